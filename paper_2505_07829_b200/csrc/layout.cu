// Layout conversion for host bindings that hand over column-major matrices.
//
// The reference's operands are Eigen matrices, stored column-major (interpreter.hpp:23-38;
// SURVEY.md §8(b)); the kernels take row-major tiles. Transposing on the host costs a
// cache-hostile pass over every element (the C++ adapter measured 70 ms in + 99 ms out at
// C3). Instead the host converts element types in storage order (a contiguous, parallel pass)
// and the device transposes: a column-major R x C matrix is a row-major C x R one, and this
// kernel writes its transpose at HBM speed.
#include <cuda_runtime.h>

#include <cstdint>

#include "bfgpu.h"
#include "common.hpp"

namespace bfgpu {

extern void note_launch();

namespace {

constexpr int TILE = 64, ROWS_PER_PASS = 16;

// dst[c, r] = src[r, c] for a rows x cols row-major src; T is the element (2 or 4 bytes).
// One 64 x 64 tile per CTA through SMEM (padded against bank conflicts), 64 x 16 threads.
template <class T>
__global__ void __launch_bounds__(TILE * ROWS_PER_PASS) transpose_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                                         int64_t rows, int64_t cols) {
  __shared__ T tile[TILE][TILE + 1];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * TILE, c0 = static_cast<int64_t>(blockIdx.x) * TILE;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int k = 0; k < TILE; k += ROWS_PER_PASS) {
    const int64_t r = r0 + ty + k, c = c0 + tx;
    if (r < rows && c < cols) tile[ty + k][tx] = src[r * cols + c];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < TILE; k += ROWS_PER_PASS) {
    const int64_t c = c0 + ty + k, r = r0 + tx;
    if (c < cols && r < rows) dst[c * rows + r] = tile[tx][ty + k];
  }
}

}  // namespace

}  // namespace bfgpu

using namespace bfgpu;

extern "C" int bf_transpose(const void* src, void* dst, int64_t rows, int64_t cols, int elem_bytes, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(src && dst && src != dst, "bf_transpose: null or aliased buffers");
    BF_CHECK_ARG(rows > 0 && cols > 0, "bf_transpose: sizes must be positive");
    BF_CHECK_ARG(elem_bytes == 2 || elem_bytes == 4 || elem_bytes == 8, "bf_transpose: element size must be 2, 4 or 8");
    BF_CHECK_ARG((cols + TILE - 1) / TILE < (1ll << 31) && (rows + TILE - 1) / TILE < 65536,
                 "bf_transpose: too large");
    const dim3 grid(static_cast<unsigned>((cols + TILE - 1) / TILE), static_cast<unsigned>((rows + TILE - 1) / TILE));
    const dim3 block(TILE, ROWS_PER_PASS);
    auto s = static_cast<cudaStream_t>(stream);
    if (elem_bytes == 2)
      transpose_kernel<uint16_t><<<grid, block, 0, s>>>(static_cast<const uint16_t*>(src), static_cast<uint16_t*>(dst),
                                                        rows, cols);
    else if (elem_bytes == 4)
      transpose_kernel<uint32_t><<<grid, block, 0, s>>>(static_cast<const uint32_t*>(src), static_cast<uint32_t*>(dst),
                                                        rows, cols);
    else
      transpose_kernel<uint64_t><<<grid, block, 0, s>>>(static_cast<const uint64_t*>(src), static_cast<uint64_t*>(dst),
                                                        rows, cols);
    BF_CUDA(cudaGetLastError());
    note_launch();
  });
}
