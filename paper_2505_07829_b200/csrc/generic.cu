// Generic block-program execution on the GPU: one float64
// SIMT kernel per operator kind of the reference IR, so that any block program that
// the fused kernels do not cover (recognizer misses, unfused lower() output, partial
// fusions) still runs entirely on the device. The host-side graph walk that drives
// these kernels is host/bfgpu_generic.cpp; it mirrors detail::eval_graph/eval_map
// (interpreter.hpp:319-472) with device-resident values.
//
// Semantics follow detail::eval_func (interpreter.hpp:263-299) in float64:
//   add, mul         elementwise on blocks, vectors or scalars          (:265-273)
//   row_shift/scale  m(i, j) + c(i) / m(i, j) * c(i)                    (:274-287)
//   row_sum          sum over columns                                   (:288)
//   dot              a * b^T                                            (:289-294)
//   outer            u * v^T                                            (:295)
//   elementwise      ScalarExpr tree, compiled to a postfix program     (:241-252, scalar_expr.hpp:66-87)
// These are correctness kernels (the fused sm_100a kernels are the performance path).
#include <cuda_runtime.h>

#include <cmath>

#include "bfgpu.h"
#include "common.hpp"

namespace bfgpu {
namespace generic {

constexpr int kMaxProg = 64;
constexpr int kMaxStack = 16;

struct ExprProgram {
  int len;
  int8_t op[kMaxProg];
  double cst[kMaxProg];
};

__global__ void binary_kernel(int op, const double* a, const double* b, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = op == BF_GX_ADD ? a[i] + b[i] : a[i] * b[i];
}

__global__ void row_op_kernel(int op, const double* m, const double* c, double* out, int64_t rows, int64_t cols) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = c[i / cols];
    out[i] = op == BF_GX_ROW_SHIFT ? m[i] + v : m[i] * v;
  }
}

// One warp per row; left-to-right partial sums per lane, then a fixed tree.
__global__ void row_sum_kernel(const double* m, double* out, int64_t rows, int64_t cols) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  double s = 0.0;
  for (int64_t j = lane; j < cols; j += 32) s += m[r * cols + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[r] = s;
}

// C[M, N] = A[M, K] * B[N, K]^T, 32x32 tiles through shared memory.
__global__ void dot_kernel(const double* A, const double* B, double* C, int64_t M, int64_t N, int64_t K) {
  __shared__ double sa[32][33], sb[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8 threads, 4 rows each
  const int64_t m0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k0 = 0; k0 < K; k0 += 32) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = ty * 4 + r;
      sa[row][tx] = (m0 + row < M && k0 + tx < K) ? A[(m0 + row) * K + k0 + tx] : 0.0;
      sb[row][tx] = (n0 + row < N && k0 + tx < K) ? B[(n0 + row) * K + k0 + tx] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double b = sb[tx][k];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] = fma(sa[ty * 4 + r][k], b, acc[r]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int64_t row = m0 + ty * 4 + r, col = n0 + tx;
    if (row < M && col < N) C[row * N + col] = acc[r];
  }
}

__global__ void outer_kernel(const double* u, const double* v, double* out, int64_t rows, int64_t cols) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = u[i / cols] * v[i % cols];
}

__global__ void elementwise_kernel(const ExprProgram prog, const double* in, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double st[kMaxStack];
    int sp = 0;
    const double x = in[i];
    for (int k = 0; k < prog.len; ++k) {
      switch (prog.op[k]) {
        case BF_GX_EXPR_VAR: st[sp++] = x; break;
        case BF_GX_EXPR_CONST: st[sp++] = prog.cst[k]; break;
        case BF_GX_EXPR_ADD: --sp; st[sp - 1] = st[sp - 1] + st[sp]; break;
        case BF_GX_EXPR_SUB: --sp; st[sp - 1] = st[sp - 1] - st[sp]; break;
        case BF_GX_EXPR_MUL: --sp; st[sp - 1] = st[sp - 1] * st[sp]; break;
        case BF_GX_EXPR_DIV: --sp; st[sp - 1] = st[sp - 1] / st[sp]; break;
        case BF_GX_EXPR_EXP: st[sp - 1] = exp(st[sp - 1]); break;
        case BF_GX_EXPR_SQRT: st[sp - 1] = sqrt(st[sp - 1]); break;
        case BF_GX_EXPR_RECIP: st[sp - 1] = 1.0 / st[sp - 1]; break;
        case BF_GX_EXPR_SQUARE: st[sp - 1] = st[sp - 1] * st[sp - 1]; break;
        case BF_GX_EXPR_SIGMOID: st[sp - 1] = 1.0 / (1.0 + exp(-st[sp - 1])); break;
        default: break;
      }
    }
    out[i] = st[0];
  }
}

inline int grid_for(int64_t n, int threads = 256) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

}  // namespace generic

extern void note_launch();

}  // namespace bfgpu

using namespace bfgpu;

extern "C" {

BF_API int bf_gx_binary(int op, const double* a, const double* b, double* out, int64_t n, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(a && b && out && n >= 0, "bf_gx_binary: bad arguments");
    BF_CHECK_ARG(op == BF_GX_ADD || op == BF_GX_MUL, "bf_gx_binary: op must be BF_GX_ADD or BF_GX_MUL");
    if (n == 0) return;
    generic::binary_kernel<<<generic::grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(op, a, b, out, n);
    BF_CUDA(cudaGetLastError());
    note_launch();
  });
}

BF_API int bf_gx_row_op(int op, const double* m, const double* c, double* out, int64_t rows, int64_t cols,
                        void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(m && c && out && rows >= 0 && cols >= 0, "bf_gx_row_op: bad arguments");
    BF_CHECK_ARG(op == BF_GX_ROW_SHIFT || op == BF_GX_ROW_SCALE, "bf_gx_row_op: op must be ROW_SHIFT or ROW_SCALE");
    if (rows * cols == 0) return;
    generic::row_op_kernel<<<generic::grid_for(rows * cols), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        op, m, c, out, rows, cols);
    BF_CUDA(cudaGetLastError());
    note_launch();
  });
}

BF_API int bf_gx_row_sum(const double* m, double* out, int64_t rows, int64_t cols, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(m && out && rows >= 0 && cols >= 0, "bf_gx_row_sum: bad arguments");
    if (rows == 0) return;
    const int64_t blocks = (rows + 7) / 8;
    BF_CHECK_ARG(blocks < (1ll << 31), "bf_gx_row_sum: too many rows");
    generic::row_sum_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(m, out, rows,
                                                                                                         cols);
    BF_CUDA(cudaGetLastError());
    note_launch();
  });
}

BF_API int bf_gx_dot(const double* a, const double* b, double* out, int64_t M, int64_t N, int64_t K, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(a && b && out && M >= 0 && N >= 0 && K >= 0, "bf_gx_dot: bad arguments");
    if (M * N == 0) return;
    BF_CHECK_ARG((M + 31) / 32 < 65536, "bf_gx_dot: too many rows");
    dim3 grid(static_cast<unsigned>((N + 31) / 32), static_cast<unsigned>((M + 31) / 32));
    generic::dot_kernel<<<grid, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(a, b, out, M, N, K);
    BF_CUDA(cudaGetLastError());
    note_launch();
  });
}

BF_API int bf_gx_outer(const double* u, const double* v, double* out, int64_t rows, int64_t cols, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(u && v && out && rows >= 0 && cols >= 0, "bf_gx_outer: bad arguments");
    if (rows * cols == 0) return;
    generic::outer_kernel<<<generic::grid_for(rows * cols), 256, 0, static_cast<cudaStream_t>(stream)>>>(u, v, out,
                                                                                                         rows, cols);
    BF_CUDA(cudaGetLastError());
    note_launch();
  });
}

BF_API int bf_gx_elementwise(const int8_t* ops, const double* consts, int len, const double* in, double* out, int64_t n,
                             void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(ops && in && out && n >= 0, "bf_gx_elementwise: bad arguments");
    BF_CHECK_ARG(len > 0 && len <= generic::kMaxProg, "bf_gx_elementwise: expression too long");
    generic::ExprProgram prog{};
    prog.len = len;
    int depth = 0, max_depth = 0;
    for (int k = 0; k < len; ++k) {
      prog.op[k] = ops[k];
      prog.cst[k] = consts ? consts[k] : 0.0;
      const int o = ops[k];
      BF_CHECK_ARG(o >= BF_GX_EXPR_VAR && o <= BF_GX_EXPR_SIGMOID, "bf_gx_elementwise: unknown opcode");
      if (o == BF_GX_EXPR_VAR || o == BF_GX_EXPR_CONST)
        ++depth;
      else if (o >= BF_GX_EXPR_ADD && o <= BF_GX_EXPR_DIV)
        --depth;
      BF_CHECK_ARG(depth >= 1, "bf_gx_elementwise: malformed postfix program");
      max_depth = depth > max_depth ? depth : max_depth;
    }
    BF_CHECK_ARG(depth == 1 && max_depth <= generic::kMaxStack, "bf_gx_elementwise: malformed postfix program");
    if (n == 0) return;
    generic::elementwise_kernel<<<generic::grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(prog, in, out, n);
    BF_CUDA(cudaGetLastError());
    note_launch();
  });
}

BF_API int bf_gx_copy2d(double* dst, int64_t dst_ld, const double* src, int64_t src_ld, int64_t rows, int64_t cols,
                        void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(dst && src && rows >= 0 && cols >= 0 && dst_ld >= cols && src_ld >= cols, "bf_gx_copy2d: bad arguments");
    if (rows * cols == 0) return;
    BF_CUDA(cudaMemcpy2DAsync(dst, dst_ld * sizeof(double), src, src_ld * sizeof(double), cols * sizeof(double), rows,
                              cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  });
}

BF_API int bf_gx_zero(double* out, int64_t n, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(out && n >= 0, "bf_gx_zero: bad arguments");
    if (n == 0) return;
    BF_CUDA(cudaMemsetAsync(out, 0, n * sizeof(double), static_cast<cudaStream_t>(stream)));
  });
}

}  // extern "C"
