// Does SS MMA throughput (M=128 N=128 K=16) depend on where A and B sit in SMEM?
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

__global__ void __launch_bounds__(128, 1) addr_bench(int iters, int aoff, int boff, int fill, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // fill: 0 = constant 1.0, 1 = pseudo-random bf16 in [-2, 2]
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
    uint32_t x = i * 2654435761u + 12345u;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    const uint32_t r = fill ? ((x & 0x807f807fu) | 0x3f003f00u) : 0x3f803f80u;
    reinterpret_cast<uint32_t*>(smem)[i] = r;
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
  if (warp == 1) {
    if (elect_one()) {
      const uint64_t ad = sdesc_kmajor_sw128(smem_u32(smem + aoff)), bd = sdesc_kmajor_sw128(smem_u32(smem + boff));
      unsigned long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ss(tmem + (it & 1) * 128, ad + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                       bd + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), idesc, kk > 0);
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  const int smem = 200 * 1024 + 1024;
  cudaFuncSetAttribute(addr_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  int cases[][2] = {{0, 32768}, {0, 65536}, {0, 98304}, {32768, 65536}, {32768, 98304}, {0, 131072}, {65536, 163840}};
  for (int fill : {0, 1})
    for (auto& c : cases) {
      addr_bench<<<148, 128, smem>>>(iters, c[0], c[1], fill, d);
      addr_bench<<<148, 128, smem>>>(iters, c[0], c[1], fill, d);
      cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("fill=%s A@%6d B@%6d: %.1f cycles/MMA  (%s)\n", fill ? "random" : "ones  ", c[0], c[1], double(h) / (iters * 8.0),
             cudaGetErrorString(cudaGetLastError()));
    }
}
