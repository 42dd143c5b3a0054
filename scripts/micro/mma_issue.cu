// Microbenchmark: how long does issuing n tcgen05.mma (SS 128x128x16) into an idle pipe block
// the issuing thread, and when does the commit barrier fire?
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

__global__ void __launch_bounds__(128, 1) issue_bench(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
  if (warp == 1 && lane == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    int k = 0;
    for (int n : {1, 2, 4, 8, 16, 32}) {
      for (int rep = 0; rep < 2; ++rep) {
        unsigned long long t0 = clock64();
        for (int i = 0; i < n; ++i) {
          const uint32_t off = ((i & 7) >> 2) * 16384 + (i & 3) * 32;
          umma_bf16_ss(tmem, sdesc_kmajor_sw128(a + off), sdesc_kmajor_sw128(b + off), idesc, i > 0);
        }
        unsigned long long t1 = clock64();
        umma_commit(&bar);
        mbar_wait(&bar, k & 1);
        ++k;
        unsigned long long t2 = clock64();
        if (rep == 1) { out[2 * (n == 1 ? 0 : n == 2 ? 1 : n == 4 ? 2 : n == 8 ? 3 : n == 16 ? 4 : 5)] = t1 - t0;
                        out[2 * (n == 1 ? 0 : n == 2 ? 1 : n == 4 ? 2 : n == 8 ? 3 : n == 16 ? 4 : 5) + 1] = t2 - t0; }
      }
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 12);
  cudaFuncSetAttribute(issue_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  issue_bench<<<1, 128, 65536>>>(d);
  cudaDeviceSynchronize();
  unsigned long long h[12]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  int ns[6] = {1, 2, 4, 8, 16, 32};
  for (int i = 0; i < 6; ++i) printf("n=%2d MMAs: issue returns after %5llu cycles, commit fires after %5llu (ideal exec %d)\n", ns[i], h[2*i], h[2*i+1], 64 * ns[i]);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
