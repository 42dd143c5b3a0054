// Cost of tcgen05.commit inside a GEMM-like MMA stream: SS M=128 N=256 K=16 MMAs in
// groups of G per k-step with a commit (to a per-stage mbarrier) after each group.
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

__global__ void __launch_bounds__(128, 1) commit_bench(int iters, int per_commit, int n256, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bars[8];
  __shared__ uint64_t done_bar;
  const uint32_t warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1); mbar_init(&done_bar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = n256 ? idesc_bf16_f32(128, 256) : idesc_bf16_f32(128, 128);
  if (warp == 1) {
    if (elect_one()) {
      const uint64_t ad = sdesc_kmajor_sw128(smem_u32(smem)), bd = sdesc_kmajor_sw128(smem_u32(smem + 32768));
      unsigned long long t0 = clock64();
      int c = 0;
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16_ss(tmem, ad + kk * 2, bd + kk * 2, idesc, 1);
        if (per_commit > 0 && (it % per_commit) == per_commit - 1) umma_commit(&bars[(c++) & 7]);
      }
      umma_commit(&done_bar);
      mbar_wait(&done_bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
    __syncwarp();
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  const int smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(commit_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  for (int n256 : {1, 0})
    for (int pc : {0, 1, 2, 4}) {
      commit_bench<<<148, 128, smem>>>(iters, pc, n256, d);
      commit_bench<<<148, 128, smem>>>(iters, pc, n256, d);
      cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double ideal = n256 ? 128 : 64;
      printf("N=%d commit every %d k-steps (4 MMAs each): %.1f cycles/MMA, eff %.1f%% (%s)\n", n256 ? 256 : 128, pc,
             double(h) / (iters * 4.0), 100 * ideal / (double(h) / (iters * 4.0)), cudaGetErrorString(cudaGetLastError()));
    }
}
