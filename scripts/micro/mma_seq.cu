// Replays the attention MMA issue sequence (per tile group: PV h0 x4, PV h1 x4, QK x8)
// with optional pieces, to find what slows the tensor pipe below 64 cycles/MMA.
//   flags bit0: commits after groups (s_full, k_empty, v_empty)
//   flags bit1: two issuing warps passing a token (tile 0 / tile 1)
//   flags bit2: mbarrier wait on an already-completed barrier before each half
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

__global__ void __launch_bounds__(128, 1) seq_bench(int iters, int flags, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bars[8];
  __shared__ uint64_t tok[2];
  __shared__ uint64_t done_bar;
  const uint32_t warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    mbar_init(&tok[0], 1); mbar_init(&tok[1], 1); mbar_init(&done_bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  // a pre-completed barrier to "wait" on
  if (threadIdx.x == 0) mbar_arrive(&bars[7]);
  __syncthreads();
  constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
  const bool two = flags & 2;
  const int my_tile = warp - 1;  // warps 1, 2
  unsigned long long t0 = clock64();
  if (warp == 1 || (two && warp == 2)) {
    const uint64_t qd0 = sdesc_kmajor_sw128(smem_u32(smem)), qd1 = sdesc_kmajor_sw128(smem_u32(smem + 32768));
    const uint64_t kd = sdesc_kmajor_sw128(smem_u32(smem + 65536)), vd = sdesc_kmajor_sw128(smem_u32(smem + 98304));
    uint32_t grp = 0;
    for (int it = 0; it < iters; ++it) {
      for (int i = 0; i < 2; ++i) {
        if (two && i != my_tile) continue;
        if (two) {
          if (i == 0) { if (grp > 0) mbar_wait(&tok[0], (grp - 1) & 1); }
          else mbar_wait(&tok[1], grp & 1);
        }
        const uint32_t ts = tmem + i * 128, to = tmem + 256 + i * 128;
        for (int h = 0; h < 2; ++h) {
          if (flags & 4) { mbar_wait(&bars[7], 0); tc_fence_after(); }
          if (elect_one()) {
#pragma unroll
            for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
              umma_bf16_ts(to, ts + kk * 8, vd + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), idesc, 1);
            if (h == 1 && (flags & 1)) umma_commit(&bars[2 + i]);
          }
          __syncwarp();
        }
        if (elect_one()) {
          const uint64_t qd = i ? qd1 : qd0;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ss(ts, qd + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4), kd + (((kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                         idesc, kk > 0);
          if (flags & 1) { umma_commit(&bars[i]); umma_commit(&bars[4 + i]); }
          if (two) mbar_arrive(&tok[1 - i]);
        }
        __syncwarp();
        ++grp;
      }
    }
    if (warp == 1) {
      if (elect_one()) umma_commit(&done_bar);
      __syncwarp();
      mbar_wait(&done_bar, 0);
      if (elect_one()) out[blockIdx.x] = clock64() - t0;
      __syncwarp();
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 8 * 148);
  const int smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(seq_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 1000;
  for (int flags : {0, 1, 4, 5, 2, 3, 7}) {
    seq_bench<<<148, 128, smem>>>(iters, flags, d);
    seq_bench<<<148, 128, smem>>>(iters, flags, d);
    cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("flags=%d (commits=%d two_issuers=%d waits=%d): %.1f cycles/MMA (%s)\n", flags, flags & 1, (flags >> 1) & 1,
           (flags >> 2) & 1, double(h) / (iters * 32.0), cudaGetErrorString(cudaGetLastError()));
  }
}
