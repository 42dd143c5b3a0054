// Microbenchmark: tcgen05.ld (32x32b.x32) throughput per SM vs. warps, and MUFU.EX2 throughput.
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

__global__ void __launch_bounds__(256, 1) tmem_ld_bench(int iters, int nwarps, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  if (warp < (uint32_t)nwarps) {
    const uint32_t lb = ((warp & 3) * 32) << 16;
    const uint32_t colbase = (warp >> 2) * 128;
    for (int it = 0; it < iters; ++it) {
      uint32_t v[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tmem + lb + colbase + c * 32, v[c]);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= v[c][e];
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * 256 + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

__global__ void __launch_bounds__(256, 1) mufu_bench(int iters, int nwarps, unsigned long long* out, float* sink) {
  const uint32_t warp = threadIdx.x / 32;
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp < (uint32_t)nwarps) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = ex2_approx(a[i]) - 1.0f;
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  sink[blockIdx.x * 256 + threadIdx.x] = s;
}

int main() {
  unsigned long long* d_out; uint32_t* sink;
  cudaMalloc(&d_out, 8 * 148); cudaMalloc(&sink, 4 * 256 * 148);
  unsigned long long h;
  const int iters = 2000;
  for (int nw : {1, 4, 8}) {
    tmem_ld_bench<<<148, 256>>>(iters, nw, d_out, sink);
    tmem_ld_bench<<<148, 256>>>(iters, nw, d_out, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    double bytes = double(iters) * nw * 32 * 128 * 4;
    printf("tcgen05.ld x32 x4: warps=%d  cycles/iter=%.1f  bytes/clk/SM=%.1f\n", nw, double(h) / iters, bytes / double(h));
  }
  for (int nw : {4, 8}) {
    mufu_bench<<<148, 256>>>(iters, nw, d_out, (float*)sink);
    mufu_bench<<<148, 256>>>(iters, nw, d_out, (float*)sink);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
    double ops = double(iters) * nw * 32 * 16;
    printf("MUFU.EX2: warps=%d  ex2/clk/SM=%.2f\n", nw, ops / double(h));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
