// FP32 FMA peak of the device, the roofline denominator of the fp32 mode (C1).
// Scalar FFMA and packed FFMA2 (fma.rn.f32x2, sm_100), 16 independent chains per thread,
// 4 warps per SM sub-partition; best of 5, CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma_peak ffma_peak.cu
#include <cstdio>

constexpr int CHAINS = 16;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(512) ffma_scalar(float* out, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(acc[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
  asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(d) : "l"(a), "l"(b));
}

__global__ void __launch_bounds__(512) ffma_packed(float* out, float a, float b) {
  unsigned long long acc[CHAINS / 2];
  const unsigned long long aa = (static_cast<unsigned long long>(__float_as_uint(a)) << 32) | __float_as_uint(a);
  const unsigned long long bb = (static_cast<unsigned long long>(__float_as_uint(b)) << 32) | __float_as_uint(b);
#pragma unroll
  for (int i = 0; i < CHAINS / 2; ++i) acc[i] = (static_cast<unsigned long long>(threadIdx.x) << 32) | i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS / 2; ++i) ffma2(acc[i], aa, bb);
  }
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS / 2; ++i) s ^= acc[i];
  if (s == 12345ull) out[threadIdx.x] = 1.f;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kind = 0; kind < 2; ++kind) {
    for (int threads : {256, 512}) {
      const int blocks = sms * (1024 / threads) * 2;
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0)
          ffma_scalar<<<blocks, threads>>>(out, 0.999f, 1e-3f);
        else
          ffma_packed<<<blocks, threads>>>(out, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      const double flops = 2.0 * CHAINS * ITERS * static_cast<double>(blocks) * threads;
      printf("{\"kind\": \"%s\", \"threads\": %d, \"blocks\": %d, \"ms\": %.4f, \"tflops\": %.2f}\n",
             kind == 0 ? "ffma" : "ffma2", threads, blocks, best, flops / best / 1e9);
    }
  }
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  return 0;
}
