// How fast can 1, 2 or 4 warps per SM sub-partition turn 64 scores per thread into bf16
// P (+ row sum)? The attention softmax's exponential phase in isolation, with P stored
// to TMEM like the kernel does (tcgen05.st x16), for each MUFU/polynomial split.
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

template <int EMU>
__device__ __forceinline__ float exp64(const float (&s)[64], float2 sc2, float2 nm2, uint32_t t_p) {
  float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int k = c * 32 + 2 * e;
      const float2 x = ffma2(make_float2(s[k], s[k + 1]), sc2, nm2);
      float2 pe;
      if ((e * (EMU / 2)) % 16 < EMU / 2) {
        pe = ex2_poly2(x);
      } else {
        pe.x = ex2_approx(x.x);
        pe.y = ex2_approx(x.y);
      }
      if (e & 1) sb = fadd2(sb, pe); else sa = fadd2(sa, pe);
      pk[e] = pack_bf16x2(pe.x, pe.y);
    }
    tmem_st_32x32b_x16(t_p + c * 16, pk);
  }
  const float2 sum = fadd2(sa, sb);
  return sum.x + sum.y;
}


// Same work at EMU = 16, written so each step pairs one MUFU pair with one polynomial pair
// (independent chains side by side) to see whether ptxas then overlaps the two pipes.
__device__ __forceinline__ float exp64_interleaved(const float (&s)[64], float2 sc2, float2 nm2, uint32_t t_p) {
  float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
      const int k = c * 32 + 2 * e;
      const float2 xm = ffma2(make_float2(s[k], s[k + 1]), sc2, nm2);
      const float2 xp = ffma2(make_float2(s[k + 2], s[k + 3]), sc2, nm2);
      float2 pm;
      pm.x = ex2_approx(xm.x);
      const float2 pp = ex2_poly2(xp);
      pm.y = ex2_approx(xm.y);
      sa = fadd2(sa, pm);
      sb = fadd2(sb, pp);
      pk[e] = pack_bf16x2(pm.x, pm.y);
      pk[e + 1] = pack_bf16x2(pp.x, pp.y);
    }
    tmem_st_32x32b_x16(t_p + c * 16, pk);
  }
  const float2 sum = fadd2(sa, sb);
  return sum.x + sum.y;
}


// Packed-half MUFU: x (fp32 pair) -> f16x2 -> ex2.approx.f16x2 (one MUFU op for two
// exponentials) -> fp32 pair for the row sum -> bf16x2 for P.
__device__ __forceinline__ float2 ex2_h2(float2 x) {
  uint32_t h, r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x.y), "f"(x.x));
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(h));
  float2 out;
  asm("{.reg .f16 lo, hi;\n mov.b32 {lo, hi}, %2;\n cvt.f32.f16 %0, lo;\n cvt.f32.f16 %1, hi;}"
      : "=f"(out.x), "=f"(out.y) : "r"(r));
  return out;
}

__device__ __forceinline__ float exp64_h2(const float (&s)[64], float2 sc2, float2 nm2, uint32_t t_p) {
  float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int k = c * 32 + 2 * e;
      const float2 x = ffma2(make_float2(s[k], s[k + 1]), sc2, nm2);
      const float2 pe = ex2_h2(x);
      if (e & 1) sb = fadd2(sb, pe); else sa = fadd2(sa, pe);
      pk[e] = pack_bf16x2(pe.x, pe.y);
    }
    tmem_st_32x32b_x16(t_p + c * 16, pk);
  }
  const float2 sum = fadd2(sa, sb);
  return sum.x + sum.y;
}

template <int EMU>
__global__ void __launch_bounds__(512, 1) exp_bench(int iters, int nwarps, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  float s[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) s[i] = -0.01f * ((threadIdx.x * 7 + i * 13) % 97);
  float acc = 0.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  if (warp < (uint32_t)nwarps) {
    const uint32_t t_p = tmem + (((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    for (int it = 0; it < iters; ++it) {
      if (EMU == 98)
        acc += exp64_h2(s, make_float2(0.18f, 0.18f), make_float2(-acc * 1e-30f, -0.5f), t_p);
      else if (EMU == 99)
        acc += exp64_interleaved(s, make_float2(0.18f, 0.18f), make_float2(-acc * 1e-30f, -0.5f), t_p);
      else
        acc += exp64<EMU>(s, make_float2(0.18f, 0.18f), make_float2(-acc * 1e-30f, -0.5f), t_p);
      tmem_wait_st();
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * 512 + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int EMU>
void run(unsigned long long* d, float* sink) {
  const int iters = 1000;
  for (int nw : {4, 8, 16}) {
    exp_bench<EMU><<<148, 512>>>(iters, nw, d, sink);
    exp_bench<EMU><<<148, 512>>>(iters, nw, d, sink);
    cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("EMU=%2d warps/SMSP=%d: %.0f cycles per 64-score step per warp-group-turn (MUFU bound %d)  %s\n", EMU, nw / 4,
           double(h) / iters, (nw / 4) * (EMU == 98 ? 32 : (64 - 64 * (EMU == 99 ? 16 : EMU) / 32)) * 8, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  unsigned long long* d; float* sink;
  cudaMalloc(&d, 8 * 148); cudaMalloc(&sink, 4 * 512 * 148);
  run<0>(d, sink); run<8>(d, sink); run<12>(d, sink); run<16>(d, sink); run<98>(d, sink);
}
