// Microbenchmark: tcgen05.mma issue rate for the attention shapes.
//   SS M=128 N=128 (S = QK^T), SS M=128 N=256 (K1 shape), TS M=128 N=128 (O += PV, A in TMEM)
// optionally with 4 or 8 warps streaming tcgen05.ld from other TMEM columns (softmax traffic).
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace bfgpu::dev;

__device__ int g_mode_st = 0;
__global__ void set_mode(int v) { g_mode_st = v; }
// MODE 0: SS N=128, 1: SS N=256, 2: TS N=128, 3: attention group sequence (TS x8, commit, SS x8, commit),
//      4: SS N=64, 5: TS N=64
template <int MODE>
__global__ void __launch_bounds__(384, 1) mma_bench(int iters, int ldwarps, unsigned long long* out, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[4];
  __shared__ volatile int done;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1); fence_barrier_init(); done = 0; }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t N = MODE == 1 ? 256 : (MODE >= 4 ? 64 : 128);
  constexpr uint32_t idesc = idesc_bf16_f32(128, N);
  unsigned long long t0 = clock64();
  if (warp == 8) {
    if (lane == 0) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          if (MODE == 3) {
            umma_bf16_ts(tmem + 256 + (it & 1) * 128, tmem + (it & 1) * 128 + kk * 8, sdesc_kmajor_sw128(b + off), idesc, 1);
          } else if (MODE == 5) {
            umma_bf16_ts(tmem + 256, tmem + 128 + kk * 8, sdesc_kmajor_sw128(b + off), idesc, 1);
          } else if (MODE == 2)
            umma_bf16_ts(tmem + 256, tmem + 128 + kk * 8, sdesc_kmajor_sw128(b + off), idesc, 1);
          else
            umma_bf16_ss(tmem + (MODE == 1 ? 256 : 384), sdesc_kmajor_sw128(a + off), sdesc_kmajor_sw128(b + off), idesc, 1);
        }
        if (MODE == 3) {
          umma_commit(&bar2[it & 1]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            umma_bf16_ss(tmem + (it & 1) * 128, sdesc_kmajor_sw128(a + off), sdesc_kmajor_sw128(b + off), idesc, kk > 0);
          }
          umma_commit(&bar2[2 + (it & 1)]);
        }
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
      done = 1;
    }
  } else if (g_mode_st == 2 && warp < (uint32_t)ldwarps) {
    // spin on an mbarrier that never completes (like idle softmax/TMA warps)
    __shared__ uint64_t never;
    if (threadIdx.x == 0) mbar_init(&never, 1);
    while (!done) mbar_try_wait(smem_u32(&never), 0);
  } else if (g_mode_st == 4 && warp < (uint32_t)ldwarps) {
    // MUFU + FFMA2 stream (softmax-like ALU load)
    float2 a = make_float2(-0.001f * lane, -0.002f * lane), b = make_float2(0.5f, 0.25f);
    float acc = 0.f;
    while (!done) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        a = ffma2(a, b, make_float2(-0.01f, -0.02f));
        acc += ex2_approx(a.x) + ex2_approx(a.y);
      }
    }
    sink[blockIdx.x * 384 + threadIdx.x] = __float_as_uint(acc);
  } else if (g_mode_st == 3 && warp < (uint32_t)ldwarps) {
    // SMEM store stream into the upper 32 KB (TMA-like write traffic)
    uint32_t k = 0;
    while (!done) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        st_shared_v4(smem_u32(smem + 65536 + ((k * 8 + u) * 32 * 16 + lane * 16) % 32768), k, u, lane, 0);
      ++k;
    }
  } else if (warp < (uint32_t)ldwarps) {
    const uint32_t lb = ((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!done) {
      uint32_t v[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tmem + lb + c * 32, v[c]);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) acc ^= v[c][lane];
      if (g_mode_st) {
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = v[e & 3][e] ^ acc;
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st_32x32b_x16(tmem + lb + (warp >> 2) * 128 + c * 16, w);
        tmem_wait_st();
      }
    }
    sink[blockIdx.x * 384 + threadIdx.x] = acc;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int MODE>
void run(const char* name, int ldw, unsigned long long* d_out, uint32_t* sink) {
  const int iters = 4000;
  cudaFuncSetAttribute(mma_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024 + 1024);
  for (int r = 0; r < 2; ++r) mma_bench<MODE><<<148, 384, 96 * 1024 + 1024>>>(iters, ldw, d_out, sink);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
  const double N = MODE == 1 ? 256 : (MODE >= 4 ? 64 : 128);
  const double cyc_per_instr = double(h) / (iters * (MODE == 3 ? 16.0 : 8.0));
  printf("%-18s ldwarps=%d  cycles/MMA(K=16)=%.1f  ideal=%.0f  eff=%.0f%%   err=%s\n", name, ldw, cyc_per_instr, N / 2,
         100.0 * (N / 2) / cyc_per_instr, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d_out; uint32_t* sink;
  cudaMalloc(&d_out, 8 * 148); cudaMalloc(&sink, 4 * 384 * 148);
  for (int st : {0}) set_mode<<<1, 1>>>(st), cudaDeviceSynchronize(), printf("side load: %s\n", st == 0 ? "tcgen05.ld" : st == 2 ? "mbarrier try_wait spinners" : st == 3 ? "st.shared stream" : "MUFU+FFMA2 stream"),
  [&] { for (int ldw : {0, 8}) {
    run<0>("SS 128x128", ldw, d_out, sink);
    run<1>("SS 128x256", ldw, d_out, sink);
    run<2>("TS 128x128", ldw, d_out, sink);
    run<3>("TSx8+SSx8 groups", ldw, d_out, sink);
    run<4>("SS 128x64", ldw, d_out, sink);
    run<5>("TS 128x64", ldw, d_out, sink);
  } }();
}
