// K2: Flash-LayerNorm + MatMul on sm_100a.
//
// Block program (final snapshot of fuse(lower(examples::layernorm_matmul())),
// reference lowering.hpp:573-581; listing in SURVEY.md §2.1):
//
//   forall m: forall n: for k:  t1 += row_sum(X[m][k]);  t2 += row_sum(square(X[m][k]))
//                               t3 += dot(X[m][k], Yt[n][k]);  t4 += row_sum(Yt[n][k])
//       mu_neg = 0 - t1/total(K);  rstd = recip(sqrt(t2/total(K) + (0 - square(t1/total(K)))))
//       O[m][n] = row_scale(add(t3, outer(mu_neg, t4)), rstd)
//
// Rules R4/R5 moved the shift and scale past the dot, so the contraction runs
// on RAW X. B200 mapping: persistent warp-specialized kernel, 128x256 output
// tiles, one M=128,N=256 tcgen05 MMA per K=16 step into double-buffered TMEM.
//   - t1, t2 (per row): statistics warps read the X tiles the TMA already
//     staged in SMEM for the MMA (no extra HBM bytes).
//   - t4 = colsum(Yt) is a property of Yt alone, identical for every m: the
//     epilogue warps, idle until the first accumulator is ready, compute a
//     1/gridDim slice of it from global memory into the workspace during the
//     first mainloop and publish it with a grid-wide release counter.
//   - epilogue: O = (acc + mu_neg * t4) * rstd -> bf16 -> TMA store.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w3 idle, w4-7 epilogue, w8-11 row statistics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "sm100.cuh"
#include "plan.hpp"
#include "tma_host.hpp"

namespace bfgpu {
namespace lnmm {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int BN = 256;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int OUT_BYTES = BM * 128 * 2;
constexpr int NUM_THREADS = 384;
constexpr int EPI_THREADS = 128;
constexpr int STATS_THREADS = 128;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t IDESC = dev::idesc_bf16_f32(128, 256);
// Dynamic SMEM is declared __align__(1024) (no static SMEM, so the window starts aligned):
// 4 x 48 KB stages + 32 KB staging + mu/rstd + barriers = 230,528 B of the 232,448 B limit.
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + OUT_BYTES + 2 * 2 * BM * 4 /*mu,rstd*/ + 128 /*barriers*/;

struct Params {
  int M, K, N;
  int Mt, Nt, kt;
  int num_tiles;
  int group;  // m-tiles per scheduling group (tiles of a group share Yt slices in L2)
  float inv_k;
  float eps;
  float* colsum;  // [N] workspace
  int* ready;     // CTAs that finished their colsum slice
};

__device__ __forceinline__ void decode(const Params& p, int t, int& m, int& n) {
  // n fastest inside a group of m-tiles: concurrent CTAs share X m-tiles and Yt slices in L2.
  const int per_group = p.group * p.Nt;
  const int g = t / per_group;
  const int r = t % per_group;
  const int gs = min(p.group, p.Mt - g * p.group);
  m = g * p.group + r % gs;
  n = r / gs;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    ln_matmul_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_y,
                     const __grid_constant__ CUtensorMap tm_o, const __nv_bfloat16* __restrict__ Yt, const Params p) {
  using namespace dev;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();  // SWIZZLE_128B tiles need 1024-byte alignment
  uint8_t* stage_base = smem;
  uint8_t* out_stage = smem + STAGES * STAGE_BYTES;
  float* s_mu = reinterpret_cast<float*>(out_stage + OUT_BYTES);  // [2][BM] : -mean
  float* s_rstd = s_mu + 2 * BM;                                  // [2][BM]
  uint64_t* full = reinterpret_cast<uint64_t*>(s_rstd + 2 * BM);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + 2);

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_y);
    tma_prefetch_desc(&tm_o);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + STATS_THREADS);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_THREADS);
      mbar_init(&sfull[a], STATS_THREADS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int m, n;
        decode(p, t, m, n);
        for (int k = 0; k < p.kt; ++k) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = stage_base + stage * STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(&tm_x, &full[stage], sa, k * BK, m * BM);
          tma_load_2d(&tm_y, &full[stage], sa + A_BYTES, k * BK, n * BN);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc = 0, aphase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * 256;
      for (int k = 0; k < p.kt; ++k) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(stage_base + stage * STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16_ss(d_tmem, sdesc_kmajor_sw128(a_addr + kk * 32), sdesc_kmajor_sw128(b_addr + kk * 32), IDESC,
                         (k | kk) != 0);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  } else if (warp >= 4 && warp < 8) {
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;
    const uint32_t etid = threadIdx.x - 4 * 32;
    const bool leader = etid == 0;
    const uint32_t out_addr = smem_u32(out_stage);

    // ---- colsum(Yt) slice for this CTA: one warp per Yt row, 16-byte loads.
    {
      const int per = (p.N + gridDim.x - 1) / gridDim.x;
      const int n0 = blockIdx.x * per, n1 = min(p.N, n0 + per);
      for (int n = n0 + static_cast<int>(q); n < n1; n += 4) {
        const uint4* rowp = reinterpret_cast<const uint4*>(Yt + static_cast<size_t>(n) * p.K);
        float s = 0.f;
        for (int c = lane; c < p.K / 8; c += 32) {
          const uint4 v = __ldg(rowp + c);
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) s += __uint_as_float(w[e] << 16) + __uint_as_float(w[e] & 0xffff0000u);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) p.colsum[n] = s;
      }
      named_bar_sync(1, EPI_THREADS);
      if (leader) {
        __threadfence();
        red_release_gpu_add(p.ready, 1);
      }
    }
    bool col_ready = false;

    uint32_t acc = 0, aphase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int m, n;
      decode(p, t, m, n);
      if (!col_ready) {
        if (leader) {
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_gpu(p.ready) < static_cast<int>(gridDim.x)) {
            __nanosleep(256);
            if (globaltimer_ns() - t0 > 20000000000ull) __trap();
          }
        }
        col_ready = true;
      }
      mbar_wait(&tfull[acc], aphase);
      mbar_wait(&sfull[acc], aphase);
      tc_fence_after();
      const float mu_neg = s_mu[acc * BM + row];
      const float rstd = s_rstd[acc * BM + row];
      const uint32_t trow = tmem_base + acc * 256 + ((q * 32) << 16);
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        if (leader) bulk_wait_read0();
        named_bar_sync(1, EPI_THREADS);  // staging buffer free
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(trow + half * 128 + j * 32, v);
          tmem_wait_ld();
          // colsum(Yt) for these 32 columns: every lane reads the same addresses (L1 broadcast).
          const int c0 = n * BN + half * 128 + j * 32;
          float cs[32];
          if (c0 + 32 <= p.N) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 f = __ldcg(reinterpret_cast<const float4*>(p.colsum + c0) + i);
              cs[4 * i] = f.x;
              cs[4 * i + 1] = f.y;
              cs[4 * i + 2] = f.z;
              cs[4 * i + 3] = f.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) cs[i] = c0 + i < p.N ? __ldcg(p.colsum + c0 + i) : 0.f;
          }
          uint32_t ov[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float o0 = (__uint_as_float(v[2 * i]) + mu_neg * cs[2 * i]) * rstd;
            const float o1 = (__uint_as_float(v[2 * i + 1]) + mu_neg * cs[2 * i + 1]) * rstd;
            ov[i] = pack_bf16x2(o0, o1);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int chunk = j * 4 + c;
            st_shared_v4(out_addr + (chunk >> 3) * (BM * 128) + sw128_offset(row, chunk & 7), ov[4 * c],
                         ov[4 * c + 1], ov[4 * c + 2], ov[4 * c + 3]);
          }
        }
        if (half == 1) {
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        fence_proxy_async_smem();
        named_bar_sync(1, EPI_THREADS);
        if (leader) {
          tma_store_2d(&tm_o, out_stage, n * BN + half * 128, m * BM);
          tma_store_2d(&tm_o, out_stage + BM * 128, n * BN + half * 128 + 64, m * BM);
          bulk_commit();
        }
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (leader) bulk_wait0();
  } else if (warp >= 8) {
    const uint32_t row = (warp - 8) * 32 + lane;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc = 0, aphase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      float s1a = 0.f, s1b = 0.f, s2a = 0.f, s2b = 0.f;
      for (int k = 0; k < p.kt; ++k) {
        mbar_wait(&full[stage], phase);
        const uint32_t base = smem_u32(stage_base + stage * STAGE_BYTES) + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 v = ld_shared_v4(base + (((c + lane) & 7) << 4));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float lo = __uint_as_float(w[e] << 16);
            const float hi = __uint_as_float(w[e] & 0xffff0000u);
            s1a += lo;
            s1b += hi;
            s2a = fmaf(lo, lo, s2a);
            s2b = fmaf(hi, hi, s2b);
          }
        }
        // Shared loads must have completed before the slot is released: the mbarrier
        // arrive does not wait for outstanding LDS, so a TMA refill could overwrite
        // the stage under an in-flight load (observed as run-to-run stats drift).
        __threadfence_block();
        mbar_arrive(&empty[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      mbar_wait(&tempty[acc], aphase ^ 1);
      const float mean = (s1a + s1b) * p.inv_k;
      // var = t2/total(K) + (0 - square(t1/total(K)))  [+ eps, 0 in the reference]
      const float var = (s2a + s2b) * p.inv_k - mean * mean + p.eps;
      s_mu[acc * BM + row] = -mean;
      s_rstd[acc * BM + row] = 1.0f / sqrtf(var);
      __threadfence_block();  // publish the STS before the arrive (SYNCS does not order it)
      mbar_arrive(&sfull[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem_base);
  }
}

}  // namespace lnmm

KernelSpec lnmm1_spec() {
  using namespace lnmm;
  KernelSpec k;
  k.name = "ln_matmul_kernel";
  k.func = reinterpret_cast<const void*>(&ln_matmul_kernel);
  k.threads = NUM_THREADS;
  k.smem_bytes = SMEM_BYTES;
  k.tmem_cols = TMEM_COLS;
  k.cluster = 1;
  k.tile_m = BM;
  k.tile_n = BN;
  k.tile_k = BK;
  k.stages = STAGES;
  k.grid_sync = true;  // colsum(Yt) published with a grid-wide counter
  return k;
}

size_t lnmm2_workspace_bytes(int64_t M, int64_t N);
void lnmm_bf16_2sm(const Plan& pl, const void* X, const void* Yt, void* O, float eps, void* ws, size_t ws_bytes,
                   cudaStream_t stream);

size_t lnmm_f32x3_workspace_bytes(int64_t M, int64_t K, int64_t N);

size_t lnmm_workspace_bytes(int64_t M, int64_t K, int64_t N, int dtype) {
  if (dtype != BF_DTYPE_BF16) return lnmm_f32x3_workspace_bytes(M, K, N);  // the 3xTF32 operands
  return std::max(align_up(static_cast<size_t>(N) * 4, 256) + 256, lnmm2_workspace_bytes(M, N));
}

void lnmm_bf16(const void* X, const void* Yt, void* O, int64_t M, int64_t K, int64_t N, float eps, int schedule,
               void* ws, size_t ws_bytes, cudaStream_t stream) {
  using namespace lnmm;
  BF_CHECK_ARG(M > 0 && K > 0 && N > 0, "bf_layernorm_matmul: sizes must be positive");
  BF_CHECK_ARG(K % 8 == 0 && N % 8 == 0, "bf_layernorm_matmul: K and N must be multiples of 8");
  BF_CHECK_ARG(M < (1ll << 31) && K < (1ll << 31) && N < (1ll << 31), "bf_layernorm_matmul: dimension too large");
  BF_CHECK_ARG(ws != nullptr && ws_bytes >= lnmm_workspace_bytes(M, K, N, BF_DTYPE_BF16),
               "bf_layernorm_matmul: workspace too small");
  const Plan pl = plan_lnmm(M, K, N, BF_DTYPE_BF16, schedule);
  if (pl.spec.cluster == 2) {
    lnmm_bf16_2sm(pl, X, Yt, O, eps, ws, ws_bytes, stream);
    return;
  }
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  float* colsum = reinterpret_cast<float*>(wsb);
  int* ready = reinterpret_cast<int*>(wsb + align_up(static_cast<size_t>(N) * 4, 256));

  const CUtensorMap tm_x = make_tmap_bf16(X, M, K, K, BK, BM);
  const CUtensorMap tm_y = make_tmap_bf16(Yt, N, K, K, BK, BN);
  const CUtensorMap tm_o = make_tmap_bf16(O, M, N, N, BK, BM);

  Params p{};
  p.M = static_cast<int>(M);
  p.K = static_cast<int>(K);
  p.N = static_cast<int>(N);
  p.Mt = static_cast<int>(pl.units);
  p.Nt = static_cast<int>((N + BN - 1) / BN);
  p.kt = static_cast<int>((K + BK - 1) / BK);
  p.group = pl.group;
  p.inv_k = 1.0f / static_cast<float>(K);
  p.eps = eps;
  p.colsum = colsum;
  p.ready = ready;
  p.num_tiles = static_cast<int>(pl.tiles);
  BF_CUDA(cudaMemsetAsync(ready, 0, sizeof(int), stream));
  launch_planned(pl, ln_matmul_kernel, stream, tm_x, tm_y, tm_o, static_cast<const __nv_bfloat16*>(Yt), p);
}

}  // namespace bfgpu
