// K3, first fusion snapshot: attention with the probabilities P as an internal
// buffered edge.
//
// Snapshot 0 of fuse(lower(examples::attention())) (internal_buffered_edges = 1):
//
//   forall m:
//     for n:  for d: t2 += dot(Q[m][d], K[n][d])
//             t6 = exp(t2 / sqrt(total(D)));  store T1[n] = t6;  t1 += row_sum(t6)
//     t8 = recip(t1)
//     forall l:  for n: t9 += dot(load T1[n], Vt[l][n])
//                O[m][l] = row_scale(t9, t8)
//
// T1 (one query block's exponentials over every key) leaves the chip, so the plan is
// two launches over (head, 128-query) tiles, with P in an HBM workspace between them:
//
//   attn_scores_kernel  S_j = Q K_j^T on tcgen05 (double-buffered in TMEM), then the
//                       softmax warps write P_j = exp2(S_j c - b) as bf16 (TMA store) and
//                       accumulate l = sum P. The base b is the running row maximum with the
//                       lazy rebase of the fused kernel (attention.cu): b moves only when
//                       the maximum grows by more than 2^8, and then l is rebased at once
//                       and the blocks already written carry their old base, recorded per
//                       (row, block); at the end of the tile those blocks are rescaled in
//                       place to the final base (significand/exponent pairs of
//                       safe_numerics.hpp:147-175, resolved before the second map reads T1).
//                       Writes 1/l per row.
//   attn_pv_kernel      O = row_scale(P Vt^T, 1/l): a persistent tcgen05 GEMM per head
//                       (M = 128 queries, N = Dv, K = keys), TMA-fed, double-buffered
//                       accumulators.
//
// Fusing the two maps (the final snapshot, attention.cu) removes the P round trip:
// 2 * BH * Sq * Skv bytes each way (2.1 GB at C2). bench.py --schedule two_phase ranks them.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "common.hpp"
#include "plan.hpp"
#include "sm100.cuh"
#include "tma_host.hpp"

namespace bfgpu {
namespace attn2 {

constexpr int BQ = 128;   // query rows per tile
constexpr int BKV = 128;  // keys per block
constexpr int NUM_THREADS = 256;
constexpr int EPI_THREADS = 128;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 units, as attention.cu

// ------------------------------------------------------------------ scores -> P
template <int D>
struct ScoreCfg {
  static constexpr int Q_BYTES = (D / 64) * BQ * 128;
  static constexpr int K_BYTES = (D / 64) * BKV * 128;
  static constexpr int KS = 4;
  static constexpr int P_BYTES = 2 * BQ * 128;  // two 64-key boxes of bf16
  static constexpr int SMEM = Q_BYTES + KS * K_BYTES + P_BYTES + 256;
  static_assert(SMEM <= 232448, "scores kernel SMEM budget");
  static constexpr uint32_t IDESC = dev::idesc_bf16_f32(128, BKV);
};

struct ScoreParams {
  int Sq, Skv, nblk, nqt, ntiles;
  float scale_log2;
  __nv_bfloat16* P;  // [BH, Sq, Skv] workspace (T1 of the program)
  float* base_hist;  // [BH * nqt * BQ][nblk]: base of each written block, per row
  float* rinv;       // [BH * Sq]: 1 / sum_j P
};

template <int D>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    attn_scores_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_p, const ScoreParams p) {
  using namespace dev;
  using C = ScoreCfg<D>;
  constexpr int KS = C::KS;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + C::Q_BYTES;
  uint8_t* sP = sK + KS * C::K_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + C::P_BYTES);
  uint64_t* q_full = bars;
  uint64_t* q_empty = q_full + 1;
  uint64_t* k_full = q_empty + 1;   // [KS]
  uint64_t* k_empty = k_full + KS;  // [KS]
  uint64_t* s_full = k_empty + KS;  // [2]
  uint64_t* s_empty = s_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + 2);
  int* fix_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_p);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], EPI_THREADS);
    }
    *fix_flag = 0;
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, qphase = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const int bh = t / p.nqt, q0 = (t % p.nqt) * BQ;
        mbar_wait(q_empty, qphase ^ 1);
        qphase ^= 1;
        mbar_arrive_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
        for (int b = 0; b < D / 64; ++b) tma_load_3d(&tm_q, q_full, sQ + b * BQ * 128, b * 64, q0, bh);
        for (int j = 0; j < p.nblk; ++j) {
          mbar_wait(&k_empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&k_full[stage], C::K_BYTES);
#pragma unroll
          for (int b = 0; b < D / 64; ++b)
            tma_load_3d(&tm_k, &k_full[stage], sK + stage * C::K_BYTES + b * BKV * 128, b * 64, j * BKV, bh);
          if (++stage == KS) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    int stage = 0;
    uint32_t phase = 0, qphase = 0;
    uint32_t sb = 0, sphase = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      mbar_wait(q_full, qphase);
      qphase ^= 1;
      for (int j = 0; j < p.nblk; ++j) {
        mbar_wait(&s_empty[sb], sphase ^ 1);
        mbar_wait(&k_full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK + stage * C::K_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk / 4) * (BQ * 128) + (kk % 4) * 32;
            umma_bf16_ss(tmem_base + sb * BKV, sdesc_kmajor_sw128(qa + off), sdesc_kmajor_sw128(ka + off), C::IDESC,
                         kk != 0);
          }
          umma_commit(&k_empty[stage]);
          umma_commit(&s_full[sb]);
          if (j == p.nblk - 1) umma_commit(q_empty);
        }
        __syncwarp();
        if (++stage == KS) {
          stage = 0;
          phase ^= 1;
        }
        sb ^= 1;
        if (sb == 0) sphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------- softmax: one row per thread
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;
    const uint32_t etid = threadIdx.x - 4 * 32;
    const bool store_leader = etid == 0;
    const uint32_t p_addr = smem_u32(sP);
    uint32_t sb = 0, sphase = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const int bh = t / p.nqt, q0 = (t % p.nqt) * BQ;
      float base = -INFINITY, l = 0.f;
      bool stale = false;  // some written block of this row carries an older base
      float* hist = p.base_hist + (static_cast<size_t>(t) * BQ + row) * p.nblk;  // this thread's row
      for (int j = 0; j < p.nblk; ++j) {
        const int valid = min(BKV, p.Skv - j * BKV);  // keys of this block inside Skv
        mbar_wait(&s_full[sb], sphase);
        tc_fence_after();
        uint32_t v[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + sb * BKV + c * 32, v[c]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&s_empty[sb]);
        sb ^= 1;
        if (sb == 0) sphase ^= 1;
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i < valid) mx = fmaxf(mx, __uint_as_float(v[c][i]));
        mx *= p.scale_log2;
        if (mx > base + RESCALE_THRESHOLD || base == -INFINITY) {
          if (base != -INFINITY) {
            l *= ex2_approx(base - mx);
            stale = true;
          }
          base = mx;
        }
        hist[j] = base;
        // the staging box is free once the previous block's TMA store has read it
        if (store_leader) bulk_wait_read0();
        named_bar_sync(1, EPI_THREADS);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int k0 = c * 32 + 2 * i;
            const float e0 = k0 < valid ? ex2_approx(fmaf(__uint_as_float(v[c][2 * i]), p.scale_log2, -base)) : 0.f;
            const float e1 =
                k0 + 1 < valid ? ex2_approx(fmaf(__uint_as_float(v[c][2 * i + 1]), p.scale_log2, -base)) : 0.f;
            l += e0 + e1;
            pk[i] = pack_bf16x2(e0, e1);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int chunk = c * 4 + u;  // 16-byte chunk of the 128 keys
            st_shared_v4(p_addr + (chunk >> 3) * (BQ * 128) + sw128_offset(row, chunk & 7), pk[4 * u],
                         pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, EPI_THREADS);
        if (store_leader) {
          tma_store_3d(&tm_p, sP, j * BKV, q0, bh);
          tma_store_3d(&tm_p, sP + BQ * 128, j * BKV + 64, q0, bh);
          bulk_commit();
        }
      }
      // blocks written under an older base: rescale them in place to the final one
      if (stale) atomicOr(fix_flag, 1);
      named_bar_sync(1, EPI_THREADS);
      const bool any = *reinterpret_cast<volatile int*>(fix_flag) != 0;
      if (any) {
        if (store_leader) {
          bulk_wait0();
          fence_proxy_async_global();
        }
        named_bar_sync(1, EPI_THREADS);
        if (stale && q0 + static_cast<int>(row) < p.Sq) {
          uint4* prow = reinterpret_cast<uint4*>(p.P + (static_cast<size_t>(bh) * p.Sq + q0 + row) * p.Skv);
          for (int j = 0; j < p.nblk; ++j) {
            const float bj = hist[j];
            if (bj == base) continue;
            const float f = ex2_approx(bj - base);
            for (int k = j * BKV / 8; k < min(p.Skv, (j + 1) * BKV) / 8; ++k) {
              uint4 w = __ldcg(prow + k);
              uint32_t* e = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
              for (int u = 0; u < 4; ++u)
                e[u] = pack_bf16x2(__uint_as_float(e[u] << 16) * f, __uint_as_float(e[u] & 0xffff0000u) * f);
              prow[k] = w;
            }
          }
        }
        named_bar_sync(1, EPI_THREADS);
        if (store_leader) *fix_flag = 0;
      }
      if (q0 + static_cast<int>(row) < p.Sq) p.rinv[static_cast<size_t>(bh) * p.Sq + q0 + row] = 1.0f / l;
    }
    if (store_leader) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<256>(tmem_base);
  }
}

// ------------------------------------------------------------------ O = row_scale(P Vt^T, 1/l)
template <int DV>
struct PvCfg {
  static constexpr int BK = 64;
  static constexpr int A_BYTES = BQ * BK * 2;
  static constexpr int B_BYTES = DV * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = DV == 128 ? 6 : 8;
  static constexpr int OUT_BYTES = (DV / 64) * BQ * 128;
  static constexpr int SMEM = STAGES * STAGE_BYTES + OUT_BYTES + 256;
  static_assert(SMEM <= 232448, "P.V kernel SMEM budget");
  static constexpr uint32_t IDESC = dev::idesc_bf16_f32(128, DV);
};

struct PvParams {
  int Sq, Skv, kt, nqt, ntiles;
  const float* rinv;
};

template <int DV>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    attn_pv_kernel(const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ CUtensorMap tm_o, const PvParams p) {
  using namespace dev;
  using C = PvCfg<DV>;
  constexpr int STAGES = C::STAGES, BK = C::BK;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint8_t* stage_base = smem;
  uint8_t* out_stage = smem + STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(out_stage + C::OUT_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_p);
    tma_prefetch_desc(&tm_v);
    tma_prefetch_desc(&tm_o);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_THREADS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<2 * DV>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const int bh = t / p.nqt, q0 = (t % p.nqt) * BQ;
        for (int k = 0; k < p.kt; ++k) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = stage_base + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_3d(&tm_p, &full[stage], sa, k * BK, q0, bh);
          tma_load_3d(&tm_v, &full[stage], sa + C::A_BYTES, k * BK, 0, bh);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0, acc = 0, aphase = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      mbar_wait(&tempty[acc], aphase ^ 1);
      tc_fence_after();
      for (int k = 0; k < p.kt; ++k) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a = smem_u32(stage_base + stage * C::STAGE_BYTES), b = a + C::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            umma_bf16_ss(tmem_base + acc * DV, sdesc_kmajor_sw128(a + kk * 32), sdesc_kmajor_sw128(b + kk * 32),
                         C::IDESC, (k | kk) != 0);
          umma_commit(&empty[stage]);
          if (k == p.kt - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;
    const uint32_t etid = threadIdx.x - 4 * 32;
    const bool store_leader = etid == 0;
    const uint32_t out_addr = smem_u32(out_stage);
    uint32_t acc = 0, aphase = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const int bh = t / p.nqt, q0 = (t % p.nqt) * BQ;
      const int grow = q0 + static_cast<int>(row);
      const float r = grow < p.Sq ? __ldg(p.rinv + static_cast<size_t>(bh) * p.Sq + grow) : 0.f;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      if (store_leader) bulk_wait_read0();
      named_bar_sync(1, EPI_THREADS);
#pragma unroll 1
      for (int j = 0; j < DV / 32; ++j) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + ((q * 32) << 16) + acc * DV + j * 32, v);
        tmem_wait_ld();
        uint32_t ov[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) ov[i] = pack_bf16x2(__uint_as_float(v[2 * i]) * r, __uint_as_float(v[2 * i + 1]) * r);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int chunk = j * 4 + c;
          st_shared_v4(out_addr + (chunk >> 3) * (BQ * 128) + sw128_offset(row, chunk & 7), ov[4 * c], ov[4 * c + 1],
                       ov[4 * c + 2], ov[4 * c + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      fence_proxy_async_smem();
      named_bar_sync(1, EPI_THREADS);
      if (store_leader) {
#pragma unroll
        for (int b = 0; b < DV / 64; ++b) tma_store_3d(&tm_o, out_stage + b * BQ * 128, b * 64, q0, bh);
        bulk_commit();
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (store_leader) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<2 * DV>(tmem_base);
  }
}

// ------------------------------------------------------------------ host side

struct Ws {
  size_t p_bytes, hist_bytes, rinv_bytes;
};

Ws layout(int64_t BH, int64_t Sq, int64_t Skv) {
  const int64_t nqt = (Sq + BQ - 1) / BQ, nblk = (Skv + BKV - 1) / BKV;
  return Ws{align_up(static_cast<size_t>(BH * Sq * Skv) * 2, 1024),
            align_up(static_cast<size_t>(BH * nqt * BQ * nblk) * 4, 256), align_up(static_cast<size_t>(BH * Sq) * 4, 256)};
}

template <int D, int DV>
void launch(const Plan& pl, const void* Q, const void* K, const void* Vt, void* O, float scale, void* ws,
            cudaStream_t stream) {
  const int64_t BH = pl.dims[0], Sq = pl.dims[1], Skv = pl.dims[2];
  const Ws w = layout(BH, Sq, Skv);
  uint8_t* wb = static_cast<uint8_t*>(ws);
  auto* P = reinterpret_cast<__nv_bfloat16*>(wb);
  float* hist = reinterpret_cast<float*>(wb + w.p_bytes);
  float* rinv = reinterpret_cast<float*>(wb + w.p_bytes + w.hist_bytes);
  const int nqt = static_cast<int>((Sq + BQ - 1) / BQ);
  const int ntiles = static_cast<int>(BH) * nqt;
  const int grid = std::min(ntiles, pl.dev.sms);

  ScoreParams sp{};
  sp.Sq = static_cast<int>(Sq);
  sp.Skv = static_cast<int>(Skv);
  sp.nblk = static_cast<int>((Skv + BKV - 1) / BKV);
  sp.nqt = nqt;
  sp.ntiles = ntiles;
  sp.scale_log2 = scale * 1.4426950408889634f;
  sp.P = P;
  sp.base_hist = hist;
  sp.rinv = rinv;
  const CUtensorMap tm_q = make_tmap_bf16_3d(Q, BH, Sq, D, 64, BQ);
  const CUtensorMap tm_k = make_tmap_bf16_3d(K, BH, Skv, D, 64, BKV);
  const CUtensorMap tm_pst = make_tmap_bf16_3d(P, BH, Sq, Skv, 64, BQ);
  ensure_smem_attr(reinterpret_cast<const void*>(&attn_scores_kernel<D>), ScoreCfg<D>::SMEM);
  attn_scores_kernel<D><<<grid, NUM_THREADS, ScoreCfg<D>::SMEM, stream>>>(tm_q, tm_k, tm_pst, sp);
  BF_CUDA(cudaGetLastError());
  note_launch();

  PvParams vp{};
  vp.Sq = static_cast<int>(Sq);
  vp.Skv = static_cast<int>(Skv);
  vp.kt = static_cast<int>((Skv + PvCfg<DV>::BK - 1) / PvCfg<DV>::BK);
  vp.nqt = nqt;
  vp.ntiles = ntiles;
  vp.rinv = rinv;
  const CUtensorMap tm_pld = make_tmap_bf16_3d(P, BH, Sq, Skv, 64, BQ);
  const CUtensorMap tm_v = make_tmap_bf16_3d(Vt, BH, DV, Skv, 64, DV);
  const CUtensorMap tm_o = make_tmap_bf16_3d(O, BH, Sq, DV, 64, BQ);
  ensure_smem_attr(reinterpret_cast<const void*>(&attn_pv_kernel<DV>), PvCfg<DV>::SMEM);
  attn_pv_kernel<DV><<<grid, NUM_THREADS, PvCfg<DV>::SMEM, stream>>>(tm_pld, tm_v, tm_o, vp);
  BF_CUDA(cudaGetLastError());
  note_launch();
}

}  // namespace attn2

size_t attention_staged_workspace_bytes(int64_t BH, int64_t Sq, int64_t Skv) {
  const attn2::Ws w = attn2::layout(BH, Sq, Skv);
  return w.p_bytes + w.hist_bytes + w.rinv_bytes;
}

KernelSpec attn_staged_spec(int D, int Dv) {
  KernelSpec k;
  k.name = "attn_scores_kernel + attn_pv_kernel";
  k.func = D == 128 ? reinterpret_cast<const void*>(&attn2::attn_scores_kernel<128>)
                    : reinterpret_cast<const void*>(&attn2::attn_scores_kernel<64>);
  k.threads = attn2::NUM_THREADS;
  k.smem_bytes = D == 128 ? attn2::ScoreCfg<128>::SMEM : attn2::ScoreCfg<64>::SMEM;
  k.tmem_cols = 256;
  k.cluster = 1;
  k.tile_m = attn2::BQ;
  k.tile_n = attn2::BKV;
  k.tile_k = D;
  k.stages = attn2::ScoreCfg<128>::KS;
  k.grid_sync = false;
  (void)Dv;
  return k;
}

// bf16 snapshot-0 entry (bf_attention_sched with BF_SCHED_STAGED).
void attention_staged_bf16(const Plan& pl, const void* Q, const void* K, const void* Vt, void* O, float scale,
                           void* ws, size_t ws_bytes, cudaStream_t stream) {
  const int64_t BH = pl.dims[0], Sq = pl.dims[1], Skv = pl.dims[2], D = pl.dims[3], Dv = pl.dims[4];
  BF_CHECK_ARG(ws != nullptr && ws_bytes >= attention_staged_workspace_bytes(BH, Sq, Skv),
               "bf_attention: workspace too small for the staged schedule");
  BF_CHECK_ARG((reinterpret_cast<uintptr_t>(ws) & 15u) == 0, "bf_attention: workspace must be 16-byte aligned");
  if (D == 128 && Dv == 128)
    attn2::launch<128, 128>(pl, Q, K, Vt, O, scale, ws, stream);
  else if (D == 128 && Dv == 64)
    attn2::launch<128, 64>(pl, Q, K, Vt, O, scale, ws, stream);
  else if (D == 64 && Dv == 128)
    attn2::launch<64, 128>(pl, Q, K, Vt, O, scale, ws, stream);
  else
    attn2::launch<64, 64>(pl, Q, K, Vt, O, scale, ws, stream);
}

}  // namespace bfgpu
