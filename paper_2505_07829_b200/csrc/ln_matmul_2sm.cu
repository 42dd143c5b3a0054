// K2 Flash-LayerNorm + MatMul, CTA-pair (cta_group::2) variant.
//
// Block program and algebra as in ln_matmul.cu: O = (X Yt^T + mu_neg (x) t4) * rstd
// with the contraction on RAW X (rules R4/R5). A cluster of two CTAs computes
// (256 H) x 256 output tiles with M=256 tcgen05 MMAs issued by the leader; each CTA
// stages its own H x 128 rows of X and half (128 rows) of the Yt tile.
//
// H = 1: 256x256 tiles, TMEM accumulators double-buffered (the epilogue of one tile
//        overlaps the next tile's mainloop), 6 stages of 32 KB.
// H = 2: 512x256 tiles (two M=256 MMAs per K step sharing the Yt half), each CTA's two
//        128x256 accumulators fill all 512 TMEM columns, 4 stages of 48 KB. A K step
//        then brings 96 KB per pair for 16.8 MFLOP instead of 64 KB for 8.4: a third less
//        L2->SMEM traffic per FLOP, the shape cuBLAS uses (nvjet 256x256_2cta per CTA),
//        which matters because these kernels run at the board power cap.
//        The next tile's MMAs into half h wait until the epilogue has drained half h.
//
// Statistics, each computed once and shared through the workspace:
//   t4 = colsum(Yt): a 1/grid slice per CTA in the epilogue-warp prologue,
//        published with a grid-wide counter (as in the 1-SM kernel);
//   t1, t2 (row sums of X and X^2) -> mu_neg, rstd: the 128 rows of a CTA's half
//        of m-unit m are reduced from global memory by the CTA whose tile (m, 0)
//        (the m-unit's first n-tile) comes next: it does so after its current
//        epilogue, one mainloop before the tile (m, 0) streams the same rows, so
//        they are still in L2 and X is read from HBM once. The statistics are
//        published with a per-row-tile release flag. Computing statistics never
//        waits, and (m, 0) precedes every (m, n) in the tile order, so every wait
//        is on work that never waits itself.
// The SMEM operand stages are read only by the tensor cores.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "sm100.cuh"
#include "plan.hpp"
#include "tma_host.hpp"

namespace bfgpu {
namespace lnmm2 {

constexpr int BM = 128;  // rows per CTA per MMA half (256 per pair and half)
#ifndef LNMM_STAT_ROWS
#define LNMM_STAT_ROWS 4
#endif
constexpr int BK = 64;
constexpr int BN = 256;
constexpr int OUT_BYTES = BM * 128 * 2;
constexpr int NUM_THREADS = 256;
constexpr int EPI_THREADS = 128;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t IDESC = dev::idesc_bf16_f32(256, 256);

template <int H>
struct Cfg {
  static constexpr int STAGES = H == 1 ? 6 : 4;
  static constexpr int A_BYTES = H * BM * BK * 2;
  static constexpr int B_BYTES = 128 * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int NUM_BARS = 2 * STAGES + 2 * 2;
  static constexpr int COLSUM_BYTES = BN * 4;  // the tile's colsum(Yt) slice, staged once per tile
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + OUT_BYTES + COLSUM_BYTES + NUM_BARS * 8 + 16;
  static_assert(SMEM_BYTES <= 232448, "K2 SMEM budget");
};

struct Params {
  int M, K, N;
  int Mt, Nt, kt;  // Mt in (256 H)-row units
  int num_tiles;
  int group;
  float inv_k;
  float eps;
  const __nv_bfloat16* X;
  const __nv_bfloat16* Yt;
  float* colsum;    // [N]
  float* row_mu;    // [M] -mean
  float* row_rstd;  // [M]
  int* col_ready;   // CTAs that published their colsum slice
  int* row_ready;   // [2*H*Mt] per 128-row tile: 1 once its statistics are published
  int staged;       // snapshot-0 schedule: statistics were computed by lnmm_stats_kernel before
                    // this launch (the program's separate `for k` map over X), nothing to wait for
};

// Snapshot 0 of fuse(lower(layernorm_matmul())) computes the row statistics in their own map
// (forall m: for k: t1 += row_sum(X), t2 += row_sum(square(X))) before the forall-n GEMM map,
// and colsum(Yt) inside it. As a launch: one warp per row of X, then per row of Yt.
__global__ void __launch_bounds__(256) lnmm_stats_kernel(const Params p) {
  using namespace dev;
  const uint32_t lane = lane_id();
  const int warps = static_cast<int>(gridDim.x * blockDim.x / 32);
  for (int r = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) / 32); r < p.M + p.N; r += warps) {
    if (r < p.M) {
      const __nv_bfloat16* rows[1] = {p.X + static_cast<size_t>(r) * p.K};
      float t1[1], t2[1], piv[1];
      warp_rows_moments_bf16<1, true>(rows, p.K, lane, t1, t2, piv);
      if (lane == 0) {
        const float dm = t1[0] * p.inv_k;
        p.row_mu[r] = -(piv[0] + dm);
        p.row_rstd[r] = 1.0f / sqrtf(t2[0] * p.inv_k - dm * dm + p.eps);
      }
    } else {
      const int n = r - p.M;
      const float2 mom = warp_row_moments_bf16(p.Yt + static_cast<size_t>(n) * p.K, p.K, lane);
      if (lane == 0) p.colsum[n] = mom.x;
    }
  }
}

__device__ __forceinline__ void decode(const Params& p, int t, int& m, int& n) {
  // Within a group of m-units, n is the slow index: every (m, 0) tile precedes (m, n>0).
  const int per_group = p.group * p.Nt;
  const int g = t / per_group;
  const int r = t % per_group;
  const int gs = min(p.group, p.Mt - g * p.group);
  m = g * p.group + r % gs;
  n = r / gs;
}

template <int H>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    ln_matmul_2sm_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_y,
                         const __grid_constant__ CUtensorMap tm_o, const Params p) {
  using namespace dev;
  using C = Cfg<H>;
  constexpr int STAGES = C::STAGES, A_BYTES = C::A_BYTES, STAGE_BYTES = C::STAGE_BYTES;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint8_t* stage_base = smem;
  uint8_t* out_stage = smem + STAGES * STAGE_BYTES;
  float* s_colsum = reinterpret_cast<float*>(out_stage + OUT_BYTES);  // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(out_stage + OUT_BYTES + C::COLSUM_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x >> 1;
  const int num_clusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_y);
    tma_prefetch_desc(&tm_o);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI_THREADS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
      for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
        int m, n;
        decode(p, t, m, n);
        // rows of MMA half h held by this CTA: m*256H + 256h + 128*rank
        const int mrow = m * 2 * H * BM + static_cast<int>(rank) * BM;
        for (int k = 0; k < p.kt; ++k) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = stage_base + stage * STAGE_BYTES;
          const uint32_t fbar = full0 + stage * 8;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
#pragma unroll
          for (int h = 0; h < H; ++h) tma_load_2d_2sm(&tm_x, fbar, sa + h * BM * BK * 2, k * BK, mrow + h * 2 * BM);
          tma_load_2d_2sm(&tm_y, fbar, sa + A_BYTES, k * BK, n * BN + static_cast<int>(rank) * 128);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t it = 0;  // tile iteration of this cluster
      for (int t = cluster_id; t < p.num_tiles; t += num_clusters, ++it) {
        // H = 1: accumulator it % 2, each completing every other tile; H = 2: both halves, every tile
        const uint32_t acc = H == 1 ? (it & 1) : 0;
        const uint32_t aphase = H == 1 ? ((it >> 1) & 1) : (it & 1);
        for (int k = 0; k < p.kt; ++k) {
          if (k == 0) {
#pragma unroll
            for (int h = 0; h < H; ++h) mbar_wait_cluster(&tempty[acc + h], aphase ^ 1);  // drained
            tc_fence_after();
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(stage_base + stage * STAGE_BYTES);
            const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
#pragma unroll
              for (int h = 0; h < H; ++h)
                umma_bf16_ss_2sm(tmem_base + (acc + h) * 256, sdesc_kmajor_sw128(a_addr + h * BM * BK * 2 + kk * 32),
                                 sdesc_kmajor_sw128(b_addr + kk * 32), IDESC, (k | kk) != 0);
            umma_commit_2sm_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) umma_commit_2sm_mc(&tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;
    const uint32_t etid = threadIdx.x - 4 * 32;
    const bool store_leader = etid == 0;
    const uint32_t out_addr = smem_u32(out_stage);
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);

    // ---- t4 = colsum(Yt): this CTA's slice, one warp per Yt row
    if (!p.staged) {
      const int per = (p.N + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
      const int n0 = static_cast<int>(blockIdx.x) * per, n1 = min(p.N, n0 + per);
      for (int n = n0 + static_cast<int>(q); n < n1; n += 4) {
        const float2 mom = warp_row_moments_bf16(p.Yt + static_cast<size_t>(n) * p.K, p.K, lane);
        if (lane == 0) p.colsum[n] = mom.x;
      }
      named_bar_sync(1, EPI_THREADS);
      if (store_leader) {
        __threadfence();
        red_release_gpu_add(p.col_ready, 1);
      }
    }
    bool col_seen = false;
    const int num_rt = (p.M + BM - 1) / BM;
    auto publish = [&](int r, float t1, float t2, float piv) {
      // moments about the pivot: t1 = sum (x - piv), t2 = sum (x - piv)^2, so
      // var = t2/total(K) + (0 - square(t1/total(K))) of the fused program [+ eps, 0 in the
      // reference] is the same quantity without the cancellation of E[x^2] - mu^2
      const float dm = t1 * p.inv_k;
      p.row_mu[r] = -(piv + dm);
      p.row_rstd[r] = 1.0f / sqrtf(t2 * p.inv_k - dm * dm + p.eps);
    };
    auto compute_row_tile = [&](int rt) {
      // kRows rows per warp at a time: these loads stream while the tensor cores run, and
      // the CTA must finish them within about one mainloop (measured at C4, TFLOP/s:
      // 1 row at a time 1456-1469, 2 rows 1509-1525, 4 rows 1512, 8 rows 1512)
      constexpr int kRows = LNMM_STAT_ROWS;
      for (int rr = kRows * static_cast<int>(q); rr < BM; rr += 4 * kRows) {
        const int r0 = rt * BM + rr;
        if (r0 >= p.M) break;
        const __nv_bfloat16* rows[kRows];
#pragma unroll
        for (int k = 0; k < kRows; ++k) rows[k] = p.X + static_cast<size_t>(min(r0 + k, p.M - 1)) * p.K;
        float t1[kRows], t2[kRows], piv[kRows];
        warp_rows_moments_bf16<kRows, true>(rows, p.K, lane, t1, t2, piv);
        if (lane == 0)
#pragma unroll
          for (int k = 0; k < kRows; ++k)
            if (r0 + k < p.M) publish(r0 + k, t1[k], t2[k], piv[k]);
      }
      named_bar_sync(1, EPI_THREADS);
      if (store_leader) {
        __threadfence();
        red_release_gpu_add(&p.row_ready[rt], 1);
      }
    };

    uint32_t it = 0;
    for (int t = cluster_id; t < p.num_tiles; t += num_clusters, ++it) {
      int m, n;
      decode(p, t, m, n);
      const uint32_t acc = H == 1 ? (it & 1) : 0;
      const uint32_t aphase = H == 1 ? ((it >> 1) & 1) : (it & 1);
      // this CTA's 128-row tiles of the output tile: m*2H + 2h + rank, h < H
      const int mt0 = m * 2 * H + static_cast<int>(rank);
      // ---- t1, t2 of this CTA's rows are produced by the CTA that owns the m-unit's
      // first n-tile (see header); in the first wave nobody ran ahead, so do it now.
      if (!p.staged && t == cluster_id && n == 0)
#pragma unroll
        for (int h = 0; h < H; ++h)
          if (mt0 + 2 * h < num_rt) compute_row_tile(mt0 + 2 * h);
      if (store_leader && !p.staged) {
        const uint64_t t0 = globaltimer_ns();
        auto rows_ready = [&] {
#pragma unroll
          for (int h = 0; h < H; ++h)  // no rows: nothing to wait for
            if (mt0 + 2 * h < num_rt && ld_acquire_gpu(&p.row_ready[mt0 + 2 * h]) < 1) return false;
          return true;
        };
        while ((!col_seen && ld_acquire_gpu(p.col_ready) < static_cast<int>(gridDim.x)) || !rows_ready()) {
          __nanosleep(128);
          if (globaltimer_ns() - t0 > 20000000000ull) __trap();
        }
      }
      col_seen = true;
      // The tile's colsum slice and this thread's row statistics, read once per tile while
      // the mainloop runs (read per 32 columns, their L2 latency sat in the epilogue's
      // critical path, which the single-buffered 512x256 tiles cannot hide).
      named_bar_sync(1, EPI_THREADS);  // statistics published (leader waited above); the
                                       // previous tile's epilogue is done with s_colsum
#pragma unroll
      for (int i = 0; i < BN / EPI_THREADS; ++i) {
        const int c = static_cast<int>(etid) * (BN / EPI_THREADS) + i;
        s_colsum[c] = n * BN + c < p.N ? __ldcg(p.colsum + n * BN + c) : 0.f;
      }
      float mu_neg_h[H], rstd_h[H];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int grow = (mt0 + 2 * h) * BM + static_cast<int>(row);
        mu_neg_h[h] = grow < p.M ? __ldcg(p.row_mu + grow) : 0.f;
        rstd_h[h] = grow < p.M ? __ldcg(p.row_rstd + grow) : 0.f;
      }
      named_bar_sync(1, EPI_THREADS);
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < H; ++h) {
        const int row0 = (mt0 + 2 * h) * BM;
        const uint32_t trow = tmem_base + (acc + h) * 256 + ((q * 32) << 16);
        const float mu_neg = h == 0 ? mu_neg_h[0] : mu_neg_h[H - 1];  // no dynamic indexing
        const float rstd = h == 0 ? rstd_h[0] : rstd_h[H - 1];
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {  // 128-column halves of the 256 columns
          if (store_leader) bulk_wait_read0();
          named_bar_sync(1, EPI_THREADS);  // staging free
#pragma unroll 1
          for (int j = 0; j < 4; ++j) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(trow + half * 128 + j * 32, v);
            float cs[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) {  // same address in every thread: broadcast
              const float4 f = reinterpret_cast<const float4*>(s_colsum + half * 128 + j * 32)[i];
              cs[4 * i] = f.x;
              cs[4 * i + 1] = f.y;
              cs[4 * i + 2] = f.z;
              cs[4 * i + 3] = f.w;
            }
            tmem_wait_ld();
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
          if (half == 1) {  // accumulator (half) drained: the next tile's MMAs may overwrite it
            tc_fence_before();
            if (leader)
              mbar_arrive(&tempty[acc + h]);
            else
              mbar_arrive_remote(tempty0 + (acc + h) * 8);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, EPI_THREADS);
          if (store_leader) {
            tma_store_2d(&tm_o, out_stage, n * BN + half * 128, row0);
            tma_store_2d(&tm_o, out_stage + BM * 128, n * BN + half * 128 + 64, row0);
            bulk_commit();
          }
        }
      }
      // Statistics for the next tile's rows if it opens an m-unit: they are read here,
      // one mainloop ahead of that tile's X stream, which then finds the rows in L2
      // (X leaves HBM once), and ahead of every other tile of the m-unit.
      const int tn = t + num_clusters;
      if (tn < p.num_tiles && !p.staged) {
        int m2, n2;
        decode(p, tn, m2, n2);
        const int mt2 = m2 * 2 * H + static_cast<int>(rank);
        if (n2 == 0)
#pragma unroll
          for (int h = 0; h < H; ++h)
            if (mt2 + 2 * h < num_rt) compute_row_tile(mt2 + 2 * h);
      }
    }
    if (store_leader) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

}  // namespace lnmm2

namespace lnmm2 {
template <int H>
KernelSpec spec_h() {
  using C = Cfg<H>;
  KernelSpec k;
  k.name = H == 1 ? "ln_matmul_2sm_kernel" : "ln_matmul_2sm_kernel<512x256>";
  k.func = reinterpret_cast<const void*>(&ln_matmul_2sm_kernel<H>);
  k.threads = NUM_THREADS;
  k.smem_bytes = C::SMEM_BYTES;
  k.tmem_cols = TMEM_COLS;
  k.cluster = 2;
  k.tile_m = 2 * H * BM;
  k.tile_n = BN;
  k.tile_k = BK;
  k.stages = C::STAGES;
  k.grid_sync = true;  // colsum counter and per-row-tile statistics flags are grid-wide
  return k;
}
}  // namespace lnmm2

// wide = true: 512x256 tiles per CTA pair (H = 2), else 256x256 (H = 1)
KernelSpec lnmm2_spec(bool wide) { return wide ? lnmm2::spec_h<2>() : lnmm2::spec_h<1>(); }

size_t lnmm2_workspace_bytes(int64_t M, int64_t N) {
  // per 128-row tile flags, for either tile height (4 ceil(M/512) >= 2 ceil(M/256))
  const size_t mt = static_cast<size_t>((M + 511) / 512) * 4;
  return align_up(static_cast<size_t>(N) * 4, 256) + 2 * align_up(static_cast<size_t>(M) * 4, 256) +
         align_up((mt + 1) * 4, 256);
}

void lnmm_bf16_2sm(const Plan& pl, const void* X, const void* Yt, void* O, float eps, void* ws, size_t ws_bytes,
                   cudaStream_t stream) {
  using namespace lnmm2;
  const int64_t M = pl.dims[0], K = pl.dims[1], N = pl.dims[2];
  BF_CHECK_ARG(ws != nullptr && ws_bytes >= lnmm2_workspace_bytes(M, N), "bf_layernorm_matmul: workspace too small");
  uint8_t* w = static_cast<uint8_t*>(ws);
  Params p{};
  p.M = static_cast<int>(M);
  p.K = static_cast<int>(K);
  p.N = static_cast<int>(N);
  const int H = pl.spec.tile_m == 512 ? 2 : 1;
  p.Mt = static_cast<int>(pl.units);
  p.Nt = static_cast<int>((N + BN - 1) / BN);
  p.kt = static_cast<int>((K + BK - 1) / BK);
  p.group = pl.group;
  p.inv_k = 1.0f / static_cast<float>(K);
  p.eps = eps;
  p.X = static_cast<const __nv_bfloat16*>(X);
  p.Yt = static_cast<const __nv_bfloat16*>(Yt);
  p.colsum = reinterpret_cast<float*>(w);
  w += align_up(static_cast<size_t>(N) * 4, 256);
  p.row_mu = reinterpret_cast<float*>(w);
  w += align_up(static_cast<size_t>(M) * 4, 256);
  p.row_rstd = reinterpret_cast<float*>(w);
  w += align_up(static_cast<size_t>(M) * 4, 256);
  p.col_ready = reinterpret_cast<int*>(w);
  p.row_ready = p.col_ready + 1;
  p.num_tiles = static_cast<int>(pl.tiles);

  const CUtensorMap tm_x = make_tmap_bf16(X, M, K, K, BK, BM);
  const CUtensorMap tm_y = make_tmap_bf16(Yt, N, K, K, BK, 128);
  const CUtensorMap tm_o = make_tmap_bf16(O, M, N, N, BK, BM);
  p.staged = pl.schedule == BF_SCHED_STAGED;
  if (p.staged) {
    // the statistics map as its own launch: 8 warps per CTA, a few rows per warp
    const int64_t warps_needed = (M + N + 3) / 4;
    const int grid = static_cast<int>(std::min<int64_t>((warps_needed + 7) / 8, static_cast<int64_t>(pl.dev.sms) * 8));
    lnmm_stats_kernel<<<grid, 256, 0, stream>>>(p);
    BF_CUDA(cudaGetLastError());
    note_launch();
  } else {
    BF_CUDA(cudaMemsetAsync(p.col_ready, 0, (static_cast<size_t>(p.Mt) * 2 * H + 1) * sizeof(int), stream));
  }
  if (H == 2)
    launch_planned(pl, ln_matmul_2sm_kernel<2>, stream, tm_x, tm_y, tm_o, p);
  else
    launch_planned(pl, ln_matmul_2sm_kernel<1>, stream, tm_x, tm_y, tm_o, p);
}

}  // namespace bfgpu
