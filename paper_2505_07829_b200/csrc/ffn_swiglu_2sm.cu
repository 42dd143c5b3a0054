// K1 Flash-RMSNorm + FFN-SwiGLU, CTA-pair (cta_group::2) variant.
//
// Same block program and tile schedule as ffn_swiglu.cu (see there for the
// listing). A cluster of two CTAs on one TPC computes 256-row tiles with
// M=256 tcgen05 MMAs issued by the pair leader. Each CTA stages its own 128
// rows of A and HALF of B:
//   gate/up tile: CTA0 holds the Wt chunk, CTA1 the Vt chunk (B = [Wt; Vt]
//                 split across the pair), so one M=256,N=256 MMA per K=16 step
//                 leaves gate | up side by side in each CTA's TMEM;
//   down tile:    CTA r holds Ut rows [n*256 + r*128, +128).
// Per SM this is 32 KB of SMEM operands per 128x256x64 step instead of 48 KB.
//
// Row statistics. r_i = 1/sqrt(sum_d x_id^2 / D + eps) depends only on the
// row, so the fused program's per-(m,n) recomputation (the `t2` accumulator)
// is done once per row here: at kernel start the epilogue warps, which are
// idle until the first accumulator is ready, reduce a 1/grid slice of X's rows
// from global memory into the workspace and publish it with a grid-wide
// release counter; gate/up epilogues read r after an acquire on that counter.
// Nothing but the MMA reads the SMEM operand stages.
//
// Synchronization:
//   full[s]  (leader) TMA bytes of both CTAs (2-SM TMA) + the leader producer's arrive
//   empty[s]          2-SM MMA commit, multicast to both CTAs
//   tfull[a]          2-SM MMA commit, multicast: accumulator a is final
//   tempty[a](leader) 256 epilogue threads of both CTAs (the peer arrives remotely)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "ffn_common.cuh"
#include "sm100.cuh"
#include "plan.hpp"
#include "tma_host.hpp"

namespace bfgpu {
namespace ffn2 {

using ffn::kDownOnly;
using ffn::kFused;
using ffn::kGateUpOnly;
using ffn::Params;
using ffn::Tile;

constexpr int BM = 128;  // rows per CTA (256 per pair)
constexpr int BK = 64;
constexpr int BF = 128;
constexpr int BN = 256;
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = 128 * BK * 2;  // 16 KB: this CTA's half of B
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int OUT_BYTES = BM * 128 * 2;
constexpr int NUM_THREADS = 256;
constexpr int EPI_THREADS = 128;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t IDESC = dev::idesc_bf16_f32(256, 256);
constexpr int NUM_BARS = 2 * STAGES + 2 * 2;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + OUT_BYTES + NUM_BARS * 8 + 16;

struct Extra {
  const __nv_bfloat16* X;  // for the row statistics
  float* rstat;            // [M] r per row
  int* stats_ready;        // CTAs that published their slice
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    ffn_swiglu_2sm_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_wt,
                          const __grid_constant__ CUtensorMap tm_vt, const __grid_constant__ CUtensorMap tm_ut,
                          const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_o,
                          const Params p, const Extra ex) {
  using namespace dev;
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  uint8_t* stage_base = smem;
  uint8_t* out_stage = smem + STAGES * STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(out_stage + OUT_BYTES);
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
    tma_prefetch_desc(&tm_wt);
    tma_prefetch_desc(&tm_vt);
    tma_prefetch_desc(&tm_ut);
    tma_prefetch_desc(&tm_h);
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
  cluster_sync();  // barrier inits and the TMEM allocation are visible pair-wide
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);  // leader's full[0]
      int iter = 0;
      for (int t = cluster_id; t < p.num_tiles; t += num_clusters, ++iter) {
        const Tile tl = ffn::decode_tile(p, t);
        const int mrow = tl.m * 2 * BM + static_cast<int>(rank) * BM;
        if (p.seg && leader) {
          // Segment sync (fused schedule without the wave sync): no cluster starts a tile past
          // the first two gate/up segments until all of those have been started, so the
          // down-projection segments begin with the clusters aligned, as after a kernel
          // boundary. Tiles before that point never wait here.
          if (t < p.seg_tiles) {
            red_release_gpu_add(p.seg, 1);
          } else if (t - num_clusters < p.seg_tiles) {  // this cluster's first tile past the point
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_gpu(p.seg) < p.seg_tiles) {
              __nanosleep(64);
              if (globaltimer_ns() - t0 > 20000000000ull) __trap();
            }
          }
        }
        if (p.wave && leader) {
          // Wave sync: start iteration i only once every cluster has started iteration i-1,
          // so the tiles of one wave (consecutive indices, which share operand row-blocks)
          // stay close enough in time to share them through L2.
          if (iter > 0) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_gpu(p.wave) < iter * num_clusters) {
              __nanosleep(64);
              if (globaltimer_ns() - t0 > 20000000000ull) __trap();
            }
          }
          red_release_gpu_add(p.wave, 1);
        }
        if (tl.kind == 1 && p.mode == kFused) {
          const int flag = tl.m * 2 + static_cast<int>(rank);
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_gpu(&p.flags[flag]) < p.Ft) {
            __nanosleep(128);
            if (globaltimer_ns() - t0 > 20000000000ull) __trap();
          }
          fence_proxy_async_global();
        }
        const int nk = tl.kind == 0 ? p.kt_d : p.kt_f;
        for (int k = 0; k < nk; ++k) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = stage_base + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint32_t fbar = full0 + stage * 8;
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE_BYTES);
          if (tl.kind == 0) {
            tma_load_2d_2sm(&tm_x, fbar, sa, k * BK, mrow);
            tma_load_2d_2sm(rank == 0 ? &tm_wt : &tm_vt, fbar, sb, k * BK, tl.j * BF);
          } else {
            tma_load_2d_2sm(&tm_h, fbar, sa, k * BK, mrow);
            tma_load_2d_2sm(&tm_ut, fbar, sb, k * BK, tl.j * BN + static_cast<int>(rank) * 128);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc = 0, aphase = 0;
      for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
        const Tile tl = ffn::decode_tile(p, t);
        const int nk = tl.kind == 0 ? p.kt_d : p.kt_f;
        mbar_wait_cluster(&tempty[acc], aphase ^ 1);  // both CTAs drained accumulator acc
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * 256;
        for (int k = 0; k < nk; ++k) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(stage_base + stage * STAGE_BYTES);
            const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              umma_bf16_ss_2sm(d_tmem, sdesc_kmajor_sw128(a_addr + kk * 32), sdesc_kmajor_sw128(b_addr + kk * 32),
                               IDESC, (k | kk) != 0);
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
        acc ^= 1;
        if (acc == 0) aphase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;
    const uint32_t etid = threadIdx.x - 4 * 32;
    const bool store_leader = etid == 0;
    const uint32_t out_addr = smem_u32(out_stage);
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);

    // ---- row statistics for a 1/gridDim slice of the rows (t2 of the fused program)
    if (p.mode != kDownOnly) {
      const int per = (p.M + static_cast<int>(gridDim.x) - 1) / static_cast<int>(gridDim.x);
      const int r0 = static_cast<int>(blockIdx.x) * per, r1 = min(p.M, r0 + per);
      // four rows per warp at a time (32 loads per lane in flight): the first epilogue waits
      // for every CTA's slice, so this prologue is on the critical path
      for (int r = r0 + 4 * static_cast<int>(q); r < r1; r += 16) {
        const __nv_bfloat16* rows[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) rows[k] = ex.X + static_cast<size_t>(min(r + k, r1 - 1)) * p.D;
        float t1[4], t2[4], piv[4];
        warp_rows_moments_bf16<4>(rows, p.D, lane, t1, t2, piv);
        if (lane == 0)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (r + k < r1) ex.rstat[r + k] = 1.0f / sqrtf(t2[k] * p.inv_d + p.eps);
      }
      named_bar_sync(1, EPI_THREADS);
      if (store_leader) {
        __threadfence();
        red_release_gpu_add(ex.stats_ready, 1);
      }
    }
    bool stats_seen = false;

    uint32_t acc = 0, aphase = 0;
    for (int t = cluster_id; t < p.num_tiles; t += num_clusters) {
      const Tile tl = ffn::decode_tile(p, t);
      const int mtile = tl.m * 2 + static_cast<int>(rank);
      float r = 0.f;
      if (tl.kind == 0) {
        if (!stats_seen) {
          if (store_leader) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_gpu(ex.stats_ready) < static_cast<int>(gridDim.x)) {
              __nanosleep(256);
              if (globaltimer_ns() - t0 > 20000000000ull) __trap();
            }
          }
          named_bar_sync(1, EPI_THREADS);
          stats_seen = true;
        }
        const int grow = mtile * BM + static_cast<int>(row);
        r = grow < p.M ? __ldcg(ex.rstat + grow) : 0.f;
      }
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t trow = tmem_base + acc * 256 + ((q * 32) << 16);
      auto release_tmem = [&] {
        tc_fence_before();
        if (leader)
          mbar_arrive(&tempty[acc]);
        else
          mbar_arrive_remote(tempty0 + acc * 8);
      };
      if (tl.kind == 0) {
        if (store_leader) bulk_wait_read0();
        named_bar_sync(1, EPI_THREADS);
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          uint32_t g[32], u[32];
          tmem_ld_32x32b_x32(trow + j * 32, g);
          tmem_ld_32x32b_x32(trow + 128 + j * 32, u);
          tmem_wait_ld();
          uint32_t hv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float g0 = r * __uint_as_float(g[2 * i]);
            const float g1 = r * __uint_as_float(g[2 * i + 1]);
            const float u0 = r * __uint_as_float(u[2 * i]);
            const float u1 = r * __uint_as_float(u[2 * i + 1]);
            hv[i] = pack_bf16x2(__fdividef(g0, 1.0f + __expf(-g0)) * u0, __fdividef(g1, 1.0f + __expf(-g1)) * u1);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int chunk = j * 4 + c;
            st_shared_v4(out_addr + (chunk >> 3) * (BM * 128) + sw128_offset(row, chunk & 7), hv[4 * c],
                         hv[4 * c + 1], hv[4 * c + 2], hv[4 * c + 3]);
          }
        }
        release_tmem();
        fence_proxy_async_smem();
        named_bar_sync(1, EPI_THREADS);
        if (store_leader) {
          tma_store_2d(&tm_h, out_stage, tl.j * BF, mtile * BM);
          tma_store_2d(&tm_h, out_stage + BM * 128, tl.j * BF + 64, mtile * BM);
          bulk_commit();
          if (p.mode == kFused) {
            bulk_wait0();
            fence_proxy_async_global();
            red_release_gpu_add(&p.flags[mtile], 1);
          }
        }
      } else {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          if (store_leader) bulk_wait_read0();
          named_bar_sync(1, EPI_THREADS);
#pragma unroll 1
          for (int j = 0; j < 4; ++j) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(trow + half * 128 + j * 32, v);
            tmem_wait_ld();
            uint32_t ov[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) ov[i] = pack_bf16x2(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int chunk = j * 4 + c;
              st_shared_v4(out_addr + (chunk >> 3) * (BM * 128) + sw128_offset(row, chunk & 7), ov[4 * c],
                           ov[4 * c + 1], ov[4 * c + 2], ov[4 * c + 3]);
            }
          }
          if (half == 1) release_tmem();
          fence_proxy_async_smem();
          named_bar_sync(1, EPI_THREADS);
          if (store_leader) {
            tma_store_2d(&tm_o, out_stage, tl.j * BN + half * 128, mtile * BM);
            tma_store_2d(&tm_o, out_stage + BM * 128, tl.j * BN + half * 128 + 64, mtile * BM);
            bulk_commit();
          }
        }
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (store_leader) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the leader's MMAs into the peer's TMEM are complete on both sides
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
  }
}

}  // namespace ffn2

KernelSpec ffn2_spec() {
  using namespace ffn2;
  KernelSpec k;
  k.name = "ffn_swiglu_2sm_kernel";
  k.func = reinterpret_cast<const void*>(&ffn_swiglu_2sm_kernel);
  k.threads = NUM_THREADS;
  k.smem_bytes = SMEM_BYTES;
  k.tmem_cols = TMEM_COLS;
  k.cluster = 2;
  k.tile_m = 2 * BM;
  k.tile_n = BN;
  k.tile_k = BK;
  k.stages = STAGES;
  k.grid_sync = true;  // row statistics, fused hand-off flags, wave/segment sync are grid-wide
  return k;
}

// Launch the CTA-pair kernel as planned. `counters` = [2*Mt flags][stats_ready][wave][seg], zeroed.
void ffn_swiglu_bf16_2sm(const Plan& pl, const void* X, const void* Wt, const void* Vt, const void* Ut, void* O,
                         void* H, float* rstat, int* counters, float eps, cudaStream_t stream) {
  using namespace ffn2;
  const int64_t M = pl.dims[0], D = pl.dims[1], F = pl.dims[2], N = pl.dims[3];
  const CUtensorMap tm_x = make_tmap_bf16(X, M, D, D, BK, BM);
  const CUtensorMap tm_wt = make_tmap_bf16(Wt, F, D, D, BK, BF);
  const CUtensorMap tm_vt = make_tmap_bf16(Vt, F, D, D, BK, BF);
  const CUtensorMap tm_ut = make_tmap_bf16(Ut, N, F, F, BK, 128);
  const CUtensorMap tm_h = make_tmap_bf16(H, M, F, F, BK, BM);
  const CUtensorMap tm_o = make_tmap_bf16(O, M, N, N, BK, BM);

  ffn::Params p{};
  p.M = static_cast<int>(M);
  p.D = static_cast<int>(D);
  p.F = static_cast<int>(F);
  p.N = static_cast<int>(N);
  p.Mt = static_cast<int>(pl.units);
  p.Ft = static_cast<int>((F + BF - 1) / BF);
  p.Nt = static_cast<int>((N + BN - 1) / BN);
  p.kt_d = static_cast<int>((D + BK - 1) / BK);
  p.kt_f = static_cast<int>((F + BK - 1) / BK);
  p.inv_d = 1.0f / static_cast<float>(D);
  p.eps = eps;
  p.flags = counters;
  p.group = pl.group;
  p.braster = pl.raster;
  int* stats_ready = counters + 2 * p.Mt;
  p.wave = pl.sync == kSyncWave ? stats_ready + 1 : nullptr;
  p.seg = nullptr;
  p.seg_tiles = 0;
  if (pl.sync == kSyncSegment) {
    // no cluster starts a tile past the first two gate/up segments before all of those started
    const int ngroups = (p.Mt + p.group - 1) / p.group;
    const int g0 = std::min(p.group, p.Mt), g1 = ngroups > 1 ? std::min(p.group, p.Mt - p.group) : 0;
    p.seg = stats_ready + 2;
    p.seg_tiles = (g0 + g1) * p.Ft;
  }
  Extra ex{static_cast<const __nv_bfloat16*>(X), rstat, stats_ready};
  auto launch = [&](int mode) {
    ffn::Params q = p;
    q.mode = mode;
    const long long a_tiles = static_cast<long long>(q.Mt) * q.Ft;
    const long long b_tiles = static_cast<long long>(q.Mt) * q.Nt;
    q.num_tiles = static_cast<int>(mode == kFused ? a_tiles + b_tiles : (mode == kGateUpOnly ? a_tiles : b_tiles));
    Plan lp = pl;
    lp.grid = std::min(pl.grid / 2, q.num_tiles) * 2;
    // the wave counter restarts for every launch (the two-phase schedule launches twice)
    if (q.wave && mode == kDownOnly) BF_CUDA(cudaMemsetAsync(q.wave, 0, sizeof(int), stream));
    launch_planned(lp, ffn_swiglu_2sm_kernel, stream, tm_x, tm_wt, tm_vt, tm_ut, tm_h, tm_o, q, ex);
  };
  if (pl.schedule == BF_FFN_FUSED) {
    launch(kFused);
  } else {
    launch(kGateUpOnly);
    launch(kDownOnly);
  }
}

}  // namespace bfgpu
