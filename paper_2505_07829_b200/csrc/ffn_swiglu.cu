// K1: Flash-RMSNorm + FFN-SwiGLU on sm_100a.
//
// Block program (final snapshot of fuse(lower(examples::rms_ffn_swiglu())),
// reference lowering.hpp:583-597, listing in SURVEY.md §2.1):
//
//   forall m: forall n: for k: for d:  t2 += row_sum(square(X[m][d]))
//                                      t3 += dot(X[m][d], Wt[k][d]); t4 += dot(X[m][d], Vt[k][d])
//                          r = recip(sqrt(t2/total(D) + eps))
//                          h = swish(row_scale(t3, r)) * row_scale(t4, r)
//                          t1 += dot(h, Ut[n][k])
//               O[m][n] = t1
//
// B200 mapping. One persistent, warp-specialized kernel runs two tile kinds
// that share one SMEM pipeline shape (A tile 128x64, B tile 256x64 bf16 per
// stage) and one TMEM shape (128 lanes x 256 fp32 columns, double buffered):
//   kind 0 "gate/up": (m, f-chunk of 128) -> one M=128,N=256 tcgen05 MMA per
//          K=16 step with B = [Wt chunk ; Vt chunk] stacked in SMEM, so the
//          gate and up products land side by side in TMEM. Stats warps read
//          the same X tiles from SMEM for sum(x^2) (rule R4: the row scale is
//          applied after the dot). The epilogue applies r, swish and the
//          Hadamard product and emits the bf16 h tile.
//   kind 1 "down": (m, n-chunk of 256) -> O tile = H[m,:] Ut[n,:]^T.
// In the fused schedule both kinds run in one launch: down tiles of m-group
// g are interleaved after gate/up tiles of group g+1 and wait on per-m-tile
// completion counters, so H is produced and consumed while L2-resident.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w3 idle, w4-7 epilogue (TMEM lanes 0-127), w8-11 row statistics.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "sm100.cuh"
#include "tma_host.hpp"
#include "ffn_common.cuh"
#include "plan.hpp"

namespace bfgpu {
namespace ffn {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int BF = 128;  // ffn columns per gate/up tile (x2 for gate+up = UMMA N 256)
constexpr int BN = 256;  // output columns per down tile
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = 256 * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int OUT_BYTES = BM * 128 * 2;  // staging for one 128x128 bf16 tile (two SW128 boxes)
constexpr int NUM_THREADS = 384;
constexpr int EPI_THREADS = 128;
constexpr int STATS_THREADS = 128;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t IDESC = dev::idesc_bf16_f32(128, 256);

constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + OUT_BYTES + 2 * BM * 4 /*rstat*/ + 256 /*barriers*/ + 1024;

__global__ void __launch_bounds__(NUM_THREADS, 1)
    ffn_swiglu_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_wt,
                      const __grid_constant__ CUtensorMap tm_vt, const __grid_constant__ CUtensorMap tm_ut,
                      const __grid_constant__ CUtensorMap tm_h, const __grid_constant__ CUtensorMap tm_o,
                      const Params p) {
  using namespace dev;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint8_t* out_stage = smem + STAGES * STAGE_BYTES;
  float* rstat = reinterpret_cast<float*>(out_stage + OUT_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(rstat + 2 * BM);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + 2);

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_wt);
    tma_prefetch_desc(&tm_vt);
    tma_prefetch_desc(&tm_ut);
    tma_prefetch_desc(&tm_h);
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
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        const Tile tl = decode_tile(p, t);
        if (tl.kind == 1 && p.mode == kFused) {
          // H rows of this m-tile must be complete (all Ft gate/up tiles).
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_gpu(&p.flags[tl.m]) < p.Ft) {
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
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          if (tl.kind == 0) {
            tma_load_2d(&tm_x, &full[stage], sa, k * BK, tl.m * BM);
            tma_load_2d(&tm_wt, &full[stage], sb, k * BK, tl.j * BF);
            tma_load_2d(&tm_vt, &full[stage], sb + B_BYTES / 2, k * BK, tl.j * BF);
          } else {
            tma_load_2d(&tm_h, &full[stage], sa, k * BK, tl.m * BM);
            tma_load_2d(&tm_ut, &full[stage], sb, k * BK, tl.j * BN);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc = 0, aphase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      const Tile tl = decode_tile(p, t);
      const int nk = tl.kind == 0 ? p.kt_d : p.kt_f;
      mbar_wait(&tempty[acc], aphase ^ 1);
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
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;
    const uint32_t row = q * 32 + lane;
    const bool leader = threadIdx.x == 4 * 32;
    uint32_t acc = 0, aphase = 0;
    uint32_t sphase = 0;  // bit a: parity of sfull[a], which completes once per gate/up tile on slot a
    const uint32_t out_addr = smem_u32(out_stage);
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      const Tile tl = decode_tile(p, t);
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t trow = tmem_base + acc * 256 + ((q * 32) << 16);
      if (tl.kind == 0) {
        mbar_wait(&sfull[acc], (sphase >> acc) & 1u);
        sphase ^= 1u << acc;
        const float r = rstat[acc * BM + row];
        if (leader) bulk_wait_read0();  // staging buffer free again
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
            const float h0 = __fdividef(g0, 1.0f + __expf(-g0)) * u0;
            const float h1 = __fdividef(g1, 1.0f + __expf(-g1)) * u1;
            hv[i] = pack_bf16x2(h0, h1);
          }
          // 32 columns = 4 chunks of 16 B; columns [64*b, 64*b+64) live in box b.
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int chunk = j * 4 + c;
            st_shared_v4(out_addr + (chunk >> 3) * (BM * 128) + sw128_offset(row, chunk & 7), hv[4 * c],
                         hv[4 * c + 1], hv[4 * c + 2], hv[4 * c + 3]);
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        fence_proxy_async_smem();
        named_bar_sync(1, EPI_THREADS);
        if (leader) {
          tma_store_2d(&tm_h, out_stage, tl.j * BF, tl.m * BM);
          tma_store_2d(&tm_h, out_stage + BM * 128, tl.j * BF + 64, tl.m * BM);
          bulk_commit();
          if (p.mode == kFused) {
            bulk_wait0();
            fence_proxy_async_global();
            red_release_gpu_add(&p.flags[tl.m], 1);
          }
        }
      } else {
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          if (leader) bulk_wait_read0();
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
          if (half == 1) {
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
          }
          fence_proxy_async_smem();
          named_bar_sync(1, EPI_THREADS);
          if (leader) {
            tma_store_2d(&tm_o, out_stage, tl.j * BN + half * 128, tl.m * BM);
            tma_store_2d(&tm_o, out_stage + BM * 128, tl.j * BN + half * 128 + 64, tl.m * BM);
            bulk_commit();
          }
        }
      }
      acc ^= 1;
      if (acc == 0) aphase ^= 1;
    }
    if (leader) bulk_wait0();
  } else if (warp >= 8) {
    // ------------------------------------------------------------ row statistics
    const uint32_t row = (warp - 8) * 32 + lane;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc = 0, aphase = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      const Tile tl = decode_tile(p, t);
      if (tl.kind == 0) {
        float ss0 = 0.f, ss1 = 0.f;
        for (int k = 0; k < p.kt_d; ++k) {
          mbar_wait(&full[stage], phase);
          const uint32_t base = smem_u32(stage_base + stage * STAGE_BYTES) + row * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            // rotate the chunk order per lane: 8 consecutive rows hit 8 distinct bank groups
            const uint4 v = ld_shared_v4(base + (((c + lane) & 7) << 4));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float lo = __uint_as_float(w[e] << 16);
              const float hi = __uint_as_float(w[e] & 0xffff0000u);
              ss0 = fmaf(lo, lo, ss0);
              ss1 = fmaf(hi, hi, ss1);
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
        rstat[acc * BM + row] = 1.0f / sqrtf((ss0 + ss1) * p.inv_d + p.eps);
        __threadfence_block();  // publish the STS before the arrive (SYNCS does not order it)
        mbar_arrive(&sfull[acc]);
      } else {
        // Down tiles carry no statistics, but the stats warps still consume every
        // stage in order: a consumer that skipped ahead could alias mbarrier
        // parities of phases two or more apart.
        for (int k = 0; k < p.kt_f; ++k) {
          mbar_wait(&full[stage], phase);
          mbar_arrive(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
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

}  // namespace ffn

// ------------------------------------------------------------------ host side

KernelSpec ffn1_spec() {
  using namespace ffn;
  KernelSpec k;
  k.name = "ffn_swiglu_kernel";
  k.func = reinterpret_cast<const void*>(&ffn_swiglu_kernel);
  k.threads = NUM_THREADS;
  k.smem_bytes = SMEM_BYTES;
  k.tmem_cols = TMEM_COLS;
  k.cluster = 1;
  k.tile_m = BM;
  k.tile_n = BN;
  k.tile_k = BK;
  k.stages = STAGES;
  k.grid_sync = true;  // fused down tiles wait on other CTAs' gate/up tiles
  return k;
}

namespace {

size_t ffn_h_bytes(int64_t M, int64_t F) { return align_up(static_cast<size_t>(M) * F * 2, 1024); }
// Counters: per m-tile completion flags (ceil(M/128) for the 1-SM kernel, 2*ceil(M/256) for
// the CTA pair, which can be one more), then the statistics, wave and segment counters.
size_t ffn_flag_count(int64_t M) { return std::max((M + 127) / 128, 2 * ((M + 255) / 256)) + 3; }
size_t ffn_flag_bytes(int64_t M) { return align_up(ffn_flag_count(M) * 4, 256); }
size_t ffn_rstat_bytes(int64_t M) { return align_up(static_cast<size_t>(M) * 4, 256); }

}  // namespace

size_t ffn_workspace_bytes(int64_t M, int64_t D, int64_t F, int64_t N) {
  (void)D;
  (void)N;
  return ffn_h_bytes(M, F) + ffn_rstat_bytes(M) + ffn_flag_bytes(M);
}

void ffn_swiglu_bf16_2sm(const Plan& pl, const void* X, const void* Wt, const void* Vt, const void* Ut, void* O,
                         void* H, float* rstat, int* counters, float eps, cudaStream_t stream);

void ffn_swiglu_bf16(const void* X, const void* Wt, const void* Vt, const void* Ut, void* O, int64_t M, int64_t D,
                     int64_t F, int64_t N, float eps, int schedule, void* ws, size_t ws_bytes, cudaStream_t stream) {
  using namespace ffn;
  BF_CHECK_ARG(M > 0 && D > 0 && F > 0 && N > 0, "bf_rms_ffn_swiglu: sizes must be positive");
  BF_CHECK_ARG(D % 8 == 0 && F % 8 == 0 && N % 8 == 0, "bf_rms_ffn_swiglu: D, F and N must be multiples of 8");
  BF_CHECK_ARG(M < (1ll << 31) && D < (1ll << 31) && F < (1ll << 31) && N < (1ll << 31),
               "bf_rms_ffn_swiglu: dimension too large");
  BF_CHECK_ARG(ws != nullptr && ws_bytes >= ffn_workspace_bytes(M, D, F, N),
               "bf_rms_ffn_swiglu: workspace too small");
  BF_CHECK_ARG(schedule == BF_FFN_FUSED || schedule == BF_FFN_TWO_PHASE, "bf_rms_ffn_swiglu: bad schedule");

  uint8_t* wsb = static_cast<uint8_t*>(ws);
  void* H = wsb;
  float* rstat = reinterpret_cast<float*>(wsb + ffn_h_bytes(M, F));
  int* counters = reinterpret_cast<int*>(wsb + ffn_h_bytes(M, F) + ffn_rstat_bytes(M));
  // counters: [flags ...][stats_ready][wave][seg], zeroed once per call
  BF_CUDA(cudaMemsetAsync(counters, 0, ffn_flag_count(M) * sizeof(int), stream));

  const Plan pl = plan_ffn(M, D, F, N, BF_DTYPE_BF16, schedule);
  if (pl.spec.cluster == 2) {
    ffn_swiglu_bf16_2sm(pl, X, Wt, Vt, Ut, O, H, rstat, counters, eps, stream);
    return;
  }

  const CUtensorMap tm_x = make_tmap_bf16(X, M, D, D, BK, BM);
  const CUtensorMap tm_wt = make_tmap_bf16(Wt, F, D, D, BK, BF);
  const CUtensorMap tm_vt = make_tmap_bf16(Vt, F, D, D, BK, BF);
  const CUtensorMap tm_ut = make_tmap_bf16(Ut, N, F, F, BK, BN);
  const CUtensorMap tm_h = make_tmap_bf16(H, M, F, F, BK, BM);
  const CUtensorMap tm_o = make_tmap_bf16(O, M, N, N, BK, BM);

  Params p{};
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
  p.braster = 0;

  auto launch = [&](int mode) {
    Params q = p;
    q.mode = mode;
    const long long a_tiles = static_cast<long long>(q.Mt) * q.Ft;
    const long long b_tiles = static_cast<long long>(q.Mt) * q.Nt;
    q.num_tiles = static_cast<int>(mode == kFused ? a_tiles + b_tiles : (mode == kGateUpOnly ? a_tiles : b_tiles));
    Plan lp = pl;
    lp.grid = std::min(pl.grid, q.num_tiles);
    launch_planned(lp, ffn_swiglu_kernel, stream, tm_x, tm_wt, tm_vt, tm_ut, tm_h, tm_o, q);
  };
  if (schedule == BF_FFN_FUSED) {
    launch(kFused);
  } else {
    launch(kGateUpOnly);
    launch(kDownOnly);
  }
}

}  // namespace bfgpu
