// fp32 mode of K2 (LayerNorm -> MatMul) on the tensor cores: three-pass TF32 ("3xTF32").
//
// The north star asks fp32 inputs to match the float64 reference within 1e-4. One TF32
// product (10-bit mantissa) misses that by two orders of magnitude, but splitting each
// operand into a TF32 head and an fp32 tail,
//     x = x_hi + x_lo,  x_hi = rna_tf32(x),  x_lo = x - x_hi  (exact in fp32),
// and accumulating x_hi y_hi + x_hi y_lo + x_lo y_hi in the fp32 TMEM accumulator leaves
// only x_lo y_lo (2^-22 relative) and the TF32 truncation of the tails (2^-21): about
// 1e-6 relative on a K = 1024 contraction, while running on tcgen05 (kind::tf32, 1.1 PF
// dense nominal) instead of the FP32 FMA pipes (73 TF/s measured).
//
// Two launches (the statistics map, then the GEMM map: the plan of the program's first
// fusion snapshot, which computes the row statistics in their own map):
//   f32_split_kernel   one warp per row. Rows of X: moments about the pivot p = x_0 give
//                      dm = mean - p and rstd; the row is shifted by p before the split
//                      (x - p is exact when |mu| >> sigma, where centring on a rounded fp32
//                      mean would not be: at |mu|/sigma = 1e4 the mean's rounding alone is
//                      5e-4 sigma), so the GEMM never sees the large common offset. Rows of
//                      Yt: split, and colsum(Yt) for the rank-1 correction of rule R5.
//                      Tails padded to Kp = 32k.
//   f32x3_gemm_kernel  128 x 128 output tiles, K split over a CTA pair; TMA-fed 3-stage
//                      ring of {X_hi, X_lo, Y_hi, Y_lo} 32-column slabs (SW128), 3 MMAs per
//                      K=8 step; each rank pushes its partial sums of the other rank's column
//                      half into the peer's SMEM (remote stores), then finalizes its own half:
//                      O = (acc0 + acc1 - dm colsum(Yt)) * rstd straight to global.
// Reference: ref::layernorm_matmul (interpreter.hpp:549-551); the block program is the
// final snapshot of fuse(lower(examples::layernorm_matmul())) (lowering.hpp:573-581).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "plan.hpp"
#include "sm100.cuh"
#include "tma_host.hpp"

namespace bfgpu {
namespace f32x3 {

// 128 x 128 output tiles (one tf32 MMA of N = 128 reads 8 KB of SMEM per 64 tensor cycles:
// SMEM and tensor pipe balance; N = 64 tiles are SMEM-bound at 1.5x). Each tile's K range is
// split over a CTA pair (cluster of 2), so a 1024^2 output still fills 128 SMs; the pair sums
// its two accumulators through distributed shared memory in a fixed order (deterministic).
constexpr int BM = 128, BN = 128, BK = 32;  // BK fp32 = one 128-byte swizzle row
constexpr int A_BYTES = BM * BK * 4;  // 16 KB
constexpr int B_BYTES = BN * BK * 4;  // 16 KB
constexpr int NUM_THREADS = 256;
// kind::tf32 instruction descriptor: D F32, A/B TF32 (format 2), both K-major, N/8, M/16
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

__device__ __forceinline__ void umma_tf32_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate,
                                             uint32_t idesc = IDESC) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// One operand of the split launch: `rows` rows of `src` ([rows, K] row-major) go to hi/lo
// ([rows, Kp], tails zero).
//   kSegLn    LayerNorm rows: moments about the pivot x_0, stat0 = rstd, stat1 = p - mean, and
//             the row is shifted by the pivot before the split;
//   kSegRms   RMSNorm rows: stat0 = 1 / sqrt(mean(x^2) + eps), the row split unshifted;
//   kSegW     weight rows: stat0 (if set) = the row sum (colsum of the transposed operand).
enum SegKind { kSegLn = 0, kSegRms = 1, kSegW = 2 };
struct SplitSeg {
  const float* src;
  float* hi;
  float* lo;
  float* stat0;
  float* stat1;
  int rows, K, Kp, kind;
};
constexpr int MAX_SEGS = 4;
struct SplitParams {
  SplitSeg seg[MAX_SEGS];
  int nseg, total_rows;
  float eps;
};

// One warp per row over the concatenated segments. A row is read once when it fits the
// registers (K <= 1024: 8 float4 per lane), else streamed twice (moments, split).
__global__ void __launch_bounds__(256) f32_split_kernel(const __grid_constant__ SplitParams p) {
  constexpr int R = 8;  // float4 per lane held in registers
  // the GEMM launch may start its prologue now; it waits for this grid before reading
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int warps = static_cast<int>(gridDim.x * blockDim.x / 32);
  for (int r = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) / 32); r < p.total_rows; r += warps) {
    int si = 0, rr = r;
    while (si + 1 < p.nseg && rr >= p.seg[si].rows) rr -= p.seg[si++].rows;
    const SplitSeg& sg = p.seg[si];
    const int K = sg.K;
    const bool vec = (K & 3) == 0;
    const float* src = sg.src + static_cast<size_t>(rr) * K;
    float4* hi = reinterpret_cast<float4*>(sg.hi + static_cast<size_t>(rr) * sg.Kp);
    float4* lo = reinterpret_cast<float4*>(sg.lo + static_cast<size_t>(rr) * sg.Kp);
    auto load4 = [&](int k4) -> float4 {  // columns [4 k4, 4 k4 + 4), zero past K
      const int k = 4 * k4;
      if (vec && k + 3 < K) return __ldg(reinterpret_cast<const float4*>(src) + k4);
      float e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) e[u] = k + u < K ? __ldg(src + k + u) : 0.f;
      return make_float4(e[0], e[1], e[2], e[3]);
    };
    const int n4 = sg.Kp / 4;
    const bool in_regs = n4 <= 32 * R;
    float4 v[R];
    if (in_regs) {
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = lane + 32 * i < n4 ? load4(lane + 32 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // LayerNorm rows: moments about the row's first element (no E[x^2] - mu^2 cancellation)
    const float piv = sg.kind == kSegLn ? __ldg(src) : 0.f;
    float s1 = 0.f, s2 = 0.f;
    auto acc = [&](float4 a, int k) {
      const float e[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u < K) {
          const float d = e[u] - piv;
          s1 += d;
          s2 = fmaf(d, d, s2);
        }
    };
    if (in_regs) {
#pragma unroll
      for (int i = 0; i < R; ++i) acc(v[i], 4 * (lane + 32 * i));
    } else {
      for (int k4 = lane; k4 < n4; k4 += 32) acc(load4(k4), 4 * k4);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      const float inv_k = 1.0f / static_cast<float>(K);
      if (sg.kind == kSegLn) {
        const float dm = s1 * inv_k;
        sg.stat0[rr] = 1.0f / sqrtf(s2 * inv_k - dm * dm + p.eps);
        sg.stat1[rr] = -dm;
      } else if (sg.kind == kSegRms) {
        sg.stat0[rr] = 1.0f / sqrtf(s2 * inv_k + p.eps);  // lowering.hpp:409-411
      } else if (sg.stat0 != nullptr) {
        sg.stat0[rr] = s1;
      }
    }
    // x - p: exact when the row sits far from zero (|mu| >> sigma), where centring on a rounded
    // fp32 mean is not
    auto split = [&](float4 a, int k4) {
      const float e[4] = {a.x, a.y, a.z, a.w};
      float h[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float x = 4 * k4 + u < K ? e[u] - piv : 0.f;
        h[u] = tf32_hi(x);
        l[u] = x - h[u];
      }
      hi[k4] = make_float4(h[0], h[1], h[2], h[3]);
      lo[k4] = make_float4(l[0], l[1], l[2], l[3]);
    };
    if (in_regs) {
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (lane + 32 * i < n4) split(v[i], lane + 32 * i);
    } else {
      for (int k4 = lane; k4 < n4; k4 += 32) split(load4(k4), k4);
    }
  }
}

// GEMM epilogues (one kernel template):
//   kLn     O = (acc + (p - mean) colsum(Yt)) * rstd                      (K2, rule R5)
//   kGate   h = silu(rstd * acc_W) * (rstd * acc_V), written as its TF32 split h_hi, h_lo
//           (the A operand of the down contraction)                       (K1, gate/up)
//   kPlain  O = acc                                                        (K1, down)
enum Mode { kLn = 0, kGate = 1, kPlain = 2 };

// BNT: output tile width. 128 everywhere; 256 for kLn/kPlain launches with enough tiles (one
// N = 256 MMA reads 12 KB of SMEM per 128 tensor cycles where two N = 128 MMAs read 16 KB, and
// these kernels are bound by SMEM bandwidth: DESIGN.md, K2 fp32).
template <int MODE, int BNT = 128>
struct GCfg {
  static constexpr int BN = BNT;
  static constexpr int B_BYTES = BNT * BK * 4;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((BNT >> 3) << 17) | ((BM >> 4) << 24);
  static constexpr int NB = MODE == kGate ? 2 : 1;  // B operands sharing the A tile
  static constexpr int STAGE_BYTES = 2 * A_BYTES + NB * 2 * B_BYTES;
  static constexpr int STAGES = STAGE_BYTES > 64 * 1024 ? 2 : 3;
  // even and odd K steps accumulate into separate sets (added in the epilogue): the tensor
  // core's accumulation is not round-to-nearest, and halving each chain keeps K1's fp32 mode
  // (two chained contractions) clear of the 1e-4 bar
  static constexpr int SET = NB * BN;
  static constexpr uint32_t TMEM_COLS = 2 * SET;
  static constexpr int RED_PITCH = NB * (BN / 2) * 4 + 16;  // pushed-half row pitch (bytes): rows on distinct banks
  static_assert(BM * RED_PITCH <= STAGES * STAGE_BYTES, "reduction buffer reuses the operand ring");
  static constexpr int SMEM = STAGES * STAGE_BYTES + 256;
  static_assert(SMEM <= 232448, "3xTF32 GEMM SMEM budget");
};

struct GemmParams {
  int M, N, kt;     // N: output columns written (kGate: the padded F of the down contraction)
  int Mt, Nt, group;  // tile raster: groups of `group` m-tiles, n slow inside a group
  int ldo;
  const float* rstd;
  const float* negdm;
  const float* colsum;
  float* O;   // kGate: h_hi
  float* O2;  // kGate: h_lo
};

template <int MODE, int BNT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    f32x3_gemm_kernel(const __grid_constant__ CUtensorMap tm_xh, const __grid_constant__ CUtensorMap tm_xl,
                      const __grid_constant__ CUtensorMap tm_yh, const __grid_constant__ CUtensorMap tm_yl,
                      const __grid_constant__ CUtensorMap tm_vh, const __grid_constant__ CUtensorMap tm_vl,
                      const GemmParams p) {
  using namespace dev;
  using C = GCfg<MODE, BNT>;
  constexpr int BN = C::BN, B_BYTES = C::B_BYTES;  // this instantiation's tile width
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // which half of K this CTA contracts
  // grouped raster: the A rows of `group` m-tiles stay in L2 while their n-tiles pass
  const int t = static_cast<int>(blockIdx.x >> 1);
  const int per_group = p.group * p.Nt, g = t / per_group, in_g = t % per_group;
  const int gm = min(p.group, p.Mt - g * p.group);
  const int m0 = (g * p.group + in_g % gm) * BM, n0 = (in_g / gm) * BN;
  const int khalf = (p.kt + 1) / 2;
  const int k_begin = rank == 0 ? 0 : khalf, k_end = rank == 0 ? khalf : p.kt;
  const int nk = k_end - k_begin;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_xh);
    tma_prefetch_desc(&tm_xl);
    tma_prefetch_desc(&tm_yh);
    tma_prefetch_desc(&tm_yl);
    if constexpr (C::NB == 2) {
      tma_prefetch_desc(&tm_vh);
      tma_prefetch_desc(&tm_vl);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: everything above overlapped the previous launch; its
  // outputs (split operands, statistics, colsum, h) are read only after it has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % C::STAGES, k = k_begin + i;
        mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        tma_load_2d(&tm_xh, &full[s], st, k * BK, m0);
        tma_load_2d(&tm_xl, &full[s], st + A_BYTES, k * BK, m0);
        tma_load_2d(&tm_yh, &full[s], st + 2 * A_BYTES, k * BK, n0);
        tma_load_2d(&tm_yl, &full[s], st + 2 * A_BYTES + B_BYTES, k * BK, n0);
        if constexpr (C::NB == 2) {
          tma_load_2d(&tm_vh, &full[s], st + 2 * A_BYTES + 2 * B_BYTES, k * BK, n0);
          tma_load_2d(&tm_vl, &full[s], st + 2 * A_BYTES + 3 * B_BYTES, k * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    for (int i = 0; i < nk; ++i) {
      const int s = i % C::STAGES;
      mbar_wait(&full[s], (i / C::STAGES) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t xh = smem_u32(smem + s * C::STAGE_BYTES), xl = xh + A_BYTES;
#pragma unroll
        for (int b = 0; b < C::NB; ++b) {
          const uint32_t yh = xh + 2 * A_BYTES + 2 * b * B_BYTES, yl = yh + B_BYTES,
                         d = tmem + (i & 1) * C::SET + b * BN;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {  // K = 8 tf32 = 32 bytes per MMA
#ifdef BF_F32X3_DBG_NOMMA  // timing only: the load pipeline alone
            if (i > 0) continue;
#endif
            const uint32_t o = kk * 32;
            // small terms first: lo*hi, hi*lo, then hi*hi
            umma_tf32_ss(d, sdesc_kmajor_sw128(xl + o), sdesc_kmajor_sw128(yh + o), (i >= 2 || kk != 0), C::IDESC);
            umma_tf32_ss(d, sdesc_kmajor_sw128(xh + o), sdesc_kmajor_sw128(yl + o), 1, C::IDESC);
            umma_tf32_ss(d, sdesc_kmajor_sw128(xh + o), sdesc_kmajor_sw128(yh + o), 1, C::IDESC);
          }
        }
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(tfull);  // nk == 0 (K <= 32 on rank 1): arrives at once, acc unused
    __syncwarp();
  }
  // Epilogue, split by columns over the pair: rank r finalizes columns [64 r, 64 r + 64) of the
  // tile. Each rank pushes its partial sums of the other half into the peer's SMEM (remote
  // stores: no round-trip latency exposed), then adds the peer's pushed half to its own TMEM
  // half in a fixed order (deterministic). The rings are free once both pairs' MMAs are done.
  constexpr int HALF = BN / 2, CH = HALF / 32;  // columns per rank, 32-column chunks per half
  const uint32_t q = warp & 3;
  const uint32_t trow = q * 32 + lane;
  const uint32_t tl = tmem + ((q * 32) << 16);
  uint8_t* red = smem + trow * C::RED_PITCH;  // [C::NB][HALF] floats per row
  if (warp >= 4) {
    mbar_wait(tfull, 0);
    tc_fence_after();
  }
  tc_fence_before();
  cluster_sync();  // A: both CTAs' accumulators are final and their operand rings idle
  if (warp >= 4) {
    const uint32_t dst = mapa_shared(smem_u32(red), rank ^ 1);
#pragma unroll 1
    for (int c = 0; c < C::NB * CH; ++c) {  // (operand b, 32-column chunk) of the peer's half
      const int b = c / CH, col = b * BN + static_cast<int>(rank ^ 1) * HALF + (c % CH) * 32;
      uint32_t v[32], v2[32];
      tmem_ld_32x32b_x32(tl + col, v);
      tmem_ld_32x32b_x32(tl + C::SET + col, v2);
      tmem_wait_ld();
      const bool two = nk > 1;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float e[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          e[u] = nk == 0 ? 0.f
                         : (two ? __uint_as_float(v[4 * i + u]) + __uint_as_float(v2[4 * i + u])
                                : __uint_as_float(v[4 * i + u]));
        const float4 f = make_float4(e[0], e[1], e[2], e[3]);
        st_cluster_v4(dst + (b * HALF + (c % CH) * 32 + 4 * i) * 4, f);
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // B: the pushed halves are visible; no remote access after this point
  if (warp >= 4) {
    tc_fence_after();
    const int row = m0 + static_cast<int>(trow);
    float r = 0.f, nd = 0.f;
    if constexpr (MODE != kPlain) r = row < p.M ? __ldg(p.rstd + row) : 0.f;
    if constexpr (MODE == kLn) nd = row < p.M ? __ldg(p.negdm + row) : 0.f;
    const bool vec = (p.N & 3) == 0 && (p.ldo & 3) == 0;
    const float4* pushed = reinterpret_cast<const float4*>(red);
#ifdef BF_F32X3_DBG_NOEPI  // timing only: no reduction or stores
    if (p.M > 0) goto epi_done;
#endif
#pragma unroll 1
    for (int c = 0; c < CH; ++c) {
      const int cbase = static_cast<int>(rank) * HALF + c * 32;  // tile column of this chunk
      uint32_t v[32], v2[32];
      tmem_ld_32x32b_x32(tl + cbase, v);
      tmem_ld_32x32b_x32(tl + C::SET + cbase, v2);
      uint32_t w[32], w2[32];
      if constexpr (C::NB == 2) {
        tmem_ld_32x32b_x32(tl + BN + cbase, w);
        tmem_ld_32x32b_x32(tl + C::SET + BN + cbase, w2);
      }
      tmem_wait_ld();
      if (row >= p.M) continue;
      const bool own = nk > 0;
      if (nk > 1) {  // fold the odd-step set into the even one (round-to-nearest fp32 adds)
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          v[u] = __float_as_uint(__uint_as_float(v[u]) + __uint_as_float(v2[u]));
          if constexpr (C::NB == 2) w[u] = __float_as_uint(__uint_as_float(w[u]) + __uint_as_float(w2[u]));
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int col = n0 + cbase + 4 * i;
        const float4 o1 = pushed[(c * 32 + 4 * i) / 4];
        float a[4] = {o1.x, o1.y, o1.z, o1.w};
        if (own) {
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] = __uint_as_float(v[4 * i + u]) + a[u];
        }
        float o[4], lo[4];
        if constexpr (MODE == kGate) {
          const float4 o2 = pushed[(HALF + c * 32 + 4 * i) / 4];
          float bb[4] = {o2.x, o2.y, o2.z, o2.w};
          if (own) {
#pragma unroll
            for (int u = 0; u < 4; ++u) bb[u] = __uint_as_float(w[4 * i + u]) + bb[u];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float gt = a[u] * r;
            const float h = col + u < p.N ? gt / (1.0f + expf(-gt)) * (bb[u] * r) : 0.f;
            o[u] = tf32_hi(h);
            lo[u] = h - o[u];
          }
        } else if constexpr (MODE == kLn) {
#pragma unroll
          for (int u = 0; u < 4; ++u) o[u] = col + u < p.N ? fmaf(nd, __ldg(p.colsum + col + u), a[u]) * r : 0.f;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) o[u] = a[u];
        }
        // stage in place (this thread's own row of the pushed buffer) for coalesced stores
        float4* st = reinterpret_cast<float4*>(red) + (c * 32 + 4 * i) / 4;
        st[0] = make_float4(o[0], o[1], o[2], o[3]);
        if constexpr (MODE == kGate) st[HALF / 4] = make_float4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    __syncwarp();
    // the warp's 32 rows x HALF columns, RPI rows per instruction (HALF * 4 contiguous bytes each)
    constexpr int LPR = HALF / 4, RPI = 32 / LPR;  // lanes per row, rows per instruction
#pragma unroll 4
    for (int k = 0; k < 32 / RPI; ++k) {
      const int cc = (static_cast<int>(lane) % LPR) * 4, col = n0 + static_cast<int>(rank) * HALF + cc;
      const int rl = RPI * k + static_cast<int>(lane) / LPR, row2 = m0 + static_cast<int>(q) * 32 + rl;
      if (row2 >= p.M) break;
      const uint8_t* srow = smem + (q * 32 + rl) * C::RED_PITCH;
      const float4 val = *reinterpret_cast<const float4*>(srow + cc * 4);
      float* out = p.O + static_cast<size_t>(row2) * p.ldo + col;
      float4 lv;
      if constexpr (MODE == kGate) lv = *reinterpret_cast<const float4*>(srow + (HALF + cc) * 4);
      if (vec && col + 3 < p.N) {
        *reinterpret_cast<float4*>(out) = val;
        if constexpr (MODE == kGate) *reinterpret_cast<float4*>(p.O2 + static_cast<size_t>(row2) * p.ldo + col) = lv;
      } else {
        const float e[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (col + u < p.N) {
            out[u] = e[u];
            if constexpr (MODE == kGate) {
              const float l4[4] = {lv.x, lv.y, lv.z, lv.w};
              p.O2[static_cast<size_t>(row2) * p.ldo + col + u] = l4[u];
            }
          }
      }
    }
#ifdef BF_F32X3_DBG_NOEPI
  epi_done:;
#endif
  }
  tc_fence_before();
  __syncthreads();  // TMEM reads done before the free
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant for large launches: 256 x 256 output tiles, M = 256 cta_group::2 MMAs
// issued by the pair leader. Each CTA stages its own 128 rows of A and 128 rows of B (hi and
// lo), so per K step a CTA writes 64 KB and its SMEM serves 96 KB to the MMAs for 4x the
// FLOPs of a 128 x 128 step (which moves 160 KB): the pair kernel is no longer bound by SMEM
// bandwidth. No K split: each CTA finalizes its own 128 rows x 256 columns. Even and odd K
// steps accumulate into two TMEM accumulators (512 columns), added once in the epilogue: the
// tensor core's accumulation is not round-to-nearest fp32, and one accumulator over K = 14336
// (K1's down GEMM at C3) measured 1.46e-4 against float64, over the 1e-4 bar; two halve the
// chain, as the K split of the single-CTA kernel does.
constexpr int P2_BN = 256, P2_STAGES = 3;
constexpr int P2_STAGE_BYTES = 2 * A_BYTES + 2 * (128 * BK * 4);  // X_hi | X_lo | Y_hi | Y_lo (this CTA's halves)
constexpr int P2_OUT_PITCH = P2_BN * 4 + 16;
static_assert(BM * P2_OUT_PITCH <= P2_STAGES * P2_STAGE_BYTES, "output staging reuses the operand ring");
constexpr int P2_SMEM = P2_STAGES * P2_STAGE_BYTES + 256;
constexpr uint32_t P2_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((P2_BN >> 3) << 17) | ((256 >> 4) << 24);

__device__ __forceinline__ void umma_tf32_ss_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(P2_IDESC), "r"(accumulate)
      : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    f32x3_pair_kernel(const __grid_constant__ CUtensorMap tm_xh, const __grid_constant__ CUtensorMap tm_xl,
                      const __grid_constant__ CUtensorMap tm_yh, const __grid_constant__ CUtensorMap tm_yl,
                      const GemmParams p) {
  static_assert(MODE == kLn || MODE == kPlain, "pair kernel epilogues");
  using namespace dev;
  constexpr int Y_BYTES = 128 * BK * 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P2_STAGES * P2_STAGE_BYTES);
  uint64_t* empty = full + P2_STAGES;
  uint64_t* tfull = empty + P2_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // grouped raster over 256 x 256 tiles
  const int t = static_cast<int>(blockIdx.x >> 1);
  const int per_group = p.group * p.Nt, g = t / per_group, in_g = t % per_group;
  const int gm = min(p.group, p.Mt - g * p.group);
  const int m0 = (g * p.group + in_g % gm) * 256, n0 = (in_g / gm) * P2_BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_xh);
    tma_prefetch_desc(&tm_xl);
    tma_prefetch_desc(&tm_yh);
    tma_prefetch_desc(&tm_yl);
    for (int s = 0; s < P2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<2 * P2_BN>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
      const int arow = m0 + static_cast<int>(rank) * 128, brow = n0 + static_cast<int>(rank) * 128;
      for (int i = 0; i < p.kt; ++i) {
        const int s = i % P2_STAGES;
        mbar_wait(&empty[s], ((i / P2_STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * P2_STAGE_BYTES;
        const uint32_t fbar = full0 + s * 8;
        if (leader) mbar_arrive_expect_tx(&full[s], 2 * P2_STAGE_BYTES);
        tma_load_2d_2sm(&tm_xh, fbar, st, i * BK, arow);
        tma_load_2d_2sm(&tm_xl, fbar, st + A_BYTES, i * BK, arow);
        tma_load_2d_2sm(&tm_yh, fbar, st + 2 * A_BYTES, i * BK, brow);
        tma_load_2d_2sm(&tm_yl, fbar, st + 2 * A_BYTES + Y_BYTES, i * BK, brow);
      }
    }
  } else if (warp == 1) {
    if (leader) {
      for (int i = 0; i < p.kt; ++i) {
        const int s = i % P2_STAGES;
        mbar_wait(&full[s], (i / P2_STAGES) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t xh = smem_u32(smem + s * P2_STAGE_BYTES), xl = xh + A_BYTES, yh = xh + 2 * A_BYTES,
                         yl = yh + Y_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t o = kk * 32;
            const uint32_t d = tmem + (i & 1) * P2_BN;  // even / odd K steps
            umma_tf32_ss_2sm(d, sdesc_kmajor_sw128(xl + o), sdesc_kmajor_sw128(yh + o), (i >= 2 || kk != 0));
            umma_tf32_ss_2sm(d, sdesc_kmajor_sw128(xh + o), sdesc_kmajor_sw128(yl + o), 1);
            umma_tf32_ss_2sm(d, sdesc_kmajor_sw128(xh + o), sdesc_kmajor_sw128(yh + o), 1);
          }
          umma_commit_2sm_mc(&empty[s], 0x3);
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit_2sm_mc(tfull, 0x3);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---- epilogue: this CTA's 128 rows x 256 columns, staged in the idle ring, stored coalesced
    const uint32_t q = warp & 3;
    const uint32_t trow = q * 32 + lane;
    const uint32_t tl = tmem + ((q * 32) << 16);
    const int row = m0 + static_cast<int>(rank) * 128 + static_cast<int>(trow);
    float r = 1.f, nd = 0.f;
    if constexpr (MODE == kLn) {
      r = row < p.M ? __ldg(p.rstd + row) : 0.f;
      nd = row < p.M ? __ldg(p.negdm + row) : 0.f;
    }
    mbar_wait(tfull, 0);  // all MMAs of the pair done: both operand rings are idle
    tc_fence_after();
    float4* srow = reinterpret_cast<float4*>(smem + trow * P2_OUT_PITCH);
#pragma unroll 1
    for (int c = 0; c < P2_BN / 32; ++c) {
      uint32_t v[32], w[32];
      tmem_ld_32x32b_x32(tl + c * 32, v);
      tmem_ld_32x32b_x32(tl + P2_BN + c * 32, w);
      tmem_wait_ld();
      const bool two = p.kt > 1;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float a = two ? __uint_as_float(v[4 * i + u]) + __uint_as_float(w[4 * i + u])
                              : __uint_as_float(v[4 * i + u]);
          if constexpr (MODE == kLn) {
            const int col = n0 + c * 32 + 4 * i + u;
            o[u] = col < p.N ? fmaf(nd, __ldg(p.colsum + col), a) * r : 0.f;
          } else {
            o[u] = a;
          }
        }
        srow[c * 8 + i] = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    __syncwarp();
    const bool vec = (p.N & 3) == 0 && (p.ldo & 3) == 0;
    const int rbase = m0 + static_cast<int>(rank) * 128 + static_cast<int>(q) * 32;
#pragma unroll 4
    for (int k = 0; k < 64; ++k) {  // 32 rows x 2 halves of 128 columns, 512 contiguous bytes each
      const int rl = k >> 1, row2 = rbase + rl;
      if (row2 >= p.M) break;
      const int cc = (k & 1) * 128 + static_cast<int>(lane) * 4, col = n0 + cc;
      const float4 val = *reinterpret_cast<const float4*>(smem + (q * 32 + rl) * P2_OUT_PITCH + cc * 4);
      float* out = p.O + static_cast<size_t>(row2) * p.ldo + col;
      if (vec && col + 3 < p.N) {
        *reinterpret_cast<float4*>(out) = val;
      } else {
        const float e[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (col + u < p.N) out[u] = e[u];
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // the leader's MMAs read this CTA's SMEM: keep both alive until the end
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<2 * P2_BN>(tmem);
  }
}

// K1's gate/up GEMM on CTA pairs: 256 x 128 tiles per B operand (W and V share the A tile),
// M = 256 MMAs with N = 128 (each CTA stages 64 rows of W and of V), even and odd K steps in
// separate accumulator sets: W | V | W' | V' = 512 TMEM columns. Per CTA and K step: 64 KB
// written by TMA and 144 KB read by the MMAs for twice the FLOPs of a 128 x 128 step.
constexpr int PG_BN = 128;                      // output columns per operand per pair tile
constexpr int PG_Y_BYTES = (PG_BN / 2) * BK * 4;  // this CTA's 64 rows of one operand slab
constexpr int PG_STAGES = 3;
constexpr int PG_STAGE_BYTES = 2 * A_BYTES + 4 * PG_Y_BYTES;  // X_hi | X_lo | W_hi | W_lo | V_hi | V_lo
constexpr int PG_OUT_PITCH = PG_BN * 4 + 16;
static_assert(2 * BM * PG_OUT_PITCH <= PG_STAGES * PG_STAGE_BYTES, "h_hi/h_lo staging reuses the operand ring");
constexpr int PG_SMEM = PG_STAGES * PG_STAGE_BYTES + 256;
constexpr uint32_t PG_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((PG_BN >> 3) << 17) | ((256 >> 4) << 24);

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    f32x3_pair_gate_kernel(const __grid_constant__ CUtensorMap tm_xh, const __grid_constant__ CUtensorMap tm_xl,
                           const __grid_constant__ CUtensorMap tm_wh, const __grid_constant__ CUtensorMap tm_wl,
                           const __grid_constant__ CUtensorMap tm_vh, const __grid_constant__ CUtensorMap tm_vl,
                           const GemmParams p) {
  using namespace dev;
  constexpr int SET = 2 * PG_BN;  // W | V
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PG_STAGES * PG_STAGE_BYTES);
  uint64_t* empty = full + PG_STAGES;
  uint64_t* tfull = empty + PG_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int t = static_cast<int>(blockIdx.x >> 1);
  const int per_group = p.group * p.Nt, g = t / per_group, in_g = t % per_group;
  const int gm = min(p.group, p.Mt - g * p.group);
  const int m0 = (g * p.group + in_g % gm) * 256, n0 = (in_g / gm) * PG_BN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_xh);
    tma_prefetch_desc(&tm_xl);
    tma_prefetch_desc(&tm_wh);
    tma_prefetch_desc(&tm_wl);
    tma_prefetch_desc(&tm_vh);
    tma_prefetch_desc(&tm_vl);
    for (int s = 0; s < PG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2sm<2 * SET>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(&full[0]), 0);
      const int arow = m0 + static_cast<int>(rank) * 128, brow = n0 + static_cast<int>(rank) * (PG_BN / 2);
      for (int i = 0; i < p.kt; ++i) {
        const int s = i % PG_STAGES;
        mbar_wait(&empty[s], ((i / PG_STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * PG_STAGE_BYTES;
        const uint32_t fbar = full0 + s * 8;
        if (leader) mbar_arrive_expect_tx(&full[s], 2 * PG_STAGE_BYTES);
        tma_load_2d_2sm(&tm_xh, fbar, st, i * BK, arow);
        tma_load_2d_2sm(&tm_xl, fbar, st + A_BYTES, i * BK, arow);
        tma_load_2d_2sm(&tm_wh, fbar, st + 2 * A_BYTES, i * BK, brow);
        tma_load_2d_2sm(&tm_wl, fbar, st + 2 * A_BYTES + PG_Y_BYTES, i * BK, brow);
        tma_load_2d_2sm(&tm_vh, fbar, st + 2 * A_BYTES + 2 * PG_Y_BYTES, i * BK, brow);
        tma_load_2d_2sm(&tm_vl, fbar, st + 2 * A_BYTES + 3 * PG_Y_BYTES, i * BK, brow);
      }
    }
  } else if (warp == 1) {
    if (leader) {
      for (int i = 0; i < p.kt; ++i) {
        const int s = i % PG_STAGES;
        mbar_wait(&full[s], (i / PG_STAGES) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t xh = smem_u32(smem + s * PG_STAGE_BYTES), xl = xh + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t o = kk * 32;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const uint32_t bh = xh + 2 * A_BYTES + 2 * b * PG_Y_BYTES, bl = bh + PG_Y_BYTES;
              const uint32_t d = tmem + (i & 1) * SET + b * PG_BN;
              asm volatile(
                  "{\n.reg .pred p;\n"
                  "setp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
                  "tcgen05.mma.cta_group::2.kind::tf32 [%0], %5, %6, %3, 1;\n"
                  "tcgen05.mma.cta_group::2.kind::tf32 [%0], %5, %2, %3, 1;\n}" ::"r"(d),
                  "l"(sdesc_kmajor_sw128(xl + o)), "l"(sdesc_kmajor_sw128(bh + o)), "r"(PG_IDESC),
                  "r"(static_cast<uint32_t>(i >= 2 || kk != 0)), "l"(sdesc_kmajor_sw128(xh + o)),
                  "l"(sdesc_kmajor_sw128(bl + o))
                  : "memory");
            }
          }
          umma_commit_2sm_mc(&empty[s], 0x3);
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit_2sm_mc(tfull, 0x3);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---- epilogue: h = silu(r a) (r b) for this CTA's 128 rows x 128 columns, as h_hi and h_lo
    const uint32_t q = warp & 3;
    const uint32_t trow = q * 32 + lane;
    const uint32_t tl = tmem + ((q * 32) << 16);
    const int row = m0 + static_cast<int>(rank) * 128 + static_cast<int>(trow);
    const float rr = row < p.M ? __ldg(p.rstd + row) : 0.f;
    mbar_wait(tfull, 0);  // all MMAs of the pair done: both operand rings are idle
    tc_fence_after();
    float4* shi = reinterpret_cast<float4*>(smem + trow * PG_OUT_PITCH);
    float4* slo = reinterpret_cast<float4*>(smem + BM * PG_OUT_PITCH + trow * PG_OUT_PITCH);
    const bool two = p.kt > 1;
#pragma unroll 1
    for (int c = 0; c < PG_BN / 32; ++c) {
      uint32_t a0[32], a1[32], b0[32], b1[32];
      tmem_ld_32x32b_x32(tl + c * 32, a0);
      tmem_ld_32x32b_x32(tl + SET + c * 32, a1);
      tmem_ld_32x32b_x32(tl + PG_BN + c * 32, b0);
      tmem_ld_32x32b_x32(tl + SET + PG_BN + c * 32, b1);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float hi[4], lo[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = 4 * i + u, col = n0 + c * 32 + e;
          const float a = two ? __uint_as_float(a0[e]) + __uint_as_float(a1[e]) : __uint_as_float(a0[e]);
          const float b = two ? __uint_as_float(b0[e]) + __uint_as_float(b1[e]) : __uint_as_float(b0[e]);
          const float gt = a * rr;
          const float h = col < p.N ? gt / (1.0f + expf(-gt)) * (b * rr) : 0.f;
          hi[u] = tf32_hi(h);
          lo[u] = h - hi[u];
        }
        shi[c * 8 + i] = make_float4(hi[0], hi[1], hi[2], hi[3]);
        slo[c * 8 + i] = make_float4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
    __syncwarp();
    const bool vec = (p.ldo & 3) == 0;
    const int rbase = m0 + static_cast<int>(rank) * 128 + static_cast<int>(q) * 32;
#pragma unroll 4
    for (int rl = 0; rl < 32; ++rl) {  // one 512-byte row segment per instruction and output
      const int row2 = rbase + rl;
      if (row2 >= p.M) break;
      const int col = n0 + static_cast<int>(lane) * 4;
      const uint8_t* sr = smem + (q * 32 + rl) * PG_OUT_PITCH + lane * 16;
      const float4 vh = *reinterpret_cast<const float4*>(sr);
      const float4 vl = *reinterpret_cast<const float4*>(sr + BM * PG_OUT_PITCH);
      float* oh = p.O + static_cast<size_t>(row2) * p.ldo + col;
      float* ol = p.O2 + static_cast<size_t>(row2) * p.ldo + col;
      if (vec && col + 3 < p.N) {
        *reinterpret_cast<float4*>(oh) = vh;
        *reinterpret_cast<float4*>(ol) = vl;
      } else {
        const float eh[4] = {vh.x, vh.y, vh.z, vh.w}, el[4] = {vl.x, vl.y, vl.z, vl.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (col + u < p.N) {
            oh[u] = eh[u];
            ol[u] = el[u];
          }
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // the leader's MMAs read this CTA's SMEM: keep both alive until the end
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm<2 * SET>(tmem);
  }
}

int64_t padded_k(int64_t K) { return (K + BK - 1) / BK * BK; }

// Tile raster group (m-tiles per group, n slow inside a group): the largest power of two whose
// hi/lo A rows (128 x Kp x 8 bytes each) fit a third of L2, but at least 8. For long
// contractions (K1's down GEMM, Kp = 14336) the slab never fits, and what matters is the shape
// of one wave of 74 CTA pairs: 8 m-tiles x ~9 n-tiles read 17 operand stripes per wave where
// 2 x 37 read 39 (16.4 -> ~7 GB of DRAM per launch at C3, ncu).
int raster_group(int64_t Mt, int64_t Kp, int64_t l2_bytes) {
  const int64_t fit = std::max<int64_t>(1, l2_bytes / 3 / (static_cast<int64_t>(BM) * Kp * 8));
  int g = 1;
  while (2 * g <= std::max<int64_t>(fit, 8) && 2 * g <= Mt) g *= 2;
  if (const char* e = std::getenv("BFGPU_F32_GROUP")) g = std::max(1, std::atoi(e));
  return g;
}

template <int MODE, int BNT = 128>
void launch_gemm(const CUtensorMap (&tm)[6], const GemmParams& gp, cudaStream_t stream) {
  using C = GCfg<MODE, BNT>;
  ensure_smem_attr(reinterpret_cast<const void*>(&f32x3_gemm_kernel<MODE, BNT>), C::SMEM);
  const int64_t tiles = static_cast<int64_t>(gp.Mt) * gp.Nt;
  BF_CHECK_ARG(2 * tiles < (1ll << 31), "fp32 mode: too many output tiles for one launch");
  // launched as a programmatic dependent of the previous launch (griddepcontrol in both)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * tiles));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, f32x3_gemm_kernel<MODE, BNT>, tm[0], tm[1], tm[2], tm[3], tm[4], tm[5], gp));
  note_launch();
}

template <int MODE>
void launch_pair(const CUtensorMap (&tm)[6], const GemmParams& gp, cudaStream_t stream) {
  ensure_smem_attr(reinterpret_cast<const void*>(&f32x3_pair_kernel<MODE>), P2_SMEM);
  const int64_t tiles = static_cast<int64_t>(gp.Mt) * gp.Nt;
  BF_CHECK_ARG(2 * tiles < (1ll << 31), "fp32 mode: too many output tiles for one launch");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * tiles));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = P2_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, f32x3_pair_kernel<MODE>, tm[0], tm[1], tm[2], tm[3], gp));
  note_launch();
}

void launch_pair_gate(const CUtensorMap (&tm)[6], const GemmParams& gp, cudaStream_t stream) {
  ensure_smem_attr(reinterpret_cast<const void*>(&f32x3_pair_gate_kernel), PG_SMEM);
  const int64_t tiles = static_cast<int64_t>(gp.Mt) * gp.Nt;
  BF_CHECK_ARG(2 * tiles < (1ll << 31), "fp32 mode: too many output tiles for one launch");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * tiles));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = PG_SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, f32x3_pair_gate_kernel, tm[0], tm[1], tm[2], tm[3], tm[4], tm[5], gp));
  note_launch();
}

void launch_split(const SplitParams& sp, int sms, cudaStream_t stream) {
  const int split_grid = static_cast<int>(std::min<int64_t>((sp.total_rows + 7) / 8, static_cast<int64_t>(sms) * 16));
  f32_split_kernel<<<split_grid, 256, 0, stream>>>(sp);
  BF_CUDA(cudaGetLastError());
  note_launch();
}

CUtensorMap tmap(const float* base, int64_t rows, int64_t Kp, int box_rows) {
  return make_tmap_2d(base, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, rows, Kp, Kp, BK, box_rows);
}

// Carves consecutive 1024-byte aligned buffers out of the workspace.
struct Carve {
  uint8_t* w;
  size_t used = 0;
  float* take(size_t floats) {
    float* r = reinterpret_cast<float*>(w + used);
    used += align_up(floats * 4, 1024);
    return r;
  }
};

}  // namespace f32x3

size_t lnmm_f32x3_workspace_bytes(int64_t M, int64_t K, int64_t N) {
  const size_t kp = static_cast<size_t>(f32x3::padded_k(K));
  return 2 * align_up(static_cast<size_t>(M) * kp * 4, 1024) + 2 * align_up(static_cast<size_t>(N) * kp * 4, 1024) +
         2 * align_up(static_cast<size_t>(M) * 4, 1024) + align_up(static_cast<size_t>(N) * 4, 1024);
}

size_t ffn_f32x3_workspace_bytes(int64_t M, int64_t D, int64_t F, int64_t N) {
  const size_t dp = static_cast<size_t>(f32x3::padded_k(D)), fp = static_cast<size_t>(f32x3::padded_k(F));
  auto a = [](size_t floats) { return align_up(floats * 4, 1024); };
  return 2 * a(M * dp) + 4 * a(F * dp) + 2 * a(N * fp) + 2 * a(M * fp) + a(M);
}

// 256 x 256 CTA-pair tiles (M = 256 MMAs, no K split) when there are at least two waves of
// them; BFGPU_F32_PAIR=0/1 forces.
bool f32x3_pair(int64_t M, int64_t N) {
  if (const char* e = std::getenv("BFGPU_F32_PAIR")) return std::atoi(e) == 1;
  return ((M + 255) / 256) * ((N + 255) / 256) >= 148;
}

// K1 fp32 on the CTA-pair kernels (gate/up: 256 x 128 tiles per operand; down: 256 x 256) is
// opt-in, BFGPU_F32_K1_PAIR=1. It is faster (C3: 11.4 vs 13.7 ms) but the pair kernels have no
// K split, so each accumulator chain is twice as long, and the two chained contractions land
// at 7.4e-5 of the 1e-4 bar instead of 3.7e-5 (fp32 modes).
bool f32x3_k1_pair() {
  const char* e = std::getenv("BFGPU_F32_K1_PAIR");
  return e != nullptr && std::atoi(e) == 1;
}

// BFGPU_F32_PAIR=1 (force the pair kernels) also drops the size threshold here.
static bool f32x3_pair_forced() {
  const char* e = std::getenv("BFGPU_F32_PAIR");
  return e != nullptr && std::atoi(e) == 1;
}

bool f32x3_pair_gate(int64_t M, int64_t F) {
  return f32x3_k1_pair() && (f32x3_pair_forced() || ((M + 255) / 256) * ((F + 127) / 128) >= 148);
}

KernelSpec f32x3_pair_gate_spec() {
  using namespace f32x3;
  KernelSpec k;
  k.name = "f32x3_pair_gate_kernel";
  k.func = reinterpret_cast<const void*>(&f32x3_pair_gate_kernel);
  k.threads = NUM_THREADS;
  k.cluster = 2;
  k.tile_m = 256;
  k.tile_n = PG_BN;
  k.tile_k = BK;
  k.smem_bytes = PG_SMEM;
  k.tmem_cols = 512;
  k.stages = PG_STAGES;
  k.grid_sync = false;
  return k;
}

// 128 x 256 tiles when there are enough of them: at least one per SM (CTA pairs x 2).
bool f32x3_wide(int64_t M, int64_t N) {
  if (const char* e = std::getenv("BFGPU_F32_BN")) return std::atoi(e) == 256;
  return ((M + f32x3::BM - 1) / f32x3::BM) * ((N + 255) / 256) >= 148;
}

KernelSpec f32x3_pair_spec(int mode) {
  using namespace f32x3;
  KernelSpec k;
  k.name = mode == kPlain ? "f32x3_pair_kernel<plain>" : "f32x3_pair_kernel<ln>";
  k.func = mode == kPlain ? reinterpret_cast<const void*>(&f32x3_pair_kernel<kPlain>)
                          : reinterpret_cast<const void*>(&f32x3_pair_kernel<kLn>);
  k.threads = NUM_THREADS;
  k.cluster = 2;  // M = 256 cta_group::2 MMAs
  k.tile_m = 256;
  k.tile_n = P2_BN;
  k.tile_k = BK;
  k.smem_bytes = P2_SMEM;
  k.tmem_cols = 2 * P2_BN;
  k.stages = P2_STAGES;
  k.grid_sync = false;
  return k;
}

KernelSpec f32x3_gemm_spec(int mode, bool wide) {
  using namespace f32x3;
  KernelSpec k;
  k.threads = NUM_THREADS;
  k.cluster = 2;  // the K range of a tile split over a CTA pair
  k.tile_m = BM;
  k.tile_n = BN;
  k.tile_k = BK;
  k.grid_sync = false;
  auto fill = [&](auto cfg, const void* func) {
    using C = decltype(cfg);
    k.func = func;
    k.smem_bytes = C::SMEM;
    k.tmem_cols = C::TMEM_COLS;
    k.stages = C::STAGES;
  };
  if (mode == kGate) {
    k.name = "f32x3_gemm_kernel<gate>";
    fill(GCfg<kGate>{}, reinterpret_cast<const void*>(&f32x3_gemm_kernel<kGate, 128>));
  } else if (mode == kPlain && wide) {
    k.name = "f32x3_gemm_kernel<plain,256>";
    fill(GCfg<kPlain, 256>{}, reinterpret_cast<const void*>(&f32x3_gemm_kernel<kPlain, 256>));
  } else if (mode == kPlain) {
    k.name = "f32x3_gemm_kernel<plain>";
    fill(GCfg<kPlain>{}, reinterpret_cast<const void*>(&f32x3_gemm_kernel<kPlain, 128>));
  } else if (wide) {
    k.name = "f32x3_gemm_kernel<ln,256>";
    fill(GCfg<kLn, 256>{}, reinterpret_cast<const void*>(&f32x3_gemm_kernel<kLn, 256>));
  } else {
    k.name = "f32x3_gemm_kernel";
    fill(GCfg<kLn>{}, reinterpret_cast<const void*>(&f32x3_gemm_kernel<kLn, 128>));
  }
  if (wide && mode != kGate) k.tile_n = 256;
  return k;
}

void lnmm_f32x3(const Plan& pl, const void* X, const void* Yt, void* O, float eps, void* ws, size_t ws_bytes,
                cudaStream_t stream) {
  using namespace f32x3;
  const int64_t M = pl.dims[0], K = pl.dims[1], N = pl.dims[2];
  const int64_t Kp = padded_k(K);
  BF_CHECK_ARG(ws != nullptr && ws_bytes >= lnmm_f32x3_workspace_bytes(M, K, N),
               "bf_layernorm_matmul: workspace too small");
  BF_CHECK_ARG((reinterpret_cast<uintptr_t>(ws) & 15u) == 0, "bf_layernorm_matmul: workspace must be 16-byte aligned");
  BF_CHECK_ARG(M < (1ll << 31) && N < (1ll << 31), "bf_layernorm_matmul: fp32 mode sizes must fit int32");
  Carve cv{static_cast<uint8_t*>(ws)};
  float *xh = cv.take(M * Kp), *xl = cv.take(M * Kp), *yh = cv.take(N * Kp), *yl = cv.take(N * Kp);
  float *rstd = cv.take(M), *negdm = cv.take(M), *colsum = cv.take(N);
  SplitParams sp{};
  sp.seg[0] = {static_cast<const float*>(X), xh, xl, rstd, negdm, static_cast<int>(M), static_cast<int>(K),
               static_cast<int>(Kp), kSegLn};
  sp.seg[1] = {static_cast<const float*>(Yt), yh, yl, colsum, nullptr, static_cast<int>(N), static_cast<int>(K),
               static_cast<int>(Kp), kSegW};
  sp.nseg = 2;
  sp.total_rows = static_cast<int>(M + N);
  sp.eps = eps;
  launch_split(sp, pl.dev.sms, stream);

  if (f32x3_pair(M, N)) {
    const CUtensorMap tp[6] = {tmap(xh, M, Kp, BM), tmap(xl, M, Kp, BM), tmap(yh, N, Kp, 128),
                               tmap(yl, N, Kp, 128), tmap(yh, N, Kp, 128), tmap(yl, N, Kp, 128)};
    GemmParams gp{};
    gp.M = static_cast<int>(M);
    gp.N = static_cast<int>(N);
    gp.ldo = static_cast<int>(N);
    gp.kt = static_cast<int>(Kp / BK);
    gp.Mt = static_cast<int>((M + 255) / 256);
    gp.Nt = static_cast<int>((N + 255) / 256);
    gp.group = raster_group(gp.Mt, 2 * Kp, pl.dev.l2_bytes);
    gp.rstd = rstd;
    gp.negdm = negdm;
    gp.colsum = colsum;
    gp.O = static_cast<float*>(O);
    launch_pair<kLn>(tp, gp, stream);
    return;
  }
  const bool wide = f32x3_wide(M, N);
  const int bn = wide ? 256 : BN;
  const CUtensorMap tm[6] = {tmap(xh, M, Kp, BM), tmap(xl, M, Kp, BM), tmap(yh, N, Kp, bn),
                             tmap(yl, N, Kp, bn), tmap(yh, N, Kp, bn), tmap(yl, N, Kp, bn)};
  GemmParams gp{};
  gp.M = static_cast<int>(M);
  gp.N = static_cast<int>(N);
  gp.ldo = static_cast<int>(N);
  gp.kt = static_cast<int>(Kp / BK);
  gp.Mt = static_cast<int>((M + BM - 1) / BM);
  gp.Nt = static_cast<int>((N + bn - 1) / bn);
  gp.group = raster_group(gp.Mt, Kp, pl.dev.l2_bytes);
  gp.rstd = rstd;
  gp.negdm = negdm;
  gp.colsum = colsum;
  gp.O = static_cast<float*>(O);
  if (wide)
    launch_gemm<kLn, 256>(tm, gp, stream);
  else
    launch_gemm<kLn>(tm, gp, stream);
}

// K1 fp32 mode on the tensor cores: split {X (RMSNorm rows), Wt, Vt, Ut}, then the gate/up GEMM
// (two B operands sharing each A tile, SwiGLU epilogue writing h as its TF32 split), then the
// down GEMM on (h_hi, h_lo) x (u_hi, u_lo). Three launches chained by programmatic dependent launch.
void ffn_f32x3(const Plan& pl, const void* X, const void* Wt, const void* Vt, const void* Ut, void* O, float eps,
               void* ws, size_t ws_bytes, cudaStream_t stream) {
  using namespace f32x3;
  const int64_t M = pl.dims[0], D = pl.dims[1], F = pl.dims[2], N = pl.dims[3];
  const int64_t Dp = padded_k(D), Fp = padded_k(F);
  BF_CHECK_ARG(ws != nullptr && ws_bytes >= ffn_f32x3_workspace_bytes(M, D, F, N),
               "bf_rms_ffn_swiglu: workspace too small");
  BF_CHECK_ARG((reinterpret_cast<uintptr_t>(ws) & 15u) == 0, "bf_rms_ffn_swiglu: workspace must be 16-byte aligned");
  BF_CHECK_ARG(M + 2 * F + N < (1ll << 31), "bf_rms_ffn_swiglu: fp32 mode sizes must fit int32");
  Carve cv{static_cast<uint8_t*>(ws)};
  float *xh = cv.take(M * Dp), *xl = cv.take(M * Dp);
  float *wh = cv.take(F * Dp), *wl = cv.take(F * Dp), *vh = cv.take(F * Dp), *vl = cv.take(F * Dp);
  float *uh = cv.take(N * Fp), *ul = cv.take(N * Fp), *hh = cv.take(M * Fp), *hl = cv.take(M * Fp);
  float* rstd = cv.take(M);
  const int m = static_cast<int>(M), d = static_cast<int>(D), f = static_cast<int>(F), n = static_cast<int>(N);
  SplitParams sp{};
  sp.seg[0] = {static_cast<const float*>(X), xh, xl, rstd, nullptr, m, d, static_cast<int>(Dp), kSegRms};
  sp.seg[1] = {static_cast<const float*>(Wt), wh, wl, nullptr, nullptr, f, d, static_cast<int>(Dp), kSegW};
  sp.seg[2] = {static_cast<const float*>(Vt), vh, vl, nullptr, nullptr, f, d, static_cast<int>(Dp), kSegW};
  sp.seg[3] = {static_cast<const float*>(Ut), uh, ul, nullptr, nullptr, n, f, static_cast<int>(Fp), kSegW};
  sp.nseg = 4;
  sp.total_rows = static_cast<int>(M + 2 * F + N);
  sp.eps = eps;
  launch_split(sp, pl.dev.sms, stream);

  if (f32x3_pair_gate(M, Fp)) {
    const CUtensorMap tp[6] = {tmap(xh, M, Dp, BM), tmap(xl, M, Dp, BM), tmap(wh, F, Dp, PG_BN / 2),
                               tmap(wl, F, Dp, PG_BN / 2), tmap(vh, F, Dp, PG_BN / 2), tmap(vl, F, Dp, PG_BN / 2)};
    GemmParams gq{};
    gq.M = m;
    gq.N = static_cast<int>(Fp);  // columns [F, Fp) of h are written as zeros (the down GEMM's K padding)
    gq.ldo = static_cast<int>(Fp);
    gq.kt = static_cast<int>(Dp / BK);
    gq.Mt = static_cast<int>((M + 255) / 256);
    gq.Nt = static_cast<int>((Fp + PG_BN - 1) / PG_BN);
    gq.group = raster_group(gq.Mt, 2 * Dp, pl.dev.l2_bytes);
    gq.rstd = rstd;
    gq.O = hh;
    gq.O2 = hl;
    launch_pair_gate(tp, gq, stream);
  } else {
  const CUtensorMap tg[6] = {tmap(xh, M, Dp, BM), tmap(xl, M, Dp, BM), tmap(wh, F, Dp, BN),
                             tmap(wl, F, Dp, BN), tmap(vh, F, Dp, BN), tmap(vl, F, Dp, BN)};
  GemmParams g1{};
  g1.M = m;
  g1.N = static_cast<int>(Fp);  // columns [F, Fp) of h are written as zeros (the down GEMM's K padding)
  g1.ldo = static_cast<int>(Fp);
  g1.kt = static_cast<int>(Dp / BK);
  g1.Mt = static_cast<int>((M + BM - 1) / BM);
  g1.Nt = static_cast<int>((Fp + BN - 1) / BN);
  g1.group = raster_group(g1.Mt, Dp, pl.dev.l2_bytes);
  g1.rstd = rstd;
  g1.O = hh;
  g1.O2 = hl;
  launch_gemm<kGate>(tg, g1, stream);
  }

  if (f32x3_k1_pair() && (f32x3_pair_forced() || ((M + 255) / 256) * ((N + 255) / 256) >= 148)) {
    const CUtensorMap tp[6] = {tmap(hh, M, Fp, BM), tmap(hl, M, Fp, BM), tmap(uh, N, Fp, 128),
                               tmap(ul, N, Fp, 128), tmap(uh, N, Fp, 128), tmap(ul, N, Fp, 128)};
    GemmParams g2{};
    g2.M = m;
    g2.N = n;
    g2.ldo = n;
    g2.kt = static_cast<int>(Fp / BK);
    g2.Mt = static_cast<int>((M + 255) / 256);
    g2.Nt = static_cast<int>((N + 255) / 256);
    g2.group = raster_group(g2.Mt, 2 * Fp, pl.dev.l2_bytes);
    g2.O = static_cast<float*>(O);
    launch_pair<kPlain>(tp, g2, stream);
    return;
  }
  const bool wide = f32x3_wide(M, N);
  const int bn = wide ? 256 : BN;
  const CUtensorMap td[6] = {tmap(hh, M, Fp, BM), tmap(hl, M, Fp, BM), tmap(uh, N, Fp, bn),
                             tmap(ul, N, Fp, bn), tmap(uh, N, Fp, bn), tmap(ul, N, Fp, bn)};
  GemmParams g2{};
  g2.M = m;
  g2.N = n;
  g2.ldo = n;
  g2.kt = static_cast<int>(Fp / BK);
  g2.Mt = static_cast<int>((M + BM - 1) / BM);
  g2.Nt = static_cast<int>((N + bn - 1) / bn);
  g2.group = raster_group(g2.Mt, Fp, pl.dev.l2_bytes);
  g2.O = static_cast<float*>(O);
  if (wide)
    launch_gemm<kPlain, 256>(td, g2, stream);
  else
    launch_gemm<kPlain>(td, g2, stream);
}

}  // namespace bfgpu
