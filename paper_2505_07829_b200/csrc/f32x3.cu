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
//                      K=8 step; rank 1 hands its partial sums over DSMEM and rank 0 writes
//                      O = (acc0 + acc1 - dm colsum(Yt)) * rstd straight to global.
// Reference: ref::layernorm_matmul (interpreter.hpp:549-551); the block program is the
// final snapshot of fuse(lower(examples::layernorm_matmul())) (lowering.hpp:573-581).
#include <cuda_runtime.h>

#include <algorithm>

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
constexpr int STAGES = 3;
constexpr int A_BYTES = BM * BK * 4;  // 16 KB
constexpr int B_BYTES = BN * BK * 4;  // 16 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int RED_PITCH = BN * 4 + 16;  // reduction buffer row pitch (bytes): rows land on distinct banks
static_assert(BM * RED_PITCH <= STAGES * STAGE_BYTES, "reduction buffer reuses the operand ring");
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256;
constexpr int NUM_THREADS = 256;
constexpr uint32_t TMEM_COLS = BN;
// kind::tf32 instruction descriptor: D F32, A/B TF32 (format 2), both K-major, N/8, M/16
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

__device__ __forceinline__ void umma_tf32_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ float4 ld_cluster_v4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

struct SplitParams {
  const float* X;
  const float* Yt;
  int M, N, K, Kp;
  float inv_k, eps;
  float* xh;
  float* xl;
  float* yh;
  float* yl;
  float* rstd;
  float* negdm;   // [M] p - mean (the shift left after subtracting the pivot)
  float* colsum;  // [N] sum_k Yt[n, k]
};

// One warp per row: rows [0, M) of X, then [M, M + N) of Yt. A row is read once when it
// fits the registers (K <= 1024: 8 float4 per lane), else streamed twice (moments, split).
__global__ void __launch_bounds__(256) f32_split_kernel(const SplitParams p) {
  constexpr int R = 8;  // float4 per lane held in registers
  // the GEMM launch may start its prologue now; it waits for this grid before reading
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int warps = static_cast<int>(gridDim.x * blockDim.x / 32);
  const bool vec = (p.K & 3) == 0;
  for (int r = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) / 32); r < p.M + p.N; r += warps) {
    const bool is_x = r < p.M;
    const int rr = is_x ? r : r - p.M;
    const float* src = (is_x ? p.X : p.Yt) + static_cast<size_t>(rr) * p.K;
    float4* hi = reinterpret_cast<float4*>((is_x ? p.xh : p.yh) + static_cast<size_t>(rr) * p.Kp);
    float4* lo = reinterpret_cast<float4*>((is_x ? p.xl : p.yl) + static_cast<size_t>(rr) * p.Kp);
    auto load4 = [&](int k4) -> float4 {  // columns [4 k4, 4 k4 + 4), zero past K
      const int k = 4 * k4;
      if (vec && k + 3 < p.K) return __ldg(reinterpret_cast<const float4*>(src) + k4);
      float e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) e[u] = k + u < p.K ? __ldg(src + k + u) : 0.f;
      return make_float4(e[0], e[1], e[2], e[3]);
    };
    const int n4 = p.Kp / 4;
    const bool in_regs = n4 <= 32 * R;
    float4 v[R];
    if (in_regs) {
#pragma unroll
      for (int i = 0; i < R; ++i) v[i] = lane + 32 * i < n4 ? load4(lane + 32 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // moments about the row's first element: no E[x^2] - mu^2 cancellation; for Yt, the sum
    const float piv = is_x ? __ldg(src) : 0.f;
    float s1 = 0.f, s2 = 0.f;
    auto acc = [&](float4 a, int k) {
      const float e[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k + u < p.K) {
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
      if (is_x) {
        const float dm = s1 * p.inv_k;
        p.rstd[rr] = 1.0f / sqrtf(s2 * p.inv_k - dm * dm + p.eps);
        p.negdm[rr] = -dm;
      } else {
        p.colsum[rr] = s1;
      }
    }
    // x - p: exact when the row sits far from zero (|mu| >> sigma), where centring on a rounded
    // fp32 mean is not
    auto split = [&](float4 a, int k4) {
      const float e[4] = {a.x, a.y, a.z, a.w};
      float h[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float x = 4 * k4 + u < p.K ? e[u] - piv : 0.f;
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

struct GemmParams {
  int M, N, kt;
  const float* rstd;
  const float* negdm;
  const float* colsum;
  float* O;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    f32x3_gemm_kernel(const __grid_constant__ CUtensorMap tm_xh, const __grid_constant__ CUtensorMap tm_xl,
                      const __grid_constant__ CUtensorMap tm_yh, const __grid_constant__ CUtensorMap tm_yl,
                      const GemmParams p) {
  using namespace dev;
  extern __shared__ __align__(1024) uint8_t smem[];
  if (smem_u32(smem) & 1023u) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();  // which half of K this CTA contracts
  const int n0 = static_cast<int>(blockIdx.x >> 1) * BN, m0 = static_cast<int>(blockIdx.y) * BM;
  const int khalf = (p.kt + 1) / 2;
  const int k_begin = rank == 0 ? 0 : khalf, k_end = rank == 0 ? khalf : p.kt;
  const int nk = k_end - k_begin;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_xh);
    tma_prefetch_desc(&tm_xl);
    tma_prefetch_desc(&tm_yh);
    tma_prefetch_desc(&tm_yl);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: everything above overlapped the split launch; the split
  // operands, statistics and colsum are read only after it has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % STAGES, k = k_begin + i;
        mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        tma_load_2d(&tm_xh, &full[s], st, k * BK, m0);
        tma_load_2d(&tm_xl, &full[s], st + A_BYTES, k * BK, m0);
        tma_load_2d(&tm_yh, &full[s], st + 2 * A_BYTES, k * BK, n0);
        tma_load_2d(&tm_yl, &full[s], st + 2 * A_BYTES + B_BYTES, k * BK, n0);
      }
    }
  } else if (warp == 1) {
    for (int i = 0; i < nk; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t xh = smem_u32(smem + s * STAGE_BYTES), xl = xh + A_BYTES, yh = xh + 2 * A_BYTES,
                       yl = yh + B_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {  // K = 8 tf32 = 32 bytes per MMA
          const uint32_t o = kk * 32;
          // small terms first: lo*hi, hi*lo, then hi*hi
          umma_tf32_ss(tmem, sdesc_kmajor_sw128(xl + o), sdesc_kmajor_sw128(yh + o), (i | kk) != 0);
          umma_tf32_ss(tmem, sdesc_kmajor_sw128(xh + o), sdesc_kmajor_sw128(yl + o), 1);
          umma_tf32_ss(tmem, sdesc_kmajor_sw128(xh + o), sdesc_kmajor_sw128(yh + o), 1);
        }
        umma_commit(&empty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) umma_commit(tfull);  // nk == 0 (K <= 32 on rank 1): arrives at once, acc unused
    __syncwarp();
  }
  const uint32_t q = warp & 3;
  const uint32_t trow = q * 32 + lane;
  uint8_t* red = smem;  // the operand ring is idle once tfull has fired
  if (warp >= 4 && rank == 1) {
    // rank 1 parks its partial sums in its own SMEM for rank 0 (zeros if it had no K steps)
    mbar_wait(tfull, 0);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + ((q * 32) << 16) + c * 32, v);
      tmem_wait_ld();
      float4* dst = reinterpret_cast<float4*>(red + trow * RED_PITCH + c * 128);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        dst[i] = nk > 0 ? make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                      __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  tc_fence_before();
  cluster_sync();  // rank 1's partials are visible cluster-wide
  if (warp >= 4 && rank == 0) {
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int row = m0 + static_cast<int>(trow);
    const uint32_t peer = mapa_shared(smem_u32(red + trow * RED_PITCH), 1);
    const float r = row < p.M ? __ldg(p.rstd + row) : 0.f, nd = row < p.M ? __ldg(p.negdm + row) : 0.f;
    float* orow = p.O + static_cast<size_t>(row) * p.N;
    const bool vec = (p.N & 3) == 0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + ((q * 32) << 16) + c * 32, v);
      tmem_wait_ld();
      if (row >= p.M) continue;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int col = n0 + c * 32 + 4 * i;
        const float4 o1 = ld_cluster_v4(peer + c * 128 + i * 16);
        const float a[4] = {__uint_as_float(v[4 * i]) + o1.x, __uint_as_float(v[4 * i + 1]) + o1.y,
                            __uint_as_float(v[4 * i + 2]) + o1.z, __uint_as_float(v[4 * i + 3]) + o1.w};
        float o[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) o[u] = col + u < p.N ? fmaf(nd, __ldg(p.colsum + col + u), a[u]) * r : 0.f;
        if (vec && col + 3 < p.N) {
          *reinterpret_cast<float4*>(orow + col) = make_float4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (col + u < p.N) orow[col + u] = o[u];
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // rank 1's SMEM stays alive until rank 0 has read it
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
}

int64_t padded_k(int64_t K) { return (K + BK - 1) / BK * BK; }

}  // namespace f32x3

size_t lnmm_f32x3_workspace_bytes(int64_t M, int64_t K, int64_t N) {
  const size_t kp = static_cast<size_t>(f32x3::padded_k(K));
  return 2 * align_up(static_cast<size_t>(M) * kp * 4, 1024) + 2 * align_up(static_cast<size_t>(N) * kp * 4, 1024) +
         2 * align_up(static_cast<size_t>(M) * 4, 256) + align_up(static_cast<size_t>(N) * 4, 256);
}

KernelSpec f32x3_gemm_spec() {
  using namespace f32x3;
  KernelSpec k;
  k.name = "f32x3_gemm_kernel";
  k.func = reinterpret_cast<const void*>(&f32x3_gemm_kernel);
  k.threads = NUM_THREADS;
  k.smem_bytes = SMEM_BYTES;
  k.tmem_cols = TMEM_COLS;
  k.cluster = 2;  // the K range of a tile split over a CTA pair
  k.tile_m = BM;
  k.tile_n = BN;
  k.tile_k = BK;
  k.stages = STAGES;
  k.grid_sync = false;
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
  BF_CHECK_ARG((M + BM - 1) / BM <= 65535, "bf_layernorm_matmul: fp32 mode supports up to 65535 x 128 rows");
  uint8_t* w = static_cast<uint8_t*>(ws);
  SplitParams sp{};
  sp.X = static_cast<const float*>(X);
  sp.Yt = static_cast<const float*>(Yt);
  sp.M = static_cast<int>(M);
  sp.N = static_cast<int>(N);
  sp.K = static_cast<int>(K);
  sp.Kp = static_cast<int>(Kp);
  sp.inv_k = 1.0f / static_cast<float>(K);
  sp.eps = eps;
  const size_t xb = align_up(static_cast<size_t>(M) * Kp * 4, 1024), yb = align_up(static_cast<size_t>(N) * Kp * 4, 1024);
  sp.xh = reinterpret_cast<float*>(w);
  sp.xl = reinterpret_cast<float*>(w + xb);
  sp.yh = reinterpret_cast<float*>(w + 2 * xb);
  sp.yl = reinterpret_cast<float*>(w + 2 * xb + yb);
  sp.rstd = reinterpret_cast<float*>(w + 2 * xb + 2 * yb);
  sp.negdm = sp.rstd + align_up(static_cast<size_t>(M) * 4, 256) / 4;
  sp.colsum = sp.negdm + align_up(static_cast<size_t>(M) * 4, 256) / 4;
  const int64_t rows = M + N;
  const int split_grid = static_cast<int>(std::min<int64_t>((rows + 7) / 8, static_cast<int64_t>(pl.dev.sms) * 16));
  f32_split_kernel<<<split_grid, 256, 0, stream>>>(sp);
  BF_CUDA(cudaGetLastError());
  note_launch();

  const CUtensorMap tm_xh = make_tmap_2d(sp.xh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, Kp, Kp, BK, BM);
  const CUtensorMap tm_xl = make_tmap_2d(sp.xl, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, Kp, Kp, BK, BM);
  const CUtensorMap tm_yh = make_tmap_2d(sp.yh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, N, Kp, Kp, BK, BN);
  const CUtensorMap tm_yl = make_tmap_2d(sp.yl, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, N, Kp, Kp, BK, BN);
  GemmParams gp{};
  gp.M = static_cast<int>(M);
  gp.N = static_cast<int>(N);
  gp.kt = static_cast<int>(Kp / BK);
  gp.rstd = sp.rstd;
  gp.negdm = sp.negdm;
  gp.colsum = sp.colsum;
  gp.O = static_cast<float*>(O);
  ensure_smem_attr(reinterpret_cast<const void*>(&f32x3_gemm_kernel), SMEM_BYTES);
  const dim3 grid(static_cast<unsigned>(2 * ((N + BN - 1) / BN)), static_cast<unsigned>((M + BM - 1) / BM));
  // launched as a programmatic dependent of the split kernel (griddepcontrol in both)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BF_CUDA(cudaLaunchKernelEx(&cfg, f32x3_gemm_kernel, tm_xh, tm_xl, tm_yh, tm_yl, gp));
  note_launch();
}

}  // namespace bfgpu
