// K3 fp32 mode on the tensor cores: flash attention with three-pass TF32 products ("3xTF32").
//
// The fp32 mode must match the float64 reference within 1e-4, which one TF32 product misses;
// splitting each operand x = x_hi + x_lo (x_hi = rna_tf32(x), x_lo = x - x_hi, exact in fp32)
// and accumulating lo*hi + hi*lo + hi*hi in the fp32 TMEM accumulator leaves ~1e-6 (as in
// csrc/f32x3.cu). Here both contractions of attention run that way:
//   S  = Q K^T    A = Q (hi/lo resident in TMEM), B = the key block (hi/lo in SMEM)
//   O += P V      A = P (hi/lo written to TMEM by the softmax), B = the Vt block (hi/lo in SMEM)
// with an exact fp32 online softmax in between (log2 domain, scale * log2(e) folded into Q;
// the base moves only when a row maximum grows by more than 2^8, the rebasing rule of
// safe_attention_rows, safe_numerics.hpp:158-170).
//
// The bf_attention C-ABI has no workspace, so the operands are split inside the kernel: TMA
// brings raw fp32 key and value blocks into a 2-slot ring, and four converter warps write hi
// and lo at the same swizzled offsets (the split is elementwise, so the SW128 layout carries
// over) into single-buffered split tiles, one block ahead of the MMAs. S is double-buffered in
// TMEM, so S(j+1) runs on the tensor pipe while the softmax works on S(j); P_hi overwrites its
// S buffer and P_lo goes to SMEM (an SS operand of PV).
//
// One CTA per (head, 128 query rows); 384 threads:
//   warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator,
//   warps 4-7 softmax + epilogue (thread = query row = TMEM lane), warps 8-11 converters.
// TMEM (512 columns): Q_hi [0, D) | Q_lo [D, 2D) | S/P_hi x2 [2D, 2D+128) | O [2D+128, +Dv).
// Block program: the final snapshot of fuse(lower(examples::attention())) (lowering.hpp:559-571).
#include <cuda_runtime.h>

#include <cmath>

#include "common.hpp"
#include "plan.hpp"
#include "sm100.cuh"
#include "tma_host.hpp"

namespace bfgpu {
namespace attn_f32x3 {

constexpr int BQ = 128, BKV = 64;
constexpr int THREADS = 384;
constexpr int RAW_SLOTS = 2;
constexpr int RAW_BYTES = 32768;  // one raw block: 64 keys x D (<= 128) fp32, or Dv (<= 128) x 64 keys
constexpr int SPLIT_BYTES = 2 * RAW_BYTES;  // hi | lo
constexpr int OFF_KS = RAW_SLOTS * RAW_BYTES;
constexpr int OFF_VS = OFF_KS + SPLIT_BYTES;
constexpr int OFF_PL = OFF_VS + SPLIT_BYTES;  // P_lo [128 rows][64 keys], two SW128 boxes of 32 keys
constexpr int PL_BYTES = 128 * 64 * 4;
constexpr int OFF_BAR = OFF_PL + PL_BYTES;
constexpr int SMEM = OFF_BAR + 256;
static_assert(SMEM <= 232448, "fp32 tensor-core attention SMEM budget");

__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// D[tmem] (+)= A[tmem] * B[smem]^T, tf32 inputs, fp32 accumulate.
__device__ __forceinline__ void umma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, tf32.
__device__ __forceinline__ void umma_tf32_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
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

// Order of the raw ring: K0, K1, V0, K2, V1, ..., K(nb-1), V(nb-2), V(nb-1). Each key block is
// split one step ahead of the value block before it, so S(j+1) can be issued while PV(j-1) runs.
__device__ __forceinline__ void ring_item(int n, int nb, bool& is_k, int& j) {
  if (n == 0) {
    is_k = true;
    j = 0;
    return;
  }
  const int m = n - 1;
  if (m / 2 + 1 < nb) {
    is_k = (m & 1) == 0;
    j = is_k ? m / 2 + 1 : m / 2;
  } else {
    is_k = false;
    j = n - nb;
  }
}

template <int D, int DV>
__global__ void __launch_bounds__(THREADS, 1)
    attn_f32x3_kernel(const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                      const float* __restrict__ Q, float* __restrict__ O, int Sq, int Skv, float qscale) {
  using namespace dev;
  static_assert((D == 64 || D == 128) && (DV == 64 || DV == 128), "head dims 64/128");
  constexpr int K_BYTES = BKV * D * 4, V_BYTES = DV * BKV * 4;
  // S is double-buffered (S(j+1) runs while the softmax works on S(j)); P_hi overwrites its S
  // buffer, P_lo goes to SMEM
  constexpr uint32_t COL_QH = 0, COL_QL = D, COL_S = 2 * D, COL_O = 2 * D + 128;
  static_assert(COL_O + DV <= 512, "TMEM budget");
  constexpr uint32_t IDESC_S = idesc_tf32(BQ, BKV), IDESC_O = idesc_tf32(BQ, DV);

  extern __shared__ __align__(1024) uint8_t smem[];
  if (dev::smem_u32(smem) & 1023u) __trap();
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* empty = full + RAW_SLOTS;
  uint64_t* ks_full = empty + RAW_SLOTS;
  uint64_t* ks_empty = ks_full + 1;
  uint64_t* vs_full = ks_empty + 1;
  uint64_t* vs_empty = vs_full + 1;
  uint64_t* q_ready = vs_empty + 1;
  uint64_t* s_full = q_ready + 1;   // [2]: one per S buffer
  uint64_t* p_ready = s_full + 2;  // [2]: keys 0-31 and 32-63 of the block written
  uint64_t* pv_done = p_ready + 2;
  uint64_t* o_full = pv_done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const uint32_t warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t lane = lane_id();
  const int h = blockIdx.y, q0 = blockIdx.x * BQ;
  const int nb = (Skv + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
    for (int s = 0; s < RAW_SLOTS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 128);
    }
    mbar_init(ks_full, 128);
    mbar_init(ks_empty, 1);
    mbar_init(vs_full, 128);
    mbar_init(vs_empty, 1);
    mbar_init(q_ready, 128);
    mbar_init(&s_full[0], 1);
    mbar_init(&s_full[1], 1);
    mbar_init(pv_done, 1);
    mbar_init(&p_ready[0], 128);
    mbar_init(&p_ready[1], 128);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- TMA: key and value blocks into the raw ring, in ring_item order
    if (lane == 0) {
      for (int i = 0; i < 2 * nb; ++i) {
        const int s = i % RAW_SLOTS;
        bool is_k;
        int j;
        ring_item(i, nb, is_k, j);
        mbar_wait(&empty[s], ((i / RAW_SLOTS) & 1) ^ 1);
        uint8_t* dst = smem + s * RAW_BYTES;
        if (is_k) {
          mbar_arrive_expect_tx(&full[s], K_BYTES);
#pragma unroll
          for (int b = 0; b < D / 32; ++b) tma_load_3d(&tm_k, &full[s], dst + b * (BKV * 128), 32 * b, j * BKV, h);
        } else {
          mbar_arrive_expect_tx(&full[s], V_BYTES);
#pragma unroll
          for (int b = 0; b < BKV / 32; ++b) tma_load_3d(&tm_v, &full[s], dst + b * (DV * 128), j * BKV + 32 * b, 0, h);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer
    const uint32_t ks = smem_u32(smem + OFF_KS), vs = smem_u32(smem + OFF_VS), pls = smem_u32(smem + OFF_PL);
    auto issue_s = [&](int j) {  // S(j) into buffer j & 1
      mbar_wait(ks_full, j & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t sb = tmem + COL_S + (j & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < D / 8; ++kk) {
          const uint32_t bo = (kk >> 2) * (BKV * 128) + (kk & 3) * 32;
          const uint64_t bh = sdesc_kmajor_sw128(ks + bo), bl = sdesc_kmajor_sw128(ks + RAW_BYTES + bo);
          // small terms first: lo*hi, hi*lo, then hi*hi
          umma_tf32_ts(sb, tmem + COL_QL + kk * 8, bh, IDESC_S, kk != 0);
          umma_tf32_ts(sb, tmem + COL_QH + kk * 8, bl, IDESC_S, 1);
          umma_tf32_ts(sb, tmem + COL_QH + kk * 8, bh, IDESC_S, 1);
        }
        umma_commit(ks_empty);
        umma_commit(&s_full[j & 1]);
      }
      __syncwarp();
    };
    mbar_wait(q_ready, 0);
    issue_s(0);
    for (int j = 0; j < nb; ++j) {
      if (j + 1 < nb) issue_s(j + 1);  // runs on the tensor pipe while the softmax works on S(j)
      mbar_wait(vs_full, j & 1);
      // PV in two halves of 32 keys: the first runs while the softmax writes the second
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        mbar_wait(&p_ready[half], j & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t pb = tmem + COL_S + (j & 1) * 64;  // P_hi over S(j)
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const int kk = 4 * half + k4;
            const uint32_t bo = (kk >> 2) * (DV * 128) + (kk & 3) * 32;
            const uint64_t bh = sdesc_kmajor_sw128(vs + bo), bl = sdesc_kmajor_sw128(vs + RAW_BYTES + bo);
            const uint64_t pl = sdesc_kmajor_sw128(pls + (kk >> 2) * (128 * 128) + (kk & 3) * 32);
            umma_tf32_ss(tmem + COL_O, pl, bh, IDESC_O, (j | kk) != 0);
            umma_tf32_ts(tmem + COL_O, pb + kk * 8, bl, IDESC_O, 1);
            umma_tf32_ts(tmem + COL_O, pb + kk * 8, bh, IDESC_O, 1);
          }
        }
        __syncwarp();
      }
      if (lane == 0) {
        umma_commit(vs_empty);
        umma_commit(pv_done);
        if (j == nb - 1) umma_commit(o_full);
      }
      __syncwarp();
    }
  } else if (warp >= 8) {
    // ---- converters: raw block -> hi | lo at the same swizzled offsets
    const int t = static_cast<int>(threadIdx.x) - 256;
    for (int i = 0; i < 2 * nb; ++i) {
      const int s = i % RAW_SLOTS;
      bool is_k;
      int j;
      ring_item(i, nb, is_k, j);
      mbar_wait(&full[s], (i / RAW_SLOTS) & 1);
      mbar_wait(is_k ? ks_empty : vs_empty, (j & 1) ^ 1);
      const float4* src = reinterpret_cast<const float4*>(smem + s * RAW_BYTES);
      float4* hi = reinterpret_cast<float4*>(smem + (is_k ? OFF_KS : OFF_VS));
      float4* lo = reinterpret_cast<float4*>(smem + (is_k ? OFF_KS : OFF_VS) + RAW_BYTES);
      const int n4 = (is_k ? K_BYTES : V_BYTES) / 16;
#pragma unroll 4
      for (int c = t; c < n4; c += 128) {
        const float4 v = src[c];
        const float4 vh = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        hi[c] = vh;
        lo[c] = make_float4(v.x - vh.x, v.y - vh.y, v.z - vh.z, v.w - vh.w);
      }
      fence_proxy_async_smem();  // generic-proxy writes -> tensor-core (async proxy) reads
      mbar_arrive(is_k ? ks_full : vs_full);
      mbar_arrive(&empty[s]);
    }
  } else if (warp >= 4) {
    // ---- softmax + epilogue: thread = query row
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t tl = tmem + (((warp & 3) * 32) << 16);
    const int grow = q0 + static_cast<int>(row);
    const float* qrow = Q + (static_cast<size_t>(h) * Sq + (grow < Sq ? grow : 0)) * D;
#pragma unroll 1
    for (int c = 0; c < D / 32; ++c) {
      uint32_t vh[32], vl[32];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 v = grow < Sq ? __ldg(reinterpret_cast<const float4*>(qrow + 32 * c) + i)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
        const float e[4] = {v.x * qscale, v.y * qscale, v.z * qscale, v.w * qscale};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float hh = tf32_hi(e[u]);
          vh[4 * i + u] = __float_as_uint(hh);
          vl[4 * i + u] = __float_as_uint(e[u] - hh);
        }
      }
      tmem_st_32x32b_x32(tl + COL_QH + 32 * c, vh);
      tmem_st_32x32b_x32(tl + COL_QL + 32 * c, vl);
    }
    tmem_wait_st();
    tc_fence_before();
    mbar_arrive(q_ready);

    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nb; ++j) {
      const uint32_t sb = COL_S + (j & 1) * 64;
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t s0[32], s1[32];
      tmem_ld_32x32b_x32(tl + sb, s0);
      tmem_ld_32x32b_x32(tl + sb + 32, s1);
      tmem_wait_ld();
      const int valid = Skv - j * BKV;  // keys of this block that exist
      float x[64];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        x[c] = c < valid ? __uint_as_float(s0[c]) : -INFINITY;
        x[32 + c] = 32 + c < valid ? __uint_as_float(s1[c]) : -INFINITY;
      }
      float mx = x[0];
#pragma unroll
      for (int c = 1; c < 64; ++c) mx = fmaxf(mx, x[c]);
      if (j == 0) {
        m_run = mx;
      } else {
        // rebase rows whose maximum grew by more than 2^8: O and l move to the new maximum (O
        // holds PV(0..j-1), complete). The TMEM accesses are warp-collective, so the whole warp
        // takes the branch and rows that keep their base scale by 1.
        const bool grow = mx > m_run + 8.0f;
        if (__any_sync(0xffffffffu, grow)) {
          mbar_wait(pv_done, (j - 1) & 1);  // O holds PV(0..j-1) only once PV(j-1) is complete
          tc_fence_after();
          const float f = grow ? ex2_approx(m_run - mx) : 1.0f;
          l_run *= f;
#pragma unroll 1
          for (int c = 0; c < DV / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tl + COL_O + 32 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * f);
            tmem_st_32x32b_x32(tl + COL_O + 32 * c, o);
          }
          if (grow) m_run = mx;
        }
      }
      float ls = 0.f;
      uint8_t* plrow = smem + OFF_PL + row * 128;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t ph[32];
        float pl[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float p = ex2_approx(x[32 * half + c] - m_run);
          ls += p;
          const float hh = tf32_hi(p);
          ph[c] = __float_as_uint(hh);
          pl[c] = p - hh;
        }
        tmem_st_32x32b_x32(tl + sb + 32 * half, ph);
        // P_lo of PV(j-1) must be consumed before it is overwritten
        if (half == 0 && j > 0) mbar_wait(pv_done, (j - 1) & 1);
        uint8_t* box = plrow + half * (128 * 128);  // keys 32 half .. +31: one SW128 box
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4*>(box + ((c ^ (row & 7)) << 4)) =
              make_float4(pl[4 * c], pl[4 * c + 1], pl[4 * c + 2], pl[4 * c + 3]);
        fence_proxy_async_smem();
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_ready[half]);  // (half 0 also covers the O rebase above)
      }
      l_run += ls;
    }
    mbar_wait(o_full, 0);
    tc_fence_after();
    const float inv = 1.0f / l_run;
    float* orow = O + (static_cast<size_t>(h) * Sq + grow) * DV;
#pragma unroll 1
    for (int c = 0; c < DV / 32; ++c) {
      uint32_t o[32];
      tmem_ld_32x32b_x32(tl + COL_O + 32 * c, o);
      tmem_wait_ld();
      if (grow < Sq) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          reinterpret_cast<float4*>(orow + 32 * c)[i] =
              make_float4(__uint_as_float(o[4 * i]) * inv, __uint_as_float(o[4 * i + 1]) * inv,
                          __uint_as_float(o[4 * i + 2]) * inv, __uint_as_float(o[4 * i + 3]) * inv);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// [batch, rows, cols] fp32, contiguous; box = 32 columns (128 bytes, SW128) x box_rows x 1.
inline CUtensorMap tmap_f32_3d(const void* base, uint64_t batch, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {cols, rows, batch};
  cuuint64_t strides[2] = {cols * 4, rows * cols * 4};
  cuuint32_t box[3] = {32, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_tiled_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed (fp32 3-D attention operand)");
  return m;
}

template <int D, int DV>
void launch(const float* Q, const float* K, const float* Vt, float* O, int64_t BH, int64_t Sq, int64_t Skv,
            float scale, cudaStream_t stream) {
  const CUtensorMap tk = tmap_f32_3d(K, BH, Skv, D, BKV);
  const CUtensorMap tv = tmap_f32_3d(Vt, BH, DV, Skv, DV);
  ensure_smem_attr(reinterpret_cast<const void*>(&attn_f32x3_kernel<D, DV>), SMEM);
  const dim3 grid(static_cast<unsigned>((Sq + BQ - 1) / BQ), static_cast<unsigned>(BH));
  attn_f32x3_kernel<D, DV><<<grid, THREADS, SMEM, stream>>>(tk, tv, Q, O, static_cast<int>(Sq), static_cast<int>(Skv),
                                                           scale * 1.4426950408889634f);
  BF_CUDA(cudaGetLastError());
  note_launch();
}

template <int D, int DV>
KernelSpec spec_t() {
  KernelSpec k;
  k.name = "attn_f32x3_kernel";
  k.func = reinterpret_cast<const void*>(&attn_f32x3_kernel<D, DV>);
  k.threads = THREADS;
  k.smem_bytes = SMEM;
  k.tmem_cols = 512;
  k.tile_m = BQ;
  k.tile_n = BKV;
  k.tile_k = D;
  k.stages = RAW_SLOTS;
  return k;
}

}  // namespace attn_f32x3

// The tensor-core fp32 attention takes head dims 64/128, Skv a multiple of 4 (TMA row pitch)
// and 16-byte aligned operands.
bool attn_f32x3_supported(int64_t D, int64_t Dv, int64_t Skv, const void* Q, const void* K, const void* Vt,
                          const void* O) {
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  return (D == 64 || D == 128) && (Dv == 64 || Dv == 128) && Skv % 4 == 0 &&
         (Q == nullptr || (a16(Q) && a16(K) && a16(Vt) && a16(O)));
}

KernelSpec attn_f32x3_spec(int D, int Dv) {
  using namespace attn_f32x3;
  if (D == 128 && Dv == 128) return spec_t<128, 128>();
  if (D == 128 && Dv == 64) return spec_t<128, 64>();
  if (D == 64 && Dv == 128) return spec_t<64, 128>();
  return spec_t<64, 64>();
}

void attention_f32x3(const float* Q, const float* K, const float* Vt, float* O, int64_t BH, int64_t Sq, int64_t Skv,
                     int64_t D, int64_t Dv, float scale, cudaStream_t stream) {
  using namespace attn_f32x3;
  BF_CHECK_ARG(Sq < (1ll << 31) && Skv < (1ll << 31), "bf_attention: sequence lengths must fit int32");
  if (D == 128 && Dv == 128)
    launch<128, 128>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
  else if (D == 128 && Dv == 64)
    launch<128, 64>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
  else if (D == 64 && Dv == 128)
    launch<64, 128>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
  else
    launch<64, 64>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
}

}  // namespace bfgpu
