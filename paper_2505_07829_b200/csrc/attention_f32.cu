// K3 fp32 mode (north star: fp32 in/out within 1e-4 of the float64 reference), tiled on the
// FP32 FMA pipes: a FlashAttention-style CTA of 64 query rows x one head, 8 warps of 8 rows,
// key/value blocks of 64 staged in SMEM, exact online softmax in fp32 per block (the rebasing
// of safe_attention_rows, safe_numerics.hpp:158-170, at every block: alpha = exp(m_old - m_new)).
//
// Block program: the final snapshot of fuse(lower(examples::attention())) (lowering.hpp:559-571),
// O = softmax(Q K^T / sqrt(D)) V with V supplied as Vt [Dv, Skv].
//
// Register tiling per warp and key block (D = Dv = 128):
//   S = Q K^T   lane l owns keys l and l + 32 of the block for the warp's 8 rows: each 4-wide
//               step of D is 10 LDS.128 (8 broadcast Q rows, 2 K rows) for 64 FMAs;
//   O += P V    lane l owns output columns l + 32k for the 8 rows: each key is 2 LDS.128
//               (broadcast P of the 8 rows) + Dv/32 LDS for 8 Dv/32 FMAs.
// SMEM rows are padded (D + 4 floats for Q/K: 16-byte aligned, conflict-free 128-bit loads per
// 8-lane phase; 65 floats for the Vt tile: conflict-free scalar loads).
#include <cuda_runtime.h>

#include <cmath>

#include "common.hpp"
#include "plan.hpp"

namespace bfgpu {
namespace attn_f32t {

constexpr int BQ = 64, BKV = 64, WARPS = 8, THREADS = WARPS * 32, RW = BQ / WARPS;  // 8 rows per warp
constexpr int VSTRIDE = BKV + 1;

template <int D, int DV>
struct Cfg {
  static constexpr int QSTRIDE = D + 4;
  static constexpr int Q_FLOATS = BQ * QSTRIDE;
  static constexpr int K_FLOATS = BKV * QSTRIDE;
  static constexpr int V_FLOATS = DV * VSTRIDE;
  static constexpr int P_FLOATS = WARPS * BKV * RW;
  static constexpr int SMEM = (Q_FLOATS + K_FLOATS + V_FLOATS + P_FLOATS) * 4;
  static_assert(SMEM <= 232448, "fp32 attention SMEM budget");
};

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }

template <int D, int DV>
__global__ void __launch_bounds__(THREADS, 1)
    attn_f32_tiled_kernel(const float* __restrict__ Q, const float* __restrict__ K, const float* __restrict__ Vt,
                          float* __restrict__ O, int Sq, int Skv, float scale) {
  using C = Cfg<D, DV>;
  constexpr int KC = DV / 32;  // output columns per lane
  extern __shared__ __align__(16) float smem[];
  float* sQ = smem;
  float* sK = sQ + C::Q_FLOATS;
  float* sV = sK + C::K_FLOATS;
  float* sP = sV + C::V_FLOATS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y, q0 = blockIdx.x * BQ;
  const float* Qh = Q + static_cast<size_t>(h) * Sq * D;
  const float* Kh = K + static_cast<size_t>(h) * Skv * D;
  const float* Vh = Vt + static_cast<size_t>(h) * DV * Skv;
  float* Oh = O + static_cast<size_t>(h) * Sq * DV;
  float* myP = sP + warp * BKV * RW;  // [key][row]

  for (int i = tid; i < BQ * D / 4; i += THREADS) {
    const int r = i / (D / 4), c4 = i % (D / 4);
    const float4 v = q0 + r < Sq ? __ldg(reinterpret_cast<const float4*>(Qh + static_cast<size_t>(q0 + r) * D) + c4)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(sQ + r * C::QSTRIDE + 4 * c4) = v;
  }

  float m_run[RW], l_run[RW], o[RW][KC];
#pragma unroll
  for (int r = 0; r < RW; ++r) {
    m_run[r] = -INFINITY;
    l_run[r] = 0.f;
#pragma unroll
    for (int k = 0; k < KC; ++k) o[r][k] = 0.f;
  }
  const bool v_vec = (Skv & 3) == 0;

  for (int n0 = 0; n0 < Skv; n0 += BKV) {
    // ---- stage the K block [64 keys][D] and the Vt block [DV][64 keys]
    for (int i = tid; i < BKV * D / 4; i += THREADS) {
      const int key = i / (D / 4), c4 = i % (D / 4);
      const float4 v = n0 + key < Skv
                           ? __ldg(reinterpret_cast<const float4*>(Kh + static_cast<size_t>(n0 + key) * D) + c4)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(sK + key * C::QSTRIDE + 4 * c4) = v;
    }
    for (int i = tid; i < DV * BKV / 4; i += THREADS) {
      const int dv = i / (BKV / 4), j4 = i % (BKV / 4);
      const int key = n0 + 4 * j4;
      const float* src = Vh + static_cast<size_t>(dv) * Skv + key;
      float e[4];
      if (v_vec && key + 3 < Skv) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src));
        e[0] = v.x, e[1] = v.y, e[2] = v.z, e[3] = v.w;
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) e[u] = key + u < Skv ? __ldg(src + u) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) sV[dv * VSTRIDE + 4 * j4 + u] = e[u];
    }
    __syncthreads();

    // ---- S = Q K^T for the warp's 8 rows, keys lane and lane + 32
    float s[RW][2];
#pragma unroll
    for (int r = 0; r < RW; ++r) s[r][0] = s[r][1] = 0.f;
    const float* qrow = sQ + warp * RW * C::QSTRIDE;
    const float* ka = sK + lane * C::QSTRIDE;
    const float* kb = sK + (lane + 32) * C::QSTRIDE;
#pragma unroll 4
    for (int d = 0; d < D; d += 4) {
      const float4 a = lds4(ka + d), b = lds4(kb + d);
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const float4 q = lds4(qrow + r * C::QSTRIDE + d);
        s[r][0] = fmaf(q.x, a.x, fmaf(q.y, a.y, fmaf(q.z, a.z, fmaf(q.w, a.w, s[r][0]))));
        s[r][1] = fmaf(q.x, b.x, fmaf(q.y, b.y, fmaf(q.z, b.z, fmaf(q.w, b.w, s[r][1]))));
      }
    }
    const bool va = n0 + lane < Skv, vb = n0 + lane + 32 < Skv;

    // ---- exact online softmax per row (warp-wide max and sum over the 64 keys)
    float alpha[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const float x0 = va ? s[r][0] * scale : -INFINITY, x1 = vb ? s[r][1] * scale : -INFINITY;
      float mx = fmaxf(x0, x1);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float m_new = fmaxf(m_run[r], mx);
      alpha[r] = expf(m_run[r] - m_new);  // 0 on the first block (m_run = -inf)
      const float p0 = expf(x0 - m_new), p1 = expf(x1 - m_new);
      float ls = p0 + p1;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
      l_run[r] = l_run[r] * alpha[r] + ls;
      m_run[r] = m_new;
      s[r][0] = p0;
      s[r][1] = p1;
    }
    // P transposed per warp: [key][row], so the PV loop reads the 8 rows of a key as 2 LDS.128
    *reinterpret_cast<float4*>(myP + lane * RW) = make_float4(s[0][0], s[1][0], s[2][0], s[3][0]);
    *reinterpret_cast<float4*>(myP + lane * RW + 4) = make_float4(s[4][0], s[5][0], s[6][0], s[7][0]);
    *reinterpret_cast<float4*>(myP + (lane + 32) * RW) = make_float4(s[0][1], s[1][1], s[2][1], s[3][1]);
    *reinterpret_cast<float4*>(myP + (lane + 32) * RW + 4) = make_float4(s[4][1], s[5][1], s[6][1], s[7][1]);
    __syncwarp();

    // ---- O = alpha O + P V
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int k = 0; k < KC; ++k) o[r][k] *= alpha[r];
    const int nvalid = min(BKV, Skv - n0);
#pragma unroll 4
    for (int j = 0; j < nvalid; ++j) {
      const float4 pa = lds4(myP + j * RW), pb = lds4(myP + j * RW + 4);
      const float p[RW] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        const float v = sV[(lane + 32 * k) * VSTRIDE + j];
#pragma unroll
        for (int r = 0; r < RW; ++r) o[r][k] = fmaf(p[r], v, o[r][k]);
      }
    }
    __syncthreads();  // the next block overwrites sK, sV (and this warp's P after its own S)
  }

#pragma unroll
  for (int r = 0; r < RW; ++r) {
    const int row = q0 + warp * RW + r;
    if (row >= Sq) continue;
    const float inv = 1.0f / l_run[r];
#pragma unroll
    for (int k = 0; k < KC; ++k) Oh[static_cast<size_t>(row) * DV + lane + 32 * k] = o[r][k] * inv;
  }
}

template <int D, int DV>
void launch(const float* Q, const float* K, const float* Vt, float* O, int64_t BH, int64_t Sq, int64_t Skv,
            float scale, cudaStream_t stream) {
  using C = Cfg<D, DV>;
  ensure_smem_attr(reinterpret_cast<const void*>(&attn_f32_tiled_kernel<D, DV>), C::SMEM);
  const dim3 grid(static_cast<unsigned>((Sq + BQ - 1) / BQ), static_cast<unsigned>(BH));
  attn_f32_tiled_kernel<D, DV><<<grid, THREADS, C::SMEM, stream>>>(Q, K, Vt, O, static_cast<int>(Sq),
                                                                   static_cast<int>(Skv), scale);
  BF_CUDA(cudaGetLastError());
  note_launch();
}

template <int D, int DV>
KernelSpec spec_t() {
  KernelSpec k;
  k.name = "attn_f32_tiled_kernel";
  k.func = reinterpret_cast<const void*>(&attn_f32_tiled_kernel<D, DV>);
  k.threads = THREADS;
  k.smem_bytes = Cfg<D, DV>::SMEM;
  k.tile_m = BQ;
  k.tile_n = BKV;
  k.tile_k = D;
  k.stages = 1;
  k.tensor = false;
  return k;
}

}  // namespace attn_f32t

bool attn_f32_tiled_supported(int64_t D, int64_t Dv) { return (D == 64 || D == 128) && (Dv == 64 || Dv == 128); }

KernelSpec attn_f32_tiled_spec(int D, int Dv) {
  if (D == 128 && Dv == 128) return attn_f32t::spec_t<128, 128>();
  if (D == 128 && Dv == 64) return attn_f32t::spec_t<128, 64>();
  if (D == 64 && Dv == 128) return attn_f32t::spec_t<64, 128>();
  return attn_f32t::spec_t<64, 64>();
}

// fp32 attention on the tiled kernel (head dims 64/128); attention_f32 (simt_f32.cu) routes here.
void attention_f32_tiled(const float* Q, const float* K, const float* Vt, float* O, int64_t BH, int64_t Sq,
                         int64_t Skv, int64_t D, int64_t Dv, float scale, cudaStream_t stream) {
  if (D == 128 && Dv == 128)
    attn_f32t::launch<128, 128>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
  else if (D == 128 && Dv == 64)
    attn_f32t::launch<128, 64>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
  else if (D == 64 && Dv == 128)
    attn_f32t::launch<64, 128>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
  else
    attn_f32t::launch<64, 64>(Q, K, Vt, O, BH, Sq, Skv, scale, stream);
}

}  // namespace bfgpu
