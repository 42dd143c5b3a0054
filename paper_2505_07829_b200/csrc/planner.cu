// Device memory / tile planner (plan.hpp) and the per-device launch state.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <sstream>
#include <tuple>
#include <utility>
#include <vector>

#include "bfgpu.h"
#include "common.hpp"
#include "plan.hpp"

namespace bfgpu {

namespace {

std::mutex g_mu;

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && v[0] ? std::atoi(v) : dflt;
}

bool env_set(const char* name) {
  const char* v = std::getenv(name);
  return v && v[0];
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

int pow2_floor(int64_t x) {
  int p = 1;
  while (static_cast<int64_t>(p) * 2 <= x) p *= 2;
  return p;
}

// Time the launch would take at the tensor-core rate of the device at ~1.9 GHz
// (8192 dense bf16 FLOP per SM per clock: one 128x256x16 MMA per 128 cycles).
double est_ms_tensor(double flops, int sms) { return flops / (static_cast<double>(sms) * 8192.0 * 1.9e9) * 1e3; }

void check_budgets(const Plan& p) {
  const KernelSpec& k = p.spec;
  if (k.smem_bytes > p.dev.smem_optin)
    throw Status(BF_ERR_INTERNAL, std::string(k.name) + ": SMEM plan " + std::to_string(k.smem_bytes) +
                                      " B exceeds the device's " + std::to_string(p.dev.smem_optin) + " B per CTA");
  if (k.tmem_cols > 512)
    throw Status(BF_ERR_INTERNAL, std::string(k.name) + ": TMEM plan exceeds 512 columns");
  if (k.tmem_cols & (k.tmem_cols - 1))
    throw Status(BF_ERR_INTERNAL, std::string(k.name) + ": TMEM allocation must be a power of two columns");
  if (k.grid_sync && p.grid > p.resident_ctas)
    throw Status(BF_ERR_INTERNAL, std::string(k.name) + ": grid exceeds co-resident capacity");
}

void finish_grid(Plan& p, int64_t launch_tiles) {
  p.resident_ctas = resident_ctas(p.spec);
  if (p.resident_ctas <= 0)
    throw Status(BF_ERR_UNSUPPORTED, std::string(p.spec.name) + ": no CTA fits on device " +
                                         std::to_string(p.dev.device) + " (SMEM/TMEM/registers)");
  const int c = p.spec.cluster;
  const int64_t units = std::min<int64_t>(launch_tiles, p.resident_ctas / c);
  p.grid = static_cast<int>(std::max<int64_t>(1, units) * c);
}

}  // namespace

const DeviceInfo& device_info(int device) {
  static std::map<int, DeviceInfo> cache;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = cache.find(device);
  if (it != cache.end()) return it->second;
  DeviceInfo d;
  d.device = device;
  int major = 0, minor = 0;
  BF_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, device));
  BF_CUDA(cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  BF_CUDA(cudaDeviceGetAttribute(&d.l2_bytes, cudaDevAttrL2CacheSize, device));
  BF_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  BF_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
  d.cc = major * 10 + minor;
  return cache.emplace(device, d).first->second;
}

void ensure_smem_attr(const void* func, int bytes) {
  static std::set<std::pair<int, const void*>> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  if (done.count({dev, func})) return;
  BF_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({dev, func});
}

int resident_ctas(const KernelSpec& k) {
  static std::map<std::pair<int, const void*>, int> cache;
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = cache.find({dev, k.func});
    if (it != cache.end()) return it->second;
  }
  ensure_smem_attr(k.func, k.smem_bytes);
  const DeviceInfo& di = device_info(dev);
  int ctas = 0;
  if (k.cluster > 1) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(di.sms / k.cluster * k.cluster));
    cfg.blockDim = dim3(static_cast<unsigned>(k.threads));
    cfg.dynamicSmemBytes = static_cast<size_t>(k.smem_bytes);
    int clusters = 0;
    BF_CUDA(cudaOccupancyMaxActiveClusters(&clusters, k.func, &cfg));
    ctas = clusters * k.cluster;
  } else {
    int per_sm = 0;
    BF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k.func, k.threads, k.smem_bytes));
    ctas = per_sm * di.sms;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  cache[{dev, k.func}] = ctas;
  return ctas;
}

// ------------------------------------------------------------------ K1
// Modeled efficiency (balanced / makespan, in k-steps) of the fused CTA-pair schedule: static
// round-robin of the tile order decode_tile() produces (ffn_common.cuh) over `clusters`, a down
// tile starting once its cluster is free and every gate/up tile of its m-unit is done.
// Epilogues, memory and clocks are ignored; what it ranks is the schedule's tail and its
// dependency stalls. C3 full size models 0.988; its 8-GPU shard (1024 rows) 0.865, where
// the measured rate is 0.85-0.88 of the full-size rate (small shards).
static double ffn_sched_eff(int64_t Mt, int64_t Ft, int64_t Nt, int64_t kt_d, int64_t kt_f, int group, int braster,
                            int clusters) {
  if (clusters <= 0 || Mt <= 0) return 0.0;
  std::vector<double> free_at(static_cast<size_t>(clusters), 0.0);
  std::vector<double> done(static_cast<size_t>(Mt), 0.0);  // last gate/up finish per m-unit
  int64_t t = 0;
  double total = 0.0;
  auto run = [&](double dur, double ready) {
    double& f = free_at[static_cast<size_t>(t++ % clusters)];
    f = std::max(f, ready) + dur;
    total += dur;
    return f;
  };
  auto seg_a = [&](int64_t g) {
    const int64_t gs = std::min<int64_t>(group, Mt - g * group);
    for (int64_t i = 0; i < gs * Ft; ++i) {
      double& d = done[static_cast<size_t>(g * group + i % gs)];
      d = std::max(d, run(static_cast<double>(kt_d), 0.0));
    }
  };
  auto seg_b = [&](int64_t g) {
    const int64_t gs = std::min<int64_t>(group, Mt - g * group);
    const int64_t bs = braster > 0 && gs > braster ? braster : gs;
    for (int64_t mb = 0; mb < gs; mb += bs) {
      const int64_t bsz = std::min(bs, gs - mb);
      for (int64_t i = 0; i < bsz * Nt; ++i)
        run(static_cast<double>(kt_f), done[static_cast<size_t>(g * group + mb + i % bsz)]);
    }
  };
  const int64_t ngroups = cdiv(Mt, group);
  seg_a(0);
  for (int64_t s = 1; s < 2 * ngroups - 1; ++s) {
    if (s & 1)
      seg_a((s + 1) / 2);
    else
      seg_b(s / 2 - 1);
  }
  seg_b(ngroups - 1);
  const double makespan = *std::max_element(free_at.begin(), free_at.end());
  return makespan > 0 ? total / clusters / makespan : 0.0;
}

static Plan make_plan_ffn(int64_t M, int64_t D, int64_t F, int64_t N, int dtype, int schedule) {
  Plan p;
  p.pattern = kPatFfn;
  p.dtype = dtype;
  p.schedule = schedule;
  p.dev = device_info(current_device());
  p.dims[0] = M, p.dims[1] = D, p.dims[2] = F, p.dims[3] = N;
  const double eb = dtype == BF_DTYPE_BF16 ? 2.0 : 4.0;
  p.flops = 2.0 * M * static_cast<double>(F) * (2.0 * D + N);
  p.algo_bytes = eb * (static_cast<double>(M) * D + 2.0 * F * D + static_cast<double>(N) * F + static_cast<double>(M) * N);
  std::ostringstream why;
  if (dtype == BF_DTYPE_F32) {
    const bool simt = env_int("BFGPU_F32_SIMT", 0) == 1;
    p.spec = simt ? simt_gemm_spec(1) : f32x3_pair_gate(M, (F + 31) / 32 * 32) ? f32x3_pair_gate_spec() : f32x3_gemm_spec(1);
    p.units = cdiv(M, p.spec.tile_m);
    p.tiles = p.units * (cdiv(F, p.spec.tile_n) + cdiv(N, p.spec.tile_n));
    p.resident_ctas = resident_ctas(p.spec);
    p.grid = static_cast<int>(std::min<int64_t>(p.units * cdiv(F, p.spec.tile_n) * p.spec.cluster, 1 << 30));
    if (simt) {
      p.group_slab_bytes = 4.0 * M * F;
      why << "override BFGPU_F32_SIMT=1: FP32 SIMT FMA; gate/up+SwiGLU kernel then the down contraction, H "
             "materialized in the fp32 workspace (" << p.group_slab_bytes / 1e6 << " MB)";
    } else {
      p.group_slab_bytes = 8.0 * M * ((F + 31) / 32 * 32);
      why << "fp32 mode: 3xTF32 on tcgen05 (x = hi + lo, three TF32 products per K step in the fp32 TMEM "
             "accumulator); a split launch writes hi/lo of X (with the RMSNorm scale), Wt, Vt, Ut, then the "
             "gate/up GEMM (two B operands per A tile, SwiGLU epilogue writing h as hi/lo, "
          << p.group_slab_bytes / 1e6 << " MB) and the down GEMM, 128x128 tiles with the K range split over a CTA "
             "pair, chained by programmatic dependent launch";
    }
    p.notes = why.str();
    check_budgets(p);
    return p;
  }
  const bool one_sm = env_int("BFGPU_FFN_1SM", 0) == 1;
  p.spec = one_sm ? ffn1_spec() : ffn2_spec();
  if (one_sm) why << "override BFGPU_FFN_1SM=1: 1-SM kernel (M=128 MMAs); ";
  else why << "CTA-pair kernel: M=256 cta_group::2 MMAs, each CTA stages its 128 rows and half of B; ";
  const int unit = p.spec.tile_m;
  p.units = cdiv(M, unit);
  const int64_t Ft = cdiv(F, 128), Nt = cdiv(N, 256);
  // Scheduling group: the m-units that stream the same weight chunks together. Larger
  // groups read the weights fewer times; the group's slab of H (rows x F bf16) must still
  // fit in L2 so the down tiles find it there. Largest power of two with the slab <= L2
  // (measured optima: 4096 rows at C3, 2048 at C5; K1).
  const int64_t rows_fit = std::max<int64_t>(unit, static_cast<int64_t>(p.dev.l2_bytes) / (2 * F));
  int group = std::min<int64_t>(pow2_floor(rows_fit / unit), p.units);
  if (env_set("BFGPU_FFN_GROUP")) {  // historical unit: 128-row tiles
    group = std::max(1, env_int("BFGPU_FFN_GROUP", 1) * 128 / unit);
    why << "override BFGPU_FFN_GROUP; ";
  }
  p.group = std::max(1, group);
  p.group_slab_bytes = 2.0 * p.group * unit * F;
  why << "group " << p.group << " m-units (" << p.group * unit << " rows): H slab " << p.group_slab_bytes / 1e6
      << " MB vs L2 " << p.dev.l2_bytes / 1e6 << " MB; ";
  const double est = est_ms_tensor(p.flops, p.dev.sms);
  if (!one_sm) {
    // Wave sync for launches long enough to run into the board power cap: there L2
    // sharing decides the clock (C5: 1016 -> 1274 TFLOP/s). Shorter launches keep the
    // clusters free-running (C3: 1.5% faster without it) with a segment sync in the
    // fused schedule.
    const int wave_env = env_set("BFGPU_FFN_WAVESYNC") ? env_int("BFGPU_FFN_WAVESYNC", 0) : -1;
    const bool wave = wave_env >= 0 ? wave_env == 1 : est >= 4.0;
    const bool seg = !wave && schedule == BF_FFN_FUSED && env_int("BFGPU_FFN_SEGSYNC", 1) != 0;
    p.sync = wave ? kSyncWave : (seg ? kSyncSegment : kSyncNone);
    why << "est " << est << " ms at the tensor rate -> "
        << (wave ? "wave sync" : (seg ? "segment sync" : "no cross-cluster sync"))
        << (wave_env >= 0 ? " (override BFGPU_FFN_WAVESYNC)" : "") << "; ";
    p.raster = env_set("BFGPU_FFN_BRASTER") ? env_int("BFGPU_FFN_BRASTER", 8) : 8;
    why << "down tiles rastered in blocks of " << p.raster << " m-units; ";
  }
  const int64_t a_tiles = p.units * Ft, b_tiles = p.units * Nt;
  p.tiles = a_tiles + b_tiles;
  if (p.tiles >= (1ll << 31)) throw Status(BF_ERR_INVALID_ARGUMENT, "bf_rms_ffn_swiglu: too many tiles");
  finish_grid(p, schedule == BF_FFN_FUSED ? p.tiles : std::max(a_tiles, b_tiles));
  if (!one_sm) {
    p.sched_eff = ffn_sched_eff(p.units, Ft, Nt, cdiv(D, 64), cdiv(F, 64), p.group, p.raster, p.grid / 2);
    why << "modeled efficiency of the fused static schedule " << p.sched_eff << "; ";
  }
  why << (schedule == BF_FFN_FUSED
              ? "fused: one persistent launch, down tiles of an m-unit wait for its gate/up tiles"
              : "two-phase: H materialized in HBM between two launches (snapshot with one internal buffered edge)");
  p.notes = why.str();
  check_budgets(p);
  return p;
}

// ------------------------------------------------------------------ K2
static Plan make_plan_lnmm(int64_t M, int64_t K, int64_t N, int dtype, int schedule) {
  Plan p;
  p.pattern = kPatLnmm;
  p.dtype = dtype;
  p.schedule = schedule;
  p.dev = device_info(current_device());
  p.dims[0] = M, p.dims[1] = K, p.dims[2] = N;
  const double eb = dtype == BF_DTYPE_BF16 ? 2.0 : 4.0;
  p.flops = 2.0 * M * static_cast<double>(K) * N;
  p.algo_bytes = eb * (static_cast<double>(M) * K + static_cast<double>(N) * K + static_cast<double>(M) * N);
  std::ostringstream why;
  if (dtype == BF_DTYPE_F32) {
    const bool simt = env_int("BFGPU_F32_SIMT", 0) == 1;
    p.spec = simt ? simt_gemm_spec(2) : f32x3_pair(M, N) ? f32x3_pair_spec(0) : f32x3_gemm_spec(0, f32x3_wide(M, N));
    p.units = cdiv(M, p.spec.tile_m);
    p.tiles = p.units * cdiv(N, p.spec.tile_n);
    p.resident_ctas = resident_ctas(p.spec);
    p.grid = static_cast<int>(std::min<int64_t>(p.tiles * p.spec.cluster, 1 << 30));
    if (simt)
      why << "override BFGPU_F32_SIMT=1: FP32 SIMT FMA, statistics and colsum(Yt) folded into the K loop of each tile";
    else
      why << "fp32 mode: 3xTF32 on tcgen05 (x = hi + lo, hi*hi + hi*lo + lo*hi in the fp32 TMEM accumulator, "
             "~1e-6 relative at K=1024, inside the 1e-4 bar that one TF32 pass misses); a split launch computes "
             "the row statistics and colsum(Yt) and writes pivot-shifted hi/lo operands (" << 8.0 * (M + N) * ((K + 31) / 32 * 32) / 1e6
          << " MB), then " << p.tiles << " 128x" << p.spec.tile_n << " tiles, each with its K range split over a CTA pair "
             "(DSMEM reduction), on a 3-stage TMA ring";
    (void)schedule;
    p.notes = why.str();
    check_budgets(p);
    return p;
  }
  const bool one_sm = env_int("BFGPU_LNMM_1SM", 0) == 1 && schedule == BF_SCHED_FUSED;
  const bool wide = !one_sm && env_int("BFGPU_LNMM_WIDE", 0) == 1;
  p.spec = one_sm ? lnmm1_spec() : lnmm2_spec(wide);
  why << (one_sm ? "override BFGPU_LNMM_1SM=1: 1-SM kernel; "
                 : (wide ? "CTA-pair kernel, 512x256 output tiles (two M=256 MMAs per K step, single-buffered "
                           "TMEM); "
                         : "CTA-pair kernel, 256x256 output tiles; "));
  const int unit = p.spec.tile_m;
  p.units = cdiv(M, unit);
  p.tiles = p.units * cdiv(N, p.spec.tile_n);
  if (p.tiles >= (1ll << 31)) throw Status(BF_ERR_INVALID_ARGUMENT, "bf_layernorm_matmul: too many tiles");
  // Group: the X rows of one group stay in L2 while its n-tiles pass (n slow inside a group).
  // Largest power of two with the X slab <= L2/3 (C4: 16 m-units = 33.5 MB; measured
  // 2/4/8/16/32 -> 993/1382/1398/1481/1386 TFLOP/s).
  const int64_t rows_fit = std::max<int64_t>(unit, static_cast<int64_t>(p.dev.l2_bytes) / 3 / (2 * K));
  int group = std::min<int64_t>(pow2_floor(rows_fit / unit), p.units);
  if (one_sm) group = 8;
  if (env_set("BFGPU_LNMM_GROUP")) {
    group = std::max(1, env_int("BFGPU_LNMM_GROUP", 1));
    why << "override BFGPU_LNMM_GROUP; ";
  }
  p.group = std::max(1, group);
  p.group_slab_bytes = 2.0 * p.group * unit * K;
  why << "group " << p.group << " m-units: X slab " << p.group_slab_bytes / 1e6 << " MB; ";
  if (schedule == BF_SCHED_STAGED)
    why << "staged (first snapshot): the row-statistics map runs as its own launch (one warp per row of X, "
           "then of Yt), then the GEMM launch reads mu, rstd and colsum(Yt) from the workspace";
  else
    why << "row statistics and colsum(Yt) computed once inside the launch and published through the workspace "
           "(grid-wide flags: cooperative launch)";
  finish_grid(p, p.tiles);
  p.notes = why.str();
  check_budgets(p);
  return p;
}

// ------------------------------------------------------------------ K3
static Plan make_plan_attention(int64_t BH, int64_t Sq, int64_t Skv, int64_t D, int64_t Dv, int dtype,
                                int schedule) {
  Plan p;
  p.pattern = kPatAttn;
  p.dtype = dtype;
  p.schedule = schedule;
  p.dev = device_info(current_device());
  p.dims[0] = BH, p.dims[1] = Sq, p.dims[2] = Skv, p.dims[3] = D, p.dims[4] = Dv;
  const double eb = dtype == BF_DTYPE_BF16 ? 2.0 : 4.0;
  p.flops = 2.0 * BH * static_cast<double>(Sq) * Skv * (D + Dv);
  p.algo_bytes = eb * BH * (static_cast<double>(Sq) * D + static_cast<double>(Skv) * D +
                            static_cast<double>(Skv) * Dv + static_cast<double>(Sq) * Dv);
  std::ostringstream why;
  if (dtype == BF_DTYPE_F32) {
    const bool simt = env_int("BFGPU_F32_SIMT", 0) == 1;
    const bool tc = !simt && attn_f32x3_supported(D, Dv, Skv, nullptr, nullptr, nullptr, nullptr);
    const bool tiled = !tc && attn_f32_tiled_supported(D, Dv);
    p.spec = tc ? attn_f32x3_spec(static_cast<int>(D), static_cast<int>(Dv))
                : tiled ? attn_f32_tiled_spec(static_cast<int>(D), static_cast<int>(Dv)) : simt_attn_spec();
    p.units = cdiv(Sq, p.spec.tile_m);
    p.tiles = p.units * BH;
    p.resident_ctas = resident_ctas(p.spec);
    p.grid = static_cast<int>(std::min<int64_t>(p.tiles, 1 << 30));
    if (tc)
      why << "fp32 mode: 3xTF32 flash attention on tcgen05 (S = QK^T and O += PV each as three TF32 products, Q and P "
             "hi/lo in TMEM, K/V blocks split in SMEM by converter warps), one CTA per (head, 128 query rows)";
    else if (tiled)
      why << "fp32 mode: FP32 FMA flash attention, one CTA per (head, 64 query rows), key blocks of 64 in SMEM";
    else
      why << "fp32 mode: FP32 SIMT online softmax (head dims outside 64/128), one CTA per (head, 16 query rows)";
    p.notes = why.str();
    check_budgets(p);
    return p;
  }
  if (schedule == BF_SCHED_STAGED) {
    p.spec = attn_staged_spec(static_cast<int>(D), static_cast<int>(Dv));
    p.units = cdiv(Sq, p.spec.tile_m);
    p.tiles = p.units * BH;
    if (p.tiles >= (1ll << 31)) throw Status(BF_ERR_INVALID_ARGUMENT, "bf_attention: too many tiles");
    finish_grid(p, p.tiles);
    p.group_slab_bytes = 2.0 * BH * static_cast<double>(Sq) * Skv;
    why << "staged (first snapshot, P buffered): scores launch writes P = exp(S - base) per (head, 128 queries) to "
           "HBM (" << p.group_slab_bytes / 1e6 << " MB), then a persistent P.Vt GEMM launch with the 1/l row scale";
    p.notes = why.str();
    check_budgets(p);
    return p;
  }
  p.emu = env_set("BFGPU_ATTN_EMU") ? env_int("BFGPU_ATTN_EMU", 8) : 8;
  if (p.emu != 0 && p.emu != 8 && p.emu != 16) p.emu = 12;
  p.spec = attn_spec(static_cast<int>(D), static_cast<int>(Dv), p.emu);
  p.units = cdiv(Sq, p.spec.tile_m);
  p.tiles = p.units * BH;
  if (p.tiles >= (1ll << 31)) throw Status(BF_ERR_INVALID_ARGUMENT, "bf_attention: too many tiles");
  finish_grid(p, p.tiles);
  why << "persistent, one CTA per SM, tile = (head, 256 query rows) as two 128-row sub-tiles ping-ponging on the "
         "tensor pipe; S|S|O|O in TMEM (" << p.spec.tmem_cols << " columns); " << p.emu
      << "/32 exponentials on the FMA pipe" << (env_set("BFGPU_ATTN_EMU") ? " (override BFGPU_ATTN_EMU)" : "");
  p.notes = why.str();
  check_budgets(p);
  return p;
}

// Plans are pure functions of (pattern, shape, dtype, schedule, device) and the process's
// environment overrides: cache them, so a launch costs a map lookup, not a plan.
namespace {
using PlanKey = std::tuple<int, int64_t, int64_t, int64_t, int64_t, int64_t, int, int, int>;

template <class Make>
const Plan& cached_plan(const PlanKey& key, Make make) {
  static std::mutex mu;
  static std::map<PlanKey, Plan> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  Plan p = make();
  std::lock_guard<std::mutex> lk(mu);
  return cache.emplace(key, std::move(p)).first->second;
}
}  // namespace

const Plan& plan_ffn(int64_t M, int64_t D, int64_t F, int64_t N, int dtype, int schedule) {
  return cached_plan(PlanKey{kPatFfn, M, D, F, N, 0, dtype, schedule, current_device()},
                     [&] { return make_plan_ffn(M, D, F, N, dtype, schedule); });
}

const Plan& plan_lnmm(int64_t M, int64_t K, int64_t N, int dtype, int schedule) {
  return cached_plan(PlanKey{kPatLnmm, M, K, N, 0, 0, dtype, schedule, current_device()},
                     [&] { return make_plan_lnmm(M, K, N, dtype, schedule); });
}

const Plan& plan_attention(int64_t BH, int64_t Sq, int64_t Skv, int64_t D, int64_t Dv, int dtype, int schedule) {
  return cached_plan(PlanKey{kPatAttn, BH, Sq, Skv, D, Dv, dtype, schedule, current_device()},
                     [&] { return make_plan_attention(BH, Sq, Skv, D, Dv, dtype, schedule); });
}

std::string plan_json(const Plan& p) {
  static const char* pat[] = {"rms_ffn_swiglu", "layernorm_matmul", "attention"};
  static const char* sync[] = {"none", "segment", "wave"};
  static const char* sched[] = {"fused", "staged"};
  auto esc = [](const std::string& s) {
    std::string o;
    for (char c : s) {
      if (c == '"' || c == '\\') o += '\\';
      o += c;
    }
    return o;
  };
  std::ostringstream j;
  j << "{\"pattern\": \"" << pat[p.pattern] << "\", \"dtype\": \"" << (p.dtype == BF_DTYPE_BF16 ? "bf16" : "f32")
    << "\", \"schedule\": \"" << sched[p.schedule ? 1 : 0] << "\", \"kernel\": \"" << p.spec.name << "\", \"engine\": \"" << (p.spec.tensor ? "tcgen05" : "fp32-simt")
    << "\", \"dims\": [" << p.dims[0] << ", " << p.dims[1] << ", " << p.dims[2] << ", " << p.dims[3] << ", "
    << p.dims[4] << "], \"tile\": [" << p.spec.tile_m << ", " << p.spec.tile_n << ", " << p.spec.tile_k
    << "], \"cluster\": " << p.spec.cluster << ", \"threads\": " << p.spec.threads << ", \"stages\": "
    << p.spec.stages << ", \"smem_bytes\": " << p.spec.smem_bytes << ", \"smem_budget\": " << p.dev.smem_optin
    << ", \"tmem_cols\": " << p.spec.tmem_cols << ", \"tmem_budget\": 512, \"units\": " << p.units
    << ", \"tiles\": " << p.tiles << ", \"grid\": " << p.grid << ", \"resident_ctas\": " << p.resident_ctas
    << ", \"cooperative\": " << (p.spec.grid_sync ? "true" : "false") << ", \"group\": " << p.group
    << ", \"group_slab_bytes\": " << p.group_slab_bytes << ", \"raster\": " << p.raster << ", \"sched_eff\": " << p.sched_eff << ", \"sync\": \""
    << sync[p.sync] << "\", \"emu\": " << p.emu << ", \"sms\": " << p.dev.sms << ", \"l2_bytes\": " << p.dev.l2_bytes
    << ", \"flops\": " << p.flops << ", \"algo_bytes\": " << p.algo_bytes << ", \"notes\": \"" << esc(p.notes)
    << "\"}";
  return j.str();
}

}  // namespace bfgpu

using namespace bfgpu;

extern "C" int bf_plan_json(int pattern, const int64_t* dims, int ndims, int dtype, int schedule, char* buf,
                            size_t len) {
  return guarded([&] {
    BF_CHECK_ARG(dims != nullptr && buf != nullptr && len > 0, "bf_plan_json: null argument");
    BF_CHECK_ARG(dtype == BF_DTYPE_BF16 || dtype == BF_DTYPE_F32, "bf_plan_json: unknown dtype");
    Plan p;
    if (pattern == BF_PATTERN_RMS_FFN_SWIGLU) {
      BF_CHECK_ARG(ndims == 4, "bf_plan_json: rms_ffn_swiglu takes {M, D, F, N}");
      p = plan_ffn(dims[0], dims[1], dims[2], dims[3], dtype, schedule);
    } else if (pattern == BF_PATTERN_LAYERNORM_MATMUL) {
      BF_CHECK_ARG(ndims == 3, "bf_plan_json: layernorm_matmul takes {M, K, N}");
      p = plan_lnmm(dims[0], dims[1], dims[2], dtype, schedule);
    } else if (pattern == BF_PATTERN_ATTENTION) {
      BF_CHECK_ARG(ndims == 5, "bf_plan_json: attention takes {BH, Sq, Skv, D, Dv}");
      p = plan_attention(dims[0], dims[1], dims[2], dims[3], dims[4], dtype, schedule);
    } else {
      throw Status(BF_ERR_INVALID_ARGUMENT, "bf_plan_json: unknown pattern");
    }
    const std::string s = plan_json(p);
    BF_CHECK_ARG(s.size() + 1 <= len, "bf_plan_json: buffer too small (" + std::to_string(s.size() + 1) + " needed)");
    std::copy(s.begin(), s.end(), buf);
    buf[s.size()] = '\0';
  });
}
