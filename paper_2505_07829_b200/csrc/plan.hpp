// Device memory / tile planner.
//
// The reference decides nothing about placement: its executor walks the block
// program with one Eigen block per operand (interpreter.hpp:319-371), and the
// fused program's map nests and port modes (ir.hpp:126-154, map_out_kind
// ir.hpp:265-276) only say WHICH values stay local to a map iteration. On the
// B200 that "local memory" has to be assigned to concrete resources, per launch:
//
//   map-local operand blocks   -> TMA-staged SMEM ring (stages x tile bytes, <= opt-in SMEM)
//   accumulating map outputs   -> TMEM accumulators (columns <= 512 per SM)
//   row statistics (t1, t2)    -> registers + a per-row workspace vector
//   broadcast operands (Wt...) -> L2 reuse across the CTAs of one scheduling group
//   buffered edges that cross  -> HBM workspace (two-phase snapshot) or the L2 group slab
//
// plan_*() makes those choices from the program, the shapes and the device
// (SM count, opt-in SMEM, L2 size, co-resident clusters), checks every budget,
// and records why. The launchers execute the plan as is; BFGPU_* environment
// variables are explicit overrides that the plan reports.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace bfgpu {

enum PatternId : int { kPatFfn = 0, kPatLnmm = 1, kPatAttn = 2 };
enum SyncKind : int { kSyncNone = 0, kSyncSegment = 1, kSyncWave = 2 };

// Static resource needs of one compiled kernel.
struct KernelSpec {
  const char* name = "";
  const void* func = nullptr;
  int threads = 0;
  int smem_bytes = 0;  // dynamic SMEM per CTA
  int tmem_cols = 0;   // TMEM columns allocated per CTA
  int cluster = 1;     // CTAs per cluster (__cluster_dims__)
  int tile_m = 0, tile_n = 0, tile_k = 0;  // output tile of one MMA unit (cluster) and its K step
  int stages = 0;                          // SMEM operand ring depth
  bool grid_sync = false;  // CTAs wait on each other through global memory: all must be co-resident
  bool tensor = true;      // tcgen05 (false: FP32 SIMT)
};

struct DeviceInfo {
  int device = 0;
  int sms = 0;
  int smem_optin = 0;  // max dynamic SMEM per CTA
  int l2_bytes = 0;
  int cc = 0;  // 100 for sm_100
};

struct Plan {
  int pattern = 0;
  int dtype = 0;
  int schedule = 0;
  KernelSpec spec;
  DeviceInfo dev;
  int64_t dims[5] = {0, 0, 0, 0, 0};
  int64_t units = 0;      // m-units (rows / tile_m) or query tiles
  int64_t tiles = 0;      // work items of the launch (all phases)
  int resident_ctas = 0;  // co-resident capacity of this kernel on the device
  int grid = 0;           // CTAs launched
  int group = 0;          // m-units per scheduling group
  int raster = 0;         // K1 down projection: m-units per raster block
  int sync = kSyncNone;
  int emu = 0;            // K3: exponentials per 32 evaluated on the FMA pipe
  double sched_eff = 0;   // K1: modeled efficiency of the static tile schedule (planner.cu)
  double flops = 0;
  double algo_bytes = 0;  // fused-minimum HBM bytes (inputs + outputs)
  double group_slab_bytes = 0;  // K1: H of one scheduling group; K2: X rows of one group
  std::string notes;      // the reasons for each choice, and any override
};

const DeviceInfo& device_info(int device);

// Raises cudaFuncAttributeMaxDynamicSharedMemorySize once per (device, kernel); thread-safe.
void ensure_smem_attr(const void* func, int bytes);

// CTAs of `k` that fit on the device at once (cluster-aware occupancy), cached per device.
int resident_ctas(const KernelSpec& k);

const Plan& plan_ffn(int64_t M, int64_t D, int64_t F, int64_t N, int dtype, int schedule);
const Plan& plan_lnmm(int64_t M, int64_t K, int64_t N, int dtype, int schedule = 0);
const Plan& plan_attention(int64_t BH, int64_t Sq, int64_t Skv, int64_t D, int64_t Dv, int dtype, int schedule = 0);
std::string plan_json(const Plan& p);

// Kernel descriptors, defined next to each kernel.
KernelSpec ffn2_spec();
KernelSpec ffn1_spec();
KernelSpec lnmm2_spec(bool wide);
KernelSpec lnmm1_spec();
KernelSpec attn_spec(int D, int Dv, int emu);
KernelSpec attn_staged_spec(int D, int Dv);
KernelSpec simt_gemm_spec(int epi);
KernelSpec f32x3_gemm_spec(int mode = 0, bool wide = false);  // 0 LayerNorm epilogue, 1 gate/up + SwiGLU, 2 plain
bool f32x3_wide(int64_t M, int64_t N);  // 128 x 256 output tiles for this launch
bool f32x3_pair(int64_t M, int64_t N);  // 256 x 256 CTA-pair tiles for this launch
KernelSpec f32x3_pair_spec(int mode);
bool f32x3_pair_gate(int64_t M, int64_t F);  // K1 fp32 gate/up GEMM on CTA pairs (opt-in)
KernelSpec f32x3_pair_gate_spec();
KernelSpec simt_attn_spec();
KernelSpec attn_f32_tiled_spec(int D, int Dv);
bool attn_f32_tiled_supported(int64_t D, int64_t Dv);
KernelSpec attn_f32x3_spec(int D, int Dv);
bool attn_f32x3_supported(int64_t D, int64_t Dv, int64_t Skv, const void* Q, const void* K, const void* Vt,
                          const void* O);  // Q == nullptr: shape check only

extern void note_launch();

// Launch `kernel` as the plan says. Kernels with grid-wide waits are launched
// cooperatively: the driver then guarantees that every CTA is resident at once
// (or rejects the launch), so a spin-wait can never wait on a CTA that was not
// scheduled, whatever else runs on other streams.
template <class... KArgs, class... Args>
void launch_planned(const Plan& pl, void (*kernel)(KArgs...), cudaStream_t stream, Args&&... args);

}  // namespace bfgpu

#include "launch.inl"
