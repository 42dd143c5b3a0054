/*
 * bfgpu.h — C-ABI of the B200 backend for Blockbuster's fused block programs.
 *
 * The reference (arXiv 2505.07829, `blockfuse`) runs every fused candidate
 * through one C++ entry point:
 *
 *   std::map<std::string, Matrix> blockfuse::execute(const BlockGraph& program,
 *       const std::map<std::string, Matrix>& inputs, const DimBinding& binding,
 *       const ExecOptions& opts = {});                 // proj/include/blockfuse/interpreter.hpp:478-487
 *
 * That walk (eval_graph -> eval_map -> eval_func, interpreter.hpp:263-472) is
 * what this library replaces for the three fully fused programs that
 * `fuse(lower(examples::X()))` emits (lowering.hpp:559-597, engine.hpp:164).
 * The C++ adapter `bfgpu::execute` (host/bfgpu_execute.hpp) keeps the
 * reference signature, recognizes the program and calls the entry points
 * below. Everything here is plain C: device pointers, sizes, a stream.
 *
 * Conventions (all entry points):
 *   - Matrices are dense row-major with the leading dimension equal to the
 *     column count. "Transposed" right operands follow the reference's block
 *     convention (lowering.hpp:159-169): Wt/Vt/Ut/Yt/K are [out, in], Vt for
 *     attention is [Dv, Skv].
 *   - All pointers are device pointers owned by the caller; outputs are
 *     fully overwritten. `stream` is a cudaStream_t (NULL = legacy stream).
 *     BF16 buffers (and workspaces) must be 16-byte aligned (TMA).
 *   - Return BF_OK (0) on success, otherwise a BF_ERR_* code; the message is
 *     available from bf_last_error() on the calling thread. This mirrors the
 *     reference's `blockfuse::Error` exceptions (ir.hpp:20-23).
 *   - Calls are reentrant per (device, stream); there is no global state
 *     besides the per-thread error string and a launch counter.
 *   - There is no CPU fallback: on a machine without an sm_100 GPU every
 *     compute entry point fails with BF_ERR_UNSUPPORTED or BF_ERR_CUDA.
 */
#ifndef BFGPU_H_
#define BFGPU_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BF_API __attribute__((visibility("default")))
#else
#define BF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BF_OK 0
#define BF_ERR_INVALID_ARGUMENT 1
#define BF_ERR_UNSUPPORTED 2
#define BF_ERR_CUDA 3
#define BF_ERR_INTERNAL 4

/* Element type of inputs and outputs. BF16 computes with fp32 accumulation
 * on the tcgen05 tensor cores; F32 is the exact fp32-in/fp32-out mode (SIMT
 * FMA, no TF32) that must match the float64 reference within 1e-4. */
#define BF_DTYPE_BF16 0
#define BF_DTYPE_F32 1

/* Schedules: which fusion snapshot of the program a launch executes.
 *   BF_SCHED_FUSED   the final snapshot of fuse(lower(examples::X())) (engine.hpp:164):
 *                    one launch, no internal buffered edge.
 *   BF_SCHED_STAGED  the first snapshot the driver emits, as its own plan:
 *                    K1  H materialized in HBM between a gate/up and a down launch;
 *                    K2  the row-statistics map (forall m: for k: sum x, sum x^2) as its
 *                        own launch before the GEMM map;
 *                    K3  P = exp(S) materialized in HBM (internal buffered edge T1) between
 *                        a scores launch and a P.Vt launch.
 * K1 FUSED: gate/up tiles hand H to the down tiles of the same m-unit inside
 * the launch, through a workspace slab that the planner sizes per scheduling
 * group. H is never re-read by a second launch, and its reads are mostly L2
 * hits, but the TMA-stored H lines do reach HBM: ncu shows DRAM writes = O + H
 * at every group size tried, including with evict-last stores and
 * discard.global.L2 after the last reader (profiles/r02_k1_h_writeback.txt). */
#define BF_SCHED_FUSED 0
#define BF_SCHED_STAGED 1
#define BF_FFN_FUSED BF_SCHED_FUSED
#define BF_FFN_TWO_PHASE BF_SCHED_STAGED

/* ------------------------------------------------------------------------
 * K1  Flash-RMSNorm + FFN-SwiGLU
 *   O = (swish(r (.) X Wt^T) (.) (r (.) X Vt^T)) Ut^T,  r_i = 1/sqrt(mean_d X_i^2 + eps)
 * Replaces: execute() on the final snapshot of fuse(lower(examples::rms_ffn_swiglu()))
 *           (lowering.hpp:583-597; dense oracle ref::rms_ffn_swiglu, interpreter.hpp:553-559).
 * Shapes: X[M,D], Wt[F,D], Vt[F,D], Ut[N,F], O[M,N]. D, F, N multiples of 8.
 * eps = 0 reproduces the reference lowering (lowering.hpp:409-411).
 * workspace: bf_rms_ffn_swiglu_workspace_bytes(...) bytes of device memory.
 * ---------------------------------------------------------------------- */
BF_API size_t bf_rms_ffn_swiglu_workspace_bytes(int64_t M, int64_t D, int64_t F, int64_t N, int dtype, int schedule);
BF_API int bf_rms_ffn_swiglu(const void* X, const void* Wt, const void* Vt, const void* Ut, void* O, int64_t M, int64_t D,
                      int64_t F, int64_t N, int dtype, float eps, int schedule, void* workspace,
                      size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * K2  Flash-LayerNorm + MatMul
 *   O = (X Yt^T - mu (x) colsum(Yt)) (.) rstd,  mu_i = mean_k X_ik,
 *   rstd_i = 1/sqrt(mean_k X_ik^2 - mu_i^2 + eps)
 * Replaces: execute() on the final snapshot of fuse(lower(examples::layernorm_matmul()))
 *           (lowering.hpp:573-581; oracle ref::layernorm_matmul, interpreter.hpp:549-551).
 * Shapes: X[M,K], Yt[N,K], O[M,N]. K, N multiples of 8. eps = 0 is the reference
 * (no eps, no gamma/beta, lowering.hpp:350-363; sigma = 0 rows give NaN like
 * the fused interpreter walk).
 * ---------------------------------------------------------------------- */
BF_API size_t bf_layernorm_matmul_workspace_bytes(int64_t M, int64_t K, int64_t N, int dtype);
BF_API int bf_layernorm_matmul(const void* X, const void* Yt, void* O, int64_t M, int64_t K, int64_t N, int dtype, float eps,
                        void* workspace, size_t workspace_bytes, void* stream);
/* Same, for either snapshot (BF_SCHED_FUSED = bf_layernorm_matmul; BF_SCHED_STAGED =
 * snapshot 1 of the driver, statistics map first, lowering.hpp:573-581). Same workspace. */
BF_API int bf_layernorm_matmul_sched(const void* X, const void* Yt, void* O, int64_t M, int64_t K, int64_t N, int dtype,
                                     float eps, int schedule, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * K3  Rediscovered FlashAttention (non-causal, no mask), online softmax
 *   O = softmax(scale * Q K^T) V, with V supplied as Vt[Dv, Skv]
 * Replaces: execute() on the final snapshot of fuse(lower(examples::attention()))
 *           (lowering.hpp:559-571) with the row-wise significand/exponent
 *           rebasing of safe_attention_rows (safe_numerics.hpp:147-175).
 * Shapes per head h in [0, BH): Q[Sq,D], K[Skv,D], Vt[Dv,Skv], O[Sq,Dv], heads
 * stored back to back. scale <= 0 selects 1/sqrt(D) (the reference's scale).
 * ---------------------------------------------------------------------- */
BF_API int bf_attention(const void* Q, const void* K, const void* Vt, void* O, int64_t BH, int64_t Sq, int64_t Skv,
                 int64_t D, int64_t Dv, int dtype, float scale, void* stream);
/* Either snapshot. BF_SCHED_FUSED needs no workspace (bf_attention). BF_SCHED_STAGED is the
 * first snapshot (P = T1 buffered; bf16 only): the workspace holds P [BH, Sq, Skv] bf16, the
 * per-(row, key block) exponent bases and 1/l, and must be 16-byte aligned. */
BF_API size_t bf_attention_workspace_bytes(int64_t BH, int64_t Sq, int64_t Skv, int64_t D, int64_t Dv, int dtype,
                                           int schedule);
BF_API int bf_attention_sched(const void* Q, const void* K, const void* Vt, void* O, int64_t BH, int64_t Sq,
                              int64_t Skv, int64_t D, int64_t Dv, int dtype, float scale, int schedule, void* workspace,
                              size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Run-time compiled kernels (any block program)
 *   Programs the fused kernels above do not cover (unfused lower() output,
 *   partial fusions, other programs) are compiled by the block-program
 *   compiler of the C++ adapter (host/bfgpu_codegen.cpp): one generated CUDA
 *   kernel per top-level operator, float64, with the numerical-safety pass
 *   (row-wise significand/exponent pairs, PAPER.md appendix). These entry
 *   points compile such source with NVRTC for sm_100a and launch it.
 * Replaces: the interpretation of eval_graph/eval_map/eval_func
 *   (interpreter.hpp:263-472): the walk happens once, at compile time.
 * bf_jit_compile: `source` is CUDA C++ with extern "C" __global__ kernels;
 *   *module stays valid for the process (cached per device and source text);
 *   the NVRTC log (warnings or errors) is copied to `log` when given.
 * bf_jit_launch: args[i] points at the i-th kernel argument (cuLaunchKernel).
 * ---------------------------------------------------------------------- */
BF_API int bf_jit_compile(const char* source, void** module, char* log, size_t log_len);
/* Compile only (NVRTC to an sm_100a cubin, discarded): needs no device. */
BF_API int bf_jit_check(const char* source, char* log, size_t log_len);
BF_API int bf_jit_launch(void* module, const char* kernel, unsigned grid_x, unsigned grid_y, unsigned block,
                         size_t dyn_smem, void* stream, void** args);

/* ------------------------------------------------------------------------
 * Device memory helpers for host bindings that do not own a CUDA runtime
 * (the C++ execute() adapter, cgo/JNI-style callers). Thin wrappers over the
 * CUDA runtime; the copies are stream-ordered and asynchronous for pinned memory.
 * ---------------------------------------------------------------------- */
BF_API void* bf_device_alloc(size_t bytes);
BF_API int bf_device_free(void* ptr);
BF_API int bf_copy_to_device(void* dst, const void* src, size_t bytes, void* stream);
BF_API int bf_copy_to_host(void* dst, const void* src, size_t bytes, void* stream);
BF_API int bf_stream_synchronize(void* stream);
/* Page-locked host memory (cudaHostAlloc, portable): staging for asynchronous copies. */
BF_API void* bf_host_alloc(size_t bytes);
BF_API int bf_host_free(void* ptr);
/* dst = src^T on the device: src is rows x cols row-major, dst cols x rows row-major,
 * elements of 2, 4 or 8 bytes, stream-ordered. A column-major (Eigen) R x C matrix is a
 * row-major C x R one, so bindings that hold column-major operands convert element types in
 * storage order on the host and let this put them in the kernels' row-major layout (and the
 * output back). Replaces the layout walk of split_into_blocks/assemble (interpreter.hpp:76-138). */
BF_API int bf_transpose(const void* src, void* dst, int64_t rows, int64_t cols, int elem_bytes, void* stream);
/* Current device of the calling thread (-1 on error) / select it. */
BF_API int bf_get_device(void);
BF_API int bf_set_device(int device);

/* ------------------------------------------------------------------------
 * Device memory / tile planner
 *   How a launch of a fused program maps onto the device: which kernel, the
 *   tile and SMEM stage ring, TMEM columns, grid and co-resident capacity,
 *   scheduling group (the L2-resident slab), cross-cluster sync, and why.
 *   The reference has no counterpart (its executor walks Eigen blocks,
 *   interpreter.hpp:319-371); the plan is the B200 reading of the fused
 *   program's map nests and port modes (ir.hpp:126-154, 265-276).
 * dims: RMS_FFN_SWIGLU {M, D, F, N}; LAYERNORM_MATMUL {M, K, N};
 *       ATTENTION {BH, Sq, Skv, D, Dv}. Writes a NUL-terminated JSON object.
 * Needs a device (the plan reads its SM count, SMEM, L2 and occupancy).
 * ---------------------------------------------------------------------- */
#define BF_PATTERN_RMS_FFN_SWIGLU 0
#define BF_PATTERN_LAYERNORM_MATMUL 1
#define BF_PATTERN_ATTENTION 2
BF_API int bf_plan_json(int pattern, const int64_t* dims, int ndims, int dtype, int schedule, char* buf,
                        size_t len);

/* ------------------------------------------------------------------------
 * Row/head-sharded multi-GPU launch (one host thread, N devices)
 *   The fused programs shard with no exchange step: rows of X for
 *   RMS_FFN_SWIGLU / LAYERNORM_MATMUL (per-row statistics; the M map is a
 *   forall, interpreter.hpp:334) and heads for ATTENTION. Shard g covers units
 *   [start, stop) of bf_shard_range (128-row aligned for rows, whole heads),
 *   runs on io[g].device with that device's pointers, and nothing crosses
 *   devices unless gather != 0: then every io[g].out_full receives the whole
 *   output (an all-gather-v: NCCL broadcasts from each shard's owner in one
 *   group over NVLink/NVSwitch when the devices are distinct, peer copies
 *   otherwise; BFGPU_GATHER=nccl|peer forces one). Reentrant per device set;
 *   concurrent execute() calls of the reference contract map to
 *   independent calls of this function.
 * Replaces: nothing in the reference (its executor is single-threaded on one
 *   host); it is the multi-GPU form of execute() for the three programs.
 * dims are the WHOLE problem's (as bf_plan_json); io[g].in[] are the shard's
 *   operands on its device: K1 {X rows, Wt, Vt, Ut}, K2 {X rows, Yt},
 *   K3 {Q, K, Vt of the shard's heads}; io[g].out the shard's output.
 *   eps_or_scale: rmsnorm/layernorm eps (K1, K2) or the softmax scale (K3).
 * ---------------------------------------------------------------------- */
typedef struct bf_shard_io {
  int device;
  const void* in[4];
  void* out;
  void* out_full;
  void* workspace;
  size_t workspace_bytes;
  void* stream;
} bf_shard_io;
BF_API int bf_shard_range(int pattern, int64_t units, int ngpu, int shard, int64_t* start, int64_t* stop);
BF_API int bf_launch_sharded(int pattern, int ngpu, const bf_shard_io* io, const int64_t* dims, int ndims, int dtype,
                             int schedule, float eps_or_scale, int gather);
/* NCCL version found at run time (libnccl.so.2 via dlopen), or -1 if none. */
BF_API int bf_nccl_version(void);

/* ------------------------------------------------------------------------
 * Introspection
 * ---------------------------------------------------------------------- */
BF_API const char* bf_last_error(void);
BF_API int bf_version(void);
/* Total kernels this library launched in the process (for launch accounting). */
BF_API uint64_t bf_kernel_launches(void);
/* 1 if device `device` is an sm_100 part this build can run on. */
BF_API int bf_device_supported(int device);

#ifdef __cplusplus
}
#endif

#endif /* BFGPU_H_ */
