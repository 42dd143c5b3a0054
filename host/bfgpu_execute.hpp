// bfgpu::execute — drop-in replacement for blockfuse::execute on B200.
//
// Same signature as the reference entry point
//   std::map<std::string, Matrix> blockfuse::execute(const BlockGraph&, const std::map<std::string, Matrix>&,
//                                                    const DimBinding&, const ExecOptions& = {})
// (proj/include/blockfuse/interpreter.hpp:478-487). Instead of walking the
// graph on the CPU in float64, it recognizes the fused candidate the fusion
// driver emitted (every snapshot of fuse(lower(examples::X())), engine.hpp:164)
// and runs it as one hand-written sm_100a kernel through the C-ABI in
// include/bfgpu.h. Any other program (unfused lower() output, partial fusions,
// programs with Misc nodes) runs on the generic float64 GPU route. There is no
// CPU fallback: every operator runs on the device.
//
// Build: against the reference headers (proj/include) and the same
// <Eigen/Dense> the reference build uses; links libbfgpu.so.
#pragma once

#include <map>
#include <string>

#include "blockfuse/interpreter.hpp"

namespace bfgpu {

enum class Precision {
  BF16,  // inputs rounded to bf16, fp32 accumulation on tcgen05 tensor cores, bf16 outputs
  F32,   // fp32 in / fp32 out on the FMA pipes (matches float64 within 1e-4)
};

// Which executor runs a program.
enum class Route {
  Auto,     // the fused sm_100a kernel if the program is a recognized fused candidate, else Generic
  Fused,    // recognized fused candidates only; anything else throws blockfuse::Error
  Generic,  // the block-program compiler (bfgpu_codegen.cpp): generated float64 kernels, any program
};

struct ExecConfig {
  Precision precision = Precision::BF16;  // fused kernels only; the generic route is float64
  void* stream = nullptr;                 // cudaStream_t; nullptr = legacy default stream
  Route route = Route::Auto;
};

enum class Pattern { RmsFfnSwiglu, LayerNormMatMul, Attention };

struct Recognized {
  Pattern pattern = Pattern::RmsFfnSwiglu;
  int snapshot = -1;                    // index into fuse(lower(example)).snapshots
  bool materializes_intermediate = false;  // snapshot keeps an internal buffered edge
  double eps = 0.0;                     // rmsnorm epsilon recovered from the program
  std::string output;                   // name of the Output node
};

// Where the time of the calling thread's last execute() on a fused kernel went.
struct ExecTiming {
  double convert_in_ms = 0;   // column-major float64 -> row-major bf16/fp32 into pinned memory (host threads),
                              // overlapped with the asynchronous uploads of the inputs before it
  double device_ms = 0;       // remaining uploads + kernel + download, after the last conversion
  double convert_out_ms = 0;  // widening the output back into the Eigen matrix
  double total_ms = 0;
  size_t h2d_bytes = 0, d2h_bytes = 0;
};
const ExecTiming& last_timing();

// Identifies `program` as one of the reference fusion driver's snapshots by the
// reference's own isomorphism test (canonical_form, serialize.hpp:370).
// Throws blockfuse::Error for anything else.
Recognized recognize(const blockfuse::BlockGraph& program);

// Any block program on the GPU in float64, compiled (host/bfgpu_codegen.cpp): one generated
// CUDA kernel per top-level operator, NVRTC-compiled for sm_100a and cached, with the
// numerical-safety pass (row-wise significand/exponent pairs; BFGPU_SAFE=0 disables it).
// Top-level Misc nodes call the executors in `opts` on host values between kernels.
std::map<std::string, blockfuse::Matrix> execute_generic(const blockfuse::BlockGraph& program,
                                                         const std::map<std::string, blockfuse::Matrix>& inputs,
                                                         const blockfuse::DimBinding& binding,
                                                         const blockfuse::ExecOptions& opts = {},
                                                         void* stream = nullptr);

// The CUDA source execute_generic generates for `program` at these inputs and binding (up to
// the first top-level Misc node), without touching a device. For inspection and tests.
std::string generic_source(const blockfuse::BlockGraph& program, const std::map<std::string, blockfuse::Matrix>& inputs,
                           const blockfuse::DimBinding& binding);

// Precision from BFGPU_PRECISION (bf16 | f32), default bf16; route from BFGPU_ROUTE
// (auto | fused | generic), default auto.
std::map<std::string, blockfuse::Matrix> execute(const blockfuse::BlockGraph& program,
                                                 const std::map<std::string, blockfuse::Matrix>& inputs,
                                                 const blockfuse::DimBinding& binding,
                                                 const blockfuse::ExecOptions& opts = {});

std::map<std::string, blockfuse::Matrix> execute(const blockfuse::BlockGraph& program,
                                                 const std::map<std::string, blockfuse::Matrix>& inputs,
                                                 const blockfuse::DimBinding& binding, const ExecConfig& cfg);

// Both of the above: route per cfg.route, Misc executors from opts (generic route).
std::map<std::string, blockfuse::Matrix> execute_routed(const blockfuse::BlockGraph& program,
                                                        const std::map<std::string, blockfuse::Matrix>& inputs,
                                                        const blockfuse::DimBinding& binding, const ExecConfig& cfg,
                                                        const blockfuse::ExecOptions& opts);

}  // namespace bfgpu
