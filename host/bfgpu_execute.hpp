// bfgpu::execute — drop-in replacement for blockfuse::execute on B200.
//
// Same signature as the reference entry point
//   std::map<std::string, Matrix> blockfuse::execute(const BlockGraph&, const std::map<std::string, Matrix>&,
//                                                    const DimBinding&, const ExecOptions& = {})
// (proj/include/blockfuse/interpreter.hpp:478-487). Instead of walking the
// graph on the CPU in float64, it recognizes the fused candidate the fusion
// driver emitted (every snapshot of fuse(lower(examples::X())), engine.hpp:164)
// and runs it as one hand-written sm_100a kernel through the C-ABI in
// include/bfgpu.h. Unrecognized programs are an error (blockfuse::Error): there
// is no CPU fallback.
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

struct ExecConfig {
  Precision precision = Precision::BF16;
  void* stream = nullptr;  // cudaStream_t; nullptr = legacy default stream
};

enum class Pattern { RmsFfnSwiglu, LayerNormMatMul, Attention };

struct Recognized {
  Pattern pattern = Pattern::RmsFfnSwiglu;
  int snapshot = -1;                    // index into fuse(lower(example)).snapshots
  bool materializes_intermediate = false;  // snapshot keeps an internal buffered edge
  double eps = 0.0;                     // rmsnorm epsilon recovered from the program
  std::string output;                   // name of the Output node
};

// Identifies `program` as one of the reference fusion driver's snapshots by the
// reference's own isomorphism test (canonical_form, serialize.hpp:370).
// Throws blockfuse::Error for anything else.
Recognized recognize(const blockfuse::BlockGraph& program);

// Precision from BFGPU_PRECISION (bf16 | f32), default bf16.
std::map<std::string, blockfuse::Matrix> execute(const blockfuse::BlockGraph& program,
                                                 const std::map<std::string, blockfuse::Matrix>& inputs,
                                                 const blockfuse::DimBinding& binding,
                                                 const blockfuse::ExecOptions& opts = {});

std::map<std::string, blockfuse::Matrix> execute(const blockfuse::BlockGraph& program,
                                                 const std::map<std::string, blockfuse::Matrix>& inputs,
                                                 const blockfuse::DimBinding& binding, const ExecConfig& cfg);

}  // namespace bfgpu
