// TEST HARNESS — compares bfgpu::execute (the drop-in adapter, GPU) against
// blockfuse::execute (the reference CPU executor) on the reference's own
// programs and random_inputs, exposed as C for tests/test_execute_gpu.py.
#include <cmath>
#include <limits>
#include <cstring>
#include <string>

#include "bfgpu_execute.hpp"
#include "blockfuse/engine.hpp"
#include "blockfuse/lowering.hpp"
#include "blockfuse/safe_numerics.hpp"

using namespace blockfuse;

namespace {

ArrayProgram example(int which, double eps) {
  if (which == 0) return examples::attention();
  if (which == 1) return examples::layernorm_matmul();
  ArrayProgram p;  // examples::rms_ffn_swiglu with an explicit rmsnorm epsilon
  NodeId x = p.input("X", "M", "D");
  NodeId wt = p.input("Wt", "K", "D", true);
  NodeId vt = p.input("Vt", "K", "D", true);
  NodeId ut = p.input("Ut", "N", "K", true);
  NodeId xn = p.op("rmsnorm", {x}, {}, eps);
  NodeId a = p.op("matmul", {xn, wt});
  NodeId b = p.op("matmul", {xn, vt});
  NodeId h = p.op("hadamard", {p.op("swish", {a}), b});
  p.output("O", p.op("matmul", {h, ut}));
  return p;
}

DimBinding parse(const char* spec) {
  DimBinding b;
  std::string s(spec);
  size_t pos = 0;
  while (pos < s.size()) {
    size_t end = s.find(',', pos);
    if (end == std::string::npos) end = s.size();
    std::string item = s.substr(pos, end - pos);
    auto eq = item.find('='), x = item.find('x');
    b.dims[item.substr(0, eq)] = {std::stoi(item.substr(eq + 1, x - eq - 1)), std::stoi(item.substr(x + 1))};
    pos = end + 1;
  }
  return b;
}

double bf16_round(double v) {
  float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

void set_msg(char* msg, int len, const std::string& s) {
  if (msg && len > 0) {
    std::strncpy(msg, s.c_str(), static_cast<size_t>(len - 1));
    msg[len - 1] = 0;
  }
}

}  // namespace

extern "C" {

// snap: fusion snapshot index, -1 final, -2 the unfused lower() program (must be rejected).
__attribute__((visibility("default"))) int bfx_compare(int which, int snap, const char* binding, int precision,
                                                       unsigned long long seed, double eps, double* rel_err,
                                                       double* norm_err, int* pattern, int* rec_snapshot,
                                                       char* msg, int msglen) {
  try {
    BlockGraph unfused = lower(example(which, eps));
    FuseResult fr = fuse(unfused);
    const BlockGraph& prog = snap == -2 ? unfused : (snap == -1 ? fr.snapshots.back().program : fr.snapshots.at(snap).program);
    DimBinding b = parse(binding);
    auto in = random_inputs(input_specs(unfused, b), seed);
    if (precision == 0)
      for (auto& [name, m] : in)
        for (long i = 0; i < m.rows(); ++i)
          for (long j = 0; j < m.cols(); ++j) m(i, j) = bf16_round(m(i, j));
    bfgpu::Recognized r = bfgpu::recognize(prog);
    *pattern = static_cast<int>(r.pattern);
    *rec_snapshot = r.snapshot;
    bfgpu::ExecConfig cfg;
    cfg.precision = precision == 0 ? bfgpu::Precision::BF16 : bfgpu::Precision::F32;
    auto got = bfgpu::execute(prog, in, b, cfg);
    auto ref = execute(prog, in, b);  // the reference CPU executor on the same program and inputs
    const Matrix& g = got.at("O");
    const Matrix& e = ref.at("O");
    double maxd = 0, maxr = 0, ss = 0;
    for (long i = 0; i < e.rows(); ++i)
      for (long j = 0; j < e.cols(); ++j) {
        maxd = std::max(maxd, std::abs(g(i, j) - e(i, j)));
        maxr = std::max(maxr, std::abs(e(i, j)));
        ss += e(i, j) * e(i, j);
      }
    *rel_err = maxd / std::max(maxr, 1e-300);
    *norm_err = maxd / std::max(std::sqrt(ss / static_cast<double>(e.size())), 1e-300);
    set_msg(msg, msglen, "ok");
    return 0;
  } catch (const std::exception& ex) {
    set_msg(msg, msglen, ex.what());
    return 1;
  }
}

// The reference's input errors through both executors on the final snapshot of `which`:
// kind 0 drops the first input, 1 adds a row to it, 2 adds a column, 3 unbinds dimension M.
// Writes blockfuse::execute's message to ref and bfgpu::execute's to ours; returns how many
// of the two threw.
__attribute__((visibility("default"))) int bfx_error_case(int which, int kind, const char* binding, char* ref,
                                                          char* ours, int len) {
  BlockGraph unfused = lower(example(which, 0.0));
  FuseResult fr = fuse(unfused);
  const BlockGraph& prog = fr.snapshots.back().program;
  DimBinding b = parse(binding);
  auto in = random_inputs(input_specs(unfused, b), 7);
  auto first = in.begin();
  if (kind == 0) {
    in.erase(first);
  } else if (kind == 1 || kind == 2) {
    Matrix& m = first->second;
    Matrix g = Matrix::Zero(m.rows() + (kind == 1), m.cols() + (kind == 2));
    g.block(0, 0, m.rows(), m.cols()) = m;
    m = g;
  } else {
    b.dims.erase("M");
  }
  int threw = 0;
  set_msg(ref, len, "no error");
  set_msg(ours, len, "no error");
  try {
    execute(prog, in, b);
  } catch (const std::exception& e) {
    set_msg(ref, len, e.what());
    ++threw;
  }
  try {
    bfgpu::execute(prog, in, b);
  } catch (const std::exception& e) {
    set_msg(ours, len, e.what());
    ++threw;
  }
  return threw;
}

// Attention snapshot `snap` on the compiled (generic) route with Q scaled by `qscale`, so the
// logits leave exp's range: max rel. error vs safe_attention_rows (safe_numerics.hpp:147)
// in *err, and the reference interpreter's own error (it overflows) in *ref_err.
__attribute__((visibility("default"))) int bfx_attention_generic(int snap, const char* binding, double qscale,
                                                                 double* err, double* ref_err, char* msg,
                                                                 int msglen) {
  try {
    BlockGraph unfused = lower(example(0, 0.0));
    FuseResult fr = fuse(unfused);
    const BlockGraph& prog = fr.snapshots.at(snap).program;
    DimBinding b = parse(binding);
    auto in = random_inputs(input_specs(unfused, b), 7);
    in["Q"] = in["Q"] * qscale;
    bfgpu::ExecConfig cfg;
    cfg.route = bfgpu::Route::Generic;
    const Matrix got = bfgpu::execute(prog, in, b, cfg).at("O");
    const Matrix safe = safe_attention_rows(in.at("Q"), in.at("K"), in.at("Vt"));
    const Matrix ref = execute(prog, in, b).at("O");
    auto rel = [&](const Matrix& m) {
      double d = 0, r = 0;
      for (long i = 0; i < safe.rows(); ++i)
        for (long j = 0; j < safe.cols(); ++j) {
          if (!std::isfinite(m(i, j))) return std::numeric_limits<double>::infinity();
          d = std::max(d, std::abs(m(i, j) - safe(i, j)));
          r = std::max(r, std::abs(safe(i, j)));
        }
      return d / std::max(r, 1e-300);
    };
    *err = rel(got);
    *ref_err = rel(ref);
    set_msg(msg, msglen, "ok");
    return 0;
  } catch (const std::exception& ex) {
    set_msg(msg, msglen, ex.what());
    return 1;
  }
}

// The block-program compiler's CUDA source for snapshot `snap` (-2: the unfused lower()
// program) at `binding` on the reference's random inputs; no device involved.
__attribute__((visibility("default"))) int bfx_generic_source(int which, int snap, const char* binding, char* out,
                                                              long outlen, char* msg, int msglen) {
  try {
    BlockGraph unfused = lower(example(which, 0.0));
    FuseResult fr = fuse(unfused);
    const BlockGraph& prog = snap == -2 ? unfused : (snap == -1 ? fr.snapshots.back().program : fr.snapshots.at(snap).program);
    DimBinding b = parse(binding);
    auto in = random_inputs(input_specs(unfused, b), 1);
    const std::string src = bfgpu::generic_source(prog, in, b);
    if (static_cast<long>(src.size()) + 1 > outlen) throw Error("source buffer too small");
    std::memcpy(out, src.c_str(), src.size() + 1);
    set_msg(msg, msglen, "ok");
    return 0;
  } catch (const std::exception& ex) {
    set_msg(msg, msglen, ex.what());
    return 1;
  }
}

__attribute__((visibility("default"))) int bfx_recognize(int which, int snap, double eps, int* pattern,
                                                         int* rec_snapshot, double* eps_out, char* msg, int msglen) {
  try {
    BlockGraph unfused = lower(example(which, eps));
    FuseResult fr = fuse(unfused);
    const BlockGraph& prog = snap == -2 ? unfused : (snap == -1 ? fr.snapshots.back().program : fr.snapshots.at(snap).program);
    bfgpu::Recognized r = bfgpu::recognize(prog);
    *pattern = static_cast<int>(r.pattern);
    *rec_snapshot = r.snapshot;
    *eps_out = r.eps;
    set_msg(msg, msglen, r.materializes_intermediate ? "materializes" : "fused");
    return 0;
  } catch (const std::exception& ex) {
    set_msg(msg, msglen, ex.what());
    return 1;
  }
}

}  // extern "C"
