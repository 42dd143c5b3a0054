// bfgpu::execute — see bfgpu_execute.hpp.
//
// Replaces the CPU walk eval_graph -> eval_map -> eval_func
// (interpreter.hpp:263-472) for the fused candidates of the three built-in
// programs. The steps mirror the reference's Input/Output handling
// (interpreter.hpp:386-420, 101-138): validate every named matrix against the
// binding totals, lay it out row-major for the device (Eigen storage is
// column-major), run the recognized kernel, and return the named output.
#include "bfgpu_execute.hpp"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "bfgpu.h"
#include "blockfuse/engine.hpp"
#include "blockfuse/lowering.hpp"
#include "blockfuse/serialize.hpp"

namespace bfgpu {

using blockfuse::BlockGraph;
using blockfuse::DimBinding;
using blockfuse::Error;
using blockfuse::Matrix;
using blockfuse::ScalarExpr;

namespace {

// ------------------------------------------------------------------ recognition

// The fused programs the reference driver emits for the three examples
// (lowering.hpp:559-597). rms_ffn_swiglu is rebuilt with the program's own
// epsilon so the isomorphism test also covers eps != 0.
blockfuse::ArrayProgram ffn_program(double eps) {
  blockfuse::ArrayProgram p;
  blockfuse::NodeId x = p.input("X", "M", "D");
  blockfuse::NodeId wt = p.input("Wt", "K", "D", true);
  blockfuse::NodeId vt = p.input("Vt", "K", "D", true);
  blockfuse::NodeId ut = p.input("Ut", "N", "K", true);
  blockfuse::NodeId xn = p.op("rmsnorm", {x}, {}, eps);
  blockfuse::NodeId a = p.op("matmul", {xn, wt});
  blockfuse::NodeId b = p.op("matmul", {xn, vt});
  blockfuse::NodeId sw = p.op("swish", {a});
  blockfuse::NodeId h = p.op("hadamard", {sw, b});
  p.output("O", p.op("matmul", {h, ut}));
  return p;
}

struct Known {
  Pattern pattern;
  int snapshot;
  bool materializes;
  std::string canon;
};

std::vector<Known> fused_candidates(Pattern pat, const blockfuse::ArrayProgram& prog) {
  std::vector<Known> out;
  blockfuse::FuseResult r = blockfuse::fuse(blockfuse::lower(prog));
  for (size_t s = 0; s < r.snapshots.size(); ++s) {
    const BlockGraph& g = r.snapshots[s].program;
    out.push_back({pat, static_cast<int>(s), blockfuse::internal_buffered_edges(g) > 0, blockfuse::canonical_form(g)});
  }
  return out;
}

const std::vector<Known>& known_static() {
  static std::once_flag once;
  static std::vector<Known> k;
  std::call_once(once, [] {
    auto a = fused_candidates(Pattern::Attention, blockfuse::examples::attention());
    auto l = fused_candidates(Pattern::LayerNormMatMul, blockfuse::examples::layernorm_matmul());
    k.insert(k.end(), a.begin(), a.end());
    k.insert(k.end(), l.begin(), l.end());
  });
  return k;
}

std::vector<Known> known_ffn(double eps) {
  static std::mutex mu;
  static std::map<double, std::vector<Known>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(eps);
  if (it == cache.end()) it = cache.emplace(eps, fused_candidates(Pattern::RmsFfnSwiglu, ffn_program(eps))).first;
  return it->second;
}

// recip(sqrt(((x / total(D)) + eps))) is the rmsnorm scale (lowering.hpp:409-411).
bool match_rms_scale(const ScalarExpr& e, double* eps) {
  using Op = ScalarExpr::Op;
  if (e.op() != Op::Recip || e.lhs().op() != Op::Sqrt) return false;
  const ScalarExpr& add = e.lhs().lhs();
  if (add.op() != Op::Add || add.lhs().op() != Op::Div || add.rhs().op() != Op::Const) return false;
  if (add.lhs().lhs().op() != Op::Var || add.lhs().rhs().op() != Op::DimTotal) return false;
  *eps = add.rhs().value();
  return true;
}

bool find_rms_eps(const BlockGraph& g, double* eps) {
  for (const auto& [id, n] : g.nodes) {
    if (n.kind == blockfuse::NodeKind::Func && n.op.kind == blockfuse::FuncKind::Elementwise &&
        match_rms_scale(n.op.expr, eps))
      return true;
    if (n.kind == blockfuse::NodeKind::Map && find_rms_eps(*n.inner, eps)) return true;
  }
  return false;
}

std::string output_name(const BlockGraph& g) {
  for (const auto& [id, n] : g.nodes)
    if (n.kind == blockfuse::NodeKind::Output) return n.name;
  throw Error("program has no output node");
}

// ------------------------------------------------------------------ layout

uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40u);  // NaN stays NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// Column-major Eigen matrix -> row-major device layout (bf16 or fp32), tiled transpose.
std::vector<uint8_t> to_device_layout(const Matrix& m, Precision prec) {
  const long R = m.rows(), C = m.cols();
  const size_t eb = prec == Precision::BF16 ? 2 : 4;
  std::vector<uint8_t> buf(static_cast<size_t>(R * C) * eb);
  constexpr long TB = 64;
  for (long i0 = 0; i0 < R; i0 += TB)
    for (long j0 = 0; j0 < C; j0 += TB)
      for (long i = i0; i < std::min(R, i0 + TB); ++i)
        for (long j = j0; j < std::min(C, j0 + TB); ++j) {
          const float f = static_cast<float>(m(i, j));
          if (prec == Precision::BF16)
            reinterpret_cast<uint16_t*>(buf.data())[i * C + j] = to_bf16(f);
          else
            reinterpret_cast<float*>(buf.data())[i * C + j] = f;
        }
  return buf;
}

Matrix from_device_layout(const std::vector<uint8_t>& buf, long R, long C, Precision prec) {
  Matrix m(R, C);
  for (long i = 0; i < R; ++i)
    for (long j = 0; j < C; ++j)
      m(i, j) = prec == Precision::BF16 ? from_bf16(reinterpret_cast<const uint16_t*>(buf.data())[i * C + j])
                                        : reinterpret_cast<const float*>(buf.data())[i * C + j];
  return m;
}

void check(int rc, const char* what) {
  if (rc != BF_OK) throw Error(std::string(what) + ": " + bf_last_error());
}

struct DeviceBuffer {
  void* p = nullptr;
  explicit DeviceBuffer(size_t bytes) {
    p = bf_device_alloc(bytes);
    if (!p) throw Error(std::string("device allocation failed: ") + bf_last_error());
  }
  ~DeviceBuffer() {
    if (p) bf_device_free(p);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};

// Named input checked against the binding the way eval_graph's Input case does (interpreter.hpp:386-403).
const Matrix& input(const std::map<std::string, Matrix>& in, const std::string& name, long rows, long cols) {
  auto it = in.find(name);
  if (it == in.end()) throw Error("missing input matrix " + name);
  if (it->second.rows() != rows) throw Error("input " + name + ": row count does not match binding");
  if (it->second.cols() != cols) throw Error("input " + name + ": column count does not match binding");
  return it->second;
}

struct Staged {
  std::vector<std::unique_ptr<DeviceBuffer>> bufs;
  void* upload(const Matrix& m, Precision prec, void* stream) {
    std::vector<uint8_t> host = to_device_layout(m, prec);
    bufs.push_back(std::make_unique<DeviceBuffer>(host.size()));
    check(bf_copy_to_device(bufs.back()->p, host.data(), host.size(), stream), "copy to device");
    check(bf_stream_synchronize(stream), "stream synchronize");  // `host` is pageable and goes out of scope
    return bufs.back()->p;
  }
  void* alloc(size_t bytes) {
    bufs.push_back(std::make_unique<DeviceBuffer>(bytes));
    return bufs.back()->p;
  }
};

Precision env_precision() {
  const char* v = std::getenv("BFGPU_PRECISION");
  if (v && (std::strcmp(v, "f32") == 0 || std::strcmp(v, "fp32") == 0)) return Precision::F32;
  return Precision::BF16;
}

Route env_route() {
  const char* v = std::getenv("BFGPU_ROUTE");
  if (v && std::strcmp(v, "fused") == 0) return Route::Fused;
  if (v && std::strcmp(v, "generic") == 0) return Route::Generic;
  return Route::Auto;
}

}  // namespace

Recognized recognize(const BlockGraph& program) {
  const std::string canon = blockfuse::canonical_form(program);
  Recognized r;
  r.output = output_name(program);
  for (const Known& k : known_static())
    if (k.canon == canon) {
      r.pattern = k.pattern;
      r.snapshot = k.snapshot;
      r.materializes_intermediate = k.materializes;
      return r;
    }
  double eps = 0.0;
  if (find_rms_eps(program, &eps))
    for (const Known& k : known_ffn(eps))
      if (k.canon == canon) {
        r.pattern = k.pattern;
        r.snapshot = k.snapshot;
        r.materializes_intermediate = k.materializes;
        r.eps = eps;
        return r;
      }
  throw Error(
      "bfgpu::execute: program is not a recognized fused candidate (attention, layernorm_matmul or "
      "rms_ffn_swiglu snapshot of the fusion driver); no CPU fallback");
}

std::map<std::string, Matrix> execute(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                      const DimBinding& binding, const ExecConfig& cfg) {
  return execute_routed(program, inputs, binding, cfg, blockfuse::ExecOptions{});
}

std::map<std::string, Matrix> execute_routed(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                             const DimBinding& binding, const ExecConfig& cfg,
                                             const blockfuse::ExecOptions& opts) {
  if (cfg.route == Route::Generic) return execute_generic(program, inputs, binding, opts, cfg.stream);
  Recognized rec;
  try {
    rec = recognize(program);
  } catch (const Error&) {
    if (cfg.route == Route::Fused) throw;
    return execute_generic(program, inputs, binding, opts, cfg.stream);
  }
  const int dt = cfg.precision == Precision::BF16 ? BF_DTYPE_BF16 : BF_DTYPE_F32;
  const size_t eb = cfg.precision == Precision::BF16 ? 2 : 4;
  void* s = cfg.stream;
  Staged st;
  long out_rows = 0, out_cols = 0;
  void* out = nullptr;
  switch (rec.pattern) {
    case Pattern::RmsFfnSwiglu: {
      const long M = binding.total("M"), D = binding.total("D"), F = binding.total("K"), N = binding.total("N");
      void* X = st.upload(input(inputs, "X", M, D), cfg.precision, s);
      void* Wt = st.upload(input(inputs, "Wt", F, D), cfg.precision, s);
      void* Vt = st.upload(input(inputs, "Vt", F, D), cfg.precision, s);
      void* Ut = st.upload(input(inputs, "Ut", N, F), cfg.precision, s);
      out_rows = M;
      out_cols = N;
      out = st.alloc(static_cast<size_t>(M * N) * eb);
      const int sched = rec.materializes_intermediate ? BF_FFN_TWO_PHASE : BF_FFN_FUSED;
      const size_t wsb = bf_rms_ffn_swiglu_workspace_bytes(M, D, F, N, dt, sched);
      void* ws = st.alloc(wsb);
      check(bf_rms_ffn_swiglu(X, Wt, Vt, Ut, out, M, D, F, N, dt, static_cast<float>(rec.eps), sched, ws, wsb, s),
            "bf_rms_ffn_swiglu");
      break;
    }
    case Pattern::LayerNormMatMul: {
      const long M = binding.total("M"), K = binding.total("K"), N = binding.total("N");
      void* X = st.upload(input(inputs, "X", M, K), cfg.precision, s);
      void* Yt = st.upload(input(inputs, "Yt", N, K), cfg.precision, s);
      out_rows = M;
      out_cols = N;
      out = st.alloc(static_cast<size_t>(M * N) * eb);
      const size_t wsb = bf_layernorm_matmul_workspace_bytes(M, K, N, dt);
      void* ws = st.alloc(wsb);
      check(bf_layernorm_matmul(X, Yt, out, M, K, N, dt, 0.0f, ws, wsb, s), "bf_layernorm_matmul");
      break;
    }
    case Pattern::Attention: {
      const long M = binding.total("M"), N = binding.total("N"), D = binding.total("D"), L = binding.total("L");
      void* Q = st.upload(input(inputs, "Q", M, D), cfg.precision, s);
      void* K = st.upload(input(inputs, "K", N, D), cfg.precision, s);
      void* Vt = st.upload(input(inputs, "Vt", L, N), cfg.precision, s);
      out_rows = M;
      out_cols = L;
      out = st.alloc(static_cast<size_t>(M * L) * eb);
      check(bf_attention(Q, K, Vt, out, 1, M, N, D, L, dt, 0.0f, s), "bf_attention");  // scale 1/sqrt(total(D))
      break;
    }
  }
  std::vector<uint8_t> host(static_cast<size_t>(out_rows * out_cols) * eb);
  check(bf_copy_to_host(host.data(), out, host.size(), s), "copy to host");
  check(bf_stream_synchronize(s), "stream synchronize");
  std::map<std::string, Matrix> result;
  result[rec.output] = from_device_layout(host, out_rows, out_cols, cfg.precision);
  return result;
}

std::map<std::string, Matrix> execute(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                      const DimBinding& binding, const blockfuse::ExecOptions& opts) {
  ExecConfig cfg;
  cfg.precision = env_precision();
  cfg.route = env_route();
  return execute_routed(program, inputs, binding, cfg, opts);  // opts.misc serves the generic route's Misc nodes
}

}  // namespace bfgpu
