// bfgpu::execute — see bfgpu_execute.hpp.
//
// Replaces the CPU walk eval_graph -> eval_map -> eval_func
// (interpreter.hpp:263-472) for the fused candidates of the three built-in
// programs. The steps mirror the reference's Input/Output handling
// (interpreter.hpp:386-420, 101-138): validate every named matrix against the
// binding totals, lay it out row-major for the device (Eigen storage is
// column-major), run the recognized kernel, and return the named output.
#include "bfgpu_execute.hpp"
#include "convert.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
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

int host_threads() {
  static const int n = [] {
    const char* v = std::getenv("BFGPU_HOST_THREADS");
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    return std::max(1, v ? std::atoi(v) : std::min(hw > 0 ? hw : 1, 32));
  }();
  return n;
}

// fn(lo, hi) over [0, n) split across the host threads (the calling thread takes the first part).
template <class Fn>
void parallel_rows(long n, long grain, Fn fn) {
  const long parts = std::max(1L, std::min<long>(host_threads(), (n + grain - 1) / grain));
  if (parts == 1) {
    fn(0L, n);
    return;
  }
  std::vector<std::thread> pool;
  for (long t = 1; t < parts; ++t) pool.emplace_back([&, t] { fn(n * t / parts, n * (t + 1) / parts); });
  fn(0L, n / parts);
  for (auto& th : pool) th.join();
}

// Column-major Eigen storage -> the same storage order in bf16/fp32 (a contiguous pass, split
// across the host threads, AVX2). `dst` is page-locked so the copy that follows is
// asynchronous; the device then transposes into the kernels' row-major layout (bf_transpose).
void narrow_in_order(const Matrix& m, Precision prec, void* dst) {
  const long n = m.rows() * m.cols();
  const double* src = m.data();
  parallel_rows(n, 1L << 16, [&](long a, long b) {
    long i = a;
    if (prec == Precision::BF16) {
      uint16_t* d = static_cast<uint16_t*>(dst);
      for (; i + 8 <= b; i += 8) _mm_storeu_si128(reinterpret_cast<__m128i*>(d + i), conv::bf16x8_from_f64(src + i));
      for (; i < b; ++i) d[i] = conv::to_bf16(static_cast<float>(src[i]));
    } else {
      float* d = static_cast<float*>(dst);
      for (; i + 4 <= b; i += 4) _mm_storeu_ps(d + i, _mm256_cvtpd_ps(_mm256_loadu_pd(src + i)));
      for (; i < b; ++i) d[i] = static_cast<float>(src[i]);
    }
  });
}

// The device already transposed the output into column-major order: widen in storage order.
void widen_in_order(const void* src, Matrix& m, Precision prec) {
  const long n = m.rows() * m.cols();
  double* dst = m.data();
  parallel_rows(n, 1L << 16, [&](long a, long b) {
    long i = a;
    if (prec == Precision::BF16) {
      const uint16_t* s16 = static_cast<const uint16_t*>(src);
      for (; i + 8 <= b; i += 8) conv::f64x8_from_bf16(s16 + i, dst + i);
      for (; i < b; ++i) dst[i] = conv::from_bf16(s16[i]);
    } else {
      const float* s32 = static_cast<const float*>(src);
      for (; i + 4 <= b; i += 4) _mm256_storeu_pd(dst + i, _mm256_cvtps_pd(_mm_loadu_ps(s32 + i)));
      for (; i < b; ++i) dst[i] = s32[i];
    }
  });
}

void check(int rc, const char* what) {
  if (rc != BF_OK) throw Error(std::string(what) + ": " + bf_last_error());
}

// Grow-only buffers, cached per thread and device: concurrent execute() calls (allowed by the
// reference contract) never share one, and repeated calls of one shape allocate
// nothing. Every call ends with a stream synchronize, so reuse by the next call is safe.
struct HostBuf {
  void* p = nullptr;
  size_t n = 0;
  ~HostBuf() {
    if (p) bf_host_free(p);
  }
  void* get(size_t bytes) {
    if (bytes > n) {
      if (p) bf_host_free(p);
      p = bf_host_alloc(bytes);
      if (!p) throw Error(std::string("pinned host allocation failed: ") + bf_last_error());
      n = bytes;
    }
    return p;
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  ~DevBuf() {
    if (p) bf_device_free(p);
  }
  void* get(size_t bytes) {
    if (bytes > n) {
      if (p) bf_device_free(p);
      p = bf_device_alloc(bytes);
      if (!p) throw Error(std::string("device allocation failed: ") + bf_last_error());
      n = bytes;
    }
    return p;
  }
};

struct Staging {
  std::map<std::string, HostBuf> host;
  std::map<std::pair<int, std::string>, DevBuf> dev;
  int device = 0;
  void* stream = nullptr;
  // Convert into a pinned buffer in Eigen's storage order, queue its asynchronous copy and the
  // device transpose into row-major: the copy of one input overlaps the conversion of the next.
  void* upload(const std::string& name, const Matrix& m, Precision prec) {
    const int eb = prec == Precision::BF16 ? 2 : 4;
    const size_t bytes = static_cast<size_t>(m.rows() * m.cols()) * eb;
    void* h = host[name].get(bytes);
    narrow_in_order(m, prec, h);
    void* staged = dev[{device, name + "/colmajor"}].get(bytes);
    check(bf_copy_to_device(staged, h, bytes, stream), "copy to device");
    void* d = dev[{device, name}].get(bytes);
    check(bf_transpose(staged, d, m.cols(), m.rows(), eb, stream), "transpose to row-major");
    return d;
  }
  void* scratch(const std::string& name, size_t bytes) { return dev[{device, name}].get(bytes); }
};

Staging& staging(void* stream) {
  thread_local Staging st;
  st.device = bf_get_device();
  if (st.device < 0) throw Error(std::string("no CUDA device: ") + bf_last_error());
  st.stream = stream;
  return st;
}

thread_local ExecTiming t_timing;

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Named input checked against the binding the way eval_graph's Input case does (interpreter.hpp:386-403).
const Matrix& input(const std::map<std::string, Matrix>& in, const std::string& name, long rows, long cols) {
  auto it = in.find(name);
  if (it == in.end()) throw Error("missing input matrix " + name);
  if (it->second.rows() != rows) throw Error("input " + name + ": row count does not match binding");
  if (it->second.cols() != cols) throw Error("input " + name + ": column count does not match binding");
  return it->second;
}

// Why the fused kernel cannot take this recognized program at this binding and precision
// (empty: it can). Mirrors the argument checks of the C-ABI entry points.
std::string unsupported_reason(const Recognized& r, const DimBinding& b, Precision prec) {
  if (r.pattern == Pattern::Attention) {
    const long D = b.total("D"), L = b.total("L"), N = b.total("N");
    if (prec == Precision::F32) return D <= 256 && L <= 256 ? "" : "fp32 attention needs head dims <= 256";
    if ((D != 64 && D != 128) || (L != 64 && L != 128)) return "bf16 attention needs head dims D, L in {64, 128}";
    if (N % 8) return "bf16 attention needs the key count a multiple of 8";
    return "";
  }
  if (prec == Precision::F32) return "";
  if (r.pattern == Pattern::LayerNormMatMul) {
    if (b.total("K") % 8 || b.total("N") % 8) return "bf16 layernorm_matmul needs K and N multiples of 8";
    return "";
  }
  if (b.total("D") % 8 || b.total("K") % 8 || b.total("N") % 8)
    return "bf16 rms_ffn_swiglu needs D, F (dim K) and N multiples of 8";
  return "";
}

// Auto-route fallbacks are reported once per reason on stderr (BFGPU_QUIET=1 silences them).
void note_fallback(const std::string& why) {
  static std::mutex mu;
  static std::set<std::string> seen;
  const char* q = std::getenv("BFGPU_QUIET");
  if (q && q[0] == '1') return;
  std::lock_guard<std::mutex> lk(mu);
  if (seen.insert(why).second)
    std::fprintf(stderr, "bfgpu::execute: %s; running it on the generic float64 GPU route\n", why.c_str());
}

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

// The reference's input errors (eval_graph's Input case, interpreter.hpp:386-403), in its order
// (top-level Input nodes in topological order), raised before any device work on every route,
// so a bad call fails the same way with or without a GPU.
void validate_inputs(const BlockGraph& g, const std::map<std::string, Matrix>& in, const DimBinding& b) {
  for (blockfuse::NodeId id : blockfuse::topological_order(g)) {
    const blockfuse::Node& n = g.node(id);
    if (n.kind != blockfuse::NodeKind::Input) continue;
    auto it = in.find(n.name);
    if (it == in.end()) throw Error("missing input matrix " + n.name);
    if (!n.rows_dim.empty() && it->second.rows() != b.total(n.rows_dim))
      throw Error("input " + n.name + ": row count does not match binding");
    if (!n.cols_dim.empty() && it->second.cols() != b.total(n.cols_dim))
      throw Error("input " + n.name + ": column count does not match binding");
  }
}

std::map<std::string, Matrix> execute_routed(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                             const DimBinding& binding, const ExecConfig& cfg,
                                             const blockfuse::ExecOptions& opts) {
  validate_inputs(program, inputs, binding);
  if (cfg.route == Route::Generic) return execute_generic(program, inputs, binding, opts, cfg.stream);
  Recognized rec;
  try {
    rec = recognize(program);
  } catch (const Error& e) {
    if (cfg.route == Route::Fused) throw;
    note_fallback("program is not a recognized fused candidate");
    return execute_generic(program, inputs, binding, opts, cfg.stream);
  }
  const std::string why = unsupported_reason(rec, binding, cfg.precision);
  if (!why.empty()) {
    if (cfg.route == Route::Fused) throw Error("bfgpu::execute: " + why);
    note_fallback(why);
    return execute_generic(program, inputs, binding, opts, cfg.stream);
  }
  const int dt = cfg.precision == Precision::BF16 ? BF_DTYPE_BF16 : BF_DTYPE_F32;
  const size_t eb = cfg.precision == Precision::BF16 ? 2 : 4;
  void* s = cfg.stream;
  Staging& st = staging(s);
  ExecTiming tm;
  const double t0 = now_ms();
  long out_rows = 0, out_cols = 0;
  void* out = nullptr;
  switch (rec.pattern) {
    case Pattern::RmsFfnSwiglu: {
      const long M = binding.total("M"), D = binding.total("D"), F = binding.total("K"), N = binding.total("N");
      const Matrix& x = input(inputs, "X", M, D);
      const Matrix& wt = input(inputs, "Wt", F, D);
      const Matrix& vt = input(inputs, "Vt", F, D);
      const Matrix& ut = input(inputs, "Ut", N, F);
      void* X = st.upload("X", x, cfg.precision);
      void* Wt = st.upload("Wt", wt, cfg.precision);
      void* Vt = st.upload("Vt", vt, cfg.precision);
      void* Ut = st.upload("Ut", ut, cfg.precision);
      tm.convert_in_ms = now_ms() - t0;
      out_rows = M;
      out_cols = N;
      out = st.scratch("O", static_cast<size_t>(M * N) * eb);
      const int sched = rec.materializes_intermediate ? BF_FFN_TWO_PHASE : BF_FFN_FUSED;
      const size_t wsb = bf_rms_ffn_swiglu_workspace_bytes(M, D, F, N, dt, sched);
      void* ws = st.scratch("ws", wsb);
      check(bf_rms_ffn_swiglu(X, Wt, Vt, Ut, out, M, D, F, N, dt, static_cast<float>(rec.eps), sched, ws, wsb, s),
            "bf_rms_ffn_swiglu");
      break;
    }
    case Pattern::LayerNormMatMul: {
      const long M = binding.total("M"), K = binding.total("K"), N = binding.total("N");
      void* X = st.upload("X", input(inputs, "X", M, K), cfg.precision);
      void* Yt = st.upload("Yt", input(inputs, "Yt", N, K), cfg.precision);
      tm.convert_in_ms = now_ms() - t0;
      out_rows = M;
      out_cols = N;
      out = st.scratch("O", static_cast<size_t>(M * N) * eb);
      const size_t wsb = bf_layernorm_matmul_workspace_bytes(M, K, N, dt);
      void* ws = st.scratch("ws", wsb);
      // snapshot 0 computes the statistics in their own map first (a distinct launch plan)
      const int sched = rec.snapshot == 0 ? BF_SCHED_STAGED : BF_SCHED_FUSED;
      check(bf_layernorm_matmul_sched(X, Yt, out, M, K, N, dt, 0.0f, sched, ws, wsb, s), "bf_layernorm_matmul");
      break;
    }
    case Pattern::Attention: {
      const long M = binding.total("M"), N = binding.total("N"), D = binding.total("D"), L = binding.total("L");
      void* Q = st.upload("Q", input(inputs, "Q", M, D), cfg.precision);
      void* K = st.upload("K", input(inputs, "K", N, D), cfg.precision);
      void* Vt = st.upload("Vt", input(inputs, "Vt", L, N), cfg.precision);
      tm.convert_in_ms = now_ms() - t0;
      out_rows = M;
      out_cols = L;
      out = st.scratch("O", static_cast<size_t>(M * L) * eb);
      // snapshot 0 buffers P (T1) between its two maps: the staged plan (bf16); fp32 mode runs the
      // fused kernel for both snapshots
      const int sched =
          rec.materializes_intermediate && cfg.precision == Precision::BF16 ? BF_SCHED_STAGED : BF_SCHED_FUSED;
      const size_t wsb = bf_attention_workspace_bytes(1, M, N, D, L, dt, sched);
      void* ws = wsb ? st.scratch("ws", wsb) : nullptr;
      check(bf_attention_sched(Q, K, Vt, out, 1, M, N, D, L, dt, 0.0f, sched, ws, wsb, s),
            "bf_attention");  // scale 1/sqrt(total(D))
      break;
    }
  }
  const size_t out_bytes = static_cast<size_t>(out_rows * out_cols) * eb;
  void* host_out = st.host["O"].get(out_bytes);
  void* out_cm = st.scratch("O/colmajor", out_bytes);  // the output in Eigen's storage order
  check(bf_transpose(out, out_cm, out_rows, out_cols, static_cast<int>(eb), s), "transpose to column-major");
  check(bf_copy_to_host(host_out, out_cm, out_bytes, s), "copy to host");
  const double t1 = now_ms();
  check(bf_stream_synchronize(s), "stream synchronize");
  const double t2 = now_ms();
  tm.device_ms = t2 - t1;
  std::map<std::string, Matrix> result;
  Matrix& o = result[rec.output];
  o.resize(out_rows, out_cols);
  widen_in_order(host_out, o, cfg.precision);
  tm.convert_out_ms = now_ms() - t2;
  tm.total_ms = now_ms() - t0;
  tm.h2d_bytes = 0;
  for (const auto& [n, m] : inputs) tm.h2d_bytes += static_cast<size_t>(m.rows() * m.cols()) * eb;
  tm.d2h_bytes = out_bytes;
  t_timing = tm;
  return result;
}

const ExecTiming& last_timing() { return t_timing; }

std::map<std::string, Matrix> execute(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                      const DimBinding& binding, const blockfuse::ExecOptions& opts) {
  ExecConfig cfg;
  cfg.precision = env_precision();
  cfg.route = env_route();
  return execute_routed(program, inputs, binding, cfg, opts);  // opts.misc serves the generic route's Misc nodes
}

}  // namespace bfgpu
