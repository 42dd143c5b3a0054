// TEST HARNESS — compares bfgpu::execute (the drop-in adapter, GPU) against
// blockfuse::execute (the reference CPU executor) on the reference's own
// programs and random_inputs, exposed as C for tests/test_execute_gpu.py.
#include <cmath>
#include <random>
#include <vector>
#include <limits>
#include <cstring>
#include <string>

#include "bfgpu_execute.hpp"
#include "convert.hpp"
#include "blockfuse/engine.hpp"
#include "blockfuse/lowering.hpp"
#include "blockfuse/safe_numerics.hpp"
#include "test_util.hpp"  // the reference's own test programs (proj/tests, compiled in place)

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

// The adapter's AVX2 conversions against their scalar forms, bit for bit, on n values mixing
// normals of every magnitude, rounding ties, subnormals, infinities and NaNs. Returns the number
// of mismatching elements (narrowing to bf16, and widening back).
__attribute__((visibility("default"))) long bfx_conversion_check(long n, unsigned long long seed) {
  std::mt19937_64 rng(seed);
  std::vector<double> x(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) {
    const uint64_t r = rng();
    switch (r % 8) {
      case 0: x[i] = std::ldexp(static_cast<double>(static_cast<int64_t>(rng())) / 9.2e18, static_cast<int>(rng() % 300) - 150); break;
      case 1: {  // an fp32 value exactly halfway between two bf16 values (ties)
        uint32_t u = static_cast<uint32_t>(rng()) & 0xffff0000u;
        u |= 0x8000u;
        float f;
        std::memcpy(&f, &u, 4);
        x[i] = std::isfinite(f) ? f : 1.0;
        break;
      }
      case 2: x[i] = std::ldexp(1.0 + static_cast<double>(rng() % 1000) / 1000.0, -130 - static_cast<int>(rng() % 20)); break;
      case 3: x[i] = (r & 16) ? std::numeric_limits<double>::infinity() : -std::numeric_limits<double>::infinity(); break;
      case 4: x[i] = std::numeric_limits<double>::quiet_NaN(); break;
      case 5: x[i] = std::ldexp(static_cast<double>(rng() % 2000000) - 1e6, static_cast<int>(rng() % 40) - 20); break;
      case 6: x[i] = (r & 16) ? 3.4e38 * 1.01 : -3.4e38 * 1.01; break;  // rounds to +-inf in fp32
      default: x[i] = static_cast<double>(static_cast<int64_t>(rng())) / 9.2e18; break;
    }
  }
  long bad = 0;
  std::vector<uint16_t> v(static_cast<size_t>(n));
  long i = 0;
  for (; i + 8 <= n; i += 8) _mm_storeu_si128(reinterpret_cast<__m128i*>(v.data() + i), bfgpu::conv::bf16x8_from_f64(x.data() + i));
  for (; i < n; ++i) v[i] = bfgpu::conv::to_bf16(static_cast<float>(x[i]));
  for (long k = 0; k < n; ++k)
    if (v[k] != bfgpu::conv::to_bf16(static_cast<float>(x[k]))) ++bad;
  std::vector<double> w(static_cast<size_t>(n));
  for (i = 0; i + 8 <= n; i += 8) bfgpu::conv::f64x8_from_bf16(v.data() + i, w.data() + i);
  for (; i < n; ++i) w[i] = bfgpu::conv::from_bf16(v[i]);
  for (long k = 0; k < n; ++k) {
    const double e = bfgpu::conv::from_bf16(v[k]);
    if (std::memcmp(&e, &w[k], 8) != 0) ++bad;
  }
  return bad;
}

// The reference interpreter's own test programs (tests/test_interpreter.cpp:46-178, built by
// tests/test_util.hpp) through the block-program compiler, against blockfuse::execute on the
// same inputs: 0 identity elementwise, 1 row sums through a map over column blocks and a
// fold, 2 relu_matmul unfused, 3 relu_matmul fused by hand, 4 the fusion driver's final
// snapshot of relu_matmul, 5 a top-level Misc node with a host executor, 6 relu_matmul with
// its M blocks permuted (the output rows must permute the same way: iteration order does not
// matter). *err = max|ours - ref| / max|ref|.
__attribute__((visibility("default"))) int bfx_interp_case(int which, double* err, char* msg, int len) {
  try {
    BlockGraph g;
    std::map<std::string, Matrix> in;
    DimBinding b;
    ExecOptions opts;
    std::string out = "R";
    auto rnd = [](long r, long c, unsigned long long seed) {
      auto m = random_inputs({{"x", r, c}}, seed);
      return m.at("x");
    };
    switch (which) {
      case 0:
        g = bftest::single_elementwise(0, 1);
        in["a"] = rnd(4, 4, 7);
        out = "b";
        break;
      case 1: {
        NodeId x = mk_input(g, g.fresh_id(), "X", ValueDesc::list_of(Base::Block, {"K"}), "", "K");
        BlockGraph mi;
        NodeId bi = mk_boundary_in(mi, g.fresh_id());
        NodeId rs = mk_func(mi, g.fresh_id(), FuncKind::RowSum);
        NodeId bo = mk_boundary_out(mi, g.fresh_id());
        mi.connect(bi, 0, rs, 0, ValueDesc::block());
        mi.connect(rs, 0, bo, 0, ValueDesc::vector());
        NodeId m = mk_map(g, g.fresh_id(), "K", std::move(mi), {PortMode::Iterate});
        NodeId red = mk_reduce(g, g.fresh_id());
        NodeId o = mk_output(g, g.fresh_id(), "S");
        g.connect(x, 0, m, 0, ValueDesc::list_of(Base::Block, {"K"}));
        g.connect(m, 0, red, 0, ValueDesc::list_of(Base::Vector, {"K"}));
        g.connect(red, 0, o, 0, ValueDesc::vector());
        b.dims["K"] = {3, 2};
        in["X"] = rnd(4, 6, 3);
        out = "S";
        break;
      }
      case 2:
      case 3:
      case 4:
      case 6:
        g = which == 3 ? bftest::relu_matmul(true) : bftest::relu_matmul(false);
        if (which == 4) g = fuse(g).snapshots.back().program;
        b.dims["M"] = {3, 2};
        b.dims["N"] = {2, 2};
        b.free_len = 4;
        in["A"] = rnd(6, 4, 13);
        in["Bt"] = rnd(4, 4, 14);
        break;
      case 5: {
        NodeId a = mk_input(g, g.fresh_id(), "a", ValueDesc::block(), "", "");
        NodeId misc = mk_misc(g, g.fresh_id(), "reverse_rows");
        NodeId o = mk_output(g, g.fresh_id(), "b");
        g.connect(a, 0, misc, 0, ValueDesc::block());
        g.connect(misc, 0, o, 0, ValueDesc::block());
        opts.misc["reverse_rows"] = [](const std::vector<Value>& v) {
          const Matrix& m = v[0].block();
          Matrix r(m.rows(), m.cols());
          for (long i = 0; i < m.rows(); ++i)
            for (long j = 0; j < m.cols(); ++j) r(i, j) = m(m.rows() - 1 - i, j);
          return std::vector<Value>{Value(std::move(r))};
        };
        in["a"] = rnd(3, 3, 11);
        out = "b";
        break;
      }
      default:
        throw Error("unknown case");
    }
    bfgpu::ExecConfig cfg;
    cfg.precision = bfgpu::Precision::F32;
    cfg.route = bfgpu::Route::Generic;
    Matrix got = bfgpu::execute_routed(g, in, b, cfg, opts).at(out);
    Matrix ref = execute(g, in, b, opts).at(out);
    if (which == 6) {  // permute A's row blocks (2 rows each): blocks 2, 0, 1
      std::map<std::string, Matrix> inp = in;
      Matrix& a = inp["A"];
      const Matrix a0 = in.at("A");
      const int order[3] = {2, 0, 1};
      for (int blk = 0; blk < 3; ++blk)
        for (long i = 0; i < 2; ++i)
          for (long j = 0; j < a0.cols(); ++j) a(2 * blk + i, j) = a0(2 * order[blk] + i, j);
      got = bfgpu::execute_routed(g, inp, b, cfg, opts).at(out);
      Matrix perm = ref;
      for (int blk = 0; blk < 3; ++blk)
        for (long i = 0; i < 2; ++i)
          for (long j = 0; j < ref.cols(); ++j) perm(2 * blk + i, j) = ref(2 * order[blk] + i, j);
      ref = perm;
    }
    double md = 0, mr = 0;
    for (long i = 0; i < ref.rows(); ++i)
      for (long j = 0; j < ref.cols(); ++j) {
        md = std::max(md, std::abs(got(i, j) - ref(i, j)));
        mr = std::max(mr, std::abs(ref(i, j)));
      }
    *err = md / std::max(mr, 1e-300);
    set_msg(msg, len, "ok");
    return 0;
  } catch (const std::exception& e) {
    set_msg(msg, len, e.what());
    return 1;
  }
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
