// bfgpu::execute_generic — the block-program compiler: any block program on the GPU, float64.
//
// Programs the fused kernels do not cover (unfused lower() output, partial fusions, programs
// of other shapes) are compiled, not interpreted. The reference executes a block program by
// walking it (eval_graph -> eval_map -> eval_func, interpreter.hpp:263-472) with one Eigen
// value per block and a deep copy per broadcast. Here the walk happens once, at compile time:
//
//   * every value gets a static type (list nest over map dims of a block / vector / scalar,
//     with the element shape from the binding and the input matrices) and a storage layout:
//     a root input is a strided view of the caller's matrix (a block of the grid is a
//     pointer offset, never a copy), a top-level value is a dense device buffer, and a value
//     local to a map iteration lives in a per-CTA scratch stack;
//   * every top-level operator becomes one generated CUDA kernel (the reference's "one kernel
//     per top-level operator" execution model, metrics.hpp kernel_count); a top-level map
//     whose outputs are collected runs its iterations as CTAs (and a perfectly nested
//     collecting map as the grid's y dimension); nested maps become loops, accumulating map
//     outputs fold in place left to right (the reference's order), and every block operator
//     is a cooperative loop over the CTA's threads;
//   * the numerical-safety pass of the paper's appendix rewrites every
//     exponential into a significand/exponent pair with one exponent per row (the row-wise
//     form that online softmax uses) and propagates the pairs through products, sums, row
//     reductions, contractions, reciprocals and accumulating maps, rebasing additions to the
//     larger exponent; values are materialized only where they leave a map iteration or the
//     program. With it, the reference's unsafe fused attention (exp without max-subtraction)
//     stays finite for any finite input, as safe_attention_rows does (safe_numerics.hpp).
//
// The generated source is compiled once per program and binding with NVRTC for sm_100a
// (bf_jit_compile, include/bfgpu.h) and cached. Misc operators are host callbacks in the
// reference (ExecOptions::misc); at top level they run on the host between kernels, inside a
// map they are rejected.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <iomanip>
#include <memory>
#include <set>
#include <sstream>
#include <vector>

#include "bfgpu.h"
#include "bfgpu_execute.hpp"

namespace bfgpu {

using blockfuse::Base;
using blockfuse::BlockGraph;
using blockfuse::DimBinding;
using blockfuse::Edge;
using blockfuse::Error;
using blockfuse::FuncKind;
using blockfuse::MapRange;
using blockfuse::Matrix;
using blockfuse::Node;
using blockfuse::NodeId;
using blockfuse::NodeKind;
using blockfuse::OutKind;
using blockfuse::PortMode;
using blockfuse::ScalarExpr;

namespace {

void check(int rc, const char* what) {
  if (rc != BF_OK) throw Error(std::string("compiled block program, ") + what + ": " + bf_last_error());
}

// ------------------------------------------------------------------ types and storage

// Static type of a value: a list nest (outermost first) of elements; an element is a block
// rows x cols, a vector of `rows` entries (cols = 1) or a scalar (1 x 1). `se`: the element is
// a significand block with one exponent per row (a vector: one per entry).
struct Ty {
  Base base = Base::Block;
  long rows = 1, cols = 1;
  std::vector<std::pair<std::string, long>> lists;
  bool se = false;
  long elem() const { return rows * cols; }
  long count() const {
    long n = 1;
    for (auto& l : lists) n *= l.second;
    return n;
  }
  Ty element() const {
    Ty t = *this;
    t.lists.clear();
    return t;
  }
};

// Where a value lives: element (i0, i1, ...) starts at p + i0*s[0] + i1*s[1] + ..., its row r
// at + r*ld (ld = 1 for vectors). SE values keep their exponents at t + sum(ik*ts[k]) + r.
struct View {
  std::string p;
  std::vector<long> s;
  long ld = 1;
  std::string t;
  std::vector<long> ts;
  Ty ty;

  View index(const std::string& i) const {
    if (ty.lists.empty()) throw Error("compiled block program: indexing a non-list value");
    View v = *this;
    v.p = "(" + p + " + (long)(" + i + ") * " + std::to_string(s[0]) + "L)";
    v.s.erase(v.s.begin());
    if (ty.se) {
      v.t = "(" + t + " + (long)(" + i + ") * " + std::to_string(ts[0]) + "L)";
      v.ts.erase(v.ts.begin());
    }
    v.ty.lists.erase(v.ty.lists.begin());
    return v;
  }
};

std::string num(double v) {
  std::ostringstream o;
  o << std::setprecision(17) << v;
  std::string s = o.str();
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// C expression of a ScalarExpr with DimTotal resolved through the binding (scalar_expr.hpp:66-87).
std::string cexpr(const ScalarExpr& e, const DimBinding& b, const std::string& x) {
  using Op = ScalarExpr::Op;
  switch (e.op()) {
    case Op::Var: return x;
    case Op::Const: return "(" + num(e.value()) + ")";
    case Op::DimTotal: return "(" + num(static_cast<double>(b.total(e.dim()))) + ")";
    case Op::Add: return "(" + cexpr(e.lhs(), b, x) + " + " + cexpr(e.rhs(), b, x) + ")";
    case Op::Sub: return "(" + cexpr(e.lhs(), b, x) + " - " + cexpr(e.rhs(), b, x) + ")";
    case Op::Mul: return "(" + cexpr(e.lhs(), b, x) + " * " + cexpr(e.rhs(), b, x) + ")";
    case Op::Div: return "(" + cexpr(e.lhs(), b, x) + " / " + cexpr(e.rhs(), b, x) + ")";
    case Op::Exp: return "exp(" + cexpr(e.lhs(), b, x) + ")";
    case Op::Sqrt: return "sqrt(" + cexpr(e.lhs(), b, x) + ")";
    case Op::Recip: return "(1.0 / " + cexpr(e.lhs(), b, x) + ")";
    case Op::Square: return "bf_sq(" + cexpr(e.lhs(), b, x) + ")";
    case Op::Sigmoid: return "(1.0 / (1.0 + exp(-" + cexpr(e.lhs(), b, x) + ")))";
  }
  throw Error("compiled block program: bad scalar expression");
}

// The expression only scales x by a constant (x / c or x * c, c free of x): it preserves an
// exponent. Returns the multiplier's C expression.
bool scales_var(const ScalarExpr& e, const DimBinding& b, std::string* mul) {
  using Op = ScalarExpr::Op;
  auto is_const = [&](const ScalarExpr& c) {
    std::function<bool(const ScalarExpr&)> f = [&](const ScalarExpr& z) {
      if (z.op() == Op::Var) return false;
      if (z.op() == Op::Const || z.op() == Op::DimTotal) return true;
      return f(z.lhs()) && (!z.has_rhs() || f(z.rhs()));
    };
    return f(c);
  };
  if ((e.op() == Op::Div || e.op() == Op::Mul) && e.lhs().op() == Op::Var && is_const(e.rhs())) {
    *mul = e.op() == Op::Div ? "(1.0 / " + cexpr(e.rhs(), b, "0.0") + ")" : cexpr(e.rhs(), b, "0.0");
    return true;
  }
  return false;
}

// ------------------------------------------------------------------ device prelude

const char* kPrelude = R"(
// Generated by bfgpu's block-program compiler (host/bfgpu_codegen.cpp). float64.
typedef long long i64;
#define BF_NEG_INF (__longlong_as_double(0xfff0000000000000LL))
__device__ __forceinline__ double bf_sq(double v) { return v * v; }
#define BF_FOR(e, n) for (long e = threadIdx.x; e < (n); e += blockDim.x)
__device__ void k_copy(double* o, long ldo, const double* a, long lda, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = a[r * lda + c]; }
}
__device__ void k_zero(double* o, long ldo, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = 0.0; }
}
__device__ void k_add(double* o, long ldo, const double* a, long lda, const double* b, long ldb, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = a[r * lda + c] + b[r * ldb + c]; }
}
__device__ void k_mul(double* o, long ldo, const double* a, long lda, const double* b, long ldb, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = a[r * lda + c] * b[r * ldb + c]; }
}
__device__ void k_row_shift(double* o, long ldo, const double* m, long ldm, const double* v, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = m[r * ldm + c] + v[r]; }
}
__device__ void k_row_scale(double* o, long ldo, const double* m, long ldm, const double* v, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = m[r * ldm + c] * v[r]; }
}
__device__ void k_row_sum(double* o, const double* m, long ldm, long R, long C) {
  BF_FOR(r, R) { double s = 0.0; for (long c = 0; c < C; ++c) s += m[r * ldm + c]; o[r] = s; }
}
// o[R, C] = a[R, K] b[C, K]^T  (dot, interpreter.hpp:289-294): 16x16 output tiles per pass
__device__ void k_dot(double* o, long ldo, const double* a, long lda, const double* b, long ldb, long R, long C,
                      long K) {
  BF_FOR(e, R * C) {
    long r = e / C, c = e % C;
    const double* x = a + r * lda;
    const double* y = b + c * ldb;
    double s = 0.0;
    for (long k = 0; k < K; ++k) s += x[k] * y[k];
    o[r * ldo + c] = s;
  }
}
__device__ void k_outer(double* o, long ldo, const double* u, const double* v, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = u[r] * v[c]; }
}
// ---- significand/exponent pairs, one exponent per row (t == 0 when an operand is plain)
__device__ __forceinline__ double bf_t(const double* t, long r) { return t ? t[r] : 0.0; }
__device__ void se_materialize(double* o, long ldo, const double* a, long lda, const double* at, long R, long C) {
  BF_FOR(e, R * C) { long r = e / C, c = e % C; o[r * ldo + c] = a[r * lda + c] * exp(bf_t(at, r)); }
}
// o = a + b with both rows rebased to z = max(ta, tb): the exponentials stay in (0, 1]
__device__ void se_add(double* o, long ldo, double* ot, const double* a, long lda, const double* at,
                       const double* b, long ldb, const double* bt, long R, long C) {
  BF_FOR(e, R * C) {
    long r = e / C, c = e % C;
    double ta = bf_t(at, r), tb = bf_t(bt, r), z = fmax(ta, tb);
    o[r * ldo + c] = a[r * lda + c] * exp(ta - z) + b[r * ldb + c] * exp(tb - z);
  }
  __syncthreads();
  BF_FOR(r, R) ot[r] = fmax(bf_t(at, r), bf_t(bt, r));
}
// o = m + v (row shift) with m[r] and v[r] rebased to their common maximum
__device__ void se_row_shift(double* o, long ldo, double* ot, const double* m, long ldm, const double* mt,
                             const double* v, const double* vt, long R, long C) {
  BF_FOR(e, R * C) {
    long r = e / C, c = e % C;
    double ta = bf_t(mt, r), tb = bf_t(vt, r), z = fmax(ta, tb);
    o[r * ldo + c] = m[r * ldm + c] * exp(ta - z) + v[r] * exp(tb - z);
  }
  __syncthreads();
  BF_FOR(r, R) ot[r] = fmax(bf_t(mt, r), bf_t(vt, r));
}
__device__ void se_sum_t(double* ot, const double* at, const double* bt, long R, double sign) {
  BF_FOR(r, R) ot[r] = bf_t(at, r) + sign * bf_t(bt, r);
}
)";

// ------------------------------------------------------------------ the compiler

struct Kernel {
  std::string name, body;
  unsigned gx = 1, gy = 1;
  long scratch = 0;  // doubles per CTA
};

class Compiler {
 public:
  Compiler(const DimBinding& b, bool safe) : b_(b), safe_(safe) {}

  // ---- scratch stack of the kernel being emitted
  long mark() const { return sp_; }
  void release(long m) { sp_ = m; }
  std::string alloc(long n) {
    std::string p = "(S + " + std::to_string(sp_) + "L)";
    sp_ += (n + 1) & ~1L;  // 16-byte aligned
    peak_ = std::max(peak_, sp_);
    return p;
  }
  View temp(const Ty& ty) {
    View v;
    v.ty = ty;
    const long n = ty.elem();
    // dense: stride of list dim k = product of the inner extents x element size
    v.s.assign(ty.lists.size(), 0);
    long acc = n;
    for (long k = static_cast<long>(ty.lists.size()) - 1; k >= 0; --k) {
      v.s[k] = acc;
      acc *= ty.lists[k].second;
    }
    v.p = alloc(acc);
    v.ld = ty.base == Base::Block ? ty.cols : 1;
    if (ty.se) {
      long tn = ty.rows;
      v.ts.assign(ty.lists.size(), 0);
      for (long k = static_cast<long>(ty.lists.size()) - 1; k >= 0; --k) {
        v.ts[k] = tn;
        tn *= ty.lists[k].second;
      }
      v.t = alloc(tn);
    }
    return v;
  }

  std::ostringstream& out() { return code_; }
  void line(const std::string& s) { code_ << std::string(static_cast<size_t>(indent_) * 2, ' ') << s << "\n"; }
  void sync() { line("__syncthreads();"); }

  // ---- element operations (views are non-list elements)
  void copy(const View& dst, const View& src) {  // dst plain or SE-shaped like src
    if (src.ty.se && !dst.ty.se) {
      line("se_materialize(" + dst.p + ", " + L(dst.ld) + ", " + src.p + ", " + L(src.ld) + ", " + src.t + ", " +
           L(src.ty.rows) + ", " + L(src.ty.cols) + ");");
    } else {
      line("k_copy(" + dst.p + ", " + L(dst.ld) + ", " + src.p + ", " + L(src.ld) + ", " + L(src.ty.rows) + ", " +
           L(src.ty.cols) + ");");
      if (src.ty.se) line("k_copy(" + dst.t + ", 1L, " + src.t + ", 1L, " + L(src.ty.rows) + ", 1L);");
    }
    sync();
  }
  View materialize(const View& v) {
    if (!v.ty.se) return v;
    Ty t = v.ty;
    t.se = false;
    View m = temp(t);
    copy(m, v);
    return m;
  }
  // acc = acc + v, folding an accumulating map output (left to right, as eval_map)
  void accumulate(const View& acc, const View& v) {
    if (acc.ty.se || v.ty.se) {
      if (!acc.ty.se) throw Error("compiled block program: accumulator kind changed across iterations");
      Ty tt = acc.ty;
      View tmp = temp(tt);
      line("se_add(" + tmp.p + ", " + L(tmp.ld) + ", " + tmp.t + ", " + acc.p + ", " + L(acc.ld) + ", " + acc.t +
           ", " + v.p + ", " + L(v.ld) + ", " + tp(v) + ", " + L(acc.ty.rows) + ", " + L(acc.ty.cols) + ");");
      sync();
      copy(acc, tmp);
    } else {
      line("k_add(" + acc.p + ", " + L(acc.ld) + ", " + acc.p + ", " + L(acc.ld) + ", " + v.p + ", " + L(v.ld) +
           ", " + L(acc.ty.rows) + ", " + L(acc.ty.cols) + ");");
      sync();
    }
  }

  View func(const Node& n, std::vector<View> in) {
    const FuncKind k = n.op.kind;
    auto same = [&](const char* op) {
      if (in[0].ty.base != in[1].ty.base) throw Error(std::string(op) + ": operand kinds differ");
      if (in[0].ty.rows != in[1].ty.rows || in[0].ty.cols != in[1].ty.cols)
        throw Error(std::string(op) + (in[0].ty.base == Base::Block ? ": block shapes differ" : ": vector lengths differ"));
    };
    for (auto& v : in)
      if (!v.ty.lists.empty()) throw Error("compiled block program: list operand of " + std::string(func_name(k)));
    switch (k) {
      case FuncKind::Add:
      case FuncKind::Mul: {
        same(k == FuncKind::Add ? "add" : "mul");
        Ty t = in[0].ty;
        t.se = safe_ && (in[0].ty.se || in[1].ty.se);
        View o = temp(t);
        if (!t.se) {
          line(std::string(k == FuncKind::Add ? "k_add(" : "k_mul(") + o.p + ", " + L(o.ld) + ", " + in[0].p + ", " +
               L(in[0].ld) + ", " + in[1].p + ", " + L(in[1].ld) + ", " + L(t.rows) + ", " + L(t.cols) + ");");
        } else if (k == FuncKind::Add) {
          line("se_add(" + o.p + ", " + L(o.ld) + ", " + o.t + ", " + in[0].p + ", " + L(in[0].ld) + ", " + tp(in[0]) +
               ", " + in[1].p + ", " + L(in[1].ld) + ", " + tp(in[1]) + ", " + L(t.rows) + ", " + L(t.cols) + ");");
        } else {  // (s1 s2, t1 + t2)
          line("k_mul(" + o.p + ", " + L(o.ld) + ", " + in[0].p + ", " + L(in[0].ld) + ", " + in[1].p + ", " +
               L(in[1].ld) + ", " + L(t.rows) + ", " + L(t.cols) + ");");
          line("se_sum_t(" + o.t + ", " + tp(in[0]) + ", " + tp(in[1]) + ", " + L(t.rows) + ", 1.0);");
        }
        sync();
        return o;
      }
      case FuncKind::RowShift:
      case FuncKind::RowScale: {
        if (in[0].ty.base != Base::Block || in[1].ty.base != Base::Vector)
          throw Error(std::string(func_name(k)) + ": expects a block and a vector");
        if (in[1].ty.rows != in[0].ty.rows)
          throw Error(std::string(func_name(k)) + ": vector length must equal block row count");
        Ty t = in[0].ty;
        t.se = safe_ && (in[0].ty.se || in[1].ty.se);
        View o = temp(t);
        const std::string R = L(t.rows), C = L(t.cols);
        if (!t.se) {
          line(std::string(k == FuncKind::RowShift ? "k_row_shift(" : "k_row_scale(") + o.p + ", " + L(o.ld) + ", " +
               in[0].p + ", " + L(in[0].ld) + ", " + in[1].p + ", " + R + ", " + C + ");");
        } else if (k == FuncKind::RowShift) {
          line("se_row_shift(" + o.p + ", " + L(o.ld) + ", " + o.t + ", " + in[0].p + ", " + L(in[0].ld) + ", " +
               tp(in[0]) + ", " + in[1].p + ", " + tp(in[1]) + ", " + R + ", " + C + ");");
        } else {
          line("k_row_scale(" + o.p + ", " + L(o.ld) + ", " + in[0].p + ", " + L(in[0].ld) + ", " + in[1].p + ", " + R +
               ", " + C + ");");
          line("se_sum_t(" + o.t + ", " + tp(in[0]) + ", " + tp(in[1]) + ", " + R + ", 1.0);");
        }
        sync();
        return o;
      }
      case FuncKind::RowSum: {
        if (in[0].ty.base != Base::Block) throw Error("row_sum: expects a block");
        Ty t;
        t.base = Base::Vector;
        t.rows = in[0].ty.rows;
        t.se = in[0].ty.se;
        View o = temp(t);
        line("k_row_sum(" + o.p + ", " + in[0].p + ", " + L(in[0].ld) + ", " + L(in[0].ty.rows) + ", " +
             L(in[0].ty.cols) + ");");
        if (t.se) line("k_copy(" + o.t + ", 1L, " + in[0].t + ", 1L, " + L(t.rows) + ", 1L);");
        sync();
        return o;
      }
      case FuncKind::Dot: {
        if (in[0].ty.base != Base::Block || in[1].ty.base != Base::Block) throw Error("dot: expects two blocks");
        if (in[0].ty.cols != in[1].ty.cols) throw Error("dot: column counts must match");
        const View b = materialize(in[1]);  // an exponent per row of b would land on output columns
        Ty t;
        t.rows = in[0].ty.rows;
        t.cols = b.ty.rows;
        t.se = in[0].ty.se;
        View o = temp(t);
        line("k_dot(" + o.p + ", " + L(o.ld) + ", " + in[0].p + ", " + L(in[0].ld) + ", " + b.p + ", " + L(b.ld) +
             ", " + L(t.rows) + ", " + L(t.cols) + ", " + L(in[0].ty.cols) + ");");
        if (t.se) line("k_copy(" + o.t + ", 1L, " + in[0].t + ", 1L, " + L(t.rows) + ", 1L);");
        sync();
        return o;
      }
      case FuncKind::Outer: {
        if (in[0].ty.base != Base::Vector || in[1].ty.base != Base::Vector) throw Error("outer: expects two vectors");
        const View v = materialize(in[1]);
        Ty t;
        t.rows = in[0].ty.rows;
        t.cols = v.ty.rows;
        t.se = in[0].ty.se;
        View o = temp(t);
        line("k_outer(" + o.p + ", " + L(o.ld) + ", " + in[0].p + ", " + v.p + ", " + L(t.rows) + ", " + L(t.cols) +
             ");");
        if (t.se) line("k_copy(" + o.t + ", 1L, " + in[0].t + ", 1L, " + L(t.rows) + ", 1L);");
        sync();
        return o;
      }
      case FuncKind::Elementwise: return elementwise(n.op.expr, in[0]);
    }
    throw Error("compiled block program: bad func kind");
  }

  View elementwise(const ScalarExpr& e, const View& a) {
    using Op = ScalarExpr::Op;
    const std::string R = L(a.ty.rows), C = L(a.ty.cols);
    std::string mul;
    if (safe_ && a.ty.se) {
      Ty t = a.ty;
      View o = temp(t);
      if (e.op() == Op::Recip && e.lhs().op() == Op::Var) {  // (s, t)^-1 = (1/s, -t)
        line("BF_FOR(e, " + R + " * " + C + ") { long r = e / " + C + ", c = e % " + C + "; " + o.p + "[r * " +
             L(o.ld) + " + c] = 1.0 / " + a.p + "[r * " + L(a.ld) + " + c]; }");
        line("se_sum_t(" + o.t + ", nullptr, " + a.t + ", " + R + ", -1.0);");
        sync();
        return o;
      }
      if (scales_var(e, b_, &mul)) {  // (s, t) * c = (s c, t)
        line("BF_FOR(e, " + R + " * " + C + ") { long r = e / " + C + ", c = e % " + C + "; " + o.p + "[r * " +
             L(o.ld) + " + c] = " + a.p + "[r * " + L(a.ld) + " + c] * " + mul + "; }");
        line("k_copy(" + o.t + ", 1L, " + a.t + ", 1L, " + R + ", 1L);");
        sync();
        return o;
      }
      return elementwise(e, materialize(a));
    }
    if (safe_ && e.op() == Op::Exp) {
      // e^f(x) as (e^(f(x) - z), z), z = the row maximum of f(x): one exponent per row
      Ty t = a.ty;
      t.se = true;
      View o = temp(t);
      const std::string f = cexpr(e.lhs(), b_, a.p + "[r * " + L(a.ld) + " + c]");
      line("BF_FOR(r, " + R + ") {");
      line("  double z = BF_NEG_INF;");
      line("  for (long c = 0; c < " + C + "; ++c) z = fmax(z, " + f + ");");
      line("  if (!(z > BF_NEG_INF)) z = 0.0;  // a row of -inf (or NaN) keeps its exponent at 0");
      line("  for (long c = 0; c < " + C + "; ++c) " + o.p + "[r * " + L(o.ld) + " + c] = exp(" + f + " - z);");
      line("  " + o.t + "[r] = z;");
      line("}");
      sync();
      return o;
    }
    View o = temp(a.ty);
    line("BF_FOR(e, " + R + " * " + C + ") { long r = e / " + C + ", c = e % " + C + "; " + o.p + "[r * " +
         L(o.ld) + " + c] = " + cexpr(e, b_, a.p + "[r * " + L(a.ld) + " + c]") + "; }");
    sync();
    return o;
  }

  // Reduce over a list (left fold from the first element, interpreter.hpp:441-451).
  View reduce(const View& in) {
    if (in.ty.lists.empty()) return in;  // accumulator form: folded by the enclosing map
    const long n = in.ty.lists[0].second;
    if (n == 0) throw Error("reduction over empty list");
    Ty et = in.ty;
    et.lists.erase(et.lists.begin());
    if (!et.lists.empty()) throw Error("reduction over nested lists is not defined");
    View acc = temp(et);
    copy(acc, in.index("0"));
    const std::string i = fresh("ri");
    line("for (long " + i + " = 1; " + i + " < " + L(n) + "; ++" + i + ") {");
    ++indent_;
    accumulate(acc, in.index(i));
    --indent_;
    line("}");
    return acc;
  }

  // A nested map: a loop over its iterations; collected outputs go to list temps, accumulating
  // outputs fold in place (eval_map, interpreter.hpp:319-371).
  std::vector<View> map(const Node& n, const std::vector<View>& in) {
    const BlockGraph& g = *n.inner;
    const long count = b_.count(n.dim);
    const long begin = n.range == MapRange::Rest ? 1 : 0;
    const long end = n.range == MapRange::First ? 1 : count;
    for (size_t p = 0; p < n.in_modes.size(); ++p)
      if (n.in_modes[p] == PortMode::Iterate) {
        if (in[p].ty.lists.empty() || in[p].ty.lists[0].second != count)
          throw Error("map over " + n.dim + ": iterated list length " +
                      std::to_string(in[p].ty.lists.empty() ? 0 : in[p].ty.lists[0].second) +
                      " does not match block count " + std::to_string(count));
      }
    // element types of the outputs: compile the body once on a throwaway emission to learn them
    std::vector<Ty> ety = body_types(n, in);
    const int nout = static_cast<int>(g.boundary_out.size());
    std::vector<View> outs(nout);
    const long extent = std::max(0L, end - begin);
    for (int p = 0; p < nout; ++p) {
      if (blockfuse::map_out_kind(n, p) == OutKind::Collect) {
        Ty t = ety[p];
        t.se = false;
        t.lists.insert(t.lists.begin(), {n.dim, extent});
        outs[p] = temp(t);
      } else {
        Ty t = ety[p];
        t.se = safe_ && t.se;
        outs[p] = temp(t);
      }
    }
    if (extent == 0) {
      if (count < 1) throw Error("map over " + n.dim + ": empty iteration range leaves accumulator undefined");
      for (int p = 0; p < nout; ++p)  // empty range: accumulators are the reduction's zero
        if (blockfuse::map_out_kind(n, p) == OutKind::Accumulate) zero(outs[p]);
      return outs;
    }
    const std::string i = fresh("i");
    line("for (long " + i + " = " + L(begin) + "; " + i + " < " + L(end) + "; ++" + i + ") {");
    ++indent_;
    body(n, in, i, begin, outs);
    --indent_;
    line("}");
    return outs;
  }

  // One iteration of map `n` with index variable `i`: evaluates the inner graph and stores its
  // boundary outputs into `outs` (collect slot i - begin, or fold into the accumulator).
  void body(const Node& n, const std::vector<View>& in, const std::string& i, long begin,
            const std::vector<View>& outs) {
    const BlockGraph& g = *n.inner;
    std::vector<View> bvals;
    for (size_t p = 0; p < n.in_modes.size(); ++p)
      bvals.push_back(n.in_modes[p] == PortMode::Iterate ? in[p].index(i) : in[p]);
    const long m = mark();
    std::vector<View> res = graph(g, bvals);
    for (size_t p = 0; p < res.size(); ++p) {
      if (blockfuse::map_out_kind(n, static_cast<int>(p)) == OutKind::Collect) {
        copy(outs[p].index("(" + i + " - " + L(begin) + ")"), res[p]);
      } else {
        line("if (" + i + " == " + L(begin) + ") {");
        ++indent_;
        copy(outs[p], res[p]);
        --indent_;
        line("} else {");
        ++indent_;
        accumulate(outs[p], res[p]);
        --indent_;
        line("}");
      }
    }
    release(m);
  }

  std::vector<Ty> body_types(const Node& n, const std::vector<View>& in) {
    // emit into a scratch buffer and discard: types are a pure function of the inputs
    std::ostringstream saved;
    saved << code_.str();
    const long sp = sp_, peak = peak_;
    const int ind = indent_, fid = fid_;
    std::vector<View> bvals;
    for (size_t p = 0; p < n.in_modes.size(); ++p)
      bvals.push_back(n.in_modes[p] == PortMode::Iterate ? in[p].index("0") : in[p]);
    std::vector<View> res = graph(*n.inner, bvals);
    std::vector<Ty> t;
    for (auto& v : res) t.push_back(v.ty);
    code_.str("");
    code_ << saved.str();
    sp_ = sp;
    peak_ = peak;
    indent_ = ind;
    fid_ = fid;
    return t;
  }

  void zero(const View& v) {
    const long n = v.ty.count();
    line("k_zero(" + v.p + ", 1L, 1L, " + L(n * v.ty.elem()) + ");");
    if (v.ty.se) line("k_zero(" + v.t + ", 1L, 1L, " + L(n * v.ty.rows) + ");");
    sync();
  }

  // Evaluates a graph level in topological order (the reference's order, ir.hpp:328).
  std::vector<View> graph(const BlockGraph& g, const std::vector<View>& boundary) {
    std::map<std::pair<NodeId, int>, View> vals;
    auto input_of = [&](NodeId id, int port) -> const View& {
      const Edge* e = g.producer(id, port);
      if (!e) throw Error("node " + std::to_string(id) + ": missing producer");
      auto it = vals.find({e->src.node, e->src.port});
      if (it == vals.end()) throw Error("value not yet computed");
      return it->second;
    };
    for (NodeId id : blockfuse::topological_order(g)) {
      const Node& n = g.node(id);
      switch (n.kind) {
        case NodeKind::BoundaryIn:
          vals[{id, 0}] =
              boundary.at(std::find(g.boundary_in.begin(), g.boundary_in.end(), id) - g.boundary_in.begin());
          break;
        case NodeKind::BoundaryOut: break;
        case NodeKind::Func: {
          std::vector<View> in;
          for (int p = 0; p < blockfuse::func_arity(n.op.kind); ++p) in.push_back(input_of(id, p));
          vals[{id, 0}] = func(n, in);
          break;
        }
        case NodeKind::Reduce: vals[{id, 0}] = reduce(input_of(id, 0)); break;
        case NodeKind::Map: {
          std::vector<View> in;
          for (int p = 0; p < blockfuse::map_in_count(n); ++p) in.push_back(input_of(id, p));
          std::vector<View> outs = map(n, in);
          for (size_t p = 0; p < outs.size(); ++p) vals[{id, static_cast<int>(p)}] = outs[p];
          break;
        }
        case NodeKind::Misc:
          throw Error("compiled block program: misc operator " + n.name +
                      " inside a map is not supported on the GPU (top-level misc operators run on the host)");
        case NodeKind::Input:
        case NodeKind::Output: throw Error("input/output node in inner graph");
      }
    }
    std::vector<View> out;
    for (NodeId bo : g.boundary_out) out.push_back(input_of(bo, 0));
    return out;
  }

  // ---- kernels for top-level operators
  Kernel top_map(const Node& n, const std::vector<View>& in, const std::vector<View>& gouts, const std::string& name) {
    begin_kernel();
    const long count = b_.count(n.dim);
    const long begin = n.range == MapRange::Rest ? 1 : 0;
    const long end = n.range == MapRange::First ? 1 : count;
    const long extent = std::max(0L, end - begin);
    bool collect_all = extent > 0;
    for (size_t p = 0; p < gouts.size(); ++p)
      if (blockfuse::map_out_kind(n, static_cast<int>(p)) != OutKind::Collect) collect_all = false;
    Kernel k;
    k.name = name;
    if (!collect_all) {
      // accumulating (or empty) top-level map: one CTA runs the iterations in order
      std::vector<View> outs = map(n, in);
      for (size_t p = 0; p < outs.size(); ++p) copy_global(gouts[p], outs[p]);
    } else {
      // iterations are independent: one CTA each (grid x), and a perfectly nested collecting
      // map of the body spreads over grid y
      const Node* inner = perfect_inner(n);
      line("const long i0 = " + L(begin) + " + (long)blockIdx.x;");
      k.gx = static_cast<unsigned>(extent);
      if (inner) {
        const long c2 = b_.count(inner->dim);
        const long b2 = inner->range == MapRange::Rest ? 1 : 0;
        const long e2 = inner->range == MapRange::First ? 1 : c2;
        k.gy = static_cast<unsigned>(e2 - b2);
        line("const long i1 = " + L(b2) + " + (long)blockIdx.y;");
        // inputs of the inner map, in terms of the outer boundary (perfect nesting: boundary
        // ports feed the inner map directly, its outputs feed the boundary outputs)
        std::vector<View> outer_b;
        for (size_t p = 0; p < n.in_modes.size(); ++p)
          outer_b.push_back(n.in_modes[p] == PortMode::Iterate ? in[p].index("i0") : in[p]);
        std::vector<View> inner_in = perfect_inputs(n, *inner, outer_b);
        std::vector<View> inner_out;
        for (size_t p = 0; p < gouts.size(); ++p) inner_out.push_back(gouts[p].index("(i0 - " + L(begin) + ")"));
        std::vector<View> sel(inner_out.size());
        for (size_t p = 0; p < inner_out.size(); ++p) sel[p] = inner_out[perfect_out_port(n, *inner, p)];
        body_global(*inner, inner_in, "i1", b2, sel);
      } else {
        std::vector<View> gsel;
        for (auto& v : gouts) gsel.push_back(v);
        body_global(n, in, "i0", begin, gsel);
      }
    }
    finish_kernel(k);
    return k;
  }

  Kernel top_func(const Node& n, const std::vector<View>& in, const View& gout, const std::string& name) {
    begin_kernel();
    Kernel k;
    k.name = name;
    View v = n.kind == NodeKind::Reduce ? reduce(in[0]) : func(n, in);
    copy_global(gout, v);
    finish_kernel(k);
    return k;
  }

  // element type of a top-level operator's outputs (dry run)
  std::vector<Ty> top_types(const Node& n, const std::vector<View>& in) {
    begin_kernel();
    std::vector<Ty> t;
    if (n.kind == NodeKind::Map) {
      for (auto& v : map(n, in)) t.push_back(v.ty);
    } else {
      View v = n.kind == NodeKind::Reduce ? reduce(in[0]) : func(n, in);
      t.push_back(v.ty);
    }
    code_.str("");
    return t;
  }

 private:
  static std::string L(long v) { return std::to_string(v) + "L"; }
  std::string tp(const View& v) const { return v.ty.se ? v.t : "nullptr"; }
  std::string fresh(const char* base) { return std::string(base) + "_" + std::to_string(fid_++); }

  void begin_kernel() {
    code_.str("");
    sp_ = peak_ = 0;
    indent_ = 1;
  }
  void finish_kernel(Kernel& k) {
    k.body = code_.str();
    k.scratch = peak_;
  }

  // a global (top-level) value receives a list or element computed in the kernel
  void copy_global(const View& dst, const View& src) {
    if (src.ty.lists.empty()) {
      copy(dst, src);
      return;
    }
    const std::string i = fresh("g");
    line("for (long " + i + " = 0; " + i + " < " + L(src.ty.lists[0].second) + "; ++" + i + ") {");
    ++indent_;
    copy_global(dst.index(i), src.index(i));
    --indent_;
    line("}");
  }

  // body of a gridded map: iteration index is a kernel coordinate, collected outputs land in
  // the global output views directly
  void body_global(const Node& n, const std::vector<View>& in, const std::string& i, long begin,
                   const std::vector<View>& gouts) {
    std::vector<View> bvals;
    for (size_t p = 0; p < n.in_modes.size(); ++p)
      bvals.push_back(n.in_modes[p] == PortMode::Iterate ? in[p].index(i) : in[p]);
    std::vector<View> res = graph(*n.inner, bvals);
    for (size_t p = 0; p < res.size(); ++p) copy_global(gouts[p].index("(" + i + " - " + L(begin) + ")"), res[p]);
  }

  // The body of top-level map `n` is exactly one collecting map fed by boundary ports and
  // feeding all boundary outputs (like forall m { forall l { ... } }): return it.
  const Node* perfect_inner(const Node& n) const {
    const BlockGraph& g = *n.inner;
    const Node* inner = nullptr;
    for (const auto& [id, nd] : g.nodes) {
      if (nd.kind == NodeKind::BoundaryIn || nd.kind == NodeKind::BoundaryOut) continue;
      if (nd.kind != NodeKind::Map || inner) return nullptr;
      inner = &nd;
    }
    if (!inner || inner->range != MapRange::Full) return nullptr;
    for (int p = 0; p < blockfuse::map_out_count(*inner); ++p)
      if (blockfuse::map_out_kind(*inner, p) != OutKind::Collect) return nullptr;
    if (static_cast<int>(g.boundary_out.size()) != blockfuse::map_out_count(*inner)) return nullptr;
    for (NodeId bo : g.boundary_out) {
      const Edge* e = g.producer(bo, 0);
      if (!e || e->src.node != inner->id) return nullptr;
    }
    for (int p = 0; p < blockfuse::map_in_count(*inner); ++p) {
      const Edge* e = g.producer(inner->id, p);
      if (!e || g.node(e->src.node).kind != NodeKind::BoundaryIn) return nullptr;
    }
    return inner;
  }
  std::vector<View> perfect_inputs(const Node& n, const Node& inner, const std::vector<View>& outer_b) const {
    const BlockGraph& g = *n.inner;
    std::vector<View> r;
    for (int p = 0; p < blockfuse::map_in_count(inner); ++p) {
      const Edge* e = g.producer(inner.id, p);
      const long k = std::find(g.boundary_in.begin(), g.boundary_in.end(), e->src.node) - g.boundary_in.begin();
      r.push_back(outer_b.at(static_cast<size_t>(k)));
    }
    return r;
  }
  // inner map output port feeding boundary output p
  size_t perfect_out_port(const Node& n, const Node& inner, size_t p) const {
    (void)inner;
    const BlockGraph& g = *n.inner;
    // boundary outputs in order; find the boundary-out whose producer port is p
    for (size_t q = 0; q < g.boundary_out.size(); ++q)
      if (g.producer(g.boundary_out[q], 0)->src.port == static_cast<int>(p)) return q;
    throw Error("compiled block program: inconsistent perfect nest");
  }

  const DimBinding& b_;
  bool safe_;
  std::ostringstream code_;
  long sp_ = 0, peak_ = 0;
  int indent_ = 1;
  int fid_ = 0;
};

// ------------------------------------------------------------------ device buffers

struct Buf {
  double* p = nullptr;
  ~Buf() {
    if (p) bf_device_free(p);
  }
};

double* device_alloc(std::vector<std::unique_ptr<Buf>>& keep, size_t n) {
  auto b = std::make_unique<Buf>();
  b->p = static_cast<double*>(bf_device_alloc(std::max<size_t>(n, 1) * sizeof(double)));
  if (!b->p) throw Error(std::string("compiled block program: device allocation failed: ") + bf_last_error());
  double* p = b->p;
  keep.push_back(std::move(b));
  return p;
}

// A dense top-level buffer for a value of type `t`, registered as bufs[slot].
View global_view(const Ty& t, int slot) {
  View v;
  v.ty = t;
  v.ty.se = false;
  v.s.assign(t.lists.size(), 0);
  long acc = t.elem();
  for (long k = static_cast<long>(t.lists.size()) - 1; k >= 0; --k) {
    v.s[k] = acc;
    acc *= t.lists[k].second;
  }
  v.ld = t.base == Base::Block ? t.cols : 1;
  v.p = "B[" + std::to_string(slot) + "]";
  return v;
}

// Host copy of a top-level value, assembled like the reference's assemble (interpreter.hpp:101-138).
Matrix assemble_host(const std::vector<double>& h, const View& v) {
  const Ty& t = v.ty;
  const long r = t.rows, c = t.cols;
  if (t.lists.size() > 2) throw Error("assemble: nested value where a block was expected");
  const long n0 = t.lists.size() > 0 ? t.lists[0].second : 1;
  const long n1 = t.lists.size() > 1 ? t.lists[1].second : 1;
  if (t.lists.size() >= 1 && n0 == 0) throw Error("assemble: empty list");
  Matrix m(n0 * r, n1 * c);
  for (long i = 0; i < n0; ++i)
    for (long j = 0; j < n1; ++j) {
      const long off = (t.lists.size() > 0 ? i * v.s[0] : 0) + (t.lists.size() > 1 ? j * v.s[1] : 0);
      for (long a = 0; a < r; ++a)
        for (long b = 0; b < c; ++b) m(i * r + a, j * c + b) = h[static_cast<size_t>(off + a * v.ld + b)];
    }
  return m;
}

blockfuse::Value to_host_value(const std::vector<double>& h, const Ty& t, long off, const std::vector<long>& s,
                               long ld, size_t depth) {
  if (depth < t.lists.size()) {
    blockfuse::ValueList l;
    for (long i = 0; i < t.lists[depth].second; ++i)
      l.push_back(to_host_value(h, t, off + i * s[depth], s, ld, depth + 1));
    return blockfuse::Value(std::move(l));
  }
  if (t.base == Base::Scalar) return blockfuse::Value(h[static_cast<size_t>(off)]);
  if (t.base == Base::Vector) {
    blockfuse::Vector v(t.rows);
    for (long i = 0; i < t.rows; ++i) v[i] = h[static_cast<size_t>(off + i)];
    return blockfuse::Value(std::move(v));
  }
  Matrix m(t.rows, t.cols);
  for (long a = 0; a < t.rows; ++a)
    for (long b = 0; b < t.cols; ++b) m(a, b) = h[static_cast<size_t>(off + a * ld + b)];
  return blockfuse::Value(std::move(m));
}

// Type of a host Value (misc operator outputs) and its dense serialization.
Ty host_type(const blockfuse::Value& v, const std::string& dim_hint) {
  if (v.is_list()) {
    if (v.list().empty()) throw Error("misc operator returned an empty list");
    Ty t = host_type(v.list()[0], dim_hint);
    t.lists.insert(t.lists.begin(), {dim_hint, static_cast<long>(v.list().size())});
    return t;
  }
  Ty t;
  if (std::holds_alternative<double>(v.v)) {
    t.base = Base::Scalar;
  } else if (std::holds_alternative<blockfuse::Vector>(v.v)) {
    t.base = Base::Vector;
    t.rows = v.vec().size();
  } else {
    t.rows = v.block().rows();
    t.cols = v.block().cols();
  }
  return t;
}

void flatten(const blockfuse::Value& v, std::vector<double>& out) {
  if (v.is_list()) {
    for (const auto& e : v.list()) flatten(e, out);
  } else if (std::holds_alternative<double>(v.v)) {
    out.push_back(v.scalar());
  } else if (std::holds_alternative<blockfuse::Vector>(v.v)) {
    for (long i = 0; i < v.vec().size(); ++i) out.push_back(v.vec()[i]);
  } else {
    const Matrix& m = v.block();
    for (long a = 0; a < m.rows(); ++a)
      for (long b = 0; b < m.cols(); ++b) out.push_back(m(a, b));
  }
}

bool safe_mode() {
  const char* v = std::getenv("BFGPU_SAFE");
  return !(v && v[0] == '0');
}

std::string module_source(const std::vector<Kernel>& ks) {
  std::ostringstream src;
  src << kPrelude;
  for (const Kernel& k : ks)
    src << "extern \"C\" __global__ void __launch_bounds__(256) " << k.name
        << "(double* const* B, double* scratch, long per_cta) {\n"
        << "  double* S = scratch + ((long)blockIdx.y * gridDim.x + blockIdx.x) * per_cta;\n"
        << "  (void)S;\n"
        << k.body << "}\n";
  return src.str();
}

// Compiles and (unless `dry` is given) runs the program. A dry run touches no device: it
// returns the generated source of the segment before the first misc operator in *dry.
std::map<std::string, Matrix> run_compiled(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                           const DimBinding& binding, const blockfuse::ExecOptions& opts,
                                           void* stream, std::string* dry) {
  Compiler cc(binding, safe_mode());
  std::vector<std::unique_ptr<Buf>> keep;
  auto device_alloc = [&](std::vector<std::unique_ptr<Buf>>& k, size_t n) -> double* {
    if (dry) return reinterpret_cast<double*>(static_cast<uintptr_t>(0x1000u * (k.size() + 1)));
    return bfgpu::device_alloc(k, n);
  };
  std::vector<double*> slots;  // bufs[] of the generated kernels
  std::map<std::pair<NodeId, int>, View> vals;
  std::map<std::string, Matrix> outputs;
  auto input_of = [&](NodeId id, int port) -> const View& {
    const Edge* e = program.producer(id, port);
    if (!e) throw Error("node " + std::to_string(id) + ": missing producer");
    auto it = vals.find({e->src.node, e->src.port});
    if (it == vals.end()) throw Error("value not yet computed");
    return it->second;
  };
  auto add_slot = [&](double* p) {
    slots.push_back(p);
    return static_cast<int>(slots.size()) - 1;
  };
  // pending kernels of the current segment (top-level nodes up to the next misc / output)
  std::vector<Kernel> pending;
  int kid = 0;
  double* dslots = nullptr;
  auto flush = [&] {
    if (pending.empty()) return;
    if (dry) {
      *dry += module_source(pending);
      pending.clear();
      return;
    }
    void* mod = nullptr;
    check(bf_jit_compile(module_source(pending).c_str(), &mod, nullptr, 0), "NVRTC compile");
    // kernel arguments: the slot table and one scratch arena sized for the largest kernel
    std::vector<double*> table = slots;
    dslots = device_alloc(keep, table.size());
    check(bf_copy_to_device(dslots, table.data(), table.size() * sizeof(double*), stream), "upload buffer table");
    long scratch_doubles = 1;
    for (const Kernel& k : pending)
      scratch_doubles = std::max(scratch_doubles, k.scratch * static_cast<long>(k.gx) * static_cast<long>(k.gy));
    double* scratch = device_alloc(keep, static_cast<size_t>(scratch_doubles));
    for (const Kernel& k : pending) {
      long per = std::max(1L, k.scratch);
      void* args[] = {&dslots, &scratch, &per};
      check(bf_jit_launch(mod, k.name.c_str(), k.gx, k.gy, 256, 0, stream, args), k.name.c_str());
    }
    check(bf_stream_synchronize(stream), "stream synchronize");  // table/scratch lifetimes end here
    pending.clear();
  };
  auto download = [&](const View& v) {
    const long n = v.ty.count() * v.ty.elem();
    std::vector<double> h(static_cast<size_t>(std::max(n, 1L)));
    flush();
    if (dry) return h;
    const long slot = std::stol(v.p.substr(2, v.p.size() - 3));
    check(bf_copy_to_host(h.data(), slots.at(static_cast<size_t>(slot)), static_cast<size_t>(n) * sizeof(double),
                          stream),
          "copy to host");
    check(bf_stream_synchronize(stream), "stream synchronize");
    return h;
  };

  for (NodeId id : blockfuse::topological_order(program)) {
    const Node& n = program.node(id);
    switch (n.kind) {
      case NodeKind::Input: {  // interpreter.hpp:386-420
        auto it = inputs.find(n.name);
        if (it == inputs.end()) throw Error("missing input matrix " + n.name);
        const Matrix& m = it->second;
        if (n.desc.base != Base::Block) throw Error("input " + n.name + ": only matrix inputs supported");
        std::vector<std::string> split_dims;
        if (!n.rows_dim.empty()) split_dims.push_back(n.rows_dim);
        if (!n.cols_dim.empty()) split_dims.push_back(n.cols_dim);
        if (n.desc.list_dims != split_dims)
          throw Error("input " + n.name + ": descriptor does not match the declared block grid");
        const long rb = n.rows_dim.empty() ? 1 : binding.count(n.rows_dim);
        const long cb = n.cols_dim.empty() ? 1 : binding.count(n.cols_dim);
        if (!n.rows_dim.empty() && m.rows() != binding.total(n.rows_dim))
          throw Error("input " + n.name + ": row count does not match binding");
        if (!n.cols_dim.empty() && m.cols() != binding.total(n.cols_dim))
          throw Error("input " + n.name + ": column count does not match binding");
        if (m.rows() % rb || m.cols() % cb) throw Error("matrix shape not divisible by block grid");
        // row-major copy of the column-major matrix; the grid is a strided view of it
        const long R = m.rows(), C = m.cols();
        std::vector<double> h(static_cast<size_t>(R * C));
        for (long j = 0; j < C; ++j)
          for (long i = 0; i < R; ++i) h[static_cast<size_t>(i * C + j)] = m.data()[j * R + i];
        double* d = device_alloc(keep, h.size());
        if (!dry) {
          check(bf_copy_to_device(d, h.data(), h.size() * sizeof(double), stream), "copy to device");
          check(bf_stream_synchronize(stream), "stream synchronize");
        }
        View v;
        v.ty.rows = R / rb;
        v.ty.cols = C / cb;
        v.ld = C;
        v.p = "B[" + std::to_string(add_slot(d)) + "]";
        if (!n.rows_dim.empty()) {
          v.ty.lists.push_back({n.rows_dim, rb});
          v.s.push_back(v.ty.rows * C);
        }
        if (!n.cols_dim.empty()) {
          v.ty.lists.push_back({n.cols_dim, cb});
          v.s.push_back(v.ty.cols);
        }
        vals[{id, 0}] = v;
        break;
      }
      case NodeKind::Output: {
        const View& v = input_of(id, 0);
        outputs[n.name] = assemble_host(download(v), v);
        break;
      }
      case NodeKind::Map:
      case NodeKind::Func:
      case NodeKind::Reduce: {
        std::vector<View> in;
        const int nin = n.kind == NodeKind::Map ? blockfuse::map_in_count(n)
                                                : (n.kind == NodeKind::Reduce ? 1 : blockfuse::func_arity(n.op.kind));
        for (int p = 0; p < nin; ++p) in.push_back(input_of(id, p));
        std::vector<Ty> tys = cc.top_types(n, in);
        std::vector<View> gouts;
        for (const Ty& t : tys) {
          Ty g = t;
          g.se = false;
          long cnt = g.count() * g.elem();
          gouts.push_back(global_view(g, add_slot(device_alloc(keep, static_cast<size_t>(cnt)))));
        }
        const std::string name = "bf_node" + std::to_string(id) + "_" + std::to_string(kid++);
        pending.push_back(n.kind == NodeKind::Map ? cc.top_map(n, in, gouts, name)
                                                  : cc.top_func(n, in, gouts[0], name));
        for (size_t p = 0; p < gouts.size(); ++p) vals[{id, static_cast<int>(p)}] = gouts[p];
        break;
      }
      case NodeKind::Misc: {  // host callback between kernels (ExecOptions::misc, interpreter.hpp:457-465)
        if (dry) {
          flush();
          return outputs;
        }
        auto it = opts.misc.find(n.name);
        if (it == opts.misc.end()) throw Error("no executor registered for misc operator " + n.name);
        std::vector<blockfuse::Value> in;
        for (int p = 0; p < n.misc_inputs; ++p) {
          const View& v = input_of(id, p);
          in.push_back(to_host_value(download(v), v.ty, 0, v.s, v.ld, 0));
        }
        std::vector<blockfuse::Value> res = it->second(in);
        for (int p = 0; p < n.misc_outputs; ++p) {
          Ty t = host_type(res.at(static_cast<size_t>(p)), n.name);
          std::vector<double> h;
          flatten(res[static_cast<size_t>(p)], h);
          double* d = device_alloc(keep, h.size());
          check(bf_copy_to_device(d, h.data(), h.size() * sizeof(double), stream), "copy to device");
          check(bf_stream_synchronize(stream), "stream synchronize");
          vals[{id, p}] = global_view(t, add_slot(d));
        }
        break;
      }
      case NodeKind::BoundaryIn:
      case NodeKind::BoundaryOut: throw Error("boundary node in root graph");
    }
  }
  flush();
  return outputs;
}

}  // namespace

std::map<std::string, Matrix> execute_generic(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                              const DimBinding& binding, const blockfuse::ExecOptions& opts,
                                              void* stream) {
  return run_compiled(program, inputs, binding, opts, stream, nullptr);
}

std::string generic_source(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                           const DimBinding& binding) {
  std::string src;
  run_compiled(program, inputs, binding, blockfuse::ExecOptions{}, nullptr, &src);
  return src;
}

}  // namespace bfgpu
