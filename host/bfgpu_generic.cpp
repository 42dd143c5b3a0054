// bfgpu::execute_generic — any block program on the GPU, in float64.
//
// The same walk as the reference's detail::eval_graph / eval_map
// (interpreter.hpp:301-472) — topological order, boundary ports, Iterate vs
// Broadcast map inputs, Collect vs Accumulate map outputs, the empty-range
// probe, left-to-right reductions, Misc executors — but every value lives in
// device memory and every operator runs as a kernel of the generic C-ABI
// (bf_gx_*, include/bfgpu.h; csrc/generic.cu). The host only walks the graph
// and moves pointers; no arithmetic happens here.
//
// Values are dense row-major float64 device buffers: a Block is rows x cols, a
// Vector is rows, a Scalar is one element, and lists hold values (the block
// grid of interpreter.hpp:76-138). Buffers come from a per-call arena with a
// size-keyed free list: all work is on one stream, so a buffer released after
// its last reader was enqueued can be reused by anything enqueued later.
#include <cstring>
#include <functional>
#include <memory>
#include <vector>

#include "bfgpu.h"
#include "bfgpu_execute.hpp"

namespace bfgpu {

using blockfuse::BlockGraph;
using blockfuse::DimBinding;
using blockfuse::Error;
using blockfuse::Matrix;
using blockfuse::Node;
using blockfuse::NodeId;
using blockfuse::NodeKind;
using blockfuse::ScalarExpr;

namespace {

void check(int rc, const char* what) {
  if (rc != BF_OK) throw Error(std::string("generic execution, ") + what + ": " + bf_last_error());
}

class Arena {
 public:
  explicit Arena(void* stream) : stream_(stream) {}
  ~Arena() {
    bf_stream_synchronize(stream_);
    for (auto& [n, v] : free_)
      for (double* p : v) bf_device_free(p);
  }
  std::shared_ptr<double> get(size_t n) {
    n = n == 0 ? 1 : n;
    double* p = nullptr;
    auto& fl = free_[n];
    if (!fl.empty()) {
      p = fl.back();
      fl.pop_back();
    } else {
      p = static_cast<double*>(bf_device_alloc(n * sizeof(double)));
      if (!p) throw Error(std::string("generic execution: device allocation failed: ") + bf_last_error());
    }
    return std::shared_ptr<double>(p, [this, n](double* q) { free_[n].push_back(q); });
  }
  void* stream() const { return stream_; }

 private:
  void* stream_;
  std::map<size_t, std::vector<double*>> free_;
};

struct DVal {
  enum Kind { Scalar, Vec, Block, List } kind = Scalar;
  std::shared_ptr<double> buf;
  long rows = 1, cols = 1;
  std::vector<DVal> list;

  long elems() const { return kind == Block ? rows * cols : (kind == Vec ? rows : 1); }
  bool is_list() const { return kind == List; }
};

DVal make_leaf(Arena& A, DVal::Kind k, long rows, long cols) {
  DVal v;
  v.kind = k;
  v.rows = rows;
  v.cols = k == DVal::Block ? cols : 1;
  v.buf = A.get(static_cast<size_t>(v.elems()));
  return v;
}

void want_same_shape(const DVal& a, const DVal& b, const char* op) {
  if (a.kind != b.kind || a.is_list()) throw Error(std::string(op) + ": operand kinds differ");
  if (a.rows != b.rows || a.cols != b.cols) throw Error(std::string(op) + ": block shapes differ");
}

DVal add_values(Arena& A, const DVal& a, const DVal& b) {  // interpreter.hpp:231-236
  if (a.is_list()) throw Error("reduction over nested lists is not defined");
  want_same_shape(a, b, "add");
  DVal out = make_leaf(A, a.kind, a.rows, a.cols);
  check(bf_gx_binary(BF_GX_ADD, a.buf.get(), b.buf.get(), out.buf.get(), a.elems(), A.stream()), "add");
  return out;
}

DVal zero_like(Arena& A, const DVal& v) {  // interpreter.hpp:310-316
  if (v.is_list()) throw Error("zero of a list value is not defined");
  DVal out = make_leaf(A, v.kind, v.rows, v.cols);
  check(bf_gx_zero(out.buf.get(), out.elems(), A.stream()), "zero");
  return out;
}

// ScalarExpr -> postfix program for bf_gx_elementwise (scalar_expr.hpp:66-87).
void compile_expr(const ScalarExpr& e, const DimBinding& b, std::vector<int8_t>& ops, std::vector<double>& cst) {
  using Op = ScalarExpr::Op;
  auto emit = [&](int op, double c = 0.0) {
    ops.push_back(static_cast<int8_t>(op));
    cst.push_back(c);
  };
  switch (e.op()) {
    case Op::Var: emit(BF_GX_EXPR_VAR); return;
    case Op::Const: emit(BF_GX_EXPR_CONST, e.value()); return;
    case Op::DimTotal: emit(BF_GX_EXPR_CONST, static_cast<double>(b.total(e.dim()))); return;
    case Op::Add:
    case Op::Sub:
    case Op::Mul:
    case Op::Div:
      compile_expr(e.lhs(), b, ops, cst);
      compile_expr(e.rhs(), b, ops, cst);
      emit(e.op() == Op::Add ? BF_GX_EXPR_ADD
                             : e.op() == Op::Sub ? BF_GX_EXPR_SUB : e.op() == Op::Mul ? BF_GX_EXPR_MUL : BF_GX_EXPR_DIV);
      return;
    case Op::Exp:
    case Op::Sqrt:
    case Op::Recip:
    case Op::Square:
    case Op::Sigmoid:
      compile_expr(e.lhs(), b, ops, cst);
      emit(e.op() == Op::Exp      ? BF_GX_EXPR_EXP
           : e.op() == Op::Sqrt   ? BF_GX_EXPR_SQRT
           : e.op() == Op::Recip  ? BF_GX_EXPR_RECIP
           : e.op() == Op::Square ? BF_GX_EXPR_SQUARE
                                  : BF_GX_EXPR_SIGMOID);
      return;
  }
  throw Error("scalar expr: bad op");
}

struct Ctx {
  Arena& A;
  const DimBinding& binding;
  const blockfuse::ExecOptions& opts;
};

DVal eval_func(const Node& n, const std::vector<DVal>& in, Ctx& c) {  // interpreter.hpp:263-299
  using blockfuse::FuncKind;
  Arena& A = c.A;
  for (const DVal& v : in)
    if (v.is_list()) throw Error(std::string("operator ") + blockfuse::func_name(n.op.kind) + ": local value expected");
  switch (n.op.kind) {
    case FuncKind::Add:
      return add_values(A, in[0], in[1]);
    case FuncKind::Mul: {
      want_same_shape(in[0], in[1], "mul");
      DVal out = make_leaf(A, in[0].kind, in[0].rows, in[0].cols);
      check(bf_gx_binary(BF_GX_MUL, in[0].buf.get(), in[1].buf.get(), out.buf.get(), in[0].elems(), A.stream()), "mul");
      return out;
    }
    case FuncKind::RowShift:
    case FuncKind::RowScale: {
      const bool shift = n.op.kind == FuncKind::RowShift;
      if (in[0].kind != DVal::Block || in[1].kind != DVal::Vec) throw Error(shift ? "row_shift: block and vector expected"
                                                                                   : "row_scale: block and vector expected");
      if (in[1].rows != in[0].rows)
        throw Error(shift ? "row_shift: vector length must equal block row count"
                          : "row_scale: vector length must equal block row count");
      DVal out = make_leaf(A, DVal::Block, in[0].rows, in[0].cols);
      check(bf_gx_row_op(shift ? BF_GX_ROW_SHIFT : BF_GX_ROW_SCALE, in[0].buf.get(), in[1].buf.get(), out.buf.get(),
                         in[0].rows, in[0].cols, A.stream()),
            "row op");
      return out;
    }
    case FuncKind::RowSum: {
      if (in[0].kind != DVal::Block) throw Error("row_sum: block expected");
      DVal out = make_leaf(A, DVal::Vec, in[0].rows, 1);
      check(bf_gx_row_sum(in[0].buf.get(), out.buf.get(), in[0].rows, in[0].cols, A.stream()), "row_sum");
      return out;
    }
    case FuncKind::Dot: {
      if (in[0].kind != DVal::Block || in[1].kind != DVal::Block) throw Error("dot: blocks expected");
      if (in[0].cols != in[1].cols) throw Error("dot: column counts must match");
      DVal out = make_leaf(A, DVal::Block, in[0].rows, in[1].rows);
      check(bf_gx_dot(in[0].buf.get(), in[1].buf.get(), out.buf.get(), in[0].rows, in[1].rows, in[0].cols, A.stream()),
            "dot");
      return out;
    }
    case FuncKind::Outer: {
      if (in[0].kind != DVal::Vec || in[1].kind != DVal::Vec) throw Error("outer: vectors expected");
      DVal out = make_leaf(A, DVal::Block, in[0].rows, in[1].rows);
      check(bf_gx_outer(in[0].buf.get(), in[1].buf.get(), out.buf.get(), in[0].rows, in[1].rows, A.stream()), "outer");
      return out;
    }
    case FuncKind::Elementwise: {
      std::vector<int8_t> ops;
      std::vector<double> cst;
      compile_expr(n.op.expr, c.binding, ops, cst);
      DVal out = make_leaf(A, in[0].kind, in[0].rows, in[0].cols);
      check(bf_gx_elementwise(ops.data(), cst.data(), static_cast<int>(ops.size()), in[0].buf.get(), out.buf.get(),
                              in[0].elems(), A.stream()),
            "elementwise");
      return out;
    }
  }
  throw Error("bad func kind");
}

// ---------------------------------------------------------------- host <-> device

DVal upload_matrix(Arena& A, const Matrix& m) {
  const long R = m.rows(), C = m.cols();
  std::vector<double> host(static_cast<size_t>(R * C));
  for (long i = 0; i < R; ++i)
    for (long j = 0; j < C; ++j) host[static_cast<size_t>(i * C + j)] = m(i, j);  // Eigen is column-major
  DVal v = make_leaf(A, DVal::Block, R, C);
  check(bf_copy_to_device(v.buf.get(), host.data(), host.size() * sizeof(double), A.stream()), "copy to device");
  check(bf_stream_synchronize(A.stream()), "stream synchronize");  // `host` is pageable and goes out of scope
  return v;
}

// split_into_blocks (interpreter.hpp:76-89), on the device
DVal split_into_blocks(Arena& A, const DVal& full, int rb, int cb) {
  if (full.rows % rb != 0 || full.cols % cb != 0) throw Error("matrix shape not divisible by block grid");
  const long br = full.rows / rb, bc = full.cols / cb;
  DVal grid;
  grid.kind = DVal::List;
  for (int i = 0; i < rb; ++i) {
    DVal row;
    row.kind = DVal::List;
    for (int j = 0; j < cb; ++j) {
      DVal blk = make_leaf(A, DVal::Block, br, bc);
      check(bf_gx_copy2d(blk.buf.get(), bc, full.buf.get() + i * br * full.cols + j * bc, full.cols, br, bc,
                         A.stream()),
            "split");
      row.list.push_back(std::move(blk));
    }
    grid.list.push_back(std::move(row));
  }
  return grid;
}

// assemble (interpreter.hpp:100-138): a leaf, a list of leaves stacked vertically, or a grid.
Matrix assemble(Arena& A, const DVal& v) {
  std::vector<std::vector<const DVal*>> rows;
  auto leaf_shape = [](const DVal& x, long& r, long& c) {
    if (x.is_list()) throw Error("assemble: nested value where a block was expected");
    r = x.rows;
    c = x.kind == DVal::Block ? x.cols : 1;
  };
  if (!v.is_list()) {
    rows.push_back({&v});
  } else {
    if (v.list.empty()) throw Error("assemble: empty list");
    for (const DVal& r : v.list) {
      if (!r.is_list()) {
        rows.push_back({&r});
        continue;
      }
      if (r.list.empty()) throw Error("assemble: empty row");
      std::vector<const DVal*> row;
      for (const DVal& cell : r.list) row.push_back(&cell);
      rows.push_back(std::move(row));
    }
  }
  long H = 0, W = -1;
  std::vector<long> row_h;
  for (const auto& row : rows) {
    long h = -1, w = 0;
    for (const DVal* cell : row) {
      long r, c;
      leaf_shape(*cell, r, c);
      if (h >= 0 && r != h) throw Error("assemble: ragged blocks");
      h = r;
      w += c;
    }
    if (W >= 0 && w != W) throw Error("assemble: ragged rows");
    W = w;
    row_h.push_back(h);
    H += h;
  }
  DVal full = make_leaf(A, DVal::Block, H, W);
  long r0 = 0;
  for (size_t i = 0; i < rows.size(); ++i) {
    long c0 = 0;
    for (const DVal* cell : rows[i]) {
      long r, c;
      leaf_shape(*cell, r, c);
      check(bf_gx_copy2d(full.buf.get() + r0 * W + c0, W, cell->buf.get(), c, r, c, A.stream()), "assemble");
      c0 += c;
    }
    r0 += row_h[i];
  }
  std::vector<double> host(static_cast<size_t>(H * W));
  check(bf_copy_to_host(host.data(), full.buf.get(), host.size() * sizeof(double), A.stream()), "copy to host");
  check(bf_stream_synchronize(A.stream()), "stream synchronize");
  Matrix m(H, W);
  for (long i = 0; i < H; ++i)
    for (long j = 0; j < W; ++j) m(i, j) = host[static_cast<size_t>(i * W + j)];
  return m;
}

// Misc operators run the caller's executor (interpreter.hpp:457-465) on host values.
blockfuse::Value to_host(Arena& A, const DVal& v) {
  if (v.is_list()) {
    blockfuse::ValueList l;
    for (const DVal& x : v.list) l.push_back(to_host(A, x));
    return blockfuse::Value(std::move(l));
  }
  std::vector<double> host(static_cast<size_t>(v.elems()));
  check(bf_copy_to_host(host.data(), v.buf.get(), host.size() * sizeof(double), A.stream()), "copy to host");
  check(bf_stream_synchronize(A.stream()), "stream synchronize");
  if (v.kind == DVal::Scalar) return blockfuse::Value(host[0]);
  if (v.kind == DVal::Vec) {
    blockfuse::Vector x(v.rows);
    for (long i = 0; i < v.rows; ++i) x[i] = host[static_cast<size_t>(i)];
    return blockfuse::Value(std::move(x));
  }
  Matrix m(v.rows, v.cols);
  for (long i = 0; i < v.rows; ++i)
    for (long j = 0; j < v.cols; ++j) m(i, j) = host[static_cast<size_t>(i * v.cols + j)];
  return blockfuse::Value(std::move(m));
}

DVal to_device(Arena& A, const blockfuse::Value& v) {
  if (v.is_list()) {
    DVal out;
    out.kind = DVal::List;
    for (const blockfuse::Value& x : v.list()) out.list.push_back(to_device(A, x));
    return out;
  }
  std::vector<double> host;
  DVal out;
  if (std::holds_alternative<double>(v.v)) {
    out = make_leaf(A, DVal::Scalar, 1, 1);
    host = {v.scalar()};
  } else if (std::holds_alternative<blockfuse::Vector>(v.v)) {
    out = make_leaf(A, DVal::Vec, v.vec().size(), 1);
    for (long i = 0; i < out.rows; ++i) host.push_back(v.vec()[i]);
  } else {
    const Matrix& m = v.block();
    out = make_leaf(A, DVal::Block, m.rows(), m.cols());
    for (long i = 0; i < out.rows; ++i)
      for (long j = 0; j < out.cols; ++j) host.push_back(m(i, j));
  }
  check(bf_copy_to_device(out.buf.get(), host.data(), host.size() * sizeof(double), A.stream()), "copy to device");
  check(bf_stream_synchronize(A.stream()), "stream synchronize");
  return out;
}

// ---------------------------------------------------------------- graph walk

struct RootIo {
  const std::map<std::string, Matrix>* inputs = nullptr;
  std::map<std::string, Matrix>* outputs = nullptr;
};

std::vector<DVal> eval_graph(const BlockGraph& g, const std::vector<DVal>& boundary, Ctx& c, RootIo io = {});

std::vector<DVal> eval_map(const Node& n, const std::vector<DVal>& in, Ctx& c) {  // interpreter.hpp:319-371
  using blockfuse::MapRange;
  using blockfuse::OutKind;
  using blockfuse::PortMode;
  const BlockGraph& inner = *n.inner;
  const int count = c.binding.count(n.dim);
  const int begin = n.range == MapRange::Rest ? 1 : 0;
  const int end = n.range == MapRange::First ? 1 : count;
  const int nin = blockfuse::map_in_count(n), nout = blockfuse::map_out_count(n);
  for (int p = 0; p < nin; ++p)
    if (n.in_modes[p] == PortMode::Iterate && static_cast<int>(in[p].list.size()) != count)
      throw Error("map over " + n.dim + ": iterated list length " + std::to_string(in[p].list.size()) +
                  " does not match block count " + std::to_string(count));
  std::vector<DVal> collected(nout), finals(nout);
  for (auto& x : collected) x.kind = DVal::List;
  bool ran = false;
  auto body = [&](int i) {
    std::vector<DVal> bvals;
    for (int p = 0; p < nin; ++p) bvals.push_back(n.in_modes[p] == PortMode::Iterate ? in[p].list[i] : in[p]);
    return eval_graph(inner, bvals, c);
  };
  for (int i = begin; i < end; ++i) {
    std::vector<DVal> outs = body(i);
    for (int p = 0; p < nout; ++p) {
      if (blockfuse::map_out_kind(n, p) == OutKind::Collect)
        collected[p].list.push_back(outs[p]);
      else
        finals[p] = ran ? add_values(c.A, finals[p], outs[p]) : outs[p];
    }
    ran = true;
  }
  if (!ran && count >= 1) {  // empty range: accumulators are the zero of the probed shape
    std::vector<DVal> outs = body(0);
    for (int p = 0; p < nout; ++p)
      if (blockfuse::map_out_kind(n, p) == OutKind::Accumulate) finals[p] = zero_like(c.A, outs[p]);
    ran = true;
  }
  std::vector<DVal> result(nout);
  for (int p = 0; p < nout; ++p) {
    if (blockfuse::map_out_kind(n, p) == OutKind::Collect)
      result[p] = std::move(collected[p]);
    else if (ran)
      result[p] = finals[p];
    else
      throw Error("map over " + n.dim + ": empty iteration range leaves accumulator undefined");
  }
  return result;
}

std::vector<DVal> eval_graph(const BlockGraph& g, const std::vector<DVal>& boundary, Ctx& c, RootIo io) {
  std::map<std::pair<NodeId, int>, DVal> vals;
  auto input_of = [&](NodeId id, int port) -> const DVal& {
    const blockfuse::Edge* e = g.producer(id, port);
    if (!e) throw Error("node " + std::to_string(id) + ": missing producer");
    auto it = vals.find({e->src.node, e->src.port});
    if (it == vals.end()) throw Error("value not yet computed");
    return it->second;
  };
  for (NodeId id : blockfuse::topological_order(g)) {
    const Node& n = g.node(id);
    switch (n.kind) {
      case NodeKind::Input: {  // interpreter.hpp:386-420
        if (!io.inputs) throw Error("input node in inner graph");
        auto it = io.inputs->find(n.name);
        if (it == io.inputs->end()) throw Error("missing input matrix " + n.name);
        const Matrix& m = it->second;
        if (n.desc.base != blockfuse::Base::Block) throw Error("input " + n.name + ": only matrix inputs supported");
        std::vector<std::string> split_dims;
        if (!n.rows_dim.empty()) split_dims.push_back(n.rows_dim);
        if (!n.cols_dim.empty()) split_dims.push_back(n.cols_dim);
        if (n.desc.list_dims != split_dims)
          throw Error("input " + n.name + ": descriptor does not match the declared block grid");
        const int rb = n.rows_dim.empty() ? 1 : c.binding.count(n.rows_dim);
        const int cb = n.cols_dim.empty() ? 1 : c.binding.count(n.cols_dim);
        if (!n.rows_dim.empty() && m.rows() != c.binding.total(n.rows_dim))
          throw Error("input " + n.name + ": row count does not match binding");
        if (!n.cols_dim.empty() && m.cols() != c.binding.total(n.cols_dim))
          throw Error("input " + n.name + ": column count does not match binding");
        DVal grid = split_into_blocks(c.A, upload_matrix(c.A, m), rb, cb);
        DVal out;
        if (n.desc.list_dims.size() == 2) {
          out = std::move(grid);
        } else if (n.desc.list_dims.size() == 1) {
          out.kind = DVal::List;
          for (DVal& row : grid.list)
            for (DVal& b : row.list) out.list.push_back(std::move(b));
        } else {
          out = grid.list[0].list[0];
        }
        vals[{id, 0}] = std::move(out);
        break;
      }
      case NodeKind::Output:
        if (!io.outputs) throw Error("output node in inner graph");
        (*io.outputs)[n.name] = assemble(c.A, input_of(id, 0));
        break;
      case NodeKind::BoundaryIn:
        vals[{id, 0}] =
            boundary.at(std::find(g.boundary_in.begin(), g.boundary_in.end(), id) - g.boundary_in.begin());
        break;
      case NodeKind::BoundaryOut:
        break;
      case NodeKind::Func: {
        std::vector<DVal> in;
        for (int p = 0; p < blockfuse::func_arity(n.op.kind); ++p) in.push_back(input_of(id, p));
        vals[{id, 0}] = eval_func(n, in, c);
        break;
      }
      case NodeKind::Reduce: {  // interpreter.hpp:435-447
        const DVal& in = input_of(id, 0);
        if (!in.is_list()) {
          vals[{id, 0}] = in;
          break;
        }
        if (in.list.empty()) throw Error("reduction over empty list");
        DVal acc = in.list[0];
        for (size_t i = 1; i < in.list.size(); ++i) acc = add_values(c.A, acc, in.list[i]);
        vals[{id, 0}] = std::move(acc);
        break;
      }
      case NodeKind::Map: {
        std::vector<DVal> in;
        for (int p = 0; p < blockfuse::map_in_count(n); ++p) in.push_back(input_of(id, p));
        std::vector<DVal> outs = eval_map(n, in, c);
        for (int p = 0; p < blockfuse::map_out_count(n); ++p) vals[{id, p}] = std::move(outs[p]);
        break;
      }
      case NodeKind::Misc: {
        auto it = c.opts.misc.find(n.name);
        if (it == c.opts.misc.end()) throw Error("no executor registered for misc operator " + n.name);
        std::vector<blockfuse::Value> in;
        for (int p = 0; p < n.misc_inputs; ++p) in.push_back(to_host(c.A, input_of(id, p)));
        std::vector<blockfuse::Value> outs = it->second(in);
        for (int p = 0; p < n.misc_outputs; ++p) vals[{id, p}] = to_device(c.A, outs.at(p));
        break;
      }
    }
  }
  std::vector<DVal> out;
  for (NodeId bo : g.boundary_out) out.push_back(input_of(bo, 0));
  return out;
}

}  // namespace

std::map<std::string, Matrix> execute_generic(const BlockGraph& program, const std::map<std::string, Matrix>& inputs,
                                              const DimBinding& binding, const blockfuse::ExecOptions& opts,
                                              void* stream) {
  Arena arena(stream);
  Ctx c{arena, binding, opts};
  std::map<std::string, Matrix> outputs;
  RootIo io{&inputs, &outputs};
  eval_graph(program, {}, c, io);
  check(bf_stream_synchronize(stream), "stream synchronize");
  return outputs;
}

}  // namespace bfgpu
