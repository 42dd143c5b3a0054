// bfgpu-cli — program-file front door of the B200 backend.
//
// Takes the reference's "blockfuse-program" v1 JSON files (bf/serialize.hpp:305-366),
// i.e. the output of the reference workflow
//     blockfuse examples X | blockfuse lower | blockfuse fuse --out-dir D
// (tools/blockfuse_main.cpp:139-181), and runs them on the GPU through the drop-in
// bfgpu::execute (host/bfgpu_execute.hpp). Subcommands and exit codes follow the
// reference CLI (tools/blockfuse_main.cpp:180-237): 0 success, 1 error, 2 inequivalent.
//
//   bfgpu-cli snapshots  <attention|layernorm-matmul|rms-swiglu> --out-dir D
//   bfgpu-cli recognize  <program.json>
//   bfgpu-cli run        <program.json> --dims M=2,N=2 [--block 4x4] [--len D=128,...]
//                        [--seed 42] [--precision bf16|f32] [--repeat R]
//   bfgpu-cli verify     <program.json> --dims ... [--block] [--len] [--trials 3]
//                        [--seed 42] [--tol T] [--precision bf16|f32]
// run/verify take --route auto|fused|generic: auto runs recognized snapshots on their
// sm_100a plans and anything else (e.g. an unfused lowered.json) through the block-program
// compiler, float64 (host/bfgpu_codegen.cpp).
//
// `snapshots` is the reference's own fuse(lower(examples::X())) (engine.hpp:164) written
// with its serializer; it exists because the reference CLI needs CLI11, absent here.
// `verify` compares the GPU result with the reference's CPU interpreter
// (blockfuse::execute, interpreter.hpp:478) on the reference's seeded inputs
// (random_inputs, interpreter.hpp:585); `run` never touches the CPU interpreter.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "bfgpu_execute.hpp"
#include "blockfuse/engine.hpp"
#include "blockfuse/lowering.hpp"
#include "blockfuse/serialize.hpp"

namespace fs = std::filesystem;
using namespace blockfuse;

namespace {

std::string read_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw Error("cannot open " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

void write_file(const std::string& path, const std::string& text) {
  std::ofstream f(path);
  if (!f) throw Error("cannot write " + path);
  f << text;
}

struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::string get(const std::string& k, const std::string& def) const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
  bool has(const std::string& k) const { return opt.count(k) != 0; }
};

Args parse_args(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    if (s == "--enable-peel") {  // the only flag without a value
      a.opt["enable-peel"] = "1";
    } else if (s.rfind("--", 0) == 0) {
      if (i + 1 >= argc) throw Error("option " + s + " needs a value");
      a.opt[s.substr(2)] = argv[++i];
    } else {
      a.pos.push_back(s);
    }
  }
  return a;
}

// Same syntax as the reference CLI: --dims "M=2,N=4", --block "4x4", --len "M=4,N=8".
DimBinding parse_binding(const Args& a) {
  DimBinding b;
  const std::string dims = a.get("dims", "");
  if (dims.empty()) throw Error("--dims is required (e.g. M=2,N=2)");
  std::istringstream is(dims);
  std::string item;
  while (std::getline(is, item, ',')) {
    auto eq = item.find('=');
    if (eq == std::string::npos) throw Error("bad --dims entry '" + item + "'");
    b.dims[item.substr(0, eq)].count = std::stoi(item.substr(eq + 1));
  }
  const std::string block = a.get("block", "4x4");
  auto x = block.find('x');
  if (x == std::string::npos) throw Error("bad --block value '" + block + "' (expected RxC)");
  const int r = std::stoi(block.substr(0, x)), c = std::stoi(block.substr(x + 1));
  if (r != c) throw Error("--block requires square blocks; use --len for per-dimension lengths");
  for (auto& [d, e] : b.dims) e.block_len = r;
  b.free_len = r;
  const std::string lens = a.get("len", "");
  std::istringstream ls(lens);
  while (!lens.empty() && std::getline(ls, item, ',')) {
    auto eq = item.find('=');
    if (eq == std::string::npos) throw Error("bad --len entry '" + item + "'");
    b.dims[item.substr(0, eq)].block_len = std::stoi(item.substr(eq + 1));
  }
  return b;
}

bfgpu::ExecConfig exec_config(const Args& a) {
  bfgpu::ExecConfig cfg;
  const std::string route = a.get("route", "auto");
  if (route == "auto")
    cfg.route = bfgpu::Route::Auto;
  else if (route == "fused")
    cfg.route = bfgpu::Route::Fused;
  else if (route == "generic")
    cfg.route = bfgpu::Route::Generic;
  else
    throw Error("--route must be auto, fused or generic");
  const std::string prec = a.get("precision", "bf16");
  if (prec == "bf16")
    cfg.precision = bfgpu::Precision::BF16;
  else if (prec == "f32")
    cfg.precision = bfgpu::Precision::F32;
  else
    throw Error("--precision must be bf16 or f32");
  return cfg;
}

const char* pattern_name(bfgpu::Pattern p) {
  switch (p) {
    case bfgpu::Pattern::RmsFfnSwiglu: return "rms_ffn_swiglu";
    case bfgpu::Pattern::LayerNormMatMul: return "layernorm_matmul";
    default: return "attention";
  }
}

BlockGraph load_block(const std::string& path) {
  ParsedProgram p = parse_program(read_file(path));
  for (const std::string& w : p.warnings) std::cerr << "bfgpu-cli: warning: " << w << "\n";
  return p.to_block();
}

int cmd_snapshots(const Args& a) {
  if (a.pos.size() != 1)
    throw Error("usage: snapshots <attention|layernorm-matmul|rms-swiglu> --out-dir D [--enable-peel]");
  const std::string name = a.pos[0];
  ArrayProgram p;
  if (name == "attention")
    p = examples::attention();
  else if (name == "layernorm-matmul")
    p = examples::layernorm_matmul();
  else if (name == "rms-swiglu")
    p = examples::rms_ffn_swiglu();
  else
    throw Error("unknown example '" + name + "'");
  const std::string dir = a.get("out-dir", "");
  if (dir.empty()) throw Error("--out-dir is required");
  fs::create_directories(dir);
  const BlockGraph lowered = lower(p);
  write_file(dir + "/lowered.json", serialize_program(lowered));
  // --enable-peel: the driver's peeling route (rule R7, off by default), as the reference CLI's
  // `fuse --enable-peel` (tools/blockfuse_main.cpp:122-126, engine.hpp:22)
  EngineConfig cfg;
  cfg.enable_peel = a.has("enable-peel");
  FuseResult r = fuse(lowered, cfg);
  for (size_t i = 0; i < r.snapshots.size(); ++i)
    write_file(dir + "/snapshot_" + std::to_string(i + 1) + ".json", serialize_program(r.snapshots[i].program));
  std::cout << "{\"example\": \"" << name << "\", \"snapshots\": " << r.snapshots.size() << "}\n";
  return 0;
}

int cmd_recognize(const Args& a) {
  if (a.pos.size() != 1) throw Error("usage: recognize <program.json>");
  const bfgpu::Recognized r = bfgpu::recognize(load_block(a.pos[0]));
  std::cout << "{\"pattern\": \"" << pattern_name(r.pattern) << "\", \"snapshot\": " << r.snapshot
            << ", \"materializes_intermediate\": " << (r.materializes_intermediate ? "true" : "false")
            << ", \"eps\": " << r.eps << ", \"output\": \"" << r.output << "\"}\n";
  return 0;
}

int cmd_run(const Args& a) {
  if (a.pos.size() != 1) throw Error("usage: run <program.json> --dims ...");
  const BlockGraph g = load_block(a.pos[0]);
  const DimBinding b = parse_binding(a);
  const bfgpu::ExecConfig cfg = exec_config(a);
  const unsigned long long seed = std::stoull(a.get("seed", "42"));
  const int repeat = std::max(1, std::stoi(a.get("repeat", "1")));
  const auto inputs = random_inputs(input_specs(g, b), seed);
  std::map<std::string, Matrix> out;
  double best_ms = 1e30, sum_ms = 0;
  bfgpu::ExecTiming best_tm;
  for (int r = 0; r < repeat; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    out = bfgpu::execute(g, inputs, b, cfg);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (r > 0 || repeat == 1) sum_ms += ms;
    if (ms < best_ms) {
      best_ms = ms;
      best_tm = bfgpu::last_timing();
    }
  }
  const double mean_ms = sum_ms / std::max(1, repeat > 1 ? repeat - 1 : 1);
  for (const auto& [name, m] : out) {
    double sum = 0, sumsq = 0;
    for (Eigen::Index i = 0; i < m.rows(); ++i)
      for (Eigen::Index j = 0; j < m.cols(); ++j) {
        sum += m(i, j);
        sumsq += m(i, j) * m(i, j);
      }
    std::printf("{\"output\": \"%s\", \"rows\": %ld, \"cols\": %ld, \"sum\": %.9g, \"rms\": %.9g, \"ms\": %.3f, "
                "\"ms_mean\": %.3f, \"repeat\": %d, \"stages_ms\": {\"convert_in\": %.3f, \"device\": %.3f, "
                "\"convert_out\": %.3f}, \"h2d_bytes\": %zu, \"d2h_bytes\": %zu}\n",
                name.c_str(), static_cast<long>(m.rows()), static_cast<long>(m.cols()), sum,
                std::sqrt(sumsq / std::max<double>(1.0, static_cast<double>(m.rows() * m.cols()))), best_ms, mean_ms,
                repeat, best_tm.convert_in_ms, best_tm.device_ms, best_tm.convert_out_ms, best_tm.h2d_bytes,
                best_tm.d2h_bytes);
  }
  return 0;
}

int cmd_verify(const Args& a) {
  if (a.pos.size() != 1) throw Error("usage: verify <program.json> --dims ...");
  const BlockGraph g = load_block(a.pos[0]);
  const DimBinding b = parse_binding(a);
  const bfgpu::ExecConfig cfg = exec_config(a);
  // which executor will run it: a fused kernel (bf16 or fp32) or the generic float64 route
  bool fused = cfg.route != bfgpu::Route::Generic;
  if (fused) {
    try {
      bfgpu::recognize(g);
    } catch (const Error&) {
      if (cfg.route == bfgpu::Route::Fused) throw;
      fused = false;
    }
  }
  const bool bf16 = fused && cfg.precision == bfgpu::Precision::BF16;
  const double tol = std::stod(a.get("tol", !fused ? "1e-10" : (bf16 ? "2e-2" : "1e-4")));
  const int trials = std::stoi(a.get("trials", "3"));
  const unsigned long long seed = std::stoull(a.get("seed", "42"));
  const auto specs = input_specs(g, b);
  double worst = 0;
  for (int t = 0; t < trials; ++t) {
    auto in = random_inputs(specs, seed + static_cast<unsigned long long>(t));
    if (bf16) {  // compare against float64 on the inputs the GPU actually sees
      for (auto& [name, m] : in)
        for (Eigen::Index i = 0; i < m.rows(); ++i)
          for (Eigen::Index j = 0; j < m.cols(); ++j) {
            const float f = static_cast<float>(m(i, j));
            uint32_t u;
            std::memcpy(&u, &f, 4);
            u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;  // round to nearest even
            float r;
            std::memcpy(&r, &u, 4);
            m(i, j) = r;
          }
    }
    const auto ref = execute(g, in, b);  // the reference's CPU interpreter (float64)
    const auto got = bfgpu::execute(g, in, b, cfg);
    for (const auto& [name, m] : ref) {
      auto it = got.find(name);
      if (it == got.end()) throw Error("backend did not produce output " + name);
      double dmax = 0, rmax = 0;
      for (Eigen::Index i = 0; i < m.rows(); ++i)
        for (Eigen::Index j = 0; j < m.cols(); ++j) {
          dmax = std::max(dmax, std::abs(m(i, j) - it->second(i, j)));
          rmax = std::max(rmax, std::abs(m(i, j)));
        }
      worst = std::max(worst, dmax / std::max(rmax, 1e-300));
    }
  }
  const bool pass = worst <= tol;
  std::cout << "route: " << (fused ? (bf16 ? "fused bf16" : "fused f32") : "generic f64") << "\n"
            << "trials: " << trials << "\n"
            << "max |gpu - reference| / max |reference|: " << worst << " (tolerance " << tol << ")\n"
            << "verdict: " << (pass ? "equivalent" : "NOT equivalent") << "\n";
  return pass ? 0 : 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: bfgpu-cli <snapshots|recognize|run|verify> ...\n";
    return 1;
  }
  try {
    const std::string cmd = argv[1];
    const Args a = parse_args(argc, argv, 2);
    if (cmd == "snapshots") return cmd_snapshots(a);
    if (cmd == "recognize") return cmd_recognize(a);
    if (cmd == "run") return cmd_run(a);
    if (cmd == "verify") return cmd_verify(a);
    throw Error("unknown subcommand '" + cmd + "'");
  } catch (const std::exception& e) {
    std::cerr << "bfgpu-cli: error: " << e.what() << "\n";
    return 1;
  }
}
