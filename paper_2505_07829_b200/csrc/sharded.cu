// Row/head-sharded multi-GPU launch from one host thread (bf_launch_sharded, include/bfgpu.h).
//
// The three fused programs shard with no exchange step: K1 and K2 rows are
// independent (per-row statistics; the reference's M map is a forall, interpreter.hpp:334) and
// K3 heads are independent. Shard g runs its own kernel on its own device with replicated
// operands; nothing crosses devices unless the caller asks for the output to be gathered.
// The gather is an all-gather-v: every shard's rows are broadcast from their owner into every
// device's full output, as one NCCL group over a single-process communicator (NVLink /
// NVSwitch), or with peer copies when devices repeat (two shards on one GPU) or NCCL is absent.
// NCCL is loaded at run time (dlopen of libnccl.so.2), so the library itself has no link
// dependency on it and uses the NCCL already in the process when there is one (torch's).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "bfgpu.h"
#include "common.hpp"

namespace bfgpu {

namespace {

struct Nccl {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return r;
    }
    r.comm_init_all = reinterpret_cast<decltype(r.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    r.broadcast = reinterpret_cast<decltype(r.broadcast)>(dlsym(h, "ncclBroadcast"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    r.get_version = reinterpret_cast<decltype(r.get_version)>(dlsym(h, "ncclGetVersion"));
    r.ok = r.comm_init_all && r.broadcast && r.group_start && r.group_end && r.error_string;
    if (!r.ok) r.why = "libnccl.so.2 lacks a needed symbol";
    return r;
  }();
  return n;
}

#define BF_NCCL(call)                                                                                          \
  do {                                                                                                         \
    ncclResult_t r_ = (call);                                                                                  \
    if (r_ != ncclSuccess) throw Status(BF_ERR_CUDA, std::string(#call) + ": " + nccl().error_string(r_));   \
  } while (0)

// One communicator set per distinct device list, created once (ncclCommInitAll is collective
// over the listed devices and expensive).
std::vector<ncclComm_t>& comms_for(const std::vector<int>& devs) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(devs);
  if (it != cache.end()) return it->second;
  std::vector<ncclComm_t> c(devs.size());
  BF_NCCL(nccl().comm_init_all(c.data(), static_cast<int>(devs.size()), devs.data()));
  return cache.emplace(devs, std::move(c)).first->second;
}

struct DeviceGuard {
  int prev = 0;
  DeviceGuard() { BF_CUDA(cudaGetDevice(&prev)); }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

int64_t units_of(int pattern, const int64_t* dims) { return dims[0]; }  // rows (M) or heads (BH)

int64_t align_of(int pattern) { return pattern == BF_PATTERN_ATTENTION ? 1 : 128; }

}  // namespace

}  // namespace bfgpu

using namespace bfgpu;

extern "C" {

int bf_shard_range(int pattern, int64_t units, int ngpu, int shard, int64_t* start, int64_t* stop) {
  return guarded([&] {
    BF_CHECK_ARG(start && stop && ngpu > 0 && shard >= 0 && shard < ngpu && units >= 0, "bf_shard_range: bad arguments");
    const int64_t a = align_of(pattern);
    const int64_t blocks = (units + a - 1) / a;
    *start = std::min(units, blocks * shard / ngpu * a);
    *stop = std::min(units, blocks * (shard + 1) / ngpu * a);
  });
}

int bf_launch_sharded(int pattern, int ngpu, const bf_shard_io* io, const int64_t* dims, int ndims, int dtype,
                      int schedule, float eps_or_scale, int gather) {
  return guarded([&] {
    BF_CHECK_ARG(ngpu > 0 && io && dims, "bf_launch_sharded: bad arguments");
    BF_CHECK_ARG(dtype == BF_DTYPE_BF16 || dtype == BF_DTYPE_F32, "bf_launch_sharded: unknown dtype");
    const int want = pattern == BF_PATTERN_RMS_FFN_SWIGLU ? 4 : pattern == BF_PATTERN_LAYERNORM_MATMUL ? 3 : 5;
    BF_CHECK_ARG(pattern >= 0 && pattern <= 2 && ndims == want, "bf_launch_sharded: pattern/dims mismatch");
    const size_t eb = dtype == BF_DTYPE_BF16 ? 2 : 4;
    const int64_t units = units_of(pattern, dims);
    // bytes of one unit of output: a row of O (K1, K2) or one head's O (K3)
    const size_t unit_bytes = eb * static_cast<size_t>(pattern == BF_PATTERN_RMS_FFN_SWIGLU ? dims[3]
                                                       : pattern == BF_PATTERN_LAYERNORM_MATMUL ? dims[2]
                                                                                                 : dims[1] * dims[4]);
    DeviceGuard guard;
    std::vector<int64_t> start(ngpu), stop(ngpu);
    for (int g = 0; g < ngpu; ++g) {
      if (bf_shard_range(pattern, units, ngpu, g, &start[g], &stop[g]) != BF_OK)
        throw Status(BF_ERR_INVALID_ARGUMENT, bf_last_error());
    }
    // ---- compute: every shard's kernel, each on its own device and stream (asynchronous)
    for (int g = 0; g < ngpu; ++g) {
      const int64_t n = stop[g] - start[g];
      if (n == 0) continue;
      BF_CUDA(cudaSetDevice(io[g].device));
      int rc;
      if (pattern == BF_PATTERN_RMS_FFN_SWIGLU)
        rc = bf_rms_ffn_swiglu(io[g].in[0], io[g].in[1], io[g].in[2], io[g].in[3], io[g].out, n, dims[1], dims[2],
                               dims[3], dtype, eps_or_scale, schedule, io[g].workspace, io[g].workspace_bytes,
                               io[g].stream);
      else if (pattern == BF_PATTERN_LAYERNORM_MATMUL)
        rc = bf_layernorm_matmul_sched(io[g].in[0], io[g].in[1], io[g].out, n, dims[1], dims[2], dtype, eps_or_scale,
                                       schedule, io[g].workspace, io[g].workspace_bytes, io[g].stream);
      else
        rc = bf_attention_sched(io[g].in[0], io[g].in[1], io[g].in[2], io[g].out, n, dims[1], dims[2], dims[3],
                                dims[4], dtype, eps_or_scale, schedule, io[g].workspace, io[g].workspace_bytes,
                                io[g].stream);
      if (rc != BF_OK) throw Status(rc, "shard " + std::to_string(g) + ": " + bf_last_error());
    }
    if (!gather) return;
    for (int g = 0; g < ngpu; ++g) BF_CHECK_ARG(io[g].out_full, "bf_launch_sharded: gather needs out_full on every shard");
    // ---- gather: all-gather-v of the shards into every device's full output
    std::vector<int> devs(ngpu);
    for (int g = 0; g < ngpu; ++g) devs[g] = io[g].device;
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const char* mode = std::getenv("BFGPU_GATHER");  // "nccl" | "peer" (default: nccl when possible)
    const bool want_peer = mode && std::strcmp(mode, "peer") == 0;
    if (distinct && !want_peer && nccl().ok) {
      std::vector<ncclComm_t>& comms = comms_for(devs);
      BF_NCCL(nccl().group_start());
      for (int r = 0; r < ngpu; ++r) {
        const size_t bytes = static_cast<size_t>(stop[r] - start[r]) * unit_bytes;
        if (bytes == 0) continue;
        for (int g = 0; g < ngpu; ++g) {
          void* dst = static_cast<uint8_t*>(io[g].out_full) + static_cast<size_t>(start[r]) * unit_bytes;
          BF_NCCL(nccl().broadcast(g == r ? io[r].out : nullptr, dst, bytes, ncclUint8, r, comms[g],
                                   static_cast<cudaStream_t>(io[g].stream)));
        }
      }
      BF_NCCL(nccl().group_end());
      return;
    }
    if (mode && std::strcmp(mode, "nccl") == 0)
      throw Status(BF_ERR_UNSUPPORTED, distinct ? "BFGPU_GATHER=nccl: " + nccl().why
                                                : "BFGPU_GATHER=nccl needs distinct devices");
    // peer copies: device g's stream waits for shard r's kernel, then pulls its rows
    std::vector<cudaEvent_t> done(ngpu);
    for (int r = 0; r < ngpu; ++r) {
      BF_CUDA(cudaSetDevice(io[r].device));
      BF_CUDA(cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming));
      BF_CUDA(cudaEventRecord(done[r], static_cast<cudaStream_t>(io[r].stream)));
    }
    for (int g = 0; g < ngpu; ++g) {
      BF_CUDA(cudaSetDevice(io[g].device));
      auto s = static_cast<cudaStream_t>(io[g].stream);
      for (int r = 0; r < ngpu; ++r) {
        const size_t bytes = static_cast<size_t>(stop[r] - start[r]) * unit_bytes;
        if (bytes == 0) continue;
        BF_CUDA(cudaStreamWaitEvent(s, done[r], 0));
        void* dst = static_cast<uint8_t*>(io[g].out_full) + static_cast<size_t>(start[r]) * unit_bytes;
        BF_CUDA(cudaMemcpyPeerAsync(dst, io[g].device, io[r].out, io[r].device, bytes, s));
      }
    }
    for (int r = 0; r < ngpu; ++r) cudaEventDestroy(done[r]);  // destruction is deferred until the waits complete
  });
}

int bf_nccl_version(void) {
  const Nccl& n = nccl();
  int v = 0;
  if (!n.ok || !n.get_version || n.get_version(&v) != ncclSuccess) return -1;
  return v;
}

}  // extern "C"
