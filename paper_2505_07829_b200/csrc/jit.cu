// Run-time compilation of generated kernels (bf_jit_*, include/bfgpu.h).
//
// The block-program compiler (host/bfgpu_codegen.cpp) emits one CUDA kernel per top-level
// operator of a program the fused kernels do not cover. This unit compiles that source with
// NVRTC straight to an sm_100a cubin, loads it with the driver API and launches it. NVRTC is
// opened at run time (dlopen libnvrtc.so.12) and the driver entry points come from the
// runtime (cudaGetDriverEntryPoint), so libbfgpu.so links neither. Modules are cached by
// source text: a program compiles once per process.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "bfgpu.h"
#include "common.hpp"

namespace bfgpu {

namespace {

struct Nvrtc {
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;
  const char* (*error_string)(nvrtcResult) = nullptr;
  std::string why;
};

const Nvrtc& nvrtc() {
  static Nvrtc n = [] {
    Nvrtc r;
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) {
      r.why = std::string("libnvrtc.so.12 not loadable: ") + dlerror();
      return r;
    }
    r.create = reinterpret_cast<decltype(r.create)>(dlsym(h, "nvrtcCreateProgram"));
    r.compile = reinterpret_cast<decltype(r.compile)>(dlsym(h, "nvrtcCompileProgram"));
    r.log_size = reinterpret_cast<decltype(r.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
    r.log = reinterpret_cast<decltype(r.log)>(dlsym(h, "nvrtcGetProgramLog"));
    r.cubin_size = reinterpret_cast<decltype(r.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
    r.cubin = reinterpret_cast<decltype(r.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
    r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "nvrtcGetErrorString"));
    if (!(r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy && r.error_string))
      r.why = "libnvrtc lacks a needed symbol";
    return r;
  }();
  return n;
}

struct Driver {
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*get_function)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
  CUresult (*func_set_attribute)(CUfunction, CUfunction_attribute, int) = nullptr;
};

template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
      !p)
    throw Status(BF_ERR_CUDA, std::string("driver entry point ") + name + " unavailable");
  return reinterpret_cast<F>(p);
}

const Driver& driver() {
  static Driver d = [] {
    Driver r;
    r.load = driver_fn<decltype(r.load)>("cuModuleLoadData");
    r.get_function = driver_fn<decltype(r.get_function)>("cuModuleGetFunction");
    r.launch = driver_fn<decltype(r.launch)>("cuLaunchKernel");
    r.func_set_attribute = driver_fn<decltype(r.func_set_attribute)>("cuFuncSetAttribute");
    return r;
  }();
  return d;
}

#define BF_CU(call)                                                                               \
  do {                                                                                            \
    CUresult r_ = (call);                                                                         \
    if (r_ != CUDA_SUCCESS) throw Status(BF_ERR_CUDA, std::string(#call) + " failed, CUresult " + \
                                                          std::to_string(static_cast<int>(r_))); \
  } while (0)

struct Module {
  int device = 0;
  CUmodule mod = nullptr;
  std::map<std::string, CUfunction> fns;
};

std::mutex g_jit_mu;

}  // namespace

void note_launch();

}  // namespace bfgpu

using namespace bfgpu;

namespace bfgpu {
namespace {

// NVRTC to an sm_100a cubin; throws with the log on failure. Needs no device.
std::vector<char> nvrtc_cubin(const char* source, char* log, size_t log_len) {
  const Nvrtc& nv = nvrtc();
  if (!nv.why.empty()) throw Status(BF_ERR_UNSUPPORTED, nv.why);
  nvrtcProgram prog = nullptr;
  if (nv.create(&prog, source, "bf_block_program.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw Status(BF_ERR_INTERNAL, "nvrtcCreateProgram failed");
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo"};
  const nvrtcResult rc = nv.compile(prog, 4, opts);
  size_t ls = 0;
  nv.log_size(prog, &ls);
  std::string text(ls, '\0');
  if (ls) nv.log(prog, text.data());
  if (log && log_len) {
    const size_t n = std::min(log_len - 1, text.size());
    std::copy(text.begin(), text.begin() + static_cast<long>(n), log);
    log[n] = '\0';
  }
  if (rc != NVRTC_SUCCESS) {
    nv.destroy(&prog);
    throw Status(BF_ERR_INTERNAL, std::string("NVRTC: ") + nv.error_string(rc) + "\n" + text);
  }
  size_t cs = 0;
  nv.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  nv.cubin(prog, cubin.data());
  nv.destroy(&prog);
  return cubin;
}

}  // namespace
}  // namespace bfgpu

extern "C" {

int bf_jit_check(const char* source, char* log, size_t log_len) {
  return guarded([&] {
    BF_CHECK_ARG(source, "bf_jit_check: null source");
    nvrtc_cubin(source, log, log_len);
  });
}

int bf_jit_compile(const char* source, void** module, char* log, size_t log_len) {
  return guarded([&] {
    BF_CHECK_ARG(source && module, "bf_jit_compile: null argument");
    static std::map<std::pair<int, std::string>, std::unique_ptr<Module>> cache;
    int dev = 0;
    BF_CUDA(cudaGetDevice(&dev));
    BF_CUDA(cudaFree(nullptr));  // make sure the primary context is current for the driver calls
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto key = std::make_pair(dev, std::string(source));
    auto it = cache.find(key);
    if (it != cache.end()) {
      *module = it->second.get();
      return;
    }
    std::vector<char> cubin = nvrtc_cubin(source, log, log_len);
    auto m = std::make_unique<Module>();
    m->device = dev;
    BF_CU(driver().load(&m->mod, cubin.data()));
    *module = m.get();
    cache.emplace(key, std::move(m));
  });
}

int bf_jit_launch(void* module, const char* kernel, unsigned grid_x, unsigned grid_y, unsigned block,
                  size_t dyn_smem, void* stream, void** args) {
  return guarded([&] {
    BF_CHECK_ARG(module && kernel && args, "bf_jit_launch: null argument");
    Module* m = static_cast<Module*>(module);
    CUfunction fn = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_jit_mu);
      auto it = m->fns.find(kernel);
      if (it == m->fns.end()) {
        BF_CU(driver().get_function(&fn, m->mod, kernel));
        if (dyn_smem > 48 * 1024)
          BF_CU(driver().func_set_attribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                            static_cast<int>(dyn_smem)));
        m->fns.emplace(kernel, fn);
      } else {
        fn = it->second;
      }
    }
    BF_CU(driver().launch(fn, grid_x, grid_y, 1, block, 1, 1, static_cast<unsigned>(dyn_smem),
                          static_cast<CUstream>(stream), args, nullptr));
    note_launch();
  });
}

}  // extern "C"
