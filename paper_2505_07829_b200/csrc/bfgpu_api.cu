// C-ABI entry points (include/bfgpu.h). Argument validation, error mapping
// and dispatch to the per-pattern kernels; no compute happens on the host.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "bfgpu.h"
#include "common.hpp"

namespace bfgpu {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int current_device() {
  int d = 0;
  BF_CUDA(cudaGetDevice(&d));
  return d;
}

int num_sms(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lk(mu);
  if (device >= static_cast<int>(cache.size())) cache.resize(device + 1, 0);
  if (cache[device] == 0) BF_CUDA(cudaDeviceGetAttribute(&cache[device], cudaDevAttrMultiProcessorCount, device));
  return cache[device];
}

// TMA tensor maps and the 16-byte vector loads need 16-byte aligned bases (the row
// strides are checked per kernel as multiples of 8 elements).
static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static void require_sm100() {
  const int dev = current_device();
  int major = 0, minor = 0;
  BF_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  BF_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0)
    throw Status(BF_ERR_UNSUPPORTED, "bfgpu kernels are built for sm_100a only (device is sm_" +
                                         std::to_string(major) + std::to_string(minor) + ")");
}

// kernels (defined in the per-pattern translation units)
size_t ffn_workspace_bytes(int64_t M, int64_t D, int64_t F, int64_t N);
void ffn_swiglu_bf16(const void* X, const void* Wt, const void* Vt, const void* Ut, void* O, int64_t M, int64_t D,
                     int64_t F, int64_t N, float eps, int schedule, void* ws, size_t ws_bytes, cudaStream_t stream);
void ffn_swiglu_f32(const void* X, const void* Wt, const void* Vt, const void* Ut, void* O, int64_t M, int64_t D,
                    int64_t F, int64_t N, float eps, void* ws, size_t ws_bytes, cudaStream_t stream);
size_t ffn_f32_workspace_bytes(int64_t M, int64_t D, int64_t F, int64_t N);

size_t lnmm_workspace_bytes(int64_t M, int64_t K, int64_t N, int dtype);
void lnmm_bf16(const void* X, const void* Yt, void* O, int64_t M, int64_t K, int64_t N, float eps, int schedule,
               void* ws, size_t ws_bytes, cudaStream_t stream);
void lnmm_f32(const void* X, const void* Yt, void* O, int64_t M, int64_t K, int64_t N, float eps, void* ws,
              size_t ws_bytes, cudaStream_t stream);

void attention_bf16(const void* Q, const void* K, const void* Vt, void* O, int64_t BH, int64_t Sq, int64_t Skv,
                    int64_t D, int64_t Dv, float scale, int schedule, void* ws, size_t ws_bytes, cudaStream_t stream);
size_t attention_staged_workspace_bytes(int64_t BH, int64_t Sq, int64_t Skv);
void attention_f32(const void* Q, const void* K, const void* Vt, void* O, int64_t BH, int64_t Sq, int64_t Skv,
                   int64_t D, int64_t Dv, float scale, cudaStream_t stream);

}  // namespace bfgpu

using namespace bfgpu;

extern "C" {

const char* bf_last_error(void) { return g_last_error.c_str(); }

int bf_version(void) { return 1; }

uint64_t bf_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int bf_device_supported(int device) {
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess) return 0;
  return major == 10 && minor == 0;
}

size_t bf_rms_ffn_swiglu_workspace_bytes(int64_t M, int64_t D, int64_t F, int64_t N, int dtype, int schedule) {
  (void)schedule;
  if (M <= 0 || D <= 0 || F <= 0 || N <= 0) return 0;
  return dtype == BF_DTYPE_F32 ? ffn_f32_workspace_bytes(M, D, F, N) : ffn_workspace_bytes(M, D, F, N);
}

int bf_rms_ffn_swiglu(const void* X, const void* Wt, const void* Vt, const void* Ut, void* O, int64_t M, int64_t D,
                      int64_t F, int64_t N, int dtype, float eps, int schedule, void* workspace,
                      size_t workspace_bytes, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(X && Wt && Vt && Ut && O, "bf_rms_ffn_swiglu: null pointer");
    BF_CHECK_ARG(dtype != BF_DTYPE_BF16 || (aligned16(X) && aligned16(Wt) && aligned16(Vt) && aligned16(Ut) &&
                                            aligned16(O) && aligned16(workspace)),
                 "bf_rms_ffn_swiglu: bf16 buffers must be 16-byte aligned");
    require_sm100();
    auto s = static_cast<cudaStream_t>(stream);
    if (dtype == BF_DTYPE_BF16)
      ffn_swiglu_bf16(X, Wt, Vt, Ut, O, M, D, F, N, eps, schedule, workspace, workspace_bytes, s);
    else if (dtype == BF_DTYPE_F32)
      ffn_swiglu_f32(X, Wt, Vt, Ut, O, M, D, F, N, eps, workspace, workspace_bytes, s);
    else
      throw Status(BF_ERR_INVALID_ARGUMENT, "bf_rms_ffn_swiglu: unknown dtype");
  });
}

size_t bf_layernorm_matmul_workspace_bytes(int64_t M, int64_t K, int64_t N, int dtype) {
  if (M <= 0 || K <= 0 || N <= 0) return 0;
  return lnmm_workspace_bytes(M, K, N, dtype);
}

int bf_layernorm_matmul(const void* X, const void* Yt, void* O, int64_t M, int64_t K, int64_t N, int dtype, float eps,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return bf_layernorm_matmul_sched(X, Yt, O, M, K, N, dtype, eps, BF_SCHED_FUSED, workspace, workspace_bytes, stream);
}

int bf_layernorm_matmul_sched(const void* X, const void* Yt, void* O, int64_t M, int64_t K, int64_t N, int dtype,
                              float eps, int schedule, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(schedule == BF_SCHED_FUSED || schedule == BF_SCHED_STAGED, "bf_layernorm_matmul: bad schedule");
    BF_CHECK_ARG(X && Yt && O, "bf_layernorm_matmul: null pointer");
    BF_CHECK_ARG(dtype != BF_DTYPE_BF16 || (aligned16(X) && aligned16(Yt) && aligned16(O) && aligned16(workspace)),
                 "bf_layernorm_matmul: bf16 buffers must be 16-byte aligned");
    require_sm100();
    auto s = static_cast<cudaStream_t>(stream);
    if (dtype == BF_DTYPE_BF16)
      lnmm_bf16(X, Yt, O, M, K, N, eps, schedule, workspace, workspace_bytes, s);
    else if (dtype == BF_DTYPE_F32)
      lnmm_f32(X, Yt, O, M, K, N, eps, workspace, workspace_bytes, s);
    else
      throw Status(BF_ERR_INVALID_ARGUMENT, "bf_layernorm_matmul: unknown dtype");
  });
}

int bf_attention(const void* Q, const void* K, const void* Vt, void* O, int64_t BH, int64_t Sq, int64_t Skv,
                 int64_t D, int64_t Dv, int dtype, float scale, void* stream) {
  return bf_attention_sched(Q, K, Vt, O, BH, Sq, Skv, D, Dv, dtype, scale, BF_SCHED_FUSED, nullptr, 0, stream);
}

size_t bf_attention_workspace_bytes(int64_t BH, int64_t Sq, int64_t Skv, int64_t D, int64_t Dv, int dtype,
                                    int schedule) {
  (void)D;
  (void)Dv;
  if (BH <= 0 || Sq <= 0 || Skv <= 0 || schedule != BF_SCHED_STAGED || dtype != BF_DTYPE_BF16) return 0;
  return attention_staged_workspace_bytes(BH, Sq, Skv);
}

int bf_attention_sched(const void* Q, const void* K, const void* Vt, void* O, int64_t BH, int64_t Sq, int64_t Skv,
                       int64_t D, int64_t Dv, int dtype, float scale, int schedule, void* workspace,
                       size_t workspace_bytes, void* stream) {
  return guarded([&] {
    BF_CHECK_ARG(schedule == BF_SCHED_FUSED || schedule == BF_SCHED_STAGED, "bf_attention: bad schedule");
    BF_CHECK_ARG(schedule == BF_SCHED_FUSED || dtype == BF_DTYPE_BF16,
                 "bf_attention: the staged (P-buffered) schedule is bf16 only");
    BF_CHECK_ARG(Q && K && Vt && O, "bf_attention: null pointer");
    BF_CHECK_ARG(dtype != BF_DTYPE_BF16 || (aligned16(Q) && aligned16(K) && aligned16(Vt) && aligned16(O)),
                 "bf_attention: bf16 buffers must be 16-byte aligned");
    require_sm100();
    auto s = static_cast<cudaStream_t>(stream);
    if (dtype == BF_DTYPE_BF16)
      attention_bf16(Q, K, Vt, O, BH, Sq, Skv, D, Dv, scale, schedule, workspace, workspace_bytes, s);
    else if (dtype == BF_DTYPE_F32)
      attention_f32(Q, K, Vt, O, BH, Sq, Skv, D, Dv, scale, s);
    else
      throw Status(BF_ERR_INVALID_ARGUMENT, "bf_attention: unknown dtype");
  });
}

void* bf_device_alloc(size_t bytes) {
  void* p = nullptr;
  const int rc = guarded([&] { BF_CUDA(cudaMalloc(&p, bytes ? bytes : 1)); });
  return rc == BF_OK ? p : nullptr;
}

int bf_device_free(void* ptr) {
  return guarded([&] { BF_CUDA(cudaFree(ptr)); });
}

int bf_copy_to_device(void* dst, const void* src, size_t bytes, void* stream) {
  return guarded([&] {
    BF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
  });
}

int bf_copy_to_host(void* dst, const void* src, size_t bytes, void* stream) {
  return guarded([&] {
    BF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
  });
}

int bf_stream_synchronize(void* stream) {
  return guarded([&] { BF_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
}

void* bf_host_alloc(size_t bytes) {
  void* p = nullptr;
  const int rc = guarded([&] { BF_CUDA(cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable)); });
  return rc == BF_OK ? p : nullptr;
}

int bf_host_free(void* ptr) {
  return guarded([&] { BF_CUDA(cudaFreeHost(ptr)); });
}

int bf_get_device(void) {
  int d = -1;
  return guarded([&] { BF_CUDA(cudaGetDevice(&d)); }) == BF_OK ? d : -1;
}

int bf_set_device(int device) {
  return guarded([&] { BF_CUDA(cudaSetDevice(device)); });
}

}  // extern "C"
