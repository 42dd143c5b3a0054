// Host-side helpers shared by the C-ABI entry points: status codes, the
// thread-local error string behind bf_last_error(), and device queries.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "bfgpu.h"

namespace bfgpu {

struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define BF_CHECK_ARG(cond, msg)                                         \
  do {                                                                  \
    if (!(cond)) throw ::bfgpu::Status(BF_ERR_INVALID_ARGUMENT, (msg)); \
  } while (0)

#define BF_CUDA(call)                                                                                    \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess)                                                                               \
      throw ::bfgpu::Status(BF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));            \
  } while (0)

// Runs `fn`, mapping exceptions to status codes and recording the message.
template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return BF_OK;
  } catch (const Status& s) {
    set_last_error(s.what());
    return s.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return BF_ERR_INTERNAL;
  }
}

int num_sms(int device);
int current_device();

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace bfgpu
