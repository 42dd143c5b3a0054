#include <cuda_runtime.h>
#include "common.hpp"
namespace bfgpu {
size_t lnmm_workspace_bytes(int64_t, int64_t, int64_t, int) { return 256; }
void lnmm_bf16(const void*, const void*, void*, int64_t, int64_t, int64_t, float, void*, size_t, cudaStream_t) {
  throw Status(BF_ERR_UNSUPPORTED, "bf16 layernorm_matmul not built yet");
}
void attention_bf16(const void*, const void*, const void*, void*, int64_t, int64_t, int64_t, int64_t, int64_t, float, cudaStream_t) {
  throw Status(BF_ERR_UNSUPPORTED, "bf16 attention not built yet");
}
}
