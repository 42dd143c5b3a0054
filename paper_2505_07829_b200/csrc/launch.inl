// Template body of launch_planned (plan.hpp).
#pragma once

#include <utility>

#include "common.hpp"

namespace bfgpu {

template <class... KArgs, class... Args>
void launch_planned(const Plan& pl, void (*kernel)(KArgs...), cudaStream_t stream, Args&&... args) {
  ensure_smem_attr(reinterpret_cast<const void*>(kernel), pl.spec.smem_bytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(pl.grid));
  cfg.blockDim = dim3(static_cast<unsigned>(pl.spec.threads));
  cfg.dynamicSmemBytes = static_cast<size_t>(pl.spec.smem_bytes);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (pl.spec.grid_sync) {
    if (pl.grid > pl.resident_ctas)
      throw Status(BF_ERR_INTERNAL, std::string(pl.spec.name) + ": plan launches " + std::to_string(pl.grid) +
                                        " CTAs but only " + std::to_string(pl.resident_ctas) + " fit at once");
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  BF_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  note_launch();
}

}  // namespace bfgpu
