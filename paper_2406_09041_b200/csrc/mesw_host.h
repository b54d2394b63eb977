// Internal host helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <utility>
#include "../../include/mesw.h"

// Record `msg` as the thread's last error and return `code`.
int mesw_fail(int code, const char* msg);
// Check for a launch error after a kernel launch.
int mesw_check_launch(const char* what);
// Programmatic dependent launch enabled (mesw_set_pdl)?
int mesw_pdl_enabled();

// Launch `k` with the PDL attribute when enabled (kernels call pdl_wait() before
// touching dependent data; see mesw_common.cuh).
template <typename... KArgs, typename... Args>
inline cudaError_t mesw_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                               Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = mesw_pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
