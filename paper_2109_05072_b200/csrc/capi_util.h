// Shared helpers of the C-ABI translation units (capi.cu, dist.cu): the
// opaque handle types and the status / error conventions of hexbp_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "internal.h"

struct hexbp_setup_s {
  hxb::Setup s;
};
struct hexbp_workspace_s {
  hxb::Workspace w;
};

namespace hxb {

inline int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return HEXBP_OK;
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  cudaGetLastError();  // clear sticky non-fatal errors
  return e == cudaErrorMemoryAllocation ? HEXBP_OUT_OF_MEMORY : HEXBP_CUDA_ERROR;
}

#define CK(call)                                               \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return hxb::cuda_status(_e, #call); \
  } while (0)

inline int invalid(const std::string& m) {
  set_error(m);
  return HEXBP_INVALID_ARGUMENT;
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace hxb
