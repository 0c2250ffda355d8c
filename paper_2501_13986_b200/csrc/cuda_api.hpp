// The CUDA driver API, resolved at run time with dlopen("libcuda.so.1") so the
// library loads (and the planner / code generator / NVRTC work) on hosts
// without a driver; compute entry points then fail with CGF_E_CUDA.
#pragma once

#include <cuda.h>

namespace cgf::drv {

#define CGF_DRV_FUNCS(X)                                                                  \
  X(cuInit) X(cuCtxGetCurrent) X(cuCtxSetCurrent) X(cuDeviceGet) X(cuDevicePrimaryCtxRetain) \
  X(cuGetErrorName) X(cuGetErrorString) X(cuModuleLoadData) X(cuModuleGetFunction)         \
  X(cuFuncSetAttribute) X(cuOccupancyMaxActiveBlocksPerMultiprocessor) X(cuCtxGetDevice)   \
  X(cuDeviceGetAttribute) X(cuLaunchKernel) X(cuMemsetD8Async) X(cuMemAlloc) X(cuMemFree)  \
  X(cuMemcpyHtoD) X(cuMemcpyDtoH) X(cuCtxSynchronize) X(cuMemcpyHtoDAsync)                 \
  X(cuMemcpyDtoHAsync) X(cuStreamSynchronize) X(cuLaunchKernelEx) X(cuFuncGetAttribute)    \
  X(cuTensorMapEncodeTiled) X(cuStreamCreate) X(cuStreamDestroy)

#define CGF_DRV_DECL(fn) extern decltype(&::fn) fn;
CGF_DRV_FUNCS(CGF_DRV_DECL)
#undef CGF_DRV_DECL

// Loads libcuda once; false (with a message) when no driver is present.
bool load(std::string* why = nullptr);

}  // namespace cgf::drv
