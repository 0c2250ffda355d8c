// NVRTC -> sm_100a cubin -> CUmodule, with a content-addressed on-disk cache.
// Uses the CUDA driver API only (no cudart), so device pointers and streams
// from any runtime (PyTorch's included) interoperate through the primary
// context.
#pragma once

#include <cuda.h>

#include <cstdint>
#include <string>

#include "codegen.hpp"

namespace cgf {

struct JitError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void cu_check(CUresult r, const char* what);
#define CU_CHECK(x) ::cgf::cu_check((x), #x)

// Makes sure a context is current on this thread (the device's primary
// context, shared with PyTorch / cudart). Returns it.
CUcontext ensure_context(int device = -1);

struct Kernel {
  CUfunction fn = nullptr;
  int threads = 0;
  int smem_bytes = 0;
  int max_grid = 0;  // resident CTAs on the whole device
  std::string name;
};

// Compiles (or loads from cache) and returns the kernel for the current
// context. Thread-safe.
Kernel load_kernel(const KernelSource& ks);

// Compile only (no device needed): returns the cubin, caching it on disk.
std::string compile_cubin(const std::string& source, const std::string& name);

std::string cache_dir();
std::string nvrtc_options_string();

}  // namespace cgf
