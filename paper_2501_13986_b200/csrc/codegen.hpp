// CUDA source generator for the CG tensor-product kernels (sm_100a).
//
// Replaces the reference's IR generator + interpreter (kernelgen::gen_forward /
// gen_backward / interpret, kernelgen.cpp:135-251, 547-675): instead of an op
// stream interpreted per row, every split subkernel becomes straight-line CUDA
// with its CG coefficients as immediates, and the whole row is one warp's
// program. Inputs are staged per unit into shared memory by the bulk-copy
// engine (cp.async.bulk + mbarrier, a D-deep per-warp ring); outputs leave
// through a per-warp staging buffer as coalesced 16-byte stores.
#pragma once

#include <string>
#include <vector>

#include "problem.hpp"

namespace cgf {

enum class Op : int { Fwd = 0, Bwd = 1, DBwd = 2 };

struct KernelConfig {
  Op op = Op::Fwd;
  bool f64 = false;
  bool w_shared = false;  // one W row for every batch row (superset of the reference API)
  bool aligned = true;    // all base pointers 16-byte aligned -> bulk copies allowed
  int warps = 4;          // warps per CTA
  int depth = 3;          // staging ring depth per warp
};

struct KernelSource {
  std::string name;
  std::string source;
  int threads = 0;
  int smem_bytes = 0;
  int units = 0;
  int bulk_ranges = 0;  // ranges moved by cp.async.bulk per row
  int sync_ranges = 0;  // ranges copied by the warp (unaligned)
};

KernelSource generate_tp_kernel(const Problem& p, const std::vector<Unit>& units,
                                const KernelConfig& cfg);

// Shared device helpers (mbarrier, bulk copy, cooperative copies), prepended
// to every generated translation unit.
const char* device_runtime_source();

}  // namespace cgf
