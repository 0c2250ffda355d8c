// CUDA source generator for the CG tensor-product kernels (sm_100a).
//
// Replaces the reference's IR generator + interpreter (kernelgen::gen_forward /
// gen_backward / interpret, kernelgen.cpp:135-251, 547-675): instead of an op
// stream interpreted per row, every split subkernel becomes straight-line CUDA
// with its CG coefficients as immediates, and a row's units run back to back
// in one warp. Inputs are staged per (unit, item) into shared memory by the
// bulk-copy engine (cp.async.bulk + mbarrier, a D-deep ring per warp); outputs
// leave through a per-warp staging buffer as coalesced 16-byte stores.
//
// The same per-subkernel code drives three loop structures:
//   Rows          batched TP: item = (row, unit); every output row-owned.
//   ConvByOutput  fused conv, row = output node s (CSR by s): for each unit,
//                 stream the row's edges and accumulate z_s in registers
//                 (conv.cpp:234-355, without the chunk fixup: rows are owned).
//   ConvByInput   fused conv, row = neighbour node d (transposed CSR):
//                 for each edge, all units; gx_d accumulated in registers,
//                 per-edge gy / gW written directly (conv.cpp:357-528).
//   ConvEdges     atomic-mode conv over an edge list in any order (ConvPlan
//                 Mode::atomic, conv.cpp:311-324): item = (edge, unit); node
//                 outputs (z at src, gx at dst) accumulate with vector float
//                 atomics, per-edge gy / gW written directly.
#pragma once

#include <string>
#include <vector>

#include "problem.hpp"

namespace cgf {

enum class Op : int { Fwd = 0, Bwd = 1, DBwd = 2 };

// What each generated kernel computes.
enum class Comp : int {
  Fwd = 0,    // z = W . cg(x, y)
  Bwd = 1,    // gx, gy, gW
  DBwd = 2,   // dx, dy, dW, dgz in one pass (unfused TP)
  DBwdZ = 3,  // conv double-backward pass 1: dgz = W.(cg(da,y)+cg(x,db)) + dC.cg(x,y)
  DBwdX = 4,  // conv double-backward pass 2: dx, dy, dW
};

enum class Loop : int { Rows = 0, ConvByOutput = 1, ConvByInput = 2, ConvEdges = 3 };

struct KernelConfig {
  Comp comp = Comp::Fwd;
  Loop loop = Loop::Rows;
  bool f64 = false;
  bool w_shared = false;  // one W row for every batch row (superset of the reference API)
  bool aligned = true;    // all base pointers 16-byte aligned -> bulk copies allowed
  int warps = 4;          // warps per CTA
  int depth = 0;          // staging ring depth per warp (0: from the slot size)
  int min_blocks = 0;     // __launch_bounds__ min blocks per SM (0: unset)
  bool sub_barrier = true;  // compiler memory barrier between subkernels
  bool y_regs = false;    // Rows loop: y / db in registers (prefetched) instead of the slot
  int max_class = 1 << 20;  // max units folded into one code body (1 = fully unrolled units)
  int merge = 1;            // chunks (same-shape units) per staged item and code body
  bool joint = false;       // emit a merged unit's chunks side by side (shared v*y[j] products); measured
                            // neutral on the TP, +15 % on the C4 conv forward (profiles/r01_ab_joint.log)
  bool merge_all = false;   // every unit in one staged item (small problems: the whole row in registers)
  bool par_bulk = false;    // lane copy: one cp.async.bulk per contiguous range, one lane each
  bool old_issue = false;   // A/B: per-range 64-bit source addresses in issue_unit
  bool y_window = false;    // stage y as a 16-byte window even when its rows are aligned (A/B)
  bool lane_copy = true;    // stage inputs with per-lane 16-byte cp.async (whole warp) instead of
                            // one lane's cp.async.bulk: no single-lane issue loop per range
  // ConvByInput over a GROUP of units (the kernel is given a unit subset):
  // gy-type per-edge outputs add to what earlier groups wrote (read-modify-
  // write in group order, deterministic) instead of overwriting.
  bool gy_accum = false;
  bool x_regs = false;      // each staged x (and dL/da) chunk loaded into registers once per item, not per sub
  bool y_item = false;      // y (and db) loaded into registers once per item, not per CG entry
  bool ffma2 = false;
  bool pair_edges = false;  // ConvByOutput FP32 forward: two edges per item as paired FP32 ops (forces EB = 2)       // with joint emission of 2 merged chunks: paired FP32 ops (FFMA2 / FMUL2)
  int edges_per_item = 1;   // ConvByOutput: consecutive edges of a row staged in one item (one wait / issue per EB edges)
  bool wait_sleep = false;  // consumer waits: mbarrier.try_wait with a suspend-time hint
  bool l2_hints = false;    // conv loops: L2 evict_last for gathered node rows, evict_first for per-edge streams
  bool unrolled_stores = false;  // staged output pieces stored by a compile-time-unrolled lane loop (else a runtime loop)
  bool pair_weights = true;  // forward, 2 merged kind-B chunks: the weight application as fma.rn.f32x2
  bool multi_sum = true;      // dy warp sums by recursive halving (warp_sum_n) instead of one butterfly per value
  bool edge_partials = false;  // ConvEdges backward: g_node_x as per-edge partial rows (O0 + eid * dim_x, plain stores)
  std::string tag;          // appended to the kernel name (e.g. the group "g1of3")
};

// Applies "k=v,flag,..." overrides (env CGF_GEN) to a config: depth=N,
// warps=N, minb=N, nobarrier, barrier, yreg, yslot, class=N, bulk (one-lane bulk copies), lanecopy,
// merge=N, joint / nojoint, ywin.
void apply_gen_flags(KernelConfig& cfg, const std::string& flags);

struct KernelSource {
  std::string name;    // entry point
  std::string module;  // cubin cache name when several entry points share one source (default: name)
  std::string source;
  int threads = 0;
  int smem_bytes = 0;
  int units = 0;
  int bulk_ranges = 0;  // ranges moved by cp.async.bulk per item
  int sync_ranges = 0;  // ranges copied by the warp (unaligned)
};

// Kernel parameters (all generated kernels share this signature):
//   (const T* X, const T* Y, const T* W, const T* GZ, const T* DA, const T* DB,
//    const T* DC, T* O0, T* O1, T* O2, T* O3, i64 rows,
//    const i64* RP, const int* NB, const int* EID)
// Rows: rows = batch rows; RP/NB/EID unused.
// ConvByOutput: rows = nodes, RP = CSR row_ptr by output node, NB[e] = the
//   neighbour read by edge e (reference `dst`); edge id = CSR position.
// ConvByInput: rows = nodes, RP = transposed row_ptr, NB[q] = output node of
//   transposed position q, EID[q] = its edge id.
// ConvEdges: rows = nodes, edges_tot = edges, EID[e] = output node (src) of
//   edge e, NB[e] = its neighbour (dst); RP unused. Node outputs must be zeroed.
// Outputs: Fwd O0=z; Bwd O0=gx O1=gy O2=gW; DBwd O0=dx O1=dy O2=dW O3=dgz;
//   DBwdZ O3=dgz; DBwdX O0=dx O1=dy O2=dW.
KernelSource generate_kernel(const Problem& p, const std::vector<Unit>& units,
                             const KernelConfig& cfg);

// Shared device helpers (mbarrier, bulk copy, cooperative copies), prepended
// to every generated translation unit.
const char* device_runtime_source();

}  // namespace cgf
