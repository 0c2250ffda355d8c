// extern "C" boundary (include/cgf.h) over the problem planner, the code
// generator and the JIT. Exceptions never cross the boundary: each maps to a
// status code plus a thread-local message.
#include "../../include/cgf.h"

#include <cuda.h>
#include <nvrtc.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>

#include "codegen.hpp"
#include "cuda_api.hpp"
#include "jit.hpp"
#include "problem.hpp"
#include "graph_ops.hpp"
#include "uvw.hpp"
#include "schedule.hpp"

struct cgf_plan {
  cgf::Problem problem;
  std::vector<cgf::Unit> units;
  std::uint32_t budget = 4096;
  cgf::ScheduleModel sched;  // the reference's per-row schedule model (counters, dumps)
  bool z_covered = true, x_covered = true;
  std::mutex mu;
  std::map<std::tuple<int, int, int, int, int, std::string>, std::shared_ptr<cgf::KernelSource>> sources;
  // uvw tensor-core path (all-C problems, shared W): generated source and the
  // device scratch (swizzled tf32 W images, gz planes, gW partials) keyed by
  // (context, stream, buffer): each call re-images W into its stream's own
  // buffers, so calls on different streams never share scratch, and calls on
  // one stream are ordered by the stream.
  std::map<std::string, std::shared_ptr<cgf::UvwSource>> uvw;  // by kernel tag
  using ScratchKey = std::tuple<CUcontext, CUstream, std::string>;
  std::map<ScratchKey, CUdeviceptr> wimg;
  std::map<ScratchKey, std::size_t> scratch_cap;  // bytes of each buffer in wimg
  // host-pointer path: two streams + double-buffered device staging per context
  static constexpr int kPipe = 4;  // max chunks in flight: H2D(c+1) | kernels(c) | D2H(c-1) | ...
  struct HostPipe {
    CUstream s[kPipe] = {};
    CUdeviceptr buf[kPipe] = {};
    std::size_t cap[kPipe] = {};
  };
  std::map<CUcontext, HostPipe> pipes;
  std::mutex host_mu;
  int uvw_bwd_ok = -1;  // uvw backward kernels generate for this problem (-1: not yet known)
  ~cgf_plan() {
    CUcontext cur = nullptr;
    if (cgf::drv::cuCtxGetCurrent) cgf::drv::cuCtxGetCurrent(&cur);
    for (auto& [key, ptr] : wimg)
      if (cur == std::get<0>(key)) cgf::drv::cuMemFree(ptr);
    for (auto& [ctx, pp] : pipes)
      if (cur == ctx) {
        for (int k = 0; k < kPipe; ++k) {
          if (pp.buf[k]) cgf::drv::cuMemFree(pp.buf[k]);
          if (pp.s[k]) cgf::drv::cuStreamDestroy(pp.s[k]);
        }
      }
  }
};

namespace {

thread_local std::string g_err;

using cgf::BudgetError;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return CGF_OK;
  } catch (const cgf::ParseError& e) {
    g_err = e.what();
    return CGF_E_PARSE;
  } catch (const cgf::ValidationError& e) {
    g_err = e.what();
    return CGF_E_VALIDATION;
  } catch (const cgf::ShapeError& e) {
    g_err = e.what();
    return CGF_E_SHAPE;
  } catch (const BudgetError& e) {
    g_err = e.what();
    return CGF_E_BUDGET;
  } catch (const cgf::TriangleError& e) {
    g_err = e.what();
    return CGF_E_TRIANGLE;
  } catch (const cgf::JitError& e) {
    g_err = e.what();
    return CGF_E_JIT;
  } catch (const cgf::CudaError& e) {
    g_err = e.what();
    return CGF_E_CUDA;
  } catch (const cgf::UnsupportedError& e) {
    g_err = e.what();
    return CGF_E_UNSUPPORTED;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return dynamic_cast<const std::invalid_argument*>(&e) ? CGF_E_INVALID : CGF_E_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CGF_E_INTERNAL;
  }
}

bool covers(const std::vector<std::pair<std::uint32_t, std::uint32_t>>& pieces, std::uint32_t dim) {
  std::vector<char> hit(dim, 0);
  for (const auto& [off, words] : pieces)
    for (std::uint32_t k = off; k < off + words && k < dim; ++k) hit[k] = 1;
  for (char c : hit)
    if (!c) return false;
  return true;
}

// Kernels that run a problem's units in G groups, one launch each (the
// generator is given the unit subset; per-row / per-edge dy-type outputs are
// summed across groups in group order, every other output has one owner):
//
//  * by-neighbour conv (backward, double-backward pass 2): each edge gathers
//    g_node_z[s] (dim_z words); with dim_z large the rows the grid touches at
//    once overflow L2 (C4 FP64: 2.4x the algorithmic DRAM bytes,
//    profiles/r01_ncu_v5_summary.txt) and the per-warp gx accumulator caps
//    occupancy at 4 warps / SM. G groups cut both G-fold.
//  * batched double-backward (and backward): seven ops per CG entry make one
//    kernel's code overflow the instruction cache (no_instruction stalls,
//    profiles/r01_ncu_v8_dbwd.txt); G smaller kernels fit.
//
// Defaults from the sweep in profiles/r02_sweep_groups.jsonl (C4 / C5 conv,
// C1 / C2 TP); CGF_CONVI_GROUPS / CGF_ROW_GROUPS(_BWD) override.
int group_env(const char* name, int nu) {
  const char* env = std::getenv(name);
  return env ? std::clamp(std::atoi(env), 1, nu) : 0;
}

int convi_groups(const cgf_plan* p, cgf::Comp comp, int dtype) {
  const int nu = static_cast<int>(p->units.size());
  if (const int g = group_env("CGF_CONVI_GROUPS", nu)) return g;
  const std::size_t zbytes = static_cast<std::size_t>(p->problem.dim_z) * (dtype == CGF_F64 ? 8 : 4);
  // Re-swept after the multi-value warp sums (profiles/r02_sweep_groups2.jsonl)
  int g = 1;
  if (comp == cgf::Comp::Bwd)  // FP64 C4: 164 -> 59 ms at G = 8, C5 FP64: 119 -> 108 ms at G = 2; FP32: G = 1
    g = dtype == CGF_F64 ? (zbytes > 32768 ? 8 : 2) : 1;
  else  // DBwdX: C4 FP32 101 -> 83 ms and FP64 267 -> 158 ms at G = 2; C5 FP32 fastest at G = 1
    g = dtype == CGF_F32 && zbytes <= 16384 ? 1 : 2;
  return std::clamp(g, 1, nu);
}

int row_groups(const cgf_plan* p, cgf::Comp comp, int dtype) {
  const int nu = static_cast<int>(p->units.size());
  if (comp != cgf::Comp::DBwd && comp != cgf::Comp::Bwd) return 1;
  if (const int g = group_env(comp == cgf::Comp::DBwd ? "CGF_ROW_GROUPS" : "CGF_ROW_GROUPS_BWD", nu)) return g;
  // backward: FP64 C2 12.4 -> 10.9 ms at G = 2 (profiles/r02_sweep_rowbwd.jsonl); FP32 G = 1 is fastest
  if (comp == cgf::Comp::Bwd) return dtype == CGF_F64 && nu >= 8 ? 2 : 1;
  // C2 FP32 33.9 -> 28.2 ms (G = 6), FP64 29.1 -> 25.0 ms (G = 2); C1 FP32 0.29 -> 0.26 ms (G = 2)
  const int g = dtype == CGF_F32 ? std::min(6, (nu + 1) / 2) : (nu >= 8 ? 2 : 1);
  return std::clamp(g, 1, nu);
}

int kernel_groups(const cgf_plan* p, cgf::Comp comp, cgf::Loop loop, int dtype) {
  if (loop == cgf::Loop::ConvByInput) return convi_groups(p, comp, dtype);
  if (loop == cgf::Loop::Rows) return row_groups(p, comp, dtype);
  return 1;
}

// n contiguous, non-empty runs of units with about equal z words each.
std::vector<std::pair<int, int>> unit_groups(const cgf_plan* p, int n) {
  const int m = static_cast<int>(p->units.size());
  n = std::clamp(n, 1, std::max(m, 1));
  std::vector<std::uint64_t> pre(m + 1, 0);  // z words of units [0, u)
  for (int u = 0; u < m; ++u) {
    pre[u + 1] = pre[u];
    for (const auto& z : p->units[u].z_pieces) pre[u + 1] += z.words;
  }
  std::vector<std::pair<int, int>> out;
  int b = 0;
  for (int g = 0; g < n; ++g) {
    int e = m;
    if (g + 1 < n) {
      e = b + 1;
      while (e < m - (n - 1 - g) && pre[e] * n < pre[m] * (g + 1)) ++e;
    }
    out.emplace_back(b, e);
    b = e;
  }
  return out;
}

// variant 1: the ConvEdges backward writing g_node_x as per-edge partial rows
// (the row-order conv backward, conv_backward_row_order)
std::shared_ptr<cgf::KernelSource> source_for(cgf_plan* p, cgf::Comp comp, cgf::Loop loop, int dtype,
                                              int w_shared, int aligned, int group = 0, int ngroups = 1,
                                              int variant = 0) {
  if (dtype != CGF_F32 && dtype != CGF_F64) throw std::invalid_argument("bad dtype");
  std::lock_guard<std::mutex> g(p->mu);
  const char* env = std::getenv("CGF_GEN");
  const std::string flags = env ? env : "";
  const auto key = std::make_tuple(static_cast<int>(comp), static_cast<int>(loop), dtype, w_shared ? 1 : 0,
                                   aligned ? 1 : 0, flags + "|" + std::to_string(group) + "/" + std::to_string(ngroups) +
                                                        "|v" + std::to_string(variant));
  auto it = p->sources.find(key);
  if (it != p->sources.end()) return it->second;
  if (w_shared && loop != cgf::Loop::Rows) throw cgf::UnsupportedError("shared weights: batched TP only");
  cgf::KernelConfig cfg;
  cfg.comp = comp;
  cfg.loop = loop;
  cfg.f64 = dtype == CGF_F64;
  cfg.w_shared = w_shared != 0;
  cfg.aligned = aligned != 0;
  cfg.edge_partials = variant == 1;
  // output stores by compile-time-unrolled lane loops: the batched double-
  // backward -2 % (FP32) / -8 % (FP64); the forward and single backward kernels
  // are 2-7 % slower with them (profiles/r02_ab_ustore.jsonl)
  cfg.unrolled_stores = comp == cgf::Comp::DBwd && loop == cgf::Loop::Rows;
  // Batched fwd / bwd keep y in registers (prefetched a row ahead); the
  // double-backward needs those registers for its three z' accumulators.
  // FP64 backward reads y from the slot instead: the 2 x dim_y doubles of
  // registers pushed it to 255 registers + stack (measured 20.3 -> 17.4 ms).
  cfg.y_regs = (loop == cgf::Loop::Rows || loop == cgf::Loop::ConvEdges) &&
               (comp == cgf::Comp::Fwd || (comp == cgf::Comp::Bwd && dtype == CGF_F32));
  // Two 32-lane chunks per staged item / code body: measured -4 % fwd, -11 %
  // bwd (TP) and -13 % (conv) in FP32; FP64 runs out of registers (keep 1).
  cfg.merge = (dtype == CGF_F32 && (comp == cgf::Comp::Fwd || comp == cgf::Comp::Bwd)) ? 2 : 1;
  // ... emitted side by side as paired FP32 ops (FFMA2 / FMUL2: one instruction
  // per chunk pair): C2 forward 8.63 -> 8.39 ms, C4 conv forward 10.40 -> 9.44
  // ms, C4 conv backward 29.9 -> 28.8 ms (profiles/r02_ab_ffma2.jsonl); same bits
  cfg.joint = cfg.ffma2 = cfg.merge == 2;
  // Measured per kernel (profiles/r01_ab_issue.log, r01_sweep_issue_bases.log):
  // the batched forward keeps the per-range 64-bit source addresses in
  // issue_unit (9.0 vs 9.15 ms; the conv forward is faster with row bases,
  // 13.9 vs 14.6 ms); the FP64 by-neighbour conv stages y as a window (145 vs
  // 155 ms).
  cfg.old_issue = comp == cgf::Comp::Fwd && loop == cgf::Loop::Rows;
  // The FP32 batched forward issues one cp.async.bulk per contiguous range
  // (8.65 vs 9.34 ms); every other kernel is faster with lane copies
  // (profiles/r01_ab_pbulk.log).
  cfg.par_bulk = comp == cgf::Comp::Fwd && loop == cgf::Loop::Rows && dtype == CGF_F32;
  cfg.y_window = dtype == CGF_F64 && loop == cgf::Loop::ConvByInput;
  // Small problems (the whole output row fits a warp's registers: <= 64 words
  // per lane) stage every unit as ONE item per row / edge. Measured
  // (profiles/r01_ab_mergeall.log): C5 conv forward 25.2 -> 13.9 ms FP32,
  // 32.1 -> 24.4 ms FP64; C1 forward / FP32 backward -4 / -6 %; the FP64
  // backward is slower (register pressure), so it keeps per-unit items.
  {
    std::uint32_t zw = 0, xw = 0;
    for (const auto& u : p->units) {
      for (const auto& z : u.z_pieces) zw += (z.words + 31) / 32;
      for (const auto& x : u.x_chunks) xw += (x.words + 31) / 32;
    }
    const bool small = zw <= 64 && xw <= 32;
    // the FP32 conv double-backward passes too: 143.9 -> 133.6 ms on C5
    // (profiles/r01_ab_mergeall2.log; the batched and atomic ones are not faster)
    const bool conv_dbwd = (comp == cgf::Comp::DBwdZ || comp == cgf::Comp::DBwdX) && dtype == CGF_F32;
    cfg.merge_all = small && (comp == cgf::Comp::Fwd || (comp == cgf::Comp::Bwd && dtype == CGF_F32) || conv_dbwd);
    // small problems' conv kernels also issue one cp.async.bulk per contiguous
    // range (C5: FP32 bwd 44.8 -> 40.5 ms, FP64 fwd 24.7 -> 21.9, FP64 bwd 140.8 -> 130.3;
    // profiles/r01_ab_pbulk_small.log); for the C2 TP's conv they are slower
    if (small && (loop == cgf::Loop::ConvByOutput || loop == cgf::Loop::ConvByInput)) cfg.par_bulk = true;
    // the large-row conv forward is latency-bound at 2 CTAs / SM (235 registers):
    // capping registers for 3 CTAs / SM measured C4 FP32 12.9 -> 11.1 ms (the
    // backward and the small-TP (C5) kernels are slower that way,
    // profiles/r02_ab_conv2.jsonl)
    // FP64 likewise: C4 FP64 19.55 -> 17.76 ms (profiles/r02_ab_conv3/4.jsonl; C5 FP64 is slower that way)
    if (!small && loop == cgf::Loop::ConvByOutput && comp == cgf::Comp::Fwd) cfg.min_blocks = 3;
    // two consecutive edges of a row per staged item for the large-row
    // by-output kernels: C4 forward FP32 11.1 -> 10.5 ms, FP64 21.3 -> 19.5 ms
    // (profiles/r02_ab_epi.jsonl); the small-TP (C5) kernels are slower
    if (!small && loop == cgf::Loop::ConvByOutput) cfg.edges_per_item = 2;
    // small problems' conv kernels (C5), profiles/r02_ab_occ.jsonl and r02_ab_pair_*.jsonl:
    //  * forward: two edges per item as paired FP32 ops (FFMA2): 14.0 -> 12.9 ms
    //  * backward: edge pairs + one slot per warp + 3 CTAs / SM (more warps beat a
    //    deeper ring here): 40.4 -> 34.5 ms
    //  * double-backward passes: one slot per warp, 4 CTAs / SM: 123 -> 116 ms
    // and the FP64 large-row backward: one slot per warp, 82.6 -> 75.4 ms (C4)
    if (small && dtype == CGF_F32 && loop == cgf::Loop::ConvByOutput && comp == cgf::Comp::Fwd) {
      cfg.pair_edges = true;
      cfg.min_blocks = 4;  // 4 CTAs / SM: C5 forward 12.96 -> 12.22 ms (profiles/r02_ab_c5occ.jsonl)
    }
    if (small && dtype == CGF_F32 && loop == cgf::Loop::ConvByInput && comp == cgf::Comp::Bwd) {
      cfg.pair_edges = true;
      cfg.depth = 1;
      cfg.min_blocks = 3;
    }
    if (small && dtype == CGF_F32 && (comp == cgf::Comp::DBwdZ || comp == cgf::Comp::DBwdX)) {
      cfg.depth = 1;
      cfg.min_blocks = 4;
    }
    if (dtype == CGF_F64 && loop == cgf::Loop::ConvByInput && comp == cgf::Comp::Bwd) cfg.depth = 1;
  }
  // FP64 double-backward family (batched and both conv passes) and the small
  // FP64 by-neighbour backward: one slot per warp beats a deeper ring (more
  // CTAs resident): C4 conv dbl-bwd 157 -> 141 ms, C2 dbl-bwd 20.3 -> 19.1 ms,
  // C5 backward 108 -> 92 ms (profiles/r02_ab_dbwd_knobs.jsonl)
  if (dtype == CGF_F64 && (comp == cgf::Comp::DBwd || comp == cgf::Comp::DBwdZ || comp == cgf::Comp::DBwdX))
    cfg.depth = 1;
  // FP32 batched double-backward: two slots per warp, C2 25.7 -> 25.4 ms (profiles/r02_ab_c2dbwd.jsonl)
  if (dtype == CGF_F32 && comp == cgf::Comp::DBwd && loop == cgf::Loop::Rows) cfg.depth = 2;
  // x chunks / y in registers once per staged item: C4 conv double-backward
  // FP64 189.6 -> 179.4 ms, FP32 91.0 -> 88.0; C2 FP64 backward 11.40 -> 10.87
  // ms; the forward kernels are neutral or slower (profiles/r02_ab_flags.jsonl)
  cfg.x_regs = cfg.y_item = (comp != cgf::Comp::Fwd && comp != cgf::Comp::Bwd) ||
                            (comp == cgf::Comp::Bwd && loop == cgf::Loop::Rows && dtype == CGF_F64);
  cgf::apply_gen_flags(cfg, flags);
  std::vector<cgf::Unit> subset;
  if (ngroups > 1) {
    const auto grp = unit_groups(p, ngroups).at(group);
    subset.assign(p->units.begin() + grp.first, p->units.begin() + grp.second);
    cfg.gy_accum = group > 0;
    cfg.tag = "g" + std::to_string(group) + "of" + std::to_string(ngroups);
  }
  auto ks = std::make_shared<cgf::KernelSource>(
      cgf::generate_kernel(p->problem, ngroups > 1 ? subset : p->units, cfg));
  p->sources.emplace(key, ks);
  return ks;
}

std::shared_ptr<cgf::UvwSource> uvw_source(cgf_plan* p, const std::string& tag);

// The backward's gy / gW kernels need more than the forward (multiplicities
// 64, l3 <= 3, their shared-memory plans): eligible when they generate.
bool uvw_backward_ok(cgf_plan* p) {
  {
    std::lock_guard<std::mutex> g(p->mu);
    if (p->uvw_bwd_ok >= 0) return p->uvw_bwd_ok == 1;
  }
  bool ok = true;
  try {
    uvw_source(p, "bwdx");
    uvw_source(p, "bwdy");
    for (std::size_t f = 0; f < p->problem.resolved.size(); f += 6) uvw_source(p, "bwdw" + std::to_string(f));
  } catch (const cgf::UnsupportedError&) {
    ok = false;
  }
  std::lock_guard<std::mutex> g(p->mu);
  p->uvw_bwd_ok = ok ? 1 : 0;
  return ok;
}

bool use_uvw(cgf_plan* p, int op, int dtype, int w_shared) {
  if ((op != CGF_OP_FORWARD && op != CGF_OP_BACKWARD) || dtype != CGF_F32 || !w_shared) return false;
  const char* env = std::getenv("CGF_UVW");
  if (env && env[0] == '0') return false;
  if (!cgf::uvw_eligible(p->problem)) return false;
  return op == CGF_OP_FORWARD || uvw_backward_ok(p);
}

std::shared_ptr<cgf::UvwSource> uvw_source(cgf_plan* p, const std::string& tag) {
  std::lock_guard<std::mutex> g(p->mu);
  auto& slot = p->uvw[tag];
  if (!slot) {
    if (tag == "fwd") slot = std::make_shared<cgf::UvwSource>(cgf::generate_uvw_forward(p->problem));
    else if (tag == "bwdx") slot = std::make_shared<cgf::UvwSource>(cgf::generate_uvw_backward_x(p->problem));
    else if (tag == "bwdy") slot = std::make_shared<cgf::UvwSource>(cgf::generate_uvw_backward_y(p->problem));
    else if (tag.rfind("bwdw", 0) == 0) {
      const int first = std::atoi(tag.c_str() + 4);
      const int count = std::min<int>(6, static_cast<int>(p->problem.resolved.size()) - first);
      slot = std::make_shared<cgf::UvwSource>(cgf::generate_uvw_backward_w(p->problem, first, count));
    }
    else throw std::logic_error("unknown uvw kernel " + tag);
  }
  return slot;
}

std::shared_ptr<cgf::KernelSource> source_for_op(cgf_plan* p, int op, int dtype, int w_shared, int aligned) {
  if (use_uvw(p, op, dtype, w_shared))
    return std::make_shared<cgf::KernelSource>(uvw_source(p, op == CGF_OP_FORWARD ? "fwd" : "bwdx")->main);
  if (op < 0 || op > 2) throw std::invalid_argument("bad op");
  return source_for(p, static_cast<cgf::Comp>(op), cgf::Loop::Rows, dtype, w_shared, aligned);
}

bool aligned16(std::initializer_list<const void*> ptrs) {
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<std::uintptr_t>(q) & 15u)) return false;
  return true;
}

struct Args {
  const void *x = nullptr, *y = nullptr, *w = nullptr, *gz = nullptr, *da = nullptr, *db = nullptr, *dc = nullptr;
  void *o0 = nullptr, *o1 = nullptr, *o2 = nullptr, *o3 = nullptr;
  std::int64_t rows = 0;
  const void *rp = nullptr, *nb = nullptr, *eid = nullptr;
  std::int64_t edges = 0;
};

void run_kernel(cgf_plan* p, cgf::Comp comp, cgf::Loop loop, int dtype, int w_shared, const Args& a, void* stream,
                int variant = 0) {
  const std::int64_t items = loop == cgf::Loop::ConvEdges ? a.edges : a.rows;
  if (items <= 0) return;
  const bool al = aligned16({a.x, a.y, a.w, a.gz, a.da, a.db, a.dc, a.o0, a.o1, a.o2, a.o3});
  const int ng = kernel_groups(p, comp, loop, dtype);
  for (int grp = 0; grp < ng; ++grp) {
    const auto ks = source_for(p, comp, loop, dtype, w_shared, al, grp, ng, variant);
    const cgf::Kernel k = cgf::load_kernel(*ks);
    const int warps = k.threads / 32;
    const std::int64_t need = (items + warps - 1) / warps;
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(need, k.max_grid));
    Args c = a;
    void* args[] = {&c.x, &c.y, &c.w, &c.gz, &c.da, &c.db, &c.dc, &c.o0, &c.o1, &c.o2, &c.o3, &c.rows,
                    &c.rp, &c.nb, &c.eid, &c.edges};
    CU_CHECK(cgf::drv::cuLaunchKernel(k.fn, grid, 1, 1, k.threads, 1, 1, k.smem_bytes,
                                      reinterpret_cast<CUstream>(stream), args, nullptr));
  }
}

// The plan's uvw scratch buffer `name` for (current context, stream), at
// least `bytes` long. Grown buffers are freed only after the stream drained
// (its earlier kernels may still read the old one).
CUdeviceptr uvw_scratch(cgf_plan* p, CUstream st, const std::string& name, std::size_t bytes) {
  CUcontext ctx = cgf::ensure_context();
  std::lock_guard<std::mutex> g(p->mu);
  const cgf_plan::ScratchKey key{ctx, st, name};
  auto it = p->wimg.find(key);
  std::size_t& cap = p->scratch_cap[key];
  if (it != p->wimg.end() && cap >= bytes) return it->second;
  if (it != p->wimg.end()) {
    CU_CHECK(cgf::drv::cuStreamSynchronize(st));
    CU_CHECK(cgf::drv::cuMemFree(it->second));
    p->wimg.erase(it);
  }
  CUdeviceptr d = 0;
  CU_CHECK(cgf::drv::cuMemAlloc(&d, std::max<std::size_t>(bytes, 256)));
  p->wimg[key] = d;
  cap = bytes;
  return d;
}

// uvw forward on the tensor cores: W -> swizzled tf32 hi / lo images (one
// small kernel), then the warp-specialised tcgen05 kernel over 128-row tiles.
// One tcgen05 uvw kernel: `in` ([rows x in_dim], TMA-staged A source: x for
// the forward, gz for the gx backward), y, the shared W (re-imaged per call),
// `out` ([rows x out_dim]).
void run_uvw(cgf_plan* p, const std::string& tag, const void* in, int in_dim, const void* y, const void* w, void* out,
             std::int64_t rows, void* stream) {
  const auto us = uvw_source(p, tag);
  const cgf::Kernel prep = cgf::load_kernel(us->prep);
  const cgf::Kernel main = cgf::load_kernel(us->main);
  CUstream st = reinterpret_cast<CUstream>(stream);
  CUdeviceptr img = uvw_scratch(p, st, tag, us->wimg_bytes);
  Args a;
  a.x = in; a.y = y; a.w = w; a.o0 = out; a.rows = rows;
  const void* wsrc = a.w;
  void* pargs[] = {&wsrc, &img};
  const unsigned pgrid = static_cast<unsigned>((p->problem.n_w + 255) / 256);
  CU_CHECK(cgf::drv::cuLaunchKernel(prep.fn, pgrid, 1, 1, 256, 1, 1, 0, st, pargs, nullptr));
  // x viewed as [rows][dim_x / 16][16] fp32; one tile = 128 rows x dx lines of
  // 16 channels' worth of one x segment, 64-byte swizzled (conflict-free
  // per-row 16-byte reads). Rows past the batch are zero-filled by the TMA.
  if (reinterpret_cast<std::uintptr_t>(a.x) & 15u) throw cgf::ShapeError("uvw path: inputs must be 16-byte aligned");
  CUtensorMap maps[4];
  const int dxs[4] = {1, 3, 5, 7};
  for (int i = 0; i < 4; ++i) {
    const cuuint64_t gdim[3] = {16, static_cast<cuuint64_t>(in_dim / 16), static_cast<cuuint64_t>(a.rows)};
    const cuuint64_t gstride[2] = {64, static_cast<cuuint64_t>(in_dim) * 4};
    const cuuint32_t box[3] = {16, static_cast<cuuint32_t>(std::min(dxs[i], in_dim / 16)), 128};
    const cuuint32_t estr[3] = {1, 1, 1};
    CU_CHECK(cgf::drv::cuTensorMapEncodeTiled(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(a.x), gdim,
                                              gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
  const void* ya = a.y;
  void* z = a.o0;
  std::int64_t nrows = a.rows;
  const void* wi = reinterpret_cast<const void*>(img);
  const std::int64_t tiles = (a.rows + us->tile_rows - 1) / us->tile_rows;
  const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(tiles, main.max_grid));
  // CGF_UVW_PROF: per-role mbarrier wait cycles (summed over CTAs), printed per call.
  CUdeviceptr prof = 0;
  if (std::getenv("CGF_UVW_PROF")) {
    CU_CHECK(cgf::drv::cuMemAlloc(&prof, 16 * 8));
    CU_CHECK(cgf::drv::cuMemsetD8Async(prof, 0, 16 * 8, st));
  }
  void* args[] = {&maps[0], &maps[1], &maps[2], &maps[3], &ya, &wi, &z, &nrows, &prof};
  CU_CHECK(cgf::drv::cuLaunchKernel(main.fn, grid, 1, 1, main.threads, 1, 1, main.smem_bytes, st, args, nullptr));
  if (prof) {
    unsigned long long h[16];
    CU_CHECK(cgf::drv::cuStreamSynchronize(st));
    CU_CHECK(cgf::drv::cuMemcpyDtoH(h, prof, sizeof h));
    cgf::drv::cuMemFree(prof);
    static const char* names[16] = {"-", "prod:aempty", "wload:wempty", "mma:sdrained(cur)", "mma:sdrained(prev)",
                                    "mma:wfull", "mma:afull", "epi:sfull", "prod:xfull", "", "", "", "xload:xempty",
                                    "", "", "kernel(cta0 cycles x ctas)"};
    std::fprintf(stderr, "cgf_uvw prof (cycles summed over CTAs, lane-0 per warp) grid=%u:\n", grid);
    for (int i = 0; i < 16; ++i)
      if (h[i]) std::fprintf(stderr, "  %-28s %14llu  (%.1f per CTA)\n", names[i], h[i], double(h[i]) / grid);
  }
}

// dL/dy and the shared dL/dW of a uvw backward: the tcgen05 gradient kernel
// (per-CTA gW partials) + a fixed-order reduction over CTAs.
void run_uvw_grad_yw(cgf_plan* p, const void* x, const void* y, const void* w, const void* gz, void* gy, void* gw,
                     std::int64_t rows, void* stream);

void memzero(void* ptr, std::size_t bytes, void* stream) {
  if (bytes) cgf::ensure_context();  // the driver entry points resolve on first use
  if (bytes) CU_CHECK(cgf::drv::cuMemsetD8Async(reinterpret_cast<CUdeviceptr>(ptr), 0, bytes, reinterpret_cast<CUstream>(stream)));
}

// Tensor maps over a [rows][dim] fp32 array viewed as [rows][dim / 16][16]:
// boxes of 128 rows x dx lines (dx = 1, 3, 5, 7), 64-byte swizzle.
void uvw_tmaps(CUtensorMap maps[4], const void* base, int dim, std::int64_t rows, unsigned box_rows = 128) {
  if (reinterpret_cast<std::uintptr_t>(base) & 15u) throw cgf::ShapeError("uvw path: inputs must be 16-byte aligned");
  const int dxs[4] = {1, 3, 5, 7};
  for (int i = 0; i < 4; ++i) {
    const cuuint64_t gdim[3] = {16, static_cast<cuuint64_t>(dim / 16), static_cast<cuuint64_t>(rows)};
    const cuuint64_t gstride[2] = {64, static_cast<cuuint64_t>(dim) * 4};
    const cuuint32_t box[3] = {16, static_cast<cuuint32_t>(std::min(dxs[i], dim / 16)), box_rows};
    const cuuint32_t estr[3] = {1, 1, 1};
    CU_CHECK(cgf::drv::cuTensorMapEncodeTiled(&maps[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), gdim,
                                              gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  }
}

void run_uvw_grad_yw(cgf_plan* p, const void* x, const void* y, const void* w, const void* gz, void* gy, void* gw,
                     std::int64_t rows, void* stream) {
  (void)w;  // the W^T images were just written by the gx kernel's prep (same call, same stream)
  CUstream st = reinterpret_cast<CUstream>(stream);
  CUtensorMap maps[4];
  uvw_tmaps(maps, x, p->problem.dim_x, rows);
  const std::int64_t tiles = (rows + 127) / 128;
  std::int64_t nrows = rows;
  const void* ya = y;
  const void* gza = gz;
  // gz -> tf32 hi / lo planes in one pre-pass: [plane][row][64] for the gy
  // kernel's A tiles and [plane][64][pitch] for the gW kernels' B tiles (plane =
  // z segment component); both kernels then TMA-load gz tiles in MMA layout
  const auto us_y = uvw_source(p, "bwdy");
  const int nplanes = us_y->dims_x;
  std::int64_t pitch = (rows + 127) / 128 * 128;
  const std::size_t ybytes = static_cast<std::size_t>(nplanes) * static_cast<std::size_t>(rows) * 64 * 4;
  const std::size_t wbytes = static_cast<std::size_t>(nplanes) * 64 * static_cast<std::size_t>(pitch) * 4;
  const CUdeviceptr pl = uvw_scratch(p, st, "gzplanes", 2 * (ybytes + wbytes));
  void* yh = reinterpret_cast<void*>(pl);
  void* yl = reinterpret_cast<void*>(pl + ybytes);
  void* wh = reinterpret_cast<void*>(pl + 2 * ybytes);
  void* wl = reinterpret_cast<void*>(pl + 2 * ybytes + wbytes);
  {
    const cgf::Kernel planes = cgf::load_kernel(us_y->prep);
    void* pargs[] = {&gza, &yh, &yl, &wh, &wl, &nrows, &pitch};
    const std::int64_t pr = us_y->prep_rows;
    const unsigned pgrid = static_cast<unsigned>(std::min<std::int64_t>((rows + pr - 1) / pr, planes.max_grid));
    CU_CHECK(cgf::drv::cuLaunchKernel(planes.fn, pgrid, 1, 1, 256, 1, 1, us_y->prep.smem_bytes, st, pargs, nullptr));
  }
  auto plane_map = [&](CUtensorMap* m, void* base, bool rows_inner) {
    const cuuint64_t gdim_y[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(nplanes)};
    const cuuint64_t gstr_y[2] = {256, static_cast<cuuint64_t>(rows) * 256};
    const cuuint32_t box_y[3] = {32, 128, 1};
    const cuuint64_t gdim_w[3] = {static_cast<cuuint64_t>(rows), 64, static_cast<cuuint64_t>(nplanes)};
    const cuuint64_t gstr_w[2] = {static_cast<cuuint64_t>(pitch) * 4, static_cast<cuuint64_t>(pitch) * 256};
    const cuuint32_t box_w[3] = {32, 64, 1};  // 128-byte lines: half the TMA requests of 64-byte ones
    const cuuint32_t estr[3] = {1, 1, 1};
    CU_CHECK(cgf::drv::cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, rows_inner ? gdim_w : gdim_y,
                                              rows_inner ? gstr_w : gstr_y, rows_inner ? box_w : box_y, estr,
                                              CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  };
  // dL/dy
  {
    const cgf::Kernel k = cgf::load_kernel(us_y->main);
    const CUdeviceptr img = uvw_scratch(p, st, "bwdx", uvw_source(p, "bwdx")->wimg_bytes);
    CUtensorMap tg[2];
    plane_map(&tg[0], yh, false);
    plane_map(&tg[1], yl, false);
    const void* wi = reinterpret_cast<const void*>(img);
    void* gya = gy;
    void* args[] = {&maps[0], &maps[1], &maps[2], &maps[3], &tg[0], &tg[1], &ya, &wi, &gya, &nrows};
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(tiles, k.max_grid));
    CU_CHECK(cgf::drv::cuLaunchKernel(k.fn, grid, 1, 1, k.threads, 1, 1, k.smem_bytes, st, args, nullptr));
  }
  // shared dL/dW: <= 6 instructions per pass (TMEM), per-CTA partials, then a
  // fixed-order reduction of each pass's weight range
  CUtensorMap tw[2];
  plane_map(&tw[0], wh, true);
  plane_map(&tw[1], wl, true);
  const int np = static_cast<int>(p->problem.resolved.size());
  for (int first = 0; first < np; first += 6) {
    const auto us = uvw_source(p, "bwdw" + std::to_string(first));
    const cgf::Kernel k = cgf::load_kernel(us->main);
    const cgf::Kernel red = cgf::load_kernel(us->prep);
    const CUdeviceptr part = uvw_scratch(p, st, "gw_part", 4ull * k.max_grid * p->problem.n_w);
    void* pa = reinterpret_cast<void*>(part);
    CUtensorMap xm[4];
    uvw_tmaps(xm, x, p->problem.dim_x, rows, static_cast<unsigned>(us->tile_rows));
    void* args[] = {&xm[0], &xm[1], &xm[2], &xm[3], &tw[0], &tw[1], &ya, &pa, &nrows};
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(tiles, k.max_grid));
    CU_CHECK(cgf::drv::cuLaunchKernel(k.fn, grid, 1, 1, k.threads, 1, 1, k.smem_bytes, st, args, nullptr));
    const int last = std::min(np, first + 6) - 1;
    int w0 = static_cast<int>(p->problem.resolved[first].w_off);
    int w1 = static_cast<int>(p->problem.resolved[last].w_off + p->problem.resolved[last].b * p->problem.resolved[last].bp);
    int nparts = static_cast<int>(grid);
    void* gwa = gw;
    void* rargs[] = {&pa, &nparts, &gwa, &w0, &w1};
    const unsigned rgrid = static_cast<unsigned>((w1 - w0 + 255) / 256);
    CU_CHECK(cgf::drv::cuLaunchKernel(red.fn, rgrid, 1, 1, 256, 1, 1, 0, st, rargs, nullptr));
  }
}

// Batched double-backward as two kernels (CGF_DBWD_SPLIT=1 / 0 overrides).
bool dbwd_split(int dtype) {
  const char* env = std::getenv("CGF_DBWD_SPLIT");
  if (env) return env[0] == '1';
  (void)dtype;
  return false;
}

// Stream-ordered device scratch.
struct Scratch {
  void* ptr = nullptr;
  void* st = nullptr;
  bool owned = true;
  Scratch(std::size_t bytes, void* stream) : st(stream) { ptr = cgf::gops::scratch_alloc(bytes, stream); }
  Scratch(void* borrowed, void* stream) : ptr(borrowed), st(stream), owned(false) {}
  ~Scratch() {
    if (owned) cgf::gops::scratch_free(ptr, st);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  template <class T> T* as() const { return static_cast<T*>(ptr); }
};

bool dbwd_split(int dtype);

// Backward / double-backward with ONE shared W on the SIMT kernels (FP64, and
// shapes or ops the tcgen05 path does not cover): the kernel writes each row's
// weight gradient into a row-indexed workspace, which a fixed-order column sum
// folds into the shared gradient; rows run in chunks so the workspace stays
// bounded (<= 2 GiB). Deterministic: the chunking depends on rows and n_w only.
void shared_w_grad(cgf_plan* p, int op, int dtype, const Args& a, void* stream) {
  const auto& pr = p->problem;
  const std::size_t es = dtype == CGF_F64 ? 8 : 4;
  std::int64_t per = std::max<std::int64_t>(1, static_cast<std::int64_t>((2ull << 30) / (pr.n_w * es)));
  if (const char* env = std::getenv("CGF_SHARED_W_CHUNK_ROWS")) per = std::max(1, std::atoi(env));  // tests
  const std::int64_t chunk = std::min(a.rows, per);
  Scratch ws(static_cast<std::size_t>(chunk) * pr.n_w * es, stream);
  const auto off = [&](const void* q, std::int64_t r0, int dim) -> const void* {
    return q ? static_cast<const char*>(q) + es * static_cast<std::size_t>(r0) * dim : nullptr;
  };
  const auto moff = [&](void* q, std::int64_t r0, int dim) -> void* {
    return q ? static_cast<char*>(q) + es * static_cast<std::size_t>(r0) * dim : nullptr;
  };
  for (std::int64_t r0 = 0; r0 < a.rows; r0 += chunk) {
    Args c = a;
    c.rows = std::min(chunk, a.rows - r0);
    c.x = off(a.x, r0, pr.dim_x);
    c.y = off(a.y, r0, pr.dim_y);
    c.gz = off(a.gz, r0, pr.dim_z);
    c.da = off(a.da, r0, pr.dim_x);
    c.db = off(a.db, r0, pr.dim_y);
    c.o0 = moff(a.o0, r0, pr.dim_x);
    c.o1 = moff(a.o1, r0, pr.dim_y);
    c.o3 = moff(a.o3, r0, pr.dim_z);
    c.o2 = ws.ptr;  // per-row weight gradients of this chunk
    if (op == CGF_OP_DOUBLE_BACKWARD && dbwd_split(dtype)) {
      run_kernel(p, cgf::Comp::DBwdZ, cgf::Loop::Rows, dtype, 1, c, stream);
      run_kernel(p, cgf::Comp::DBwdX, cgf::Loop::Rows, dtype, 1, c, stream);
    } else {
      run_kernel(p, static_cast<cgf::Comp>(op), cgf::Loop::Rows, dtype, 1, c, stream);
    }
    cgf::gops::column_sum(dtype == CGF_F64, ws.ptr, c.rows, pr.n_w, a.o2, r0 > 0, stream);
  }
}

void launch(cgf_plan* p, int op, int dtype, int w_shared, std::int64_t rows, const void* x,
            const void* y, const void* w, const void* gz, const void* da, const void* db,
            const void* dc, void* o0, void* o1, void* o2, void* o3, void* stream) {
  if (rows < 0) throw cgf::ShapeError("rows must be non-negative");
  if (rows == 0) return;
  if (op < 0 || op > 2) throw std::invalid_argument("bad op");
  const std::size_t es = dtype == CGF_F64 ? 8 : 4;
  const auto& pr = p->problem;
  // Outputs the kernel never touches must still read as zero.
  if (op != CGF_OP_BACKWARD && !p->z_covered) memzero(op == CGF_OP_FORWARD ? o0 : o3, es * rows * pr.dim_z, stream);
  if (op != CGF_OP_FORWARD && !p->x_covered) memzero(o0, es * rows * pr.dim_x, stream);
  Args a;
  a.x = x; a.y = y; a.w = w; a.gz = gz; a.da = da; a.db = db; a.dc = dc;
  a.o0 = o0; a.o1 = o1; a.o2 = o2; a.o3 = o3; a.rows = rows;
  if (use_uvw(p, op, dtype, w_shared)) {
    if (op == CGF_OP_FORWARD) {
      run_uvw(p, "fwd", x, pr.dim_x, y, w, o0, rows, stream);
    } else {
      // backward, shared W: gx on the tensor cores (transposed forward);
      // gy and gW by the uvw gradient kernel.
      run_uvw(p, "bwdx", gz, pr.dim_z, y, w, o0, rows, stream);
      run_uvw_grad_yw(p, x, y, w, gz, o1, o2, rows, stream);
    }
    return;
  }
  if (w_shared && op != CGF_OP_FORWARD) {
    shared_w_grad(p, op, dtype, a, stream);
    return;
  }
  if (op == CGF_OP_DOUBLE_BACKWARD && dbwd_split(dtype)) {
    // two passes over the rows: dL/dgz, then (dL/dx, dL/dy, dL/dW)
    run_kernel(p, cgf::Comp::DBwdZ, cgf::Loop::Rows, dtype, w_shared, a, stream);
    run_kernel(p, cgf::Comp::DBwdX, cgf::Loop::Rows, dtype, w_shared, a, stream);
    return;
  }
  run_kernel(p, static_cast<cgf::Comp>(op), cgf::Loop::Rows, dtype, w_shared, a, stream);
}

void need(const void* ptr, const char* what) {
  if (!ptr) throw std::invalid_argument(std::string("null pointer: ") + what);
}

struct DevBuf {
  CUdeviceptr p = 0;
  explicit DevBuf(std::size_t bytes) {
    if (bytes) CU_CHECK(cgf::drv::cuMemAlloc(&p, bytes));
  }
  ~DevBuf() {
    if (p) cgf::drv::cuMemFree(p);
  }
  void* get() const { return reinterpret_cast<void*>(p); }
};

// Per-edge output node of a CSR (row_ptr by output node), on the host.
std::vector<std::int32_t> csr_sources(std::int64_t nodes, std::int64_t edges, const std::int64_t* row_ptr) {
  need(row_ptr, "row_ptr");
  if (row_ptr[0] != 0 || row_ptr[nodes] != edges) throw std::invalid_argument("row_ptr does not span the edge list");
  std::vector<std::int32_t> src(static_cast<std::size_t>(std::max<std::int64_t>(edges, 1)));
  for (std::int64_t v = 0; v < nodes; ++v) {
    if (row_ptr[v + 1] < row_ptr[v]) throw std::invalid_argument("row_ptr is not monotone");
    for (std::int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) src[e] = static_cast<std::int32_t>(v);
  }
  return src;
}

// Host-side validation of an edge list (atomic mode needs no order).
void check_edge_list(std::int64_t nodes, std::int64_t edges, const std::int32_t* src, const std::int32_t* dst) {
  if (edges == 0) return;
  need(src, "src");
  need(dst, "dst");
  for (std::int64_t e = 0; e < edges; ++e)
    if (src[e] < 0 || src[e] >= nodes || dst[e] < 0 || dst[e] >= nodes)
      throw std::invalid_argument("edge endpoint out of range");
}

// Atomic-mode conv (Mode::atomic, conv.cpp:311-324 / 470-486) over an edge
// list: one item per (edge, unit); z / gx contributions accumulate at the
// edge's src / dst nodes with float atomics into zeroed node arrays.
void conv_atomic(cgf_plan* p, int dtype, cgf::Comp comp, std::int64_t out_nodes, std::int64_t in_nodes,
                 std::int64_t edges, const std::int32_t* src, const std::int32_t* dst, Args a, void* stream) {
  if (out_nodes < 0 || in_nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
  if (edges > 0 && (out_nodes == 0 || in_nodes == 0)) throw cgf::ShapeError("edges without nodes");
  const std::size_t es = dtype == CGF_F64 ? 8 : 4;
  const auto& pr = p->problem;
  // z-type outputs live on the output nodes, x-type ones on the neighbours
  if (a.o3 || comp == cgf::Comp::Fwd) memzero(comp == cgf::Comp::Fwd ? a.o0 : a.o3, es * out_nodes * pr.dim_z, stream);
  if (comp != cgf::Comp::Fwd) memzero(a.o0, es * in_nodes * pr.dim_x, stream);
  if (edges == 0) return;
  need(src, "src"); need(dst, "dst");
  a.rows = out_nodes;
  a.edges = edges;
  a.eid = src;
  a.nb = dst;
  run_kernel(p, comp, cgf::Loop::ConvEdges, dtype, 0, a, stream);
}


// Per-edge output node of a device CSR, for the CSR entry points called with
// CGF_CONV_ATOMIC and for the unfused backward's g_node_z gather.
struct CsrSrc : Scratch {
  CsrSrc(const std::int64_t* row_ptr, std::int64_t nodes, std::int64_t edges, void* stream)
      : Scratch(edges > 0 ? 4ull * edges : 0, stream) {
    if (edges <= 0) return;
    need(row_ptr, "row_ptr");
    cgf::gops::rowptr_expand(row_ptr, nodes, as<std::int32_t>(), stream);
  }
  const std::int32_t* get() const { return as<const std::int32_t>(); }
};

// Atomic-mode conv given only the transposed CSR (the shard backward's
// arguments): the edge list is rebuilt in edge order on the device.
void atomic_transposed(cgf_plan* p, int dtype, cgf::Comp comp, std::int64_t out_nodes, std::int64_t in_nodes,
                       std::int64_t edges, const std::int64_t* t_row_ptr, const std::int32_t* t_out,
                       const std::int32_t* t_eid, const void* x, const void* y, const void* w, const void* gz,
                       const void* da, const void* db, const void* dc, void* o0, void* o1, void* o2, void* o3,
                       void* stream) {
  Scratch el(edges > 0 ? 8ull * edges : 0, stream);
  if (edges > 0) {
    need(t_out, "t_src"); need(t_eid, "t_eid");
    cgf::gops::untranspose(t_row_ptr, in_nodes, t_out, t_eid, el.as<std::int32_t>(), el.as<std::int32_t>() + edges,
                           stream);
  }
  Args a;
  a.x = x; a.y = y; a.w = w; a.gz = gz; a.da = da; a.db = db; a.dc = dc;
  a.o0 = o0; a.o1 = o1; a.o2 = o2; a.o3 = o3;
  conv_atomic(p, dtype, comp, out_nodes, in_nodes, edges, el.as<std::int32_t>(), el.as<std::int32_t>() + edges, a,
              stream);
}

// Conv backward traversal ("beware the g_node_z gather"). By
// neighbour (default kernel, transposed CSR): each edge gathers g_node_z[s]
// (dim_z words) and g_node_x[d] is summed in the warp. Row order: the edges in
// CSR order (consecutive edges share s, so g_node_z[s] is re-read from cache),
// g_node_x as per-edge partial rows (2 dim_x words of extra DRAM traffic per
// edge: written, read back) and a segmented sum over the transposed CSR.
// Chooser (whole-graph calls): CGF_CONV_BWD=row | nbr, else by neighbour. The
// traffic model favours row order whenever dim_z > 2 dim_x (C4: 9,088 vs 2,304
// words per edge; C5: 1,632 vs 576), but the kernels are issue-bound and the
// per-(edge, unit) ConvEdges kernel measured 3.3x (C4 FP32) to 23x (C5 FP32)
// slower than the by-neighbour one (profiles/r02_ab_rowbwd.jsonl), so the
// measured default is by neighbour for every problem.
bool conv_bwd_row_order(const cgf_plan* p, int dtype) {
  (void)p; (void)dtype;
  const char* e = std::getenv("CGF_CONV_BWD");
  return e && std::strcmp(e, "row") == 0;
}

// Whole graph only (cgf_conv_backward): src / nbr per edge in CSR order.
void conv_backward_row_order(cgf_plan* p, int dtype, std::int64_t nodes, std::int64_t edges,
                             const std::int64_t* row_ptr, const std::int32_t* nbr, const std::int64_t* t_row_ptr,
                             const std::int32_t* t_eid, const void* x, const void* y, const void* w, const void* gz,
                             void* gx, void* gy, void* gw, void* stream) {
  const std::size_t es = dtype == CGF_F64 ? 8 : 4;
  const auto& pr = p->problem;
  if (nodes == 0) return;
  if (edges == 0) {
    memzero(gx, es * nodes * pr.dim_x, stream);
    return;
  }
  need(x, "node_x"); need(nbr, "nbr"); need(y, "edge_y"); need(w, "edge_w"); need(gz, "g_node_z");
  need(t_row_ptr, "t_row_ptr"); need(t_eid, "t_eid"); need(gy, "g_edge_y"); need(gw, "g_edge_w"); need(gx, "g_node_x");
  const CsrSrc src(row_ptr, nodes, edges, stream);
  Scratch part(es * edges * pr.dim_x, stream);
  if (!p->x_covered) memzero(part.ptr, es * edges * pr.dim_x, stream);
  Args a;
  a.x = x; a.y = y; a.w = w; a.gz = gz;
  a.o0 = part.ptr; a.o1 = gy; a.o2 = gw;
  a.rows = nodes;
  a.edges = edges;
  a.eid = src.get();
  a.nb = nbr;
  run_kernel(p, cgf::Comp::Bwd, cgf::Loop::ConvEdges, dtype, 0, a, stream, 1);
  cgf::gops::segment_sum(dtype == CGF_F64, part.ptr, t_row_ptr, t_eid, gx, nodes, pr.dim_x, stream);
}

// Unfused comparator (conv.cpp:530-616): gather x per edge, batched TP over
// |E| rows, then per-node sums in edge order. The output node's edges are
// positions [rp[v], rp[v+1]) of the edge list, through ridx when the list is
// not in CSR order.
// Workspace of the unfused path: 256-byte aligned pieces.
std::size_t ws_round(std::size_t b) { return (b + 255) / 256 * 256; }
std::size_t unfused_ws(const cgf::Problem& pr, int dtype, int op, std::int64_t edges) {
  const std::size_t es = dtype == CGF_F64 ? 8 : 4, E = static_cast<std::size_t>(std::max<std::int64_t>(edges, 0));
  if (op == 0) return ws_round(es * E * pr.dim_x) + ws_round(es * E * pr.dim_z);
  return 2 * ws_round(es * E * pr.dim_x) + ws_round(es * E * pr.dim_z) + ws_round(4 * E);
}
struct Carver {
  char* base;
  void* carve(std::size_t b) {
    void* r = base;
    base += ws_round(b);
    return r;
  }
};

void unfused_fwd(cgf_plan* p, int dtype, std::int64_t nodes, std::int64_t edges, const std::int64_t* rp,
                 const std::int32_t* ridx, const std::int32_t* nbr, const void* node_x, const void* edge_y,
                 const void* edge_w, void* node_z, void* ws, std::size_t ws_bytes, void* stream) {
  if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
  if (nodes == 0) return;
  need(node_z, "node_z");
  const auto& pr = p->problem;
  const bool f64 = dtype == CGF_F64;
  const std::size_t es = f64 ? 8 : 4;
  if (edges == 0) {
    memzero(node_z, es * nodes * pr.dim_z, stream);
    return;
  }
  need(rp, "row_ptr"); need(nbr, "nbr"); need(node_x, "node_x"); need(edge_y, "edge_y"); need(edge_w, "edge_w");
  const std::size_t want = unfused_ws(pr, dtype, 0, edges);
  if (ws && ws_bytes < want) throw std::invalid_argument("unfused conv: workspace too small");
  Scratch all = ws ? Scratch(ws, stream) : Scratch(want, stream);
  Carver cv{all.as<char>()};
  Scratch xg(cv.carve(es * edges * pr.dim_x), stream), ze(cv.carve(es * edges * pr.dim_z), stream);
  cgf::gops::gather_rows(f64, node_x, nbr, xg.ptr, edges, pr.dim_x, stream);
  launch(p, CGF_OP_FORWARD, dtype, 0, edges, xg.ptr, edge_y, edge_w, nullptr, nullptr, nullptr, nullptr, ze.ptr,
         nullptr, nullptr, nullptr, stream);
  cgf::gops::segment_sum(f64, ze.ptr, rp, ridx, node_z, nodes, pr.dim_z, stream);
}

// src / nbr per edge (any order); (t_rp, t_idx) buckets the edges by nbr in
// edge order.
void unfused_bwd(cgf_plan* p, int dtype, std::int64_t nodes, std::int64_t edges, const std::int32_t* src,
                 const std::int32_t* nbr, const std::int64_t* t_rp, const std::int32_t* t_idx, const void* node_x,
                 const void* edge_y, const void* edge_w, const void* g_node_z, void* g_node_x, void* g_edge_y,
                 void* g_edge_w, char* ws, void* stream) {
  if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
  if (nodes == 0) return;
  need(g_node_x, "g_node_x");
  const auto& pr = p->problem;
  const bool f64 = dtype == CGF_F64;
  const std::size_t es = f64 ? 8 : 4;
  if (edges == 0) {
    memzero(g_node_x, es * nodes * pr.dim_x, stream);
    return;
  }
  need(src, "src"); need(nbr, "nbr"); need(t_rp, "t_row_ptr"); need(t_idx, "t_eid");
  need(node_x, "node_x"); need(edge_y, "edge_y"); need(edge_w, "edge_w"); need(g_node_z, "g_node_z");
  need(g_edge_y, "g_edge_y"); need(g_edge_w, "g_edge_w");
  Carver cv{ws};  // the caller sized it with unfused_ws(op 1); the last piece (src) is the caller's
  Scratch xg(cv.carve(es * edges * pr.dim_x), stream), gzg(cv.carve(es * edges * pr.dim_z), stream),
      gxe(cv.carve(es * edges * pr.dim_x), stream);
  cgf::gops::gather_rows(f64, node_x, nbr, xg.ptr, edges, pr.dim_x, stream);
  cgf::gops::gather_rows(f64, g_node_z, src, gzg.ptr, edges, pr.dim_z, stream);
  launch(p, CGF_OP_BACKWARD, dtype, 0, edges, xg.ptr, edge_y, edge_w, gzg.ptr, nullptr, nullptr, nullptr, gxe.ptr,
         g_edge_y, g_edge_w, nullptr, stream);
  cgf::gops::segment_sum(f64, gxe.ptr, t_rp, t_idx, g_node_x, nodes, pr.dim_x, stream);
}

// Stable bucket of an edge list by key on the host: rp[nodes + 1], idx.
void host_bucket(std::int64_t nodes, std::int64_t edges, const std::int32_t* key, std::vector<std::int64_t>& rp,
                 std::vector<std::int32_t>& idx) {
  rp.assign(static_cast<std::size_t>(nodes) + 1, 0);
  for (std::int64_t e = 0; e < edges; ++e) ++rp[static_cast<std::size_t>(key[e]) + 1];
  for (std::int64_t v = 0; v < nodes; ++v) rp[v + 1] += rp[v];
  std::vector<std::int64_t> next(rp.begin(), rp.end() - 1);
  idx.assign(static_cast<std::size_t>(std::max<std::int64_t>(edges, 1)), 0);
  for (std::int64_t e = 0; e < edges; ++e) idx[next[key[e]]++] = static_cast<std::int32_t>(e);
}

}  // namespace

namespace cgf {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace cgf

extern "C" {

const char* cgf_last_error(void) { return g_err.c_str(); }

const char* cgf_version(void) {
  static std::string v;
  if (v.empty()) {
    int a = 0, b = 0;
    nvrtcVersion(&a, &b);
    v = "cgf 0.1.0 nvrtc " + std::to_string(a) + "." + std::to_string(b) + " sm_100a";
  }
  return v.c_str();
}

int cgf_cg_block(int l1, int l2, int l3, int cap, int* i, int* j, int* k, double* v) {
  int n = 0;
  const int rc = guarded([&] {
    const auto b = cgf::cg_block(l1, l2, l3);
    n = static_cast<int>(b->entries.size());
    for (int e = 0; e < n && e < cap; ++e) {
      i[e] = b->entries[e].i;
      j[e] = b->entries[e].j;
      k[e] = b->entries[e].k;
      v[e] = b->entries[e].v;
    }
  });
  return rc == CGF_OK ? n : -rc;
}

int cgf_plan_create(const char* problem_json, int lane_width, uint32_t budget_words, cgf_plan** out) {
  return guarded([&] {
    need(problem_json, "problem_json");
    need(out, "out");
    *out = nullptr;
    auto p = std::make_unique<cgf_plan>();
    p->problem = cgf::parse_problem_json(problem_json, lane_width > 0 ? lane_width : 32);
    p->budget = budget_words ? budget_words : 4096;
    // The reference's schedule under the budget: its admission check (every
    // subkernel's x + y + w + z words fit, scheduler.cpp:161-170) raises
    // BudgetError here, and its phases drive the ExecStats counters.
    p->sched = cgf::build_schedule_model(p->problem, p->budget);
    p->units = cgf::plan_units(p->problem);
    std::vector<std::pair<std::uint32_t, std::uint32_t>> zs, xs;
    for (const auto& s : p->problem.subs) {
      zs.emplace_back(s.z_off, s.b * s.dz());
      xs.emplace_back(s.x_off, s.bp * s.dx());
    }
    p->z_covered = covers(zs, p->problem.dim_z);
    p->x_covered = covers(xs, p->problem.dim_x);
    *out = p.release();
  });
}

void cgf_plan_destroy(cgf_plan* plan) { delete plan; }

int cgf_plan_dims(const cgf_plan* p, int64_t dims[6]) {
  return guarded([&] {
    need(p, "plan");
    dims[0] = p->problem.dim_x;
    dims[1] = p->problem.dim_y;
    dims[2] = p->problem.dim_z;
    dims[3] = p->problem.n_w;
    dims[4] = static_cast<int64_t>(p->problem.subs.size());
    dims[5] = static_cast<int64_t>(p->units.size());
  });
}

int cgf_plan_flops(const cgf_plan* p, uint64_t flops[3]) {
  return guarded([&] {
    need(p, "plan");
    flops[0] = p->problem.fwd_flops_per_row();
    flops[1] = p->problem.bwd_flops_per_row();
    flops[2] = 3 * flops[0] + 4 * flops[1];
  });
}

int cgf_plan_source(cgf_plan* p, int op, int dtype, int w_shared, int aligned, char* buf, int cap) {
  int n = 0;
  const int rc = guarded([&] {
    need(p, "plan");
    const auto ks = source_for_op(p, op, dtype, w_shared, aligned);
    n = static_cast<int>(ks->source.size());
    if (buf && cap > 0) {
      const int m = std::min(cap - 1, n);
      std::memcpy(buf, ks->source.data(), m);
      buf[m] = 0;
    }
  });
  return rc == CGF_OK ? n : -rc;
}

int cgf_plan_compile(cgf_plan* p, int op, int dtype, int w_shared, int aligned) {
  return guarded([&] {
    need(p, "plan");
    if (use_uvw(p, op, dtype, w_shared)) {
      // every tcgen05 kernel of the op and its prep / reduction kernel
      std::vector<std::string> tags = {op == CGF_OP_FORWARD ? "fwd" : "bwdx"};
      if (op == CGF_OP_BACKWARD) {
        tags.push_back("bwdy");
        for (std::size_t f = 0; f < p->problem.resolved.size(); f += 6) tags.push_back("bwdw" + std::to_string(f));
      }
      for (const auto& tag : tags) {
        const auto us = uvw_source(p, tag);
        for (const auto* k : {&us->main, &us->prep})
          if (!k->source.empty()) cgf::compile_cubin(k->source, k->module.empty() ? k->name : k->module);
      }
      return;
    }
    const auto ks = source_for_op(p, op, dtype, w_shared, aligned);
    cgf::compile_cubin(ks->source, ks->module.empty() ? ks->name : ks->module);
  });
}

int cgf_tp_forward(cgf_plan* p, int dtype, const void* x, const void* y, const void* w, void* z,
                   int64_t rows, int w_shared, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (rows > 0) {
      need(x, "x"); need(y, "y"); need(w, "w"); need(z, "z");
    }
    launch(p, CGF_OP_FORWARD, dtype, w_shared, rows, x, y, w, nullptr, nullptr, nullptr, nullptr, z,
           nullptr, nullptr, nullptr, stream);
  });
}

int cgf_tp_backward(cgf_plan* p, int dtype, const void* x, const void* y, const void* w, const void* gz,
                    void* gx, void* gy, void* gw, int64_t rows, int w_shared, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (rows > 0) {
      need(x, "x"); need(y, "y"); need(w, "w"); need(gz, "gz");
      need(gx, "gx"); need(gy, "gy"); need(gw, "gw");
    }
    launch(p, CGF_OP_BACKWARD, dtype, w_shared, rows, x, y, w, gz, nullptr, nullptr, nullptr, gx, gy,
           gw, nullptr, stream);
  });
}

int cgf_tp_double_backward(cgf_plan* p, int dtype, const void* x, const void* y, const void* w,
                           const void* gz, const void* da, const void* db, const void* dc, void* ox,
                           void* oy, void* ow, void* ogz, int64_t rows, int w_shared, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (rows > 0) {
      need(x, "x"); need(y, "y"); need(w, "w"); need(gz, "gz"); need(da, "da"); need(db, "db");
      need(dc, "dc"); need(ox, "ox"); need(oy, "oy"); need(ow, "ow"); need(ogz, "ogz");
    }
    launch(p, CGF_OP_DOUBLE_BACKWARD, dtype, w_shared, rows, x, y, w, gz, da, db, dc, ox, oy, ow, ogz,
           stream);
  });
}

namespace {

struct HostCall {
  std::size_t es;
  std::vector<std::unique_ptr<DevBuf>> bufs;
  void* in(const void* h, std::size_t n) {
    bufs.push_back(std::make_unique<DevBuf>(n * es));
    if (n) CU_CHECK(cgf::drv::cuMemcpyHtoD(reinterpret_cast<CUdeviceptr>(bufs.back()->get()), h, n * es));
    return bufs.back()->get();
  }
  void* out(std::size_t n) {
    bufs.push_back(std::make_unique<DevBuf>(n * es));
    return bufs.back()->get();
  }
  void back(void* h, const void* d, std::size_t n) {
    if (n) CU_CHECK(cgf::drv::cuMemcpyDtoH(h, reinterpret_cast<CUdeviceptr>(d), n * es));
  }
};

}  // namespace

}  // extern "C"

namespace {

// Host-pointer path: rows stream through the GPU in chunks, each chunk on one
// of kPipe streams with its own device staging, so one chunk's host->device
// copy, another's kernels and a third's device->host copy overlap (PCIe is
// full duplex: the two directions run on separate copy engines). Staging is
// cached per plan and context. A shared-W backward reduces over all rows, so
// it runs as one chunk.
//
// op CGF_OP_FORWARD / BACKWARD / DOUBLE_BACKWARD, or kFwdBwd: forward and
// backward of the same rows in one pass (inputs x, y, w, gz; outputs z, gx,
// gy, gw), so x, y and W cross PCIe once for both.
constexpr int kFwdBwd = 3;

void run_host(cgf_plan* p, int op, int dtype, int w_shared, std::int64_t rows, const void* const in[7],
              void* const out[4]) {
  const auto& pr = p->problem;
  const std::size_t es = dtype == CGF_F64 ? 8 : 4;
  const bool ws = w_shared != 0;
  const std::size_t iw[7] = {static_cast<std::size_t>(pr.dim_x), static_cast<std::size_t>(pr.dim_y), pr.n_w,
                             static_cast<std::size_t>(pr.dim_z), static_cast<std::size_t>(pr.dim_x),
                             static_cast<std::size_t>(pr.dim_y), pr.n_w};
  const bool irow[7] = {true, true, !ws, true, true, true, !ws};
  std::size_t ow[4] = {0, 0, 0, 0};
  bool orow[4] = {true, true, true, true};
  if (op == CGF_OP_FORWARD) {
    ow[0] = pr.dim_z;
  } else if (op == kFwdBwd) {  // z, gx, gy, gw
    ow[0] = pr.dim_z; ow[1] = pr.dim_x; ow[2] = pr.dim_y; ow[3] = pr.n_w; orow[3] = !ws;
  } else {
    ow[0] = pr.dim_x; ow[1] = pr.dim_y; ow[2] = pr.n_w; orow[2] = !ws;
    if (op == CGF_OP_DOUBLE_BACKWARD) ow[3] = pr.dim_z;
  }
  std::size_t row_words = 0, fixed_words = 0;
  for (int i = 0; i < 7; ++i)
    if (in[i]) (irow[i] ? row_words : fixed_words) += iw[i];
  for (int i = 0; i < 4; ++i)
    if (out[i]) (orow[i] ? row_words : fixed_words) += ow[i];
  const bool one_chunk = ws && op != CGF_OP_FORWARD;
  std::int64_t chunk = rows;
  // staging per chunk (CGF_HOST_CHUNK_MB, default 256: 146 -> 140 ms per C2 e2e step
  // vs 128, profiles/r02_sweep_e2e.jsonl): large enough that each
  // copy runs at PCIe speed, small enough that the pipeline fills quickly;
  // CGF_HOST_DEPTH (2..4, default 3) chunks in flight
  const char* mb_env = std::getenv("CGF_HOST_CHUNK_MB");
  const char* dp_env = std::getenv("CGF_HOST_DEPTH");
  const std::size_t chunk_bytes = (mb_env ? std::max(1, std::atoi(mb_env)) : 256) * (1ull << 20);
  const int K = dp_env ? std::clamp(std::atoi(dp_env), 2, static_cast<int>(cgf_plan::kPipe)) : 3;
  if (!one_chunk) {
    const std::int64_t target = static_cast<std::int64_t>(chunk_bytes / std::max<std::size_t>(1, row_words * es));
    chunk = std::min<std::int64_t>(rows, std::max<std::int64_t>(1024, target / 128 * 128));
  }
  const std::size_t need = (fixed_words + static_cast<std::size_t>(chunk) * row_words) * es + 11 * 256;
  CUcontext ctx = cgf::ensure_context();
  std::lock_guard<std::mutex> call_lock(p->host_mu);  // one host call per plan at a time (shared staging)
  cgf_plan::HostPipe* pipe;
  {
    std::lock_guard<std::mutex> g(p->mu);
    pipe = &p->pipes[ctx];
  }
  if (!pipe->s[0])
    for (int k = 0; k < cgf_plan::kPipe; ++k) CU_CHECK(cgf::drv::cuStreamCreate(&pipe->s[k], CU_STREAM_NON_BLOCKING));
  for (int k = 0; k < K; ++k)
    if (!pipe->buf[k] || pipe->cap[k] < need) {
      if (pipe->buf[k]) {
        CU_CHECK(cgf::drv::cuStreamSynchronize(pipe->s[k]));
        cgf::drv::cuMemFree(pipe->buf[k]);
        pipe->buf[k] = 0;
      }
      CU_CHECK(cgf::drv::cuMemAlloc(&pipe->buf[k], need));
      pipe->cap[k] = need;
    }
  // chunk sequence: full chunks, with (CGF_HOST_RAMP, default on) the first and
  // last ones split into 1/8, 1/4, 1/2 pieces, so the pipeline fills (first
  // H2D alone) and drains (last D2H alone) in a small piece's time: C2 e2e step
  // 147.2 -> 146.0 and 152.3 -> 150.5 ms (profiles/r02_sweep_e2e_ramp.jsonl)
  std::vector<std::pair<std::int64_t, std::int64_t>> pieces;  // (first row, rows)
  {
    const char* ramp_env = std::getenv("CGF_HOST_RAMP");
    const bool ramp = !one_chunk && !(ramp_env && std::atoi(ramp_env) == 0) && rows >= 4 * chunk;
    std::vector<std::int64_t> sizes;
    if (ramp) {
      const std::int64_t q = std::max<std::int64_t>(128, chunk / 8 / 128 * 128);
      const std::int64_t h = std::max<std::int64_t>(128, chunk / 4 / 128 * 128);
      const std::int64_t half = std::max<std::int64_t>(128, chunk / 2 / 128 * 128);
      const std::int64_t ends[3] = {q, h, half};
      std::int64_t left = rows - 2 * (q + h + half);
      for (std::int64_t v : ends) sizes.push_back(v);
      for (; left > 0; left -= chunk) sizes.push_back(std::min(chunk, left));
      for (int i = 2; i >= 0; --i) sizes.push_back(ends[i]);
    } else {
      for (std::int64_t left = rows; left > 0; left -= chunk) sizes.push_back(std::min(chunk, left));
    }
    std::int64_t r = 0;
    for (std::int64_t v : sizes) {
      pieces.emplace_back(r, v);
      r += v;
    }
  }
  const std::int64_t nchunks = static_cast<std::int64_t>(pieces.size());
  for (std::int64_t c = 0; c < nchunks; ++c) {
    const int k = static_cast<int>(c % K);
    CUstream st = pipe->s[k];
    const std::int64_t r0 = pieces[c].first, n = pieces[c].second;
    std::size_t off = 0;
    auto carve = [&](std::size_t words) {
      const CUdeviceptr d = pipe->buf[k] + off;
      off += (words * es + 255) / 256 * 256;
      return d;
    };
    void* din[7] = {};
    for (int i = 0; i < 7; ++i) {
      if (!in[i]) continue;
      const std::size_t words = irow[i] ? iw[i] * static_cast<std::size_t>(n) : iw[i];
      const CUdeviceptr d = carve(irow[i] ? iw[i] * static_cast<std::size_t>(chunk) : iw[i]);
      din[i] = reinterpret_cast<void*>(d);
      if (irow[i] || c < K) {  // a shared W is uploaded once per staging buffer
        const char* h = static_cast<const char*>(in[i]) + (irow[i] ? es * iw[i] * static_cast<std::size_t>(r0) : 0);
        CU_CHECK(cgf::drv::cuMemcpyHtoDAsync(d, h, words * es, st));
      }
    }
    void* dout[4] = {};
    for (int i = 0; i < 4; ++i)
      if (out[i]) dout[i] = reinterpret_cast<void*>(carve(orow[i] ? ow[i] * static_cast<std::size_t>(chunk) : ow[i]));
    if (op == kFwdBwd) {
      launch(p, CGF_OP_FORWARD, dtype, w_shared, n, din[0], din[1], din[2], nullptr, nullptr, nullptr, nullptr, dout[0],
             nullptr, nullptr, nullptr, st);
      launch(p, CGF_OP_BACKWARD, dtype, w_shared, n, din[0], din[1], din[2], din[3], nullptr, nullptr, nullptr, dout[1],
             dout[2], dout[3], nullptr, st);
    } else {
      launch(p, op, dtype, w_shared, n, din[0], din[1], din[2], din[3], din[4], din[5], din[6], dout[0], dout[1],
             dout[2], dout[3], st);
    }
    for (int i = 0; i < 4; ++i) {
      if (!out[i]) continue;
      const std::size_t words = orow[i] ? ow[i] * static_cast<std::size_t>(n) : ow[i];
      char* h = static_cast<char*>(out[i]) + (orow[i] ? es * ow[i] * static_cast<std::size_t>(r0) : 0);
      CU_CHECK(cgf::drv::cuMemcpyDtoHAsync(h, reinterpret_cast<CUdeviceptr>(dout[i]), words * es, st));
    }
  }
  for (int k = 0; k < K; ++k) CU_CHECK(cgf::drv::cuStreamSynchronize(pipe->s[k]));
}

}  // namespace

extern "C" {

int cgf_tp_forward_host(cgf_plan* p, int dtype, const void* x, const void* y, const void* w, void* z,
                        int64_t rows, int w_shared) {
  return guarded([&] {
    need(p, "plan");
    if (rows <= 0) return;
    const void* in[7] = {x, y, w, nullptr, nullptr, nullptr, nullptr};
    void* out[4] = {z, nullptr, nullptr, nullptr};
    run_host(p, CGF_OP_FORWARD, dtype, w_shared, rows, in, out);
  });
}

int cgf_tp_backward_host(cgf_plan* p, int dtype, const void* x, const void* y, const void* w,
                         const void* gz, void* gx, void* gy, void* gw, int64_t rows, int w_shared) {
  return guarded([&] {
    need(p, "plan");
    if (rows <= 0) return;
    const void* in[7] = {x, y, w, gz, nullptr, nullptr, nullptr};
    void* out[4] = {gx, gy, gw, nullptr};
    run_host(p, CGF_OP_BACKWARD, dtype, w_shared, rows, in, out);
  });
}

int cgf_tp_forward_backward_host(cgf_plan* p, int dtype, const void* x, const void* y, const void* w,
                                 const void* gz, void* z, void* gx, void* gy, void* gw, int64_t rows, int w_shared) {
  return guarded([&] {
    need(p, "plan");
    if (rows <= 0) return;
    need(x, "x"); need(y, "y"); need(w, "w"); need(gz, "gz");
    need(z, "z"); need(gx, "gx"); need(gy, "gy"); need(gw, "gw");
    if (w_shared) {  // the shared gW reduces over every row: two passes
      const void* fin[7] = {x, y, w, nullptr, nullptr, nullptr, nullptr};
      void* fout[4] = {z, nullptr, nullptr, nullptr};
      run_host(p, CGF_OP_FORWARD, dtype, w_shared, rows, fin, fout);
      const void* bin[7] = {x, y, w, gz, nullptr, nullptr, nullptr};
      void* bout[4] = {gx, gy, gw, nullptr};
      run_host(p, CGF_OP_BACKWARD, dtype, w_shared, rows, bin, bout);
      return;
    }
    const void* in[7] = {x, y, w, gz, nullptr, nullptr, nullptr};
    void* out[4] = {z, gx, gy, gw};
    run_host(p, kFwdBwd, dtype, w_shared, rows, in, out);
  });
}

int cgf_tp_double_backward_host(cgf_plan* p, int dtype, const void* x, const void* y, const void* w,
                                const void* gz, const void* da, const void* db, const void* dc,
                                void* ox, void* oy, void* ow, void* ogz, int64_t rows, int w_shared) {
  return guarded([&] {
    need(p, "plan");
    if (rows <= 0) return;
    const void* in[7] = {x, y, w, gz, da, db, dc};
    void* out[4] = {ox, oy, ow, ogz};
    run_host(p, CGF_OP_DOUBLE_BACKWARD, dtype, w_shared, rows, in, out);
  });
}

int cgf_tp_stats(const cgf_plan* p, int op, int64_t rows, int w_shared, uint64_t stats[3]) {
  (void)w_shared;
  return guarded([&] {
    need(p, "plan");
    need(stats, "stats");
    if (rows < 0) throw cgf::ShapeError("rows must be non-negative");
    const auto& m = p->sched;
    const std::uint64_t R = static_cast<std::uint64_t>(rows);
    const std::uint64_t f[3] = {m.fwd_loads, m.fwd_stores, m.fwd_flops}, b[3] = {m.bwd_loads, 0, m.bwd_flops};
    for (int k = 0; k < 3; ++k) {
      switch (op) {
        case CGF_OP_FORWARD: stats[k] = R * f[k]; break;
        case CGF_OP_BACKWARD: stats[k] = R * b[k]; break;
        case CGF_OP_DOUBLE_BACKWARD: stats[k] = R * (3 * f[k] + 4 * b[k]); break;
        default: throw std::invalid_argument("bad op");
      }
    }
  });
}

int cgf_tp_traffic(const cgf_plan* p, int op, int64_t rows, int w_shared, uint64_t words[2]) {
  return guarded([&] {
    need(p, "plan");
    need(words, "words");
    const auto& pr = p->problem;
    const std::uint64_t R = static_cast<std::uint64_t>(rows);
    const std::uint64_t W = w_shared ? pr.n_w : R * pr.n_w;
    const std::uint64_t X = R * pr.dim_x, Y = R * pr.dim_y, Z = R * pr.dim_z;
    switch (op) {
      case CGF_OP_FORWARD: words[0] = X + Y + W; words[1] = Z; break;
      case CGF_OP_BACKWARD: words[0] = X + Y + W + Z; words[1] = X + Y + W; break;
      case CGF_OP_DOUBLE_BACKWARD: words[0] = 3 * (X + Y + W) + Z; words[1] = X + Y + W + Z; break;
      default: throw std::invalid_argument("bad op");
    }
  });
}

namespace {
int copy_out(const std::string& t, char* buf, int cap) {
  if (buf && cap > 0) {
    const int m = std::min<int>(cap - 1, static_cast<int>(t.size()));
    std::memcpy(buf, t.data(), m);
    buf[m] = 0;
  }
  return static_cast<int>(t.size());
}
}  // namespace

int cgf_plan_schedule_json(const cgf_plan* p, char* buf, int cap) {
  int n = 0;
  const int rc = guarded([&] {
    need(p, "plan");
    n = copy_out(cgf::schedule_json(p->problem, p->sched), buf, cap);
  });
  return rc == CGF_OK ? n : -rc;
}

int cgf_plan_listing(const cgf_plan* p, int pos, int backward, char* buf, int cap) {
  int n = 0;
  const int rc = guarded([&] {
    need(p, "plan");
    if (pos < 0 || pos >= static_cast<int>(p->problem.subs.size())) throw std::invalid_argument("subkernel position out of range");
    n = copy_out(cgf::listing_text(p->problem.subs[pos], backward != 0), buf, cap);
  });
  return rc == CGF_OK ? n : -rc;
}

int cgf_conv_stats(const cgf_plan* p, int op, int mode, int unfused, int64_t nodes, int64_t edges,
                   uint64_t st[4]) {
  return guarded([&] {
    need(p, "plan");
    need(st, "stats");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (mode != CGF_CONV_DETERMINISTIC && mode != CGF_CONV_ATOMIC) throw std::invalid_argument("bad conv mode");
    const auto& pr = p->problem;
    const std::uint64_t E = static_cast<std::uint64_t>(edges), V = static_cast<std::uint64_t>(nodes);
    const std::uint64_t dx = pr.dim_x, dy = pr.dim_y, dz = pr.dim_z, nw = pr.n_w;
    const bool atomic = mode == CGF_CONV_ATOMIC;
    if (op == CGF_OP_FORWARD) {
      if (unfused) {  // gather x per edge, TP over |E| rows, per-node sums of |E| z rows
        st[0] = E * (2 * dx + dy + nw); st[1] = E * (dx + dz); st[2] = E;
      } else {  // per edge: x[nbr] (L2), y_e, W_e; z once per row, or one reduction per edge
        st[0] = E * (dx + dy + nw); st[1] = atomic ? E * dz : V * dz; st[2] = atomic ? E : V;
      }
      st[3] = E * p->sched.fwd_flops;
    } else if (op == CGF_OP_BACKWARD) {
      if (unfused) {
        st[0] = E * (2 * dx + dy + nw + dz); st[1] = E * (2 * dx + dy + nw); st[2] = E;
      } else {
        st[0] = E * (dx + dy + nw + dz); st[1] = (atomic ? E : V) * dx + E * (dy + nw); st[2] = (atomic ? E : V) + E;
      }
      st[3] = E * p->sched.bwd_flops;
    } else {
      throw std::invalid_argument("bad op");
    }
  });
}

// ------------------------------------------------------------- convolution --

int cgf_plan_kernel_source(cgf_plan* p, int comp, int loop, int dtype, int w_shared, int aligned, char* buf,
                           int cap) {
  int n = 0;
  const int rc = guarded([&] {
    need(p, "plan");
    if (comp < 0 || comp > 4 || loop < 0 || loop > 3) throw std::invalid_argument("bad comp / loop");
    const auto ks = source_for(p, static_cast<cgf::Comp>(comp), static_cast<cgf::Loop>(loop), dtype, w_shared, aligned);
    n = static_cast<int>(ks->source.size());
    if (buf && cap > 0) {
      const int m = std::min(cap - 1, n);
      std::memcpy(buf, ks->source.data(), m);
      buf[m] = 0;
    }
  });
  return rc == CGF_OK ? n : -rc;
}

int cgf_plan_kernel_groups(const cgf_plan* p, int comp, int loop, int dtype) {
  if (!p || comp < 0 || comp > 4 || loop < 0 || loop > 3) return -CGF_E_INVALID;
  return kernel_groups(p, static_cast<cgf::Comp>(comp), static_cast<cgf::Loop>(loop), dtype);
}

int cgf_plan_kernel_source_group(cgf_plan* p, int comp, int loop, int dtype, int w_shared, int aligned, int group,
                                 char* buf, int cap) {
  int n = 0;
  const int rc = guarded([&] {
    need(p, "plan");
    if (comp < 0 || comp > 4 || loop < 0 || loop > 3) throw std::invalid_argument("bad comp / loop");
    const int ng = cgf_plan_kernel_groups(p, comp, loop, dtype);
    if (group < 0 || group >= ng) throw std::invalid_argument("kernel group out of range");
    const auto ks = source_for(p, static_cast<cgf::Comp>(comp), static_cast<cgf::Loop>(loop), dtype, w_shared, aligned,
                               group, ng);
    n = copy_out(ks->source, buf, cap);
  });
  return rc == CGF_OK ? n : -rc;
}

int cgf_plan_kernel_compile(cgf_plan* p, int comp, int loop, int dtype, int w_shared, int aligned) {
  return guarded([&] {
    need(p, "plan");
    if (comp < 0 || comp > 4 || loop < 0 || loop > 3) throw std::invalid_argument("bad comp / loop");
    const int ng = kernel_groups(p, static_cast<cgf::Comp>(comp), static_cast<cgf::Loop>(loop), dtype);
    for (int grp = 0; grp < ng; ++grp) {
      const auto ks = source_for(p, static_cast<cgf::Comp>(comp), static_cast<cgf::Loop>(loop), dtype, w_shared,
                                 aligned, grp, ng);
      cgf::compile_cubin(ks->source, ks->name);
    }
  });
}

int cgf_conv_transpose_shard_host(int64_t out_nodes, int64_t in_nodes, int64_t edges, const int64_t* row_ptr,
                                  const int32_t* nbr, int64_t* t_row_ptr, int32_t* t_out, int32_t* t_eid) {
  return guarded([&] {
    if (out_nodes < 0 || in_nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    need(t_row_ptr, "t_row_ptr");
    if (out_nodes > 0) need(row_ptr, "row_ptr");
    if (edges > 0) { need(nbr, "nbr"); need(t_out, "t_src"); need(t_eid, "t_eid"); }
    if (out_nodes > 0 && (row_ptr[0] != 0 || row_ptr[out_nodes] != edges))
      throw std::invalid_argument("row_ptr does not span the edge list");
    if (out_nodes == 0 && edges != 0) throw std::invalid_argument("row_ptr does not span the edge list");
    // Stable counting sort by neighbour (conv.cpp:135-151): within a bucket
    // edges keep CSR order, i.e. ascending output node.
    std::vector<int64_t> cnt(static_cast<size_t>(in_nodes) + 1, 0);
    for (int64_t e = 0; e < edges; ++e) {
      if (nbr[e] < 0 || nbr[e] >= in_nodes) throw std::invalid_argument("neighbour index out of range");
      ++cnt[static_cast<size_t>(nbr[e]) + 1];
    }
    for (int64_t v = 0; v < in_nodes; ++v) cnt[v + 1] += cnt[v];
    std::memcpy(t_row_ptr, cnt.data(), sizeof(int64_t) * (static_cast<size_t>(in_nodes) + 1));
    for (int64_t s = 0; s < out_nodes; ++s)
      for (int64_t e = row_ptr[s]; e < row_ptr[s + 1]; ++e) {
        const int64_t q = cnt[nbr[e]]++;
        t_out[q] = static_cast<int32_t>(s);
        t_eid[q] = static_cast<int32_t>(e);
      }
  });
}

int cgf_conv_transpose_host(int64_t nodes, int64_t edges, const int64_t* row_ptr, const int32_t* nbr,
                            int64_t* t_row_ptr, int32_t* t_out, int32_t* t_eid) {
  return cgf_conv_transpose_shard_host(nodes, nodes, edges, row_ptr, nbr, t_row_ptr, t_out, t_eid);
}

int cgf_conv_forward_shard(cgf_plan* p, int dtype, int64_t out_nodes, int64_t in_nodes, int64_t edges,
                           const int64_t* row_ptr, const int32_t* nbr, const void* node_x, const void* edge_y,
                           const void* edge_w, void* node_z, int mode, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (mode != CGF_CONV_DETERMINISTIC && mode != CGF_CONV_ATOMIC) throw std::invalid_argument("bad conv mode");
    if (out_nodes < 0 || in_nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (out_nodes == 0) return;
    need(row_ptr, "row_ptr"); need(node_z, "node_z");
    if (mode == CGF_CONV_ATOMIC) {  // Mode::atomic over the shard's CSR expanded to an edge list
      const CsrSrc src(row_ptr, out_nodes, edges, stream);
      Args a;
      a.x = node_x; a.y = edge_y; a.w = edge_w; a.o0 = node_z;
      conv_atomic(p, dtype, cgf::Comp::Fwd, out_nodes, in_nodes, edges, src.get(), nbr, a, stream);
      return;
    }
    if (edges > 0) { need(node_x, "node_x"); need(nbr, "nbr"); need(edge_y, "edge_y"); need(edge_w, "edge_w"); }
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    if (!p->z_covered) memzero(node_z, es * out_nodes * p->problem.dim_z, stream);
    Args a;
    a.x = node_x; a.y = edge_y; a.w = edge_w; a.o0 = node_z; a.rows = out_nodes;
    a.rp = row_ptr; a.nb = nbr; a.edges = edges;
    run_kernel(p, cgf::Comp::Fwd, cgf::Loop::ConvByOutput, dtype, 0, a, stream);
  });
}

int cgf_conv_forward(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr, const int32_t* nbr,
                     const void* node_x, const void* edge_y, const void* edge_w, void* node_z, int mode, void* stream) {
  if (mode == CGF_CONV_ATOMIC)
    return guarded([&] {
      need(p, "plan");
      const CsrSrc src(row_ptr, nodes, edges, stream);
      if (cgf_conv_forward_atomic(p, dtype, nodes, edges, src.get(), nbr, node_x, edge_y, edge_w, node_z, stream) != CGF_OK)
        throw std::runtime_error(g_err);
    });
  return cgf_conv_forward_shard(p, dtype, nodes, nodes, edges, row_ptr, nbr, node_x, edge_y, edge_w, node_z, mode,
                                stream);
}

int cgf_conv_backward_shard(cgf_plan* p, int dtype, int64_t out_nodes, int64_t in_nodes, int64_t edges,
                            const int64_t* t_row_ptr, const int32_t* t_out, const int32_t* t_eid, const void* node_x,
                            const void* edge_y, const void* edge_w, const void* g_node_z, void* g_node_x,
                            void* g_edge_y, void* g_edge_w, int mode, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (mode != CGF_CONV_DETERMINISTIC && mode != CGF_CONV_ATOMIC) throw std::invalid_argument("bad conv mode");
    if (out_nodes < 0 || in_nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (in_nodes == 0) return;
    need(t_row_ptr, "t_row_ptr"); need(node_x, "node_x"); need(g_node_x, "g_node_x");
    if (mode == CGF_CONV_ATOMIC) {
      // the transposed CSR as an edge list in transposed order: position q
      // is edge t_eid[q] = (t_src[q], its neighbour); per-edge outputs are
      // addressed through t_eid, so the edge arrays are permuted views
      atomic_transposed(p, dtype, cgf::Comp::Bwd, out_nodes, in_nodes, edges, t_row_ptr, t_out, t_eid, node_x, edge_y,
                        edge_w, g_node_z, nullptr, nullptr, nullptr, g_node_x, g_edge_y, g_edge_w, nullptr, stream);
      return;
    }
    if (edges > 0) {
      need(g_node_z, "g_node_z"); need(t_out, "t_src"); need(t_eid, "t_eid"); need(edge_y, "edge_y");
      need(edge_w, "edge_w"); need(g_edge_y, "g_edge_y"); need(g_edge_w, "g_edge_w");
    }
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    if (!p->x_covered) memzero(g_node_x, es * in_nodes * p->problem.dim_x, stream);
    Args a;
    a.x = node_x; a.y = edge_y; a.w = edge_w; a.gz = g_node_z;
    a.o0 = g_node_x; a.o1 = g_edge_y; a.o2 = g_edge_w; a.rows = in_nodes;
    a.rp = t_row_ptr; a.nb = t_out; a.eid = t_eid; a.edges = edges;
    run_kernel(p, cgf::Comp::Bwd, cgf::Loop::ConvByInput, dtype, 0, a, stream);
  });
}

int cgf_conv_backward(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                      const int32_t* nbr, const int64_t* t_row_ptr, const int32_t* t_out, const int32_t* t_eid,
                      const void* node_x, const void* edge_y, const void* edge_w, const void* g_node_z,
                      void* g_node_x, void* g_edge_y, void* g_edge_w, int mode, void* stream) {
  if (mode == CGF_CONV_ATOMIC)
    return guarded([&] {
      need(p, "plan");
      const CsrSrc src(row_ptr, nodes, edges, stream);
      if (cgf_conv_backward_atomic(p, dtype, nodes, edges, src.get(), nbr, node_x, edge_y, edge_w, g_node_z, g_node_x,
                                   g_edge_y, g_edge_w, stream) != CGF_OK)
        throw std::runtime_error(g_err);
    });
  if (mode == CGF_CONV_DETERMINISTIC && conv_bwd_row_order(p, dtype))
    return guarded([&] {
      need(p, "plan");
      conv_backward_row_order(p, dtype, nodes, edges, row_ptr, nbr, t_row_ptr, t_eid, node_x, edge_y, edge_w, g_node_z,
                              g_node_x, g_edge_y, g_edge_w, stream);
    });
  return cgf_conv_backward_shard(p, dtype, nodes, nodes, edges, t_row_ptr, t_out, t_eid, node_x, edge_y, edge_w,
                                 g_node_z, g_node_x, g_edge_y, g_edge_w, mode, stream);
}

int cgf_conv_double_backward_shard(cgf_plan* p, int dtype, int64_t out_nodes, int64_t in_nodes, int64_t edges,
                                   const int64_t* row_ptr, const int32_t* nbr, const int64_t* t_row_ptr,
                                   const int32_t* t_out, const int32_t* t_eid, const void* node_x,
                                   const void* edge_y, const void* edge_w, const void* g_node_z, const void* d_gx,
                                   const void* d_gy, const void* d_gw, void* o_node_x, void* o_edge_y,
                                   void* o_edge_w, void* o_g_node_z, int mode, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (mode != CGF_CONV_DETERMINISTIC && mode != CGF_CONV_ATOMIC) throw std::invalid_argument("bad conv mode");
    if (out_nodes < 0 || in_nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (mode == CGF_CONV_ATOMIC) {  // one pass over the edge list (dx at dst, dgz at src)
      if (out_nodes > 0) need(row_ptr, "row_ptr");
      if (edges > 0) need(nbr, "nbr");
      const CsrSrc src(row_ptr, out_nodes, edges, stream);
      Args a;
      a.x = node_x; a.y = edge_y; a.w = edge_w; a.gz = g_node_z; a.da = d_gx; a.db = d_gy; a.dc = d_gw;
      a.o0 = o_node_x; a.o1 = o_edge_y; a.o2 = o_edge_w; a.o3 = o_g_node_z;
      conv_atomic(p, dtype, cgf::Comp::DBwd, out_nodes, in_nodes, edges, src.get(), nbr, a, stream);
      return;
    }
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    // Pass 1, by output node: dL/dg_node_z = sum_e op3 + op6 + op7.
    if (out_nodes > 0) {
      need(row_ptr, "row_ptr"); need(o_g_node_z, "o_g_node_z");
      if (!p->z_covered) memzero(o_g_node_z, es * out_nodes * p->problem.dim_z, stream);
      Args a;
      a.x = node_x; a.y = edge_y; a.w = edge_w; a.da = d_gx; a.db = d_gy; a.dc = d_gw;
      a.o3 = o_g_node_z; a.rows = out_nodes; a.rp = row_ptr; a.nb = nbr; a.edges = edges;
      run_kernel(p, cgf::Comp::DBwdZ, cgf::Loop::ConvByOutput, dtype, 0, a, stream);
    }
    // Pass 2, by neighbour node (transposed CSR): dL/dnode_x = sum_e op1.gx + op2.gx,
    // per edge dL/dy = op1.gy + op2.gy and dL/dW = op4.gw + op5.gw.
    if (in_nodes > 0) {
      need(t_row_ptr, "t_row_ptr"); need(o_node_x, "o_node_x");
      if (!p->x_covered) memzero(o_node_x, es * in_nodes * p->problem.dim_x, stream);
      Args b;
      b.x = node_x; b.y = edge_y; b.w = edge_w; b.gz = g_node_z; b.da = d_gx; b.db = d_gy; b.dc = d_gw;
      b.o0 = o_node_x; b.o1 = o_edge_y; b.o2 = o_edge_w; b.rows = in_nodes;
      b.rp = t_row_ptr; b.nb = t_out; b.eid = t_eid; b.edges = edges;
      run_kernel(p, cgf::Comp::DBwdX, cgf::Loop::ConvByInput, dtype, 0, b, stream);
    }
  });
}

int cgf_conv_double_backward(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                             const int32_t* nbr, const int64_t* t_row_ptr, const int32_t* t_out,
                             const int32_t* t_eid, const void* node_x, const void* edge_y, const void* edge_w,
                             const void* g_node_z, const void* d_gx, const void* d_gy, const void* d_gw,
                             void* o_node_x, void* o_edge_y, void* o_edge_w, void* o_g_node_z, int mode,
                             void* stream) {
  if (mode == CGF_CONV_ATOMIC)
    return guarded([&] {
      need(p, "plan");
      const CsrSrc src(row_ptr, nodes, edges, stream);
      if (cgf_conv_double_backward_atomic(p, dtype, nodes, edges, src.get(), nbr, node_x, edge_y, edge_w, g_node_z, d_gx,
                                          d_gy, d_gw, o_node_x, o_edge_y, o_edge_w, o_g_node_z, stream) != CGF_OK)
        throw std::runtime_error(g_err);
    });
  return cgf_conv_double_backward_shard(p, dtype, nodes, nodes, edges, row_ptr, nbr, t_row_ptr, t_out, t_eid,
                                        node_x, edge_y, edge_w, g_node_z, d_gx, d_gy, d_gw, o_node_x, o_edge_y,
                                        o_edge_w, o_g_node_z, mode, stream);
}

// ---- atomic-mode conv over an edge list ----------------------------------

int cgf_conv_forward_atomic(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int32_t* src, const int32_t* dst,
                            const void* node_x, const void* edge_y, const void* edge_w, void* node_z, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (nodes > 0) need(node_z, "node_z");
    if (edges > 0) { need(node_x, "node_x"); need(edge_y, "edge_y"); need(edge_w, "edge_w"); }
    Args a;
    a.x = node_x; a.y = edge_y; a.w = edge_w; a.o0 = node_z;
    conv_atomic(p, dtype, cgf::Comp::Fwd, nodes, nodes, edges, src, dst, a, stream);
  });
}

int cgf_conv_backward_atomic(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                             const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                             const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (nodes > 0) need(g_node_x, "g_node_x");
    if (edges > 0) {
      need(node_x, "node_x"); need(edge_y, "edge_y"); need(edge_w, "edge_w"); need(g_node_z, "g_node_z");
      need(g_edge_y, "g_edge_y"); need(g_edge_w, "g_edge_w");
    }
    Args a;
    a.x = node_x; a.y = edge_y; a.w = edge_w; a.gz = g_node_z;
    a.o0 = g_node_x; a.o1 = g_edge_y; a.o2 = g_edge_w;
    conv_atomic(p, dtype, cgf::Comp::Bwd, nodes, nodes, edges, src, dst, a, stream);
  });
}

int cgf_conv_double_backward_atomic(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                    const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                    const void* g_node_z, const void* d_gx, const void* d_gy, const void* d_gw,
                                    void* o_node_x, void* o_edge_y, void* o_edge_w, void* o_g_node_z, void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (nodes > 0) { need(o_node_x, "o_node_x"); need(o_g_node_z, "o_g_node_z"); }
    if (edges > 0) {
      need(node_x, "node_x"); need(edge_y, "edge_y"); need(edge_w, "edge_w"); need(g_node_z, "g_node_z");
      need(d_gx, "d_gx"); need(d_gy, "d_gy"); need(d_gw, "d_gw"); need(o_edge_y, "o_edge_y"); need(o_edge_w, "o_edge_w");
    }
    Args a;
    a.x = node_x; a.y = edge_y; a.w = edge_w; a.gz = g_node_z; a.da = d_gx; a.db = d_gy; a.dc = d_gw;
    a.o0 = o_node_x; a.o1 = o_edge_y; a.o2 = o_edge_w; a.o3 = o_g_node_z;
    conv_atomic(p, dtype, cgf::Comp::DBwd, nodes, nodes, edges, src, dst, a, stream);
  });
}

// ---- unfused gather -> batched TP -> scatter (conv.cpp:530-616) ---------

int cgf_conv_unfused_forward(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                             const int32_t* nbr, const void* node_x, const void* edge_y, const void* edge_w,
                             void* node_z, void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    need(p, "plan");
    unfused_fwd(p, dtype, nodes, edges, row_ptr, nullptr, nbr, node_x, edge_y, edge_w, node_z, workspace,
                workspace_bytes, stream);
  });
}

int cgf_conv_unfused_backward(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                              const int32_t* nbr, const int64_t* t_row_ptr, const int32_t* t_eid, const void* node_x,
                              const void* edge_y, const void* edge_w, const void* g_node_z, void* g_node_x,
                              void* g_edge_y, void* g_edge_w, void* workspace, size_t workspace_bytes,
                              void* stream) {
  return guarded([&] {
    need(p, "plan");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (nodes == 0) return;
    const std::size_t want = unfused_ws(p->problem, dtype, 1, edges);
    if (workspace && workspace_bytes < want) throw std::invalid_argument("unfused conv: workspace too small");
    Scratch all = workspace ? Scratch(workspace, stream) : Scratch(want, stream);
    // per-edge output node in the workspace's tail
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    const std::size_t E = static_cast<std::size_t>(edges);
    std::int32_t* src = reinterpret_cast<std::int32_t*>(all.as<char>() + 2 * ws_round(es * E * p->problem.dim_x) +
                                                        ws_round(es * E * p->problem.dim_z));
    if (edges > 0) {
      need(row_ptr, "row_ptr");
      cgf::gops::rowptr_expand(row_ptr, nodes, src, stream);
    }
    unfused_bwd(p, dtype, nodes, edges, src, nbr, t_row_ptr, t_eid, node_x, edge_y, edge_w, g_node_z, g_node_x,
                g_edge_y, g_edge_w, all.as<char>(), stream);
  });
}

size_t cgf_conv_unfused_workspace(const cgf_plan* p, int dtype, int op, int64_t edges) {
  return p ? unfused_ws(p->problem, dtype, op, edges) : 0;
}

// ---- graph construction on the device (conv.cpp:64-151) -----------------

int cgf_graph_make(int64_t nodes, int64_t edges, const int32_t* src, const int32_t* dst, int allow_self_loops,
                   int64_t* row_ptr, int32_t* nbr, int32_t* out_src, int64_t* out_edges, void* stream) {
  return guarded([&] {
    need(row_ptr, "row_ptr"); need(out_edges, "out_edges");
    if (edges > 0) { need(src, "src"); need(dst, "dst"); need(nbr, "nbr"); }
    cgf::ensure_context();
    *out_edges = cgf::gops::make_graph(nodes, edges, src, dst, allow_self_loops != 0, row_ptr, nbr, out_src, stream);
  });
}

int cgf_graph_transpose(int64_t out_nodes, int64_t in_nodes, int64_t edges, const int64_t* row_ptr,
                        const int32_t* nbr, int64_t* t_row_ptr, int32_t* t_src, int32_t* t_eid, void* stream) {
  return guarded([&] {
    if (out_nodes < 0 || in_nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    need(t_row_ptr, "t_row_ptr");
    if (edges > 0) { need(row_ptr, "row_ptr"); need(nbr, "nbr"); need(t_src, "t_src"); need(t_eid, "t_eid"); }
    cgf::ensure_context();
    cgf::gops::transpose(out_nodes, in_nodes, edges, row_ptr, nbr, t_row_ptr, t_src, t_eid, stream);
  });
}

int cgf_graph_radius(int64_t n, const double* pos, double r_cut, int64_t* row_ptr, int32_t* nbr, int64_t cap,
                     int64_t* out_edges, void* stream) {
  return guarded([&] {
    need(out_edges, "out_edges");
    if (n > 0) need(pos, "pos");
    cgf::ensure_context();
    *out_edges = cgf::gops::radius_graph(n, pos, r_cut, row_ptr, nbr, cap, stream);
  });
}

// ---- host-pointer conv (the C++ drop-in shim's path) ---------------------
// Copies the graph and arrays in, runs the device entry points on the
// default stream, copies results back. Mode::atomic runs the atomic
// edge-list kernels (cgf_conv_*_atomic_host) over the CSR's expanded sources.
int cgf_conv_forward_host(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                          const int32_t* nbr, const void* node_x, const void* edge_y, const void* edge_w,
                          void* node_z, int mode) {
  return guarded([&] {
    need(p, "plan");
    if (mode != CGF_CONV_DETERMINISTIC && mode != CGF_CONV_ATOMIC) throw std::invalid_argument("bad conv mode");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (nodes == 0) return;
    if (mode == CGF_CONV_ATOMIC) {
      const auto src = csr_sources(nodes, edges, row_ptr);
      if (cgf_conv_forward_atomic_host(p, dtype, nodes, edges, src.data(), nbr, node_x, edge_y, edge_w, node_z) != CGF_OK)
        throw std::runtime_error(g_err);
      return;
    }
    cgf::ensure_context();
    const auto& pr = p->problem;
    const std::size_t V = static_cast<std::size_t>(nodes), E = static_cast<std::size_t>(edges);
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    HostCall hi{1, {}};
    void* drp = hi.in(row_ptr, (V + 1) * 8);
    void* dnb = hi.in(nbr, E * 4);
    void* dx = h.in(node_x, V * pr.dim_x);
    void* dy = h.in(edge_y, E * pr.dim_y);
    void* dw = h.in(edge_w, E * pr.n_w);
    void* dz = h.out(V * pr.dim_z);
    const int rc = cgf_conv_forward(p, dtype, nodes, edges, static_cast<const int64_t*>(drp),
                                    static_cast<const int32_t*>(dnb), dx, dy, dw, dz, CGF_CONV_DETERMINISTIC, nullptr);
    if (rc != CGF_OK) throw std::runtime_error(g_err);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(node_z, dz, V * pr.dim_z);
  });
}

int cgf_conv_backward_host(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                           const int32_t* nbr, const void* node_x, const void* edge_y, const void* edge_w,
                           const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w, int mode) {
  return guarded([&] {
    need(p, "plan");
    if (mode != CGF_CONV_DETERMINISTIC && mode != CGF_CONV_ATOMIC) throw std::invalid_argument("bad conv mode");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (nodes == 0) return;
    if (mode == CGF_CONV_ATOMIC) {
      const auto src = csr_sources(nodes, edges, row_ptr);
      if (cgf_conv_backward_atomic_host(p, dtype, nodes, edges, src.data(), nbr, node_x, edge_y, edge_w, g_node_z,
                                        g_node_x, g_edge_y, g_edge_w) != CGF_OK)
        throw std::runtime_error(g_err);
      return;
    }
    cgf::ensure_context();
    const auto& pr = p->problem;
    const std::size_t V = static_cast<std::size_t>(nodes), E = static_cast<std::size_t>(edges);
    std::vector<int64_t> trp(V + 1);
    std::vector<int32_t> tsrc(std::max<std::size_t>(E, 1)), teid(std::max<std::size_t>(E, 1));
    int rc = cgf_conv_transpose_host(nodes, edges, row_ptr, nbr, trp.data(), tsrc.data(), teid.data());
    if (rc != CGF_OK) throw std::invalid_argument(g_err);
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    HostCall hi{1, {}};
    void* dtrp = hi.in(trp.data(), (V + 1) * 8);
    void* dts = hi.in(tsrc.data(), E * 4);
    void* dte = hi.in(teid.data(), E * 4);
    void* dx = h.in(node_x, V * pr.dim_x);
    void* dy = h.in(edge_y, E * pr.dim_y);
    void* dw = h.in(edge_w, E * pr.n_w);
    void* dgz = h.in(g_node_z, V * pr.dim_z);
    void* ogx = h.out(V * pr.dim_x);
    void* ogy = h.out(E * pr.dim_y);
    void* ogw = h.out(E * pr.n_w);
    rc = cgf_conv_backward(p, dtype, nodes, edges, nullptr, nullptr, static_cast<const int64_t*>(dtrp),
                           static_cast<const int32_t*>(dts), static_cast<const int32_t*>(dte), dx, dy, dw, dgz, ogx,
                           ogy, ogw, CGF_CONV_DETERMINISTIC, nullptr);
    if (rc != CGF_OK) throw std::runtime_error(g_err);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(g_node_x, ogx, V * pr.dim_x);
    h.back(g_edge_y, ogy, E * pr.dim_y);
    h.back(g_edge_w, ogw, E * pr.n_w);
  });
}

int cgf_conv_forward_atomic_host(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                 const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                 void* node_z) {
  return guarded([&] {
    need(p, "plan");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (nodes == 0) return;
    check_edge_list(nodes, edges, src, dst);
    cgf::ensure_context();
    const auto& pr = p->problem;
    const std::size_t V = static_cast<std::size_t>(nodes), E = static_cast<std::size_t>(edges);
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    HostCall hi{1, {}};
    void* ds = hi.in(src, E * 4);
    void* dd = hi.in(dst, E * 4);
    void* dx = h.in(node_x, V * pr.dim_x);
    void* dy = h.in(edge_y, E * pr.dim_y);
    void* dw = h.in(edge_w, E * pr.n_w);
    void* dz = h.out(V * pr.dim_z);
    if (cgf_conv_forward_atomic(p, dtype, nodes, edges, static_cast<const int32_t*>(ds), static_cast<const int32_t*>(dd),
                                dx, dy, dw, dz, nullptr) != CGF_OK)
      throw std::runtime_error(g_err);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(node_z, dz, V * pr.dim_z);
  });
}

int cgf_conv_backward_atomic_host(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                  const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                  const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w) {
  return guarded([&] {
    need(p, "plan");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (nodes == 0) return;
    check_edge_list(nodes, edges, src, dst);
    cgf::ensure_context();
    const auto& pr = p->problem;
    const std::size_t V = static_cast<std::size_t>(nodes), E = static_cast<std::size_t>(edges);
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    HostCall hi{1, {}};
    void* ds = hi.in(src, E * 4);
    void* dd = hi.in(dst, E * 4);
    void* dx = h.in(node_x, V * pr.dim_x);
    void* dy = h.in(edge_y, E * pr.dim_y);
    void* dw = h.in(edge_w, E * pr.n_w);
    void* dgz = h.in(g_node_z, V * pr.dim_z);
    void* ogx = h.out(V * pr.dim_x);
    void* ogy = h.out(E * pr.dim_y);
    void* ogw = h.out(E * pr.n_w);
    if (cgf_conv_backward_atomic(p, dtype, nodes, edges, static_cast<const int32_t*>(ds),
                                 static_cast<const int32_t*>(dd), dx, dy, dw, dgz, ogx, ogy, ogw, nullptr) != CGF_OK)
      throw std::runtime_error(g_err);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(g_node_x, ogx, V * pr.dim_x);
    h.back(g_edge_y, ogy, E * pr.dim_y);
    h.back(g_edge_w, ogw, E * pr.n_w);
  });
}

int cgf_conv_unfused_forward_host(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                  const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                  void* node_z) {
  return guarded([&] {
    need(p, "plan");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (nodes == 0) return;
    check_edge_list(nodes, edges, src, dst);
    cgf::ensure_context();
    const auto& pr = p->problem;
    const std::size_t V = static_cast<std::size_t>(nodes), E = static_cast<std::size_t>(edges);
    std::vector<std::int64_t> rp;
    std::vector<std::int32_t> ridx;
    host_bucket(nodes, edges, src, rp, ridx);
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    HostCall hi{1, {}};
    void* drp = hi.in(rp.data(), (V + 1) * 8);
    void* dri = hi.in(ridx.data(), E * 4);
    void* dd = hi.in(dst, E * 4);
    void* dx = h.in(node_x, V * pr.dim_x);
    void* dy = h.in(edge_y, E * pr.dim_y);
    void* dw = h.in(edge_w, E * pr.n_w);
    void* dz = h.out(V * pr.dim_z);
    unfused_fwd(p, dtype, nodes, edges, static_cast<const std::int64_t*>(drp), static_cast<const std::int32_t*>(dri),
                static_cast<const std::int32_t*>(dd), dx, dy, dw, dz, nullptr, 0, nullptr);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(node_z, dz, V * pr.dim_z);
  });
}

int cgf_conv_unfused_backward_host(cgf_plan* p, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                   const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                   const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w) {
  return guarded([&] {
    need(p, "plan");
    if (nodes < 0 || edges < 0) throw cgf::ShapeError("negative graph size");
    if (nodes == 0) return;
    check_edge_list(nodes, edges, src, dst);
    cgf::ensure_context();
    const auto& pr = p->problem;
    const std::size_t V = static_cast<std::size_t>(nodes), E = static_cast<std::size_t>(edges);
    std::vector<std::int64_t> trp;
    std::vector<std::int32_t> tidx;
    host_bucket(nodes, edges, dst, trp, tidx);
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    HostCall hi{1, {}};
    void* ds = hi.in(src, E * 4);
    void* dd = hi.in(dst, E * 4);
    void* dtrp = hi.in(trp.data(), (V + 1) * 8);
    void* dti = hi.in(tidx.data(), E * 4);
    void* dx = h.in(node_x, V * pr.dim_x);
    void* dy = h.in(edge_y, E * pr.dim_y);
    void* dw = h.in(edge_w, E * pr.n_w);
    void* dgz = h.in(g_node_z, V * pr.dim_z);
    void* ogx = h.out(V * pr.dim_x);
    void* ogy = h.out(E * pr.dim_y);
    void* ogw = h.out(E * pr.n_w);
    Scratch ws(unfused_ws(pr, dtype, 1, edges), nullptr);
    unfused_bwd(p, dtype, nodes, edges, static_cast<const std::int32_t*>(ds), static_cast<const std::int32_t*>(dd),
                static_cast<const std::int64_t*>(dtrp), static_cast<const std::int32_t*>(dti), dx, dy, dw, dgz, ogx,
                ogy, ogw, ws.as<char>(), nullptr);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(g_node_x, ogx, V * pr.dim_x);
    h.back(g_edge_y, ogy, E * pr.dim_y);
    h.back(g_edge_w, ogw, E * pr.n_w);
  });
}

}  // extern "C"
