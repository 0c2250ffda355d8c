// extern "C" boundary (include/cgf.h) over the problem planner, the code
// generator and the JIT. Exceptions never cross the boundary: each maps to a
// status code plus a thread-local message.
#include "../../include/cgf.h"

#include <cuda.h>
#include <nvrtc.h>

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

struct cgf_plan {
  cgf::Problem problem;
  std::vector<cgf::Unit> units;
  std::uint32_t budget = 4096;
  bool z_covered = true, x_covered = true;
  std::mutex mu;
  std::map<std::tuple<int, int, int, int>, std::shared_ptr<cgf::KernelSource>> sources;
};

namespace {

thread_local std::string g_err;

struct BudgetError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

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

std::shared_ptr<cgf::KernelSource> source_for(cgf_plan* p, int op, int dtype, int w_shared, int aligned) {
  if (op < 0 || op > 2) throw std::invalid_argument("bad op");
  if (dtype != CGF_F32 && dtype != CGF_F64) throw std::invalid_argument("bad dtype");
  std::lock_guard<std::mutex> g(p->mu);
  const auto key = std::make_tuple(op, dtype, w_shared ? 1 : 0, aligned ? 1 : 0);
  auto it = p->sources.find(key);
  if (it != p->sources.end()) return it->second;
  if (w_shared && op != CGF_OP_FORWARD)
    throw cgf::UnsupportedError("shared-weight backward / double-backward needs the uvw tensor-core path");
  cgf::KernelConfig cfg;
  cfg.op = static_cast<cgf::Op>(op);
  cfg.f64 = dtype == CGF_F64;
  cfg.w_shared = w_shared != 0;
  cfg.aligned = aligned != 0;
  auto ks = std::make_shared<cgf::KernelSource>(cgf::generate_tp_kernel(p->problem, p->units, cfg));
  p->sources.emplace(key, ks);
  return ks;
}

bool aligned16(std::initializer_list<const void*> ptrs) {
  for (const void* q : ptrs)
    if (q && (reinterpret_cast<std::uintptr_t>(q) & 15u)) return false;
  return true;
}

void launch(cgf_plan* p, int op, int dtype, int w_shared, std::int64_t rows, const void* x,
            const void* y, const void* w, const void* gz, const void* da, const void* db,
            const void* dc, void* o0, void* o1, void* o2, void* o3, void* stream) {
  if (rows < 0) throw cgf::ShapeError("rows must be non-negative");
  if (rows == 0) return;
  const bool al = aligned16({x, y, w, gz, da, db, dc, o0, o1, o2, o3});
  const auto ks = source_for(p, op, dtype, w_shared, al);
  const cgf::Kernel k = cgf::load_kernel(*ks);
  CUstream s = reinterpret_cast<CUstream>(stream);
  const std::size_t es = dtype == CGF_F64 ? 8 : 4;
  const auto& pr = p->problem;
  // Outputs the kernel never touches must still read as zero.
  if (op != CGF_OP_BACKWARD && !p->z_covered) {
    void* zo = op == CGF_OP_FORWARD ? o0 : o3;
    CU_CHECK(cgf::drv::cuMemsetD8Async(reinterpret_cast<CUdeviceptr>(zo), 0, es * rows * pr.dim_z, s));
  }
  if (op != CGF_OP_FORWARD && !p->x_covered)
    CU_CHECK(cgf::drv::cuMemsetD8Async(reinterpret_cast<CUdeviceptr>(o0), 0, es * rows * pr.dim_x, s));
  const int warps = k.threads / 32;
  const std::int64_t need = (rows + warps - 1) / warps;
  const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(need, k.max_grid));
  void* args[] = {&x, &y, &w, &gz, &da, &db, &dc, &o0, &o1, &o2, &o3, &rows};
  CU_CHECK(cgf::drv::cuLaunchKernel(k.fn, grid, 1, 1, k.threads, 1, 1, k.smem_bytes, s, args, nullptr));
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

}  // namespace

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
    // The reference's admission check: every subkernel's working set
    // (x + y + w + z words) must fit the per-worker budget (scheduler.cpp:161-170).
    for (const auto& s : p->problem.subs) {
      const std::uint32_t ws = s.bp * s.dx() + s.dy() + (s.kind == cgf::Kind::B ? s.b : s.b * s.bp) + s.b * s.dz();
      if (ws > p->budget)
        throw BudgetError("budget " + std::to_string(p->budget) + " words below working set " + std::to_string(ws) +
                          " of subkernel (l=(" + std::to_string(s.l1) + "," + std::to_string(s.l2) + "," +
                          std::to_string(s.l3) + "), b=" + std::to_string(s.b) + ", b'=" + std::to_string(s.bp) + ")");
    }
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
    const auto ks = source_for(p, op, dtype, w_shared, aligned);
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
    const auto ks = source_for(p, op, dtype, w_shared, aligned);
    cgf::compile_cubin(ks->source, ks->name);
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

int cgf_tp_forward_host(cgf_plan* p, int dtype, const void* x, const void* y, const void* w, void* z,
                        int64_t rows, int w_shared) {
  return guarded([&] {
    need(p, "plan");
    if (rows <= 0) return;
    cgf::ensure_context();
    const auto& pr = p->problem;
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    const std::size_t R = static_cast<std::size_t>(rows);
    void* dx = h.in(x, R * pr.dim_x);
    void* dy = h.in(y, R * pr.dim_y);
    void* dw = h.in(w, (w_shared ? 1 : R) * pr.n_w);
    void* dz = h.out(R * pr.dim_z);
    launch(p, CGF_OP_FORWARD, dtype, w_shared, rows, dx, dy, dw, nullptr, nullptr, nullptr, nullptr, dz,
           nullptr, nullptr, nullptr, nullptr);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(z, dz, R * pr.dim_z);
  });
}

int cgf_tp_backward_host(cgf_plan* p, int dtype, const void* x, const void* y, const void* w,
                         const void* gz, void* gx, void* gy, void* gw, int64_t rows, int w_shared) {
  return guarded([&] {
    need(p, "plan");
    if (rows <= 0) return;
    cgf::ensure_context();
    const auto& pr = p->problem;
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    const std::size_t R = static_cast<std::size_t>(rows), RW = w_shared ? 1 : R;
    void* dx = h.in(x, R * pr.dim_x);
    void* dy = h.in(y, R * pr.dim_y);
    void* dw = h.in(w, RW * pr.n_w);
    void* dg = h.in(gz, R * pr.dim_z);
    void* ox = h.out(R * pr.dim_x);
    void* oy = h.out(R * pr.dim_y);
    void* ow = h.out(RW * pr.n_w);
    launch(p, CGF_OP_BACKWARD, dtype, w_shared, rows, dx, dy, dw, dg, nullptr, nullptr, nullptr, ox, oy, ow,
           nullptr, nullptr);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(gx, ox, R * pr.dim_x);
    h.back(gy, oy, R * pr.dim_y);
    h.back(gw, ow, RW * pr.n_w);
  });
}

int cgf_tp_double_backward_host(cgf_plan* p, int dtype, const void* x, const void* y, const void* w,
                                const void* gz, const void* da, const void* db, const void* dc,
                                void* ox, void* oy, void* ow, void* ogz, int64_t rows, int w_shared) {
  return guarded([&] {
    need(p, "plan");
    if (rows <= 0) return;
    cgf::ensure_context();
    const auto& pr = p->problem;
    HostCall h{dtype == CGF_F64 ? 8u : 4u, {}};
    const std::size_t R = static_cast<std::size_t>(rows), RW = w_shared ? 1 : R;
    void* dx = h.in(x, R * pr.dim_x);
    void* dy = h.in(y, R * pr.dim_y);
    void* dw = h.in(w, RW * pr.n_w);
    void* dg = h.in(gz, R * pr.dim_z);
    void* a = h.in(da, R * pr.dim_x);
    void* b = h.in(db, R * pr.dim_y);
    void* c = h.in(dc, RW * pr.n_w);
    void* o0 = h.out(R * pr.dim_x);
    void* o1 = h.out(R * pr.dim_y);
    void* o2 = h.out(RW * pr.n_w);
    void* o3 = h.out(R * pr.dim_z);
    launch(p, CGF_OP_DOUBLE_BACKWARD, dtype, w_shared, rows, dx, dy, dw, dg, a, b, c, o0, o1, o2, o3, nullptr);
    CU_CHECK(cgf::drv::cuCtxSynchronize());
    h.back(ox, o0, R * pr.dim_x);
    h.back(oy, o1, R * pr.dim_y);
    h.back(ow, o2, RW * pr.n_w);
    h.back(ogz, o3, R * pr.dim_z);
  });
}

int cgf_tp_stats(const cgf_plan* p, int op, int64_t rows, int w_shared, uint64_t stats[3]) {
  return guarded([&] {
    need(p, "plan");
    const auto& pr = p->problem;
    const std::uint64_t R = static_cast<std::uint64_t>(rows);
    const std::uint64_t W = w_shared ? pr.n_w : R * pr.n_w;
    const std::uint64_t X = R * pr.dim_x, Y = R * pr.dim_y, Z = R * pr.dim_z;
    const std::uint64_t f = pr.fwd_flops_per_row(), b = pr.bwd_flops_per_row();
    switch (op) {
      case CGF_OP_FORWARD: stats[0] = X + Y + W; stats[1] = Z; stats[2] = R * f; break;
      case CGF_OP_BACKWARD: stats[0] = X + Y + W + Z; stats[1] = X + Y + W; stats[2] = R * b; break;
      case CGF_OP_DOUBLE_BACKWARD:
        stats[0] = 2 * (X + Y + W) + Z + X + Y + W;
        stats[1] = X + Y + W + Z;
        stats[2] = R * (3 * f + 4 * b);
        break;
      default: throw std::invalid_argument("bad op");
    }
  });
}

}  // extern "C"
