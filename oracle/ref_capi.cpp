// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrapper around the UNMODIFIED reference library (cgforge, built
// out-of-tree from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libcgforge_ref.so). It lets the Python tests, the golden-fixture
// script and bench.py's cpu_baseline / --impl reference arm drive the
// reference's own public C++ API (tpspec::parse_problem_json ->
// scheduler::split_multiplicities -> build_schedule -> engine::TpPlan,
// conv::ConvPlan) on flat host arrays.
//
// Every entry point copies caller arrays into the reference's std::vector
// containers, calls the reference, and copies results back; the timing entry
// points (cgr_bench_*) time only the reference call itself, with the CLI's
// methodology (median of `iters` after `warmup`, tools/cgforge.cpp:336-348).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cgforge/cg.hpp"
#include "cgforge/conv.hpp"
#include "cgforge/array_io.hpp"
#include "cgforge/engine.hpp"
#include "cgforge/kernelgen.hpp"
#include "cgforge/rng.hpp"
#include "cgforge/scheduler.hpp"
#include "cgforge/tpspec.hpp"

using namespace cgforge;

namespace {

thread_local std::string g_err;

struct RefPlan {
  tpspec::ValidatedProblem split;
  scheduler::Schedule sched;
  std::unique_ptr<engine::TpPlan> plan;
};

template <typename T>
std::vector<T> vec(const T* p, std::size_t n) {
  return std::vector<T>(p, p + n);
}

template <typename T>
void out(const std::vector<T>& v, T* p) {
  std::memcpy(p, v.data(), sizeof(T) * v.size());
}

engine::Options opts(int workers, int interpreted) {
  engine::Options o;
  o.workers = workers > 0 ? workers : static_cast<int>(std::thread::hardware_concurrency());
  o.mode = interpreted ? engine::ExecMode::interpreted : engine::ExecMode::specialized;
  return o;
}

void put_stats(const engine::ExecStats& st, std::uint64_t* stats) {
  if (!stats) return;
  stats[0] = st.loads_words;
  stats[1] = st.stores_words;
  stats[2] = st.flops;
}

template <typename T>
int tp_forward(void* h, std::int64_t rows, const T* x, const T* y, const T* w, T* z, int workers,
               int interpreted, std::uint64_t* stats) {
  try {
    auto* rp = static_cast<RefPlan*>(h);
    const auto& p = rp->split;
    engine::Batch<T> b;
    b.rows = rows;
    b.x = vec(x, static_cast<std::size_t>(rows) * p.dim_x);
    b.y = vec(y, static_cast<std::size_t>(rows) * p.dim_y);
    b.w = vec(w, static_cast<std::size_t>(rows) * p.total_weights);
    std::vector<T> zz;
    put_stats(rp->plan->forward(b, zz, opts(workers, interpreted)), stats);
    out(zz, z);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename T>
int tp_backward(void* h, std::int64_t rows, const T* x, const T* y, const T* w, const T* gz,
                T* gx, T* gy, T* gw, int workers, int interpreted, std::uint64_t* stats) {
  try {
    auto* rp = static_cast<RefPlan*>(h);
    const auto& p = rp->split;
    engine::Batch<T> b;
    b.rows = rows;
    b.x = vec(x, static_cast<std::size_t>(rows) * p.dim_x);
    b.y = vec(y, static_cast<std::size_t>(rows) * p.dim_y);
    b.w = vec(w, static_cast<std::size_t>(rows) * p.total_weights);
    engine::Grads<T> g;
    put_stats(rp->plan->backward(b, vec(gz, static_cast<std::size_t>(rows) * p.dim_z), g,
                                 opts(workers, interpreted)),
              stats);
    out(g.x, gx);
    out(g.y, gy);
    out(g.w, gw);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename T>
int tp_double_backward(void* h, std::int64_t rows, const T* x, const T* y, const T* w,
                       const T* gz, const T* da, const T* db, const T* dc, T* ox, T* oy, T* ow,
                       T* ogz, int seven_call, int workers, std::uint64_t* stats) {
  try {
    auto* rp = static_cast<RefPlan*>(h);
    const auto& p = rp->split;
    const auto nx = static_cast<std::size_t>(rows) * p.dim_x;
    const auto ny = static_cast<std::size_t>(rows) * p.dim_y;
    const auto nw = static_cast<std::size_t>(rows) * p.total_weights;
    const auto nz = static_cast<std::size_t>(rows) * p.dim_z;
    engine::Batch<T> b;
    b.rows = rows;
    b.x = vec(x, nx);
    b.y = vec(y, ny);
    b.w = vec(w, nw);
    engine::Grads<T> up;
    up.x = vec(da, nx);
    up.y = vec(db, ny);
    up.w = vec(dc, nw);
    engine::DoubleGrads<T> o;
    put_stats(rp->plan->double_backward(
                  b, vec(gz, nz), up, o,
                  seven_call ? engine::DispatchStyle::seven_call : engine::DispatchStyle::fused,
                  opts(workers, 0)),
              stats);
    out(o.x, ox);
    out(o.y, oy);
    out(o.w, ow);
    out(o.gz, ogz);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

conv::GraphCSR make_csr(std::int64_t nodes, std::int64_t ne, const std::int32_t* src,
                        const std::int32_t* dst) {
  std::vector<conv::Edge> edges(static_cast<std::size_t>(ne));
  for (std::int64_t e = 0; e < ne; ++e) edges[e] = {src[e], dst[e]};
  return conv::make_graph(nodes, std::move(edges));
}

void put_cstats(const conv::ConvStats& st, std::uint64_t* stats) {
  if (!stats) return;
  stats[0] = st.loads_words;
  stats[1] = st.stores_words;
  stats[2] = st.output_store_ops;
  stats[3] = st.flops;
}

template <typename T>
int conv_forward(void* h, std::int64_t nodes, std::int64_t ne, const std::int32_t* src,
                 const std::int32_t* dst, const T* node_x, const T* edge_y, const T* edge_w,
                 T* node_z, int atomic, int workers, int chunks, int unfused,
                 std::uint64_t* stats) {
  try {
    auto* rp = static_cast<RefPlan*>(h);
    const auto& p = rp->split;
    const auto g = make_csr(nodes, ne, src, dst);
    if (g.edge_count() != ne) throw std::invalid_argument("edge list not strictly sorted/unique");
    std::vector<T> nz;
    const auto nx = vec(node_x, static_cast<std::size_t>(nodes) * p.dim_x);
    const auto ey = vec(edge_y, static_cast<std::size_t>(ne) * p.dim_y);
    const auto ew = vec(edge_w, static_cast<std::size_t>(ne) * p.total_weights);
    if (unfused) {
      put_cstats(conv::unfused_forward(*rp->plan, g, nx, ey, ew, nz, opts(workers, 0)), stats);
    } else {
      conv::ConvOptions co;
      co.workers = opts(workers, 0).workers;
      co.chunks = chunks > 0 ? chunks : 16;
      const conv::ConvPlan cp(*rp->plan);
      put_cstats(cp.forward(g, nx, ey, ew, nz,
                            atomic ? conv::Mode::atomic : conv::Mode::deterministic, co),
                 stats);
    }
    out(nz, node_z);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename T>
int conv_backward(void* h, std::int64_t nodes, std::int64_t ne, const std::int32_t* src,
                  const std::int32_t* dst, const T* node_x, const T* edge_y, const T* edge_w,
                  const T* g_node_z, T* g_node_x, T* g_edge_y, T* g_edge_w, int atomic,
                  int workers, int chunks, int unfused, std::uint64_t* stats) {
  try {
    auto* rp = static_cast<RefPlan*>(h);
    const auto& p = rp->split;
    const auto g = make_csr(nodes, ne, src, dst);
    if (g.edge_count() != ne) throw std::invalid_argument("edge list not strictly sorted/unique");
    const auto perm = conv::transpose_permutation(g);
    const auto nx = vec(node_x, static_cast<std::size_t>(nodes) * p.dim_x);
    const auto ey = vec(edge_y, static_cast<std::size_t>(ne) * p.dim_y);
    const auto ew = vec(edge_w, static_cast<std::size_t>(ne) * p.total_weights);
    const auto gnz = vec(g_node_z, static_cast<std::size_t>(nodes) * p.dim_z);
    std::vector<T> gx, gy, gw;
    if (unfused) {
      put_cstats(conv::unfused_backward(*rp->plan, g, nx, ey, ew, gnz, gx, gy, gw,
                                        opts(workers, 0)),
                 stats);
    } else {
      conv::ConvOptions co;
      co.workers = opts(workers, 0).workers;
      co.chunks = chunks > 0 ? chunks : 16;
      const conv::ConvPlan cp(*rp->plan);
      put_cstats(cp.backward(g, perm, nx, ey, ew, gnz, gx, gy, gw,
                             atomic ? conv::Mode::atomic : conv::Mode::deterministic, co),
                 stats);
    }
    out(gx, g_node_x);
    out(gy, g_edge_y);
    out(gw, g_edge_w);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename F>
double median_s(int warmup, int iters, F&& body) {
  for (int i = 0; i < warmup; ++i) body();
  std::vector<double> t;
  for (int i = 0; i < std::max(iters, 1); ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    body();
    const auto t1 = std::chrono::steady_clock::now();
    t.push_back(std::chrono::duration<double>(t1 - t0).count());
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

// op bit mask: 1 forward, 2 backward, 4 double_backward. Inputs are the
// reference's own random_batch / NormalGen draws (cgforge.cpp:357-386).
template <typename T>
int bench_tp(void* h, std::int64_t rows, int ops, int warmup, int iters, int workers,
             std::uint64_t seed, double* secs) {
  try {
    auto* rp = static_cast<RefPlan*>(h);
    const auto& p = rp->split;
    const auto in = engine::random_batch<T>(p, rows, seed);
    const auto o = opts(workers, 0);
    std::vector<T> z;
    rp->plan->forward(in, z, o);
    secs[0] = secs[1] = secs[2] = 0.0;
    if (ops & 1) secs[0] = median_s(warmup, iters, [&] { rp->plan->forward(in, z, o); });
    const std::vector<T> gz = rng::NormalGen(seed + 1).normal_vec<T>(z.size());
    if (ops & 2) {
      engine::Grads<T> g;
      secs[1] = median_s(warmup, iters, [&] { rp->plan->backward(in, gz, g, o); });
    }
    if (ops & 4) {
      engine::Grads<T> up;
      up.x = rng::NormalGen(seed + 2).normal_vec<T>(in.x.size());
      up.y = rng::NormalGen(seed + 3).normal_vec<T>(in.y.size());
      up.w = rng::NormalGen(seed + 4).normal_vec<T>(in.w.size());
      engine::DoubleGrads<T> dg;
      secs[2] = median_s(warmup, iters, [&] {
        rp->plan->double_backward(in, gz, up, dg, engine::DispatchStyle::fused, o);
      });
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

template <typename T>
int bench_conv(void* h, int lattice_n, double r_cut, int ops, int warmup, int iters, int workers,
               std::uint64_t seed, double* secs, std::int64_t* edges) {
  try {
    auto* rp = static_cast<RefPlan*>(h);
    const auto& p = rp->split;
    const auto g = conv::radius_graph(conv::cubic_lattice(lattice_n, lattice_n, lattice_n, 1.0),
                                      r_cut);
    *edges = g.edge_count();
    const auto nv = static_cast<std::size_t>(g.node_count), ne = static_cast<std::size_t>(*edges);
    rng::NormalGen gen(seed);
    const auto node_x = gen.normal_vec<T>(nv * p.dim_x);
    const auto edge_y = gen.normal_vec<T>(ne * p.dim_y);
    const auto edge_w = gen.normal_vec<T>(ne * p.total_weights);
    const conv::ConvPlan cp(*rp->plan);
    conv::ConvOptions co;
    co.workers = opts(workers, 0).workers;
    std::vector<T> node_z;
    secs[0] = secs[1] = 0.0;
    cp.forward(g, node_x, edge_y, edge_w, node_z, conv::Mode::deterministic, co);
    if (ops & 1)
      secs[0] = median_s(warmup, iters, [&] {
        cp.forward(g, node_x, edge_y, edge_w, node_z, conv::Mode::deterministic, co);
      });
    if (ops & 2) {
      const auto perm = conv::transpose_permutation(g);
      const auto gnz = rng::NormalGen(seed + 1).normal_vec<T>(node_z.size());
      std::vector<T> gx, gy, gw;
      secs[1] = median_s(warmup, iters, [&] {
        cp.backward(g, perm, node_x, edge_y, edge_w, gnz, gx, gy, gw, conv::Mode::deterministic,
                    co);
      });
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* cgr_last_error() { return g_err.c_str(); }

// Parses + validates (tpspec.cpp:105-130), splits (scheduler.cpp:32-81),
// schedules (scheduler.cpp:139-389) and compiles a TpPlan (engine.cpp:92).
void* cgr_plan_create(const char* problem_json, std::uint32_t budget, int lane_width) {
  try {
    auto vr = tpspec::parse_problem_json(problem_json);
    if (!vr.ok()) {
      g_err.clear();
      for (const auto& v : vr.violations) {
        g_err += "instruction " + std::to_string(v.instruction_index) + ": " + v.message + "; ";
      }
      return nullptr;
    }
    auto rp = std::make_unique<RefPlan>();
    rp->split = scheduler::split_multiplicities(*vr.problem, lane_width > 0 ? lane_width : 32);
    rp->sched = scheduler::build_schedule(rp->split, budget);
    rp->plan = std::make_unique<engine::TpPlan>(rp->split, rp->sched);
    return rp.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void cgr_plan_destroy(void* h) { delete static_cast<RefPlan*>(h); }

// dims[0..3] = dim_x, dim_y, dim_z, total_weights; dims[4] = split count;
// dims[5] = phases; dims[6] = strategy; traffic[0..2] = loads, stores, flops
// per row (scheduler.cpp:391-404).
void cgr_plan_info(void* h, std::int64_t* dims, std::uint64_t* traffic) {
  auto* rp = static_cast<RefPlan*>(h);
  dims[0] = rp->split.dim_x;
  dims[1] = rp->split.dim_y;
  dims[2] = rp->split.dim_z;
  dims[3] = rp->split.total_weights;
  dims[4] = static_cast<std::int64_t>(rp->split.resolved.size());
  dims[5] = static_cast<std::int64_t>(rp->sched.phases.size());
  dims[6] = static_cast<std::int64_t>(rp->sched.strategy);
  traffic[0] = rp->sched.traffic.loads_words;
  traffic[1] = rp->sched.traffic.stores_words;
  traffic[2] = rp->sched.traffic.flops;
}

// Per split subkernel (schedule order): kind, l1, l2, l3, b, b', x_off,
// y_off, z_off, w_off, w_row_stride, fwd flops, bwd flops. 13 ints each.
int cgr_plan_split(void* h, std::int64_t* rows, int cap) {
  auto* rp = static_cast<RefPlan*>(h);
  const auto& s = rp->split;
  const int n = static_cast<int>(s.resolved.size());
  for (int pos = 0; pos < n && pos < cap; ++pos) {
    const auto& r = s.resolved[rp->sched.order[pos]];
    std::int64_t* o = rows + 13 * pos;
    o[0] = r.kind == tpspec::Kind::B ? 0 : 1;
    o[1] = r.l1;
    o[2] = r.l2;
    o[3] = r.l3;
    o[4] = r.b;
    o[5] = r.b_prime;
    o[6] = r.x_offset;
    o[7] = r.y_offset;
    o[8] = r.z_offset;
    o[9] = r.weight_offset;
    o[10] = r.w_row_stride;
    o[11] = static_cast<std::int64_t>(kernelgen::flop_count(kernelgen::gen_forward(r)));
    o[12] = static_cast<std::int64_t>(kernelgen::flop_count(kernelgen::gen_backward(r)));
  }
  return n;
}

// Listing text of gen_forward/gen_backward (kernelgen.cpp:305-360) for
// split subkernel `pos`; returns the length written (truncated to cap).
int cgr_emit_text(void* h, int pos, int backward, char* buf, int cap) {
  auto* rp = static_cast<RefPlan*>(h);
  const auto& r = rp->split.resolved.at(rp->sched.order.at(pos));
  const std::string t =
      kernelgen::emit_text(backward ? kernelgen::gen_backward(r) : kernelgen::gen_forward(r));
  const int n = std::min<int>(cap - 1, static_cast<int>(t.size()));
  std::memcpy(buf, t.data(), n);
  buf[n] = 0;
  return static_cast<int>(t.size());
}

// array_io::save_array (array_io.cpp:15-38), for byte comparisons.
int cgr_save_array(const char* base, const void* data, std::int64_t rows, std::int64_t cols, int f64) {
  try {
    if (f64) array_io::save_array(base, static_cast<const double*>(data), rows, cols);
    else array_io::save_array(base, static_cast<const float*>(data), rows, cols);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// scheduler::schedule_to_json of the plan's schedule (scheduler.cpp:406-445).
int cgr_schedule_json(void* h, char* buf, int cap) {
  auto* rp = static_cast<RefPlan*>(h);
  const std::string t = scheduler::schedule_to_json(rp->split, rp->sched);
  const int n = std::min<int>(cap - 1, static_cast<int>(t.size()));
  std::memcpy(buf, t.data(), n);
  buf[n] = 0;
  return static_cast<int>(t.size());
}

int cgr_cg_block(int l1, int l2, int l3, int cap, int* i, int* j, int* k, double* v) {
  try {
    const auto b = cg::cg_block(l1, l2, l3);
    const int n = static_cast<int>(b->entries.size());
    for (int e = 0; e < n && e < cap; ++e) {
      i[e] = b->entries[e].i;
      j[e] = b->entries[e].j;
      k[e] = b->entries[e].k;
      v[e] = b->entries[e].v;
    }
    return n;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// rng::NormalGen(seed) stream (rng.hpp:14-53), continuing across calls via a
// handle so multi-array draws keep the reference's order.
void* cgr_rng_new(std::uint64_t seed) { return new rng::NormalGen(seed); }
void cgr_rng_free(void* g) { delete static_cast<rng::NormalGen*>(g); }
void cgr_rng_normal(void* g, double* o, std::int64_t n) {
  auto* gen = static_cast<rng::NormalGen*>(g);
  for (std::int64_t e = 0; e < n; ++e) o[e] = gen->normal();
}

// radius_graph(cubic_lattice(n,n,n,spacing), r_cut) (conv.cpp:89-164).
// Returns the edge count; fills src/dst when cap allows.
std::int64_t cgr_lattice_graph(int n, double spacing, double r_cut, std::int32_t* src,
                               std::int32_t* dst, std::int64_t cap) {
  const auto g = conv::radius_graph(conv::cubic_lattice(n, n, n, spacing), r_cut);
  for (std::int64_t e = 0; e < g.edge_count() && e < cap; ++e) {
    src[e] = g.edges[e].src;
    dst[e] = g.edges[e].dst;
  }
  return g.edge_count();
}

void cgr_transpose_permutation(std::int64_t nodes, std::int64_t ne, const std::int32_t* src,
                               const std::int32_t* dst, std::int64_t* perm) {
  const auto g = make_csr(nodes, ne, src, dst);
  const auto p = conv::transpose_permutation(g);
  std::memcpy(perm, p.data(), sizeof(std::int64_t) * p.size());
}

#define CGR_TYPED(SUF, T)                                                                     \
  int cgr_tp_forward_##SUF(void* h, std::int64_t rows, const T* x, const T* y, const T* w,   \
                           T* z, int workers, int interp, std::uint64_t* st) {               \
    return tp_forward<T>(h, rows, x, y, w, z, workers, interp, st);                          \
  }                                                                                           \
  int cgr_tp_backward_##SUF(void* h, std::int64_t rows, const T* x, const T* y, const T* w,  \
                            const T* gz, T* gx, T* gy, T* gw, int workers, int interp,        \
                            std::uint64_t* st) {                                              \
    return tp_backward<T>(h, rows, x, y, w, gz, gx, gy, gw, workers, interp, st);            \
  }                                                                                           \
  int cgr_tp_double_backward_##SUF(void* h, std::int64_t rows, const T* x, const T* y,       \
                                   const T* w, const T* gz, const T* da, const T* db,         \
                                   const T* dc, T* ox, T* oy, T* ow, T* ogz, int seven,       \
                                   int workers, std::uint64_t* st) {                          \
    return tp_double_backward<T>(h, rows, x, y, w, gz, da, db, dc, ox, oy, ow, ogz, seven,   \
                                 workers, st);                                                \
  }                                                                                           \
  int cgr_conv_forward_##SUF(void* h, std::int64_t nodes, std::int64_t ne,                   \
                             const std::int32_t* src, const std::int32_t* dst, const T* nx,   \
                             const T* ey, const T* ew, T* nz, int atomic, int workers,        \
                             int chunks, int unfused, std::uint64_t* st) {                    \
    return conv_forward<T>(h, nodes, ne, src, dst, nx, ey, ew, nz, atomic, workers, chunks,  \
                           unfused, st);                                                      \
  }                                                                                           \
  int cgr_conv_backward_##SUF(void* h, std::int64_t nodes, std::int64_t ne,                  \
                              const std::int32_t* src, const std::int32_t* dst, const T* nx,  \
                              const T* ey, const T* ew, const T* gnz, T* gnx, T* gey, T* gew, \
                              int atomic, int workers, int chunks, int unfused,               \
                              std::uint64_t* st) {                                            \
    return conv_backward<T>(h, nodes, ne, src, dst, nx, ey, ew, gnz, gnx, gey, gew, atomic,  \
                            workers, chunks, unfused, st);                                    \
  }                                                                                           \
  int cgr_bench_tp_##SUF(void* h, std::int64_t rows, int ops, int warmup, int iters,         \
                         int workers, std::uint64_t seed, double* secs) {                     \
    return bench_tp<T>(h, rows, ops, warmup, iters, workers, seed, secs);                    \
  }                                                                                           \
  int cgr_bench_conv_##SUF(void* h, int n, double rc, int ops, int warmup, int iters,        \
                           int workers, std::uint64_t seed, double* secs, std::int64_t* e) {  \
    return bench_conv<T>(h, n, rc, ops, warmup, iters, workers, seed, secs, e);              \
  }

CGR_TYPED(f32, float)
CGR_TYPED(f64, double)

}  // extern "C"
