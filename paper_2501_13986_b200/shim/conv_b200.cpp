// Drop-in replacement for cgforge's src/conv.cpp (include/cgforge/conv.hpp,
// unchanged): the fused convolution and the unfused gather -> TP -> scatter
// comparator (gather, batched TP, per-node sums) run on the B200 kernels
// through the C ABI; the graph utilities
// (XYZ loading, CSR build, radius graph, transpose permutation, lattice) are
// host code with the reference's contracts (conv.hpp:20-91).
//
// ConvStats follow a store/load model of the GPU kernels: the fused conv
// writes each output row once (output_store_ops = |V|, stores |V| dim_z) and
// streams y, W per edge plus x per edge from L2; the unfused path stores one
// z row per edge and reads the gathered x twice (gather + TP). Mode::atomic
// runs the atomic edge-list kernels (no sortedness or permutation required,
// as in conv.cpp:240 / 371-374).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cgforge/conv.hpp"
#include "plan_impl_b200.hpp"

namespace cgforge::conv {

using engine::b200::check;
using engine::b200::dtype;

// ---- graph utilities ---------------------------------------------------------

Geometry load_xyz(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw XyzError("cannot open " + path);
  std::string text;
  if (!std::getline(f, text)) throw XyzError("missing atom count line");
  long count = 0;
  {
    const char* b = text.c_str();
    char* end = nullptr;
    count = std::strtol(b, &end, 10);
    bool ok = end != b;
    for (const char* q = end; ok && *q; ++q) ok = std::isspace(static_cast<unsigned char>(*q)) != 0;
    if (!ok) throw XyzError("line 1: malformed atom count \"" + text + "\"");
  }
  if (count < 0) throw XyzError("line 1: negative atom count");
  std::getline(f, text);  // comment (may be absent when count == 0)
  Geometry g;
  for (int line = 3; std::getline(f, text); ++line) {
    if (text.find_first_not_of(" \t\r\n") == std::string::npos) continue;
    std::istringstream in(text);
    std::string el;
    std::array<double, 3> r{};
    if (!(in >> el >> r[0] >> r[1] >> r[2]))
      throw XyzError("line " + std::to_string(line) + ": expected `El x y z`, got \"" + text + "\"");
    if (!std::isfinite(r[0]) || !std::isfinite(r[1]) || !std::isfinite(r[2]))
      throw XyzError("line " + std::to_string(line) + ": non-finite coordinate");
    g.species.push_back(el);
    g.positions.push_back(r);
  }
  if (static_cast<long>(g.positions.size()) != count)
    throw XyzError("atom count line says " + std::to_string(count) + " but file has " +
                   std::to_string(g.positions.size()) + " rows");
  return g;
}

GraphCSR make_graph(std::int64_t node_count, std::vector<Edge> edges, bool allow_self_loops) {
  for (const Edge& e : edges) {
    const bool in_range = e.src >= 0 && e.dst >= 0 && e.src < node_count && e.dst < node_count;
    if (!in_range) throw std::invalid_argument("make_graph: edge endpoint out of range");
    if (e.src == e.dst && !allow_self_loops)
      throw std::invalid_argument("make_graph: self-loop (" + std::to_string(e.src) + ")");
  }
  // sort by (src, dst) via one 64-bit key, then drop duplicates
  std::vector<std::uint64_t> key(edges.size());
  for (std::size_t i = 0; i < edges.size(); ++i)
    key[i] = (static_cast<std::uint64_t>(edges[i].src) << 32) | static_cast<std::uint32_t>(edges[i].dst);
  std::sort(key.begin(), key.end());
  key.erase(std::unique(key.begin(), key.end()), key.end());
  GraphCSR g;
  g.node_count = node_count;
  g.edges.resize(key.size());
  g.row_ptr.assign(static_cast<std::size_t>(node_count) + 1, 0);
  for (std::size_t i = 0; i < key.size(); ++i) {
    g.edges[i] = {static_cast<std::int32_t>(key[i] >> 32), static_cast<std::int32_t>(key[i] & 0xffffffffu)};
    ++g.row_ptr[static_cast<std::size_t>(g.edges[i].src) + 1];
  }
  for (std::size_t v = 1; v < g.row_ptr.size(); ++v) g.row_ptr[v] += g.row_ptr[v - 1];
  return g;
}

GraphCSR radius_graph(const Geometry& geo, double r_cut) {
  if (!(r_cut > 0.0)) throw std::invalid_argument("radius_graph: r_cut must be positive");
  const std::int64_t n = geo.size();
  std::vector<Edge> edges;
  if (n > 0) {
    // Bin atoms into cubic cells of side r_cut (cell ids sorted), then test
    // the 27 neighbouring cells of each atom.
    std::array<double, 3> lo = geo.positions[0];
    for (const auto& p : geo.positions)
      for (int d = 0; d < 3; ++d) lo[d] = std::min(lo[d], p[d]);
    auto cell = [&](const std::array<double, 3>& p, int d) {
      return static_cast<std::int64_t>(std::floor((p[d] - lo[d]) / r_cut));
    };
    std::array<std::int64_t, 3> ext{1, 1, 1};
    for (const auto& p : geo.positions)
      for (int d = 0; d < 3; ++d) ext[d] = std::max(ext[d], cell(p, d) + 1);
    auto cid = [&](std::int64_t a, std::int64_t b, std::int64_t c) { return (a * ext[1] + b) * ext[2] + c; };
    std::vector<std::pair<std::int64_t, std::int32_t>> bins(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i)
      bins[i] = {cid(cell(geo.positions[i], 0), cell(geo.positions[i], 1), cell(geo.positions[i], 2)),
                 static_cast<std::int32_t>(i)};
    std::sort(bins.begin(), bins.end());
    const double r2 = r_cut * r_cut;
    for (std::int64_t i = 0; i < n; ++i) {
      const auto& pi = geo.positions[i];
      const std::int64_t c0 = cell(pi, 0), c1 = cell(pi, 1), c2 = cell(pi, 2);
      for (std::int64_t a = c0 - 1; a <= c0 + 1; ++a)
        for (std::int64_t b = c1 - 1; b <= c1 + 1; ++b)
          for (std::int64_t c = c2 - 1; c <= c2 + 1; ++c) {
            if (a < 0 || b < 0 || c < 0 || a >= ext[0] || b >= ext[1] || c >= ext[2]) continue;
            const std::int64_t id = cid(a, b, c);
            auto it = std::lower_bound(bins.begin(), bins.end(), std::make_pair(id, std::int32_t(-1)));
            for (; it != bins.end() && it->first == id; ++it) {
              const std::int32_t j = it->second;
              if (j == i) continue;
              const auto& pj = geo.positions[j];
              const double dx = pi[0] - pj[0], dy = pi[1] - pj[1], dz = pi[2] - pj[2];
              if (dx * dx + dy * dy + dz * dz <= r2) edges.push_back({static_cast<std::int32_t>(i), j});
            }
          }
    }
  }
  return make_graph(n, std::move(edges));
}

std::vector<std::int64_t> transpose_permutation(const GraphCSR& g) {
  // position of each edge in the CSR of the reversed graph: a stable bucket
  // fill by dst (edges arrive in (src, dst) order, so src ascends per bucket)
  std::vector<std::int64_t> next(static_cast<std::size_t>(g.node_count) + 1, 0);
  for (const Edge& e : g.edges) ++next[static_cast<std::size_t>(e.dst) + 1];
  for (std::size_t v = 1; v < next.size(); ++v) next[v] += next[v - 1];
  std::vector<std::int64_t> perm(g.edges.size());
  for (std::size_t e = 0; e < g.edges.size(); ++e) perm[e] = next[static_cast<std::size_t>(g.edges[e].dst)]++;
  return perm;
}

Geometry cubic_lattice(int nx, int ny, int nz, double spacing) {
  Geometry g;
  g.positions.reserve(static_cast<std::size_t>(nx) * ny * nz);
  for (int a = 0; a < nx; ++a)
    for (int b = 0; b < ny; ++b)
      for (int c = 0; c < nz; ++c) {
        g.positions.push_back({a * spacing, b * spacing, c * spacing});
        g.species.emplace_back("C");
      }
  return g;
}

std::string graph_to_json(const GraphCSR& g) {
  std::string s = "{\"edges\":[";
  for (std::size_t e = 0; e < g.edges.size(); ++e) {
    s += e ? ",[" : "[";
    s += std::to_string(g.edges[e].src) + "," + std::to_string(g.edges[e].dst) + "]";
  }
  return s + "],\"nodes\":" + std::to_string(g.node_count) + "}";
}

// ---- fused convolution on the GPU -------------------------------------------

namespace {

const tpspec::ValidatedProblem& prob(const engine::TpPlan& p) { return p.problem(); }

template <typename T>
void require_conv_shapes(const tpspec::ValidatedProblem& p, const GraphCSR& g, const std::vector<T>& node_x,
                         const std::vector<T>& edge_y, const std::vector<T>& edge_w) {
  const auto V = static_cast<std::size_t>(g.node_count), E = static_cast<std::size_t>(g.edge_count());
  if (node_x.size() != V * static_cast<std::size_t>(p.dim_x)) throw engine::ShapeError("conv: node_x shape mismatch");
  if (edge_y.size() != E * static_cast<std::size_t>(p.dim_y)) throw engine::ShapeError("conv: edge_y shape mismatch");
  if (edge_w.size() != E * p.total_weights) throw engine::ShapeError("conv: edge_w shape mismatch");
}

void require_sorted(const GraphCSR& g) {
  for (std::size_t e = 1; e < g.edges.size(); ++e) {
    const Edge &a = g.edges[e - 1], &b = g.edges[e];
    if (a.src > b.src || (a.src == b.src && a.dst >= b.dst))
      throw std::invalid_argument("conv: deterministic mode requires edges sorted by first coordinate");
  }
}

std::vector<std::int32_t> neighbours(const GraphCSR& g) {
  std::vector<std::int32_t> nb(g.edges.size());
  for (std::size_t e = 0; e < g.edges.size(); ++e) nb[e] = g.edges[e].dst;
  return nb;
}

// The CSR row pointer rebuilt from the (sorted) edge list: the reference's
// conv reads only g.edges (conv.cpp:234-528), so a GraphCSR whose row_ptr is
// stale or missing must still work.
std::vector<std::int64_t> row_ptr_of(const GraphCSR& g) {
  std::vector<std::int64_t> rp(static_cast<std::size_t>(g.node_count) + 1, 0);
  for (const auto& e : g.edges) {
    if (e.src < 0 || e.src >= g.node_count || e.dst < 0 || e.dst >= g.node_count)
      throw std::invalid_argument("conv: edge endpoint out of range");
    ++rp[static_cast<std::size_t>(e.src) + 1];
  }
  for (std::size_t v = 1; v < rp.size(); ++v) rp[v] += rp[v - 1];
  return rp;
}

// ConvStats from libcgf's store / load model of the GPU kernels (cgf_conv_stats).
ConvStats conv_stats(const engine::TpPlan& plan, int op, Mode mode, bool unfused, const GraphCSR& g) {
  std::uint64_t s[4] = {0, 0, 0, 0};
  check(cgf_conv_stats(plan.impl().gpu, op, mode == Mode::atomic ? CGF_CONV_ATOMIC : CGF_CONV_DETERMINISTIC,
                       unfused ? 1 : 0, g.node_count, g.edge_count(), s));
  ConvStats st;
  st.loads_words = s[0];
  st.stores_words = s[1];
  st.output_store_ops = s[2];
  st.flops = s[3];
  return st;
}

std::vector<std::int32_t> sources(const GraphCSR& g) {
  std::vector<std::int32_t> s(g.edges.size());
  for (std::size_t e = 0; e < g.edges.size(); ++e) s[e] = g.edges[e].src;
  return s;
}

}  // namespace

template <typename T>
ConvStats ConvPlan::forward(const GraphCSR& g, const std::vector<T>& node_x, const std::vector<T>& edge_y,
                            const std::vector<T>& edge_w, std::vector<T>& node_z, Mode mode,
                            const ConvOptions&) const {
  const auto& p = prob(*plan_);
  require_conv_shapes(p, g, node_x, edge_y, edge_w);
  if (mode == Mode::deterministic) require_sorted(g);
  node_z.assign(static_cast<std::size_t>(g.node_count) * p.dim_z, T(0));
  const auto nb = neighbours(g);
  if (g.node_count > 0 && mode == Mode::atomic)
    check(cgf_conv_forward_atomic_host(plan_->impl().gpu, dtype<T>(), g.node_count, g.edge_count(), sources(g).data(),
                                       nb.data(), node_x.data(), edge_y.data(), edge_w.data(), node_z.data()));
  else if (g.node_count > 0)
    check(cgf_conv_forward_host(plan_->impl().gpu, dtype<T>(), g.node_count, g.edge_count(), row_ptr_of(g).data(),
                                nb.data(), node_x.data(), edge_y.data(), edge_w.data(), node_z.data(),
                                CGF_CONV_DETERMINISTIC));
  return conv_stats(*plan_, CGF_OP_FORWARD, mode, false, g);
}

template <typename T>
ConvStats ConvPlan::backward(const GraphCSR& g, const std::vector<std::int64_t>& perm, const std::vector<T>& node_x,
                             const std::vector<T>& edge_y, const std::vector<T>& edge_w,
                             const std::vector<T>& g_node_z, std::vector<T>& g_node_x, std::vector<T>& g_edge_y,
                             std::vector<T>& g_edge_w, Mode mode, const ConvOptions&) const {
  const auto& p = prob(*plan_);
  require_conv_shapes(p, g, node_x, edge_y, edge_w);
  if (g_node_z.size() != static_cast<std::size_t>(g.node_count) * p.dim_z)
    throw engine::ShapeError("conv: g_node_z shape mismatch");
  if (mode == Mode::deterministic) {
    require_sorted(g);
    if (perm.size() != g.edges.size()) throw engine::ShapeError("conv: transpose permutation size mismatch");
  }
  g_node_x.assign(node_x.size(), T(0));
  g_edge_y.assign(edge_y.size(), T(0));
  g_edge_w.assign(edge_w.size(), T(0));
  const auto nb = neighbours(g);
  if (g.node_count > 0 && mode == Mode::atomic)
    check(cgf_conv_backward_atomic_host(plan_->impl().gpu, dtype<T>(), g.node_count, g.edge_count(),
                                        sources(g).data(), nb.data(), node_x.data(), edge_y.data(), edge_w.data(),
                                        g_node_z.data(), g_node_x.data(), g_edge_y.data(), g_edge_w.data()));
  else if (g.node_count > 0)
    check(cgf_conv_backward_host(plan_->impl().gpu, dtype<T>(), g.node_count, g.edge_count(), row_ptr_of(g).data(),
                                 nb.data(), node_x.data(), edge_y.data(), edge_w.data(), g_node_z.data(),
                                 g_node_x.data(), g_edge_y.data(), g_edge_w.data(), CGF_CONV_DETERMINISTIC));
  return conv_stats(*plan_, CGF_OP_BACKWARD, mode, false, g);
}

// ---- unfused gather -> batched TP -> scatter (the GPU TP on gathered rows) --

template <typename T>
ConvStats unfused_forward(const engine::TpPlan& plan, const GraphCSR& g, const std::vector<T>& node_x,
                          const std::vector<T>& edge_y, const std::vector<T>& edge_w, std::vector<T>& node_z,
                          const engine::Options&) {
  const auto& p = prob(plan);
  require_conv_shapes(p, g, node_x, edge_y, edge_w);
  node_z.assign(static_cast<std::size_t>(g.node_count) * p.dim_z, T(0));
  // gather, batched TP and per-node sums in edge order, all on the GPU
  if (g.node_count > 0)
    check(cgf_conv_unfused_forward_host(plan.impl().gpu, dtype<T>(), g.node_count, g.edge_count(), sources(g).data(),
                                        neighbours(g).data(), node_x.data(), edge_y.data(), edge_w.data(),
                                        node_z.data()));
  return conv_stats(plan, CGF_OP_FORWARD, Mode::deterministic, true, g);
}

template <typename T>
ConvStats unfused_backward(const engine::TpPlan& plan, const GraphCSR& g, const std::vector<T>& node_x,
                           const std::vector<T>& edge_y, const std::vector<T>& edge_w, const std::vector<T>& g_node_z,
                           std::vector<T>& g_node_x, std::vector<T>& g_edge_y, std::vector<T>& g_edge_w,
                           const engine::Options&) {
  const auto& p = prob(plan);
  require_conv_shapes(p, g, node_x, edge_y, edge_w);
  g_node_x.assign(node_x.size(), T(0));
  g_edge_y.assign(edge_y.size(), T(0));
  g_edge_w.assign(edge_w.size(), T(0));
  if (g.node_count > 0)
    check(cgf_conv_unfused_backward_host(plan.impl().gpu, dtype<T>(), g.node_count, g.edge_count(),
                                         sources(g).data(), neighbours(g).data(), node_x.data(), edge_y.data(),
                                         edge_w.data(), g_node_z.data(), g_node_x.data(), g_edge_y.data(),
                                         g_edge_w.data()));
  return conv_stats(plan, CGF_OP_BACKWARD, Mode::deterministic, true, g);
}

#define CGF_CONV_INST(T)                                                                                            \
  template ConvStats ConvPlan::forward<T>(const GraphCSR&, const std::vector<T>&, const std::vector<T>&,            \
                                          const std::vector<T>&, std::vector<T>&, Mode, const ConvOptions&) const;  \
  template ConvStats ConvPlan::backward<T>(const GraphCSR&, const std::vector<std::int64_t>&, const std::vector<T>&, \
                                           const std::vector<T>&, const std::vector<T>&, const std::vector<T>&,     \
                                           std::vector<T>&, std::vector<T>&, std::vector<T>&, Mode,                 \
                                           const ConvOptions&) const;                                               \
  template ConvStats unfused_forward<T>(const engine::TpPlan&, const GraphCSR&, const std::vector<T>&,              \
                                        const std::vector<T>&, const std::vector<T>&, std::vector<T>&,              \
                                        const engine::Options&);                                                    \
  template ConvStats unfused_backward<T>(const engine::TpPlan&, const GraphCSR&, const std::vector<T>&,             \
                                         const std::vector<T>&, const std::vector<T>&, const std::vector<T>&,       \
                                         std::vector<T>&, std::vector<T>&, std::vector<T>&, const engine::Options&);
CGF_CONV_INST(float)
CGF_CONV_INST(double)
#undef CGF_CONV_INST

}  // namespace cgforge::conv
