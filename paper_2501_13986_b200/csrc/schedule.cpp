// The reference's phase plan, counters and dumps (schedule.hpp), restated on
// the product's split problem. The subkernels are already in the reference's
// normalised order (Problem::subs: stable sort by z offset,
// scheduler.cpp:146-151); Sub::split_index maps them back to the split order
// the reference's `order` / `split_map` refer to.
#include "schedule.hpp"

#include <algorithm>
#include <array>
#include <charconv>
#include <cstdio>
#include <functional>
#include <map>
#include <sstream>
#include <tuple>

namespace cgf {

namespace {

using Ids = std::vector<std::uint32_t>;

bool has(const Ids& v, std::uint32_t id) { return std::find(v.begin(), v.end(), id) != v.end(); }

Ids sorted_unique(Ids v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  return v;
}

// The four operands of one subkernel as resources (scheduler.cpp:106-131):
// x chunk, y segment, W slice (B: b words; C: b x b' tile of the row-major
// W[w][u] block), z piece.
std::array<SchedResource, 4> operands(const Sub& s) {
  const std::uint32_t xw = static_cast<std::uint32_t>(s.bp * s.dx());
  const std::uint32_t zw = static_cast<std::uint32_t>(s.b * s.dz());
  const std::uint32_t yw = static_cast<std::uint32_t>(s.dy());
  SchedResource w = s.kind == Kind::B
                        ? SchedResource{Space::W, s.w_off, 1, static_cast<std::uint32_t>(s.b), static_cast<std::uint32_t>(s.b)}
                        : SchedResource{Space::W, s.w_off, static_cast<std::uint32_t>(s.b),
                                        static_cast<std::uint32_t>(s.bp), s.w_stride};
  return {SchedResource{Space::X, s.x_off, 1, xw, xw}, SchedResource{Space::Y, s.y_off, 1, yw, yw}, w,
          SchedResource{Space::Z, s.z_off, 1, zw, zw}};
}

struct Plan {
  const Problem& p;
  std::uint32_t budget;
  std::vector<SchedResource> res;
  std::vector<std::array<std::uint32_t, 4>> need;  // per position: x, y, w, z resource ids

  std::uint64_t words(const Ids& ids) const {
    std::uint64_t w = 0;
    for (auto id : ids) w += res[id].words();
    return w;
  }
  bool is_z(std::uint32_t id) const { return res[id].space == Space::Z; }

  void intern_all() {
    std::map<std::tuple<int, std::uint32_t, std::uint32_t, std::uint32_t, std::uint32_t>, std::uint32_t> seen;
    for (const auto& s : p.subs) {
      std::array<std::uint32_t, 4> ids{};
      const auto ops = operands(s);
      for (int k = 0; k < 4; ++k) {
        const auto& r = ops[k];
        const auto key = std::make_tuple(static_cast<int>(r.space), r.offset, r.rows, r.cols, r.row_stride);
        auto it = seen.find(key);
        if (it == seen.end()) {
          it = seen.emplace(key, static_cast<std::uint32_t>(res.size())).first;
          res.push_back(r);
        }
        ids[k] = it->second;
      }
      need.push_back(ids);
    }
  }

  // distinct operands of position `pos`, in x, y, w, z order
  Ids operands_of(std::size_t pos) const {
    Ids v;
    for (auto id : need[pos])
      if (!has(v, id)) v.push_back(id);
    return v;
  }

  // first position >= from that reads or writes resource id (npos: never)
  std::size_t next_use(std::uint32_t id, std::size_t from) const {
    for (std::size_t q = from; q < need.size(); ++q)
      if (has(Ids(need[q].begin(), need[q].end()), id)) return q;
    return need.size();
  }

  void single_phase(ScheduleModel& m) const {
    SchedPhase ph;
    for (std::uint32_t id = 0; id < res.size(); ++id) {
      ph.resident.push_back(id);
      (is_z(id) ? ph.z_flush : ph.loaded).push_back(id);
    }
    for (std::uint32_t q = 0; q < need.size(); ++q) ph.instructions.push_back(q);
    m.strategy = Strategy::SinglePhase;
    m.phases.push_back(std::move(ph));
  }

  // x and y stay resident; runs of positions writing one z piece (with their
  // weights) are packed into phases up to the budget.
  bool stream_z(ScheduleModel& m) const {
    Ids xy;
    for (std::uint32_t id = 0; id < res.size(); ++id)
      if (res[id].space == Space::X || res[id].space == Space::Y) xy.push_back(id);
    const std::uint64_t xy_words = words(xy);
    struct Run {
      std::uint32_t z;
      Ids pos, w;
    };
    std::vector<Run> runs;
    for (std::uint32_t q = 0; q < need.size(); ++q) {
      if (runs.empty() || runs.back().z != need[q][3]) runs.push_back({need[q][3], {}, {}});
      runs.back().pos.push_back(q);
      runs.back().w.push_back(need[q][2]);
    }
    for (auto& r : runs) r.w = sorted_unique(r.w);
    if (xy_words > budget) return false;
    for (const auto& r : runs)
      if (xy_words + res[r.z].words() + words(r.w) > budget) return false;
    m.strategy = Strategy::StreamZ;
    for (std::size_t i = 0; i < runs.size();) {
      SchedPhase ph;
      std::uint64_t used = xy_words;
      for (; i < runs.size(); ++i) {
        const std::uint64_t extra = res[runs[i].z].words() + words(runs[i].w);
        if (used + extra > budget && !ph.instructions.empty()) break;
        used += extra;
        ph.z_flush.push_back(runs[i].z);
        ph.loaded.insert(ph.loaded.end(), runs[i].w.begin(), runs[i].w.end());
        ph.instructions.insert(ph.instructions.end(), runs[i].pos.begin(), runs[i].pos.end());
      }
      ph.z_flush = sorted_unique(ph.z_flush);
      if (m.phases.empty()) {
        ph.loaded.insert(ph.loaded.end(), xy.begin(), xy.end());
      } else {
        ph.retained = xy;
      }
      ph.loaded = sorted_unique(ph.loaded);
      Ids all = ph.loaded;
      all.insert(all.end(), ph.retained.begin(), ph.retained.end());
      all.insert(all.end(), ph.z_flush.begin(), ph.z_flush.end());
      ph.resident = sorted_unique(all);
      m.phases.push_back(std::move(ph));
    }
    return true;
  }

  // Fill scratch until the next position does not fit; carry over the
  // resources used soonest (Belady on the known stream).
  void greedy(ScheduleModel& m) const {
    m.strategy = Strategy::Greedy;
    const std::size_t n = need.size();
    Ids carried;
    std::size_t q = 0;
    while (q < n) {
      SchedPhase ph;
      ph.retained = carried;
      Ids live = carried;
      std::uint64_t used = words(live);
      for (; q < n; ++q) {
        Ids miss;
        for (auto id : operands_of(q))
          if (!has(live, id)) miss.push_back(id);
        const std::uint64_t extra = words(miss);
        if (used + extra > budget) break;
        live.insert(live.end(), miss.begin(), miss.end());
        ph.loaded.insert(ph.loaded.end(), miss.begin(), miss.end());
        used += extra;
        ph.instructions.push_back(static_cast<std::uint32_t>(q));
      }
      if (ph.instructions.empty()) {
        // the carried set blocks the next position: flush its z pieces alone
        if (carried.empty()) throw BudgetError("greedy scheduling failed to place an instruction");
        for (auto id : carried)
          if (is_z(id)) ph.z_flush.push_back(id);
        if (!ph.z_flush.empty()) {
          ph.resident = carried;
          ph.retained.clear();
          m.phases.push_back(std::move(ph));
        }
        carried.clear();
        continue;
      }
      ph.resident = live;
      Ids keep;
      if (q < n) {
        const Ids next = operands_of(q);
        const std::uint64_t next_words = words(next);
        std::vector<std::pair<std::size_t, std::uint32_t>> cand;  // (next use, id)
        for (auto id : live) {
          if (has(next, id)) continue;
          const std::size_t nu = next_use(id, q);
          if (nu < n) cand.emplace_back(nu, id);
        }
        std::sort(cand.begin(), cand.end());
        std::uint64_t kept = 0;
        for (const auto& [nu, id] : cand) {
          (void)nu;
          if (next_words + kept + res[id].words() <= budget) {
            keep.push_back(id);
            kept += res[id].words();
          }
        }
        for (auto id : next)
          if (has(live, id)) keep.push_back(id);
        keep = sorted_unique(keep);
      }
      for (auto id : live)
        if (is_z(id) && !has(keep, id)) ph.z_flush.push_back(id);
      carried = keep;
      m.phases.push_back(std::move(ph));
    }
  }
};

std::string sub_name(const Sub& s) {
  return "subkernel " + std::to_string(s.split_index) + " (" + (s.kind == Kind::B ? "B" : "C") + ", l=(" +
         std::to_string(s.l1) + "," + std::to_string(s.l2) + "," + std::to_string(s.l3) + "), b=" +
         std::to_string(s.b) + ", b'=" + std::to_string(s.bp) + ")";
}

}  // namespace

ScheduleModel build_schedule_model(const Problem& p, std::uint32_t budget) {
  Plan pl{p, budget, {}, {}};
  // admission: every subkernel's working set fits (scheduler.cpp:161-170)
  for (const auto& s : p.subs) {
    std::uint64_t ws = 0;
    for (const auto& r : operands(s)) ws += r.words();
    if (ws > budget)
      throw BudgetError("budget " + std::to_string(budget) + " words below working set " + std::to_string(ws) +
                        " of " + sub_name(s));
  }
  pl.intern_all();
  ScheduleModel m;
  m.budget = budget;
  for (const auto& s : p.subs) m.order.push_back(static_cast<std::uint32_t>(s.split_index));
  std::uint64_t total = 0;
  for (const auto& r : pl.res) total += r.words();
  if (total <= budget) pl.single_phase(m);
  else if (!pl.stream_z(m)) pl.greedy(m);
  m.resources = pl.res;
  // Counters (engine.cpp:115-168): the forward reads each phase's newly
  // loaded x / y / w and stores its flushed z; the backward reads the same
  // plus every z piece that is not carried over (g_z staged), and stores
  // nothing (it accumulates straight into gx / gy / gw).
  for (const auto& ph : m.phases) {
    for (auto id : ph.resident) {
      const bool z = pl.is_z(id), loaded = has(ph.loaded, id), kept = has(ph.retained, id);
      if (!z && loaded) {
        m.fwd_loads += pl.res[id].words();
        m.bwd_loads += pl.res[id].words();
      }
      if (z && !kept) m.bwd_loads += pl.res[id].words();
    }
    for (auto id : ph.z_flush) m.fwd_stores += pl.res[id].words();
  }
  m.fwd_flops = p.fwd_flops_per_row();
  m.bwd_flops = p.bwd_flops_per_row();
  return m;
}

// ---------------------------------------------------------------- JSON ---
namespace {

// A minimal writer reproducing the reference's dump(2) output: keys in sorted
// order, 2-space indent, number arrays inline, doubles in shortest round-trip
// form with a trailing ".0" for integral values.
struct JW {
  std::ostringstream o;
  int ind = 0;
  void nl() { o << "\n" << std::string(2 * ind, ' '); }
  // arrays of numbers stay on one line: [0,1,2]
  void arr(const std::vector<std::uint32_t>& v) {
    o << "[";
    for (std::size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
    o << "]";
  }
};

std::string dbl(double v) {
  char b[64];
  auto r = std::to_chars(b, b + sizeof b, v);
  std::string s(b, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

const char* space_name(Space s) {
  switch (s) {
    case Space::X: return "x";
    case Space::Y: return "y";
    case Space::W: return "w";
    case Space::Z: return "z";
  }
  return "?";
}

}  // namespace

std::string schedule_json(const Problem& p, const ScheduleModel& s) {
  // each object is a list of (key, writer) pairs emitted in sorted key order
  using Field = std::pair<std::string, std::function<void(JW&)>>;
  std::function<void(JW&, std::vector<Field>)> obj = [&](JW& w, std::vector<Field> f) {
    std::sort(f.begin(), f.end(), [](const Field& a, const Field& b) { return a.first < b.first; });
    w.o << "{";
    ++w.ind;
    for (std::size_t i = 0; i < f.size(); ++i) {
      w.nl();
      w.o << "\"" << f[i].first << "\": ";
      f[i].second(w);
      if (i + 1 < f.size()) w.o << ",";
    }
    --w.ind;
    w.nl();
    w.o << "}";
  };
  auto num = [](std::uint64_t v) { return [v](JW& w) { w.o << v; }; };
  auto str = [](std::string v) { return [v](JW& w) { w.o << "\"" << v << "\""; }; };
  auto list = [&](auto items, auto each) {
    return [items, each, &obj](JW& w) {
      if (items.empty()) {
        w.o << "[]";
        return;
      }
      w.o << "[";
      ++w.ind;
      for (std::size_t i = 0; i < items.size(); ++i) {
        w.nl();
        obj(w, each(items[i]));
        if (i + 1 < items.size()) w.o << ",";
      }
      --w.ind;
      w.nl();
      w.o << "]";
    };
  };
  static const char* strategy[] = {"single_phase", "stream_z", "greedy"};
  std::vector<const Sub*> split(p.subs.size());
  for (const auto& sb : p.subs) split[sb.split_index] = &sb;
  const double ai = (s.fwd_loads + s.fwd_stores) ? static_cast<double>(s.fwd_flops) /
                                                       (8.0 * static_cast<double>(s.fwd_loads + s.fwd_stores))
                                                 : 0.0;
  JW w;
  obj(w, {
             {"budget_words", num(s.budget)},
             {"order", [&](JW& j) { j.arr(s.order); }},
             {"phases", list(s.phases,
                             [&](const SchedPhase& ph) {
                               return std::vector<Field>{
                                   {"instructions", [&ph](JW& j) { j.arr(ph.instructions); }},
                                   {"loaded", [&ph](JW& j) { j.arr(ph.loaded); }},
                                   {"resident", [&ph](JW& j) { j.arr(ph.resident); }},
                                   {"retained", [&ph](JW& j) { j.arr(ph.retained); }},
                                   {"z_flush", [&ph](JW& j) { j.arr(ph.z_flush); }}};
                             })},
             {"resources", list(s.resources,
                                [&](const SchedResource& r) {
                                  return std::vector<Field>{{"cols", num(r.cols)},
                                                            {"offset", num(r.offset)},
                                                            {"row_stride", num(r.row_stride)},
                                                            {"rows", num(r.rows)},
                                                            {"space", str(space_name(r.space))}};
                                })},
             {"split_map", list(split,
                                [&](const Sub* sb) {
                                  return std::vector<Field>{{"b", num(sb->b)},
                                                            {"b_prime", num(sb->bp)},
                                                            {"instruction", num(sb->origin)},
                                                            {"kind", str(sb->kind == Kind::B ? "B" : "C")},
                                                            {"w_row_stride", num(sb->w_stride)},
                                                            {"weight_offset", num(sb->w_off)},
                                                            {"x_offset", num(sb->x_off)},
                                                            {"y_offset", num(sb->y_off)},
                                                            {"z_offset", num(sb->z_off)}};
                                })},
             {"strategy", str(strategy[static_cast<int>(s.strategy)])},
             {"traffic",
              [&](JW& j) {
                obj(j, {{"arithmetic_intensity_fp64", [ai](JW& k) { k.o << dbl(ai); }},
                        {"flops", num(s.fwd_flops)},
                        {"loads_words", num(s.fwd_loads)},
                        {"stores_words", num(s.fwd_stores)}});
              }},
         });
  return w.o.str();
}

// ------------------------------------------------------------- listing ---
namespace {

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// "name" for one register, "name[0:n]" for a group of n > 1
std::string grp(const char* name, int n) {
  return std::string(name) + (n == 1 ? "[0]" : "[0:" + std::to_string(n) + "]");
}

std::string mem(const char* arr, std::uint32_t base, std::uint32_t stride) {
  std::string s = std::string(arr) + "[@" + std::to_string(base);
  if (stride) s += "+" + std::to_string(stride) + "t";
  return s + "]";
}

std::string reg(const char* name, int i) { return std::string(name) + "[" + std::to_string(i) + "]"; }

}  // namespace

std::string listing_text(const Sub& s, bool backward) {
  const int dx = s.dx(), dy = s.dy(), dz = s.dz(), b = s.b, bp = s.bp;
  const bool B = s.kind == Kind::B;
  const int lanes = std::max(b, bp);
  const std::string L = " |" + std::to_string(bp) + "L";
  const std::string wtile = "[@" + std::to_string(s.w_off) + ",s" + std::to_string(s.w_stride) + "|" +
                            std::to_string(b) + "x" + std::to_string(bp) + "]";
  std::ostringstream o;
  // one load op with every operand binding
  o << "load   " << grp("x", dx) << " = " << mem("X", s.x_off, dx) << " |" << bp << "L  " << grp("y", dy) << " = "
    << mem("Y", s.y_off, 0) << " |" << bp << "L";
  if (backward) o << "  " << grp("gz", dz) << " = " << mem("GZ", s.z_off, dz) << " |" << b << "L";
  if (B) o << "  w = " << mem("W", s.w_off, 1) << " |" << b << "L";
  o << "\n";
  (void)lanes;
  if (!backward) {
    for (const auto& e : s.cg->entries)
      o << "fma    " << reg("z", e.k) << " += " << g17(e.v) << " * " << reg("x", e.i) << " * " << reg("y", e.j) << L
        << "\n";
    if (B)
      for (int k = 0; k < dz; ++k) o << "scale  " << reg("out", k) << " += w * " << reg("z", k) << " |" << b << "L\n";
    else
      o << "matmul " << grp("out", dz) << " += W" << wtile << " * " << grp("z", dz) << "\n";
    o << "acc    " << mem("Z", s.z_off, dz) << " += " << grp("out", dz) << " |" << b << "L\n";
    return o.str();
  }
  if (B)
    for (int k = 0; k < dz; ++k) o << "scale  " << reg("gzp", k) << " += w * " << reg("gz", k) << " |" << b << "L\n";
  else
    o << "matmul " << grp("gzp", dz) << " += W^T" << wtile << " * " << grp("gz", dz) << "\n";
  for (const auto& e : s.cg->entries) {
    const std::string v = g17(e.v);
    o << "fma    " << reg("gx", e.i) << " += " << v << " * " << reg("y", e.j) << " * " << reg("gzp", e.k) << L << "\n";
    o << "fma    " << reg("gy", e.j) << " += " << v << " * " << reg("x", e.i) << " * " << reg("gzp", e.k) << L << "\n";
    o << "fma    " << reg("z", e.k) << " += " << v << " * " << reg("x", e.i) << " * " << reg("y", e.j) << L << "\n";
  }
  o << "reduce " << grp("gy", dy) << " over " << bp << "L\n";
  o << "acc    " << mem("GY", s.y_off, 0) << " += " << grp("gy", dy) << " |lane0\n";
  o << "acc    " << mem("GX", s.x_off, dx) << " += " << grp("gx", dx) << L << "\n";
  if (B) {
    for (int k = 0; k < dz; ++k) o << "scale  gw += " << reg("gz", k) << " * " << reg("z", k) << " |" << b << "L\n";
    o << "acc    " << mem("GW", s.w_off, 1) << " += gw |" << b << "L\n";
  } else {
    o << "outer  GW" << wtile << " += " << grp("gz", dz) << " (x) " << grp("z", dz) << "\n";
  }
  return o.str();
}

}  // namespace cgf
