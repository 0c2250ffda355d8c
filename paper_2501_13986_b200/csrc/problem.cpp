#include "problem.hpp"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <complex>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <numeric>
#include <sstream>
#include <tuple>

namespace cgf {

// ================================================================ irreps ==
int Irreps::dim() const {
  int d = 0;
  for (const auto& b : blocks) d += b.dim();
  return d;
}

int Irreps::offset(int seg) const {
  int d = 0;
  for (int k = 0; k < seg; ++k) d += blocks[k].dim();
  return d;
}

std::string Irreps::str() const {
  std::ostringstream os;
  for (size_t k = 0; k < blocks.size(); ++k)
    os << (k ? " + " : "") << blocks[k].mult << 'x' << blocks[k].l << (blocks[k].odd ? 'o' : 'e');
  return os.str();
}

Irreps parse_irreps(const std::string& text) {
  Irreps out;
  size_t pos = 0;
  auto ws = [&] {
    while (pos < text.size() && std::isspace(static_cast<unsigned char>(text[pos]))) ++pos;
  };
  ws();
  bool first = true;
  while (first || pos < text.size()) {
    if (!first) {
      if (text[pos] != '+') throw ParseError("expected '+' between irreps blocks near \"" + text.substr(pos) + "\"");
      ++pos;
      ws();
    }
    first = false;
    const size_t start = pos;
    while (pos < text.size() && !std::isspace(static_cast<unsigned char>(text[pos])) && text[pos] != '+') ++pos;
    const std::string tok = text.substr(start, pos - start);
    if (tok.empty()) throw ParseError("empty irreps token in \"" + text + "\"");
    const size_t x = tok.find('x');
    const auto bad = [&](const char* why) { return ParseError("bad irreps token \"" + tok + "\": " + why); };
    if (x == std::string::npos || x == 0 || x + 2 > tok.size() - 0 || tok.size() - x - 1 < 2)
      throw bad("expected <mult>x<l><e|o>");
    const std::string ms = tok.substr(0, x), ls = tok.substr(x + 1, tok.size() - x - 2);
    const char par = tok.back();
    if (par != 'e' && par != 'o') throw bad("parity must be 'e' or 'o'");
    for (char c : ms) if (!std::isdigit(static_cast<unsigned char>(c))) throw bad("multiplicity is not a number");
    for (char c : ls) if (!std::isdigit(static_cast<unsigned char>(c))) throw bad("l is not a number");
    long m = 0, l = 0;
    try {
      m = std::stol(ms);
      l = std::stol(ls);
    } catch (...) {
      throw bad("number out of range");
    }
    if (m <= 0) throw bad("multiplicity must be positive");
    out.blocks.push_back({static_cast<int>(m), static_cast<int>(l), par == 'o'});
    ws();
  }
  return out;
}

// ==================================================================== CG ==
namespace {

double fact(int n) {
  // Exact through 33! by 128-bit integer products, then one rounding.
  unsigned __int128 a = 1;
  for (int k = 2; k <= n; ++k) a *= static_cast<unsigned>(k);
  return static_cast<double>(a);
}

double racah(int l1, int l2, int l3, int m1, int m2, int m3) {
  if (m1 + m2 != m3) return 0.0;
  const double pre = std::sqrt((2.0 * l3 + 1.0) * fact(l1 + l2 - l3) * fact(l1 - l2 + l3) *
                               fact(-l1 + l2 + l3) / fact(l1 + l2 + l3 + 1)) *
                     std::sqrt(fact(l3 + m3) * fact(l3 - m3) * fact(l1 - m1) * fact(l1 + m1) *
                               fact(l2 - m2) * fact(l2 + m2));
  const int lo = std::max({0, l2 - l3 - m1, l1 - l3 + m2});
  const int hi = std::min({l1 + l2 - l3, l1 - m1, l2 + m2});
  double s = 0.0;
  for (int k = lo; k <= hi; ++k)
    s += ((k & 1) ? -1.0 : 1.0) / (fact(k) * fact(l1 + l2 - l3 - k) * fact(l1 - m1 - k) *
                                    fact(l2 + m2 - k) * fact(l3 - l2 + m1 + k) * fact(l3 - l1 - m2 + k));
  return pre * s;
}

using cd = std::complex<double>;

// Complex -> real spherical-harmonic basis, row = real index p, column =
// complex index m, both shifted by +l; Condon-Shortley phase on p > 0.
std::vector<cd> real_basis(int l) {
  const int d = 2 * l + 1;
  const double h = 1.0 / std::sqrt(2.0);
  std::vector<cd> u(static_cast<size_t>(d) * d, cd(0.0, 0.0));
  auto U = [&](int r, int c) -> cd& { return u[static_cast<size_t>(r) * d + c]; };
  U(l, l) = 1.0;
  for (int m = 1; m <= l; ++m) {
    const double cs = (m & 1) ? -1.0 : 1.0;
    U(l + m, l + m) = cs * h;
    U(l + m, l - m) = h;
    U(l - m, l + m) = cd(0.0, -cs * h);
    U(l - m, l - m) = cd(0.0, h);
  }
  return u;
}

CGBlock build(int l1, int l2, int l3) {
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  const auto u1 = real_basis(l1), u2 = real_basis(l2), u3 = real_basis(l3);
  std::vector<cd> t(static_cast<size_t>(d1) * d2 * d3);
  for (int m1 = -l1; m1 <= l1; ++m1)
    for (int m2 = -l2; m2 <= l2; ++m2) {
      const int m3 = m1 + m2;
      if (std::abs(m3) > l3) continue;
      const double c = racah(l1, l2, l3, m1, m2, m3);
      if (c == 0.0) continue;
      for (int i = 0; i < d1; ++i) {
        const cd f1 = u1[static_cast<size_t>(i) * d1 + l1 + m1];
        if (f1 == 0.0) continue;
        for (int j = 0; j < d2; ++j) {
          const cd f2 = u2[static_cast<size_t>(j) * d2 + l2 + m2];
          if (f2 == 0.0) continue;
          for (int k = 0; k < d3; ++k) {
            const cd f3 = std::conj(u3[static_cast<size_t>(k) * d3 + l3 + m3]);
            if (f3 == 0.0) continue;
            t[(static_cast<size_t>(i) * d2 + j) * d3 + k] += f1 * f2 * f3 * c;
          }
        }
      }
    }
  cd top = 0.0;
  for (const auto& v : t)
    if (std::abs(v) > std::abs(top)) top = v;
  if (std::abs(top) > 0.0) {
    const cd ph = std::conj(top) / std::abs(top);
    for (auto& v : t) v *= ph;
  }
  CGBlock b{l1, l2, l3, {}};
  for (int k = 0; k < d3; ++k)
    for (int i = 0; i < d1; ++i)
      for (int j = 0; j < d2; ++j) {
        const cd v = t[(static_cast<size_t>(i) * d2 + j) * d3 + k];
        if (std::abs(v.imag()) > 1e-12) throw std::runtime_error("cg_block: imaginary residue");
        if (std::abs(v.real()) > 1e-12) b.entries.push_back({i, j, k, v.real()});
      }
  std::vector<double> nrm(d3, 0.0);
  for (const auto& e : b.entries) nrm[e.k] += e.v * e.v;
  for (auto& e : b.entries)
    if (nrm[e.k] > 0.0) e.v /= std::sqrt(nrm[e.k]);
  return b;
}

}  // namespace

std::shared_ptr<const CGBlock> cg_block(int l1, int l2, int l3) {
  if (l1 < 0 || l2 < 0 || l3 < 0) throw std::invalid_argument("cg_block: negative l");
  if (l3 < std::abs(l1 - l2) || l3 > l1 + l2)
    throw TriangleError("cg_block: triangle rule violated for (" + std::to_string(l1) + "," +
                        std::to_string(l2) + "," + std::to_string(l3) + ")");
  if (l1 + l2 + l3 + 1 > 33) throw UnsupportedError("cg_block: l1+l2+l3 too large");
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, std::shared_ptr<const CGBlock>> memo;
  std::lock_guard<std::mutex> g(mu);
  auto& slot = memo[{l1, l2, l3}];
  if (!slot) slot = std::make_shared<const CGBlock>(build(l1, l2, l3));
  return slot;
}

// ================================================================ tpspec ==
std::uint64_t Sub::fwd_flops() const {
  const std::uint64_t nnz = cg->entries.size();
  std::uint64_t f = 3ull * bp * nnz;
  f += kind == Kind::B ? 2ull * b * dz() : 2ull * b * bp * dz();
  return f;
}

std::uint64_t Sub::bwd_flops() const {
  const std::uint64_t nnz = cg->entries.size();
  const std::uint64_t mm = kind == Kind::B ? 2ull * b * dz() : 2ull * b * bp * dz();
  return mm + 9ull * bp * nnz + (bp > 1 ? std::uint64_t(dy()) * (bp - 1) : 0) + mm;
}

std::uint64_t Problem::fwd_flops_per_row() const {
  std::uint64_t f = 0;
  for (const auto& s : subs) f += s.fwd_flops();
  return f;
}
std::uint64_t Problem::bwd_flops_per_row() const {
  std::uint64_t f = 0;
  for (const auto& s : subs) f += s.bwd_flops();
  return f;
}

Problem make_problem(const Irreps& x, const Irreps& y, const Irreps& z,
                     const std::vector<Instruction>& ins, int lane_width) {
  if (lane_width <= 0) throw std::invalid_argument("lane_width <= 0");
  Problem p;
  p.x_ir = x;
  p.y_ir = y;
  p.z_ir = z;
  p.instructions = ins;
  p.dim_x = x.dim();
  p.dim_y = y.dim();
  p.dim_z = z.dim();
  p.lane_width = lane_width;
  std::vector<std::string> viol;
  auto flag = [&](size_t n, const std::string& m) {
    viol.push_back("instruction " + std::to_string(n) + ": " + m);
  };
  std::uint32_t w_off = 0;
  for (size_t n = 0; n < ins.size(); ++n) {
    const auto& in = ins[n];
    bool ok = true;
    if (in.x_seg < 1 || in.x_seg > int(x.blocks.size())) { flag(n, "x segment index " + std::to_string(in.x_seg) + " out of range"); ok = false; }
    if (in.y_seg < 1 || in.y_seg > int(y.blocks.size())) { flag(n, "y segment index " + std::to_string(in.y_seg) + " out of range"); ok = false; }
    if (in.z_seg < 1 || in.z_seg > int(z.blocks.size())) { flag(n, "z segment index " + std::to_string(in.z_seg) + " out of range"); ok = false; }
    if (!ok) continue;
    const auto &bx = x.blocks[in.x_seg - 1], &by = y.blocks[in.y_seg - 1], &bz = z.blocks[in.z_seg - 1];
    if (by.mult != 1) flag(n, "y segment multiplicity must be 1 (unsupported pattern), got " + std::to_string(by.mult));
    if (in.kind == Kind::B && bx.mult != bz.mult)
      flag(n, "kind B requires mult(x_seg) == mult(z_seg), got " + std::to_string(bx.mult) + " vs " + std::to_string(bz.mult));
    if (bz.l < std::abs(bx.l - by.l) || bz.l > bx.l + by.l)
      flag(n, "triangle rule violated: (" + std::to_string(bx.l) + "," + std::to_string(by.l) + "," + std::to_string(bz.l) + ")");
    if ((bx.odd != by.odd) != bz.odd) flag(n, "parity rule violated: p_x * p_y != p_z");
    Sub s;
    s.kind = in.kind;
    s.l1 = bx.l;
    s.l2 = by.l;
    s.l3 = bz.l;
    s.b = bz.mult;
    s.bp = bx.mult;
    s.x_off = x.offset(in.x_seg - 1);
    s.y_off = y.offset(in.y_seg - 1);
    s.z_off = z.offset(in.z_seg - 1);
    s.w_off = w_off;
    s.w_stride = in.kind == Kind::B ? 1 : bx.mult;
    s.origin = static_cast<int>(n);
    w_off += in.kind == Kind::B ? s.b : s.b * s.bp;
    p.resolved.push_back(s);
  }
  p.n_w = w_off;
  if (!viol.empty()) {
    std::string m;
    for (const auto& v : viol) m += (m.empty() ? "" : "; ") + v;
    throw ValidationError(m);
  }
  for (auto& s : p.resolved) s.cg = cg_block(s.l1, s.l2, s.l3);
  // Split (scheduler.cpp:32-81): B chunks x and z lanes together; C chunks z
  // rows outer, x columns inner, keeping the original W row stride.
  std::vector<Sub> split;
  for (const auto& r : p.resolved) {
    if (r.kind == Kind::B) {
      for (int c0 = 0; c0 < r.b; c0 += lane_width) {
        Sub s = r;
        s.b = s.bp = std::min(lane_width, r.b - c0);
        s.x_off = r.x_off + c0 * r.dx();
        s.z_off = r.z_off + c0 * r.dz();
        s.w_off = r.w_off + c0;
        split.push_back(s);
      }
    } else {
      for (int r0 = 0; r0 < r.b; r0 += lane_width)
        for (int c0 = 0; c0 < r.bp; c0 += lane_width) {
          Sub s = r;
          s.b = std::min(lane_width, r.b - r0);
          s.bp = std::min(lane_width, r.bp - c0);
          s.x_off = r.x_off + c0 * r.dx();
          s.z_off = r.z_off + r0 * r.dz();
          s.w_off = r.w_off + r0 * r.w_stride + c0;
          split.push_back(s);
        }
    }
  }
  for (size_t i = 0; i < split.size(); ++i) split[i].split_index = static_cast<int>(i);
  std::stable_sort(split.begin(), split.end(),
                   [](const Sub& a, const Sub& b) { return a.z_off < b.z_off; });
  p.subs = std::move(split);
  return p;
}

// ------------------------------------------------------------ tiny JSON --
namespace {

struct JVal {
  enum T { Null, Num, Str, Arr, Obj, Bool } t = Null;
  double num = 0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal& at(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw ParseError("problem JSON: missing key \"" + k + "\"");
  }
};

struct JParser {
  const std::string& s;
  size_t i = 0;
  void ws() { while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i; }
  [[noreturn]] void fail(const char* m) { throw ParseError(std::string("problem JSON: ") + m + " at offset " + std::to_string(i)); }
  JVal value() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    JVal v;
    const char c = s[i];
    if (c == '{') {
      v.t = JVal::Obj;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') { ++i; return v; }
      for (;;) {
        ws();
        if (i >= s.size() || s[i] != '"') fail("expected key");
        std::string k = string();
        ws();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        v.obj.emplace_back(k, value());
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == '}') { ++i; break; }
        fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.t = JVal::Arr;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') { ++i; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i < s.size() && s[i] == ',') { ++i; continue; }
        if (i < s.size() && s[i] == ']') { ++i; break; }
        fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.t = JVal::Str;
      v.str = string();
    } else if (c == 't' || c == 'f' || c == 'n') {
      const char* w = c == 't' ? "true" : c == 'f' ? "false" : "null";
      if (s.compare(i, std::strlen(w), w) != 0) fail("bad literal");
      i += std::strlen(w);
      v.t = c == 'n' ? JVal::Null : JVal::Bool;
      v.num = c == 't';
    } else {
      size_t used = 0;
      try {
        v.num = std::stod(s.substr(i), &used);
      } catch (...) {
        fail("bad number");
      }
      i += used;
      v.t = JVal::Num;
    }
    return v;
  }
  std::string string() {
    std::string out;
    ++i;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\' && i + 1 < s.size()) ++i;
      out += s[i++];
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
};

}  // namespace

Problem parse_problem_json(const std::string& text, int lane_width) {
  JParser jp{text};
  const JVal root = jp.value();
  if (root.t != JVal::Obj) throw ParseError("problem JSON: expected an object");
  auto str = [](const JVal& v, const char* what) {
    if (v.t != JVal::Str) throw ParseError(std::string("problem JSON: \"") + what + "\" must be a string");
    return v.str;
  };
  const Irreps x = parse_irreps(str(root.at("x"), "x"));
  const Irreps y = parse_irreps(str(root.at("y"), "y"));
  const Irreps z = parse_irreps(str(root.at("z"), "z"));
  const JVal& ia = root.at("instructions");
  if (ia.t != JVal::Arr) throw ParseError("problem JSON: \"instructions\" must be an array");
  std::vector<Instruction> ins;
  for (const auto& t : ia.arr) {
    if (t.t != JVal::Arr || t.arr.size() != 4 || t.arr[0].t != JVal::Num || t.arr[1].t != JVal::Num ||
        t.arr[2].t != JVal::Num || t.arr[3].t != JVal::Str)
      throw ParseError("instruction must be [x_seg, y_seg, z_seg, \"B\"|\"C\"]");
    Instruction in;
    in.x_seg = static_cast<int>(t.arr[0].num);
    in.y_seg = static_cast<int>(t.arr[1].num);
    in.z_seg = static_cast<int>(t.arr[2].num);
    if (t.arr[3].str == "B") in.kind = Kind::B;
    else if (t.arr[3].str == "C") in.kind = Kind::C;
    else throw ParseError("instruction kind must be \"B\" or \"C\", got \"" + t.arr[3].str + "\"");
    ins.push_back(in);
  }
  return make_problem(x, y, z, ins, lane_width);
}

// ========================================================== unit planning ==
int Unit::x_chunk_of(const Sub& s) const {
  for (size_t k = 0; k < x_chunks.size(); ++k)
    if (x_chunks[k].off == s.x_off) return static_cast<int>(k);
  return -1;
}
int Unit::z_piece_of(const Sub& s) const {
  for (size_t k = 0; k < z_pieces.size(); ++k)
    if (z_pieces[k].off == s.z_off) return static_cast<int>(k);
  return -1;
}

std::vector<Unit> plan_units(const Problem& p) {
  const int n = static_cast<int>(p.subs.size());
  std::vector<int> parent(n);
  std::iota(parent.begin(), parent.end(), 0);
  std::function<int(int)> find = [&](int a) { return parent[a] == a ? a : parent[a] = find(parent[a]); };
  std::map<std::uint32_t, int> by_x, by_z;
  for (int s = 0; s < n; ++s) {
    for (auto* m : {&by_x, &by_z}) {
      const std::uint32_t key = m == &by_x ? p.subs[s].x_off : p.subs[s].z_off;
      auto it = m->find(key);
      if (it == m->end()) m->emplace(key, s);
      else parent[find(s)] = find(it->second);
    }
  }
  std::map<int, int> unit_of_root;  // ordered by first subkernel (schedule order)
  std::vector<Unit> units;
  for (int s = 0; s < n; ++s) {
    const int r = find(s);
    auto it = unit_of_root.find(r);
    if (it == unit_of_root.end()) {
      it = unit_of_root.emplace(r, static_cast<int>(units.size())).first;
      units.emplace_back();
    }
    Unit& u = units[it->second];
    u.subs.push_back(s);
    const Sub& sb = p.subs[s];
    if (u.x_chunk_of(sb) < 0) u.x_chunks.push_back({sb.x_off, static_cast<std::uint32_t>(sb.bp * sb.dx())});
    if (u.z_piece_of(sb) < 0) u.z_pieces.push_back({sb.z_off, static_cast<std::uint32_t>(sb.b * sb.dz())});
  }
  return units;
}

}  // namespace cgf
