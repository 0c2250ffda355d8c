#include "codegen.hpp"

#include <algorithm>
#include <cstdio>
#include <map>
#include <sstream>

namespace cgf {

const char* device_runtime_source() {
  return R"RT(
typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;
#define DEVI __device__ __forceinline__

DEVI u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
DEVI void mbar_init(u64* b, u32 n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(b)), "r"(n) : "memory");
}
DEVI void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
DEVI void mbar_expect_tx(u64* b, u32 bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}"
               :: "r"(smem_addr(b)), "r"(bytes) : "memory");
}
DEVI bool mbar_try(u64* b, u32 parity) {
  u32 ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_addr(b)), "r"(parity) : "memory");
  return ok != 0;
}
DEVI void mbar_wait(u64* b, u32 parity) { while (!mbar_try(b, parity)) { } }
DEVI void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier (bytes).
DEVI void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
template <class T> DEVI void coop_load(T* dst, const T* __restrict__ src, int n, int lane) {
  for (int i = lane; i < n; i += 32) dst[i] = __ldg(src + i);
}
template <class T> DEVI void coop_store(T* __restrict__ dst, const T* src, int n, int lane) {
  for (int i = lane; i < n; i += 32) dst[i] = src[i];
}
// 16-byte vector stores, streaming (evict-first) — outputs are written once.
DEVI void coop_store16(void* dst, const void* src, int n16, int lane) {
  const float4* s = (const float4*)src;
  float4* d = (float4*)dst;
  for (int i = lane; i < n16; i += 32) __stcs(d + i, s[i]);
}
template <class T> DEVI T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
)RT";
}

namespace {

std::string hexd(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}

struct SlotRange {
  std::string arr;  // kernel parameter name
  std::string stride;  // row stride expression (words)
  std::uint32_t off = 0, words = 0, slot_off = 0;
  bool bulk = false;
};

struct UnitLayout {
  std::vector<SlotRange> ranges;
  std::map<std::uint32_t, std::uint32_t> x_slot, a_slot, gz_slot;  // row offset -> slot offset
  std::map<int, std::uint32_t> w_slot, c_slot;                      // sub index -> slot offset
  std::uint32_t words = 0, bulk_bytes = 0;
};

class Gen {
 public:
  Gen(const Problem& p, const std::vector<Unit>& units, const KernelConfig& cfg)
      : p_(p), units_(units), cfg_(cfg), sz_(cfg.f64 ? 8 : 4) {}

  KernelSource run();

 private:
  const Problem& p_;
  const std::vector<Unit>& units_;
  KernelConfig cfg_;
  int sz_;
  std::ostringstream o_;
  std::vector<UnitLayout> lay_;
  int max_dz_ = 1, max_dx_ = 1, max_piece_ = 1;
  bool has_c_ = false;
  std::uint32_t scr_words_ = 0, off_zs_ = 0, off_wt_ = 0, off_ct_ = 0;

  bool bwd() const { return cfg_.op != Op::Fwd; }
  bool dbl() const { return cfg_.op == Op::DBwd; }
  std::uint32_t align_words() const { return 16u / sz_; }
  std::uint32_t up(std::uint32_t w) const { return (w + align_words() - 1) / align_words() * align_words(); }
  bool aligned16(std::uint64_t words) const { return (words * sz_) % 16 == 0; }

  void layout();
  void add_range(UnitLayout& L, const std::string& arr, std::uint32_t stride, std::uint32_t off,
                 std::uint32_t words, std::uint32_t& slot_off);
  void emit_issue();
  void emit_unit(int u);
  void emit_store(const std::string& dst, std::uint32_t stride, std::uint32_t off,
                  std::uint32_t words, const std::string& guard_rows, int width,
                  const std::string& reg);
  std::string wsrc(const Sub& s, const std::string& arr) const;
};

void Gen::add_range(UnitLayout& L, const std::string& arr, std::uint32_t stride, std::uint32_t off,
                    std::uint32_t words, std::uint32_t& slot_off) {
  SlotRange r;
  r.arr = arr;
  r.stride = std::to_string(stride);
  r.off = off;
  r.words = words;
  r.slot_off = L.words;
  r.bulk = cfg_.aligned && aligned16(stride) && aligned16(off) && aligned16(words);
  slot_off = r.slot_off;
  L.words = up(L.words + words);
  if (r.bulk) L.bulk_bytes += words * sz_;
  L.ranges.push_back(r);
}

void Gen::layout() {
  for (const auto& s : p_.subs) {
    max_dz_ = std::max(max_dz_, s.dz());
    max_dx_ = std::max(max_dx_, s.dx());
    max_piece_ = std::max({max_piece_, s.b * s.dz(), s.bp * s.dx()});
    if (s.kind == Kind::C) has_c_ = true;
  }
  for (const auto& u : units_) {
    UnitLayout L;
    std::uint32_t so = 0;
    for (const auto& xc : u.x_chunks) {
      add_range(L, "X", p_.dim_x, xc.off, xc.words, so);
      L.x_slot[xc.off] = so;
      if (dbl()) {
        add_range(L, "DA", p_.dim_x, xc.off, xc.words, so);
        L.a_slot[xc.off] = so;
      }
    }
    if (!cfg_.w_shared) {
      for (int si : u.subs) {
        const Sub& s = p_.subs[si];
        if (s.kind != Kind::B) continue;
        add_range(L, "W", p_.n_w, s.w_off, s.b, so);
        L.w_slot[si] = so;
        if (dbl()) {
          add_range(L, "DC", p_.n_w, s.w_off, s.b, so);
          L.c_slot[si] = so;
        }
      }
    }
    if (bwd()) {
      for (const auto& zp : u.z_pieces) {
        add_range(L, "GZ", p_.dim_z, zp.off, zp.words, so);
        L.gz_slot[zp.off] = so;
      }
    }
    L.words = std::max<std::uint32_t>(L.words, align_words());
    lay_.push_back(std::move(L));
  }
  // Per-warp scratch: output staging, plus z' staging and W / dC tiles for uvw.
  const std::uint32_t stage = up(static_cast<std::uint32_t>(std::max(max_piece_, 32 * max_dx_)));
  scr_words_ = stage;
  off_zs_ = scr_words_;
  if (has_c_) {
    scr_words_ += up(2u * 32u * max_dz_);
    off_wt_ = scr_words_;
    scr_words_ += up(32u * 33u);
    off_ct_ = scr_words_;
    if (dbl()) scr_words_ += up(32u * 33u);
  }
}

std::string Gen::wsrc(const Sub& s, const std::string& arr) const {
  // Global base of this subkernel's weight tile for the current row.
  if (cfg_.w_shared) return "(" + arr + " + " + std::to_string(s.w_off) + ")";
  return "(" + arr + " + row * (i64)" + std::to_string(p_.n_w) + " + " + std::to_string(s.w_off) + ")";
}

void Gen::emit_issue() {
  o_ << "DEVI void issue_unit(int u, i64 row, T* sl, u64* bar, const T* __restrict__ X,"
        " const T* __restrict__ W, const T* __restrict__ GZ, const T* __restrict__ DA,"
        " const T* __restrict__ DC) {\n"
        "  fence_proxy_async();\n  switch (u) {\n";
  for (size_t u = 0; u < lay_.size(); ++u) {
    const auto& L = lay_[u];
    o_ << "  case " << u << ":\n    mbar_expect_tx(bar, " << L.bulk_bytes << "u);\n";
    for (const auto& r : L.ranges)
      if (r.bulk)
        o_ << "    bulk_g2s(sl + " << r.slot_off << ", " << r.arr << " + row * (i64)" << r.stride
           << " + " << r.off << ", " << r.words * sz_ << "u, bar);\n";
    o_ << "    break;\n";
  }
  o_ << "  default: break;\n  }\n}\n\n";
}

void Gen::emit_store(const std::string& dst, std::uint32_t stride, std::uint32_t off,
                     std::uint32_t words, const std::string& guard_rows, int width,
                     const std::string& reg) {
  // Lane r owns `width` consecutive words of the piece; stage through smem so
  // the global store is coalesced (and 16-byte vectorised when aligned).
  o_ << "      if (lane < " << guard_rows << ") {";
  for (int k = 0; k < width; ++k) o_ << " scr[lane * " << width << " + " << k << "] = " << reg << "[" << k << "];";
  o_ << " }\n      __syncwarp();\n";
  const bool vec = cfg_.aligned && aligned16(stride) && aligned16(off) && aligned16(words);
  if (vec)
    o_ << "      coop_store16(" << dst << " + row * (i64)" << stride << " + " << off << ", scr, "
       << words * sz_ / 16 << ", lane);\n";
  else
    o_ << "      coop_store(" << dst << " + row * (i64)" << stride << " + " << off << ", scr, " << words
       << ", lane);\n";
  o_ << "      __syncwarp();\n";
}

void Gen::emit_unit(int ui) {
  const Unit& u = units_[ui];
  const UnitLayout& L = lay_[ui];
  o_ << "    { // ---- unit " << ui << ": " << u.subs.size() << " subkernels\n";
  o_ << "      T* sl = wsm + slot * " << "SLOT_WORDS;\n";
  o_ << "      mbar_wait(&bars[slot], phase);\n";
  bool any_sync = false;
  for (const auto& r : L.ranges)
    if (!r.bulk) {
      o_ << "      coop_load(sl + " << r.slot_off << ", " << r.arr << " + row * (i64)" << r.stride << " + "
         << r.off << ", " << r.words << ", lane);\n";
      any_sync = true;
    }
  if (any_sync) o_ << "      __syncwarp();\n";

  // Output accumulators: per x chunk (gx / dx) and per z piece (z / dgz).
  std::map<std::uint32_t, int> xdx, zdz;
  std::map<std::uint32_t, int> xb, zb;
  for (int si : u.subs) {
    const Sub& s = p_.subs[si];
    xdx[s.x_off] = s.dx();
    xb[s.x_off] = s.bp;
    zdz[s.z_off] = s.dz();
    zb[s.z_off] = s.b;
  }
  if (bwd())
    for (size_t c = 0; c < u.x_chunks.size(); ++c)
      o_ << "      T gx" << c << "[" << xdx[u.x_chunks[c].off] << "] = {};\n";
  if (cfg_.op != Op::Bwd)
    for (size_t z = 0; z < u.z_pieces.size(); ++z)
      o_ << "      T pz" << z << "[" << zdz[u.z_pieces[z].off] << "] = {};\n";

  for (int si : u.subs) {
    const Sub& s = p_.subs[si];
    const int dx = s.dx(), dz = s.dz();
    const int xc = u.x_chunk_of(s), zc = u.z_piece_of(s);
    const std::uint32_t xs = L.x_slot.at(s.x_off);
    o_ << "      { // sub " << si << ": " << (s.kind == Kind::B ? "B" : "C") << " l=(" << s.l1 << ","
       << s.l2 << "," << s.l3 << ") b=" << s.b << " b'=" << s.bp << " nnz=" << s.cg->entries.size()
       << "\n";
    // x (and da) lanes t < b'
    o_ << "        T xv[" << dx << "];";
    if (dbl()) o_ << " T av[" << dx << "];";
    o_ << "\n        if (lane < " << s.bp << ") {";
    for (int i = 0; i < dx; ++i) o_ << " xv[" << i << "] = sl[" << xs << " + lane * " << dx << " + " << i << "];";
    if (dbl())
      for (int i = 0; i < dx; ++i)
        o_ << " av[" << i << "] = sl[" << L.a_slot.at(s.x_off) << " + lane * " << dx << " + " << i << "];";
    o_ << " } else {";
    for (int i = 0; i < dx; ++i) o_ << " xv[" << i << "] = 0;";
    if (dbl())
      for (int i = 0; i < dx; ++i) o_ << " av[" << i << "] = 0;";
    o_ << " }\n";
    // gz (lanes t < b), uniform access for C
    std::string gzs;
    if (bwd()) {
      gzs = std::to_string(L.gz_slot.at(s.z_off));
      if (s.kind == Kind::B) {
        o_ << "        T gz[" << dz << "];\n        if (lane < " << s.b << ") {";
        for (int k = 0; k < dz; ++k) o_ << " gz[" << k << "] = sl[" << gzs << " + lane * " << dz << " + " << k << "];";
        o_ << " } else {";
        for (int k = 0; k < dz; ++k) o_ << " gz[" << k << "] = 0;";
        o_ << " }\n";
      }
    }
    // weights for B: per lane scalar
    if (s.kind == Kind::B) {
      auto wexpr = [&](const std::string& arr, const std::map<int, std::uint32_t>& slot) {
        if (cfg_.w_shared) return "__ldg(" + wsrc(s, arr) + " + lane)";
        return "sl[" + std::to_string(slot.at(si)) + " + lane]";
      };
      o_ << "        const T wt = (lane < " << s.b << ") ? " << wexpr("W", L.w_slot) << " : (T)0;\n";
      if (dbl()) o_ << "        const T ct = (lane < " << s.b << ") ? " << wexpr("DC", L.c_slot) << " : (T)0;\n";
    }
    // W^T g_z (bwd): gzp (and gzc for dbl: dC^T g_z)
    if (bwd()) {
      o_ << "        T gzp[" << dz << "];";
      if (dbl()) o_ << " T gzc[" << dz << "];";
      o_ << "\n";
      if (s.kind == Kind::B) {
        for (int k = 0; k < dz; ++k) {
          o_ << "        gzp[" << k << "] = wt * gz[" << k << "];";
          if (dbl()) o_ << " gzc[" << k << "] = ct * gz[" << k << "];";
          o_ << "\n";
        }
      } else {
        o_ << "        {";
        for (int k = 0; k < dz; ++k) {
          o_ << " gzp[" << k << "] = 0;";
          if (dbl()) o_ << " gzc[" << k << "] = 0;";
        }
        o_ << "\n          const T* wg = " << wsrc(s, "W") << ";\n";
        if (dbl()) o_ << "          const T* cg = " << wsrc(s, "DC") << ";\n";
        o_ << "#pragma unroll 2\n          for (int r = 0; r < " << s.b << "; ++r) {\n"
           << "            const T wv = (lane < " << s.bp << ") ? __ldg(wg + r * " << s.w_stride << " + lane) : (T)0;\n";
        if (dbl())
          o_ << "            const T cv = (lane < " << s.bp << ") ? __ldg(cg + r * " << s.w_stride << " + lane) : (T)0;\n";
        for (int k = 0; k < dz; ++k) {
          o_ << "            { const T g = sl[" << gzs << " + r * " << dz << " + " << k << "]; gzp[" << k
             << "] = fma(wv, g, gzp[" << k << "]);";
          if (dbl()) o_ << " gzc[" << k << "] = fma(cv, g, gzc[" << k << "]);";
          o_ << " }\n";
        }
        o_ << "          }\n        }\n";
      }
    }
    // The unrolled CG stream: one line per nonzero entry.
    if (cfg_.op == Op::Fwd) {
      o_ << "        T zp[" << dz << "] = {};\n";
      for (const auto& e : s.cg->entries)
        o_ << "        zp[" << e.k << "] = fma((T)" << hexd(e.v) << " * y[" << s.y_off + e.j << "], xv[" << e.i
           << "], zp[" << e.k << "]);\n";
    } else if (cfg_.op == Op::Bwd) {
      o_ << "        T zp[" << dz << "] = {};\n";
      for (const auto& e : s.cg->entries) {
        const std::string v = "(T)" + hexd(e.v);
        const std::string yj = "y[" + std::to_string(s.y_off + e.j) + "]";
        o_ << "        { const T c = " << v << " * " << yj << "; gx" << xc << "[" << e.i << "] = fma(c, gzp["
           << e.k << "], gx" << xc << "[" << e.i << "]); zp[" << e.k << "] = fma(c, xv[" << e.i << "], zp["
           << e.k << "]); gy[" << s.y_off + e.j << "] = fma(" << v << " * xv[" << e.i << "], gzp[" << e.k
           << "], gy[" << s.y_off + e.j << "]); }\n";
      }
    } else {
      o_ << "        T zx[" << dz << "] = {}; T za[" << dz << "] = {}; T zb[" << dz << "] = {};\n";
      for (const auto& e : s.cg->entries) {
        const std::string v = "(T)" + hexd(e.v);
        const std::string J = std::to_string(s.y_off + e.j), I = std::to_string(e.i), K = std::to_string(e.k);
        const std::string X = std::to_string(xc);
        o_ << "        { const T cy = " << v << " * y[" << J << "]; const T cb = " << v << " * db[" << J
           << "];\n"
           << "          gx" << X << "[" << I << "] = fma(cb, gzp[" << K << "], fma(cy, gzc[" << K << "], gx" << X
           << "[" << I << "]));\n"
           << "          gy[" << J << "] = fma(" << v << " * av[" << I << "], gzp[" << K << "], fma(" << v
           << " * xv[" << I << "], gzc[" << K << "], gy[" << J << "]));\n"
           << "          zx[" << K << "] = fma(cy, xv[" << I << "], zx[" << K << "]); za[" << K
           << "] = fma(cy, av[" << I << "], za[" << K << "]); zb[" << K << "] = fma(cb, xv[" << I << "], zb[" << K
           << "]); }\n";
      }
    }
    // Weight application / weight gradients.
    const std::string nw = std::to_string(p_.n_w);
    if (cfg_.op == Op::Fwd) {
      if (s.kind == Kind::B) {
        for (int k = 0; k < dz; ++k) o_ << "        pz" << zc << "[" << k << "] = fma(wt, zp[" << k << "], pz" << zc << "[" << k << "]);\n";
      } else {
        o_ << "        if (lane < " << s.bp << ") {";
        for (int k = 0; k < dz; ++k) o_ << " zs[lane * " << dz << " + " << k << "] = zp[" << k << "];";
        o_ << " }\n        { const T* wg = " << wsrc(s, "W") << ";\n"
           << "#pragma unroll 4\n          for (int r = 0; r < " << s.b << "; ++r) if (lane < " << s.bp
           << ") wts[r * 33 + lane] = __ldg(wg + r * " << s.w_stride << " + lane); }\n"
           << "        __syncwarp();\n        if (lane < " << s.b << ") {\n#pragma unroll 4\n"
           << "          for (int c = 0; c < " << s.bp << "; ++c) { const T wv = wts[lane * 33 + c];";
        for (int k = 0; k < dz; ++k) o_ << " pz" << zc << "[" << k << "] = fma(wv, zs[c * " << dz << " + " << k << "], pz" << zc << "[" << k << "]);";
        o_ << " }\n        }\n        __syncwarp();\n";
      }
    } else if (cfg_.op == Op::Bwd) {
      if (s.kind == Kind::B) {
        o_ << "        { T g = 0;";
        for (int k = 0; k < dz; ++k) o_ << " g = fma(gz[" << k << "], zp[" << k << "], g);";
        o_ << " if (lane < " << s.b << ") O2[row * (i64)" << nw << " + " << s.w_off << " + lane] = g; }\n";
      } else {
        o_ << "#pragma unroll 2\n        for (int r = 0; r < " << s.b << "; ++r) { T g = 0;";
        for (int k = 0; k < dz; ++k) o_ << " g = fma(sl[" << gzs << " + r * " << dz << " + " << k << "], zp[" << k << "], g);";
        o_ << " if (lane < " << s.bp << ") O2[row * (i64)" << nw << " + " << s.w_off << " + r * " << s.w_stride
           << " + lane] = g; }\n";
      }
    } else {  // DBwd
      if (s.kind == Kind::B) {
        for (int k = 0; k < dz; ++k)
          o_ << "        pz" << zc << "[" << k << "] = fma(ct, zx[" << k << "], fma(wt, za[" << k << "] + zb[" << k
             << "], pz" << zc << "[" << k << "]));\n";
        o_ << "        { T g = 0;";
        for (int k = 0; k < dz; ++k) o_ << " g = fma(gz[" << k << "], za[" << k << "] + zb[" << k << "], g);";
        o_ << " if (lane < " << s.b << ") O2[row * (i64)" << nw << " + " << s.w_off << " + lane] = g; }\n";
      } else {
        o_ << "        if (lane < " << s.bp << ") {";
        for (int k = 0; k < dz; ++k)
          o_ << " zs[lane * " << dz << " + " << k << "] = za[" << k << "] + zb[" << k << "]; zs[" << 32 * dz
             << " + lane * " << dz << " + " << k << "] = zx[" << k << "];";
        o_ << " }\n        { const T* wg = " << wsrc(s, "W") << "; const T* cg = " << wsrc(s, "DC") << ";\n"
           << "#pragma unroll 4\n          for (int r = 0; r < " << s.b << "; ++r) if (lane < " << s.bp
           << ") { wts[r * 33 + lane] = __ldg(wg + r * " << s.w_stride << " + lane); cts[r * 33 + lane] = __ldg(cg + r * "
           << s.w_stride << " + lane); } }\n"
           << "        __syncwarp();\n        if (lane < " << s.b << ") {\n#pragma unroll 4\n"
           << "          for (int c = 0; c < " << s.bp << "; ++c) { const T wv = wts[lane * 33 + c]; const T cv = cts[lane * 33 + c];";
        for (int k = 0; k < dz; ++k)
          o_ << " pz" << zc << "[" << k << "] = fma(cv, zs[" << 32 * dz << " + c * " << dz << " + " << k
             << "], fma(wv, zs[c * " << dz << " + " << k << "], pz" << zc << "[" << k << "]));";
        o_ << " }\n        }\n        __syncwarp();\n";
        o_ << "#pragma unroll 2\n        for (int r = 0; r < " << s.b << "; ++r) { T g = 0;";
        for (int k = 0; k < dz; ++k)
          o_ << " g = fma(sl[" << gzs << " + r * " << dz << " + " << k << "], za[" << k << "] + zb[" << k << "], g);";
        o_ << " if (lane < " << s.bp << ") O2[row * (i64)" << nw << " + " << s.w_off << " + r * " << s.w_stride
           << " + lane] = g; }\n";
      }
    }
    o_ << "      }\n";
  }
  // Stores of owned outputs.
  if (bwd())
    for (size_t c = 0; c < u.x_chunks.size(); ++c) {
      const auto& xc = u.x_chunks[c];
      emit_store("O0", p_.dim_x, xc.off, xc.words, std::to_string(xb[xc.off]), xdx[xc.off], "gx" + std::to_string(c));
    }
  if (cfg_.op != Op::Bwd)
    for (size_t z = 0; z < u.z_pieces.size(); ++z) {
      const auto& zp = u.z_pieces[z];
      emit_store(cfg_.op == Op::Fwd ? "O0" : "O3", p_.dim_z, zp.off, zp.words, std::to_string(zb[zp.off]),
                 zdz[zp.off], "pz" + std::to_string(z));
    }
  // Release the slot: refill it with unit n + D.
  o_ << "      if (lane == 0 && n + D < total) {\n"
        "        const i64 m = n + D; const i64 rr2 = m / NU; const int u2 = (int)(m - rr2 * NU);\n"
        "        issue_unit(u2, gwarp + rr2 * nwarp, sl, &bars[slot], X, W, GZ, DA, DC);\n      }\n"
        "      ++n; if (++slot == D) { slot = 0; phase ^= 1u; }\n    }\n";
}

KernelSource Gen::run() {
  layout();
  std::uint32_t slot_words = 0;
  int bulk = 0, sync = 0;
  for (const auto& L : lay_) {
    slot_words = std::max(slot_words, L.words);
    for (const auto& r : L.ranges) (r.bulk ? bulk : sync)++;
  }
  // Fit the ring into shared memory: shrink depth, then warps.
  int depth = cfg_.depth, warps = cfg_.warps;
  auto warp_bytes = [&](int d) { return (static_cast<std::uint64_t>(d) * slot_words + scr_words_) * sz_; };
  const std::uint64_t budget = 200 * 1024;
  while (depth > 1 && warp_bytes(depth) * warps + 8ull * depth * warps > budget) --depth;
  while (warps > 1 && warp_bytes(depth) * warps + 8ull * depth * warps > budget) --warps;
  if (warp_bytes(depth) * warps + 8ull * depth * warps > 227 * 1024)
    throw UnsupportedError("problem too large for one warp's shared-memory slot (" +
                           std::to_string(warp_bytes(1)) + " bytes)");
  const std::uint64_t wb = (warp_bytes(depth) + 127) / 128 * 128;
  const char* opn[] = {"fwd", "bwd", "dbwd"};
  KernelSource ks;
  ks.name = std::string("cgf_tp_") + opn[static_cast<int>(cfg_.op)] + (cfg_.f64 ? "_f64" : "_f32") +
            (cfg_.w_shared ? "_ws" : "") + (cfg_.aligned ? "" : "_u");
  ks.threads = warps * 32;
  ks.smem_bytes = static_cast<int>(wb * warps + 8ull * depth * warps);
  ks.units = static_cast<int>(units_.size());
  ks.bulk_ranges = bulk;
  ks.sync_ranges = sync;

  o_ << device_runtime_source();
  o_ << "\n// Generated for: x = " << p_.x_ir.str() << " | y = " << p_.y_ir.str() << " | z = " << p_.z_ir.str()
     << "\n// " << p_.subs.size() << " split subkernels in " << units_.size() << " units; op " << opn[static_cast<int>(cfg_.op)]
     << "\n";
  o_ << "typedef " << (cfg_.f64 ? "double" : "float") << " T;\n";
  o_ << "#define NW " << warps << "\n#define D " << depth << "\n#define NU " << units_.size()
     << "\n#define SLOT_WORDS " << slot_words << "\n#define WARP_BYTES " << wb << "\n\n";
  emit_issue();
  o_ << "extern \"C\" __global__ void __launch_bounds__(NW * 32) " << ks.name
     << "(const T* __restrict__ X, const T* __restrict__ Y, const T* __restrict__ W,"
        " const T* __restrict__ GZ, const T* __restrict__ DA, const T* __restrict__ DB,"
        " const T* __restrict__ DC, T* __restrict__ O0, T* __restrict__ O1, T* __restrict__ O2,"
        " T* __restrict__ O3, i64 rows) {\n"
        "  extern __shared__ __align__(128) unsigned char smem_raw[];\n"
        "  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;\n"
        "  T* wsm = (T*)(smem_raw + wid * WARP_BYTES);\n"
        "  T* scr = wsm + D * SLOT_WORDS;\n";
  if (has_c_)
    o_ << "  T* zs = scr + " << off_zs_ << "; T* wts = scr + " << off_wt_ << ";" << (dbl() ? " T* cts = scr + " + std::to_string(off_ct_) + ";" : "")
       << "\n";
  o_ << "  u64* bars = (u64*)(smem_raw + NW * WARP_BYTES) + wid * D;\n"
        "  if (lane == 0) { for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1); mbar_fence_init(); }\n"
        "  __syncwarp();\n"
        "  const i64 gwarp = (i64)blockIdx.x * NW + wid, nwarp = (i64)gridDim.x * NW;\n"
        "  const i64 my_rows = gwarp < rows ? (rows - 1 - gwarp) / nwarp + 1 : 0;\n"
        "  const i64 total = my_rows * NU;\n"
        "  if (lane == 0)\n"
        "    for (int d = 0; d < D && d < total; ++d) {\n"
        "      const i64 rr = d / NU; const int u = (int)(d - rr * NU);\n"
        "      issue_unit(u, gwarp + rr * nwarp, wsm + d * SLOT_WORDS, &bars[d], X, W, GZ, DA, DC);\n"
        "    }\n"
        "  i64 n = 0; int slot = 0; u32 phase = 0;\n";
  const int dy = p_.dim_y;
  o_ << "  T y[" << dy << "], yn[" << dy << "];\n";
  if (dbl()) o_ << "  T db[" << dy << "], dbn[" << dy << "];\n";
  o_ << "  if (my_rows > 0) {";
  for (int j = 0; j < dy; ++j) {
    o_ << " yn[" << j << "] = __ldg(Y + gwarp * " << dy << " + " << j << ");";
    if (dbl()) o_ << " dbn[" << j << "] = __ldg(DB + gwarp * " << dy << " + " << j << ");";
  }
  o_ << " }\n";
  o_ << "  for (i64 rr = 0; rr < my_rows; ++rr) {\n    const i64 row = gwarp + rr * nwarp;\n";
  o_ << "   ";
  for (int j = 0; j < dy; ++j) {
    o_ << " y[" << j << "] = yn[" << j << "];";
    if (dbl()) o_ << " db[" << j << "] = dbn[" << j << "];";
  }
  o_ << "\n    if (rr + 1 < my_rows) {";
  for (int j = 0; j < dy; ++j) {
    o_ << " yn[" << j << "] = __ldg(Y + (row + nwarp) * " << dy << " + " << j << ");";
    if (dbl()) o_ << " dbn[" << j << "] = __ldg(DB + (row + nwarp) * " << dy << " + " << j << ");";
  }
  o_ << " }\n";
  if (bwd()) o_ << "    T gy[" << dy << "] = {};\n";
  for (size_t u = 0; u < units_.size(); ++u) emit_unit(static_cast<int>(u));
  if (bwd()) {
    for (int j0 = 0; j0 < dy; j0 += 32) {
    o_ << "    { T mine = 0;\n";
    for (int j = j0; j < std::min(dy, j0 + 32); ++j) o_ << "      { const T s = warp_sum(gy[" << j << "]); if (lane == " << j - j0 << ") mine = s; }\n";
    o_ << "      if (lane < " << std::min(dy - j0, 32) << ") O1[row * (i64)" << dy << " + " << j0 << " + lane] = mine; }\n";
    }
  }
  o_ << "  }\n}\n";
  ks.source = o_.str();
  return ks;
}

}  // namespace

KernelSource generate_tp_kernel(const Problem& p, const std::vector<Unit>& units,
                                const KernelConfig& cfg) {
  Gen g(p, units, cfg);
  return g.run();
}

}  // namespace cgf
