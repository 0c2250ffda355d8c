#include "codegen.hpp"

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <functional>
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
// try_wait with a suspend-time hint (ns): a waiting warp is suspended by the
// hardware until the phase completes or the hint expires, not spinning.
DEVI bool mbar_try_sleep(u64* b, u32 parity) {
  u32 ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_addr(b)), "r"(parity), "r"(1000000u) : "memory");
  return ok != 0;
}
DEVI void mbar_wait_sleep(u64* b, u32 parity) { while (!mbar_try_sleep(b, parity)) { } }
DEVI void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier (bytes).
DEVI void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
// 16-byte async copy global -> shared by one thread (LDGSTS, L2 only).
DEVI void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(smem_addr(dst)), "l"(src) : "memory");
}
// L2 eviction priorities (conv loops): gathered node rows that neighbouring
// items re-read are kept (evict_last), per-edge streams go first (evict_first).
DEVI u64 l2_policy_last() { u64 p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
DEVI u64 l2_policy_first() { u64 p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
DEVI void cp_async16_h(void* dst, const void* src, u64 pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"(smem_addr(dst)), "l"(src), "l"(pol) : "memory");
}
DEVI void bulk_g2s_h(void* dst, const void* src, u32 bytes, u64* bar, u64 pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol) : "memory");
}
// Arrive on the mbarrier once all of this thread's prior cp.async completed
// (the barrier counts one arrival per lane).
DEVI void cp_async_arrive(u64* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" :: "r"(smem_addr(b)) : "memory");
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
// The same with the count known at compile time: the lane loop is unrolled
// (no per-iteration index / compare / branch / descriptor moves).
template <int N> DEVI void coop_store16n(void* dst, const void* src, int lane) {
  const float4* s = (const float4*)src;
  float4* d = (float4*)dst;
#pragma unroll
  for (int i0 = 0; i0 < N; i0 += 32)
    if (N % 32 == 0 || i0 + lane < N) __stcs(d + i0 + lane, s[i0 + lane]);
}
template <int N, class T> DEVI void coop_storen(T* __restrict__ dst, const T* src, int lane) {
#pragma unroll
  for (int i0 = 0; i0 < N; i0 += 32)
    if (N % 32 == 0 || i0 + lane < N) dst[i0 + lane] = src[i0 + lane];
}
// Atomic accumulation of a staged run into global memory (atomic-mode conv):
// 16-byte vector reductions for FP32, scalar for FP64; results unused -> RED.
DEVI void coop_red16(float* dst, const float* src, int n16, int lane) {
  for (int i = lane; i < n16; i += 32) {
    const float4 v = ((const float4*)src)[i];
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"((float4*)dst + i), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
  }
}
DEVI void coop_red16(double* dst, const double* src, int n16, int lane) {
  for (int i = lane; i < 2 * n16; i += 32) atomicAdd(dst + i, src[i]);
}
template <class T> DEVI void coop_red(T* dst, const T* src, int n, int lane) {
  for (int i = lane; i < n; i += 32) atomicAdd(dst + i, src[i]);
}
// Paired FP32 (sm_100 FFMA2 / FMUL2): each half is an IEEE fma / mul of its
// operands; scalar register pairs are allocated adjacently by ptxas.
DEVI void fma2s(float a, float b0, float b1, float& c0, float& c1) {
  u64 A, B, C;
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(c0), "f"(c1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(C));
}
DEVI void fma2v(float a0, float a1, float b0, float b1, float& c0, float& c1) {
  u64 A, B, C;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(C) : "f"(c0), "f"(c1));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(C) : "l"(A), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(C));
}
DEVI void mul2v(float a0, float a1, float b0, float b1, float& r0, float& r1) {
  u64 A, B, R;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r0), "=f"(r1) : "l"(R));
}
DEVI void mul2s(float a, float b0, float b1, float& r0, float& r1) {
  u64 A, B, R;
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(B) : "f"(b0), "f"(b1));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(R) : "l"(A), "l"(B));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r0), "=f"(r1) : "l"(R));
}
template <class T> DEVI T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Warp sums of 2^P per-lane values at once, by recursive halving: in the round
// with lane offset o each lane keeps half of its values and adds the partner's
// copy of that half (lanes with bit o set keep the upper half), so the values
// in flight halve every round; the remaining rounds are plain butterflies.
// Every lane returns the total of value index warp_sum_n_idx<P>(lane); the
// lanes sharing the top P lane bits hold the same (bit-identical) total.
// 2^P (+1 .. 5-P) shuffles instead of 5 per value.
template <class T, int P> DEVI T warp_sum_n(T* v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < P; ++r) {
    const int o = 16 >> r, k = (1 << P) >> (r + 1);
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < k; ++i) {
      const T snd = up ? v[i] : v[i + k];
      const T kp = up ? v[i + k] : v[i];
      v[i] = kp + __shfl_xor_sync(0xffffffffu, snd, o);
    }
  }
  T t = v[0];
#pragma unroll
  for (int o = 16 >> P; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}
template <int P> DEVI int warp_sum_n_idx(int lane) {
  int j = 0;
#pragma unroll
  for (int r = 0; r < P; ++r) j = (j << 1) | ((lane >> (4 - r)) & 1);
  return j;
}
)RT";
}


namespace {

std::string hexd(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}

std::string S(long long v) { return std::to_string(v); }

// base + kc * step, as source text (kc: the runtime chunk index of a class).
std::string O(long long base, long long step) {
  if (step == 0) return S(base);
  return "(" + S(base) + " + kc * " + S(step) + ")";
}

enum class Src { Row, Nbr, Edge };

struct SlotRange {
  std::string arr;           // kernel parameter name
  std::uint32_t stride = 0;  // words per indexed row
  Src src = Src::Row;
  long long off = 0, step = 0;  // word offset within the row (affine in kc)
  std::uint32_t words = 0, slot_off = 0;
  bool bulk = false;
  bool window = false;  // y-like: copy the 16-byte aligned window around the row
};

// A class is a run of units with identical code whose global offsets are
// affine in a chunk index kc (the 32-lane chunks of the same instructions).
// One code body per class keeps the per-row program small enough for the
// instruction cache.
struct UClass {
  int u0 = 0, n = 1;
  std::vector<long long> sx, sz, sw;    // per sub position: x_off, z_off, w_off steps
  std::vector<long long> xstep, zstep;  // per x chunk / z piece
};

struct Layout {
  std::vector<SlotRange> ranges;
  std::map<std::uint32_t, std::uint32_t> x_slot, a_slot, gz_slot;  // u0 offset -> slot offset
  std::map<int, std::uint32_t> w_slot, c_slot;                      // sub position -> slot offset
  std::uint32_t words = 0, fixed_bulk_bytes = 0;
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
  std::vector<UClass> cls_;
  std::vector<Layout> lay_;  // per class
  int max_dz_ = 1, max_dx_ = 1, max_piece_ = 1;
  bool has_c_ = false;
  std::uint32_t scr_words_ = 0, off_zs_ = 0, off_wt_ = 0, off_ct_ = 0, off_gya_ = 0, off_gxs_ = 0;
  // ConvByInput: the row's gx-type accumulator holds only this kernel's x
  // chunks, packed: class k's unit kc, chunk c sits at
  // gx_base_[k] + kc * gx_unit_[k] + gx_pre_[k][c] (affine in kc).
  std::vector<std::uint32_t> gx_base_, gx_unit_;
  std::vector<std::vector<std::uint32_t>> gx_pre_;
  std::uint32_t gx_words_ = 0;

  bool reads_gz() const { return cfg_.comp == Comp::Bwd || cfg_.comp == Comp::DBwd || cfg_.comp == Comp::DBwdX; }
  bool dual() const { return cfg_.comp == Comp::DBwd || cfg_.comp == Comp::DBwdZ || cfg_.comp == Comp::DBwdX; }
  bool out_x() const { return cfg_.comp == Comp::Bwd || cfg_.comp == Comp::DBwd || cfg_.comp == Comp::DBwdX; }
  bool out_z() const { return cfg_.comp == Comp::Fwd || cfg_.comp == Comp::DBwd || cfg_.comp == Comp::DBwdZ; }
  bool out_y() const { return out_x(); }
  bool out_w() const { return out_x(); }
  bool conv() const { return cfg_.loop != Loop::Rows; }
  bool by_input() const { return cfg_.loop == Loop::ConvByInput; }
  bool edges() const { return cfg_.loop == Loop::ConvEdges; }
  bool yreg() const { return cfg_.y_regs && (cfg_.loop == Loop::Rows || edges()); }
  bool gy_flush() const { return out_y() && (dual() || cfg_.f64); }
  // by-output forward, FP32, kind B only: two edges per item as paired ops
  bool pair_edges() const {
    return cfg_.pair_edges && cfg_.loop == Loop::ConvByOutput && cfg_.comp == Comp::Fwd && !cfg_.f64 && !has_c_ &&
           cfg_.lane_copy;
  }
  // by-neighbour backward, FP32, kind B, one unit (small problems), no groups
  bool pair_edges_bwd() const {
    return cfg_.pair_edges && cfg_.loop == Loop::ConvByInput && cfg_.comp == Comp::Bwd && !cfg_.f64 && !has_c_ &&
           cfg_.lane_copy && units_.size() == 1 && cls_.size() == 1 && !cfg_.gy_accum && !gy_flush();
  }
  int eb() const {
    if (pair_edges() || pair_edges_bwd()) return 2;
    return cfg_.loop == Loop::ConvByOutput && cfg_.lane_copy ? std::max(1, cfg_.edges_per_item) : 1;
  }
  Src x_src() const { return cfg_.loop == Loop::ConvByOutput || edges() ? Src::Nbr : Src::Row; }
  Src z_src() const { return cfg_.loop == Loop::ConvByInput ? Src::Nbr : Src::Row; }
  Src e_src() const { return conv() ? Src::Edge : Src::Row; }
  const char* idx(Src s) const { return s == Src::Row ? "row" : s == Src::Nbr ? "nbr" : "eid"; }
  std::uint32_t A() const { return 16u / sz_; }
  std::uint32_t up(std::uint32_t w) const { return (w + A() - 1) / A() * A(); }
  bool al16(long long words) const { return (words * sz_) % 16 == 0; }

  void classify();
  void add(Layout& L, const std::string& arr, std::uint32_t stride, Src src, long long off, long long step,
           std::uint32_t words, std::uint32_t& so, bool window = false);
  void layout();
  std::string range_src(const SlotRange& r) const;
  void emit_issue();
  void emit_wait_and_sync(int k, bool with_wait = true);
  void emit_release();
  void emit_store(const std::string& dst, const std::string& rowexpr, std::uint32_t stride, long long off,
                  long long step, std::uint32_t words, int guard_rows, int width, const std::string& reg,
                  bool atomic = false);
  void emit_unit_body(int k, const std::function<void(int)>& post_sub = {});
  void emit_unit_body_edge_pair(int k);
  void emit_unit_body_edge_pair_bwd(int k);
  std::string wsrc(const Sub& s, long long step, const std::string& arr) const;
  void emit_gy_reduce(const std::string& rowexpr, const std::string& arr = "gy");
  void emit_multi_sum(int n, const std::function<std::string(int)>& src, const std::string& use);
  void emit_gy_flush_row(const std::string& rowexpr);
  void emit_gy_resume(const std::string& rowexpr);
  void emit_class_loop_open(int k);
  void emit_class_loop_close(int k);
  void emit_rows_loop();
  void emit_conv_loop();
  const Unit& U0(int k) const { return units_[cls_[k].u0]; }
};

bool same_shape(const Problem& p, const Unit& a, const Unit& b) {
  if (a.subs.size() != b.subs.size() || a.x_chunks.size() != b.x_chunks.size() ||
      a.z_pieces.size() != b.z_pieces.size())
    return false;
  for (size_t q = 0; q < a.subs.size(); ++q) {
    const Sub &s = p.subs[a.subs[q]], &t = p.subs[b.subs[q]];
    if (s.kind != t.kind || s.l1 != t.l1 || s.l2 != t.l2 || s.l3 != t.l3 || s.b != t.b || s.bp != t.bp ||
        s.y_off != t.y_off || s.w_stride != t.w_stride || a.x_chunk_of(s) != b.x_chunk_of(t) ||
        a.z_piece_of(s) != b.z_piece_of(t))
      return false;
  }
  for (size_t c = 0; c < a.x_chunks.size(); ++c)
    if (a.x_chunks[c].words != b.x_chunks[c].words) return false;
  for (size_t z = 0; z < a.z_pieces.size(); ++z)
    if (a.z_pieces[z].words != b.z_pieces[z].words) return false;
  return true;
}

void Gen::classify() {
  const int nu = static_cast<int>(units_.size());
  int u = 0;
  while (u < nu) {
    UClass c;
    c.u0 = u;
    c.n = 1;
    const Unit& a = units_[u];
    auto diff = [&](const Unit& b, std::vector<long long>& sx, std::vector<long long>& sz,
                    std::vector<long long>& sw, std::vector<long long>& xs, std::vector<long long>& zs) {
      for (size_t q = 0; q < a.subs.size(); ++q) {
        const Sub &s = p_.subs[a.subs[q]], &t = p_.subs[b.subs[q]];
        sx.push_back(static_cast<long long>(t.x_off) - s.x_off);
        sz.push_back(static_cast<long long>(t.z_off) - s.z_off);
        sw.push_back(static_cast<long long>(t.w_off) - s.w_off);
      }
      for (size_t q = 0; q < a.x_chunks.size(); ++q)
        xs.push_back(static_cast<long long>(b.x_chunks[q].off) - a.x_chunks[q].off);
      for (size_t q = 0; q < a.z_pieces.size(); ++q)
        zs.push_back(static_cast<long long>(b.z_pieces[q].off) - a.z_pieces[q].off);
    };
    c.sx.assign(a.subs.size(), 0);
    c.sz.assign(a.subs.size(), 0);
    c.sw.assign(a.subs.size(), 0);
    c.xstep.assign(a.x_chunks.size(), 0);
    c.zstep.assign(a.z_pieces.size(), 0);
    while (u + c.n < nu && c.n < cfg_.max_class && same_shape(p_, a, units_[u + c.n])) {
      std::vector<long long> sx, sz, sw, xs, zs;
      diff(units_[u + c.n], sx, sz, sw, xs, zs);
      if (c.n == 1) {
        c.sx = sx; c.sz = sz; c.sw = sw; c.xstep = xs; c.zstep = zs;
      } else {
        bool ok = true;
        for (size_t q = 0; q < sx.size() && ok; ++q)
          ok = sx[q] == c.n * c.sx[q] && sz[q] == c.n * c.sz[q] && sw[q] == c.n * c.sw[q];
        for (size_t q = 0; q < xs.size() && ok; ++q) ok = xs[q] == c.n * c.xstep[q];
        for (size_t q = 0; q < zs.size() && ok; ++q) ok = zs[q] == c.n * c.zstep[q];
        if (!ok) break;
      }
      ++c.n;
    }
    if (c.n == 1) {
      c.sx.assign(a.subs.size(), 0);
      c.sz.assign(a.subs.size(), 0);
      c.sw.assign(a.subs.size(), 0);
      c.xstep.assign(a.x_chunks.size(), 0);
      c.zstep.assign(a.z_pieces.size(), 0);
    }
    cls_.push_back(c);
    u += c.n;
  }
}

void Gen::add(Layout& L, const std::string& arr, std::uint32_t stride, Src src, long long off, long long step,
              std::uint32_t words, std::uint32_t& so, bool window) {
  SlotRange r;
  r.arr = arr;
  r.stride = stride;
  r.src = src;
  r.off = off;
  r.step = step;
  r.words = words;
  r.window = window;
  r.slot_off = L.words;
  if (window) {
    r.bulk = cfg_.aligned;
    L.words = up(L.words + words + 2 * A());
  } else {
    r.bulk = cfg_.aligned && al16(stride) && al16(off) && al16(step) && al16(words);
    L.words = up(L.words + words);
    if (r.bulk) L.fixed_bulk_bytes += words * sz_;
  }
  so = r.slot_off;
  L.ranges.push_back(r);
}

void Gen::layout() {
  for (const auto& s : p_.subs) {
    max_dz_ = std::max(max_dz_, s.dz());
    max_dx_ = std::max(max_dx_, s.dx());
    max_piece_ = std::max({max_piece_, s.b * s.dz(), s.bp * s.dx()});
    if (s.kind == Kind::C) has_c_ = true;
  }
  const std::uint32_t nw = cfg_.w_shared ? 0 : p_.n_w;
  for (size_t k = 0; k < cls_.size(); ++k) {
    const UClass& C = cls_[k];
    const Unit& u = units_[C.u0];
    Layout L;
    std::uint32_t so = 0;
    if (!yreg()) {
      // y rows are copied as a 16-byte aligned window unless they are aligned
      // themselves (dim_y * sizeof(T) % 16 == 0): then a plain range
      const bool win = cfg_.y_window || !al16(p_.dim_y);
      add(L, "Y", p_.dim_y, e_src(), 0, 0, p_.dim_y, so, win);
      if (dual()) add(L, "DB", p_.dim_y, e_src(), 0, 0, p_.dim_y, so, win);
    }
    for (size_t c = 0; c < u.x_chunks.size(); ++c) {
      const auto& xc = u.x_chunks[c];
      add(L, "X", p_.dim_x, x_src(), xc.off, C.xstep[c], xc.words, so);
      L.x_slot[xc.off] = so;
      if (dual()) {
        add(L, "DA", p_.dim_x, x_src(), xc.off, C.xstep[c], xc.words, so);
        L.a_slot[xc.off] = so;
      }
    }
    if (!cfg_.w_shared) {
      // in source order, so slices adjacent in the W row are adjacent in the
      // slot too (one contiguous copy for the parallel-bulk issue)
      std::vector<int> order(u.subs.size());
      for (size_t q = 0; q < order.size(); ++q) order[q] = static_cast<int>(q);
      std::stable_sort(order.begin(), order.end(),
                       [&](int a, int b) { return p_.subs[u.subs[a]].w_off < p_.subs[u.subs[b]].w_off; });
      for (int qi : order) {
        const Sub& s = p_.subs[u.subs[qi]];
        if (s.kind != Kind::B) continue;
        add(L, "W", nw, e_src(), s.w_off, C.sw[qi], s.b, so);
        L.w_slot[qi] = so;
      }
      if (dual())
        for (int qi : order) {
          const Sub& s = p_.subs[u.subs[qi]];
          if (s.kind != Kind::B) continue;
          add(L, "DC", nw, e_src(), s.w_off, C.sw[qi], s.b, so);
          L.c_slot[qi] = so;
        }
    }
    if (reads_gz()) {
      for (size_t z = 0; z < u.z_pieces.size(); ++z) {
        add(L, "GZ", p_.dim_z, z_src(), u.z_pieces[z].off, C.zstep[z], u.z_pieces[z].words, so);
        L.gz_slot[u.z_pieces[z].off] = so;
      }
    }
    L.words = std::max<std::uint32_t>(L.words, A());
    lay_.push_back(std::move(L));
  }
  for (size_t k = 0; k < cls_.size(); ++k) {
    const Unit& u = units_[cls_[k].u0];
    std::vector<std::uint32_t> pre;
    std::uint32_t w = 0;
    for (const auto& xc : u.x_chunks) {
      pre.push_back(w);
      w += xc.words;
    }
    gx_base_.push_back(gx_words_);
    gx_unit_.push_back(w);
    gx_pre_.push_back(pre);
    gx_words_ += w * static_cast<std::uint32_t>(cls_[k].n);
  }
  const std::uint32_t stage = up(static_cast<std::uint32_t>(std::max(max_piece_, 32 * max_dx_)));
  scr_words_ = stage;
  off_gya_ = scr_words_;
  scr_words_ += up(static_cast<std::uint32_t>(p_.dim_y));
  off_gxs_ = scr_words_;
  if (by_input()) scr_words_ += up(gx_words_);
  off_zs_ = scr_words_;
  if (has_c_) {
    scr_words_ += up(2u * 32u * max_dz_);
    off_wt_ = scr_words_;
    scr_words_ += up(32u * 33u);
    off_ct_ = scr_words_;
    if (dual()) scr_words_ += up(32u * 33u);
  }
}

std::string Gen::wsrc(const Sub& s, long long step, const std::string& arr) const {
  if (cfg_.w_shared) return "(" + arr + " + " + O(s.w_off, step) + ")";
  return "(" + arr + " + " + idx(e_src()) + " * (i64)" + S(p_.n_w) + " + " + O(s.w_off, step) + ")";
}

std::string Gen::range_src(const SlotRange& r) const {
  const std::string I = (r.arr == "W" || r.arr == "DC") && cfg_.w_shared ? "0" : idx(r.src);
  return r.arr + " + " + I + " * (i64)" + S(r.stride) + " + " + O(r.off, r.step);
}

// issue_unit(u, ...): start the item's copies into its slot. u is the flat
// unit index -> (class, kc).
//   lane copy (default): every lane issues 16-byte cp.async pieces; pass t
//     gives lane l piece 32 t + l of the concatenation of the class's fixed
//     ranges. The 64-bit row bases of the source arrays are computed once per
//     item; a lane's piece is a compile-time (base, offset) pair selected by
//     its lane range. Completion: one cp.async.mbarrier arrive per lane.
//     (A table-driven variant -- one L1 table load per pass -- measured 1.8x
//     slower on the TP backward: the load latency sat on the critical path.)
//   parallel bulk (par_bulk, with lane copy): lane i issues one cp.async.bulk
//     (TMA 1-D) for the class's i-th contiguous range, lane 0 arms the mbarrier
//     with the item's byte count: one instruction per range, in parallel.
//   bulk: lane 0 arms the mbarrier and issues one cp.async.bulk per range.
void Gen::emit_issue() {
  const bool lc = cfg_.lane_copy;
  const bool pb = lc && cfg_.par_bulk;
  // distinct (array, index) source bases of the fixed ranges
  std::vector<std::pair<std::string, Src>> bases;
  auto base_id = [&](const SlotRange& r) {
    const std::pair<std::string, Src> key{r.arr, ((r.arr == "W" || r.arr == "DC") && cfg_.w_shared) ? Src::Row : r.src};
    for (size_t i = 0; i < bases.size(); ++i)
      if (bases[i] == key) return static_cast<int>(i);
    bases.push_back(key);
    return static_cast<int>(bases.size()) - 1;
  };
  if (lc)
    for (const auto& L : lay_)
      for (const auto& r : L.ranges)
        if (r.bulk && !r.window) base_id(r);
  const bool hints = cfg_.l2_hints && conv();
  // a range re-read by neighbouring items (node rows) vs a per-edge stream
  auto keep = [&](const SlotRange& r) { return r.src != Src::Edge; };
  auto pol = [&](const SlotRange& r) { return std::string(keep(r) ? "PL" : "PF"); };
  o_ << "__device__ __noinline__ void issue_unit(int u, i64 row, i64 nbr, i64 eid, i64 rows_tot, i64 edges_tot, T* sl,"
        " u64* bar, const T* __restrict__ X, const T* __restrict__ Y, const T* __restrict__ W,"
        " const T* __restrict__ GZ, const T* __restrict__ DA, const T* __restrict__ DB, const T* __restrict__ DC"
     << (lc ? ", int lane" : "") << (lc ? ", bool v_" : "") << ") {\n"
        "  (void)nbr; (void)eid; (void)rows_tot; (void)edges_tot;\n"
     << (lc && !pb ? "" : "  fence_proxy_async();\n")
     << (hints ? "  const u64 PL = l2_policy_last(), PF = l2_policy_first();\n" : "");
  int wlane = 31;  // parallel bulk: window ranges take lanes 31, 30, ...
  if (lc) {
    for (size_t i = 0; i < bases.size(); ++i) {
      const auto& [arr, src] = bases[i];
      std::uint32_t stride = 0;
      for (const auto& L : lay_)
        for (const auto& r : L.ranges)
          if (r.arr == arr) stride = r.stride;
      const std::string I = ((arr == "W" || arr == "DC") && cfg_.w_shared) ? "0" : idx(src);
      o_ << "  const char* B" << i << " = (const char*)(" << arr << " + " << I << " * (i64)" << stride << ");\n";
    }
    o_ << "  char* sb = (char*)sl;\n";
    if (pb) o_ << "  u32 tx = 0; const char* s_ = nullptr; int d_ = 0; u32 b_ = 0;" << (hints ? " u64 p_ = 0;" : "") << "\n";
    // v_ false: an item slot past the row's last edge (multi-edge items) --
    // no copies, but the lane still arrives so the barrier count holds
    o_ << "  if (v_) {\n";
    // window ranges (y, db): same slot offsets in every class (laid out first)
    for (const auto& r : lay_[0].ranges) {
      if (!(r.bulk && r.window)) continue;
      if (pb) {
        // one lane per window range (from lane 31 down), bytes into the item's tx
        const std::string I = r.src == Src::Edge ? "eid" : "row";
        const std::string tot = r.src == Src::Edge && conv() ? "edges_tot" : "rows_tot";
        o_ << "  { const i64 b0 = " << I << " * " << r.stride << ", a0 = b0 & ~(i64)" << A() - 1 << ", a1 = (b0 + "
           << r.words << " + " << A() - 1 << ") & ~(i64)" << A() - 1 << ";\n    if (a1 <= " << tot << " * (i64)" << r.stride
           << ") { const u32 n_ = (u32)((a1 - a0) * sizeof(T)); tx += n_; if (lane == " << wlane << ") { s_ = (const char*)("
           << r.arr << " + a0); d_ = " << r.slot_off * sz_ << "; b_ = n_;" << (hints ? " p_ = " + pol(r) + ";" : "")
           << " } } }\n";
        --wlane;
        continue;
      }
      const std::string I = r.src == Src::Edge ? "eid" : "row";
      const std::string tot = r.src == Src::Edge && conv() ? "edges_tot" : "rows_tot";
      o_ << "  { const i64 b0 = " << I << " * " << r.stride << ", a0 = b0 & ~(i64)" << A() - 1 << ", a1 = (b0 + " << r.words
         << " + " << A() - 1 << ") & ~(i64)" << A() - 1 << ";\n    if (a1 <= " << tot << " * (i64)" << r.stride
         << ") { const int n16 = (int)((a1 - a0) * sizeof(T) / 16); for (int c = lane; c < n16; c += 32) cp_async16(sb + "
         << r.slot_off * sz_ << " + 16 * c, (const char*)(" << r.arr << " + a0) + 16 * c); } }\n";
    }
  }
  for (size_t k = 0; k < cls_.size(); ++k) {
    const UClass& C = cls_[k];
    const Layout& L = lay_[k];
    o_ << "  " << (k ? "else " : "") << "if (u < " << C.u0 + C.n << ") {\n    const int kc = u - " << C.u0
       << "; (void)kc;\n";
    if (pb) {
      // contiguous runs of fixed ranges (same base, adjacent source and slot)
      struct Run { int base; long long off, step; std::uint32_t dst, bytes; };
      std::vector<Run> runs;
      std::uint32_t fixed = 0;
      for (const auto& r : L.ranges) {
        if (!r.bulk || r.window) continue;
        const Run x{base_id(r), r.off * sz_, r.step * sz_, r.slot_off * static_cast<std::uint32_t>(sz_),
                    r.words * static_cast<std::uint32_t>(sz_)};
        fixed += x.bytes;
        if (!runs.empty()) {
          Run& b = runs.back();
          if (b.base == x.base && b.step == x.step && b.off + b.bytes == x.off && b.dst + b.bytes == x.dst) {
            b.bytes += x.bytes;
            continue;
          }
        }
        runs.push_back(x);
      }
      if (runs.size() > static_cast<size_t>(wlane + 1))
        throw UnsupportedError("parallel bulk issue: more ranges than lanes");
      o_ << "    tx += " << fixed << "u;\n";
      for (size_t i = 0; i < runs.size(); ++i)
        o_ << "    " << (i ? "else " : "") << "if (lane == " << i << ") { s_ = B" << runs[i].base << " + "
           << O(runs[i].off, runs[i].step) << "; d_ = " << runs[i].dst << "; b_ = " << runs[i].bytes << "u;"
           << (hints ? std::string(" p_ = ") + (bases[runs[i].base].second != Src::Edge ? "PL" : "PF") + ";" : "")
           << " }\n";
    } else if (lc) {
      std::vector<std::pair<int, int>> pieces;  // (range, piece)
      for (size_t ri = 0; ri < L.ranges.size(); ++ri) {
        const auto& r = L.ranges[ri];
        if (!r.bulk || r.window) continue;
        for (std::uint32_t c = 0; c < r.words * sz_ / 16; ++c) pieces.emplace_back(static_cast<int>(ri), static_cast<int>(c));
      }
      for (size_t t0 = 0; t0 < pieces.size(); t0 += 32) {
        const size_t t1 = std::min(pieces.size(), t0 + 32);
        o_ << "    { const char* s_ = nullptr; int d_ = 0;" << (hints ? " u64 p_ = 0;" : "") << "\n";
        size_t a = t0;
        bool first = true;
        while (a < t1) {
          size_t b = a;
          while (b < t1 && pieces[b].first == pieces[a].first) ++b;
          const auto& r = L.ranges[pieces[a].first];
          // lane l of this run copies piece (pieces[a].second + l - a + t0) of range r
          const long long p0 = pieces[a].second - static_cast<long long>(a - t0);
          if (cfg_.old_issue)  // A/B: the 64-bit row address per range (pre-bases form)
            o_ << "      " << (first ? "" : "else ") << "if (lane < " << b - t0 << ") { s_ = (const char*)(" << range_src(r)
               << ") + " << 16 * p0 << "; d_ = " << r.slot_off * sz_ + 16 * p0 << "; }\n";
          else
            o_ << "      " << (first ? "" : "else ") << "if (lane < " << b - t0 << ") { s_ = B" << base_id(r) << " + "
               << O(r.off * sz_ + 16 * p0, r.step * sz_) << "; d_ = " << r.slot_off * sz_ + 16 * p0 << ";"
               << (hints ? " p_ = " + pol(r) + ";" : "") << " }\n";
          first = false;
          a = b;
        }
        if (hints)
          o_ << "      if (lane < " << t1 - t0 << ") cp_async16_h(sb + d_ + 16 * lane, s_ + 16 * lane, p_); }\n";
        else
          o_ << "      if (lane < " << t1 - t0 << ") cp_async16(sb + d_ + 16 * lane, s_ + 16 * lane); }\n";
      }
    } else {
      o_ << "    u32 tx = " << L.fixed_bulk_bytes << "u; (void)tx;\n";
      for (const auto& r : L.ranges)
        if (r.bulk && r.window) {
          const std::string I = r.src == Src::Edge ? "eid" : "row";
          const std::string tot = r.src == Src::Edge && conv() ? "edges_tot" : "rows_tot";
          o_ << "    const i64 b0_" << r.arr << " = " << I << " * " << r.stride << ", a0_" << r.arr << " = b0_" << r.arr
             << " & ~(i64)" << A() - 1 << ", a1_" << r.arr << " = (b0_" << r.arr << " + " << r.words << " + " << A() - 1
             << ") & ~(i64)" << A() - 1 << ";\n    const bool ok_" << r.arr << " = a1_" << r.arr << " <= " << tot
             << " * (i64)" << r.stride << ";\n    if (ok_" << r.arr << ") tx += (u32)((a1_" << r.arr << " - a0_" << r.arr
             << ") * sizeof(T));\n";
        }
      o_ << "    mbar_expect_tx(bar, tx);\n";
      for (const auto& r : L.ranges) {
        if (!r.bulk) continue;
        if (r.window)
          o_ << "    if (ok_" << r.arr << ") bulk_g2s(sl + " << r.slot_off << ", " << r.arr << " + a0_" << r.arr
             << ", (u32)((a1_" << r.arr << " - a0_" << r.arr << ") * sizeof(T)), bar);\n";
        else
          o_ << "    bulk_g2s(sl + " << r.slot_off << ", " << range_src(r) << ", " << r.words * sz_ << "u, bar);\n";
      }
    }
    o_ << "  }\n";
  }
  if (lc) o_ << "  }\n";
  if (pb)
    o_ << "  if (lane == 0) mbar_expect_tx(bar, tx);\n  __syncwarp();\n  if (b_) "
       << (hints ? "bulk_g2s_h(sb + d_, s_, b_, bar, p_);\n" : "bulk_g2s(sb + d_, s_, b_, bar);\n");
  else if (lc)
    o_ << "  cp_async_arrive(bar);\n";
  o_ << "}\n\n";
}

void Gen::emit_wait_and_sync(int k, bool with_wait) {
  const Layout& L = lay_[k];
  if (with_wait)
    o_ << "      T* sl = wsm + slot * SLOT_WORDS;\n      " << (cfg_.wait_sleep ? "mbar_wait_sleep" : "mbar_wait")
       << "(&bars[slot], phase);\n";
  bool sync = false;
  for (const auto& r : L.ranges) {
    if ((r.arr == "Y" || r.arr == "DB") && !r.window)
      o_ << "      const int " << (r.arr == "Y" ? "ys" : "dbs") << " = " << r.slot_off << ";\n";
    if (r.window) {
      const std::string I = r.src == Src::Edge ? "eid" : "row";
      const std::string tot = r.src == Src::Edge && conv() ? "edges_tot" : "rows";
      const std::string var = r.arr == "Y" ? "ys" : "dbs";
      if (r.bulk) {
        o_ << "      int " << var << ";\n      { const i64 b0 = " << I << " * " << r.stride << "; const i64 a0 = b0 & ~(i64)"
           << A() - 1 << "; const i64 a1 = (b0 + " << r.words << " + " << A() - 1 << ") & ~(i64)" << A() - 1 << ";\n"
           << "        if (a1 <= " << tot << " * (i64)" << r.stride << ") " << var << " = " << r.slot_off
           << " + (int)(b0 - a0);\n        else { " << var << " = " << r.slot_off << "; coop_load(sl + "
           << r.slot_off << ", " << r.arr << " + b0, " << r.words << ", lane); __syncwarp(); } }\n";
      } else {
        o_ << "      const int " << var << " = " << r.slot_off << ";\n      coop_load(sl + " << r.slot_off << ", "
           << r.arr << " + " << I << " * (i64)" << r.stride << ", " << r.words << ", lane);\n";
        sync = true;
      }
      continue;
    }
    if (r.bulk) continue;
    o_ << "      coop_load(sl + " << r.slot_off << ", " << range_src(r) << ", " << r.words << ", lane);\n";
    sync = true;
  }
  if (sync) o_ << "      __syncwarp();\n";
}

void Gen::emit_release() {
  o_ << "      __syncwarp();\n      " << (cfg_.lane_copy ? "" : "if (lane == 0) ") << "producer_next();\n"
        "      if (++slot == D) { slot = 0; phase ^= 1u; }\n";
}

void Gen::emit_store(const std::string& dst, const std::string& rowexpr, std::uint32_t stride, long long off,
                     long long step, std::uint32_t words, int guard_rows, int width, const std::string& reg,
                     bool atomic) {
  o_ << "      if (lane < " << guard_rows << ") {";
  for (int k = 0; k < width; ++k) o_ << " scr[lane * " << width << " + " << k << "] = " << reg << "[" << k << "];";
  o_ << " }\n      __syncwarp();\n";
  const bool vec = cfg_.aligned && al16(stride) && al16(off) && al16(step) && al16(words);
  const std::string at = dst + " + " + rowexpr + " * (i64)" + S(stride) + " + " + O(off, step);
  if (atomic)
    o_ << "      " << (vec ? "coop_red16(" : "coop_red(") << at << ", scr, " << (vec ? words * sz_ / 16 : words)
       << ", lane);\n";
  else if (!cfg_.unrolled_stores)
    o_ << "      " << (vec ? "coop_store16(" : "coop_store(") << at << ", scr, " << (vec ? words * sz_ / 16 : words)
       << ", lane);\n";
  else if (vec)
    o_ << "      coop_store16n<" << words * sz_ / 16 << ">(" << at << ", scr, lane);\n";
  else
    o_ << "      coop_storen<" << words << ">(" << at << ", scr, lane);\n";
  o_ << "      __syncwarp();\n";
}

// Compute of one unit (class k, chunk kc) on its staged slot. The caller
// declares x-chunk accumulators ax<c> (when the unit owns them) and z-piece
// accumulators pz<c>. A unit merged from m same-shape chunks (merge_units)
// is emitted sub by sub with its m chunks side by side: the lane-uniform CG
// products v*y[j] (and v*db[j]) are computed once and feed all m chunks.
void Gen::emit_unit_body(int k, const std::function<void(int)>& post_sub) {
  const UClass& Cl = cls_[k];
  const Unit& u = U0(k);
  const Layout& L = lay_[k];
  const std::string nw = S(p_.n_w);
  // weight-gradient rows: per item (with shared W the caller passes a per-row
  // workspace and reduces it over rows)
  const std::string wrow = idx(e_src());
  const int nsub = static_cast<int>(u.subs.size());
  const int m = (cfg_.joint && u.merged > 1 && nsub % u.merged == 0) ? u.merged : 1;
  const int n = nsub / m;
  const bool need_gzc = cfg_.comp == Comp::DBwd || cfg_.comp == Comp::DBwdX;
  const bool zx_on = cfg_.comp == Comp::Fwd || cfg_.comp == Comp::Bwd || cfg_.comp == Comp::DBwd || cfg_.comp == Comp::DBwdZ;
  const bool zab = cfg_.comp == Comp::DBwd || cfg_.comp == Comp::DBwdZ || cfg_.comp == Comp::DBwdX;
  const bool gfl = gy_flush();
  const bool yq = !yreg() && (m > 1 || cfg_.y_item);
  // paired FP32 emission of two merged chunks (FFMA2)
  const bool f2 = cfg_.ffma2 && m == 2 && !cfg_.f64;
  if (yq) {
    // joint chunks: the item's y (and db) into registers once, so the products
    // below are shared across chunks; otherwise y is read from the slot at each
    // use (no registers held across the item)
    o_ << "      T yq[" << p_.dim_y << "];" << (dual() ? " T dbq[" + S(p_.dim_y) + "];" : "");
    for (int j = 0; j < p_.dim_y; ++j)
      o_ << " yq[" << j << "] = sl[ys + " << j << "];" << (dual() ? " dbq[" + S(j) + "] = sl[dbs + " + S(j) + "];" : "");
    o_ << "\n";
  }
  if (cfg_.x_regs) {
    // the unit's x (and dL/da) chunks into registers once: every sub reading a
    // chunk then takes it from there instead of reloading the slot
    for (size_t c = 0; c < u.x_chunks.size(); ++c) {
      int dxc = 1, bpc = 0;
      for (int si : u.subs)
        if (p_.subs[si].x_off == u.x_chunks[c].off) {
          dxc = p_.subs[si].dx();
          bpc = p_.subs[si].bp;
        }
      const std::uint32_t xs = L.x_slot.at(u.x_chunks[c].off);
      o_ << "      T xr" << c << "[" << dxc << "];" << (dual() ? " T ar" + S(c) + "[" + S(dxc) + "];" : "")
         << "\n      if (lane < " << bpc << ") {";
      for (int i = 0; i < dxc; ++i) o_ << " xr" << c << "[" << i << "] = sl[" << xs << " + lane * " << dxc << " + " << i << "];";
      if (dual())
        for (int i = 0; i < dxc; ++i)
          o_ << " ar" << c << "[" << i << "] = sl[" << L.a_slot.at(u.x_chunks[c].off) << " + lane * " << dxc << " + " << i
             << "];";
      o_ << " } else {";
      for (int i = 0; i < dxc; ++i) o_ << " xr" << c << "[" << i << "] = 0;" << (dual() ? " ar" + S(c) + "[" + S(i) + "] = 0;" : "");
      o_ << " }\n";
    }
  }
  auto Y = [&](int j) { return yreg() ? "y[" + S(j) + "]" : yq ? "yq[" + S(j) + "]" : "sl[ys + " + S(j) + "]"; };
  auto DB = [&](int j) { return yreg() ? "db[" + S(j) + "]" : yq ? "dbq[" + S(j) + "]" : "sl[dbs + " + S(j) + "]"; };
  for (int g = 0; g < n; ++g) {
    if (g && cfg_.sub_barrier) o_ << "      asm volatile(\"\" ::: \"memory\");\n";
    const Sub& s0 = p_.subs[u.subs[g]];
    const int dx = s0.dx(), dz = s0.dz();
    o_ << "      { // sub";
    for (int c = 0; c < m; ++c) o_ << " " << u.subs[g + c * n];
    o_ << ": " << (s0.kind == Kind::B ? "B" : "C") << " l=(" << s0.l1 << "," << s0.l2 << "," << s0.l3 << ") b=" << s0.b
       << " b'=" << s0.bp << " nnz=" << s0.cg->entries.size() << (m > 1 ? " x" + S(m) + " chunks" : "") << "\n";
    // two merged kind-B chunks of a backward: their gz*w products and their gW
    // chains go out as paired FP32 ops (each half the same op, same bits)
    bool pair_b = false;
    if (f2 && cfg_.pair_weights && cfg_.comp == Comp::Bwd) {
      const Sub& s1 = p_.subs[u.subs[g + n]];
      pair_b = s0.kind == Kind::B && s1.kind == Kind::B && s1.dz() == dz && !cfg_.w_shared;
    }
    // ---- per-chunk operands ----
    for (int c = 0; c < m; ++c) {
      const int qi = g + c * n;
      const Sub& s = p_.subs[u.subs[qi]];
      const std::string X = "_" + S(c);
      const long long swq = Cl.sw[qi];
      if (gfl && out_y()) o_ << "        T gyl" << X << "[" << s.dy() << "] = {};\n";
      const std::uint32_t xs = L.x_slot.at(s.x_off);
      if (cfg_.x_regs) {
        const int xc = u.x_chunk_of(s);
        o_ << "        T xv" << X << "[" << dx << "];" << (dual() ? " T av" + X + "[" + S(dx) + "];" : "") << "\n       ";
        for (int i = 0; i < dx; ++i)
          o_ << " xv" << X << "[" << i << "] = xr" << xc << "[" << i << "];" << (dual() ? " av" + X + "[" + S(i) + "] = ar" + S(xc) + "[" + S(i) + "];" : "");
        o_ << "\n";
      } else {
      o_ << "        T xv" << X << "[" << dx << "];" << (dual() ? " T av" + X + "[" + S(dx) + "];" : "")
         << "\n        if (lane < " << s.bp << ") {";
      for (int i = 0; i < dx; ++i) o_ << " xv" << X << "[" << i << "] = sl[" << xs << " + lane * " << dx << " + " << i << "];";
      if (dual())
        for (int i = 0; i < dx; ++i)
          o_ << " av" << X << "[" << i << "] = sl[" << L.a_slot.at(s.x_off) << " + lane * " << dx << " + " << i << "];";
      o_ << " } else {";
      for (int i = 0; i < dx; ++i) o_ << " xv" << X << "[" << i << "] = 0;";
      if (dual())
        for (int i = 0; i < dx; ++i) o_ << " av" << X << "[" << i << "] = 0;";
      o_ << " }\n";
      }
      std::string gzs;
      if (reads_gz()) {
        gzs = S(L.gz_slot.at(s.z_off));
        if (s.kind == Kind::B) {
          o_ << "        T gz" << X << "[" << dz << "];\n        if (lane < " << s.b << ") {";
          for (int kk = 0; kk < dz; ++kk) o_ << " gz" << X << "[" << kk << "] = sl[" << gzs << " + lane * " << dz << " + " << kk << "];";
          o_ << " } else {";
          for (int kk = 0; kk < dz; ++kk) o_ << " gz" << X << "[" << kk << "] = 0;";
          o_ << " }\n";
        }
      }
      if (s.kind == Kind::B) {
        auto wexpr = [&](const std::string& arr, const std::map<int, std::uint32_t>& slot) {
          if (cfg_.w_shared) return "__ldg(" + wsrc(s, swq, arr) + " + lane)";
          return "sl[" + S(slot.at(qi)) + " + lane]";
        };
        o_ << "        const T wt" << X << " = (lane < " << s.b << ") ? " << wexpr("W", L.w_slot) << " : (T)0;\n";
        if (dual()) o_ << "        const T ct" << X << " = (lane < " << s.b << ") ? " << wexpr("DC", L.c_slot) << " : (T)0;\n";
      }
      if (reads_gz()) {
        o_ << "        T gzp" << X << "[" << dz << "];" << (need_gzc ? " T gzc" + X + "[" + S(dz) + "];" : "") << "\n";
        if (s.kind == Kind::B && pair_b) {
          if (c == 1)  // both chunks' operands are in place now
            for (int kk = 0; kk < dz; ++kk)
              o_ << "        mul2v(wt_0, wt_1, gz_0[" << kk << "], gz_1[" << kk << "], gzp_0[" << kk << "], gzp_1[" << kk << "]);\n";
        } else if (s.kind == Kind::B) {
          for (int kk = 0; kk < dz; ++kk)
            o_ << "        gzp" << X << "[" << kk << "] = wt" << X << " * gz" << X << "[" << kk << "];"
               << (need_gzc ? " gzc" + X + "[" + S(kk) + "] = ct" + X + " * gz" + X + "[" + S(kk) + "];" : "") << "\n";
        } else {
          o_ << "        {";
          for (int kk = 0; kk < dz; ++kk)
            o_ << " gzp" << X << "[" << kk << "] = 0;" << (need_gzc ? " gzc" + X + "[" + S(kk) + "] = 0;" : "");
          o_ << "\n          const T* wg = " << wsrc(s, swq, "W") << ";\n";
          if (need_gzc) o_ << "          const T* cg = " << wsrc(s, swq, "DC") << ";\n";
          o_ << "#pragma unroll 2\n          for (int r = 0; r < " << s.b << "; ++r) {\n"
             << "            const T wv = (lane < " << s.bp << ") ? __ldg(wg + r * " << s.w_stride << " + lane) : (T)0;\n";
          if (need_gzc)
            o_ << "            const T cv = (lane < " << s.bp << ") ? __ldg(cg + r * " << s.w_stride << " + lane) : (T)0;\n";
          for (int kk = 0; kk < dz; ++kk) {
            o_ << "            { const T g = sl[" << gzs << " + r * " << dz << " + " << kk << "]; gzp" << X << "[" << kk
               << "] = fma(wv, g, gzp" << X << "[" << kk << "]);";
            if (need_gzc) o_ << " gzc" << X << "[" << kk << "] = fma(cv, g, gzc" << X << "[" << kk << "]);";
            o_ << " }\n";
          }
          o_ << "          }\n        }\n";
        }
      }
      if (zx_on) o_ << "        T zx" << X << "[" << dz << "] = {};\n";
      if (zab) o_ << "        T za" << X << "[" << dz << "] = {}; T zb" << X << "[" << dz << "] = {};\n";
    }
    // ---- the unrolled CG stream (one line per nonzero entry, all chunks) ----
    for (const auto& e : s0.cg->entries) {
      const std::string v = "(T)" + hexd(e.v), I = S(e.i), K = S(e.k);
      const int J = s0.y_off + e.j;
      // v * (a0, a1) into (r0, r1): a paired multiply, or (|v| = 1, exact either way) a copy
      auto mul2 = [&](const std::string& a0, const std::string& a1, const std::string& r0, const std::string& r1) {
        if (e.v == 1.0) return " " + r0 + " = " + a0 + "; " + r1 + " = " + a1 + ";";
        if (e.v == -1.0) return " " + r0 + " = -" + a0 + "; " + r1 + " = -" + a1 + ";";
        return " mul2s(" + v + ", " + a0 + ", " + a1 + ", " + r0 + ", " + r1 + ");";
      };
      std::ostringstream l;
      l << "        { const T cy = " << v << " * " << Y(J) << ";";
      if (dual()) l << " const T cb = " << v << " * " << DB(J) << ";";
      if (f2) {
        // the two chunks' identical streams as paired FP32 ops (FFMA2 / FMUL2:
        // one instruction per pair, each half an IEEE fma / mul -> the same
        // bits as the scalar form)
        const Sub& s_0 = p_.subs[u.subs[g]];
        const Sub& s_1 = p_.subs[u.subs[g + n]];
        const std::string A0 = "ax" + S(u.x_chunk_of(s_0)), A1 = "ax" + S(u.x_chunk_of(s_1));
        auto GYc = [&](int c, const Sub& s) { return gfl ? "gyl_" + S(c) + "[" + S(e.j) + "]" : "gy[" + S(s.y_off + e.j) + "]"; };
        if (zx_on) l << " fma2s(cy, xv_0[" << I << "], xv_1[" << I << "], zx_0[" << K << "], zx_1[" << K << "]);";
        if (zab)
          l << " fma2s(cy, av_0[" << I << "], av_1[" << I << "], za_0[" << K << "], za_1[" << K << "]);"
            << " fma2s(cb, xv_0[" << I << "], xv_1[" << I << "], zb_0[" << K << "], zb_1[" << K << "]);";
        if (need_gzc) {
          // AX = fma(cb, gzp, fma(cy, gzc, AX)); GY = fma(v a, gzp, fma(v x, gzc, GY)) per chunk
          l << " fma2s(cy, gzc_0[" << K << "], gzc_1[" << K << "], " << A0 << "[" << I << "], " << A1 << "[" << I << "]);"
            << " fma2s(cb, gzp_0[" << K << "], gzp_1[" << K << "], " << A0 << "[" << I << "], " << A1 << "[" << I << "]);"
            << " { T t0_, t1_, u0_, u1_;" << mul2("xv_0[" + I + "]", "xv_1[" + I + "]", "t0_", "t1_")
            << mul2("av_0[" + I + "]", "av_1[" + I + "]", "u0_", "u1_");
          if (gfl)
            l << " fma2v(t0_, t1_, gzc_0[" << K << "], gzc_1[" << K << "], " << GYc(0, s_0) << ", " << GYc(1, s_1) << ");"
              << " fma2v(u0_, u1_, gzp_0[" << K << "], gzp_1[" << K << "], " << GYc(0, s_0) << ", " << GYc(1, s_1) << "); }";
          else
            l << " " << GYc(0, s_0) << " = fma(u0_, gzp_0[" << K << "], fma(t0_, gzc_0[" << K << "], " << GYc(0, s_0) << "));"
              << " " << GYc(1, s_1) << " = fma(u1_, gzp_1[" << K << "], fma(t1_, gzc_1[" << K << "], " << GYc(1, s_1) << ")); }";
        }
        if (cfg_.comp == Comp::Bwd) {
          l << " fma2s(cy, gzp_0[" << K << "], gzp_1[" << K << "], " << A0 << "[" << I << "], " << A1 << "[" << I << "]);"
            << " { T t0_, t1_;" << mul2("xv_0[" + I + "]", "xv_1[" + I + "]", "t0_", "t1_");
          if (gfl)
            l << " fma2v(t0_, t1_, gzp_0[" << K << "], gzp_1[" << K << "], " << GYc(0, s_0) << ", " << GYc(1, s_1) << "); }";
          else
            l << " " << GYc(0, s_0) << " = fma(t0_, gzp_0[" << K << "], " << GYc(0, s_0) << "); " << GYc(1, s_1)
              << " = fma(t1_, gzp_1[" << K << "], " << GYc(1, s_1) << "); }";
        }
        l << " }\n";
        o_ << l.str();
        continue;
      }
      for (int c = 0; c < m; ++c) {
        const int qi = g + c * n;
        const Sub& s = p_.subs[u.subs[qi]];
        const std::string X = "_" + S(c);
        const std::string AX = "ax" + S(u.x_chunk_of(s));
        auto GY = [&](int j) { return gfl ? "gyl" + X + "[" + S(j) + "]" : "gy[" + S(s.y_off + j) + "]"; };
        if (zx_on) l << " zx" << X << "[" << K << "] = fma(cy, xv" << X << "[" << I << "], zx" << X << "[" << K << "]);";
        if (zab)
          l << " za" << X << "[" << K << "] = fma(cy, av" << X << "[" << I << "], za" << X << "[" << K << "]); zb" << X << "[" << K
            << "] = fma(cb, xv" << X << "[" << I << "], zb" << X << "[" << K << "]);";
        if (cfg_.comp == Comp::Bwd)
          l << " " << AX << "[" << I << "] = fma(cy, gzp" << X << "[" << K << "], " << AX << "[" << I << "]);"
            << " " << GY(e.j) << " = fma(" << v << " * xv" << X << "[" << I << "], gzp" << X << "[" << K << "], " << GY(e.j) << ");";
        if (need_gzc)
          l << " " << AX << "[" << I << "] = fma(cb, gzp" << X << "[" << K << "], fma(cy, gzc" << X << "[" << K << "], " << AX
            << "[" << I << "]));"
            << " " << GY(e.j) << " = fma(" << v << " * av" << X << "[" << I << "], gzp" << X << "[" << K << "], fma(" << v
            << " * xv" << X << "[" << I << "], gzc" << X << "[" << K << "], " << GY(e.j) << "));";
      }
      l << " }\n";
      o_ << l.str();
    }
    // ---- per-chunk epilogues ----
    // forward, kind B, two merged chunks: the per-channel weight application of
    // both chunks as one paired FP32 op per component (fma.rn.f32x2: each half
    // the same fma as before, so the bits do not change)
    bool w_paired = false;
    if (f2 && out_z() && cfg_.comp == Comp::Fwd && cfg_.pair_weights) {
      const Sub& s0 = p_.subs[u.subs[g]];
      const Sub& s1 = p_.subs[u.subs[g + n]];
      if (s0.kind == Kind::B && s1.kind == Kind::B && s0.dz() == dz && s1.dz() == dz) {
        const std::string P0 = "pz" + S(u.z_piece_of(s0)), P1 = "pz" + S(u.z_piece_of(s1));
        if (P0 != P1)
        for (int kk = 0; kk < dz; ++kk)
          o_ << "        fma2v(wt_0, wt_1, zx_0[" << kk << "], zx_1[" << kk << "], " << P0 << "[" << kk << "], " << P1
             << "[" << kk << "]);\n";
        w_paired = P0 != P1;
      }
    }
    for (int c = 0; c < m; ++c) {
      const int qi = g + c * n;
      const Sub& s = p_.subs[u.subs[qi]];
      const std::string X = "_" + S(c);
      const std::string PZ = "pz" + S(u.z_piece_of(s));
      const long long swq = Cl.sw[qi];
      const std::string gzs = reads_gz() ? S(L.gz_slot.at(s.z_off)) : "";
      // weight application (z-type outputs)
      if (out_z() && !w_paired) {
        const bool dzm = cfg_.comp != Comp::Fwd;  // dgz = W.(za+zb) + dC.zx
        if (s.kind == Kind::B) {
          for (int kk = 0; kk < dz; ++kk) {
            if (dzm)
              o_ << "        " << PZ << "[" << kk << "] = fma(ct" << X << ", zx" << X << "[" << kk << "], fma(wt" << X << ", za" << X
                 << "[" << kk << "] + zb" << X << "[" << kk << "], " << PZ << "[" << kk << "]));\n";
            else
              o_ << "        " << PZ << "[" << kk << "] = fma(wt" << X << ", zx" << X << "[" << kk << "], " << PZ << "[" << kk << "]);\n";
          }
        } else {
          o_ << "        if (lane < " << s.bp << ") {";
          for (int kk = 0; kk < dz; ++kk) {
            if (dzm)
              o_ << " zs[lane * " << dz << " + " << kk << "] = za" << X << "[" << kk << "] + zb" << X << "[" << kk << "]; zs["
                 << 32 * dz << " + lane * " << dz << " + " << kk << "] = zx" << X << "[" << kk << "];";
            else
              o_ << " zs[lane * " << dz << " + " << kk << "] = zx" << X << "[" << kk << "];";
          }
          o_ << " }\n        { const T* wg = " << wsrc(s, swq, "W") << ";"
             << (dzm ? " const T* cg = " + wsrc(s, swq, "DC") + ";" : "") << "\n"
             << "#pragma unroll 4\n          for (int r = 0; r < " << s.b << "; ++r) if (lane < " << s.bp
             << ") { wts[r * 33 + lane] = __ldg(wg + r * " << s.w_stride << " + lane);";
          if (dzm) o_ << " cts[r * 33 + lane] = __ldg(cg + r * " << s.w_stride << " + lane);";
          o_ << " } }\n        __syncwarp();\n        if (lane < " << s.b << ") {\n#pragma unroll 4\n"
             << "          for (int c = 0; c < " << s.bp << "; ++c) { const T wv = wts[lane * 33 + c];"
             << (dzm ? " const T cv = cts[lane * 33 + c];" : "");
          for (int kk = 0; kk < dz; ++kk) {
            if (dzm)
              o_ << " " << PZ << "[" << kk << "] = fma(cv, zs[" << 32 * dz << " + c * " << dz << " + " << kk
                 << "], fma(wv, zs[c * " << dz << " + " << kk << "], " << PZ << "[" << kk << "]));";
            else
              o_ << " " << PZ << "[" << kk << "] = fma(wv, zs[c * " << dz << " + " << kk << "], " << PZ << "[" << kk << "]);";
          }
          o_ << " }\n        }\n        __syncwarp();\n";
        }
      }
      // weight gradients (per sub, written directly)
      if (out_w()) {
        auto zk = [&](int kk) {
          return cfg_.comp == Comp::Bwd ? "zx" + X + "[" + S(kk) + "]" : "(za" + X + "[" + S(kk) + "] + zb" + X + "[" + S(kk) + "])";
        };
        if (s.kind == Kind::B && pair_b) {
          if (c == 1) {  // both chunks' chains side by side
            const int q0 = g;
            const Sub& sa = p_.subs[u.subs[q0]];
            o_ << "        { T g0 = 0, g1 = 0;";
            for (int kk = 0; kk < dz; ++kk)
              o_ << " fma2v(gz_0[" << kk << "], gz_1[" << kk << "], zx_0[" << kk << "], zx_1[" << kk << "], g0, g1);";
            o_ << " if (lane < " << sa.b << ") O2[" << wrow << " * (i64)" << nw << " + " << O(sa.w_off, Cl.sw[q0])
               << " + lane] = g0; if (lane < " << s.b << ") O2[" << wrow << " * (i64)" << nw << " + " << O(s.w_off, swq)
               << " + lane] = g1; }\n";
          }
        } else if (s.kind == Kind::B) {
          o_ << "        { T g = 0;";
          for (int kk = 0; kk < dz; ++kk) o_ << " g = fma(gz" << X << "[" << kk << "], " << zk(kk) << ", g);";
          o_ << " if (lane < " << s.b << ") O2[" << wrow << " * (i64)" << nw << " + " << O(s.w_off, swq) << " + lane] = g; }\n";
        } else {
          o_ << "#pragma unroll 2\n        for (int r = 0; r < " << s.b << "; ++r) { T g = 0;";
          for (int kk = 0; kk < dz; ++kk)
            o_ << " g = fma(sl[" << gzs << " + r * " << dz << " + " << kk << "], " << zk(kk) << ", g);";
          o_ << " if (lane < " << s.bp << ") O2[" << wrow << " * (i64)" << nw << " + " << O(s.w_off, swq) << " + r * "
             << s.w_stride << " + lane] = g; }\n";
        }
      }
      if (gfl && out_y())  // each gya entry is always updated by the same lane (same dy -> same mapping)
        emit_multi_sum(s.dy(), [&](int j) { return "gyl" + X + "[" + S(j) + "]"; },
                       "gya[" + S(s.y_off) + " + j_] += s_;");
    }
    o_ << "      }\n";
    if (post_sub)
      for (int c = 0; c < m; ++c) post_sub(g + c * n);
  }
}

// The forward of two edges of a row (sub-slots sb_ and sb_ + LW, y in ya_ /
// yb_) side by side as paired FP32 ops; edge b's contribution is added after
// edge a's in every z piece (and skipped when the item has one edge).
// v * (a0, a1) into (r0, r1) as emitted code: a paired multiply, or for
// |v| = 1 (exact either way) a copy / negation
std::string mul2_coef(double v, const std::string& a0, const std::string& a1, const std::string& r0, const std::string& r1) {
  if (v == 1.0) return " " + r0 + " = " + a0 + "; " + r1 + " = " + a1 + ";";
  if (v == -1.0) return " " + r0 + " = -" + a0 + "; " + r1 + " = -" + a1 + ";";
  return " mul2s((T)" + hexd(v) + ", " + a0 + ", " + a1 + ", " + r0 + ", " + r1 + ");";
}

void Gen::emit_unit_body_edge_pair(int k) {
  const Unit& u = U0(k);
  const Layout& L = lay_[k];
  for (int q = 0; q < static_cast<int>(u.subs.size()); ++q) {
    const Sub& s = p_.subs[u.subs[q]];
    const int dx = s.dx(), dz = s.dz();
    const std::uint32_t xs = L.x_slot.at(s.x_off), ws = L.w_slot.at(q);
    const std::string PZ = "pz" + S(u.z_piece_of(s));
    if (q && cfg_.sub_barrier) o_ << "      asm volatile(\"\" ::: \"memory\");\n";
    o_ << "      { // sub " << u.subs[q] << " (edge pair): l=(" << s.l1 << "," << s.l2 << "," << s.l3 << ") nnz="
       << s.cg->entries.size() << "\n        T xa[" << dx << "], xb[" << dx << "];\n        if (lane < " << s.bp << ") {";
    for (int i = 0; i < dx; ++i)
      o_ << " xa[" << i << "] = sb_[" << xs << " + lane * " << dx << " + " << i << "]; xb[" << i << "] = sb_[LW + " << xs
         << " + lane * " << dx << " + " << i << "];";
    o_ << " } else {";
    for (int i = 0; i < dx; ++i) o_ << " xa[" << i << "] = 0; xb[" << i << "] = 0;";
    o_ << " }\n        const T wa = (lane < " << s.b << ") ? sb_[" << ws << " + lane] : (T)0, wb = (lane < " << s.b
       << ") ? sb_[LW + " << ws << " + lane] : (T)0;\n        T za[" << dz << "] = {}, zb[" << dz << "] = {};\n";
    for (const auto& e : s.cg->entries) {
      const int J = s.y_off + e.j;
      o_ << "        { T ca_, cb_;" << mul2_coef(e.v, "ya_[" + S(J) + "]", "yb_[" + S(J) + "]", "ca_", "cb_") << " fma2v(ca_, cb_, xa["
         << e.i << "], xb[" << e.i << "], za[" << e.k << "], zb[" << e.k << "]); }\n";
    }
    for (int kk = 0; kk < dz; ++kk)
      o_ << "        " << PZ << "[" << kk << "] = fma(wa, za[" << kk << "], " << PZ << "[" << kk << "]); if (two_) " << PZ << "["
         << kk << "] = fma(wb, zb[" << kk << "], " << PZ << "[" << kk << "]);\n";
    o_ << "      }\n";
  }
}

// The backward of two edges into node d (sub-slots sb_ / sb_ + LW; x is the
// node's row, the same for both) side by side as paired FP32 ops. Per-edge
// accumulators axa / axb, gya / gyb and the gW of each edge keep the
// one-edge-per-item order of every addition.
void Gen::emit_unit_body_edge_pair_bwd(int k) {
  const Unit& u = U0(k);
  const Layout& L = lay_[k];
  const std::string nw = S(p_.n_w);
  for (int q = 0; q < static_cast<int>(u.subs.size()); ++q) {
    const Sub& s = p_.subs[u.subs[q]];
    const int dx = s.dx(), dz = s.dz();
    const std::uint32_t xs = L.x_slot.at(s.x_off), ws = L.w_slot.at(q), gs = L.gz_slot.at(s.z_off);
    const std::string AX = S(u.x_chunk_of(s));
    if (q && cfg_.sub_barrier) o_ << "      asm volatile(\"\" ::: \"memory\");\n";
    o_ << "      { // sub " << u.subs[q] << " (edge pair): l=(" << s.l1 << "," << s.l2 << "," << s.l3 << ") nnz="
       << s.cg->entries.size() << "\n        T xv[" << dx << "], ga[" << dz << "], gb[" << dz << "];\n        if (lane < "
       << s.bp << ") {";
    for (int i = 0; i < dx; ++i) o_ << " xv[" << i << "] = sb_[" << xs << " + lane * " << dx << " + " << i << "];";
    o_ << " } else {";
    for (int i = 0; i < dx; ++i) o_ << " xv[" << i << "] = 0;";
    o_ << " }\n        if (lane < " << s.b << ") {";
    for (int kk = 0; kk < dz; ++kk)
      o_ << " ga[" << kk << "] = sb_[" << gs << " + lane * " << dz << " + " << kk << "]; gb[" << kk << "] = sb_[LW + " << gs
         << " + lane * " << dz << " + " << kk << "];";
    o_ << " } else {";
    for (int kk = 0; kk < dz; ++kk) o_ << " ga[" << kk << "] = 0; gb[" << kk << "] = 0;";
    o_ << " }\n        const T wa = (lane < " << s.b << ") ? sb_[" << ws << " + lane] : (T)0, wb = (lane < " << s.b
       << ") ? sb_[LW + " << ws << " + lane] : (T)0;\n        T pa[" << dz << "], pb[" << dz << "], za[" << dz
       << "] = {}, zb[" << dz << "] = {};\n       ";
    for (int kk = 0; kk < dz; ++kk)
      o_ << (cfg_.pair_weights ? " mul2v(wa, wb, ga[" + S(kk) + "], gb[" + S(kk) + "], pa[" + S(kk) + "], pb[" + S(kk) + "]);"
                               : " pa[" + S(kk) + "] = wa * ga[" + S(kk) + "]; pb[" + S(kk) + "] = wb * gb[" + S(kk) + "];");
    o_ << "\n";
    for (const auto& e : s.cg->entries) {
      const std::string v = "(T)" + hexd(e.v), I = S(e.i), K = S(e.k), Jg = S(s.y_off + e.j);
      o_ << "        { T ca_, cb_;" << mul2_coef(e.v, "ya_[" + Jg + "]", "yb_[" + Jg + "]", "ca_", "cb_")
         << " fma2v(ca_, cb_, pa[" << K << "], pb[" << K << "], axa" << AX << "[" << I << "], axb" << AX << "[" << I << "]);"
         << " { const T t_ = " << v << " * xv[" << I << "]; fma2s(t_, pa[" << K << "], pb[" << K << "], gya[" << Jg
         << "], gyb[" << Jg << "]); }"
         << " fma2s(xv[" << I << "], ca_, cb_, za[" << K << "], zb[" << K << "]); }\n";
    }
    o_ << "        { T ea = 0, eb = 0;";
    for (int kk = 0; kk < dz; ++kk) o_ << " fma2v(ga[" << kk << "], gb[" << kk << "], za[" << kk << "], zb[" << kk << "], ea, eb);";
    o_ << "\n          if (lane < " << s.b << ") { O2[eida * (i64)" << nw << " + " << s.w_off << " + lane] = ea; if (two_) O2[eidb * (i64)"
       << nw << " + " << s.w_off << " + lane] = eb; } }\n      }\n";
  }
}

// The warp sums of n <= 32 per-lane values src(0 .. n-1) in one recursive-
// halving reduction (warp_sum_n); `use(j, s)` consumes total j in one lane.
void Gen::emit_multi_sum(int n, const std::function<std::string(int)>& src, const std::string& use) {
  if (n == 1 || !cfg_.multi_sum) {  // one butterfly per value (CGF_GEN=nomsum: the A/B baseline)
    for (int j = 0; j < n; ++j)
      o_ << "      { const T s_ = warp_sum(" << src(j) << "); if (lane == " << j << ") { const int j_ = " << j << "; "
         << use << " } }\n";
    return;
  }
  // split n into reductions of 2^P values (zero-padded) minimising issued
  // instructions: a halving round costs 2 selects + a shuffle + an add per value
  // pair (FP64: 4 + 2 + 1), a plain round a shuffle + an add (FP64: 2 + 1)
  const int pair = cfg_.f64 ? 7 : 4, plain = cfg_.f64 ? 3 : 2;
  auto cost = [&](int P) { return pair * ((1 << P) - 1) + plain * (5 - P); };
  std::vector<int> best(n + 1, 1 << 30), pick(n + 1, 0);
  best[0] = 0;
  for (int m = 1; m <= n; ++m)
    for (int P = 0; P <= 5; ++P) {
      const int c = cost(P) + best[m - std::min(m, 1 << P)];
      if (c < best[m]) { best[m] = c; pick[m] = P; }
    }
  for (int done = 0; done < n;) {
    const int P = pick[n - done], cnt = std::min(n - done, 1 << P);
    o_ << "      { T v_[" << (1 << P) << "] = {";
    for (int j = 0; j < (1 << P); ++j) o_ << (j ? ", " : "") << (j < cnt ? src(done + j) : std::string("(T)0"));
    o_ << "};\n        const T s_ = warp_sum_n<T, " << P << ">(v_); const int j_ = " << done << " + warp_sum_n_idx<" << P
       << ">(lane);\n        if ((lane & " << (1 << (5 - P)) - 1 << ") == 0 && j_ < " << done + cnt << ") { " << use
       << " } }\n";
    done += cnt;
  }
}

void Gen::emit_gy_reduce(const std::string& rowexpr, const std::string& arr) {
  const int dy = p_.dim_y;
  for (int j0 = 0; j0 < dy; j0 += 32) {
    const int n = std::min(dy - j0, 32);
    emit_multi_sum(n, [&](int j) { return arr + "[" + S(j0 + j) + "]"; },
                   "O1[" + rowexpr + " * (i64)" + S(dy) + " + " + S(j0) + " + j_] " + (cfg_.gy_accum ? "+=" : "=") + " s_;");
  }
}

// A later group of a grouped kernel continues the running dy sum where the
// earlier groups left it (in O1): the per-sub additions then happen in the
// same order as in one ungrouped kernel, so any grouping gives bit-identical
// dy (and a single-edge conv equals one TP call bitwise).
void Gen::emit_gy_resume(const std::string& rowexpr) {
  o_ << "    for (int j = lane; j < " << p_.dim_y << "; j += 32) gya[j] = O1[" << rowexpr << " * (i64)" << p_.dim_y
     << " + j];\n    __syncwarp();\n";
}

void Gen::emit_gy_flush_row(const std::string& rowexpr) {
  o_ << "    __syncwarp();\n    for (int j = lane; j < " << p_.dim_y << "; j += 32) { O1[" << rowexpr << " * (i64)"
     << p_.dim_y << " + j] = gya[j]; gya[j] = 0; }\n    __syncwarp();\n";
}

std::string zero_init(const std::string& name, int n) { return "T " + name + "[" + S(n) + "] = {};"; }

void Gen::emit_class_loop_open(int k) {
  const UClass& C = cls_[k];
  if (C.n > 1)
    o_ << "#pragma unroll 1\n    for (int kc = 0; kc < " << C.n << "; ++kc) { // ---- class " << k << ": units "
       << C.u0 << ".." << C.u0 + C.n - 1 << "\n";
  else
    o_ << "    { const int kc = 0; (void)kc; // ---- class " << k << ": unit " << C.u0 << "\n";
}

void Gen::emit_class_loop_close(int) { o_ << "    }\n"; }

void Gen::emit_rows_loop() {
  if (yreg())
    o_ << "  T y[" << p_.dim_y << "], yn[" << p_.dim_y << "];"
       << (dual() ? " T db[" + S(p_.dim_y) + "], dbn[" + S(p_.dim_y) + "];" : "") << "\n";
  o_ << "  i64 pn = 0;  // next item to issue (lane 0)\n"
        "#define producer_next() do { if (pn < total) {\\\n"
        "    const i64 rr_ = pn / NU; const int u_ = (int)(pn - rr_ * NU); const i64 r_ = gwarp + rr_ * nwarp;\\\n"
        "    const int s_ = (int)(pn % D);\\\n"
     << (edges() ? "    issue_unit(u_, (i64)EID[r_], (i64)NB[r_], r_, rows, edges_tot,"
                 : "    issue_unit(u_, r_, r_, r_, rows, rows,")
     << " wsm + s_ * SLOT_WORDS, &bars[s_], X, Y, W, GZ, DA, DB, DC" << (cfg_.lane_copy ? ", lane, true" : "") << ");\\\n"
        "    ++pn; } } while (0)\n"
        "  " << (cfg_.lane_copy ? "" : "if (lane == 0) ") << "for (int d = 0; d < D; ++d) producer_next();\n"
        "  int slot = 0; u32 phase = 0;\n"
        "  for (i64 rr = 0; rr < my_rows; ++rr) {\n";
  // the item index: a batch row, or (atomic conv) an edge with its output node
  // (row = src) and neighbour (nbr = dst)
  const std::string it = edges() ? "eid" : "row";
  if (edges())
    o_ << "    const i64 eid = gwarp + rr * nwarp;\n    const i64 row = EID[eid], nbr = NB[eid];\n";
  else
    o_ << "    const i64 row = gwarp + rr * nwarp;\n    const i64 nbr = row, eid = row; (void)nbr; (void)eid;\n";
  if (yreg()) {
    const int dy = p_.dim_y;
    o_ << "    if (rr == 0) {";
    for (int j = 0; j < dy; ++j) {
      o_ << " yn[" << j << "] = __ldg(Y + " << it << " * " << dy << " + " << j << ");";
      if (dual()) o_ << " dbn[" << j << "] = __ldg(DB + " << it << " * " << dy << " + " << j << ");";
    }
    o_ << " }\n   ";
    for (int j = 0; j < dy; ++j)
      o_ << " y[" << j << "] = yn[" << j << "];" << (dual() ? " db[" + S(j) + "] = dbn[" + S(j) + "];" : "");
    o_ << "\n    if (rr + 1 < my_rows) {";
    for (int j = 0; j < dy; ++j) {
      o_ << " yn[" << j << "] = __ldg(Y + (" << it << " + nwarp) * " << dy << " + " << j << ");";
      if (dual()) o_ << " dbn[" << j << "] = __ldg(DB + (" << it << " + nwarp) * " << dy << " + " << j << ");";
    }
    o_ << " }\n";
  }
  if (out_y() && !gy_flush()) o_ << "    " << zero_init("gy", p_.dim_y) << "\n";
  if (gy_flush() && cfg_.gy_accum) emit_gy_resume(it);
  for (size_t k = 0; k < cls_.size(); ++k) {
    const UClass& C = cls_[k];
    const Unit& u = U0(static_cast<int>(k));
    emit_class_loop_open(static_cast<int>(k));
    std::map<std::uint32_t, int> xdx, xb, zdz, zb;
    for (int si : u.subs) {
      const Sub& s = p_.subs[si];
      xdx[s.x_off] = s.dx();
      xb[s.x_off] = s.bp;
      zdz[s.z_off] = s.dz();
      zb[s.z_off] = s.b;
    }
    if (out_x())
      for (size_t c = 0; c < u.x_chunks.size(); ++c) o_ << "      " << zero_init("ax" + S(c), xdx[u.x_chunks[c].off]) << "\n";
    if (out_z())
      for (size_t z = 0; z < u.z_pieces.size(); ++z) o_ << "      " << zero_init("pz" + S(z), zdz[u.z_pieces[z].off]) << "\n";
    emit_wait_and_sync(static_cast<int>(k));
    // Store every owned output right after the last subkernel that writes it.
    std::map<int, std::vector<int>> x_done, z_done;
    for (size_t c = 0; c < u.x_chunks.size(); ++c) {
      int last = 0;
      for (size_t q = 0; q < u.subs.size(); ++q)
        if (p_.subs[u.subs[q]].x_off == u.x_chunks[c].off) last = static_cast<int>(q);
      x_done[last].push_back(static_cast<int>(c));
    }
    for (size_t z = 0; z < u.z_pieces.size(); ++z) {
      int last = 0;
      for (size_t q = 0; q < u.subs.size(); ++q)
        if (p_.subs[u.subs[q]].z_off == u.z_pieces[z].off) last = static_cast<int>(q);
      z_done[last].push_back(static_cast<int>(z));
    }
    emit_unit_body(static_cast<int>(k), [&](int q) {
      if (out_x())
        for (int c : x_done[q]) {
          const auto& xc = u.x_chunks[c];
          emit_store("O0", edges() ? (cfg_.edge_partials ? "eid" : "nbr") : "row", p_.dim_x, xc.off, C.xstep[c],
                     xc.words, xb[xc.off], xdx[xc.off], "ax" + S(c), edges() && !cfg_.edge_partials);
        }
      if (out_z())
        for (int z : z_done[q]) {
          const auto& zp = u.z_pieces[z];
          emit_store(cfg_.comp == Comp::Fwd ? "O0" : "O3", "row", p_.dim_z, zp.off, C.zstep[z], zp.words, zb[zp.off],
                     zdz[zp.off], "pz" + S(z), edges());
        }
    });
    emit_release();
    emit_class_loop_close(static_cast<int>(k));
  }
  if (out_y()) {
    if (gy_flush())
      emit_gy_flush_row(it);
    else
      emit_gy_reduce(it);
  }
  o_ << "  }\n";
}

void Gen::emit_conv_loop() {
  const bool bi = by_input();
  // The producer (lane 0) walks (row, unit, edge) [ByOutput] or (row, edge,
  // unit) [ByInput]; the neighbour / edge-id of the NEXT edge is loaded one
  // step ahead so the index fetch never sits on the critical path.
  o_ << "  i64 pk = 0, pq = 0, pq1 = 0, pq0 = 0, pnb = 0, peid = 0; int pu = 0;\n"
        "#define prow(k) (gwarp + (k) * nwarp)\n"
        "#define seek() do { while (pk < my_rows) { const i64 r_ = prow(pk); pq0 = pq = RP[r_]; pq1 = RP[r_ + 1]; if (pq < pq1) break; ++pk; } } while (0)\n"
        "#define fetch_idx() do { if (pk < my_rows) { pnb = NB[pq]; peid = " << (bi ? "EID[pq]" : "pq") << "; } } while (0)\n"
        "  " << (cfg_.lane_copy ? "" : "if (lane == 0) ") << "{ seek(); fetch_idx(); }\n"
        "  int pslot = 0;\n"
        "#define producer_next() do { if (pk < my_rows) {\\\n"
        "    const i64 r_ = prow(pk);\\\n";
  if (eb() > 1) {
    // EB consecutive edges of the row per item, each in its own sub-slot
    o_ << "    for (int e_ = 0; e_ < EB; ++e_) { const bool v_ = pq + e_ < pq1; const i64 q_ = v_ ? pq + e_ : pq;\\\n"
          "      issue_unit(pu, r_, (i64)NB[q_], " << (bi ? "(i64)EID[q_]" : "q_") << ", rows, edges_tot, wsm + pslot * SLOT_WORDS + e_ * LW, &bars[pslot],"
          " X, Y, W, GZ, DA, DB, DC, lane, v_); }\\\n"
          "    if (++pslot == D) pslot = 0;\\\n"
          "    pq += EB; if (pq >= pq1) { pq = pq0; if (++pu == NU) { pu = 0; ++pk; seek(); } }\\\n";
  } else {
    o_ << "    issue_unit(pu, r_, pnb, peid, rows, edges_tot, wsm + pslot * SLOT_WORDS, &bars[pslot], X, Y, W, GZ, DA, DB, DC"
       << (cfg_.lane_copy ? ", lane, true" : "") << ");\\\n"
          "    if (++pslot == D) pslot = 0;\\\n";
    o_ << (bi ? "    if (++pu == NU) { pu = 0; if (++pq == pq1) { ++pk; seek(); } fetch_idx(); }\\\n"
              : "    if (++pq == pq1) { pq = pq0; if (++pu == NU) { pu = 0; ++pk; seek(); } } fetch_idx();\\\n");
  }
  o_ << "  } } while (0)\n"
        "  " << (cfg_.lane_copy ? "" : "if (lane == 0) ") << "for (int d = 0; d < D; ++d) producer_next();\n"
        "  int slot = 0; u32 phase = 0;\n"
        "  for (i64 k = 0; k < my_rows; ++k) {\n    const i64 row = prow(k);\n"
        "    const i64 q0 = RP[row], q1 = RP[row + 1];\n";
  if (!bi) {
    for (size_t k = 0; k < cls_.size(); ++k) {
      const UClass& C = cls_[k];
      const Unit& u = U0(static_cast<int>(k));
      std::map<std::uint32_t, int> zdz, zb;
      for (int si : u.subs) {
        zdz[p_.subs[si].z_off] = p_.subs[si].dz();
        zb[p_.subs[si].z_off] = p_.subs[si].b;
      }
      emit_class_loop_open(static_cast<int>(k));
      for (size_t z = 0; z < u.z_pieces.size(); ++z) o_ << "      " << zero_init("pz" + S(z), zdz[u.z_pieces[z].off]) << "\n";
      if (pair_edges()) {
        // two edges per item computed as paired FP32 ops (FFMA2 / FMUL2);
        // each z piece still accumulates edge by edge in order (same bits)
        o_ << "      for (i64 q = q0; q < q1; q += 2) {\n      T* sb_ = wsm + slot * SLOT_WORDS;\n      "
           << (cfg_.wait_sleep ? "mbar_wait_sleep" : "mbar_wait") << "(&bars[slot], phase);\n"
           << "      const bool two_ = q + 1 < q1;\n      T ya_[" << p_.dim_y << "], yb_[" << p_.dim_y << "];\n";
        for (int h = 0; h < 2; ++h) {
          o_ << "      { const i64 eid = q + (two_ ? " << h << " : 0); const i64 nbr = NB[eid]; (void)nbr; T* sl = sb_ + "
             << h << " * LW;\n";
          emit_wait_and_sync(static_cast<int>(k), false);
          o_ << "       ";
          for (int j = 0; j < p_.dim_y; ++j) o_ << " y" << (h ? "b" : "a") << "_[" << j << "] = sl[ys + " << j << "];";
          o_ << " }\n";
        }
        emit_unit_body_edge_pair(static_cast<int>(k));
        emit_release();
        o_ << "      }\n";
      } else if (eb() > 1) {
        o_ << "      for (i64 q = q0; q < q1; q += EB) {\n      T* sb_ = wsm + slot * SLOT_WORDS;\n      "
           << (cfg_.wait_sleep ? "mbar_wait_sleep" : "mbar_wait") << "(&bars[slot], phase);\n"
           << "      const int ne_ = (int)(q1 - q < EB ? q1 - q : EB);\n#pragma unroll 1\n"
           << "      for (int e_ = 0; e_ < ne_; ++e_) {\n      const i64 eid = q + e_; const i64 nbr = NB[eid]; (void)nbr;\n"
           << "      T* sl = sb_ + e_ * LW;\n";
        emit_wait_and_sync(static_cast<int>(k), false);
        emit_unit_body(static_cast<int>(k));
        o_ << "      }\n";
        emit_release();
        o_ << "      }\n";
      } else {
        o_ << "      for (i64 q = q0; q < q1; ++q) {\n      const i64 eid = q; const i64 nbr = NB[q]; (void)nbr;\n";
        emit_wait_and_sync(static_cast<int>(k));
        emit_unit_body(static_cast<int>(k));
        emit_release();
        o_ << "      }\n";
      }
      for (size_t z = 0; z < u.z_pieces.size(); ++z) {
        const auto& zp = u.z_pieces[z];
        emit_store(cfg_.comp == Comp::Fwd ? "O0" : "O3", "row", p_.dim_z, zp.off, C.zstep[z], zp.words, zb[zp.off],
                   zdz[zp.off], "pz" + S(z));
      }
      emit_class_loop_close(static_cast<int>(k));
    }
  } else {
    // gx-type outputs accumulate over the row's edges in the warp's shared
    // gxs[dim_x]; each item adds its register partials (lane-owned, conflict-free).
    if (pair_edges_bwd()) {
      // two edges of the node per item as paired FP32 ops; every output is
      // still accumulated edge by edge in order (same bits as one edge per item)
      const Unit& u = U0(0);
      std::map<std::uint32_t, int> xdx, xb;
      for (int si : u.subs) {
        xdx[p_.subs[si].x_off] = p_.subs[si].dx();
        xb[p_.subs[si].x_off] = p_.subs[si].bp;
      }
      o_ << "    for (i64 q = q0; q < q1; q += 2) {\n      const bool two_ = q + 1 < q1;\n"
            "      const i64 eida = EID[q], eidb = EID[two_ ? q + 1 : q];\n"
         << "      " << zero_init("gya", p_.dim_y) << " " << zero_init("gyb", p_.dim_y) << "\n";
      for (size_t c = 0; c < u.x_chunks.size(); ++c)
        o_ << "      " << zero_init("axa" + S(c), xdx[u.x_chunks[c].off]) << " "
           << zero_init("axb" + S(c), xdx[u.x_chunks[c].off]) << "\n";
      o_ << "      T* sb_ = wsm + slot * SLOT_WORDS;\n      " << (cfg_.wait_sleep ? "mbar_wait_sleep" : "mbar_wait")
         << "(&bars[slot], phase);\n      T ya_[" << p_.dim_y << "], yb_[" << p_.dim_y << "];\n";
      for (int h = 0; h < 2; ++h) {
        o_ << "      { const i64 eid = " << (h ? "eidb" : "eida") << "; const i64 nbr = NB[q + (two_ ? " << h
           << " : 0)]; (void)nbr; T* sl = sb_ + " << h << " * LW;\n";
        emit_wait_and_sync(0, false);
        o_ << "       ";
        for (int j = 0; j < p_.dim_y; ++j) o_ << " y" << (h ? "b" : "a") << "_[" << j << "] = sl[ys + " << j << "];";
        o_ << " }\n";
      }
      emit_unit_body_edge_pair_bwd(0);
      for (const char* h : {"a", "b"}) {
        if (h[0] == 'b') o_ << "      if (two_) {\n";
        for (size_t c = 0; c < u.x_chunks.size(); ++c) {
          const auto& xc = u.x_chunks[c];
          const int dx = xdx[xc.off];
          o_ << "      if (lane < " << xb[xc.off] << ") {";
          for (int i = 0; i < dx; ++i)
            o_ << " gxs[" << gx_base_[0] + gx_pre_[0][c] << " + lane * " << dx << " + " << i << "] += ax" << h << c << "["
               << i << "];";
          o_ << " }\n";
        }
        if (h[0] == 'b') o_ << "      }\n";
      }
      emit_release();
      emit_gy_reduce("eida", "gya");
      o_ << "    if (two_) {\n";
      emit_gy_reduce("eidb", "gyb");
      o_ << "    }\n    }\n";
    } else {
    o_ << "    for (i64 q = q0; q < q1; ++q) {\n      const i64 eid = EID[q]; const i64 nbr = NB[q]; (void)nbr;\n";
    if (out_y() && !gy_flush()) o_ << "      " << zero_init("gy", p_.dim_y) << "\n";
    if (gy_flush() && cfg_.gy_accum) emit_gy_resume("eid");
    for (size_t k = 0; k < cls_.size(); ++k) {
      const Unit& u = U0(static_cast<int>(k));
      std::map<std::uint32_t, int> xdx, xb;
      for (int si : u.subs) {
        xdx[p_.subs[si].x_off] = p_.subs[si].dx();
        xb[p_.subs[si].x_off] = p_.subs[si].bp;
      }
      emit_class_loop_open(static_cast<int>(k));
      for (size_t c = 0; c < u.x_chunks.size(); ++c) o_ << "      " << zero_init("ax" + S(c), xdx[u.x_chunks[c].off]) << "\n";
      emit_wait_and_sync(static_cast<int>(k));
      emit_unit_body(static_cast<int>(k));
      for (size_t c = 0; c < u.x_chunks.size(); ++c) {
        const auto& xc = u.x_chunks[c];
        const int dx = xdx[xc.off];
        o_ << "      if (lane < " << xb[xc.off] << ") {";
        for (int i = 0; i < dx; ++i)
          o_ << " gxs[" << O(gx_base_[k] + gx_pre_[k][c], gx_unit_[k]) << " + lane * " << dx << " + " << i << "] += ax" << c
             << "[" << i << "];";
        o_ << " }\n";
      }
      emit_release();
      emit_class_loop_close(static_cast<int>(k));
    }
    if (out_y()) {
      if (gy_flush())
        emit_gy_flush_row("eid");
      else
        emit_gy_reduce("eid");
    }
    o_ << "    }\n";
    }
    // the row's packed x chunks -> their places in the output row
    o_ << "    __syncwarp();\n";
    for (size_t k = 0; k < cls_.size(); ++k) {
      const UClass& C = cls_[k];
      const Unit& u = U0(static_cast<int>(k));
      o_ << "#pragma unroll 1\n    for (int kc = 0; kc < " << C.n << "; ++kc) {\n";
      for (size_t c = 0; c < u.x_chunks.size(); ++c) {
        const auto& xc = u.x_chunks[c];
        const bool vec = cfg_.aligned && al16(p_.dim_x) && al16(xc.off) && al16(C.xstep[c]) && al16(xc.words) &&
                         al16(gx_base_[k] + gx_pre_[k][c]) && al16(gx_unit_[k]);
        const std::string at = "O0 + row * (i64)" + S(p_.dim_x) + " + " + O(xc.off, C.xstep[c]);
        const std::string from = "gxs + " + O(gx_base_[k] + gx_pre_[k][c], gx_unit_[k]);
        if (!cfg_.unrolled_stores)
          o_ << "      " << (vec ? "coop_store16(" : "coop_store(") << at << ", " << from << ", "
             << (vec ? xc.words * sz_ / 16 : xc.words) << ", lane);\n";
        else if (vec)
          o_ << "      coop_store16n<" << xc.words * sz_ / 16 << ">(" << at << ", " << from << ", lane);\n";
        else
          o_ << "      coop_storen<" << xc.words << ">(" << at << ", " << from << ", lane);\n";
      }
      o_ << "    }\n";
    }
    o_ << "    __syncwarp();\n    for (int j = lane; j < " << gx_words_ << "; j += 32) gxs[j] = 0;\n    __syncwarp();\n";
  }
  o_ << "  }\n";
}

KernelSource Gen::run() {
  if (conv() && cfg_.w_shared) throw UnsupportedError("shared weights are not supported in the fused convolution");
  if (cfg_.loop == Loop::ConvByOutput && !(cfg_.comp == Comp::Fwd || cfg_.comp == Comp::DBwdZ))
    throw UnsupportedError("ConvByOutput computes z-type outputs only");
  if (cfg_.loop == Loop::ConvByInput && !(cfg_.comp == Comp::Bwd || cfg_.comp == Comp::DBwdX))
    throw UnsupportedError("ConvByInput computes x-type outputs only");
  // (the split double-backward passes also run on batched rows: two smaller
  // kernels instead of one that overflows the instruction cache)
  if (edges() && (cfg_.comp == Comp::DBwdZ || cfg_.comp == Comp::DBwdX))
    throw UnsupportedError("the atomic edge-list conv runs the double-backward in one pass");
  classify();
  layout();
  std::uint32_t slot_words = 0;
  int bulk = 0, sync = 0;
  for (const auto& L : lay_) {
    slot_words = std::max(slot_words, L.words);
    for (const auto& r : L.ranges) (r.bulk ? bulk : sync)++;
  }
  const std::uint32_t lw = up(slot_words);  // one edge's sub-slot (multi-edge items)
  if (eb() > 1) slot_words = lw * static_cast<std::uint32_t>(eb());
  // Default ring depth: ~12 KB of staged inputs per warp, 2..4 slots.
  int depth = cfg_.depth > 0 ? cfg_.depth
                             : static_cast<int>(std::clamp<std::uint64_t>(12288 / std::max<std::uint64_t>(1, slot_words * sz_), 2, 4));
  int warps = cfg_.warps;
  auto warp_bytes = [&](int d) { return (static_cast<std::uint64_t>(d) * slot_words + scr_words_) * sz_; };
  const std::uint64_t budget = 224 * 1024;  // of the 227 KB a CTA may use
  while (depth > 1 && warp_bytes(depth) * warps + 8ull * depth * warps > budget) --depth;
  while (warps > 1 && warp_bytes(depth) * warps + 8ull * depth * warps > budget) --warps;
  if (warp_bytes(depth) * warps + 8ull * depth * warps > 227 * 1024)
    throw UnsupportedError("problem too large for one warp's shared-memory slot (" + S(warp_bytes(1)) + " bytes)");
  const std::uint64_t wb = (warp_bytes(depth) + 127) / 128 * 128;
  static const char* compn[] = {"fwd", "bwd", "dbwd", "dbwdz", "dbwdx"};
  static const char* loopn[] = {"tp", "convo", "convi", "conve"};
  KernelSource ks;
  ks.name = std::string("cgf_") + loopn[static_cast<int>(cfg_.loop)] + "_" + compn[static_cast<int>(cfg_.comp)] +
            (cfg_.f64 ? "_f64" : "_f32") + (cfg_.w_shared ? "_ws" : "") + (cfg_.aligned ? "" : "_u") +
            (cfg_.tag.empty() ? "" : "_" + cfg_.tag);
  ks.threads = warps * 32;
  ks.smem_bytes = static_cast<int>(wb * warps + 8ull * depth * warps);
  ks.units = static_cast<int>(units_.size());
  ks.bulk_ranges = bulk;
  ks.sync_ranges = sync;

  o_ << device_runtime_source();
  o_ << "\n// Generated for: x = " << p_.x_ir.str() << " | y = " << p_.y_ir.str() << " | z = " << p_.z_ir.str()
     << "\n// " << p_.subs.size() << " split subkernels in " << units_.size() << " units / " << cls_.size()
     << " code classes; " << ks.name << "\n";
  o_ << "typedef " << (cfg_.f64 ? "double" : "float") << " T;\n";
  o_ << "#define NW " << warps << "\n#define D " << depth << "\n#define NU " << units_.size() << "\n#define SLOT_WORDS "
     << slot_words << "\n#define WARP_BYTES " << wb << "\n#define EB " << eb() << "\n#define LW " << lw << "\n\n";
  emit_issue();
  o_ << "extern \"C\" __global__ void __launch_bounds__(NW * 32"
     << (cfg_.min_blocks > 0 ? ", " + S(cfg_.min_blocks) : "") << ") " << ks.name
     << "(const T* __restrict__ X, const T* __restrict__ Y, const T* __restrict__ W,"
        " const T* __restrict__ GZ, const T* __restrict__ DA, const T* __restrict__ DB,"
        " const T* __restrict__ DC, T* __restrict__ O0, T* __restrict__ O1, T* __restrict__ O2,"
        " T* __restrict__ O3, i64 rows, const i64* __restrict__ RP, const int* __restrict__ NB,"
        " const int* __restrict__ EID, i64 edges_tot) {\n"
        "  extern __shared__ __align__(128) unsigned char smem_raw[];\n"
        "  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;\n"
        "  T* wsm = (T*)(smem_raw + wid * WARP_BYTES);\n"
        "  T* scr = wsm + D * SLOT_WORDS;\n";
  if (has_c_)
    o_ << "  T* zs = scr + " << off_zs_ << "; T* wts = scr + " << off_wt_ << ";"
       << (dual() ? " T* cts = scr + " + S(off_ct_) + ";" : "") << " (void)zs; (void)wts;\n";
  o_ << "  T* gya = scr + " << off_gya_ << "; (void)gya;\n"
     << "  for (int j = lane; j < " << p_.dim_y << "; j += 32) gya[j] = 0;\n";
  if (by_input())
    o_ << "  T* gxs = scr + " << off_gxs_ << ";\n  for (int j = lane; j < " << gx_words_ << "; j += 32) gxs[j] = 0;\n";
  o_ << "  u64* bars = (u64*)(smem_raw + NW * WARP_BYTES) + wid * D;\n"
        "  if (lane == 0) { for (int d = 0; d < D; ++d) mbar_init(&bars[d], " << (cfg_.lane_copy && !cfg_.par_bulk ? 32 : 1) * eb() << "); mbar_fence_init(); }\n"
        "  __syncwarp();\n"
        "  const i64 gwarp = (i64)blockIdx.x * NW + wid, nwarp = (i64)gridDim.x * NW;\n"
        "  const i64 n_items = " << (edges() ? "edges_tot" : "rows") << ";\n"
        "  const i64 my_rows = gwarp < n_items ? (n_items - 1 - gwarp) / nwarp + 1 : 0;\n"
        "  const i64 total = my_rows * NU; (void)total;\n";
  if (conv() && !edges())
    emit_conv_loop();
  else
    emit_rows_loop();
  o_ << "}\n";
  ks.source = o_.str();
  return ks;
}

}  // namespace

void apply_gen_flags(KernelConfig& cfg, const std::string& flags) {
  std::stringstream ss(flags);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    if (tok.empty()) continue;
    const auto eq = tok.find('=');
    const std::string k = tok.substr(0, eq);
    const int v = eq == std::string::npos ? 0 : std::atoi(tok.c_str() + eq + 1);
    if (k == "depth") cfg.depth = std::max(0, v);
    else if (k == "warps") cfg.warps = std::max(1, v);
    else if (k == "minb") cfg.min_blocks = std::max(0, v);
    else if (k == "nobarrier") cfg.sub_barrier = false;
    else if (k == "barrier") cfg.sub_barrier = true;
    else if (k == "yreg") cfg.y_regs = true;
    else if (k == "yslot") cfg.y_regs = false;
    else if (k == "class") cfg.max_class = std::max(1, v);
    else if (k == "bulk") cfg.lane_copy = false;
    else if (k == "merge") cfg.merge = std::max(1, v);
    else if (k == "lanecopy") cfg.lane_copy = true;
    else if (k == "nojoint") cfg.joint = false;
    else if (k == "ywin") cfg.y_window = true;
    else if (k == "oldissue") cfg.old_issue = true;
    else if (k == "pbulk") cfg.par_bulk = true;
    else if (k == "mergeall") cfg.merge_all = true;
    else if (k == "nomergeall") cfg.merge_all = false;
    else if (k == "nopbulk") cfg.par_bulk = false;
    else if (k == "newissue") cfg.old_issue = false;
    else if (k == "noywin") cfg.y_window = false;
    else if (k == "joint") cfg.joint = true;
    else if (k == "epi") cfg.edges_per_item = std::max(1, v);
    else if (k == "pairedges") cfg.pair_edges = true;
    else if (k == "nopairedges") cfg.pair_edges = false;
    else if (k == "ffma2") cfg.ffma2 = true;
    else if (k == "noffma2") cfg.ffma2 = false;
    else if (k == "waitsleep") cfg.wait_sleep = true;
    else if (k == "nowaitsleep") cfg.wait_sleep = false;
    else if (k == "edgepart") cfg.edge_partials = true;
    else if (k == "nomsum") cfg.multi_sum = false;
    else if (k == "loopstores") cfg.unrolled_stores = false;
    else if (k == "ustores") cfg.unrolled_stores = true;
    else if (k == "pairw") cfg.pair_weights = true;
    else if (k == "nopairw") cfg.pair_weights = false;
    else if (k == "l2hint") cfg.l2_hints = true;
    else if (k == "nol2hint") cfg.l2_hints = false;
    else if (k == "xregs") cfg.x_regs = true;
    else if (k == "noxregs") cfg.x_regs = false;
    else if (k == "yitem") cfg.y_item = true;
    else if (k == "noyitem") cfg.y_item = false;
  }
}

namespace {
// Merges runs of up to `m` consecutive same-shape units (the 32-lane chunks of
// the same instructions) into one unit: one staging item and one code body
// then cover m chunks, so the per-item bookkeeping and the lane-uniform CG
// products (v * y[j], shared by every chunk) are paid once per m chunks.
std::vector<Unit> merge_units(const Problem& p, const std::vector<Unit>& units, int m) {
  if (m <= 1) return units;
  std::vector<Unit> out;
  size_t i = 0;
  while (i < units.size()) {
    size_t j = i + 1;
    while (j < units.size() && static_cast<int>(j - i) < m && same_shape(p, units[i], units[j])) ++j;
    Unit u = units[i];
    u.merged = static_cast<int>(j - i);
    for (size_t k = i + 1; k < j; ++k) {
      const Unit& v = units[k];
      u.subs.insert(u.subs.end(), v.subs.begin(), v.subs.end());
      for (const auto& c : v.x_chunks) {
        bool have = false;
        for (const auto& e : u.x_chunks) have = have || e.off == c.off;
        if (!have) u.x_chunks.push_back(c);
      }
      for (const auto& z : v.z_pieces) {
        bool have = false;
        for (const auto& e : u.z_pieces) have = have || e.off == z.off;
        if (!have) u.z_pieces.push_back(z);
      }
    }
    out.push_back(std::move(u));
    i = j;
  }
  return out;
}
}  // namespace

// All units as one (one staged item per row / edge): for problems whose whole
// output row fits a warp's registers (merge_all).
std::vector<Unit> fuse_units(const std::vector<Unit>& units) {
  Unit u;
  for (const auto& v : units) {
    u.subs.insert(u.subs.end(), v.subs.begin(), v.subs.end());
    u.x_chunks.insert(u.x_chunks.end(), v.x_chunks.begin(), v.x_chunks.end());
    u.z_pieces.insert(u.z_pieces.end(), v.z_pieces.begin(), v.z_pieces.end());
  }
  return {u};
}

KernelSource generate_kernel(const Problem& p, const std::vector<Unit>& units, const KernelConfig& cfg) {
  const std::vector<Unit> merged = cfg.merge_all ? fuse_units(units) : merge_units(p, units, cfg.merge);
  Gen g(p, merged, cfg);
  return g.run();
}

}  // namespace cgf
