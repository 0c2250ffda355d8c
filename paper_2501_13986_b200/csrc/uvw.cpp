#include "uvw.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <sstream>

namespace cgf {

namespace {

constexpr int kTileRows = 128;
constexpr int kProdWarps = 8;     // 2 per SM sub-partition: thread = (row, 16 channels)
constexpr int kMmaWarp = 8;
constexpr int kEpiWarp0 = 9;      // warps 9..12: one per TMEM lane quadrant (warp % 4)
constexpr int kWarps = 13;
constexpr int kTmemCols = 512;
constexpr int kASlotBytes = 2 * kTileRows * 128;  // hi + lo, 128 rows x 32 fp32, SW128 K-major

std::string S(long long v) { return std::to_string(v); }

std::string hexd(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return b;
}

struct Seg {
  std::uint32_t z_off = 0;
  int dz = 1, n = 0, col = 0;
  std::vector<int> ins;  // indices into p.resolved
};

}  // namespace

bool uvw_eligible(const Problem& p, std::string* why) {
  auto no = [&](const std::string& m) {
    if (why) *why = m;
    return false;
  };
  if (p.resolved.empty()) return no("no instructions");
  for (const auto& s : p.resolved) {
    if (s.kind != Kind::C) return no("not all instructions are uvw (kind C)");
    if (s.b % 16 || s.b > 256) return no("z multiplicity must be a multiple of 16 and <= 256");
    if (s.bp % 32) return no("x multiplicity must be a multiple of 32");
    if (s.dz() * s.b > kTmemCols) return no("z segment accumulator exceeds TMEM");
    if (s.dx() > 7 || s.dz() > 7) return no("l > 3 not supported by the tensor-core path");
  }
  if (p.dim_z % 4 || p.dim_x % 4) return no("dim_x / dim_z must be multiples of 4");
  for (const auto& s : p.resolved)
    if (s.z_off % 4 || s.x_off % 4) return no("segment offsets must be multiples of 4");
  return true;
}

UvwSource generate_uvw_forward(const Problem& p) {
  std::string why;
  if (!uvw_eligible(p, &why)) throw UnsupportedError("uvw tensor-core path: " + why);
  const auto& R = p.resolved;
  const int np = static_cast<int>(R.size());

  // ---- output segments: every instruction writing one z segment shares its
  // TMEM accumulator; largest first, columns assigned around a 512-col ring.
  std::vector<Seg> segs;
  {
    std::map<std::uint32_t, int> by_z;
    for (int q = 0; q < np; ++q) {
      auto it = by_z.find(R[q].z_off);
      if (it == by_z.end()) {
        by_z[R[q].z_off] = static_cast<int>(segs.size());
        Seg s;
        s.z_off = R[q].z_off;
        s.dz = R[q].dz();
        s.n = R[q].b;
        segs.push_back(s);
        segs.back().ins.push_back(q);
      } else {
        segs[it->second].ins.push_back(q);
      }
    }
    std::stable_sort(segs.begin(), segs.end(), [](const Seg& a, const Seg& b) { return a.dz * a.n > b.dz * b.n; });
    int cur = 0;
    for (auto& s : segs) {
      const int cols = s.dz * s.n;
      if (cur + cols > kTmemCols) cur = 0;
      s.col = cur;
      cur += cols;
    }
  }
  const int ns = static_cast<int>(segs.size());
  auto overlap = [&](int a, int b) {
    const int a0 = segs[a].col, a1 = a0 + segs[a].dz * segs[a].n;
    const int b0 = segs[b].col, b1 = b0 + segs[b].dz * segs[b].n;
    return a0 < b1 && b0 < a1;
  };
  // Before the first MMA into segment s of tile t, wait until every
  // overlapping segment's previous accumulator was drained: those earlier in
  // the order from tile t, those at or after s from tile t-1.
  std::vector<unsigned> wait_cur(ns, 0), wait_prev(ns, 0);
  for (int s = 0; s < ns; ++s)
    for (int o = 0; o < ns; ++o)
      if (overlap(s, o)) (o < s ? wait_cur[s] : wait_prev[s]) |= 1u << o;

  // ---- units: (instruction, 32-channel block) in segment order
  struct U {
    int ins, cb, seg, dz, n;
    bool first, last;
    std::size_t wimg;
  };
  std::vector<U> units;
  int max_n = 16;
  for (const auto& s : segs) max_n = std::max(max_n, s.n);
  const int wslot = 2 * max_n * 128;  // hi + lo, N rows x 32 fp32
  std::size_t wimg = 0;
  std::vector<std::size_t> wimg_of(np, 0);
  for (int q = 0; q < np; ++q) {
    wimg_of[q] = wimg;
    wimg += static_cast<std::size_t>(R[q].bp / 32) * wslot;
  }
  for (int si = 0; si < ns; ++si) {
    const auto& s = segs[si];
    for (size_t t = 0; t < s.ins.size(); ++t) {
      const int q = s.ins[t];
      const int nb = R[q].bp / 32;
      for (int cb = 0; cb < nb; ++cb)
        units.push_back({q, cb, si, s.dz, s.n, t == 0 && cb == 0, t + 1 == s.ins.size() && cb + 1 == nb,
                         wimg_of[q] + static_cast<std::size_t>(cb) * wslot});
    }
  }
  const int nu = static_cast<int>(units.size());
  const int a_slots = std::min(6, (227 * 1024 - 3 * wslot - 1536) / kASlotBytes);
  if (a_slots < 2) throw UnsupportedError("uvw tensor-core path: shared memory too small");
  const int smem = 1024 /*align*/ + a_slots * kASlotBytes + 3 * wslot + 512 /*barriers*/;

  std::ostringstream o;
  if (std::getenv("CGF_UVW_DEBUG")) o << "#define CGF_UVW_DEBUG 1\n";
  o << device_runtime_source();
  o << R"(
// ---- tcgen05 / TMEM helpers (sm_100a) ----
// Bounded wait: a barrier that never completes traps after ~4 s with its tag
// instead of hanging the device.
DEVI u64 gtimer() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
DEVI void mbar_wait_t(u64* b, u32 parity, int tag) {
  if (mbar_try(b, parity)) return;
  const u64 t0 = gtimer();
  for (u32 it = 1;; ++it) {
    if (mbar_try(b, parity)) return;
    if ((it & 1023u) == 0 && gtimer() - t0 > 4000000000ull) {
      printf("cgf_uvw: mbarrier timeout tag=%d block=%d thread=%d parity=%u\n", tag, blockIdx.x, threadIdx.x, parity);
      __trap();
    }
  }
}
DEVI void mbar_arrive(u64* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_addr(b)) : "memory"); }
DEVI void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
DEVI void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// D[tmem] (+)= A[smem] * B[smem]^T, tf32 inputs, fp32 accumulate, single CTA.
DEVI void tc_mma(u32 d, u64 a, u64 b, u32 idesc, u32 acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// Arrive on an mbarrier once every previously issued tcgen05.mma completed.
DEVI void tc_commit(u64* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(b)) : "memory");
}
DEVI void tc_ld8(u32 taddr, float* v) {
  u32 r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
DEVI void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups
// 1024 B apart (SBO), version 1 (sm_100).
DEVI u64 sdesc(u32 saddr) {
  return (u64)((saddr & 0x3FFFFu) >> 4) | ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
}
// Instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M = 128, N.
DEVI constexpr u32 idesc_tf32(int n) { return (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(n >> 3) << 17) | ((u32)(128 >> 4) << 24); }
// tf32 split: hi keeps the top 19 bits (exactly representable), lo the rest.
DEVI float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }
// Byte offset of element (m, c) of a 128 x 32 fp32 K-major SW128 tile.
DEVI u32 sw128(int m, int chunk) { return (u32)((m >> 3) * 1024 + (m & 7) * 128 + ((chunk ^ (m & 7)) << 4)); }
)";
  o << "\n// uvw forward: x = " << p.x_ir.str() << " | y = " << p.y_ir.str() << " | z = " << p.z_ir.str() << "\n";
  o << "// " << np << " instructions, " << ns << " z segments, " << nu << " units / 128-row tile, " << a_slots
    << " A slots\n";
  o << "#define DIMX " << p.dim_x << "\n#define DIMY " << p.dim_y << "\n#define DIMZ " << p.dim_z << "\n#define NW_ "
    << p.n_w << "\n#define NS " << a_slots << "\n#define WSLOT " << wslot << "\n#define NSEG " << ns << "\n";

  // ---- prep kernel: shared W -> per-(instruction, channel block) images
  o << "extern \"C\" __global__ void cgf_uvw_prep_f32(const float* __restrict__ W, float* __restrict__ img) {\n"
       "  const int t = blockIdx.x * blockDim.x + threadIdx.x;\n  int e = t;\n";
  for (int q = 0; q < np; ++q) {
    const auto& s = R[q];
    const int cnt = s.b * s.bp;
    o << "  if (e < " << cnt << ") { const int r = e / " << s.bp << ", c = e % " << s.bp << ", cb = c >> 5, cl = c & 31;\n"
      << "    const float v = W[" << s.w_off << " + r * " << s.w_stride << " + c]; const float h = tf32_hi(v);\n"
      << "    char* base = (char*)img + " << wimg_of[q] << " + (size_t)cb * WSLOT;\n"
      << "    const u32 off = (u32)((r >> 3) * 1024 + (r & 7) * 128 + (((cl >> 2) ^ (r & 7)) << 4) + (cl & 3) * 4);\n"
      << "    *(float*)(base + off) = h; *(float*)(base + " << s.b * 128 << " + off) = v - h; return; }\n"
      << "  e -= " << cnt << ";\n";
  }
  o << "}\n\n";

  // ---- producer: one function per instruction (CG coefficients as immediates)
  for (int q = 0; q < np; ++q) {
    const auto& s = R[q];
    const int dx = s.dx(), dz = s.dz();
    o << "// instruction " << q << ": l=(" << s.l1 << "," << s.l2 << "," << s.l3 << ") b=" << s.b << " b'=" << s.bp
      << " nnz=" << s.cg->entries.size() << "\n";
    o << "DEVI void produce_" << q << "(const float* __restrict__ xr, const float* yv, bool valid, int m, int sub,"
         " unsigned char* abase, u64* afull, u64* aempty, u32& seq) {\n";
    o << "  float q[" << dz << "][" << dx << "];\n#pragma unroll\n  for (int k = 0; k < " << dz
      << "; ++k)\n#pragma unroll\n    for (int i = 0; i < " << dx << "; ++i) q[k][i] = 0.f;\n";
    for (const auto& e : s.cg->entries)
      o << "  q[" << e.k << "][" << e.i << "] = fmaf((float)" << hexd(e.v) << ", yv[" << s.y_off + e.j << "], q[" << e.k
        << "][" << e.i << "]);\n";
    o << "  float xv[" << 16 * dx << "];\n"
      << "  if (valid) {\n#pragma unroll\n    for (int t = 0; t < " << 4 * dx
      << "; ++t) { const float4 v = __ldg((const float4*)xr + t); xv[4*t] = v.x; xv[4*t+1] = v.y; xv[4*t+2] = v.z; xv[4*t+3] = v.w; }\n"
      << "  } else {\n#pragma unroll\n    for (int t = 0; t < " << 16 * dx << "; ++t) xv[t] = 0.f;\n  }\n";
    o << "#pragma unroll\n  for (int k = 0; k < " << dz << "; ++k) {\n"
      << "    const u32 slot = seq % NS, ph = (seq / NS) & 1u;\n"
      << "    mbar_wait_t(&aempty[slot], ph ^ 1u, 1);\n"
      << "    unsigned char* hi = abase + slot * " << kASlotBytes << "; unsigned char* lo = hi + " << kASlotBytes / 2 << ";\n"
      << "#pragma unroll\n    for (int g = 0; g < 4; ++g) {\n"
      << "      float h[4], l[4];\n#pragma unroll\n      for (int cc = 0; cc < 4; ++cc) {\n"
      << "        const int c = 4 * g + cc; float z = 0.f;\n#pragma unroll\n        for (int i = 0; i < " << dx
      << "; ++i) z = fmaf(q[k][i], xv[c * " << dx << " + i], z);\n"
      << "        h[cc] = tf32_hi(z); l[cc] = z - h[cc];\n      }\n"
      << "      const u32 off = sw128(m, 4 * sub + g);\n"
      << "      *(float4*)(hi + off) = make_float4(h[0], h[1], h[2], h[3]);\n"
      << "      *(float4*)(lo + off) = make_float4(l[0], l[1], l[2], l[3]);\n    }\n"
      << "    fence_proxy_async();\n    __syncwarp();\n    if ((threadIdx.x & 31) == 0) mbar_arrive(&afull[slot]);\n"
      << "    ++seq;\n  }\n}\n\n";
  }

  // ---- unit / segment tables
  auto arr = [&](const char* name, const std::vector<long long>& v) {
    o << "__constant__ int " << name << "[" << std::max<size_t>(1, v.size()) << "] = {";
    for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
    if (v.empty()) o << "0";
    o << "};\n";
  };
  {
    std::vector<long long> udz, ucol, un, ufirst, ulast, useg, uw;
    for (const auto& u : units) {
      udz.push_back(u.dz);
      ucol.push_back(segs[u.seg].col);
      un.push_back(u.n);
      ufirst.push_back(u.first);
      ulast.push_back(u.last);
      useg.push_back(u.seg);
      uw.push_back(static_cast<long long>(u.wimg));
    }
    arr("U_DZ", udz);
    arr("U_COL", ucol);
    arr("U_N", un);
    arr("U_FIRST", ufirst);
    arr("U_LAST", ulast);
    arr("U_SEG", useg);
    arr("U_WIMG", uw);
    std::vector<long long> sz, sdz, sn, scol, swc, swp;
    for (int si = 0; si < ns; ++si) {
      sz.push_back(segs[si].z_off);
      sdz.push_back(segs[si].dz);
      sn.push_back(segs[si].n);
      scol.push_back(segs[si].col);
      swc.push_back(wait_cur[si]);
      swp.push_back(wait_prev[si]);
    }
    arr("S_ZOFF", sz);
    arr("S_DZ", sdz);
    arr("S_N", sn);
    arr("S_COL", scol);
    arr("S_WAITCUR", swc);
    arr("S_WAITPREV", swp);
  }
  o << "#define NU " << nu << "\n\n";

  // ---- the main kernel
  o << "extern \"C\" __global__ void __launch_bounds__(" << kWarps * 32 << ", 1) cgf_uvw_fwd_f32("
       "const float* __restrict__ X, const float* __restrict__ Y, const float* __restrict__ WIMG, "
       "const float* __restrict__ GZ, const float* __restrict__ DA, const float* __restrict__ DB, "
       "const float* __restrict__ DC, float* __restrict__ Z, float* __restrict__ O1, float* __restrict__ O2, "
       "float* __restrict__ O3, i64 rows, const i64* __restrict__ RP, const int* __restrict__ NB, "
       "const int* __restrict__ EID, i64 edges_tot) {\n"
       "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
       "  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);\n"
       "  unsigned char* abase = sm;\n"
       "  unsigned char* wbase = sm + NS * "
    << kASlotBytes << ";\n"
       "  u64* bars = (u64*)(wbase + 3 * WSLOT);\n"
       "  u64* afull = bars; u64* aempty = afull + NS; u64* wfull = aempty + NS; u64* wempty = wfull + 3;\n"
       "  u64* sfull = wempty + 3; u64* sdrained = sfull + NSEG;\n"
       "  u32* tmem_slot = (u32*)(sdrained + NSEG);\n"
       "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
       "  const i64 ntiles = (rows + 127) / 128;\n"
       "  if (threadIdx.x == 0) {\n"
       "    for (int i = 0; i < NS; ++i) { mbar_init(&afull[i], "
    << kProdWarps
    << "); mbar_init(&aempty[i], 1); }\n"
       "    for (int i = 0; i < 3; ++i) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], 1); }\n"
       "    for (int i = 0; i < NSEG; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sdrained[i], 4); }\n"
       "    mbar_fence_init();\n  }\n"
       "  if (warp == "
    << kMmaWarp
    << ") {\n"
       "    asm volatile(\"tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\" :: \"r\"(smem_addr(tmem_slot)));\n"
       "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\");\n"
       "  }\n"
       "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n"
       "  const u32 tmem = *tmem_slot;\n\n";

  // producers
  o << "  if (warp < " << kProdWarps
    << ") {\n"
       "    const int m = 32 * (warp & 3) + lane, sub = warp >> 2;\n"
       "    u32 seq = 0;\n"
       "    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
       "      const i64 row = tile * 128 + m;\n"
       "      const bool valid = row < rows;\n"
       "      { const i64 nrow = row + (i64)gridDim.x * 128;  // warm L2 with the next tile's x row\n"
       "        if (nrow < rows) { const char* px = (const char*)(X + nrow * DIMX);\n"
       "          for (int b = sub * 128; b < DIMX * 4; b += 256) asm volatile(\"prefetch.global.L2 [%0];\" :: \"l\"(px + b)); } }\n"
       "      float yv[DIMY];\n"
       "#pragma unroll\n      for (int j = 0; j < DIMY; ++j) yv[j] = valid ? __ldg(Y + row * DIMY + j) : 0.f;\n"
       "      const float* xrow = X + (valid ? row : 0) * DIMX;\n";
  for (const auto& u : units) {
    const auto& s = R[u.ins];
    const long long c0 = static_cast<long long>(u.cb) * 32;
    o << "      produce_" << u.ins << "(xrow + " << s.x_off << " + (" << c0 << " + 16 * sub) * " << s.dx()
      << ", yv, valid, m, sub, abase, afull, aempty, seq);\n";
  }
  o << "    }\n  }\n";

  // MMA issuer
  o << "  else if (warp == " << kMmaWarp
    << ") {\n"
       "    if (lane == 0) {\n"
       "      u32 seq = 0, gu = 0; i64 lt = 0;\n"
       "      const i64 my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;\n"
       "      const i64 total_units = my_tiles * NU;\n"
       "      auto load_w = [&](u32 g) {  // W ring of 3, loaded two units ahead\n"
       "        const int u = (int)(g % NU); const u32 sl = g % 3u;\n"
       "        if (g >= 3) mbar_wait_t(&wempty[sl], (g / 3u - 1u) & 1u, 2);\n"
       "        mbar_expect_tx(&wfull[sl], WSLOT);\n"
       "        bulk_g2s(wbase + sl * WSLOT, (const char*)WIMG + U_WIMG[u], WSLOT, &wfull[sl]);\n"
       "      };\n"
       "      if (total_units > 0) load_w(0);\n"
       "      if (total_units > 1) load_w(1);\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {\n"
       "        for (int u = 0; u < NU; ++u, ++gu) {\n"
       "          if (U_FIRST[u]) {\n"
       "            const int s = U_SEG[u];\n"
       "            for (int o = 0; o < NSEG; ++o) {\n"
       "              if (S_WAITCUR[s] >> o & 1) mbar_wait_t(&sdrained[o], (u32)(lt & 1), 3);\n"
       "              if ((S_WAITPREV[s] >> o & 1) && lt > 0) mbar_wait_t(&sdrained[o], (u32)((lt - 1) & 1), 4);\n"
       "            }\n"
       "            tc_fence_after();\n"
       "          }\n"
       "          const u32 wsl = gu % 3u;\n"
       "          mbar_wait_t(&wfull[wsl], (gu / 3u) & 1u, 5);\n"
       "          tc_fence_after();\n"
       "          const u32 wad = smem_addr(wbase + wsl * WSLOT);\n"
       "          const int n = U_N[u];\n"
       "          const u32 idesc = idesc_tf32(n);\n"
       "          for (int k = 0; k < U_DZ[u]; ++k) {\n"
       "            const u32 slot = seq % NS, ph = (seq / NS) & 1u;\n"
       "            mbar_wait_t(&afull[slot], ph, 6);\n"
       "            tc_fence_after();\n"
       "            const u32 aad = smem_addr(abase + slot * "
    << kASlotBytes
    << ");\n"
       "            const u32 d = tmem + (u32)(U_COL[u] + k * n);\n"
       "#pragma unroll\n"
       "            for (int ps = 0; ps < 3; ++ps) {  // 3xTF32: hi*hi + hi*lo + lo*hi\n"
       "              const u32 ao = ps == 2 ? "
    << kASlotBytes / 2
    << "u : 0u, bo = ps == 1 ? (u32)(n * 128) : 0u;\n"
       "#pragma unroll\n"
       "              for (int ks = 0; ks < 4; ++ks)\n"
       "                tc_mma(d, sdesc(aad + ao + ks * 32), sdesc(wad + bo + ks * 32), idesc,\n"
       "                       (U_FIRST[u] && ps == 0 && ks == 0) ? 0u : 1u);\n"
       "            }\n"
       "            tc_commit(&aempty[slot]);\n"
       "            ++seq;\n"
       "          }\n"
       "          tc_commit(&wempty[wsl]);\n"
       "#ifdef CGF_UVW_DEBUG\n"
       "          if (gu == 0) { mbar_wait_t(&aempty[0], 0, 9); printf(\"cgf_uvw dbg: unit 0 aempty[0] done\\n\");\n"
       "            mbar_wait_t(&aempty[4], 0, 10); printf(\"cgf_uvw dbg: unit 0 aempty[4] done\\n\");\n"
       "            mbar_wait_t(&wempty[0], 0, 11); printf(\"cgf_uvw dbg: unit 0 wempty[0] done\\n\"); }\n"
       "#endif\n"
       "          if (U_LAST[u]) tc_commit(&sfull[U_SEG[u]]);\n"
       "          if (gu + 2 < total_units) load_w(gu + 2);  // waits for unit gu-1 only\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n";

  // epilogue: per segment (compile-time dz, n), TMEM -> registers -> z row
  o << "  else {\n"
       "    const int qd = warp & 3, m = 32 * qd + lane;\n"
       "    const u32 tq = tmem + ((u32)(32 * qd) << 16);\n"
       "    i64 lt = 0;\n"
       "    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {\n"
       "      const i64 row = tile * 128 + m;\n"
       "      const bool valid = row < rows;\n";
  for (int si = 0; si < ns; ++si) {
    const auto& sg = segs[si];
    o << "      { // segment " << si << ": z[" << sg.z_off << " ...) dz=" << sg.dz << " n=" << sg.n << " cols [" << sg.col
      << ", " << sg.col + sg.dz * sg.n << ")\n"
      << "        mbar_wait_t(&sfull[" << si << "], (u32)(lt & 1), 7);\n        tc_fence_after();\n"
      << "        float* zr = Z + (valid ? row : 0) * DIMZ + " << sg.z_off << ";\n"
      << "#pragma unroll 1\n        for (int r0 = 0; r0 < " << sg.n << "; r0 += 8) {\n"
      << "          float v[" << sg.dz << "][8];\n";
    for (int k = 0; k < sg.dz; ++k)
      o << "          tc_ld8(tq + (u32)(" << sg.col + k * sg.n << " + r0), v[" << k << "]);\n";
    o << "          tc_wait_ld();\n          if (valid) {\n            float4* dst = (float4*)(zr + r0 * " << sg.dz << ");\n";
    for (int t = 0; t < 2 * sg.dz; ++t) {
      o << "            __stcs(dst + " << t << ", make_float4(";
      for (int a = 0; a < 4; ++a) {
        const int f = 4 * t + a, rr = f / sg.dz, kk = f % sg.dz;
        o << (a ? ", " : "") << "v[" << kk << "][" << rr << "]";
      }
      o << "));\n";
    }
    o << "          }\n        }\n        tc_fence_before();\n        __syncwarp();\n"
      << "        if (lane == 0) mbar_arrive(&sdrained[" << si << "]);\n      }\n";
  }
  o << "    }\n  }\n";
  o <<        "  tc_fence_before();\n"
       "  __syncthreads();\n"
       "  if (warp == "
    << kMmaWarp
    << ") {\n"
       "    tc_fence_after();\n"
       "    asm volatile(\"tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\" :: \"r\"(tmem));\n"
       "  }\n"
       "}\n";

  UvwSource out;
  out.main.name = "cgf_uvw_fwd_f32";
  out.main.source = o.str();
  out.main.threads = kWarps * 32;
  out.main.smem_bytes = smem;
  out.main.units = nu;
  out.prep = out.main;
  out.prep.name = "cgf_uvw_prep_f32";
  out.prep.threads = 256;
  out.prep.smem_bytes = 0;
  out.main.module = out.prep.module = "cgf_uvw_fwd_f32";
  out.wimg_bytes = wimg;
  return out;
}

}  // namespace cgf
