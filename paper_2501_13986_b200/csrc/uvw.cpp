#include "uvw.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <sstream>

namespace cgf {

namespace {

constexpr int kTileRows = 128;
constexpr int kProdWarps = 8;     // producer warps (default; 8 measured 3.28 ms vs 3.59 ms for 16 on C3); MMA warp, 4 epilogue warps, TMA warp follow




constexpr int kTmemCols = 512;
constexpr int kCh = 16;           // channels per unit = K of one A block (64 B rows, SW64)
constexpr int kASlotBytes = 2 * kTileRows * kCh * 4;  // hi + lo, 128 rows x 16 fp32

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
    if (s.bp % kCh) return no("x multiplicity must be a multiple of 16");
    if (s.dz() * s.b > kTmemCols - 64) return no("z segment accumulator exceeds TMEM");
    if (s.dx() > 7 || s.dz() > 7) return no("l > 3 not supported by the tensor-core path");
  }
  if (p.dim_z % 4 || p.dim_x % kCh) return no("dim_x must be a multiple of 16 and dim_z of 4");
  for (const auto& s : p.resolved)
    if (s.z_off % 4 || s.x_off % kCh) return no("x segment offsets must be multiples of 16, z of 4");
  return true;
}

namespace {
UvwSource generate_uvw_impl(const Problem& p, const std::string& tag, bool w_transposed);

// Device helpers shared by the uvw kernels (tcgen05 / TMEM / TMA / mbarrier).
const char* uvw_helpers() {
  return R"(
// ---- tcgen05 / TMEM / TMA helpers (sm_100a) ----
struct __align__(64) TMap { unsigned long long v[16]; };  // CUtensorMap
DEVI u64 gtimer() { u64 t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
// Bounded wait: a barrier that never completes traps after ~4 s with its tag
// instead of hanging the device.
#ifdef CGF_UVW_PROF
__shared__ unsigned long long prof_s[16];
#endif
DEVI void mbar_wait_t(u64* b, u32 parity, int tag) {
  if (mbar_try(b, parity)) return;
#ifdef CGF_UVW_PROF
  const long long c0 = clock64();
  while (!mbar_try(b, parity)) { }
  if ((threadIdx.x & 31) == 0) atomicAdd(&prof_s[tag], (unsigned long long)(clock64() - c0));
  return;
#endif
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
DEVI void tc_st8(u32 taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                  "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                  "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])) : "memory");
}
DEVI void tc_st16(u32 taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                  "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                  "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
                  "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
                  "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
                  "r"(__float_as_uint(v[15])) : "memory");
}
DEVI void tc_st4(u32 taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
               :: "r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                  "r"(__float_as_uint(v[3])) : "memory");
}
DEVI u32 elect_one() {
  u32 p;
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n selp.u32 %0, 1, 0, e;\n}" : "=r"(p));
  return p;
}
DEVI void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem]^T (A: 128 lanes x 8 tf32 columns)
DEVI void tc_mma_ts(u32 d, u32 a, u64 b, u32 idesc, u32 acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
               :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// 3-D TMA tile load global -> shared, completion on an mbarrier (bytes).
DEVI void tma_load3(void* dst, const TMap* map, int c0, int c1, int c2, u64* bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
               :: "r"(smem_addr(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_addr(bar)) : "memory");
}
// Shared-memory matrix descriptor: K-major, 64-byte swizzle (rows of 16 fp32),
// 8-row groups 512 B apart (SBO), version 1 (sm_100).
DEVI u64 sdesc64(u32 saddr) {
  return (u64)((saddr & 0x3FFFFu) >> 4) | ((u64)1 << 16) | ((u64)(512 >> 4) << 32) | ((u64)1 << 46) | ((u64)4 << 61);
}
// K-major, 128-byte swizzle (rows of 32 fp32), 8-row groups 1024 B apart.
DEVI u64 sdesc128(u32 saddr) {
  return (u64)((saddr & 0x3FFFFu) >> 4) | ((u64)1 << 16) | ((u64)(1024 >> 4) << 32) | ((u64)1 << 46) | ((u64)2 << 61);
}
// Instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M = 128, N.
DEVI constexpr u32 idesc_tf32(int n) { return (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(n >> 3) << 17) | ((u32)(128 >> 4) << 24); }
// tf32 split: hi keeps the top 19 bits (exactly representable), lo the rest.
// 16-byte shared-memory load through an explicit .shared address (a generic
// pointer into the slot compiled to LD.E: generic-space loads, longer latency)
DEVI float4 lds128(const unsigned char* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(smem_addr(p)));
  return v;
}
DEVI float2 lds64(const unsigned char* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(smem_addr(p)));
  return v;
}
DEVI void sts128(unsigned char* p, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" :: "r"(smem_addr(p)), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
DEVI void sts32(unsigned char* p, float v) { asm volatile("st.shared.f32 [%0], %1;" :: "r"(smem_addr(p)), "f"(v) : "memory"); }
DEVI float tf32_hi(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }
// Byte offset of 16-byte chunk `chunk` of row m in a K-major SW64 tile (64 B rows).
DEVI u32 sw64(int m, int chunk) { return (u32)((m >> 3) * 512 + (m & 7) * 64 + ((chunk ^ ((m >> 1) & 3)) << 4)); }
)";
}
}  // namespace

UvwSource generate_uvw_forward(const Problem& p) {
  std::string why;
  if (!uvw_eligible(p, &why)) throw UnsupportedError("uvw tensor-core path: " + why);
  return generate_uvw_impl(p, "fwd", false);
}

// gx = dL/dx is the forward contraction of the TRANSPOSED problem: for each
// instruction, gx[l1 seg][c][i] += sum_r W[r][c] sum_{(i,j,k)} v y[j] gz[l3 seg][r][k]
// (kernelgen.cpp:222-226 with gzp = W^T gz), i.e. x <-> gz, l1 <-> l3,
// b <-> b', CG entries (i,j,k) -> (k,j,i) and W read transposed. The same
// generator then emits the tcgen05 kernel (A = CG(gz, y) in TMEM, B = W^T).
UvwSource generate_uvw_backward_x(const Problem& p) {
  std::string why;
  if (!uvw_eligible(p, &why)) throw UnsupportedError("uvw tensor-core path: " + why);
  Problem t = p;
  std::swap(t.x_ir, t.z_ir);
  std::swap(t.dim_x, t.dim_z);
  for (auto& s : t.resolved) {
    std::swap(s.x_off, s.z_off);
    std::swap(s.l1, s.l3);
    std::swap(s.b, s.bp);
    auto cg = std::make_shared<CGBlock>(*s.cg);
    std::swap(cg->l1, cg->l3);
    for (auto& e : cg->entries) std::swap(e.i, e.k);
    std::stable_sort(cg->entries.begin(), cg->entries.end(), [](const CGEntry& a, const CGEntry& b) {
      return a.k != b.k ? a.k < b.k : a.i != b.i ? a.i < b.i : a.j < b.j;
    });
    s.cg = cg;
  }
  if (!uvw_eligible(t, &why)) throw UnsupportedError("uvw tensor-core backward: " + why);
  return generate_uvw_impl(t, "bwdx", true);
}


// Shared pieces of the two uvw gradient kernels (gy, shared gW).
namespace {

struct GradInfo {
  int np = 0, max_dx = 1, wslot = 0, xslot = 0;
  std::vector<std::size_t> wimg_of;
};

GradInfo grad_info(const Problem& p) {
  std::string why;
  if (!uvw_eligible(p, &why)) throw UnsupportedError("uvw tensor-core path: " + why);
  GradInfo g;
  const auto& R = p.resolved;
  g.np = static_cast<int>(R.size());
  int max_bp = 16;
  for (const auto& s : R) {
    if (s.b != 64 || s.bp != 64) throw UnsupportedError("uvw gradient kernels: multiplicities must be 64");
    g.max_dx = std::max(g.max_dx, s.dx());
    max_bp = std::max(max_bp, s.bp);
  }
  // W^T images of the gx kernel's prep: per instruction, b / 16 images of
  // [b' rows][16 fp32] hi + lo (same offsets as generate_uvw_backward_x).
  g.wslot = 2 * max_bp * kCh * 4;
  std::size_t w = 0;
  for (const auto& s : R) {
    g.wimg_of.push_back(w);
    w += static_cast<std::size_t>(s.b / kCh) * g.wslot;
  }
  g.xslot = (kTileRows * kCh * g.max_dx * 4 + 1023) / 1024 * 1024;
  return g;
}

void emit_grad_tables(std::ostringstream& o, const Problem& p) {
  const auto& R = p.resolved;
  auto arr = [&](const char* name, const std::vector<long long>& v) {
    o << "__constant__ int " << name << "[" << std::max<size_t>(1, v.size()) << "] = {";
    for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
    o << "};\n";
  };
  std::vector<long long> dz, dx, zoff, xc, woff;
  for (const auto& s : R) {
    dz.push_back(s.dz());
    dx.push_back(s.dx());
    zoff.push_back(s.z_off);
    xc.push_back(s.x_off / kCh);
    woff.push_back(s.w_off);
  }
  arr("P_DZ", dz);
  arr("P_DX", dx);
  arr("P_ZOFF", zoff);
  arr("P_XC", xc);
  arr("P_WOFF", woff);
}

const char* grad_helpers() {
  return R"(
DEVI void tc_ld32(u32 taddr, float* v) {
  u32 r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
DEVI void prod_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// element (row r of the operand, K index k) of a K-major SW128 tile whose K
// runs over 32 batch rows (one 128-byte line per operand row, 16-byte chunks
// XOR the row's index in its 8-row atom): 32 lanes holding consecutive K of
// one operand row store 128 contiguous bytes
DEVI u32 kmaj128(int r, int k) { return (u32)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ r) & 7) << 4) + (k & 3) * 4); }
)";
}

// x tile -> this thread's 8 channels x dx floats (the forward producer's read)
void emit_x_read(std::ostringstream& o, int dx) {
  o << "  float xv[" << 8 * dx << "];\n#pragma unroll\n  for (int t = 0; t < " << 2 * dx << "; ++t) {\n"
    << "    const int g = " << 2 * dx << " * sub + t, L = m * " << dx << " + (g >> 2), j = g & 3;\n"
    << "    const float4 v = lds128(xs + L * 64 + ((j ^ ((L >> 1) & 3)) << 4));\n"
    << "    xv[4 * t] = v.x; xv[4 * t + 1] = v.y; xv[4 * t + 2] = v.z; xv[4 * t + 3] = v.w;\n  }\n"
    << "  fence_proxy_async();\n  __syncwarp();\n  if ((threadIdx.x & 31) == 0) mbar_arrive(xempty);\n";
}

const char* grad_kernel_head() {
  return
       "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
       "  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);\n"
       "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
       "  const i64 ntiles = (rows + 127) / 128;\n";
}

}  // namespace

// dL/dy of a uvw backward with shared W (kernel "cgf_uvw_bwdy_f32"). Per
// 128-row tile and unit (instruction q, component k):
//   gzp_k[row, c] = sum_r gz[row][q.z][r][k] W_q[r][c]     tcgen05: M=128 rows, N=64 (c), K=64 (r), 3xTF32
//   gy[row, j]   += sum_{(i,j,k)} v sum_c x[row][q.x][c][i] gzp_k[row, c]          SIMT (producers)
// (kernelgen.cpp:222-226: gy accumulates v x[i] gzp[k]). The gz_k tile is the
// K-major A operand; B is the gx kernel's W^T image; gzp is read back from
// TMEM by the producers, which hold x for the same 8 channels.
UvwSource generate_uvw_backward_y(const Problem& p) {
  const GradInfo g = grad_info(p);
  const auto& R = p.resolved;
  const int np = g.np;
  int max_dz = 1;
  for (const auto& sq : R) max_dz = std::max(max_dz, sq.dz());
  if (64 * max_dz > 512) throw UnsupportedError("uvw gy kernel: l3 too large");
  // gz planes: for every z segment and component k, the 64 channels of gz
  // contiguous per row ([plane][row][64], tf32 hi and lo arrays), written by
  // the pre-pass so the gy kernel can TMA-load gz_k tiles in the MMA layout.
  std::map<std::uint32_t, int> plane_of_seg;
  int nplanes = 0;
  std::vector<std::pair<std::uint32_t, int>> segs;  // (z_off, dz) in plane order
  for (const auto& sq : R)
    if (!plane_of_seg.count(sq.z_off)) {
      plane_of_seg[sq.z_off] = nplanes;
      nplanes += sq.dz();
      segs.push_back({sq.z_off, sq.dz()});
    }
  const int gz_bytes = 2 * kTileRows * 64 * 4;
  // gz_k tiles move as halves (32 r: hi + lo, 32 KB) through a ring of NGH
  // stages, so the loader runs ahead of the MMAs (one whole-tile buffer left
  // every k's TMA latency exposed): 3.71 -> 2.99 ms with 3 stages and a
  // 2-tile x ring (profiles/r02_ab_gy.txt)
  const int ngh = std::getenv("CGF_UVW_GY_NGH") ? std::clamp(std::atoi(std::getenv("CGF_UVW_GY_NGH")), 2, 6) : 3;
  const int nx = std::getenv("CGF_UVW_GY_NX") ? std::atoi(std::getenv("CGF_UVW_GY_NX")) : 2;
  const int smem = 1024 + ngh * (gz_bytes / 2) + nx * g.xslot + 4 * g.wslot + 1024 + 128 * p.dim_y * 4;
  if (smem > 227 * 1024) throw UnsupportedError("uvw gy kernel: shared memory too small");
  std::ostringstream o;
  if (std::getenv("CGF_UVW_DEBUG")) o << "#define CGF_UVW_DEBUG 1\n";
  o << device_runtime_source() << uvw_helpers() << grad_helpers();
  o << "// uvw gy: " << np << " instructions, " << nplanes << " gz planes\n#define DIMX " << p.dim_x << "\n#define DIMY "
    << p.dim_y << "\n#define DIMZ " << p.dim_z << "\n#define NP " << np << "\n#define WSLOT " << g.wslot
    << "\n#define XSLOT " << g.xslot << "\n#define GZB " << gz_bytes << "\n#define NGH " << ngh << "\n#define NX " << nx << "\n#define NPLANES "
    << nplanes << "\n";
  emit_grad_tables(o, p);
  {
    o << "__constant__ int P_WIMG[" << np << "] = {";
    for (int q = 0; q < np; ++q) o << (q ? "," : "") << g.wimg_of[q];
    o << "};\n__constant__ int P_PLANE[" << np << "] = {";
    for (int q = 0; q < np; ++q) o << (q ? "," : "") << plane_of_seg.at(R[q].z_off);
    o << "};\n";
  }
  // ---- pre-pass (one read of gz): tf32 hi / lo planes for both gradient
  // kernels, one block per 32 rows staged in shared memory:
  //   gy:  YH / YL [plane][row][64 r]      (the gy MMA's A tiles, K = r)
  //   gW:  WH / WL [plane][64 r][pitch]    (the gW MMA's B tiles, K = rows)
  // rows per block: 32 (3 blocks / SM, 128-byte gW-plane segments) measured
  // 2.41 ms against 3.15 ms for 16 rows (6 blocks / SM, half-line segments;
  // profiles/r02_ab_planes.txt)
  const int pr = std::getenv("CGF_UVW_PLANE_ROWS") ? std::atoi(std::getenv("CGF_UVW_PLANE_ROWS")) : 32;
  if (pr != 16 && pr != 32) throw UnsupportedError("CGF_UVW_PLANE_ROWS must be 16 or 32");
  o << "#define PR " << pr << "\n";
  o << "extern \"C\" __global__ void __launch_bounds__(256) cgf_uvw_bwd_planes_f32(const float* __restrict__ GZ,"
       " float* __restrict__ YH, float* __restrict__ YL, float* __restrict__ WH, float* __restrict__ WL, i64 rows,"
       " i64 pitch) {\n"
       "  extern __shared__ float t[];  // [PR][DIMZ + 1] (odd pitch: conflict-free column reads)\n"
       "  const i64 chunks = (rows + PR - 1) / PR;\n"
       "  for (i64 cbk = blockIdx.x; cbk < chunks; cbk += gridDim.x) {\n"
       "    const i64 r0 = cbk * PR;\n"
       "    __syncthreads();\n"
       "    for (int e = threadIdx.x; e < PR / 4 * DIMZ; e += 256) {  // 16-byte loads\n"
       "      const int rr = e / (DIMZ / 4), c = 4 * (e - rr * (DIMZ / 4));\n"
       "      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);\n"
       "      if (r0 + rr < rows) v = __ldg((const float4*)(GZ + (r0 + rr) * DIMZ + c));\n"
       "      float* d = t + rr * (DIMZ + 1) + c; d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;\n    }\n"
       "    __syncthreads();\n";
  for (size_t si = 0; si < segs.size(); ++si) {
    const auto [zoff, dz] = segs[si];
    const int pl0 = plane_of_seg.at(zoff);
    o << "    // segment " << si << ": z offset " << zoff << ", " << dz << " components, planes " << pl0 << ".."
      << pl0 + dz - 1 << "\n"
      // gy planes: 4 consecutive r per 16-byte store
      << "    for (int e = threadIdx.x; e < PR * 16 * " << dz << "; e += 256) {\n"
      << "      const int j = e & 15, rr = (e >> 4) % PR, k = (e >> 4) / PR;\n"
      << "      if (r0 + rr < rows) {\n"
      << "        const float* sr = t + rr * (DIMZ + 1) + " << zoff << " + k;\n"
      << "        float v[4], h[4];\n#pragma unroll\n        for (int a = 0; a < 4; ++a) { v[a] = sr[(4 * j + a) * " << dz
      << "]; h[a] = tf32_hi(v[a]); }\n"
      << "        const i64 o = ((i64)(" << pl0 << " + k) * rows + r0 + rr) * 64 + 4 * j;\n"
      << "        __stcs((float4*)(YH + o), make_float4(h[0], h[1], h[2], h[3]));\n"
      << "        __stcs((float4*)(YL + o), make_float4(v[0] - h[0], v[1] - h[1], v[2] - h[2], v[3] - h[3]));\n      }\n    }\n"
      // gW planes: 4 consecutive rows per 16-byte store
      << "    for (int e = threadIdx.x; e < PR / 4 * 64 * " << dz << "; e += 256) {\n"
      << "      const int q4 = e % (PR / 4), r = (e / (PR / 4)) & 63, k = e / (PR / 4) / 64;\n"
      << "      float v[4], h[4];\n#pragma unroll\n      for (int a = 0; a < 4; ++a) { v[a] = t[(4 * q4 + a) * (DIMZ + 1) + "
      << zoff << " + r * " << dz << " + k]; h[a] = tf32_hi(v[a]); }\n"
      << "      const i64 o = ((i64)(" << pl0 << " + k) * 64 + r) * pitch + r0 + 4 * q4;\n"
      << "      if (r0 + 4 * q4 < rows) {\n"
      << "        __stcs((float4*)(WH + o), make_float4(h[0], h[1], h[2], h[3]));\n"
      << "        __stcs((float4*)(WL + o), make_float4(v[0] - h[0], v[1] - h[1], v[2] - h[2], v[3] - h[3]));\n      }\n    }\n";
  }
  o << "  }\n}\n\n";
  // per instruction: x once per 16-channel block, then every component k
  // against gzp_k (TMEM columns 64 k of this thread's lane)
  for (int q = 0; q < np; ++q) {
    const auto& sq = R[q];
    const int dx = sq.dx(), dz = sq.dz();
    o << "DEVI void gyq_" << q << "(int cb, const unsigned char* xs, int m, int sub, u32 tq, float* gy, u64* xempty) {\n";
    emit_x_read(o, dx);
    for (int k = 0; k < dz; ++k) {
      std::set<int> is;
      for (const auto& e : sq.cg->entries)
        if (e.k == k) is.insert(e.i);
      if (is.empty()) continue;
      o << "  { // k = " << k << "\n    float gp[8];\n    tc_ld8(tq + " << 64 * k << " + cb * 16 + 8 * sub, gp);\n"
        << "    tc_wait_ld();\n";
      for (int i : is) o << "    float xg" << i << " = 0.f;\n";
      o << "#pragma unroll\n    for (int c = 0; c < 8; ++c) {\n";
      for (int i : is) o << "      xg" << i << " = fmaf(xv[c * " << dx << " + " << i << "], gp[c], xg" << i << ");\n";
      o << "    }\n";
      for (const auto& e : sq.cg->entries)
        if (e.k == k)
          o << "    gy[" << sq.y_off + e.j << "] = fmaf((float)" << hexd(e.v) << ", xg" << e.i << ", gy[" << sq.y_off + e.j
            << "]);\n";
      o << "  }\n";
    }
    o << "}\n\n";
  }
  // warps: 0-7 producers (gy), 8 MMA, 9 x TMA, 10 W images, 11 gz TMA
  o << "extern \"C\" __global__ void __launch_bounds__(384, 1) cgf_uvw_bwdy_f32("
       "const __grid_constant__ TMap tx1, const __grid_constant__ TMap tx3, const __grid_constant__ TMap tx5, "
       "const __grid_constant__ TMap tx7, const __grid_constant__ TMap tgh, const __grid_constant__ TMap tgl, "
       "const float* __restrict__ Y, const float* __restrict__ WIMG, float* __restrict__ GY, i64 rows) {\n"
    << grad_kernel_head()
    << "  unsigned char* gzt = sm;                 // NGH half tiles of gz_k [rows][32 r]: hi 16 KB, lo 16 KB (TMA)\n"
       "  unsigned char* xs0 = gzt + NGH * (GZB / 2);  // x tile ring (TMA, SW64)\n"
       "  unsigned char* ws = xs0 + NX * XSLOT;    // W^T images of one instruction (4 r-blocks)\n"
       "  u64* bars = (u64*)(ws + 4 * WSLOT);\n"
       "  u64* gz_full = bars; u64* gz_empty = bars + NGH; u64* gzp_full = bars + 2 * NGH; u64* gzp_empty = gzp_full + 1;\n"
       "  u64* w_full = gzp_empty + 1; u64* w_empty = w_full + 1; u64* x_full = w_empty + 1; u64* x_empty = x_full + NX;\n"
       "  u32* tmem_slot = (u32*)(x_empty + NX);\n"
       "  float* gys = (float*)(bars + 32);\n"
       "  if (threadIdx.x == 0) {\n"
       "    for (int i = 0; i < NGH; ++i) { mbar_init(&gz_full[i], 1); mbar_init(&gz_empty[i], 1); }\n"
       "    mbar_init(gzp_full, 1); mbar_init(gzp_empty, 8);\n"
       "    mbar_init(w_full, 1); mbar_init(w_empty, 1);\n"
       "    for (int i = 0; i < NX; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 8); }\n"
       "    mbar_fence_init();\n  }\n"
       "  if (warp == 8) {\n"
       "    asm volatile(\"tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\" :: \"r\"(smem_addr(tmem_slot)));\n"
       "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\");\n"
       "  }\n"
       "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n"
       "  const u32 tmem = *tmem_slot;\n"
       "  if (warp < 8) {\n"
       "    const int m = 32 * (warp & 3) + lane, sub = warp >> 2;\n"
       "    const u32 tq = tmem + ((u32)(32 * (warp & 3)) << 16);\n"
       "    u32 uq = 0, gx = 0;\n"
       "    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
       "      const i64 row = tile * 128 + m;\n"
       "      const bool valid = row < rows;\n"
       "      float gy[DIMY];\n"
       "#pragma unroll\n      for (int j = 0; j < DIMY; ++j) gy[j] = 0.f;\n"
       "#pragma unroll 1\n      for (int q = 0; q < NP; ++q, ++uq) {\n"
       "        mbar_wait_t(gzp_full, uq & 1u, 22);\n"
       "        tc_fence_after();\n"
       "#pragma unroll 1\n        for (int cb = 0; cb < 4; ++cb, ++gx) {\n"
       "          const u32 xsl = gx % NX;\n"
       "          mbar_wait_t(&x_full[xsl], (gx / NX) & 1u, 23);\n"
       "          const unsigned char* xs = xs0 + xsl * XSLOT;\n"
       "          switch (q) {\n";
  for (int q = 0; q < np; ++q)
    o << "            case " << q << ": gyq_" << q << "(cb, xs, m, sub, tq, gy, &x_empty[xsl]); break;\n";
  o << "          }\n"
       "        }\n"
       "        tc_fence_before();\n        __syncwarp();\n"
       "        if (lane == 0) mbar_arrive(gzp_empty);\n"
       "      }\n"
       "      if (sub == 1) {\n#pragma unroll\n        for (int j = 0; j < DIMY; ++j) gys[m * DIMY + j] = gy[j];\n      }\n"
       "      prod_sync();\n"
       "      if (sub == 0 && valid) {\n#pragma unroll\n        for (int j = 0; j < DIMY; ++j) GY[row * DIMY + j] = gy[j] + gys[m * DIMY + j];\n      }\n"
       "      prod_sync();\n"
       "    }\n"
       "  }\n"
       "  else if (warp == 8) {\n"
       "    const u64 gzh0 = sdesc128(smem_addr(gzt));\n"
       "    const u64 wd = sdesc64(smem_addr(ws));\n"
       "    const u32 id_gzp = idesc_tf32(64);\n"
       "    u32 ug = 0, uq = 0;\n"
       "    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
       "      for (int q = 0; q < NP; ++q, ++uq) {\n"
       "        mbar_wait_t(w_full, uq & 1u, 25);\n"
       "        mbar_wait_t(gzp_empty, (uq & 1u) ^ 1u, 27);\n"
       "        tc_fence_after();\n"
       "        const int dz = P_DZ[q];\n"
       "        for (int k = 0; k < dz; ++k) {\n"
       "          const u32 dg = tmem + 64 * k;\n"
       "          for (int j = 0; j < 2; ++j, ++ug) {  // r-block j: one half-tile stage\n"
       "            const u32 hs = ug % NGH;\n"
       "            mbar_wait_t(&gz_full[hs], (ug / NGH) & 1u, 26);\n"
       "            tc_fence_after();\n"
       "            if (elect_one()) {\n"
       "              const u64 gzh = gzh0 + (u64)((hs * (GZB / 2)) >> 4), gzl = gzh + (u64)((GZB / 4) >> 4);\n"
       "#pragma unroll\n              for (int t = 0; t < 4; ++t) {\n"
       // gz (A): SW128, [128 rows][32 r] per half; W^T (B): SW64 blocks of 16
       "                const int s = 4 * j + t;\n"
       "                const u64 ao = (u64)((t * 32) >> 4);\n"
       "                const u64 bo = (u64)(((s >> 1) * WSLOT + (s & 1) * 32) >> 4);\n"
       "                tc_mma(dg, gzh + ao, wd + bo, id_gzp, s ? 1u : 0u);\n"
       "                tc_mma(dg, gzh + ao, wd + bo + (u64)((64 * 64) >> 4), id_gzp, 1u);\n"
       "                tc_mma(dg, gzl + ao, wd + bo, id_gzp, 1u);\n"
       "              }\n"
       "              tc_commit(&gz_empty[hs]);\n"
       "              if (k == dz - 1 && j == 1) { tc_commit(gzp_full); tc_commit(w_empty); }\n"
       "            }\n"
       "            __syncwarp();\n"
       "          }\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "  }\n"
       "  else if (warp == 9) {\n"
       "    if (lane == 0) {\n"
       "      u32 gx = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x)\n"
       "        for (int q = 0; q < NP; ++q)\n"
       "          for (int cb = 0; cb < 4; ++cb, ++gx) {\n"
       "            const u32 xsl = gx % NX;\n"
       "            mbar_wait_t(&x_empty[xsl], ((gx / NX) & 1u) ^ 1u, 29);\n"
       "            const int dx = P_DX[q];\n"
       "            mbar_expect_tx(&x_full[xsl], 128 * 64 * dx);\n"
       "            const TMap* mp = dx == 1 ? &tx1 : dx == 3 ? &tx3 : dx == 5 ? &tx5 : &tx7;\n"
       "            tma_load3(xs0 + xsl * XSLOT, mp, 0, P_XC[q] + cb * dx, (int)(tile * 128), &x_full[xsl]);\n"
       "          }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n"
       "  else if (warp == 10) {\n"
       "    if (lane == 0) {\n"
       "      u32 wg = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x)\n"
       "        for (int q = 0; q < NP; ++q, ++wg) {\n"
       "          mbar_wait_t(w_empty, (wg & 1u) ^ 1u, 30);\n"
       "          mbar_expect_tx(w_full, 4 * WSLOT);\n"
       "          bulk_g2s(ws, (const char*)WIMG + P_WIMG[q], 4 * WSLOT, w_full);\n"
       "        }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n"
       "  else if (warp == 11) {\n"
       // gz_k tiles from the planes: 2 r-blocks of [128 rows][32] (SW128,
       // 128-byte box lines) for hi and for lo, the MMA's K-major A layout
       "    if (lane == 0) {\n"
       "      u32 ug = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x)\n"
       "        for (int q = 0; q < NP; ++q)\n"
       "          for (int k = 0; k < P_DZ[q]; ++k)\n"
       "            for (int j = 0; j < 2; ++j, ++ug) {\n"
       "              const u32 hs = ug % NGH;\n"
       "              unsigned char* d = gzt + hs * (GZB / 2);\n"
       "              mbar_wait_t(&gz_empty[hs], ((ug / NGH) & 1u) ^ 1u, 31);\n"
       "              mbar_expect_tx(&gz_full[hs], GZB / 2);\n"
       "              tma_load3(d, &tgh, 32 * j, (int)(tile * 128), P_PLANE[q] + k, &gz_full[hs]);\n"
       "              tma_load3(d + GZB / 4, &tgl, 32 * j, (int)(tile * 128), P_PLANE[q] + k, &gz_full[hs]);\n"
       "            }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n"
       "  tc_fence_before();\n  __syncthreads();\n"
       "  if (warp == 8) { tc_fence_after(); asm volatile(\"tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\" :: \"r\"(tmem)); }\n"
       "}\n";
  UvwSource out;
  out.main.name = out.main.module = "cgf_uvw_bwdy_f32";
  out.main.source = o.str();
  out.main.threads = 384;
  out.main.smem_bytes = smem;
  out.prep = out.main;
  out.prep.name = "cgf_uvw_bwd_planes_f32";
  out.prep.threads = 256;
  out.prep.smem_bytes = pr * (p.dim_z + 1) * 4;
  out.prep_rows = pr;
  out.wimg_bytes = 0;
  out.dims_x = nplanes;  // number of gz planes (the caller sizes the plane buffers)
  return out;
}

// The shared-W gradient dL/dW of a uvw backward (kernel "cgf_uvw_bwdw<first>_f32")
// for instructions [first, first + count) (count <= 6: one 64-column TMEM
// accumulator each):
//   gW_q[r][c] += sum_row sum_k gz[row][q.z][r][k] z'_k[row][c],  z'_k = CG(x, y)[.., k]
// (kernelgen.cpp:639-650 summed over rows): tcgen05 M=64 (c), N=64 (r), K = 32
// batch rows per stage, both operands K-major over the rows (SW128), 3xTF32.
// The z' tiles are written transposed by the producers (double buffered), the
// gz^T tiles come by TMA from the transposed gz planes (cgf_uvw_bwd_planes_f32)
// through a ring of NGZ stages that runs ahead of the MMAs.
// Accumulators live in TMEM across all tiles of the CTA and are written once
// as this CTA's partial; `prep` sums the partials over CTAs in a fixed order
// (deterministic).
UvwSource generate_uvw_backward_w(const Problem& p, int first, int count) {
  const GradInfo g = grad_info(p);
  const auto& R = p.resolved;
  if (count < 1 || count > 6 || first < 0 || first + count > g.np) throw std::logic_error("bad gW instruction range");
  constexpr int kRows = 32;                       // batch rows per stage (the MMA's K)
  const int tb = 2 * 64 * kRows * 4;              // hi + lo of a [64][64 rows] K-major tile
  const int xslot = (kRows * kCh * g.max_dx * 4 + 1023) / 1024 * 1024;
  // x: the instruction's whole x segment (4 16-channel tiles) is loaded once
  // per (tile, instruction) and reused by all its components k, double
  // buffered so the next instruction's segment lands while this one is used
  // (single-buffered, the producers spent a third of their time waiting on it)
  const int nx = 4;  // x tiles per instruction
  // staging depths: gz^T tiles (the loader runs ahead of the MMAs) and x
  // segments; with two of each the pass was TMA-latency bound (no MMAs and no
  // producer math still took 2.0 of 2.7 ms, profiles/r02_ab_gw.txt); 6 gz^T
  // stages: 2.64 + 2.92 -> 2.20 + 2.34 ms (r02_ab_gw2.txt; more z' stages: no
  // change, r02_ab_gw3.txt)
  const int ngz = std::getenv("CGF_UVW_NGZ") ? std::clamp(std::atoi(std::getenv("CGF_UVW_NGZ")), 2, 8) : 6;
  const int nxb = std::getenv("CGF_UVW_NXB") ? std::clamp(std::atoi(std::getenv("CGF_UVW_NXB")), 2, 4) : 2;
  const int nzs = std::getenv("CGF_UVW_NZS") ? std::clamp(std::atoi(std::getenv("CGF_UVW_NZS")), 2, 4) : 2;  // z' stages
  const int smem = 1024 + (ngz + nzs) * tb + nxb * nx * xslot + 1024;
  if (smem > 227 * 1024) throw UnsupportedError("uvw gW kernel: shared memory too small");
  const std::string kname = "cgf_uvw_bwdw" + S(first) + "_f32";
  // gz planes (same numbering as the pre-pass): segment component -> plane
  std::map<std::uint32_t, int> plane_of_seg;
  int nplanes = 0;
  for (const auto& sq : R)
    if (!plane_of_seg.count(sq.z_off)) {
      plane_of_seg[sq.z_off] = nplanes;
      nplanes += sq.dz();
    }
  std::ostringstream o;
  if (std::getenv("CGF_UVW_DEBUG")) o << "#define CGF_UVW_DEBUG 1\n";
  o << device_runtime_source() << uvw_helpers() << grad_helpers();
  // experiment knobs (A/B only): 16 = no MMAs, 32 = producers skip the z' values
  o << "#define UVW_EXP " << (std::getenv("CGF_UVW_EXP") ? std::atoi(std::getenv("CGF_UVW_EXP")) : 0) << "\n";
  o << "// uvw gW: instructions [" << first << ", " << first + count << ")\n#define DIMX " << p.dim_x
    << "\n#define DIMY " << p.dim_y << "\n#define DIMZ " << p.dim_z << "\n#define NW_ " << p.n_w << "\n#define Q0 "
    << first << "\n#define Q1 " << first + count << "\n#define XSLOT " << xslot << "\n#define TB " << tb
    << "\n#define KR " << kRows << "\n#define NX " << nx << "\n#define NGZ " << ngz << "\n#define NXB " << nxb << "\n#define NZS " << nzs << "\n";
  emit_grad_tables(o, p);
  o << "__constant__ int P_PLANE[" << R.size() << "] = {";
  for (size_t q = 0; q < R.size(); ++q) o << (q ? "," : "") << plane_of_seg.at(R[q].z_off);
  o << "};\n";
  // producer thread (row m < 32, sub < 8) owns channels [2 sub, 2 sub + 2) of
  // every 16-channel block: per (instruction, component) stage the CG·y
  // coefficients are formed once, then the 4 blocks' x reads (float2) and
  // z'_k values for its 2 channels
  for (int q = first; q < first + count; ++q) {
    const auto& sq = R[q];
    const int dx = sq.dx(), dz = sq.dz();
    o << "DEVI void zw_" << q << "(int k, const unsigned char* xs0, const float* yv, int m, int sub, unsigned char* zt) {\n"
      << "  switch (k) {\n";
    for (int k = 0; k < dz; ++k) {
      std::map<int, std::string> qk;
      for (const auto& e : sq.cg->entries) {
        if (e.k != k) continue;
        std::string& t = qk[e.i];
        t += (t.empty() ? "" : " + ") + std::string("(float)") + hexd(e.v) + " * yv[" + S(sq.y_off + e.j) + "]";
      }
      o << "  case " << k << ": {\n";
      for (const auto& [i, ex] : qk) o << "    const float q" << i << " = " << ex << ";\n";
      o << "#pragma unroll\n    for (int cb = 0; cb < 4; ++cb) {\n"
        << "      const unsigned char* xs = xs0 + cb * XSLOT;\n"
        << "      float xv[" << 2 * dx << "];\n#pragma unroll\n      for (int t = 0; t < " << dx << "; ++t) {\n"
        // float2 index f2 = dx * sub + t of the row's 16 dx floats: line f2 / 8, chunk (f2 / 2) & 3, half f2 & 1
        << "        const int f2 = " << dx << " * sub + t, L = m * " << dx << " + (f2 >> 3), j = (f2 >> 1) & 3;\n"
        << "        const float2 v = lds64(xs + L * 64 + ((j ^ ((L >> 1) & 3)) << 4) + 8 * (f2 & 1));\n"
        << "        xv[2 * t] = v.x; xv[2 * t + 1] = v.y;\n      }\n"
        << "#pragma unroll\n      for (int c = 0; c < 2; ++c) {\n        float zc = 0.f;\n";
      for (const auto& kv : qk) o << "        zc = fmaf(q" << kv.first << ", xv[c * " << dx << " + " << kv.first << "], zc);\n";
      o << "        const float h = tf32_hi(zc);\n        const u32 off = kmaj128(16 * cb + 2 * sub + c, m);\n"
        << "        sts32(zt + off, h); sts32(zt + TB / 2 + off, zc - h);\n      }\n    }\n    break; }\n";
    }
    o << "  }\n}\n\n";
  }
  o << "extern \"C\" __global__ void " << kname << "_reduce(const float* __restrict__ part, int nparts, "
       "float* __restrict__ gw, int w0, int w1) {\n"
       "  const int e = w0 + blockIdx.x * blockDim.x + threadIdx.x;\n  if (e >= w1) return;\n"
       "  float s = 0.f;\n  for (int c = 0; c < nparts; ++c) s += part[(size_t)c * NW_ + e];\n  gw[e] = s;\n}\n\n";
  // warps: 0-7 producers (z'), 8 MMA, 9 x TMA, 10 gz TMA
  o << "extern \"C\" __global__ void __launch_bounds__(352, 1) " << kname << "("
       "const __grid_constant__ TMap tx1, const __grid_constant__ TMap tx3, const __grid_constant__ TMap tx5, "
       "const __grid_constant__ TMap tx7, const __grid_constant__ TMap tgh, const __grid_constant__ TMap tgl, "
       "const float* __restrict__ Y, float* __restrict__ PART, i64 rows) {\n"
       "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
       "  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);\n"
       "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
       "  const i64 ntiles = (rows + KR - 1) / KR;\n"
       "  unsigned char* gzt = sm;                 // NGZ x gz_k^T tile [r][KR rows] K-major: hi, lo after TB/2\n"
       "  unsigned char* zt = sm + NGZ * TB;       // NZS x z'_k^T tile [c][KR rows] K-major\n"
       "  unsigned char* xs0 = zt + NZS * TB;      // NXB x segments of one instruction: NX tiles each (TMA, SW64)\n"
       "  u64* bars = (u64*)(xs0 + NXB * NX * XSLOT);\n"
       "  u64* gz_full = bars; u64* gz_empty = bars + NGZ; u64* z_full = gz_empty + NGZ; u64* z_empty = z_full + NZS;\n"
       "  u64* x_full = z_empty + NZS; u64* x_empty = x_full + NXB; u64* done = x_empty + NXB;\n"
       "  u32* tmem_slot = (u32*)(done + 1);\n"
       "  if (threadIdx.x == 0) {\n"
       "    for (int i = 0; i < NGZ; ++i) { mbar_init(&gz_full[i], 1); mbar_init(&gz_empty[i], 1); }\n"
       "    for (int i = 0; i < NZS; ++i) { mbar_init(&z_full[i], 8); mbar_init(&z_empty[i], 1); }\n"
       "    for (int i = 0; i < NXB; ++i) { mbar_init(&x_full[i], 1); mbar_init(&x_empty[i], 8); }\n"
       "    mbar_init(done, 1);\n    mbar_fence_init();\n  }\n"
       "  if (warp == 8) {\n"
       "    asm volatile(\"tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\" :: \"r\"(smem_addr(tmem_slot)));\n"
       "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\");\n"
       "  }\n"
       "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n"
       "  const u32 tmem = *tmem_slot;\n"
       "  if (warp < 8) {\n"
       "    const int m = lane, sub = warp;\n"
       "    u32 ug = 0, uq = 0;\n"
       "    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
       "      const i64 row = tile * KR + m;\n"
       "      const bool valid = row < rows;\n"
       "      float yv[DIMY];\n"
       "#pragma unroll\n      for (int j = 0; j < DIMY; ++j) yv[j] = valid ? __ldg(Y + row * DIMY + j) : 0.f;\n"
       "#pragma unroll 1\n      for (int q = Q0; q < Q1; ++q, ++uq) {\n"
       "        const int dz = P_DZ[q];\n"
       "        const u32 xb = uq % NXB;\n"
       "        mbar_wait_t(&x_full[xb], (uq / NXB) & 1u, 23);\n"
       "#pragma unroll 1\n        for (int k = 0; k < dz; ++k, ++ug) {\n"
       "          const u32 zs = ug % NZS;\n"
       "          unsigned char* z = zt + zs * TB;\n"
       "          mbar_wait_t(&z_empty[zs], ((ug / NZS) & 1u) ^ 1u, 21);\n"
       "          {\n"
       "            const unsigned char* xs = xs0 + (xb * NX) * XSLOT;\n"
       "            if (!(UVW_EXP & 32)) switch (q) {\n";
  for (int q = first; q < first + count; ++q)
    o << "              case " << q << ": zw_" << q << "(k, xs, yv, m, sub, z); break;\n";
  o << "            }\n"
       "          }\n"
       "          fence_proxy_async();\n          __syncwarp();\n          if (lane == 0) mbar_arrive(&z_full[zs]);\n"
       "        }\n"
       // the x segment's generic reads are done: release it to the next TMA
       "        fence_proxy_async();\n        __syncwarp();\n        if (lane == 0) mbar_arrive(&x_empty[xb]);\n"
       "      }\n"
       "    }\n"
       // this CTA's partial: M=64 accumulators use lanes 0-15 of each 32-lane
       // quadrant: quadrant w holds c in [16 w, 16 w + 16), all 64 r columns
       "    mbar_wait_t(done, 0, 24);\n    tc_fence_after();\n"
       "    if (warp < 4) {\n"
       "      const u32 tq = tmem + ((u32)(32 * warp) << 16);\n"
       "      const int c = 16 * warp + lane;\n"
       "      float* pr = PART + (size_t)blockIdx.x * NW_;\n"
       "      for (int q = Q0; q < Q1; ++q) {\n"
       "        float v[32];\n"
       "        for (int h = 0; h < 2; ++h) {\n"
       "          tc_ld32(tq + 64 * (q - Q0) + 32 * h, v);\n          tc_wait_ld();\n"
       "          if (lane < 16) {\n"
       "#pragma unroll\n            for (int j = 0; j < 32; ++j) pr[P_WOFF[q] + (32 * h + j) * 64 + c] = v[j];\n"
       "          }\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "  }\n"
       "  else if (warp == 8) {\n"
       "    const u64 gh0 = sdesc128(smem_addr(gzt)), zh0 = sdesc128(smem_addr(zt));\n"
       "    const u32 id_w = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(64 >> 3) << 17) | ((u32)(64 >> 4) << 24);\n"
       "    u32 ug = 0; i64 lt = 0;\n"
       "    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {\n"
       "      for (int q = Q0; q < Q1; ++q) {\n"
       "        const int dz = P_DZ[q];\n"
       "        for (int k = 0; k < dz; ++k, ++ug) {\n"
          "          const u32 st = ug % NZS, ph = (ug / NZS) & 1u, gs = ug % NGZ;\n"
       "          mbar_wait_t(&gz_full[gs], (ug / NGZ) & 1u, 26);\n"
       "          mbar_wait_t(&z_full[st], ph, 28);\n"
       "          tc_fence_after();\n"
       "          if (elect_one()) {\n"
       "            const u64 gh = gh0 + (u64)((gs * TB) >> 4), gl = gh + (u64)((TB / 2) >> 4);\n"
       "            const u64 zh = zh0 + (u64)((st * TB) >> 4), zl = zh + (u64)((TB / 2) >> 4);\n"
       "            const u32 dw = tmem + 64 * (q - Q0);\n"
       "            const u32 first = (lt == 0 && k == 0) ? 1u : 0u;\n"
       "#pragma unroll\n            for (int s = 0; s < KR / 8; ++s) {\n"
       // z' (A) and gz (B): SW128, one 128-byte line of 32 batch rows per operand row
       // (z' was SW64 with 16-row blocks: its producer stores were 2-way bank conflicted)
       "              const u64 o = (u64)(((s >> 2) * 8192 + (s & 3) * 32) >> 4);\n"
       "              const u64 ob = (u64)(((s >> 2) * 8192 + (s & 3) * 32) >> 4);\n"
       "              if (!(UVW_EXP & 16)) {\n"
       "              tc_mma(dw, zh + o, gh + ob, id_w, (first && s == 0) ? 0u : 1u);\n"
       "              tc_mma(dw, zh + o, gl + ob, id_w, 1u);\n"
       "              tc_mma(dw, zl + o, gh + ob, id_w, 1u);\n"
       "              }\n"
       "            }\n"
       "            tc_commit(&gz_empty[gs]);\n            tc_commit(&z_empty[st]);\n"
       "          }\n"
       "          __syncwarp();\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "    if (elect_one()) tc_commit(done);\n    __syncwarp();\n"
       "  }\n"
       "  else if (warp == 9) {\n"
       "    if (lane == 0) {\n"
       "      u32 uq = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x)\n"
       "        for (int q = Q0; q < Q1; ++q, ++uq) {\n"
       "          const u32 xb = uq % NXB;\n"
       "          mbar_wait_t(&x_empty[xb], ((uq / NXB) & 1u) ^ 1u, 29);\n"
       "          const int dx = P_DX[q];\n"
       "          if (UVW_EXP & 64) { mbar_arrive(&x_full[xb]); continue; }\n"
       "          mbar_expect_tx(&x_full[xb], 4 * KR * 64 * dx);\n"
       "          const TMap* mp = dx == 1 ? &tx1 : dx == 3 ? &tx3 : dx == 5 ? &tx5 : &tx7;\n"
       "          for (int cb = 0; cb < 4; ++cb)\n"
       "            tma_load3(xs0 + (xb * NX + cb) * XSLOT, mp, 0, P_XC[q] + cb * dx, (int)(tile * KR), &x_full[xb]);\n"
       "        }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n"
       "  else if (warp == 10) {\n"
       // gz_k^T tiles from the transposed planes: KR / 32 K blocks of
       // [64 r][32 rows] (SW128, 128-byte box lines), hi and lo: the K-major B
       // layout of the MMA
       "    if (lane == 0) {\n"
       "      u32 ug = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x)\n"
       "        for (int q = Q0; q < Q1; ++q)\n"
       "          for (int k = 0; k < P_DZ[q]; ++k, ++ug) {\n"
       "            const u32 st = ug % NGZ;\n"
       "            mbar_wait_t(&gz_empty[st], ((ug / NGZ) & 1u) ^ 1u, 31);\n"
       "            if (UVW_EXP & 128) { mbar_arrive(&gz_full[st]); continue; }\n"
       "            mbar_expect_tx(&gz_full[st], TB);\n"
       "            unsigned char* d = gzt + st * TB;\n"
       "            for (int b = 0; b < KR / 32; ++b) {\n"
       "              tma_load3(d + b * 8192, &tgh, (int)(tile * KR) + 32 * b, 0, P_PLANE[q] + k, &gz_full[st]);\n"
       "              tma_load3(d + TB / 2 + b * 8192, &tgl, (int)(tile * KR) + 32 * b, 0, P_PLANE[q] + k, &gz_full[st]);\n"
       "            }\n"
       "          }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n"
       "  tc_fence_before();\n  __syncthreads();\n"
       "  if (warp == 8) { tc_fence_after(); asm volatile(\"tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\" :: \"r\"(tmem)); }\n"
       "}\n";
  UvwSource out;
  out.main.name = out.main.module = kname;
  out.main.source = o.str();
  out.main.threads = 352;
  out.main.smem_bytes = smem;
  out.prep = out.main;
  out.prep.name = kname + "_reduce";
  out.prep.threads = 256;
  out.prep.smem_bytes = 0;
  out.tile_rows = kRows;
  return out;
}

namespace {

UvwSource generate_uvw_impl(const Problem& p, const std::string& tag, bool w_transposed) {
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
  }
  // TMEM plan: the A ring (na blocks of hi + lo, 32 columns each) sits at the
  // top, accumulators below it. Segments are allocated around the accumulator
  // ring in processing order; pick the order (and the deepest A ring) whose
  // accumulator reuse leaves the fewest back-to-back waits on an epilogue drain.
  int na = 0;
  {
    std::vector<int> perm(segs.size());
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = static_cast<int>(i);
    int best_score = 1 << 30;
    std::vector<Seg> best;
    const int na_max = std::getenv("CGF_UVW_NA") ? std::atoi(std::getenv("CGF_UVW_NA")) : 4;  // A/B knob
    for (int cand = na_max; cand >= 2 && best.empty(); --cand) {
      const int cap = kTmemCols - 32 * cand;
      bool fits = true;
      for (const auto& sg : segs) fits = fits && sg.dz * sg.n <= cap;
      if (!fits) continue;
      std::sort(perm.begin(), perm.end());
      int iters = 0;
      do {
        std::vector<Seg> o2;
        for (int i : perm) o2.push_back(segs[i]);
        int cur = 0;
        for (auto& sg : o2) {
          const int cols = sg.dz * sg.n;
          if (cur + cols > cap) cur = 0;
          sg.col = cur;
          cur += cols;
        }
        auto ov = [&](const Seg& a, const Seg& b) {
          return a.col < b.col + b.dz * b.n && b.col < a.col + a.dz * a.n;
        };
        int score = 0;
        const int k = static_cast<int>(o2.size());
        for (int i = 1; i < k; ++i) score += ov(o2[i], o2[i - 1]);
        if (k > 1) score += ov(o2[0], o2[k - 1]);
        if (score < best_score) {
          best_score = score;
          best = o2;
        }
      } while (++iters < 5040 && std::next_permutation(perm.begin(), perm.end()));
      if (!best.empty()) na = cand;
    }
    if (best.empty()) throw UnsupportedError("uvw tensor-core path: z segment accumulators exceed TMEM");
    segs = best;
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

  // ---- units: (instruction, 16-channel block) in segment order
  struct U {
    int ins, cb, seg, dz, n, dx;
    bool first, last;
    std::size_t wimg;
  };
  std::vector<U> units;
  int max_n = 16, max_dx = 1;
  for (const auto& s : segs) max_n = std::max(max_n, s.n);
  for (const auto& s : R) max_dx = std::max(max_dx, s.dx());
  const int wslot = 2 * max_n * kCh * 4;                           // hi + lo images, N rows x 16 fp32
  const int xslot = (kTileRows * kCh * max_dx * 4 + 1023) / 1024 * 1024;  // 128 rows x 16 channels x dx
  std::size_t wimg = 0;
  std::vector<std::size_t> wimg_of(np, 0);
  for (int q = 0; q < np; ++q) {
    wimg_of[q] = wimg;
    wimg += static_cast<std::size_t>(R[q].bp / kCh) * wslot;
  }
  // CGF_UVW_ORDER=1: within a segment, channel-block-major (instructions of
  // different dx alternate, so cheap and expensive producer units interleave)
  const int uorder = std::getenv("CGF_UVW_ORDER") ? std::atoi(std::getenv("CGF_UVW_ORDER")) : 0;
  for (int si = 0; si < ns; ++si) {
    const auto& s = segs[si];
    std::vector<std::pair<int, int>> qc;  // (instruction, channel block)
    int maxnb = 0;
    for (int q : s.ins) maxnb = std::max(maxnb, R[q].bp / kCh);
    if (uorder == 1) {
      for (int cb = 0; cb < maxnb; ++cb)
        for (int q : s.ins)
          if (cb < R[q].bp / kCh) qc.push_back({q, cb});
    } else {
      for (int q : s.ins)
        for (int cb = 0; cb < R[q].bp / kCh; ++cb) qc.push_back({q, cb});
    }
    for (size_t t = 0; t < qc.size(); ++t) {
      const int q = qc[t].first, cb = qc[t].second;
      units.push_back({q, cb, si, s.dz, s.n, R[q].dx(), t == 0, t + 1 == qc.size(),
                       wimg_of[q] + static_cast<std::size_t>(cb) * wslot});
    }
  }
  const int nu = static_cast<int>(units.size());
  // producer warps (2 or 4 per SM sub-partition; thread = (row, 16 * 4 / pw
  // channels)) and x-tile ring depth; env overrides for A/B runs.
  const int pw = std::getenv("CGF_UVW_PW") ? std::atoi(std::getenv("CGF_UVW_PW")) : kProdWarps;
  const int nx = std::getenv("CGF_UVW_NX") ? std::atoi(std::getenv("CGF_UVW_NX")) : 3;
  if (pw != 4 && pw != 8 && pw != 16) throw UnsupportedError("CGF_UVW_PW must be 4, 8 or 16");
  const int cpt = kCh * 4 / pw;  // channels per producer thread
  const int nwr = std::getenv("CGF_UVW_NW") ? std::atoi(std::getenv("CGF_UVW_NW")) : 6;  // W ring depth
  // A blocks per TMEM-store round (<= NS / 2 so a batch is written while the other half is consumed);
  // batches of 2 measured 3.45 ms vs 3.36 ms for 1 (profiles/r01_uvw_kb.log), so 1 is the default
  const int kb = std::max(1, std::min(std::getenv("CGF_UVW_KB") ? std::atoi(std::getenv("CGF_UVW_KB")) : 1, na / 2));
  // every producer thread arrives on afull / xempty (no __syncwarp; CGF_UVW_ARV=0
  // restores lane-0 arrives), and the x slot is released after the unit's last
  // A block (CGF_UVW_XREL=0: right after the reads): together C3 forward
  // 2.79 -> 2.75 ms (profiles/r02_ab_uvw5.jsonl)
  const bool pipe_req = std::getenv("CGF_UVW_PIPE") && std::atoi(std::getenv("CGF_UVW_PIPE")) == 1;
  const bool all_arrive = !pipe_req && !(std::getenv("CGF_UVW_ARV") && std::atoi(std::getenv("CGF_UVW_ARV")) == 0);
  const bool xrel_late = !(std::getenv("CGF_UVW_XREL") && std::atoi(std::getenv("CGF_UVW_XREL")) == 0);
  const bool pipe = std::getenv("CGF_UVW_PIPE") && std::atoi(std::getenv("CGF_UVW_PIPE")) == 1;
  // warps: producers | MMA | 4 epilogue | W loader | x loader
  const int mma_warp = pw, wload_warp = pw + 5, xload_warp = pw + 6, nwarps = pw + 7;
  // epilogue staging: per epilogue warp, 32 rows x (8 dz + 4) floats, so each
  // z row piece leaves as contiguous full-sector stores (each thread's own-row
  // float4 stores touched 32 lines per instruction, half a sector each)
  int max_dz = 1;
  for (const auto& sg : segs) max_dz = std::max(max_dz, sg.dz);
  // staged epilogue: C3 forward 3.19 -> 2.79 ms, gx 15.48 -> 15.05 ms of the
  // backward (profiles/r02_ab_uvw2.jsonl); CGF_UVW_EPI=0 restores row stores
  const bool epi_stage = !(std::getenv("CGF_UVW_EPI") && std::atoi(std::getenv("CGF_UVW_EPI")) == 0);
  const int epi_stride = 8 * max_dz + 4;
  const int epi_bytes = epi_stage ? 4 * 32 * epi_stride * 4 : 0;
  const int smem = 1024 /*align*/ + nx * xslot + nwr * wslot + 1024 /*barriers*/ + epi_bytes;
  if (smem > 227 * 1024) throw UnsupportedError("uvw tensor-core path: shared memory too small");
  const int acol0 = kTmemCols - 32 * na;  // A ring columns [acol0, 512)

  std::ostringstream o;
  if (std::getenv("CGF_UVW_DEBUG")) o << "#define CGF_UVW_DEBUG 1\n";
  if (std::getenv("CGF_UVW_PROF")) o << "#define CGF_UVW_PROF 1\n";
  // experiment knobs (A/B only): 1 = epilogue skips stores, 2 = one MMA pass
  // instead of three, 4 = producers skip the TMEM stores
  o << "#define UVW_EXP " << (std::getenv("CGF_UVW_EXP") ? std::atoi(std::getenv("CGF_UVW_EXP")) : 0) << "\n";
  o << device_runtime_source();
  o << uvw_helpers();
  o << "\n// uvw forward: x = " << p.x_ir.str() << " | y = " << p.y_ir.str() << " | z = " << p.z_ir.str() << "\n";
  o << "// " << np << " instructions, " << ns << " z segments, " << nu << " units / 128-row tile, " << na
    << " TMEM A blocks\n";
  o << "#define DIMX " << p.dim_x << "\n#define DIMY " << p.dim_y << "\n#define DIMZ " << p.dim_z << "\n#define NS "
    << na << "\n#define ACOL0 " << acol0 << "\n#define NX " << nx << "\n#define NWR " << nwr << "\n#define WSLOT " << wslot << "\n#define XSLOT " << xslot << "\n#define NSEG " << ns
    << "\n";

  // ---- prep kernel: shared W -> per-(instruction, 16-channel block) images
  const std::string kname = "cgf_uvw_" + tag + "_f32", pname = "cgf_uvw_" + tag + "_prep_f32";
  o << "extern \"C\" __global__ void " << pname << "(const float* __restrict__ W, float* __restrict__ img) {\n"
       "  const int t = blockIdx.x * blockDim.x + threadIdx.x;\n  int e = t;\n";
  for (int q = 0; q < np; ++q) {
    const auto& s = R[q];
    const int cnt = s.b * s.bp;
    o << "  if (e < " << cnt << ") { const int r = e / " << s.bp << ", c = e % " << s.bp << ", cb = c >> 4, cl = c & 15;\n"
      << "    const float v = W[" << s.w_off << " + "
      << (w_transposed ? "c * " + S(s.w_stride) + " + r" : "r * " + S(s.w_stride) + " + c") << "]; const float h = tf32_hi(v);\n"
      << "    char* base = (char*)img + " << wimg_of[q] << " + (size_t)cb * WSLOT;\n"
      << "    const u32 off = sw64(r, cl >> 2) + (cl & 3) * 4;\n"
      << "    *(float*)(base + off) = h; *(float*)(base + " << s.b * kCh * 4 << " + off) = v - h; return; }\n"
      << "  e -= " << cnt << ";\n";
  }
  o << "}\n\n";

  // ---- producer: one function per instruction (CG coefficients as immediates).
  // Thread (row m, sub) owns channels [8 sub, 8 sub + 8) of the unit's 16.
  for (int q = 0; q < np; ++q) {
    const auto& s = R[q];
    const int dx = s.dx(), dz = s.dz();
    o << "// instruction " << q << ": l=(" << s.l1 << "," << s.l2 << "," << s.l3 << ") b=" << s.b << " b'=" << s.bp
      << " nnz=" << s.cg->entries.size() << "\n";
    o << "DEVI void produce_" << q << "(const unsigned char* xs, const float* yv, int m, int sub,"
         " u32 tq, u64* afull, u64* aempty, u64* xempty, u32& slot, u32& ph, u32& pend, u32& pslot) {\n";
    // x: cpt channels x dx floats = cpt * dx / 4 float4 chunks of the staged SW64 tile
    const int nch = cpt * dx / 4;
    o << "  float xv[" << cpt * dx << "];\n#pragma unroll\n  for (int t = 0; t < " << nch
      << "; ++t) {\n    const int g = " << nch << " * sub + t, L = m * " << dx
      << " + (g >> 2), j = g & 3;\n    const float4 v = lds128(xs + L * 64 + ((j ^ ((L >> 1) & 3)) << 4));\n"
         "    xv[4 * t] = v.x; xv[4 * t + 1] = v.y; xv[4 * t + 2] = v.z; xv[4 * t + 3] = v.w;\n  }\n"
         // generic-proxy reads of the slot must be ordered before the next
         // TMA (async proxy) write into it: without this fence the refill
         // raced the reads (measured: corrupted rows).
         "";
    // release of the x slot: right after the reads (default), or (CGF_UVW_XREL=1)
    // after the unit's last A block, when the fence has no loads left to wait on
    const std::string xrel = std::string(std::getenv("CGF_UVW_EXP") && (std::atoi(std::getenv("CGF_UVW_EXP")) & 8) ? "" : "  fence_proxy_async();\n") +
                             (all_arrive ? "  mbar_arrive(xempty);\n" : "  __syncwarp();\n  if ((threadIdx.x & 31) == 0) mbar_arrive(xempty);\n");
    if (!xrel_late) o << xrel;
    o << "  float q[" << dz << "][" << dx << "];\n#pragma unroll\n  for (int k = 0; k < " << dz
      << "; ++k)\n#pragma unroll\n    for (int i = 0; i < " << dx << "; ++i) q[k][i] = 0.f;\n";
    for (const auto& e : s.cg->entries)
      o << "  q[" << e.k << "][" << e.i << "] = fmaf((float)" << hexd(e.v) << ", yv[" << s.y_off + e.j << "], q[" << e.k
        << "][" << e.i << "]);\n";
    // A block k -> TMEM columns [ACOL0 + 32 slot, +32): hi in the first 16, lo in
    // the next 16; this thread's row is its TMEM lane, its channels its columns.
    // Blocks go out in batches of kb: all of a batch's values are computed
    // before its slots are awaited, and one tcgen05.wait::st + fence + arrive
    // round covers the batch (the per-block round trip dominated the loop).
    if (pipe) {
      // Software-pipelined TMEM stores: block k's stores are issued, and their
      // completion (tcgen05.wait::st) + the afull arrive happen only after
      // block k+1's values are computed -- the store round trip overlaps the
      // next block's FMAs instead of stalling the warp (pend / pslot carry the
      // outstanding block across units; the caller flushes it at the end).
      for (int k = 0; k < dz; ++k) {
        o << "  {\n    float h[" << cpt << "], l[" << cpt << "];\n#pragma unroll\n    for (int c = 0; c < " << cpt
          << "; ++c) {\n      float z = 0.f;\n#pragma unroll\n      for (int i = 0; i < " << dx
          << "; ++i) z = fmaf(q[" << k << "][i], xv[c * " << dx << " + i], z);\n"
          << "      h[c] = tf32_hi(z); l[c] = z - h[c];\n    }\n"
          << "    if (pend) { tc_wait_st(); tc_fence_before(); __syncwarp(); if ((threadIdx.x & 31) == 0) mbar_arrive(&afull[pslot]); pend = 0; }\n"
          << "    mbar_wait_t(&aempty[slot], ph ^ 1u, 1);\n    tc_fence_after();\n"
          << "    { const u32 ta = tq + ACOL0 + 32 * slot + " << cpt << " * sub;\n"
          << "      if (!(UVW_EXP & 4)) { tc_st" << cpt << "(ta, h); tc_st" << cpt << "(ta + 16, l); } }\n"
          << "    pslot = slot; pend = 1;\n    if (++slot == NS) { slot = 0; ph ^= 1u; }\n  }\n";
      }
      if (xrel_late) o << xrel;
      o << "}\n\n";
      continue;
    }
    for (int k0 = 0; k0 < dz; k0 += kb) {
      const int nk = std::min(kb, dz - k0);
      o << "  {\n    float h[" << nk << "][" << cpt << "], l[" << nk << "][" << cpt << "];\n";
      for (int t = 0; t < nk; ++t)
        o << "#pragma unroll\n    for (int c = 0; c < " << cpt << "; ++c) {\n"
          << "      float z = 0.f;\n#pragma unroll\n      for (int i = 0; i < " << dx
          << "; ++i) z = fmaf(q[" << k0 + t << "][i], xv[c * " << dx << " + i], z);\n"
          << "      h[" << t << "][c] = tf32_hi(z); l[" << t << "][c] = z - h[" << t << "][c];\n    }\n";
      o << "    u32 s_ = slot, p_ = ph;\n";
      for (int t = 0; t < nk; ++t) {
        o << "    mbar_wait_t(&aempty[s_], p_ ^ 1u, 1);\n";
        if (t == 0) o << "    tc_fence_after();\n";
        o << "    { const u32 ta = tq + ACOL0 + 32 * s_ + " << cpt << " * sub;\n"
          << "      if (!(UVW_EXP & 4)) { tc_st" << cpt << "(ta, h[" << t << "]); tc_st" << cpt << "(ta + 16, l[" << t << "]); } }\n"
          << "    if (++s_ == NS) { s_ = 0; p_ ^= 1u; }\n";
      }
      o << "    tc_wait_st();\n    tc_fence_before();\n"
        << (all_arrive ? "    { u32 a_ = slot;" : "    __syncwarp();\n    if ((threadIdx.x & 31) == 0) { u32 a_ = slot;");
      for (int t = 0; t < nk; ++t) o << " mbar_arrive(&afull[a_]);" << (t + 1 < nk ? " if (++a_ == NS) a_ = 0;" : "");
      o << " }\n    slot = s_; ph = p_;\n  }\n";
    }
    if (xrel_late) o << xrel;
    o << "}\n\n";
  }

  // ---- unit / segment tables
  auto arr = [&](const char* name, const std::vector<long long>& v) {
    o << "__constant__ int " << name << "[" << std::max<size_t>(1, v.size()) << "] = {";
    for (size_t i = 0; i < v.size(); ++i) o << (i ? "," : "") << v[i];
    if (v.empty()) o << "0";
    o << "};\n";
  };
  {
    std::vector<long long> udz, ucol, un, ufirst, ulast, useg, uw, udx, uxc, uins;
    for (const auto& u : units) {
      uins.push_back(u.ins);
      udz.push_back(u.dz);
      ucol.push_back(segs[u.seg].col);
      un.push_back(u.n);
      ufirst.push_back(u.first);
      ulast.push_back(u.last);
      useg.push_back(u.seg);
      uw.push_back(static_cast<long long>(u.wimg));
      udx.push_back(u.dx);
      uxc.push_back((R[u.ins].x_off + static_cast<long long>(u.cb) * kCh * u.dx) / kCh);  // TMA coordinate 1
    }
    arr("U_DZ", udz);
    arr("U_COL", ucol);
    arr("U_N", un);
    arr("U_FIRST", ufirst);
    arr("U_LAST", ulast);
    arr("U_SEG", useg);
    arr("U_WIMG", uw);
    arr("U_DX", udx);
    arr("U_XC", uxc);
    arr("U_INS", uins);
    std::vector<long long> swc, swp;
    for (int si = 0; si < ns; ++si) {
      swc.push_back(wait_cur[si]);
      swp.push_back(wait_prev[si]);
    }
    arr("S_WAITCUR", swc);
    arr("S_WAITPREV", swp);
  }
  o << "#define NU " << nu << "\n\n";

  // ---- the main kernel
  o << "extern \"C\" __global__ void __launch_bounds__(" << nwarps * 32 << ", 1) " << kname << "("
       "const __grid_constant__ TMap tx1, const __grid_constant__ TMap tx3, const __grid_constant__ TMap tx5, "
       "const __grid_constant__ TMap tx7, const float* __restrict__ Y, const float* __restrict__ WIMG, "
       "float* __restrict__ Z, i64 rows, unsigned long long* __restrict__ prof) {\n"
       "#ifdef CGF_UVW_PROF\n  if (threadIdx.x < 16) prof_s[threadIdx.x] = 0;\n  const long long kc0 = clock64();\n#endif\n"
       "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n"
       "  unsigned char* sm = (unsigned char*)(((unsigned long long)smem_raw + 1023) & ~1023ull);\n"
       "  unsigned char* xbase = sm;\n"
       "  unsigned char* wbase = xbase + NX * XSLOT;\n"
       "  u64* bars = (u64*)(wbase + NWR * WSLOT);\n"
       "  u64* afull = bars; u64* aempty = afull + NS; u64* wfull = aempty + NS; u64* wempty = wfull + NWR;\n"
       "  u64* xfull = wempty + NWR; u64* xempty = xfull + NX;\n"
       "  u64* sfull = xempty + NX; u64* sdrained = sfull + NSEG;\n"
       "  u32* tmem_slot = (u32*)(sdrained + NSEG);\n"
       "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n"
       "  const i64 ntiles = (rows + 127) / 128;\n"
       "  const i64 my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;\n"
       "  if (threadIdx.x == 0) {\n"
       "    for (int i = 0; i < NS; ++i) { mbar_init(&afull[i], "
    << (all_arrive ? pw * 32 : pw)
    << "); mbar_init(&aempty[i], 1); }\n"
       "    for (int i = 0; i < NWR; ++i) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], 1); }\n"
       "    for (int i = 0; i < NX; ++i) { mbar_init(&xfull[i], 1); mbar_init(&xempty[i], "
    << (all_arrive ? pw * 32 : pw)
    << "); }\n"
       "    for (int i = 0; i < NSEG; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sdrained[i], 4); }\n"
       "    mbar_fence_init();\n  }\n"
       "  if (warp == "
    << mma_warp
    << ") {\n"
       "    asm volatile(\"tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\" :: \"r\"(smem_addr(tmem_slot)));\n"
       "    asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\");\n"
       "  }\n"
       "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n"
       "  const u32 tmem = 0;  // all 512 columns are ours: the allocation starts at lane 0, column 0\n"
       "  if (threadIdx.x == 0 && *tmem_slot != 0) { printf(\"cgf_uvw: unexpected TMEM base %u\\n\", *tmem_slot); __trap(); }\n\n";

  // producers
  o << "  if (warp < " << pw
    << ") {\n"
       "    const int m = 32 * (warp & 3) + lane, sub = warp >> 2;\n"
       "    const u32 tq = tmem + ((u32)(32 * (warp & 3)) << 16);\n"
       "    u32 slot = 0, ph = 0, gx = 0, pend = 0, pslot = 0;\n"
       "    for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
       "      const i64 row = tile * 128 + m;\n"
       "      const bool valid = row < rows;\n"
       "      float yv[DIMY];\n"
       "#pragma unroll\n      for (int j = 0; j < DIMY; ++j) yv[j] = valid ? __ldg(Y + row * DIMY + j) : 0.f;\n";
  // runtime unit loop, one switch arm per instruction: the body stays
  // instruction-cache resident (the unrolled unit sequence was i-cache bound)
  o << "#pragma unroll 1\n      for (int u = 0; u < NU; ++u) {\n"
       "        const u32 xs_ = gx % NX; mbar_wait_t(&xfull[xs_], (gx / NX) & 1u, 8); ++gx;\n"
       "        const unsigned char* xsl = xbase + xs_ * XSLOT;\n"
       "        switch (U_INS[u]) {\n";
  for (int q = 0; q < np; ++q)
    o << "          case " << q << ": produce_" << q << "(xsl, yv, m, sub, tq, afull, aempty, &xempty[xs_], slot, ph, pend, pslot); break;\n";
  o << "        }\n      }\n";
  o << "    }\n"
       "    if (pend) { tc_wait_st(); tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&afull[pslot]); }\n"
       "  }\n";

  // MMA issuer
  o << "  else if (warp == " << mma_warp
    << ") {\n"
       // The whole warp walks the schedule (so every loop value is warp-uniform
       // and lives in uniform registers) and one elected lane issues each
       // tcgen05.mma / commit. TMEM addresses are compile-time: the kernel owns
       // all 512 columns, so the allocation base is column 0 (checked below).
       // The naive lane-0 loop with per-MMA descriptor rebuilds measured
       // ~150 cycles per MMA (tools/tc_bench.cu); this form is tensor-bound.
       "    {\n"
       "      const u64 wd0 = sdesc64(smem_addr(wbase));\n"
       "      u32 slot = 0, ph = 0, wsl = 0, wph = 0; i64 lt = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {\n"
       "        for (int u = 0; u < NU; ++u) {\n"
       "          if (U_FIRST[u]) {\n"
       "            const int s = U_SEG[u];\n"
       "            for (int o = 0; o < NSEG; ++o) {\n"
       "              if (S_WAITCUR[s] >> o & 1) mbar_wait_t(&sdrained[o], (u32)(lt & 1), 3);\n"
       "              if ((S_WAITPREV[s] >> o & 1) && lt > 0) mbar_wait_t(&sdrained[o], (u32)((lt - 1) & 1), 4);\n"
       "            }\n"
       "            tc_fence_after();\n"
       "          }\n"
       "          mbar_wait_t(&wfull[wsl], wph, 5);\n"
       "          tc_fence_after();\n"
       "          const int n = U_N[u];\n"
       "          const u32 idesc = idesc_tf32(n), first = U_FIRST[u];\n"
       "          const u64 bh = wd0 + (u64)(wsl * (WSLOT >> 4)), bl = bh + (u64)((n * 64) >> 4);\n"
       "          const u32 dbase = (u32)U_COL[u];\n"
       "          for (int k = 0; k < U_DZ[u]; ++k) {\n"
       "            mbar_wait_t(&afull[slot], ph, 6);\n"
       "            tc_fence_after();\n"
       "            const u32 ah = ACOL0 + 32 * slot, al = ah + 16;\n"
       "            const u32 d = dbase + (u32)(k * n);\n"
       "            if (elect_one()) {\n"
       // 3xTF32: hi*hi + hi*lo + lo*hi, two K=8 steps (A: +8 columns, B: +32 B) each
       "              tc_mma_ts(d, ah, bh, idesc, first ? 0u : 1u);\n"
       "              tc_mma_ts(d, ah + 8, bh + 2, idesc, 1u);\n"
       "              if (!(UVW_EXP & 2)) {\n"
       "              tc_mma_ts(d, ah, bl, idesc, 1u);\n"
       "              tc_mma_ts(d, ah + 8, bl + 2, idesc, 1u);\n"
       "              tc_mma_ts(d, al, bh, idesc, 1u);\n"
       "              tc_mma_ts(d, al + 8, bh + 2, idesc, 1u);\n"
       "              }\n"
       "              tc_commit(&aempty[slot]);\n"
       "            }\n"
       "            __syncwarp();\n"
       "            if (++slot == NS) { slot = 0; ph ^= 1u; }\n"
       "          }\n"
       "          if (elect_one()) {\n"
       "            tc_commit(&wempty[wsl]);\n"
       "            if (U_LAST[u]) tc_commit(&sfull[U_SEG[u]]);\n"
       "          }\n"
       "          __syncwarp();\n"
       "          if (++wsl == NWR) { wsl = 0; wph ^= 1u; }\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "  }\n";

  // TMA loaders, one warp each so neither ring's wait blocks the other:
  // W images (ring of NWR, 1-D bulk copies) and x tiles (ring of NX, 3-D
  // tensor copies), both in unit order.
  o << "  else if (warp == " << wload_warp
    << ") {\n"
       "    if (lane == 0) {\n"
       "      u32 gu = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
       "        for (int u = 0; u < NU; ++u, ++gu) {\n"
       "          const u32 ws = gu % NWR;\n"
       "          mbar_wait_t(&wempty[ws], ((gu / NWR) & 1u) ^ 1u, 2);\n"
       "          mbar_expect_tx(&wfull[ws], WSLOT);\n"
       "          bulk_g2s(wbase + ws * WSLOT, (const char*)WIMG + U_WIMG[u], WSLOT, &wfull[ws]);\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n"
       "  else if (warp == "
    << xload_warp
    << ") {\n"
       "    if (lane == 0) {\n"
       "      u32 gu = 0;\n"
       "      for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {\n"
       "        for (int u = 0; u < NU; ++u, ++gu) {\n"
       "          const u32 xs = gu % NX;\n"
       "          mbar_wait_t(&xempty[xs], ((gu / NX) & 1u) ^ 1u, 12);\n"
       "          const int dx = U_DX[u];\n"
       "          mbar_expect_tx(&xfull[xs], 128 * 64 * dx);\n"
       "          const TMap* mp = dx == 1 ? &tx1 : dx == 3 ? &tx3 : dx == 5 ? &tx5 : &tx7;\n"
       "          tma_load3(xbase + xs * XSLOT, mp, 0, U_XC[u], (int)(tile * 128), &xfull[xs]);\n"
       "        }\n"
       "      }\n"
       "    }\n"
       "    __syncwarp();\n"
       "  }\n";

  // epilogue: per segment (compile-time dz, n), TMEM -> registers -> z row
  o << "  else {\n"
       "    const int qd = warp & 3, m = 32 * qd + lane;\n"
    << (epi_stage ? "    float* stg = (float*)((unsigned char*)bars + 1024) + qd * " + S(32 * epi_stride) + ";\n" : "")
    << ""
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
    if (epi_stage) {
      // rows -> the warp's staging rows (stride 8 dz + 4 floats: conflict-free
      // v4 stores), then lanes walk the 32 rows' contiguous 8 dz floats
      const int st = 8 * sg.dz + 4, nq = 2 * sg.dz;
      o << "          tc_wait_ld();\n          {\n            float* sr = stg + lane * " << st << ";\n";
      for (int t = 0; t < nq; ++t) {
        o << "            sts128((unsigned char*)(sr + " << 4 * t << "), make_float4(";
        for (int a = 0; a < 4; ++a) {
          const int f = 4 * t + a, rr = f / sg.dz, kk = f % sg.dz;
          o << (a ? ", " : "") << "v[" << kk << "][" << rr << "]";
        }
        o << "));\n";
      }
      o << "          }\n          __syncwarp();\n"
        << "          if (!(UVW_EXP & 1))\n"
        << "          for (int i = lane; i < " << 32 * nq << "; i += 32) {\n"
        << "            const int rw = i / " << nq << ", pq = i - rw * " << nq << ";\n"
        << "            const i64 grow = tile * 128 + 32 * qd + rw;\n"
        << "            if (grow < rows) __stcs((float4*)(Z + grow * DIMZ + " << sg.z_off << " + r0 * " << sg.dz
        << ") + pq, lds128((const unsigned char*)(stg + rw * " << st << " + 4 * pq)));\n          }\n"
        << "          __syncwarp();\n";
      o << "        }\n        tc_fence_before();\n        __syncwarp();\n";
    } else {
    o << "          tc_wait_ld();\n          if (valid && !(UVW_EXP & 1)) {\n            float4* dst = (float4*)(zr + r0 * " << sg.dz << ");\n";
    for (int t = 0; t < 2 * sg.dz; ++t) {
      o << "            __stcs(dst + " << t << ", make_float4(";
      for (int a = 0; a < 4; ++a) {
        const int f = 4 * t + a, rr = f / sg.dz, kk = f % sg.dz;
        o << (a ? ", " : "") << "v[" << kk << "][" << rr << "]";
      }
      o << "));\n";
    }
    o << "          }\n        }\n        tc_fence_before();\n        __syncwarp();\n";
    }
    o << ""
      << "        if (lane == 0) mbar_arrive(&sdrained[" << si << "]);\n      }\n";
  }
  o << "    }\n  }\n";
  o << "  tc_fence_before();\n"
       "  __syncthreads();\n"
       "#ifdef CGF_UVW_PROF\n  if (threadIdx.x < 16) atomicAdd(&prof[threadIdx.x], prof_s[threadIdx.x]);\n"
       "  if (threadIdx.x == 0) atomicAdd(&prof[15], (unsigned long long)(clock64() - kc0));\n#endif\n"
       "  if (warp == "
    << mma_warp
    << ") {\n"
       "    tc_fence_after();\n"
       "    asm volatile(\"tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\" :: \"r\"(*tmem_slot));\n"
       "  }\n"
       "}\n";

  UvwSource out;
  out.main.name = kname;
  out.main.source = o.str();
  out.main.threads = nwarps * 32;
  out.main.smem_bytes = smem;
  out.main.units = nu;
  out.prep = out.main;
  out.prep.name = pname;
  out.prep.threads = 256;
  out.prep.smem_bytes = 0;
  out.main.module = out.prep.module = kname;
  out.wimg_bytes = wimg;
  out.dims_x = p.dim_x;
  return out;
}

}  // namespace

}  // namespace cgf
