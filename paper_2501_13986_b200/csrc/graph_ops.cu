// Device graph utilities (conv.cpp:64-151) and the unfused convolution's
// gather / segmented-sum kernels (conv.cpp:530-616) for sm_100a.
//
// All of this is HBM- or latency-bound integer and copy work: the kernels are
// grid-stride loops sized to the SM count, with 16-byte vector accesses where
// the row width allows; the sorts are CUB's device radix sort (a library
// primitive, like cuBLAS for a GEMM). Integer outputs are bit-identical to the
// reference's host construction (tests/test_gpu_graph.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cub/cub.cuh>
#include <string>

#include "graph_ops.hpp"
#include "problem.hpp"

namespace cgf::gops {

namespace {

using i64 = long long;
using u64 = unsigned long long;

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}
#define CK(x) ck((x), #x)

int g_sms = 0;
unsigned grid_for(i64 items, int threads) {
  if (!g_sms) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const i64 need = (items + threads - 1) / threads;
  return static_cast<unsigned>(std::max<i64>(1, std::min<i64>(need, static_cast<i64>(g_sms) * 16)));
}

int bits_for(i64 v) {  // bits needed to represent 0..v
  int b = 1;
  while (b < 63 && (static_cast<u64>(1) << b) <= static_cast<u64>(std::max<i64>(v, 1))) ++b;
  return b;
}

// RAII stream-ordered buffer
struct Buf {
  void* p = nullptr;
  cudaStream_t st;
  Buf(std::size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) CK(cudaMallocAsync(&p, bytes, st));
  }
  ~Buf() {
    if (p) cudaFreeAsync(p, st);
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// ---- kernels ----------------------------------------------------------------

__global__ void k_gather(const char* __restrict__ src, const int* __restrict__ idx, char* __restrict__ dst, i64 n,
                         int row_bytes, int vec) {
  const int lane = threadIdx.x & 31;
  const i64 w0 = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
  const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
  for (i64 r = w0; r < n; r += nw) {
    const char* s = src + static_cast<i64>(idx[r]) * row_bytes;
    char* d = dst + r * row_bytes;
    if (vec) {
      const int n16 = row_bytes / 16;
      for (int i = lane; i < n16; i += 32) __stcs(reinterpret_cast<float4*>(d) + i, __ldg(reinterpret_cast<const float4*>(s) + i));
    } else {
      const int n4 = row_bytes / 4;
      for (int i = lane; i < n4; i += 32) reinterpret_cast<float*>(d)[i] = reinterpret_cast<const float*>(s)[i];
    }
  }
}

template <class T, class V, int W>
__global__ void k_segsum(const T* __restrict__ rows, const i64* __restrict__ rp, const int* __restrict__ idx,
                         T* __restrict__ out, i64 nodes, int dim, int vec) {
  const int ncol = vec ? dim / W : dim;
  const i64 total = nodes * ncol;
  for (i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 v = t / ncol;
    const int c = static_cast<int>(t - v * ncol);
    const i64 q0 = rp[v], q1 = rp[v + 1];
    if (vec) {
      T acc[W];
#pragma unroll
      for (int k = 0; k < W; ++k) acc[k] = T(0);
      for (i64 q = q0; q < q1; ++q) {
        const i64 e = idx ? idx[q] : q;
        const V r = __ldg(reinterpret_cast<const V*>(rows + e * dim) + c);
        const T* rr = reinterpret_cast<const T*>(&r);
#pragma unroll
        for (int k = 0; k < W; ++k) acc[k] += rr[k];
      }
      V o;
      T* oo = reinterpret_cast<T*>(&o);
#pragma unroll
      for (int k = 0; k < W; ++k) oo[k] = acc[k];
      reinterpret_cast<V*>(out + v * dim)[c] = o;
    } else {
      T acc = T(0);
      for (i64 q = q0; q < q1; ++q) acc += rows[(idx ? idx[q] : q) * static_cast<i64>(dim) + c];
      out[v * dim + c] = acc;
    }
  }
}

__global__ void k_expand(const i64* __restrict__ rp, i64 nodes, int* __restrict__ src) {
  for (i64 v = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; v < nodes;
       v += static_cast<i64>(gridDim.x) * blockDim.x)
    for (i64 e = rp[v]; e < rp[v + 1]; ++e) src[e] = static_cast<int>(v);
}

// dst[c] (+)= sum over r < rows of src[r * n + c], summed in row order (the
// shared-W weight gradient's reduction over per-row partials; deterministic).
template <typename T>
__global__ void k_colsum(const T* __restrict__ src, i64 rows, i64 n, i64 ld, T* __restrict__ dst, int accumulate) {
  for (i64 c = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; c < n;
       c += static_cast<i64>(gridDim.x) * blockDim.x) {
    T acc = accumulate ? dst[c] : T(0);
    i64 r = 0;
    for (; r + 8 <= rows; r += 8) {
      T v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldg(src + (r + k) * ld + c);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
    }
    for (; r < rows; ++r) acc += __ldg(src + r * ld + c);
    dst[c] = acc;
  }
}

// transposed CSR -> edge list in edge order: position q of bucket d is edge
// t_eid[q] = (t_src[q], d)
__global__ void k_untranspose(const i64* __restrict__ trp, i64 in_nodes, const int* __restrict__ t_src,
                              const int* __restrict__ t_eid, int* __restrict__ src, int* __restrict__ dst) {
  for (i64 d = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; d < in_nodes;
       d += static_cast<i64>(gridDim.x) * blockDim.x)
    for (i64 q = trp[d]; q < trp[d + 1]; ++q) {
      const int e = t_eid[q];
      src[e] = t_src[q];
      dst[e] = static_cast<int>(d);
    }
}

__global__ void k_validate(const int* __restrict__ src, const int* __restrict__ dst, i64 edges, i64 nodes,
                           int allow_self, u64* first_bad) {
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < edges;
       e += static_cast<i64>(gridDim.x) * blockDim.x) {
    const int s = src[e], d = dst[e];
    const bool bad = s < 0 || s >= nodes || d < 0 || d >= nodes || (!allow_self && s == d);
    if (bad) atomicMin(first_bad, static_cast<u64>(e));
  }
}

__global__ void k_keys(const int* __restrict__ src, const int* __restrict__ dst, i64 edges, u64* __restrict__ keys) {
  for (i64 e = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; e < edges;
       e += static_cast<i64>(gridDim.x) * blockDim.x)
    keys[e] = (static_cast<u64>(static_cast<unsigned>(src[e])) << 32) | static_cast<unsigned>(dst[e]);
}

__global__ void k_split(const u64* __restrict__ keys, i64 n, int* __restrict__ nbr, int* __restrict__ src) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    nbr[i] = static_cast<int>(keys[i] & 0xffffffffull);
    if (src) src[i] = static_cast<int>(keys[i] >> 32);
  }
}

template <class K>
__device__ i64 lower_bound(const K* a, i64 n, K key) {
  i64 lo = 0, hi = n;
  while (lo < hi) {
    const i64 mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// rp[v] = first position whose key >= v << shift, for v in [0, nodes]
template <class K>
__global__ void k_rowptr(const K* __restrict__ keys, i64 n, i64 nodes, int shift, i64* __restrict__ rp) {
  for (i64 v = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; v <= nodes;
       v += static_cast<i64>(gridDim.x) * blockDim.x)
    rp[v] = v == nodes ? n : lower_bound<K>(keys, n, static_cast<K>(static_cast<u64>(v) << shift));
}

__global__ void k_iota(int* a, i64 n) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    a[i] = static_cast<int>(i);
}

__global__ void k_take(const int* __restrict__ table, const int* __restrict__ idx, int* __restrict__ out, i64 n) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    out[i] = table[idx[i]];
}

// ---- radius graph -----------------------------------------------------------

constexpr int kCellBits = 21;  // per-axis cell coordinate bits in a 63-bit cell key
constexpr i64 kCellMax = (1ll << kCellBits) - 1;

__global__ void k_min3(const double* __restrict__ pos, i64 n, double* __restrict__ lo) {
  __shared__ double red[3][1024];
  double m[3] = {pos[0], pos[1], pos[2]};
  for (i64 i = threadIdx.x; i < n; i += blockDim.x)
    for (int d = 0; d < 3; ++d) m[d] = fmin(m[d], pos[3 * i + d]);
  for (int d = 0; d < 3; ++d) red[d][threadIdx.x] = m[d];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int d = 0; d < 3; ++d) red[d][threadIdx.x] = fmin(red[d][threadIdx.x], red[d][threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x < 3) lo[threadIdx.x] = red[threadIdx.x][0];
}

__device__ __forceinline__ i64 cell_coord(double p, double lo, double r) { return static_cast<i64>(floor(__ddiv_rn(__dsub_rn(p, lo), r))); }

__global__ void k_cells(const double* __restrict__ pos, i64 n, const double* __restrict__ lo, double r,
                        u64* __restrict__ key, int* __restrict__ overflow) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    u64 k = 0;
    for (int d = 0; d < 3; ++d) {
      const i64 c = cell_coord(pos[3 * i + d], lo[d], r);
      if (c < 0 || c > kCellMax) *overflow = 1;
      k = (k << kCellBits) | static_cast<u64>(c & kCellMax);
    }
    key[i] = k;
  }
}

// One thread per atom: scan the 27 neighbouring cells (binary search in the
// cell-sorted atom list); count, or write the (i, j) keys at row_ptr[i].
__global__ void k_pairs(const double* __restrict__ pos, i64 n, const double* __restrict__ lo, double r, double r2,
                        const u64* __restrict__ skey, const int* __restrict__ satom, i64* __restrict__ count,
                        const i64* __restrict__ rp, u64* __restrict__ out) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const double px = pos[3 * i], py = pos[3 * i + 1], pz = pos[3 * i + 2];
    const i64 c0 = cell_coord(px, lo[0], r), c1 = cell_coord(py, lo[1], r), c2 = cell_coord(pz, lo[2], r);
    i64 cnt = 0;
    i64 w = out ? rp[i] : 0;
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const i64 a = c0 + dx, b = c1 + dy, c = c2 + dz;
          if (a < 0 || b < 0 || c < 0 || a > kCellMax || b > kCellMax || c > kCellMax) continue;
          const u64 key = (static_cast<u64>(a) << (2 * kCellBits)) | (static_cast<u64>(b) << kCellBits) | static_cast<u64>(c);
          for (i64 k = lower_bound<u64>(skey, n, key); k < n && skey[k] == key; ++k) {
            const int j = satom[k];
            if (j == i) continue;
            const double ddx = __dsub_rn(px, pos[3 * j]), ddy = __dsub_rn(py, pos[3 * j + 1]),
                         ddz = __dsub_rn(pz, pos[3 * j + 2]);
            // (ddx*ddx + ddy*ddy) + ddz*ddz, each rounded: the reference is built with -ffp-contract=off
            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(ddy, ddy)), __dmul_rn(ddz, ddz));
            if (d2 <= r2) {
              if (out) out[w++] = (static_cast<u64>(i) << 32) | static_cast<unsigned>(j);
              ++cnt;
            }
          }
        }
    if (count) count[i] = cnt;
  }
}

template <class F>
void cub_call(cudaStream_t st, F&& f) {
  std::size_t bytes = 0;
  CK(f(nullptr, bytes));
  Buf tmp(std::max<std::size_t>(bytes, 16), st);
  CK(f(tmp.p, bytes));
}

}  // namespace

// ---- unfused conv data movement -------------------------------------------

void gather_rows(bool f64, const void* src, const std::int32_t* idx, void* dst, std::int64_t n, int dim, void* stream) {
  if (n <= 0) return;
  const int rb = dim * (f64 ? 8 : 4);
  const int vec = (rb % 16 == 0) && !(reinterpret_cast<std::uintptr_t>(src) & 15) && !(reinterpret_cast<std::uintptr_t>(dst) & 15);
  k_gather<<<grid_for(n * 32, 256), 256, 0, S(stream)>>>(static_cast<const char*>(src), idx, static_cast<char*>(dst), n,
                                                         rb, vec);
  CK(cudaGetLastError());
}

void segment_sum(bool f64, const void* rows, const std::int64_t* rp, const std::int32_t* idx, void* out,
                 std::int64_t nodes, int dim, void* stream) {
  if (nodes <= 0) return;
  const bool al = !(reinterpret_cast<std::uintptr_t>(rows) & 15) && !(reinterpret_cast<std::uintptr_t>(out) & 15);
  if (f64) {
    const int vec = al && dim % 2 == 0;
    const i64 items = nodes * (vec ? dim / 2 : dim);
    k_segsum<double, double2, 2><<<grid_for(items, 256), 256, 0, S(stream)>>>(
        static_cast<const double*>(rows), reinterpret_cast<const i64*>(rp), idx, static_cast<double*>(out), nodes, dim, vec);
  } else {
    const int vec = al && dim % 4 == 0;
    const i64 items = nodes * (vec ? dim / 4 : dim);
    k_segsum<float, float4, 4><<<grid_for(items, 256), 256, 0, S(stream)>>>(
        static_cast<const float*>(rows), reinterpret_cast<const i64*>(rp), idx, static_cast<float*>(out), nodes, dim, vec);
  }
  CK(cudaGetLastError());
}

void rowptr_expand(const std::int64_t* rp, std::int64_t nodes, std::int32_t* src, void* stream) {
  if (nodes <= 0) return;
  k_expand<<<grid_for(nodes, 256), 256, 0, S(stream)>>>(reinterpret_cast<const i64*>(rp), nodes, src);
  CK(cudaGetLastError());
}

void column_sum(bool f64, const void* src, std::int64_t rows, std::int64_t n, void* dst, bool accumulate,
                void* stream, std::int64_t ld) {
  if (n <= 0) return;
  if (ld <= 0) ld = n;
  const int acc = accumulate ? 1 : 0;
  if (f64)
    k_colsum<double><<<grid_for(n, 128), 128, 0, S(stream)>>>(static_cast<const double*>(src), rows, n, ld,
                                                              static_cast<double*>(dst), acc);
  else
    k_colsum<float><<<grid_for(n, 128), 128, 0, S(stream)>>>(static_cast<const float*>(src), rows, n, ld,
                                                             static_cast<float*>(dst), acc);
  CK(cudaGetLastError());
}

void untranspose(const std::int64_t* t_row_ptr, std::int64_t in_nodes, const std::int32_t* t_src,
                 const std::int32_t* t_eid, std::int32_t* src, std::int32_t* dst, void* stream) {
  if (in_nodes <= 0) return;
  k_untranspose<<<grid_for(in_nodes, 256), 256, 0, S(stream)>>>(reinterpret_cast<const i64*>(t_row_ptr), in_nodes,
                                                                 t_src, t_eid, src, dst);
  CK(cudaGetLastError());
}

// ---- graph construction ---------------------------------------------------

std::int64_t make_graph(std::int64_t nodes, std::int64_t edges, const std::int32_t* src, const std::int32_t* dst,
                        bool allow_self_loops, std::int64_t* row_ptr, std::int32_t* nbr, std::int32_t* out_src,
                        void* stream) {
  const cudaStream_t st = S(stream);
  if (nodes < 0 || edges < 0) throw ShapeError("negative graph size");
  if (edges > 0) {
    Buf bad(sizeof(u64), st);
    CK(cudaMemsetAsync(bad.p, 0xff, sizeof(u64), st));
    k_validate<<<grid_for(edges, 256), 256, 0, st>>>(src, dst, edges, nodes, allow_self_loops ? 1 : 0, bad.as<u64>());
    CK(cudaGetLastError());
    u64 first = 0;
    CK(cudaMemcpyAsync(&first, bad.p, sizeof first, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (first != ~0ull) {
      int sd[2];
      CK(cudaMemcpy(&sd[0], src + first, 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(&sd[1], dst + first, 4, cudaMemcpyDeviceToHost));
      if (sd[0] < 0 || sd[0] >= nodes || sd[1] < 0 || sd[1] >= nodes)
        throw std::invalid_argument("make_graph: edge endpoint out of range");
      throw std::invalid_argument("make_graph: self-loop (" + std::to_string(sd[0]) + ")");
    }
  }
  std::int64_t m = 0;
  if (edges > 0) {
    Buf keys(8 * edges, st), sorted(8 * edges, st), uniq(8 * edges, st), num(8, st);
    k_keys<<<grid_for(edges, 256), 256, 0, st>>>(src, dst, edges, keys.as<u64>());
    CK(cudaGetLastError());
    const int end_bit = 32 + bits_for(nodes);
    cub_call(st, [&](void* t, std::size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, keys.as<u64>(), sorted.as<u64>(), edges, 0, end_bit, st);
    });
    cub_call(st, [&](void* t, std::size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted.as<u64>(), uniq.as<u64>(), num.as<i64>(), edges, st);
    });
    CK(cudaMemcpyAsync(&m, num.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    k_split<<<grid_for(m, 256), 256, 0, st>>>(uniq.as<u64>(), m, nbr, out_src);
    CK(cudaGetLastError());
    k_rowptr<u64><<<grid_for(nodes + 1, 256), 256, 0, st>>>(uniq.as<u64>(), m, nodes, 32, reinterpret_cast<i64*>(row_ptr));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));  // scratch is freed stream-ordered; results ready on return
  } else {
    CK(cudaMemsetAsync(row_ptr, 0, 8 * (nodes + 1), st));
    CK(cudaStreamSynchronize(st));
  }
  return m;
}

void transpose(std::int64_t out_nodes, std::int64_t in_nodes, std::int64_t edges, const std::int64_t* row_ptr,
               const std::int32_t* nbr, std::int64_t* t_row_ptr, std::int32_t* t_src, std::int32_t* t_eid,
               void* stream) {
  const cudaStream_t st = S(stream);
  if (edges <= 0) {
    CK(cudaMemsetAsync(t_row_ptr, 0, 8 * (in_nodes + 1), st));
    return;
  }
  Buf src(4 * edges, st), iota(4 * edges, st), skeys(4 * edges, st);
  rowptr_expand(row_ptr, out_nodes, src.as<int>(), stream);
  k_iota<<<grid_for(edges, 256), 256, 0, st>>>(iota.as<int>(), edges);
  CK(cudaGetLastError());
  // LSD radix sort is stable: within a neighbour bucket edges keep their CSR
  // (ascending output node) order, as conv.cpp:135-151's counting fill.
  const int end_bit = bits_for(in_nodes);
  cub_call(st, [&](void* t, std::size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, nbr, skeys.as<int>(), iota.as<int>(), t_eid, edges, 0, end_bit, st);
  });
  k_rowptr<int><<<grid_for(in_nodes + 1, 256), 256, 0, st>>>(skeys.as<int>(), edges, in_nodes, 0,
                                                               reinterpret_cast<i64*>(t_row_ptr));
  CK(cudaGetLastError());
  k_take<<<grid_for(edges, 256), 256, 0, st>>>(src.as<int>(), t_eid, t_src, edges);
  CK(cudaGetLastError());
}

std::int64_t radius_graph(std::int64_t n, const double* pos, double r_cut, std::int64_t* row_ptr, std::int32_t* nbr,
                          std::int64_t cap, void* stream) {
  if (!(r_cut > 0.0)) throw std::invalid_argument("radius_graph: r_cut must be positive");
  if (n < 0) throw ShapeError("negative atom count");
  const cudaStream_t st = S(stream);
  if (n == 0) {
    if (row_ptr) CK(cudaMemsetAsync(row_ptr, 0, 8, st));
    CK(cudaStreamSynchronize(st));
    return 0;
  }
  if (n > INT_MAX) throw UnsupportedError("radius_graph: more than 2^31 atoms");
  const double r2 = r_cut * r_cut;
  Buf lo(3 * 8, st), key(8 * n, st), skey(8 * n, st), atom(4 * n, st), satom(4 * n, st), flag(4, st),
      cnt(8 * (n + 1), st), rp_own(row_ptr ? 0 : 8 * (n + 1), st);
  i64* rp = row_ptr ? reinterpret_cast<i64*>(row_ptr) : rp_own.as<i64>();
  k_min3<<<1, 1024, 0, st>>>(pos, n, lo.as<double>());
  CK(cudaMemsetAsync(flag.p, 0, 4, st));
  k_cells<<<grid_for(n, 256), 256, 0, st>>>(pos, n, lo.as<double>(), r_cut, key.as<u64>(), flag.as<int>());
  k_iota<<<grid_for(n, 256), 256, 0, st>>>(atom.as<int>(), n);
  CK(cudaGetLastError());
  cub_call(st, [&](void* t, std::size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, key.as<u64>(), skey.as<u64>(), atom.as<int>(), satom.as<int>(), n, 0,
                                           3 * kCellBits, st);
  });
  CK(cudaMemsetAsync(cnt.as<i64>() + n, 0, 8, st));
  k_pairs<<<grid_for(n, 128), 128, 0, st>>>(pos, n, lo.as<double>(), r_cut, r2, skey.as<u64>(), satom.as<int>(),
                                             cnt.as<i64>(), nullptr, nullptr);
  CK(cudaGetLastError());
  cub_call(st, [&](void* t, std::size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt.as<i64>(), rp, n + 1, st);
  });
  int overflow = 0;
  i64 total = 0;
  CK(cudaMemcpyAsync(&overflow, flag.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&total, rp + n, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (overflow) throw UnsupportedError("radius_graph: geometry spans more than 2^21 cells per axis");
  if (total > INT_MAX) throw UnsupportedError("radius_graph: more than 2^31 edges");
  if (!nbr) return total;
  if (cap < total) throw std::invalid_argument("radius_graph: nbr capacity " + std::to_string(cap) + " < " +
                                               std::to_string(total) + " edges");
  if (total > 0) {
    Buf pairs(8 * total, st), spairs(8 * total, st);
    k_pairs<<<grid_for(n, 128), 128, 0, st>>>(pos, n, lo.as<double>(), r_cut, r2, skey.as<u64>(), satom.as<int>(),
                                               nullptr, rp, pairs.as<u64>());
    CK(cudaGetLastError());
    // rows are already grouped by i; the sort orders each row's neighbours
    cub_call(st, [&](void* t, std::size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, pairs.as<u64>(), spairs.as<u64>(), total, 0, 32 + bits_for(n), st);
    });
    k_split<<<grid_for(total, 256), 256, 0, st>>>(spairs.as<u64>(), total, nbr, nullptr);
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(st));
  return total;
}

void* scratch_alloc(std::size_t bytes, void* stream) {
  void* p = nullptr;
  if (bytes) CK(cudaMallocAsync(&p, bytes, S(stream)));
  return p;
}

void scratch_free(void* p, void* stream) {
  if (p) cudaFreeAsync(p, S(stream));
}

}  // namespace cgf::gops
