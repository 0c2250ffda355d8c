// Multi-GPU fused convolution behind the C ABI (include/cgf.h, "multi-GPU"):
// the destination partition of paper_2501_13986_b200/dist.py for C / C++
// callers, with NCCL (resolved at run time from libnccl.so.2, the instance the
// caller's process already loaded when there is one) over NVLink for the one
// exchange per direction:
//   forward          all-gather of node_x into the padded [world x chunk] layout,
//                    then the local fused conv (cgf_conv_forward_shard);
//   backward         local by-neighbour conv -> partial g_node_x for every
//                    padded row; all-to-all (grouped ncclSend / ncclRecv) of
//                    the partials and a rank-ordered sum on the device, so
//                    the result is bitwise independent of NCCL's algorithm;
//   double-backward  all-gathers of node_x and dL/dg_node_x, local passes,
//                    the same ordered reduction of dL/dnode_x.
// cgf_dist_allreduce_ordered is the shared-W gradient all-reduce (C3
// replicas): all-gather of the ranks' gradients + a rank-ordered sum.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/cgf.h"
#include "graph_ops.hpp"
#include "problem.hpp"

struct cgf_conv_shard {
  int world = 1, rank = 0;
  std::int64_t out_nodes = 0, in_nodes = 0, chunk = 1, edges = 0, node0 = 0, edge0 = 0;
  // device CSR of the shard (rows = owned output nodes, nbr in the padded
  // neighbour space) and its transposed CSR
  void *row_ptr = nullptr, *nbr = nullptr, *t_row_ptr = nullptr, *t_src = nullptr, *t_eid = nullptr;
  // overlap (dist.DistConvPlan's scheme): [la, lb) = the longest run of output
  // rows whose neighbours are all this rank's nodes (they run during the
  // all-gather), [oa, ob) = this rank's own slot of the neighbour rows (they run
  // during the exchange); both 4-aligned. The collectives of an overlapped call
  // run on `comm_stream`, ordered against the caller's stream by the events.
  std::int64_t la = 0, lb = 0, oa = 0, ob = 0;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~cgf_conv_shard() {
    for (void* p : {row_ptr, nbr, t_row_ptr, t_src, t_eid})
      if (p) cudaFree(p);
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (comm_stream) cudaStreamDestroy(comm_stream);
  }
};

namespace {

struct Nccl {
  decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&::ncclCommInitRank) commInitRank = nullptr;
  decltype(&::ncclCommDestroy) commDestroy = nullptr;
  decltype(&::ncclAllGather) allGather = nullptr;
  decltype(&::ncclSend) send = nullptr;
  decltype(&::ncclRecv) recv = nullptr;
  decltype(&::ncclGroupStart) groupStart = nullptr;
  decltype(&::ncclGroupEnd) groupEnd = nullptr;
  decltype(&::ncclGetErrorString) errorString = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the caller's NCCL, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL not available (libnccl.so.2): ") + dlerror();
      return;
    }
#define CGF_NCCL(f, sym) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, sym)); if (!n.f) err = "libnccl lacks " sym;
    CGF_NCCL(getUniqueId, "ncclGetUniqueId")
    CGF_NCCL(commInitRank, "ncclCommInitRank")
    CGF_NCCL(commDestroy, "ncclCommDestroy")
    CGF_NCCL(allGather, "ncclAllGather")
    CGF_NCCL(send, "ncclSend")
    CGF_NCCL(recv, "ncclRecv")
    CGF_NCCL(groupStart, "ncclGroupStart")
    CGF_NCCL(groupEnd, "ncclGroupEnd")
    CGF_NCCL(errorString, "ncclGetErrorString")
#undef CGF_NCCL
  });
  if (!err.empty()) throw cgf::CudaError(err);
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw cgf::CudaError(std::string(what) + ": " + nccl().errorString(r));
}

void cuda_check(cudaError_t r, const char* what) {
  if (r != cudaSuccess) throw cgf::CudaError(std::string(what) + ": " + cudaGetErrorString(r));
}

// Forwards the error of a cgf_* call made from here (message kept).
struct Forwarded : std::runtime_error {
  int code;
  Forwarded(int c, const char* m) : std::runtime_error(m), code(c) {}
};
void rc_check(int rc) {
  if (rc != CGF_OK) throw Forwarded(rc, cgf_last_error());
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return CGF_OK;
  } catch (const Forwarded& e) {
    cgf::set_last_error(e.what());
    return e.code;
  } catch (const cgf::ShapeError& e) {
    cgf::set_last_error(e.what());
    return CGF_E_SHAPE;
  } catch (const cgf::CudaError& e) {
    cgf::set_last_error(e.what());
    return CGF_E_CUDA;
  } catch (const std::invalid_argument& e) {
    cgf::set_last_error(e.what());
    return CGF_E_INVALID;
  } catch (const std::exception& e) {
    cgf::set_last_error(e.what());
    return CGF_E_INTERNAL;
  }
}

// Output-node ranges of ~|E| / P edges each (dist.partition_bounds): boundary
// r is the first node whose row starts at or after round(r |E| / P)
// (round half to even, as numpy), clamped monotone.
std::vector<std::int64_t> partition_bounds(std::int64_t nodes, const std::int64_t* rp, int world) {
  std::vector<std::int64_t> b(world + 1);
  const std::int64_t E = rp[nodes];
  for (int r = 0; r <= world; ++r) {
    if (E == 0) {
      b[r] = nodes * r / world;
      continue;
    }
    const auto t = static_cast<std::int64_t>(std::nearbyint(static_cast<double>(r) * static_cast<double>(E) / world));
    b[r] = std::lower_bound(rp, rp + nodes + 1, t) - rp;
  }
  b[0] = 0;
  b[world] = nodes;
  for (int r = 0; r <= world; ++r) {
    b[r] = std::min(b[r], nodes);
    if (r) b[r] = std::max(b[r], b[r - 1]);
  }
  return b;
}

template <typename T>
void* upload(const std::vector<T>& v) {
  void* d = nullptr;
  cuda_check(cudaMalloc(&d, std::max<std::size_t>(1, v.size()) * sizeof(T)), "cudaMalloc");
  if (!v.empty()) cuda_check(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy");
  return d;
}

struct DevScratch {
  void* p = nullptr;
  void* st = nullptr;
  DevScratch(std::size_t bytes, void* stream) : st(stream) { p = cgf::gops::scratch_alloc(bytes, stream); }
  ~DevScratch() { cgf::gops::scratch_free(p, st); }
  char* c() const { return static_cast<char*>(p); }
};

ncclDataType_t nccl_type(int dtype) { return dtype == CGF_F64 ? ncclFloat64 : ncclFloat32; }

// [out_nodes x dim] local rows -> [world * chunk x dim] padded rows on every rank
void all_gather(const cgf_conv_shard* sh, int dtype, void* comm, const void* local, int dim, void* all,
                DevScratch& pad, void* stream) {
  const std::size_t es = dtype == CGF_F64 ? 8 : 4, row = es * dim;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cuda_check(cudaMemsetAsync(pad.p, 0, row * sh->chunk, st), "cudaMemsetAsync");
  if (sh->out_nodes)
    cuda_check(cudaMemcpyAsync(pad.p, local, row * sh->out_nodes, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
  nccl_check(nccl().allGather(pad.p, all, static_cast<std::size_t>(sh->chunk) * dim, nccl_type(dtype),
                              static_cast<ncclComm_t>(comm), st),
             "ncclAllGather");
}

// [world * chunk x dim] partial sums on every rank -> this rank's [out_nodes x
// dim] totals: all-to-all of the chunks, then the sum over ranks in rank order.
void ordered_reduce(const cgf_conv_shard* sh, int dtype, void* comm, const void* partial, int dim, void* out,
                    void* stream) {
  const std::size_t es = dtype == CGF_F64 ? 8 : 4, block = es * dim * static_cast<std::size_t>(sh->chunk);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevScratch parts(block * sh->world, stream);
  const auto& n = nccl();
  nccl_check(n.groupStart(), "ncclGroupStart");
  for (int r = 0; r < sh->world; ++r) {
    nccl_check(n.send(static_cast<const char*>(partial) + block * r, block / es, nccl_type(dtype),
                      r, static_cast<ncclComm_t>(comm), st), "ncclSend");
    nccl_check(n.recv(parts.c() + block * r, block / es, nccl_type(dtype), r, static_cast<ncclComm_t>(comm), st),
               "ncclRecv");
  }
  nccl_check(n.groupEnd(), "ncclGroupEnd");
  // parts viewed as [world][chunk * dim]: the first out_nodes * dim columns
  cgf::gops::column_sum(dtype == CGF_F64, parts.p, sh->world, static_cast<std::int64_t>(sh->out_nodes) * dim, out,
                        false, stream, static_cast<std::int64_t>(sh->chunk) * dim);
}

// Overlapped collectives: on by default for P > 1 in the deterministic mode;
// CGF_DIST_OVERLAP=0 turns them off, =force also overlaps on one rank (tests).
bool overlap_on(const cgf_conv_shard* sh, int mode) {
  const char* e = std::getenv("CGF_DIST_OVERLAP");
  if (mode != CGF_CONV_DETERMINISTIC || (e && std::strcmp(e, "0") == 0)) return false;
  return sh->world > 1 || (e && std::strcmp(e, "force") == 0);
}

std::int64_t ceil4(std::int64_t v) { return (v + 3) / 4 * 4; }
std::int64_t floor4(std::int64_t v) { return v / 4 * 4; }

}  // namespace

extern "C" {

int cgf_nccl_unique_id(char id[128]) {
  return guarded([&] {
    ncclUniqueId u;
    nccl_check(nccl().getUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, u.internal, 128);
  });
}

int cgf_nccl_comm_create(int world, int rank, const char id[128], void** comm) {
  return guarded([&] {
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    ncclComm_t c = nullptr;
    nccl_check(nccl().commInitRank(&c, world, u, rank), "ncclCommInitRank");
    *comm = c;
  });
}

int cgf_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (comm) nccl_check(nccl().commDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

int cgf_conv_shard_create(int64_t nodes, int64_t edges, const int64_t* row_ptr, const int32_t* nbr, int world,
                          int rank, cgf_conv_shard** out) {
  return guarded([&] {
    if (!out || !row_ptr || (edges > 0 && !nbr)) throw std::invalid_argument("null pointer");
    if (world < 1 || rank < 0 || rank >= world) throw cgf::ShapeError("rank outside world");
    if (nodes < 0 || edges < 0 || row_ptr[0] != 0 || row_ptr[nodes] != edges)
      throw std::invalid_argument("row_ptr does not span the edge list");
    const auto b = partition_bounds(nodes, row_ptr, world);
    auto sh = std::make_unique<cgf_conv_shard>();
    sh->world = world;
    sh->rank = rank;
    for (int r = 0; r < world; ++r) sh->chunk = std::max(sh->chunk, b[r + 1] - b[r]);
    sh->in_nodes = world * sh->chunk;
    const std::int64_t s0 = b[rank], s1 = b[rank + 1], e0 = row_ptr[s0], e1 = row_ptr[s1];
    sh->node0 = s0;
    sh->out_nodes = s1 - s0;
    sh->edge0 = e0;
    sh->edges = e1 - e0;
    std::vector<std::int64_t> rp(sh->out_nodes + 1);
    for (std::int64_t v = 0; v <= sh->out_nodes; ++v) rp[v] = row_ptr[s0 + v] - e0;
    std::vector<std::int32_t> nb(sh->edges);
    for (std::int64_t e = 0; e < sh->edges; ++e) {
      const std::int64_t g = nbr[e0 + e];
      if (g < 0 || g >= nodes) throw std::invalid_argument("neighbour index out of range");
      const int owner = static_cast<int>(std::upper_bound(b.begin(), b.end(), g) - b.begin()) - 1;
      nb[e] = static_cast<std::int32_t>(owner * sh->chunk + g - b[owner]);
    }
    std::vector<std::int64_t> trp(sh->in_nodes + 1);
    std::vector<std::int32_t> tsrc(std::max<std::int64_t>(sh->edges, 1)), teid(std::max<std::int64_t>(sh->edges, 1));
    rc_check(cgf_conv_transpose_shard_host(sh->out_nodes, sh->in_nodes, sh->edges, rp.data(), nb.data(), trp.data(),
                                           tsrc.data(), teid.data()));
    {  // overlap ranges (dist.GraphShard.local_rows / own_rows)
      const std::int64_t lo = static_cast<std::int64_t>(rank) * sh->chunk, hi = lo + sh->out_nodes;
      std::int64_t a = 0, ba = 0, bb = 0;
      for (std::int64_t v = 0; v <= sh->out_nodes; ++v) {
        bool inner = v < sh->out_nodes;
        for (std::int64_t e = inner ? rp[v] : 0; inner && e < rp[v + 1]; ++e) inner = nb[e] >= lo && nb[e] < hi;
        if (inner) continue;
        if (v - a > bb - ba) { ba = a; bb = v; }
        a = v + 1;
      }
      sh->la = ceil4(ba);
      sh->lb = floor4(bb);
      if (sh->la >= sh->lb) sh->la = sh->lb = 0;
      sh->oa = ceil4(lo);
      sh->ob = floor4(lo + sh->chunk);
      if (sh->oa >= sh->ob) sh->oa = sh->ob = 0;
      cuda_check(cudaStreamCreateWithFlags(&sh->comm_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      for (auto& e : sh->ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    }
    sh->row_ptr = upload(rp);
    sh->nbr = upload(nb);
    sh->t_row_ptr = upload(trp);
    sh->t_src = upload(tsrc);
    sh->t_eid = upload(teid);
    *out = sh.release();
  });
}

void cgf_conv_shard_destroy(cgf_conv_shard* sh) { delete sh; }

int cgf_conv_shard_info(const cgf_conv_shard* sh, int64_t info[6]) {
  return guarded([&] {
    if (!sh || !info) throw std::invalid_argument("null pointer");
    const int64_t v[6] = {sh->out_nodes, sh->in_nodes, sh->chunk, sh->edges, sh->node0, sh->edge0};
    std::memcpy(info, v, sizeof v);
  });
}

int cgf_dist_conv_forward(cgf_plan* plan, int dtype, const cgf_conv_shard* sh, void* comm, const void* node_x,
                          const void* edge_y, const void* edge_w, void* node_z, int mode, void* stream) {
  return guarded([&] {
    if (!plan || !sh || !comm) throw std::invalid_argument("null pointer");
    int64_t d[6];
    rc_check(cgf_plan_dims(plan, d));
    const int dx = static_cast<int>(d[0]), dz = static_cast<int>(d[2]);
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    const auto rp = static_cast<const int64_t*>(sh->row_ptr);
    const auto nb = static_cast<const int32_t*>(sh->nbr);
    // the collective must not depend on this rank's ranges (an empty range just
    // moves all rows after the all-gather)
    if (!overlap_on(sh, mode)) {
      DevScratch pad(es * dx * sh->chunk, stream), all(es * dx * sh->in_nodes, stream);
      all_gather(sh, dtype, comm, node_x, dx, all.p, pad, stream);
      rc_check(cgf_conv_forward_shard(plan, dtype, sh->out_nodes, sh->in_nodes, sh->edges, rp, nb, all.p, edge_y,
                                      edge_w, node_z, mode, stream));
      return;
    }
    // in-place all-gather on the comm stream while the local-neighbour rows run
    cudaStream_t st = static_cast<cudaStream_t>(stream), cs = sh->comm_stream;
    const std::size_t row = es * dx;
    DevScratch all(row * sh->in_nodes, stream);
    char* own = all.c() + row * sh->rank * sh->chunk;
    cuda_check(cudaMemsetAsync(own + row * sh->out_nodes, 0, row * (sh->chunk - sh->out_nodes), st), "cudaMemsetAsync");
    if (sh->out_nodes)
      cuda_check(cudaMemcpyAsync(own, node_x, row * sh->out_nodes, cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
    cuda_check(cudaEventRecord(sh->ev[0], st), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(cs, sh->ev[0], 0), "cudaStreamWaitEvent");
    nccl_check(nccl().allGather(own, all.p, static_cast<std::size_t>(sh->chunk) * dx, nccl_type(dtype),
                                static_cast<ncclComm_t>(comm), cs), "ncclAllGather");
    cuda_check(cudaEventRecord(sh->ev[1], cs), "cudaEventRecord");
    char* z = static_cast<char*>(node_z);
    auto rows = [&](std::int64_t r0, std::int64_t r1) {
      if (r0 < r1)
        rc_check(cgf_conv_forward_shard(plan, dtype, r1 - r0, sh->in_nodes, sh->edges, rp + r0, nb, all.p, edge_y,
                                        edge_w, z + es * dz * r0, mode, stream));
    };
    rows(sh->la, sh->lb);
    cuda_check(cudaStreamWaitEvent(st, sh->ev[1], 0), "cudaStreamWaitEvent");
    rows(0, sh->la);
    rows(sh->lb, sh->out_nodes);
  });
}

int cgf_dist_conv_backward(cgf_plan* plan, int dtype, const cgf_conv_shard* sh, void* comm, const void* node_x,
                           const void* edge_y, const void* edge_w, const void* g_node_z, void* g_node_x,
                           void* g_edge_y, void* g_edge_w, int mode, void* stream) {
  return guarded([&] {
    if (!plan || !sh || !comm) throw std::invalid_argument("null pointer");
    int64_t d[6];
    rc_check(cgf_plan_dims(plan, d));
    const int dx = static_cast<int>(d[0]);
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    DevScratch pad(es * dx * sh->chunk, stream), all(es * dx * sh->in_nodes, stream),
        part(es * dx * sh->in_nodes, stream);
    all_gather(sh, dtype, comm, node_x, dx, all.p, pad, stream);
    const auto trp = static_cast<const int64_t*>(sh->t_row_ptr);
    const auto tsrc = static_cast<const int32_t*>(sh->t_src);
    const auto teid = static_cast<const int32_t*>(sh->t_eid);
    if (!overlap_on(sh, mode)) {
      rc_check(cgf_conv_backward_shard(plan, dtype, sh->out_nodes, sh->in_nodes, sh->edges, trp, tsrc, teid, all.p,
                                       edge_y, edge_w, g_node_z, part.p, g_edge_y, g_edge_w, mode, stream));
      ordered_reduce(sh, dtype, comm, part.p, dx, g_node_x, stream);
      return;
    }
    // other ranks' neighbour rows first; their partials travel (comm stream)
    // while the own rows run; then the rank-ordered sum, as ordered_reduce
    cudaStream_t st = static_cast<cudaStream_t>(stream), cs = sh->comm_stream;
    const std::size_t row = es * dx, block = row * static_cast<std::size_t>(sh->chunk);
    auto rows = [&](std::int64_t r0, std::int64_t r1) {
      if (r0 < r1)
        rc_check(cgf_conv_backward_shard(plan, dtype, sh->out_nodes, r1 - r0, sh->edges, trp + r0, tsrc, teid,
                                         all.c() + row * r0, edge_y, edge_w, g_node_z, part.c() + row * r0, g_edge_y,
                                         g_edge_w, mode, stream));
    };
    rows(0, sh->oa);
    rows(sh->ob, sh->in_nodes);
    DevScratch parts(block * sh->world, stream);
    cuda_check(cudaEventRecord(sh->ev[0], st), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(cs, sh->ev[0], 0), "cudaStreamWaitEvent");
    const auto& n = nccl();
    nccl_check(n.groupStart(), "ncclGroupStart");
    for (int r = 0; r < sh->world; ++r) {
      if (r == sh->rank) continue;
      nccl_check(n.send(part.c() + block * r, block / es, nccl_type(dtype), r, static_cast<ncclComm_t>(comm), cs),
                 "ncclSend");
      nccl_check(n.recv(parts.c() + block * r, block / es, nccl_type(dtype), r, static_cast<ncclComm_t>(comm), cs),
                 "ncclRecv");
    }
    nccl_check(n.groupEnd(), "ncclGroupEnd");
    cuda_check(cudaEventRecord(sh->ev[1], cs), "cudaEventRecord");
    rows(sh->oa, sh->ob);
    cuda_check(cudaMemcpyAsync(parts.c() + block * sh->rank, part.c() + block * sh->rank, block,
                               cudaMemcpyDeviceToDevice, st), "cudaMemcpyAsync");
    cuda_check(cudaStreamWaitEvent(st, sh->ev[1], 0), "cudaStreamWaitEvent");
    cgf::gops::column_sum(dtype == CGF_F64, parts.p, sh->world, static_cast<std::int64_t>(sh->out_nodes) * dx,
                          g_node_x, false, stream, static_cast<std::int64_t>(sh->chunk) * dx);
  });
}

int cgf_dist_conv_double_backward(cgf_plan* plan, int dtype, const cgf_conv_shard* sh, void* comm,
                                  const void* node_x, const void* edge_y, const void* edge_w, const void* g_node_z,
                                  const void* d_gx, const void* d_gy, const void* d_gw, void* o_node_x,
                                  void* o_edge_y, void* o_edge_w, void* o_g_node_z, int mode, void* stream) {
  return guarded([&] {
    if (!plan || !sh || !comm) throw std::invalid_argument("null pointer");
    int64_t d[6];
    rc_check(cgf_plan_dims(plan, d));
    const int dx = static_cast<int>(d[0]);
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    DevScratch pad(es * dx * sh->chunk, stream), xall(es * dx * sh->in_nodes, stream),
        dall(es * dx * sh->in_nodes, stream), part(es * dx * sh->in_nodes, stream);
    all_gather(sh, dtype, comm, node_x, dx, xall.p, pad, stream);
    all_gather(sh, dtype, comm, d_gx, dx, dall.p, pad, stream);
    rc_check(cgf_conv_double_backward_shard(
        plan, dtype, sh->out_nodes, sh->in_nodes, sh->edges, static_cast<const int64_t*>(sh->row_ptr),
        static_cast<const int32_t*>(sh->nbr), static_cast<const int64_t*>(sh->t_row_ptr),
        static_cast<const int32_t*>(sh->t_src), static_cast<const int32_t*>(sh->t_eid), xall.p, edge_y, edge_w,
        g_node_z, dall.p, d_gy, d_gw, part.p, o_edge_y, o_edge_w, o_g_node_z, mode, stream));
    ordered_reduce(sh, dtype, comm, part.p, dx, o_node_x, stream);
  });
}

int cgf_dist_allreduce_ordered(int dtype, void* comm, int world, void* buf, int64_t count, void* stream) {
  return guarded([&] {
    if (!comm || (count > 0 && !buf)) throw std::invalid_argument("null pointer");
    if (world < 1 || count < 0) throw cgf::ShapeError("bad world / count");
    if (count == 0) return;
    const std::size_t es = dtype == CGF_F64 ? 8 : 4;
    DevScratch all(es * count * world, stream);
    nccl_check(nccl().allGather(buf, all.p, count, nccl_type(dtype), static_cast<ncclComm_t>(comm),
                                static_cast<cudaStream_t>(stream)),
               "ncclAllGather");
    cgf::gops::column_sum(dtype == CGF_F64, all.p, world, count, buf, false, stream, count);
  });
}

}  // extern "C"
