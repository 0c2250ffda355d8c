// Device-side graph utilities and the unfused convolution's data movement
// (SURVEY.md §8f rows 2-3). All functions take device pointers and enqueue on
// `stream` (a CUstream / cudaStream_t); the ones returning a count
// synchronise the stream to read it. Errors throw cgf::CudaError (CUDA
// failures) or std::invalid_argument (bad graphs, with the reference's
// messages).
#pragma once

#include <cstdint>

namespace cgf::gops {

// ---- unfused gather -> TP -> scatter (conv::unfused_forward / backward,
// conv.cpp:530-616) ---------------------------------------------------------

// dst[r, :] = src[idx[r], :] for r < n rows of `dim` words (T = f32 / f64).
void gather_rows(bool f64, const void* src, const std::int32_t* idx, void* dst, std::int64_t n, int dim, void* stream);

// out[v, :] = sum over q in [rp[v], rp[v+1]) of rows[idx ? idx[q] : q, :],
// summed sequentially in q order from zero (the reference's scatter order).
void segment_sum(bool f64, const void* rows, const std::int64_t* rp, const std::int32_t* idx, void* out,
                 std::int64_t nodes, int dim, void* stream);

// src[e] = v for e in [rp[v], rp[v+1]) (CSR -> per-edge output node).
void rowptr_expand(const std::int64_t* rp, std::int64_t nodes, std::int32_t* src, void* stream);

// dst[c] = (accumulate ? dst[c] : 0) + sum over r < rows of src[r * ld + c]
// (c < n; ld = 0 means n), in row order (deterministic).
void column_sum(bool f64, const void* src, std::int64_t rows, std::int64_t n, void* dst, bool accumulate,
                void* stream, std::int64_t ld = 0);

// Transposed CSR (t_row_ptr by neighbour, t_src, t_eid) -> the edge list in
// edge order: src[e], dst[e] (the atomic-mode shard backward's input).
void untranspose(const std::int64_t* t_row_ptr, std::int64_t in_nodes, const std::int32_t* t_src,
                 const std::int32_t* t_eid, std::int32_t* src, std::int32_t* dst, void* stream);

// ---- graph construction (conv.cpp:64-151) ---------------------------------

// make_graph (conv.cpp:64-87): validates (first offending edge in edge order
// decides the error, as in the reference), sorts by (src, dst), drops
// duplicates; row_ptr[nodes + 1], nbr[<= edges], out_src[<= edges] (may be
// null). Returns the deduplicated edge count.
std::int64_t make_graph(std::int64_t nodes, std::int64_t edges, const std::int32_t* src, const std::int32_t* dst,
                        bool allow_self_loops, std::int64_t* row_ptr, std::int32_t* nbr, std::int32_t* out_src,
                        void* stream);

// Transposed CSR (transpose_permutation, conv.cpp:135-151): a stable bucket of
// the edges by neighbour. t_row_ptr[in_nodes + 1], t_src[q] = output node,
// t_eid[q] = edge id (perm[t_eid[q]] == q).
void transpose(std::int64_t out_nodes, std::int64_t in_nodes, std::int64_t edges, const std::int64_t* row_ptr,
               const std::int32_t* nbr, std::int64_t* t_row_ptr, std::int32_t* t_src, std::int32_t* t_eid,
               void* stream);

// radius_graph (conv.cpp:89-133) over pos[n][3] (FP64): cells of side r_cut
// from the minimum corner, candidates from the 27 neighbouring cells, edge
// (i, j) for i != j with |r_i - r_j|^2 <= r_cut^2 (evaluated without FMA
// contraction, as the reference's -ffp-contract=off build). With nbr == null
// only counts. Writes row_ptr[n + 1] and nbr[E] (needs cap >= E). Returns E.
std::int64_t radius_graph(std::int64_t n, const double* pos, double r_cut, std::int64_t* row_ptr, std::int32_t* nbr,
                          std::int64_t cap, void* stream);

// Stream-ordered scratch.
void* scratch_alloc(std::size_t bytes, void* stream);
void scratch_free(void* p, void* stream);

}  // namespace cgf::gops
