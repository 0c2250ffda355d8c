/*
 * cgf.h — C ABI of the B200-native CG tensor-product kernels (libcgf.so).
 *
 * This is the drop-in boundary for the reference's C++ operator API
 * (/root/reference/proj/include/cgforge/ headers). The reference has no C ABI, no
 * plugin registry and no FFI: its callers construct engine::TpPlan /
 * conv::ConvPlan objects directly. Each entry point below replaces one of
 * those calls (file:line cited per function); INTEGRATION.md shows the ctypes
 * binding and the header-compatible C++ shim a maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only. Array pointers passed to cgf_tp_* and
 *    cgf_conv_* are DEVICE pointers (CUDA global memory, any allocator); the
 *    *_host variants take host pointers and do the copies themselves.
 *  - Layouts are the reference's: row-major [rows x dim], irreps segments
 *    [mult][2l+1] mult-major, weights concatenated per instruction with kind C
 *    stored W[w][u] (tpspec.hpp:16-20).
 *  - Outputs are fully overwritten (the reference zero-fills then accumulates,
 *    engine.cpp:270-274).
 *  - `stream` is a CUstream / cudaStream_t (0 = legacy default stream).
 *  - Every function returns CGF_OK or an error code; the message of the last
 *    error on the calling thread is cgf_last_error(). Codes map 1:1 onto the
 *    reference's exception types.
 *  - No CPU fallback: without a usable CUDA device the compute calls return
 *    CGF_E_CUDA.
 */
#ifndef CGF_H
#define CGF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum cgf_status {
  CGF_OK = 0,
  CGF_E_PARSE = 1,       /* irreps::ParseError, malformed problem JSON (irreps.hpp:58, tpspec.hpp:88-91) */
  CGF_E_VALIDATION = 2,  /* tpspec::validate violations (tpspec.hpp:70-84) */
  CGF_E_SHAPE = 3,       /* engine::ShapeError (engine.hpp:62-64) */
  CGF_E_BUDGET = 4,      /* scheduler::BudgetError (scheduler.hpp:74-76) */
  CGF_E_TRIANGLE = 5,    /* cg::TriangleError (cg.hpp:40-42) */
  CGF_E_INVALID = 6,     /* std::invalid_argument, e.g. unsorted edges (conv.cpp:196-205) */
  CGF_E_CUDA = 7,        /* CUDA driver error / no device */
  CGF_E_JIT = 8,         /* NVRTC compilation of a generated kernel failed */
  CGF_E_UNSUPPORTED = 9, /* configuration outside this build's coverage */
  CGF_E_INTERNAL = 10    /* std::logic_error (engine.cpp:48, 126) */
};

enum cgf_dtype { CGF_F32 = 0, CGF_F64 = 1 };
enum cgf_op { CGF_OP_FORWARD = 0, CGF_OP_BACKWARD = 1, CGF_OP_DOUBLE_BACKWARD = 2 };

typedef struct cgf_plan cgf_plan;

/* Thread-local message of the last failing call on this thread. */
const char* cgf_last_error(void);
/* Library version string ("cgf <semver> nvrtc <maj.min> sm_100a"). */
const char* cgf_version(void);

/* ---- descriptors -------------------------------------------------------- */

/* Real-basis CG block <l1 l2 l3>, entries sorted (k,i,j), per-k orthonormal.
 * Replaces cg::cg_block (cg.hpp:55, cg.cpp:138-160). Returns the entry count
 * (arrays filled up to cap) or -(error code). */
int cgf_cg_block(int l1, int l2, int l3, int cap, int* i, int* j, int* k, double* v);

/* Parse + validate + split + plan. Replaces tpspec::parse_problem_json
 * (tpspec.hpp:88-91) -> scheduler::split_multiplicities (scheduler.hpp:82-84)
 * -> scheduler::build_schedule (scheduler.hpp:86-89) -> engine::TpPlan ctor
 * (engine.hpp:73). lane_width: multiplicity split width (<= 0: 32).
 * budget_words: the reference's per-worker scratch budget; kept for API
 * parity — a budget below the largest subkernel working set is rejected with
 * CGF_E_BUDGET exactly as build_schedule does (scheduler.cpp:161-170); 0 means
 * the reference default 4096. Kernels are generated and compiled lazily. */
int cgf_plan_create(const char* problem_json, int lane_width, uint32_t budget_words, cgf_plan** out);
void cgf_plan_destroy(cgf_plan* plan);

/* dims = {dim_x, dim_y, dim_z, total_weights, split_subkernels, units}. */
int cgf_plan_dims(const cgf_plan* plan, int64_t dims[6]);
/* Reference flop rule per row (kernelgen::flop_count, kernelgen.cpp:253-276):
 * flops = {forward, backward, double_backward(= 3 fwd + 4 bwd)}. */
int cgf_plan_flops(const cgf_plan* plan, uint64_t flops[3]);
/* Generated CUDA source for (op, dtype, w_shared, aligned); returns its length
 * (copies up to cap-1 bytes + NUL). Debug / inspection only. */
int cgf_plan_source(cgf_plan* plan, int op, int dtype, int w_shared, int aligned, char* buf, int cap);
/* Generate + NVRTC-compile (sm_100a) ahead of time; no device needed. */
int cgf_plan_compile(cgf_plan* plan, int op, int dtype, int w_shared, int aligned);

/* ---- batched tensor product (device pointers) --------------------------- */

/* z[rows x dim_z] = TP(x, y, W). Replaces TpPlan::forward (engine.hpp:82-83,
 * engine.cpp:278-283). w_shared != 0: w is ONE row used for every batch row
 * (a superset of the reference API, which stores W per row). */
int cgf_tp_forward(cgf_plan* plan, int dtype, const void* x, const void* y, const void* w, void* z,
                   int64_t rows, int w_shared, void* stream);

/* (gx, gy, gw) = backward(x, y, W, gz). Replaces TpPlan::backward
 * (engine.hpp:85-87, engine.cpp:285-295). */
int cgf_tp_backward(cgf_plan* plan, int dtype, const void* x, const void* y, const void* w,
                    const void* gz, void* gx, void* gy, void* gw, int64_t rows, int w_shared,
                    void* stream);

/* Given (da, db, dC) = upstream gradients of (gx, gy, gw), returns
 * (dL/dx, dL/dy, dL/dW, dL/dgz) in one fused pass. Replaces
 * TpPlan::double_backward (engine.hpp:89-95, engine.cpp:297-392). */
int cgf_tp_double_backward(cgf_plan* plan, int dtype, const void* x, const void* y, const void* w,
                           const void* gz, const void* da, const void* db, const void* dc,
                           void* ox, void* oy, void* ow, void* ogz, int64_t rows, int w_shared,
                           void* stream);

/* Host-pointer variants: allocate device buffers, copy in, run, copy out,
 * synchronise. The semantics of the reference's std::vector API
 * (TpPlan::forward/backward/double_backward on host Batch<T>). */
int cgf_tp_forward_host(cgf_plan* plan, int dtype, const void* x, const void* y, const void* w,
                        void* z, int64_t rows, int w_shared);
int cgf_tp_backward_host(cgf_plan* plan, int dtype, const void* x, const void* y, const void* w,
                         const void* gz, void* gx, void* gy, void* gw, int64_t rows, int w_shared);
/* Forward and backward of the same rows in ONE pipelined host pass (a
 * training step's TP: z = TP(x, y, W) and (gx, gy, gw) from a given gz, as
 * TpPlan::forward followed by TpPlan::backward, engine.hpp:82-88): x, y and W
 * cross PCIe once, and host->device / device->host copies of different row
 * chunks overlap. Same results as the two calls. */
int cgf_tp_forward_backward_host(cgf_plan* plan, int dtype, const void* x, const void* y, const void* w,
                                 const void* gz, void* z, void* gx, void* gy, void* gw, int64_t rows,
                                 int w_shared);
int cgf_tp_double_backward_host(cgf_plan* plan, int dtype, const void* x, const void* y,
                                const void* w, const void* gz, const void* da, const void* db,
                                const void* dc, void* ox, void* oy, void* ow, void* ogz,
                                int64_t rows, int w_shared);

/* The counters the reference's TpPlan returns (engine::ExecStats,
 * engine.hpp:19-30) for `rows` rows of `op`: {loads_words, stores_words,
 * flops} of the reference's per-row schedule model (the plan's budget),
 * computed here (scheduler.cpp:139-404, engine.cpp:115-168):
 *   forward          = traffic_report x rows (test_engine.cpp:350-363);
 *   backward         = phases' loaded x/y/w + staged g_z words, no stores,
 *                      backward flops, x rows (engine_impl.hpp:143-181);
 *   double_backward  = 3 forward + 4 backward rows (engine.cpp:350-391).
 * w_shared is accepted for symmetry and does not change the model. */
int cgf_tp_stats(const cgf_plan* plan, int op, int64_t rows, int w_shared, uint64_t stats[3]);
/* The GPU kernels' compulsory traffic of one call in words: {loads, stores},
 * each input read once and each output written once (the
 * roofline's algorithmic bytes = words x sizeof(T)). */
int cgf_tp_traffic(const cgf_plan* plan, int op, int64_t rows, int w_shared, uint64_t words[2]);
/* scheduler::schedule_to_json (scheduler.cpp:406-445) of the plan's schedule
 * model: same document, byte for byte. Returns the length (copies up to cap-1
 * bytes + NUL). */
int cgf_plan_schedule_json(const cgf_plan* plan, char* buf, int cap);
/* kernelgen::emit_text(gen_forward / gen_backward) of split subkernel `pos`
 * in schedule order (kernelgen.cpp:305-360): the op stream whose CG
 * coefficients the generated kernels carry as immediates. Returns the length. */
int cgf_plan_listing(const cgf_plan* plan, int pos, int backward, char* buf, int cap);

/* ConvStats (conv.hpp:78-91) of one conv call under the GPU kernels' store /
 * load model: op CGF_OP_FORWARD / CGF_OP_BACKWARD, mode CGF_CONV_* (fused),
 * or unfused != 0 for the gather -> TP -> scatter comparator. stats =
 * {loads_words, stores_words, output_store_ops, flops}. The fused
 * deterministic conv writes each output row once (output_store_ops = nodes);
 * atomic mode reduces once per edge; the unfused path stores one row per edge. */
int cgf_conv_stats(const cgf_plan* plan, int op, int mode, int unfused, int64_t nodes, int64_t edges,
                   uint64_t stats[4]);

/* ---- kernel introspection ------------------------------------------------ */

/* comp: 0 fwd, 1 bwd, 2 fused double-backward, 3 conv dbwd pass 1 (dgz),
 * 4 conv dbwd pass 2 (dx, dy, dW). loop: 0 batched rows, 1 conv by output
 * node, 2 conv by neighbour node (transposed CSR). */
int cgf_plan_kernel_source(cgf_plan* plan, int comp, int loop, int dtype, int w_shared, int aligned, char* buf,
                           int cap);
int cgf_plan_kernel_compile(cgf_plan* plan, int comp, int loop, int dtype, int w_shared, int aligned);
/* Kernels per call of (comp, loop): the by-neighbour conv and the batched
 * double-backward run their units in groups, one kernel each,
 * and one group's source. */
int cgf_plan_kernel_groups(const cgf_plan* plan, int comp, int loop, int dtype);
int cgf_plan_kernel_source_group(cgf_plan* plan, int comp, int loop, int dtype, int w_shared, int aligned,
                                 int group, char* buf, int cap);

/* ---- fused tensor product + graph convolution (device pointers) ---------- */

/* Edge convention of the reference (conv.hpp:15-18): edge e = (s, d)
 * contributes node_z[s] += TP(node_x[d], edge_y[e], edge_w[e]). The graph is
 * the reference's GraphCSR (conv.hpp:44-50): edges sorted strictly by (s, d),
 * row_ptr[nodes + 1] (int64) by output node s, nbr[e] = d (int32).
 * Deterministic: every output row is owned by one warp and summed in edge
 * order; no atomics. */
enum cgf_conv_mode { CGF_CONV_DETERMINISTIC = 0, CGF_CONV_ATOMIC = 1 };

/* Transposed CSR for the backward traversal (conv::transpose_permutation,
 * conv.cpp:135-151, on host arrays): t_row_ptr[nodes + 1] by neighbour d,
 * t_src[q] = output node s of transposed position q, t_eid[q] = its edge id
 * (so perm[t_eid[q]] == q). */
int cgf_conv_transpose_host(int64_t nodes, int64_t edges, const int64_t* row_ptr, const int32_t* nbr,
                            int64_t* t_row_ptr, int32_t* t_src, int32_t* t_eid);

/* node_z = sum over edges (ConvPlan::forward, conv.hpp:99-102, conv.cpp:234-355). */
int cgf_conv_forward(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                     const int32_t* nbr, const void* node_x, const void* edge_y, const void* edge_w,
                     void* node_z, int mode, void* stream);

/* (g_node_x, g_edge_y, g_edge_w) from g_node_z (ConvPlan::backward,
 * conv.hpp:106-111, conv.cpp:357-528): g_node_x accumulated per neighbour
 * over the transposed CSR, per-edge gradients written directly. */
int cgf_conv_backward(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                      const int32_t* nbr, const int64_t* t_row_ptr, const int32_t* t_src, const int32_t* t_eid,
                      const void* node_x, const void* edge_y, const void* edge_w, const void* g_node_z,
                      void* g_node_x, void* g_edge_y, void* g_edge_w, int mode, void* stream);

/* Conv double-backward (no reference entry point; composed per SURVEY.md §8c):
 * given (d_gx, d_gy, d_gw) = upstream gradients of the backward outputs,
 * returns (dL/dnode_x, dL/dedge_y, dL/dedge_w, dL/dg_node_z). Two passes:
 * by output node (dg_node_z) and by neighbour node (the rest). */
int cgf_conv_double_backward(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                             const int32_t* nbr, const int64_t* t_row_ptr, const int32_t* t_src,
                             const int32_t* t_eid, const void* node_x, const void* edge_y, const void* edge_w,
                             const void* g_node_z, const void* d_gx, const void* d_gy, const void* d_gw,
                             void* o_node_x, void* o_edge_y, void* o_edge_w, void* o_g_node_z, int mode,
                             void* stream);

/* ---- atomic-mode convolution (ConvPlan Mode::atomic, conv.hpp:70,
 * conv.cpp:311-324 and 470-486) -------------------------------------------
 * The graph is an edge list in ANY order: edge e = (src[e], dst[e]), int32.
 * No sorting, CSR or transposed permutation. One warp item per (edge, unit);
 * node_z[src] and g_node_x[dst] accumulate with float atomics (16-byte vector
 * reductions in FP32), so results vary in the last bits between runs; per-edge
 * gradients are written directly. The double-backward runs in one pass.
 * The CSR entry points above also accept mode = CGF_CONV_ATOMIC: they expand
 * row_ptr to per-edge sources on the device and call these. */
int cgf_conv_forward_atomic(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                            const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                            void* node_z, void* stream);
int cgf_conv_backward_atomic(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                             const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                             const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w, void* stream);
int cgf_conv_double_backward_atomic(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                    const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                    const void* g_node_z, const void* d_gx, const void* d_gy, const void* d_gw,
                                    void* o_node_x, void* o_edge_y, void* o_edge_w, void* o_g_node_z, void* stream);

/* Host-pointer variants (copies in and out, default stream, synchronous). The
 * transposed CSR for the backward is built internally. With mode =
 * CGF_CONV_ATOMIC the CSR variants run the atomic kernels. */
int cgf_conv_forward_host(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                          const int32_t* nbr, const void* node_x, const void* edge_y, const void* edge_w,
                          void* node_z, int mode);
int cgf_conv_backward_host(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                           const int32_t* nbr, const void* node_x, const void* edge_y, const void* edge_w,
                           const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w, int mode);
/* Host-pointer atomic mode over an edge list in any order (the shim's
 * ConvPlan Mode::atomic path: no sortedness requirement, conv.cpp:240). */
int cgf_conv_forward_atomic_host(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                 const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                 void* node_z);
int cgf_conv_backward_atomic_host(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                  const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                  const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w);

/* ---- unfused comparator (conv::unfused_forward / unfused_backward,
 * conv.cpp:530-616) on the GPU -----------------------------------------------
 * Gathers node rows per edge (|E| x dim_x, and |E| x dim_z of g_node_z for the
 * backward), runs the batched TP kernels over |E| rows, and sums the per-edge
 * rows into the nodes in edge order (deterministic segmented sums over the
 * CSR / transposed CSR). Device workspace of |E| (dim_x + dim_z) words
 * (backward: |E| (2 dim_x + dim_z) + |E| int32); it exists to quantify what
 * the fused kernels save. */
int cgf_conv_unfused_forward(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                             const int32_t* nbr, const void* node_x, const void* edge_y, const void* edge_w,
                             void* node_z, void* workspace, size_t workspace_bytes, void* stream);
int cgf_conv_unfused_backward(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int64_t* row_ptr,
                              const int32_t* nbr, const int64_t* t_row_ptr, const int32_t* t_eid, const void* node_x,
                              const void* edge_y, const void* edge_w, const void* g_node_z, void* g_node_x,
                              void* g_edge_y, void* g_edge_w, void* workspace, size_t workspace_bytes,
                              void* stream);
/* Device workspace the unfused calls need (op 0 forward, 1 backward). With
 * workspace == NULL they allocate it stream-ordered per call instead. */
size_t cgf_conv_unfused_workspace(const cgf_plan* plan, int dtype, int op, int64_t edges);
/* Host-pointer variants over an edge list in any order (the reference's
 * unfused_forward / unfused_backward take any GraphCSR edge order). */
int cgf_conv_unfused_forward_host(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                  const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                  void* node_z);
int cgf_conv_unfused_backward_host(cgf_plan* plan, int dtype, int64_t nodes, int64_t edges, const int32_t* src,
                                   const int32_t* dst, const void* node_x, const void* edge_y, const void* edge_w,
                                   const void* g_node_z, void* g_node_x, void* g_edge_y, void* g_edge_w);

/* ---- graph construction on the device (conv.cpp:64-151) ------------------
 * Device pointers; the calls returning a count synchronise `stream`.
 * cgf_graph_make = conv::make_graph (conv.cpp:64-87): validates (the first
 * offending edge decides: "make_graph: edge endpoint out of range" /
 * "make_graph: self-loop (s)", CGF_E_INVALID), sorts by (src, dst), removes
 * duplicates. row_ptr[nodes + 1]; nbr / out_src (nullable) need room for
 * `edges` entries; *out_edges = the deduplicated count.
 * cgf_graph_transpose = transpose_permutation (conv.cpp:135-151) as a
 * transposed CSR (see cgf_conv_transpose_shard_host).
 * cgf_graph_radius = conv::radius_graph (conv.cpp:89-133) over pos[n][3]
 * (FP64): *out_edges = |E|; with nbr == NULL it only counts, else nbr needs
 * cap >= |E| entries and row_ptr[n + 1] is written. */
int cgf_graph_make(int64_t nodes, int64_t edges, const int32_t* src, const int32_t* dst, int allow_self_loops,
                   int64_t* row_ptr, int32_t* nbr, int32_t* out_src, int64_t* out_edges, void* stream);
int cgf_graph_transpose(int64_t out_nodes, int64_t in_nodes, int64_t edges, const int64_t* row_ptr,
                        const int32_t* nbr, int64_t* t_row_ptr, int32_t* t_src, int32_t* t_eid, void* stream);
int cgf_graph_radius(int64_t n, const double* pos, double r_cut, int64_t* row_ptr, int32_t* nbr, int64_t cap,
                     int64_t* out_edges, void* stream);

/* ---- sharded convolution (multi-GPU, destination-partitioned) ------------
 * One rank owns a contiguous range of out_nodes output nodes and their edges
 * (SURVEY.md §8e). Node-indexed inputs read through nbr (node_x, d_gx) and the
 * x-type outputs (g_node_x, o_node_x) span in_nodes rows — the all-gathered
 * neighbour space; output-node arrays (node_z, g_node_z, o_g_node_z) span
 * out_nodes rows; edge arrays span the shard's edges. row_ptr[out_nodes + 1]
 * is rebased to the shard; t_row_ptr[in_nodes + 1] / t_src / t_eid are the
 * shard's transposed CSR (t_src local to the shard). The x-type outputs are
 * the shard's PARTIAL sums; the caller reduce-scatters them across ranks.
 * With out_nodes == in_nodes and a whole graph these are the calls above. */
int cgf_conv_transpose_shard_host(int64_t out_nodes, int64_t in_nodes, int64_t edges, const int64_t* row_ptr,
                                  const int32_t* nbr, int64_t* t_row_ptr, int32_t* t_src, int32_t* t_eid);
int cgf_conv_forward_shard(cgf_plan* plan, int dtype, int64_t out_nodes, int64_t in_nodes, int64_t edges,
                           const int64_t* row_ptr, const int32_t* nbr, const void* node_x, const void* edge_y,
                           const void* edge_w, void* node_z, int mode, void* stream);
int cgf_conv_backward_shard(cgf_plan* plan, int dtype, int64_t out_nodes, int64_t in_nodes, int64_t edges,
                            const int64_t* t_row_ptr, const int32_t* t_src, const int32_t* t_eid,
                            const void* node_x, const void* edge_y, const void* edge_w, const void* g_node_z,
                            void* g_node_x, void* g_edge_y, void* g_edge_w, int mode, void* stream);
int cgf_conv_double_backward_shard(cgf_plan* plan, int dtype, int64_t out_nodes, int64_t in_nodes, int64_t edges,
                                   const int64_t* row_ptr, const int32_t* nbr, const int64_t* t_row_ptr,
                                   const int32_t* t_src, const int32_t* t_eid, const void* node_x,
                                   const void* edge_y, const void* edge_w, const void* g_node_z, const void* d_gx,
                                   const void* d_gy, const void* d_gw, void* o_node_x, void* o_edge_y,
                                   void* o_edge_w, void* o_g_node_z, int mode, void* stream);

/* ---- array files (array_io.cpp:15-68) --------------------------------------
 * The reference CLI's array format: <base>.bin raw little-endian values and a
 * <base>.json sidecar {"cols":C,"dtype":"fp32"|"fp64","rows":R}. Files written
 * here are byte-identical to the reference's save_array. cgf_array_load reads
 * into a host buffer (device = 0) or, through pinned staging, into device
 * memory on `stream` (device != 0); `capacity` is in elements. */
int cgf_array_save(const char* base, int dtype, const void* host_data, int64_t rows, int64_t cols);
int cgf_array_meta(const char* base, int64_t shape[2], int* dtype);
int cgf_array_load(const char* base, int dtype, void* dst, int64_t capacity, int device, void* stream);

/* ---- multi-GPU fused convolution (destination-partitioned, NCCL) ----------
 * One process (or thread) per GPU, one rank each. The reference runs the conv
 * on one host only (conv.cpp:234-528); SURVEY.md §8e's partition: rank r owns
 * a contiguous range of output nodes (~|E|/P edges) with their node rows and
 * their edges' y / W. Per call one exchange: the forward all-gathers node_x
 * (padded [world x chunk] layout), the backward reduces the partial g_node_x
 * with an all-to-all (ncclSend / ncclRecv) and a rank-ordered sum on the device
 * (bitwise independent of NCCL's algorithm), the double-backward does both.
 * NCCL is resolved at run time from libnccl.so.2 (the caller's instance when
 * already loaded); `nccl_comm` is an ncclComm_t of `world` ranks. */
typedef struct cgf_conv_shard cgf_conv_shard;
/* NCCL bootstrap for callers without NCCL headers: a 128-byte unique id on
 * one rank, shared out of band, then one communicator per rank. */
int cgf_nccl_unique_id(char id[128]);
int cgf_nccl_comm_create(int world, int rank, const char id[128], void** nccl_comm);
int cgf_nccl_comm_destroy(void* nccl_comm);
/* Rank `rank`'s shard of a host GraphCSR (row_ptr int64 [nodes + 1], nbr
 * int32, sorted by (src, dst)): device CSR + transposed CSR in the padded
 * neighbour space. info = {out_nodes, in_nodes, chunk, edges, node0, edge0}:
 * the rank passes node rows [node0, node0 + out_nodes) and edges
 * [edge0, edge0 + edges) of the global arrays. */
int cgf_conv_shard_create(int64_t nodes, int64_t edges, const int64_t* row_ptr, const int32_t* nbr, int world,
                          int rank, cgf_conv_shard** shard);
int cgf_conv_shard_info(const cgf_conv_shard* shard, int64_t info[6]);
void cgf_conv_shard_destroy(cgf_conv_shard* shard);
/* ConvPlan::forward / backward (conv.hpp:99-111) and the double-backward over
 * the partition; device pointers to the rank's rows, mode CGF_CONV_*. With
 * P > 1 in the deterministic mode the forward's all-gather runs on the shard's
 * own stream while the rows whose neighbours are all local compute, and the
 * backward's exchange runs while the rank's own neighbour rows compute (events
 * order both against `stream`); results are bit-identical to the unoverlapped
 * path, which CGF_DIST_OVERLAP=0 selects. */
int cgf_dist_conv_forward(cgf_plan* plan, int dtype, const cgf_conv_shard* shard, void* nccl_comm,
                          const void* node_x, const void* edge_y, const void* edge_w, void* node_z, int mode,
                          void* stream);
int cgf_dist_conv_backward(cgf_plan* plan, int dtype, const cgf_conv_shard* shard, void* nccl_comm,
                           const void* node_x, const void* edge_y, const void* edge_w, const void* g_node_z,
                           void* g_node_x, void* g_edge_y, void* g_edge_w, int mode, void* stream);
int cgf_dist_conv_double_backward(cgf_plan* plan, int dtype, const cgf_conv_shard* shard, void* nccl_comm,
                                  const void* node_x, const void* edge_y, const void* edge_w, const void* g_node_z,
                                  const void* d_gx, const void* d_gy, const void* d_gw, void* o_node_x,
                                  void* o_edge_y, void* o_edge_w, void* o_g_node_z, int mode, void* stream);
/* Deterministic all-reduce (sum) of `count` words in place: all-gather + a
 * rank-ordered sum (the shared-W gradient of data-parallel replicas). */
int cgf_dist_allreduce_ordered(int dtype, void* nccl_comm, int world, void* buf, int64_t count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CGF_H */
