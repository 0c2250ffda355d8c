/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the parity tests.
 *
 * A plain-C restatement of the reference's hot path (cgforge, /root/reference/proj):
 *   - rng::NormalGen                         (include/cgforge/rng.hpp:14-53)
 *   - cg::complex_cg / build_block           (src/cg.cpp:25-134)
 *   - kernelgen gen_forward/gen_backward + interpret, direct mode
 *                                            (src/kernelgen.cpp:135-251, 547-675)
 *   - engine::TpPlan forward/backward/double_backward (fused style)
 *                                            (src/engine.cpp:224-391)
 *   - conv::ConvPlan forward/backward (deterministic edge order) and the
 *     composed conv double-backward oracle
 *                                            (src/conv.cpp:234-528)
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the product never does.
 *
 * A problem is passed as its multiplicity-SPLIT subkernel list in schedule
 * order (stable sort by z offset, scheduler.cpp:146-151), CGO_SUB_FIELDS
 * int32 per subkernel:
 *   kind(0=B uvu, 1=C uvw), l1, l2, l3, b, b', x_off, y_off, z_off, w_off, w_row_stride
 * oracle/oracle.py builds it from the problem JSON (tpspec.cpp:8-130,
 * scheduler.cpp:32-81).
 */
#ifndef CGORACLE_H
#define CGORACLE_H
#include <stdint.h>

#define CGO_SUB_FIELDS 11

typedef struct {
  uint64_t mt[312];
  int idx;
  int have_spare;
  double spare;
} cgo_rng;

void cgo_rng_init(cgo_rng* g, uint64_t seed);
uint64_t cgo_rng_bits(cgo_rng* g);
double cgo_rng_normal(cgo_rng* g);
/* normal_vec<T>: n draws cast to T, continuing the stream of g. */
void cgo_rng_fill_f64(cgo_rng* g, double* out, int64_t n);
void cgo_rng_fill_f32(cgo_rng* g, float* out, int64_t n);
int cgo_rng_size(void);

double cgo_factorial(int n);
double cgo_complex_cg(int l1, int l2, int l3, int m1, int m2, int m3);
/* Real-basis block, entries sorted (k,i,j). Returns nnz (or -1 on error). */
int cgo_cg_block(int l1, int l2, int l3, int cap, int* i, int* j, int* k, double* v);

typedef struct {
  const int32_t* subs;
  int32_t n;
  int32_t dim_x, dim_y, dim_z, n_w;
} cgo_problem;

#define CGO_DECL(SUF, T)                                                                        \
  int cgo_tp_forward_##SUF(const cgo_problem* p, const T* x, const T* y, const T* w, T* z,     \
                           int64_t rows, int w_shared);                                         \
  int cgo_tp_backward_##SUF(const cgo_problem* p, const T* x, const T* y, const T* w,          \
                            const T* gz, T* gx, T* gy, T* gw, int64_t rows, int w_shared);      \
  int cgo_tp_double_backward_##SUF(const cgo_problem* p, const T* x, const T* y, const T* w,   \
                                   const T* gz, const T* da, const T* db, const T* dc, T* ox,   \
                                   T* oy, T* ow, T* ogz, int64_t rows, int w_shared);           \
  int cgo_conv_forward_##SUF(const cgo_problem* p, int64_t nodes, int64_t ne,                  \
                             const int64_t* row_ptr, const int32_t* nbr, const T* node_x,       \
                             const T* edge_y, const T* edge_w, T* node_z, int w_shared);        \
  int cgo_conv_backward_##SUF(const cgo_problem* p, int64_t nodes, int64_t ne,                 \
                              const int32_t* src, const int32_t* nbr, const T* node_x,          \
                              const T* edge_y, const T* edge_w, const T* g_node_z, T* g_node_x, \
                              T* g_edge_y, T* g_edge_w, int w_shared);                          \
  int cgo_conv_double_backward_##SUF(                                                           \
      const cgo_problem* p, int64_t nodes, int64_t ne, const int32_t* src, const int32_t* nbr,  \
      const T* node_x, const T* edge_y, const T* edge_w, const T* g_node_z, const T* d_gx,      \
      const T* d_gy, const T* d_gw, T* o_node_x, T* o_edge_y, T* o_edge_w, T* o_g_node_z,       \
      int w_shared);

CGO_DECL(f32, float)
CGO_DECL(f64, double)

#endif
