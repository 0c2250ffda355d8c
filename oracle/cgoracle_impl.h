/* TEST INFRASTRUCTURE ONLY — included twice by cgoracle.c with T = float /
 * double and SUF = f32 / f64. Per-row semantics are the reference IR
 * interpreter's in direct (single-phase) mode: the op order of gen_forward /
 * gen_backward (kernelgen.cpp:135-251) evaluated as interpret<T> does
 * (kernelgen.cpp:547-675), one lane at a time (lanes never interact except in
 * reduce_lanes and the W matmuls, which are restated explicitly). */
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define FN(name) CAT(name, SUF)


/* z += TP(x, y, w) for one row; z accumulates (engine zeroes it first,
 * engine.cpp:232). One pass over subkernels in schedule order. */
static void FN(fwd_row)(const cgo_problem* p, const T* x, const T* y, const T* w, T* z) {
  for (int s = 0; s < p->n; ++s) {
    const int32_t* d = SUB(p, s);
    const cg_entries* cg = cg_get(d[F_L1], d[F_L2], d[F_L3]);
    const int dx = 2 * d[F_L1] + 1, dz = 2 * d[F_L3] + 1;
    const int b = d[F_B], bp = d[F_BP];
    const int lanes = b > bp ? b : bp;
    /* z' per lane (kSlotZ), zeroed as an accum group (kernelgen.cpp:327). */
    T zp[64][MAXW];
    T outv[64][MAXW];
    for (int t = 0; t < lanes; ++t)
      for (int k = 0; k < dz; ++k) zp[t][k] = outv[t][k] = (T)0;
    /* fma z'[k] += (T(v) * x[i]) * y[j] over bp lanes (kernelgen.cpp:340-342, 585-592). */
    for (int t = 0; t < bp; ++t) {
      const T* xt = x + d[F_XO] + t * dx;
      const T* yy = y + d[F_YO];
      for (int e = 0; e < cg->n; ++e) {
        const T v = (T)cg->v[e];
        zp[t][cg->k[e]] += v * xt[cg->i[e]] * yy[cg->j[e]];
      }
    }
    if (d[F_KIND] == 0) {
      /* scale out[k] += w * z'[k] over b lanes (kernelgen.cpp:344-347). */
      for (int t = 0; t < b; ++t) {
        const T wt = w[d[F_WO] + t];
        for (int k = 0; k < dz; ++k) outv[t][k] += wt * zp[t][k];
      }
    } else {
      /* apply_w: out[r][s] = sum_c W[r,c] z'[c][s], c order (kernelgen.cpp:609-623). */
      for (int r = 0; r < b; ++r)
        for (int q = 0; q < dz; ++q) {
          T acc = outv[r][q];
          for (int c = 0; c < bp; ++c) acc += w[d[F_WO] + r * d[F_WS] + c] * zp[c][q];
          outv[r][q] = acc;
        }
    }
    /* acc Z[z_off + t*dz + k] += out[k] over b lanes (kernelgen.cpp:353-354). */
    for (int t = 0; t < b; ++t)
      for (int k = 0; k < dz; ++k) z[d[F_ZO] + t * dz + k] += outv[t][k];
  }
}

/* gx, gy, gw += backward(x, y, w, gz) for one row (kernelgen.cpp:180-251). */
static void FN(bwd_row)(const cgo_problem* p, const T* x, const T* y, const T* w, const T* gz,
                        T* gx, T* gy, T* gw) {
  for (int s = 0; s < p->n; ++s) {
    const int32_t* d = SUB(p, s);
    const cg_entries* cg = cg_get(d[F_L1], d[F_L2], d[F_L3]);
    const int dx = 2 * d[F_L1] + 1, dy = 2 * d[F_L2] + 1, dz = 2 * d[F_L3] + 1;
    const int b = d[F_B], bp = d[F_BP];
    const int lanes = b > bp ? b : bp;
    T gzp[64][MAXW], lgx[64][MAXW], lgy[64][MAXW], zp[64][MAXW], lgw[64];
    for (int t = 0; t < lanes; ++t) {
      for (int k = 0; k < MAXW; ++k) gzp[t][k] = lgx[t][k] = lgy[t][k] = zp[t][k] = (T)0;
      lgw[t] = (T)0;
    }
    const T* gzr = gz + d[F_ZO];
    if (d[F_KIND] == 0) {
      for (int t = 0; t < b; ++t) {
        const T wt = w[d[F_WO] + t];
        for (int k = 0; k < dz; ++k) gzp[t][k] += wt * gzr[t * dz + k];
      }
    } else {
      /* apply_wt: gzp[c][s] = sum_r W[r,c] gz[r][s], r order (kernelgen.cpp:625-637). */
      for (int c = 0; c < bp; ++c)
        for (int q = 0; q < dz; ++q) {
          T acc = gzp[c][q];
          for (int r = 0; r < b; ++r) acc += w[d[F_WO] + r * d[F_WS] + c] * gzr[r * dz + q];
          gzp[c][q] = acc;
        }
    }
    for (int t = 0; t < bp; ++t) {
      const T* xt = x + d[F_XO] + t * dx;
      const T* yy = y + d[F_YO];
      for (int e = 0; e < cg->n; ++e) {
        const T v = (T)cg->v[e];
        const int i = cg->i[e], j = cg->j[e], k = cg->k[e];
        lgx[t][i] += v * yy[j] * gzp[t][k];
        lgy[t][j] += v * xt[i] * gzp[t][k];
        zp[t][k] += v * xt[i] * yy[j];
      }
    }
    /* reduce_lanes: lane 0 sums lanes 1..bp-1 in order (kernelgen.cpp:599-608). */
    for (int q = 0; q < dy; ++q) {
      T acc = lgy[0][q];
      for (int t = 1; t < bp; ++t) acc += lgy[t][q];
      gy[d[F_YO] + q] += acc;
    }
    for (int t = 0; t < bp; ++t)
      for (int i = 0; i < dx; ++i) gx[d[F_XO] + t * dx + i] += lgx[t][i];
    if (d[F_KIND] == 0) {
      for (int t = 0; t < b; ++t) {
        for (int k = 0; k < dz; ++k) lgw[t] += gzr[t * dz + k] * zp[t][k];
        gw[d[F_WO] + t] += lgw[t];
      }
    } else {
      /* outer_acc: GW[r,c] = GW[r,c] + sum_s gz[r][s] z'[c][s] (kernelgen.cpp:639-650). */
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < bp; ++c) {
          T* g = gw + d[F_WO] + r * d[F_WS] + c;
          T acc = *g;
          for (int q = 0; q < dz; ++q) acc += gzr[r * dz + q] * zp[c][q];
          *g = acc;
        }
    }
  }
}

static void FN(zero)(T* a, int64_t n) {
  for (int64_t e = 0; e < n; ++e) a[e] = (T)0;
}

int FN(cgo_tp_forward)(const cgo_problem* p, const T* x, const T* y, const T* w, T* z,
                       int64_t rows, int w_shared) {
  if (prepare(p)) return -1;
  FN(zero)(z, rows * p->dim_z);
  for (int64_t r = 0; r < rows; ++r)
    FN(fwd_row)(p, x + r * p->dim_x, y + r * p->dim_y, w + (w_shared ? 0 : r * p->n_w),
                z + r * p->dim_z);
  return 0;
}

/* w_shared: one weight row for all rows; the shared gradient is the row sum of
 * the per-row gradients, accumulated in double (gap 1). */
int FN(cgo_tp_backward)(const cgo_problem* p, const T* x, const T* y, const T* w, const T* gz,
                        T* gx, T* gy, T* gw, int64_t rows, int w_shared) {
  if (prepare(p)) return -1;
  FN(zero)(gx, rows * p->dim_x);
  FN(zero)(gy, rows * p->dim_y);
  T* tmp = NULL;
  double* acc = NULL;
  if (w_shared) {
    tmp = (T*)malloc(sizeof(T) * (size_t)p->n_w);
    acc = (double*)calloc((size_t)p->n_w, sizeof(double));
  } else {
    FN(zero)(gw, rows * p->n_w);
  }
  for (int64_t r = 0; r < rows; ++r) {
    T* gwr = gw + r * p->n_w;
    if (w_shared) {
      FN(zero)(tmp, p->n_w);
      gwr = tmp;
    }
    FN(bwd_row)(p, x + r * p->dim_x, y + r * p->dim_y, w + (w_shared ? 0 : r * p->n_w),
                gz + r * p->dim_z, gx + r * p->dim_x, gy + r * p->dim_y, gwr);
    if (w_shared)
      for (int q = 0; q < p->n_w; ++q) acc[q] += (double)tmp[q];
  }
  if (w_shared) {
    for (int q = 0; q < p->n_w; ++q) gw[q] = (T)acc[q];
    free(tmp);
    free(acc);
  }
  return 0;
}

/* Fused double-backward (engine.cpp:350-391): op3+op6+op7 -> dL/dgz,
 * op1+op2 -> dL/dx, dL/dy, op4+op5 -> dL/dW. */
static void FN(dbwd_row)(const cgo_problem* p, const T* x, const T* y, const T* w, const T* gz,
                         const T* da, const T* db, const T* dc, T* ox, T* oy, T* ow, T* ogz,
                         T* dump_x, T* dump_y, T* dump_w) {
  FN(fwd_row)(p, da, y, w, ogz);                           /* op3 */
  FN(fwd_row)(p, x, db, w, ogz);                           /* op6 */
  FN(fwd_row)(p, x, y, dc, ogz);                           /* op7 */
  FN(bwd_row)(p, da, db, w, gz, ox, oy, dump_w);           /* op1 */
  FN(bwd_row)(p, x, y, dc, gz, ox, oy, dump_w);            /* op2 */
  FN(bwd_row)(p, da, y, w, gz, dump_x, dump_y, ow);        /* op4 */
  FN(bwd_row)(p, x, db, w, gz, dump_x, dump_y, ow);        /* op5 */
}

int FN(cgo_tp_double_backward)(const cgo_problem* p, const T* x, const T* y, const T* w,
                               const T* gz, const T* da, const T* db, const T* dc, T* ox, T* oy,
                               T* ow, T* ogz, int64_t rows, int w_shared) {
  if (prepare(p)) return -1;
  T* dump_x = (T*)calloc((size_t)p->dim_x, sizeof(T));
  T* dump_y = (T*)calloc((size_t)p->dim_y, sizeof(T));
  T* dump_w = (T*)calloc((size_t)p->n_w, sizeof(T));
  T* tmp = (T*)calloc((size_t)p->n_w, sizeof(T));
  double* acc = (double*)calloc((size_t)p->n_w, sizeof(double));
  FN(zero)(ox, rows * p->dim_x);
  FN(zero)(oy, rows * p->dim_y);
  FN(zero)(ogz, rows * p->dim_z);
  if (!w_shared) FN(zero)(ow, rows * p->n_w);
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t wo = w_shared ? 0 : r * p->n_w;
    T* owr = ow + wo;
    if (w_shared) {
      FN(zero)(tmp, p->n_w);
      owr = tmp;
    }
    FN(dbwd_row)(p, x + r * p->dim_x, y + r * p->dim_y, w + wo, gz + r * p->dim_z,
                 da + r * p->dim_x, db + r * p->dim_y, dc + wo, ox + r * p->dim_x,
                 oy + r * p->dim_y, owr, ogz + r * p->dim_z, dump_x, dump_y, dump_w);
    if (w_shared)
      for (int q = 0; q < p->n_w; ++q) acc[q] += (double)tmp[q];
  }
  if (w_shared)
    for (int q = 0; q < p->n_w; ++q) ow[q] = (T)acc[q];
  free(dump_x);
  free(dump_y);
  free(dump_w);
  free(tmp);
  free(acc);
  return 0;
}

/* Conv forward, deterministic (conv.cpp:234-355): edges sorted by (src, nbr);
 * node_z[src] = sum, in edge order, of each edge's TP output, where each edge
 * output is a fresh zero-initialised TP (conv.cpp:213-230, 303-310). */
int FN(cgo_conv_forward)(const cgo_problem* p, int64_t nodes, int64_t ne,
                         const int64_t* row_ptr, const int32_t* nbr, const T* node_x,
                         const T* edge_y, const T* edge_w, T* node_z, int w_shared) {
  if (prepare(p)) return -1;
  (void)ne;
  T* eo = (T*)malloc(sizeof(T) * (size_t)p->dim_z);
  T* acc = (T*)malloc(sizeof(T) * (size_t)p->dim_z);
  for (int64_t v = 0; v < nodes; ++v) {
    FN(zero)(acc, p->dim_z);
    for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
      FN(zero)(eo, p->dim_z);
      FN(fwd_row)(p, node_x + (int64_t)nbr[e] * p->dim_x, edge_y + e * p->dim_y,
                  edge_w + (w_shared ? 0 : e * p->n_w), eo);
      for (int k = 0; k < p->dim_z; ++k) acc[k] += eo[k];
    }
    T* zr = node_z + v * p->dim_z;
    for (int k = 0; k < p->dim_z; ++k) zr[k] = (T)0 + acc[k];
  }
  free(eo);
  free(acc);
  return 0;
}

/* Stable counting sort of edges by neighbour: the transposed CSR traversal
 * order of conv.cpp:135-151, 384-389. Returns by_pos (position -> edge). */
static int64_t* FN(transposed_order)(int64_t nodes, int64_t ne, const int32_t* nbr) {
  int64_t* cnt = (int64_t*)calloc((size_t)nodes + 1, sizeof(int64_t));
  int64_t* by_pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne > 0 ? ne : 1));
  for (int64_t e = 0; e < ne; ++e) cnt[nbr[e] + 1]++;
  for (int64_t v = 0; v < nodes; ++v) cnt[v + 1] += cnt[v];
  for (int64_t e = 0; e < ne; ++e) by_pos[cnt[nbr[e]]++] = e;
  free(cnt);
  return by_pos;
}

/* Conv backward, deterministic (conv.cpp:357-528): per-edge g_edge_y / g_edge_w;
 * g_node_x[nbr] accumulated over the transposed traversal (nbr-major, src
 * ascending). */
int FN(cgo_conv_backward)(const cgo_problem* p, int64_t nodes, int64_t ne, const int32_t* src,
                          const int32_t* nbr, const T* node_x, const T* edge_y, const T* edge_w,
                          const T* g_node_z, T* g_node_x, T* g_edge_y, T* g_edge_w,
                          int w_shared) {
  if (prepare(p)) return -1;
  int64_t* by_pos = FN(transposed_order)(nodes, ne, nbr);
  FN(zero)(g_node_x, nodes * p->dim_x);
  FN(zero)(g_edge_y, ne * p->dim_y);
  T* tmpw = (T*)calloc((size_t)p->n_w, sizeof(T));
  double* accw = (double*)calloc((size_t)p->n_w, sizeof(double));
  if (!w_shared) FN(zero)(g_edge_w, ne * p->n_w);
  for (int64_t q = 0; q < ne; ++q) {
    const int64_t e = by_pos[q];
    const int32_t s = src[e], d = nbr[e];
    T* gw = g_edge_w + e * p->n_w;
    if (w_shared) {
      FN(zero)(tmpw, p->n_w);
      gw = tmpw;
    }
    FN(bwd_row)(p, node_x + (int64_t)d * p->dim_x, edge_y + e * p->dim_y,
                edge_w + (w_shared ? 0 : e * p->n_w), g_node_z + (int64_t)s * p->dim_z,
                g_node_x + (int64_t)d * p->dim_x, g_edge_y + e * p->dim_y, gw);
    if (w_shared)
      for (int k = 0; k < p->n_w; ++k) accw[k] += (double)tmpw[k];
  }
  if (w_shared)
    for (int k = 0; k < p->n_w; ++k) g_edge_w[k] = (T)accw[k];
  free(tmpw);
  free(accw);
  free(by_pos);
  return 0;
}

/* Conv double-backward oracle composed per SURVEY.md §8c: for each edge
 * e = (s, d): TpPlan::double_backward on (x = node_x[d], y_e, W_e,
 * gz = g_node_z[s], a = d_gx[d], b = d_gy[e], C = d_gw[e]); dL/dx scattered to
 * d, dL/dgz scattered to s (edge order), dL/dy and dL/dW per edge. */
int FN(cgo_conv_double_backward)(const cgo_problem* p, int64_t nodes, int64_t ne,
                                 const int32_t* src, const int32_t* nbr, const T* node_x,
                                 const T* edge_y, const T* edge_w, const T* g_node_z,
                                 const T* d_gx, const T* d_gy, const T* d_gw, T* o_node_x,
                                 T* o_edge_y, T* o_edge_w, T* o_g_node_z, int w_shared) {
  if (prepare(p)) return -1;
  T* ox = (T*)malloc(sizeof(T) * (size_t)p->dim_x);
  T* ogz = (T*)malloc(sizeof(T) * (size_t)p->dim_z);
  T* ow = (T*)malloc(sizeof(T) * (size_t)p->n_w);
  double* accw = (double*)calloc((size_t)p->n_w, sizeof(double));
  T* dump_x = (T*)calloc((size_t)p->dim_x, sizeof(T));
  T* dump_y = (T*)calloc((size_t)p->dim_y, sizeof(T));
  T* dump_w = (T*)calloc((size_t)p->n_w, sizeof(T));
  FN(zero)(o_node_x, nodes * p->dim_x);
  FN(zero)(o_g_node_z, nodes * p->dim_z);
  FN(zero)(o_edge_y, ne * p->dim_y);
  if (!w_shared) FN(zero)(o_edge_w, ne * p->n_w);
  for (int64_t e = 0; e < ne; ++e) {
    const int32_t s = src[e], d = nbr[e];
    const int64_t wo = w_shared ? 0 : e * p->n_w;
    FN(zero)(ox, p->dim_x);
    FN(zero)(ogz, p->dim_z);
    FN(zero)(ow, p->n_w);
    FN(dbwd_row)(p, node_x + (int64_t)d * p->dim_x, edge_y + e * p->dim_y, edge_w + wo,
                 g_node_z + (int64_t)s * p->dim_z, d_gx + (int64_t)d * p->dim_x,
                 d_gy + e * p->dim_y, d_gw + wo, ox, o_edge_y + e * p->dim_y, ow, ogz, dump_x,
                 dump_y, dump_w);
    for (int k = 0; k < p->dim_x; ++k) o_node_x[(int64_t)d * p->dim_x + k] += ox[k];
    for (int k = 0; k < p->dim_z; ++k) o_g_node_z[(int64_t)s * p->dim_z + k] += ogz[k];
    if (w_shared)
      for (int k = 0; k < p->n_w; ++k) accw[k] += (double)ow[k];
    else
      for (int k = 0; k < p->n_w; ++k) o_edge_w[e * p->n_w + k] = ow[k];
  }
  if (w_shared)
    for (int k = 0; k < p->n_w; ++k) o_edge_w[k] = (T)accw[k];
  free(ox);
  free(ogz);
  free(ow);
  free(accw);
  free(dump_x);
  free(dump_y);
  free(dump_w);
  return 0;
}

#undef FN
#undef CAT
#undef CAT2
