/* TEST INFRASTRUCTURE ONLY — see cgoracle.h. Built with -ffp-contract=off,
 * like the reference library (src/CMakeLists.txt:15), so every product and sum
 * below rounds exactly as the reference's does. */
#include "cgoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng ---
 * std::mt19937_64 (the engine rng::NormalGen wraps, rng.hpp:16) and the
 * NormalGen transform: 53-bit uniform (rng.hpp:18-20), Box-Muller with a
 * cached spare (rng.hpp:22-35). */
#define MT_N 312
#define MT_M 156
#define MT_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x7FFFFFFFULL

void cgo_rng_init(cgo_rng* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int n = 1; n < MT_N; ++n)
    g->mt[n] = 6364136223846793005ULL * (g->mt[n - 1] ^ (g->mt[n - 1] >> 62)) + (uint64_t)n;
  g->idx = MT_N;
  g->have_spare = 0;
  g->spare = 0.0;
}

int cgo_rng_size(void) { return (int)sizeof(cgo_rng); }

static void mt_refill(cgo_rng* g) {
  for (int n = 0; n < MT_N; ++n) {
    const uint64_t y = (g->mt[n] & MT_UPPER) | (g->mt[(n + 1) % MT_N] & MT_LOWER);
    g->mt[n] = g->mt[(n + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? MT_A : 0ULL);
  }
  g->idx = 0;
}

uint64_t cgo_rng_bits(cgo_rng* g) {
  if (g->idx >= MT_N) mt_refill(g);
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

static double rng_uniform(cgo_rng* g) { return (double)(cgo_rng_bits(g) >> 11) * 0x1.0p-53; }

double cgo_rng_normal(cgo_rng* g) {
  if (g->have_spare) {
    g->have_spare = 0;
    return g->spare;
  }
  double u1 = rng_uniform(g);
  while (u1 <= 0.0) u1 = rng_uniform(g);
  const double u2 = rng_uniform(g);
  const double r = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  g->spare = r * sin(a);
  g->have_spare = 1;
  return r * cos(a);
}

void cgo_rng_fill_f64(cgo_rng* g, double* out, int64_t n) {
  for (int64_t e = 0; e < n; ++e) out[e] = cgo_rng_normal(g);
}
void cgo_rng_fill_f32(cgo_rng* g, float* out, int64_t n) {
  for (int64_t e = 0; e < n; ++e) out[e] = (float)cgo_rng_normal(g);
}

/* ----------------------------------------------------------------- CG ---
 * Exact factorials through 128-bit integers (irreps.cpp:13-27), the Racah sum
 * (cg.cpp:25-54), and the real-basis block (cg.cpp:58-134). Complex values are
 * carried as (re, im) pairs; the products below reproduce the libstdc++
 * std::complex<double> operations the reference uses term by term. */
double cgo_factorial(int n) {
  if (n < 0 || n > 33) return NAN;
  unsigned __int128 acc = 1;
  for (int k = 2; k <= n; ++k) acc *= (unsigned)k;
  return (double)acc;
}

static int imax3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
static int imin3(int a, int b, int c) { return a < b ? (a < c ? a : c) : (b < c ? b : c); }

double cgo_complex_cg(int l1, int l2, int l3, int m1, int m2, int m3) {
  if (m1 + m2 != m3) return 0.0;
  const double pre =
      sqrt((2.0 * l3 + 1.0) * cgo_factorial(l1 + l2 - l3) * cgo_factorial(l1 - l2 + l3) *
           cgo_factorial(-l1 + l2 + l3) / cgo_factorial(l1 + l2 + l3 + 1)) *
      sqrt(cgo_factorial(l3 + m3) * cgo_factorial(l3 - m3) * cgo_factorial(l1 - m1) *
           cgo_factorial(l1 + m1) * cgo_factorial(l2 - m2) * cgo_factorial(l2 + m2));
  const int k0 = imax3(0, l2 - l3 - m1, l1 - l3 + m2);
  const int k1 = imin3(l1 + l2 - l3, l1 - m1, l2 + m2);
  double s = 0.0;
  for (int k = k0; k <= k1; ++k) {
    const double sg = (k % 2 == 0) ? 1.0 : -1.0;
    s += sg / (cgo_factorial(k) * cgo_factorial(l1 + l2 - l3 - k) * cgo_factorial(l1 - m1 - k) *
               cgo_factorial(l2 + m2 - k) * cgo_factorial(l3 - l2 + m1 + k) *
               cgo_factorial(l3 - l1 - m2 + k));
  }
  return pre * s;
}

typedef struct {
  double re, im;
} cpx;

static cpx cmul(cpx a, cpx b) {
  cpx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}

/* Entry (row p, column m) of the complex->real change of basis, both indices
 * shifted by +l (irreps.cpp:164-178). */
static cpx basis(int l, int p, int m) {
  const double h = 1.0 / sqrt(2.0);
  cpx z = {0.0, 0.0};
  if (p == l && m == l) {
    z.re = 1.0;
    return z;
  }
  const int a = p - l, b = m - l;
  if (a > 0) {
    const double cs = (a % 2 == 0) ? 1.0 : -1.0;
    if (b == a) z.re = cs * h;
    if (b == -a) z.re = h;
  } else if (a < 0) {
    const int q = -a;
    const double cs = (q % 2 == 0) ? 1.0 : -1.0;
    if (b == q) z.im = -cs * h;
    if (b == -q) z.im = h;
  }
  return z;
}

#define CGO_LMAX 12
typedef struct {
  int n;
  int* i;
  int* j;
  int* k;
  double* v;
} cg_entries;
static cg_entries* g_memo[CGO_LMAX + 1][CGO_LMAX + 1][CGO_LMAX + 1];

static cg_entries* build_block(int l1, int l2, int l3) {
  const int d1 = 2 * l1 + 1, d2 = 2 * l2 + 1, d3 = 2 * l3 + 1;
  const size_t nt = (size_t)d1 * d2 * d3;
  cpx* t = (cpx*)calloc(nt, sizeof(cpx));
#define AT(i, j, k) t[((size_t)(i) * d2 + (j)) * d3 + (k)]
  for (int m1 = -l1; m1 <= l1; ++m1) {
    for (int m2 = -l2; m2 <= l2; ++m2) {
      const int m3 = m1 + m2;
      if (abs(m3) > l3) continue;
      const double c = cgo_complex_cg(l1, l2, l3, m1, m2, m3);
      if (c == 0.0) continue;
      for (int i = 0; i < d1; ++i) {
        const cpx f1 = basis(l1, i, l1 + m1);
        if (f1.re == 0.0 && f1.im == 0.0) continue;
        for (int j = 0; j < d2; ++j) {
          const cpx f2 = basis(l2, j, l2 + m2);
          if (f2.re == 0.0 && f2.im == 0.0) continue;
          for (int k = 0; k < d3; ++k) {
            cpx f3 = basis(l3, k, l3 + m3);
            f3.im = -f3.im; /* conj */
            if (f3.re == 0.0 && f3.im == 0.0) continue;
            cpx p = cmul(cmul(f1, f2), f3);
            p.re *= c;
            p.im *= c;
            AT(i, j, k).re += p.re;
            AT(i, j, k).im += p.im;
          }
        }
      }
    }
  }
  /* Largest-magnitude entry becomes real positive (cg.cpp:98-106). */
  cpx top = {0.0, 0.0};
  double top_abs = 0.0;
  for (size_t e = 0; e < nt; ++e) {
    const double a = hypot(t[e].re, t[e].im);
    if (a > top_abs) {
      top = t[e];
      top_abs = a;
    }
  }
  if (top_abs > 0.0) {
    const cpx ph = {top.re / top_abs, -top.im / top_abs};
    for (size_t e = 0; e < nt; ++e) t[e] = cmul(t[e], ph);
  }
  cg_entries* out = (cg_entries*)calloc(1, sizeof(cg_entries));
  out->i = (int*)malloc(sizeof(int) * nt);
  out->j = (int*)malloc(sizeof(int) * nt);
  out->k = (int*)malloc(sizeof(int) * nt);
  out->v = (double*)malloc(sizeof(double) * nt);
  for (int k = 0; k < d3; ++k)
    for (int i = 0; i < d1; ++i)
      for (int j = 0; j < d2; ++j) {
        const cpx v = AT(i, j, k);
        if (fabs(v.im) > 1e-12) { /* reference throws (cg.cpp:114-117) */
          out->n = -1;
          free(t);
          return out;
        }
        if (fabs(v.re) > 1e-12) {
          out->i[out->n] = i;
          out->j[out->n] = j;
          out->k[out->n] = k;
          out->v[out->n] = v.re;
          out->n++;
        }
      }
#undef AT
  /* Per-k unit norm (cg.cpp:124-129). */
  double* nrm = (double*)calloc((size_t)d3, sizeof(double));
  for (int e = 0; e < out->n; ++e) nrm[out->k[e]] += out->v[e] * out->v[e];
  for (int e = 0; e < out->n; ++e) {
    const double q = nrm[out->k[e]];
    if (q > 0.0) out->v[e] /= sqrt(q);
  }
  free(nrm);
  free(t);
  return out;
}

static int triangle(int l1, int l2, int l3) { return l3 >= abs(l1 - l2) && l3 <= l1 + l2; }

static const cg_entries* cg_get(int l1, int l2, int l3) {
  if (l1 < 0 || l2 < 0 || l3 < 0 || l1 > CGO_LMAX || l2 > CGO_LMAX || l3 > CGO_LMAX) return NULL;
  if (!triangle(l1, l2, l3) || l1 + l2 + l3 + 1 > 33) return NULL;
  cg_entries* e = g_memo[l1][l2][l3];
  if (!e) {
    e = build_block(l1, l2, l3);
    g_memo[l1][l2][l3] = e;
  }
  return e->n < 0 ? NULL : e;
}

int cgo_cg_block(int l1, int l2, int l3, int cap, int* i, int* j, int* k, double* v) {
  const cg_entries* e = cg_get(l1, l2, l3);
  if (!e) return -1;
  for (int n = 0; n < e->n && n < cap; ++n) {
    i[n] = e->i[n];
    j[n] = e->j[n];
    k[n] = e->k[n];
    v[n] = e->v[n];
  }
  return e->n;
}

/* Builds every block a problem needs before any (possibly threaded) sweep. */
static int prepare(const cgo_problem* p) {
  for (int s = 0; s < p->n; ++s) {
    const int32_t* d = p->subs + CGO_SUB_FIELDS * s;
    if (!cg_get(d[1], d[2], d[3])) return -1;
    if (d[4] > 64 || d[5] > 64 || d[4] < 1 || d[5] < 1) return -2;
  }
  return 0;
}

#define SUB(p, s) ((p)->subs + CGO_SUB_FIELDS * (s))
enum { F_KIND, F_L1, F_L2, F_L3, F_B, F_BP, F_XO, F_YO, F_ZO, F_WO, F_WS };
/* Lane register groups sized for l <= 12 (kernelgen.hpp:24); <= 64 lanes. */
#define MAXW 25

#define T float
#define SUF f32
#include "cgoracle_impl.h"
#undef T
#undef SUF

#define T double
#define SUF f64
#include "cgoracle_impl.h"
#undef T
#undef SUF
