/*
 * sgw_oracle.c -- CPU restatement of the reference sgweno hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see sgw_oracle.h).  Compiled with
 * -O2 -ffp-contract=off so every expression below rounds exactly like the
 * reference headers built the same way; tests/test_oracle_pin.py checks that
 * against oracle/_ref/libsgwref.so (the reference headers themselves) and the
 * committed golden fixtures.
 *
 * Citations: /root/reference/proj/include/sgweno/<file>:<line>.
 */
#define _GNU_SOURCE
#include "sgw_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static double sqr(double x) { return x * x; } /* weno.hpp:31 */

/* Member-level parallelism of the oracle (OpenMP; 1 = serial, the default).
 * Members are independent within a step given dt (timestep.hpp:156-165 loops
 * over them serially), so every result is bitwise the same for any count. */
static int g_threads = 1;
void sgwo_set_threads(int n) { g_threads = (n < 1) ? 1 : n; }
int sgwo_get_threads(void) { return g_threads; }

/* ------------------------------------------------------------------------ */
/* grid.hpp                                                                  */
/* ------------------------------------------------------------------------ */

/* grid.hpp:57-79: recursion emits tuples in lexicographic order already. */
static int enum_rec(int d, int nl, int lo_sum, int k, int used, int* cur, int* out, int cap,
                    int count) {
  if (k == d - 1) {
    int last = lo_sum - used;
    if (last < 0) last = 0;
    for (; last + used <= nl; ++last) {
      cur[k] = last;
      if (used + last >= lo_sum) {
        if (out && count < cap)
          for (int q = 0; q < d; ++q) out[count * d + q] = cur[q];
        ++count;
      }
    }
    return count;
  }
  for (int l = 0; l + used <= nl; ++l) {
    cur[k] = l;
    count = enum_rec(d, nl, lo_sum, k + 1, used + l, cur, out, cap, count);
  }
  return count;
}

int sgwo_enumerate_levels(int d, int nl, int* out, int cap) {
  if (d < 1 || d > 4 || nl < d - 1) return -1;
  int cur[4] = {0, 0, 0, 0};
  int lo_sum = nl - d + 1;
  if (lo_sum < 0) lo_sum = 0;
  return enum_rec(d, nl, lo_sum, 0, 0, cur, out, cap, 0);
}

/* combine.hpp:27-43 */
static long long binomial(int n, int k) {
  if (k < 0 || k > n) return 0;
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

int sgwo_combination_coefficients(int d, int nl, long long* coef) {
  if (d < 1 || d > 4 || nl < d - 1) return SGWO_EINVAL;
  for (int j = 0; j < d; ++j) coef[j] = (j % 2 == 0 ? 1 : -1) * binomial(d - 1, j);
  return SGWO_OK;
}

/* grid.hpp:110-133 */
void sgwo_member_geometry(const sgwo_domain* dom, const int* level, int* points, double* spacing) {
  for (int k = 0; k < dom->d; ++k) {
    int cells = dom->root_cells[k] << level[k];
    points[k] = cells + (dom->bc[k] == SGWO_ZERO ? 1 : 0);
    double rootH = (dom->upper[k] - dom->lower[k]) / dom->root_cells[k];
    spacing[k] = ldexp(rootH, -level[k]);
  }
}

size_t sgwo_member_points(const sgwo_domain* dom, const int* level) {
  int pts[4];
  double sp[4];
  sgwo_member_geometry(dom, level, pts, sp);
  size_t n = 1;
  for (int k = 0; k < dom->d; ++k) n *= (size_t)pts[k];
  return n;
}

static int family_levels(const sgwo_domain* dom, int** levels_out) {
  int n = sgwo_enumerate_levels(dom->d, dom->nl, NULL, 0);
  if (n < 0) return -1;
  int* lv = (int*)malloc(sizeof(int) * (size_t)n * (size_t)dom->d);
  sgwo_enumerate_levels(dom->d, dom->nl, lv, n);
  *levels_out = lv;
  return n;
}

size_t sgwo_family_total_points(const sgwo_domain* dom) {
  int* lv;
  int n = family_levels(dom, &lv);
  if (n < 0) return 0;
  size_t tot = 0;
  for (int m = 0; m < n; ++m) tot += sgwo_member_points(dom, lv + m * dom->d);
  free(lv);
  return tot;
}

size_t sgwo_finest_points(const sgwo_domain* dom) {
  int lv[4];
  for (int k = 0; k < dom->d; ++k) lv[k] = dom->nl;
  return sgwo_member_points(dom, lv);
}

/* ------------------------------------------------------------------------ */
/* weno.hpp                                                                  */
/* ------------------------------------------------------------------------ */

static const double kLinearWeight0 = 0.1; /* weno.hpp:25-27 */
static const double kLinearWeight1 = 0.6;
static const double kLinearWeight2 = 0.3;
static const double kSixth = 1.0 / 6.0; /* weno.hpp:29 */

/* weno.hpp:36-44 */
void sgwo_smoothness_indicators(const double* s, double* b) {
  b[0] = (13.0 / 12.0) * sqr(s[0] - 2.0 * s[1] + s[2]) + 0.25 * sqr(s[0] - 4.0 * s[1] + 3.0 * s[2]);
  b[1] = (13.0 / 12.0) * sqr(s[1] - 2.0 * s[2] + s[3]) + 0.25 * sqr(s[1] - s[3]);
  b[2] = (13.0 / 12.0) * sqr(s[2] - 2.0 * s[3] + s[4]) + 0.25 * sqr(3.0 * s[2] - 4.0 * s[3] + s[4]);
}

/* weno.hpp:60-72 */
double sgwo_weno5_flux_positive(const double* s, double eps, int mode) {
  const double c0 = kSixth * (2.0 * s[0] - 7.0 * s[1] + 11.0 * s[2]);
  const double c1 = kSixth * (-s[1] + 5.0 * s[2] + 2.0 * s[3]);
  const double c2 = kSixth * (2.0 * s[2] + 5.0 * s[3] - s[4]);
  if (mode == SGWO_WENO_LINEAR) return kLinearWeight0 * c0 + kLinearWeight1 * c1 + kLinearWeight2 * c2;
  double b[3];
  sgwo_smoothness_indicators(s, b);
  const double a0 = kLinearWeight0 / sqr(eps + b[0]);
  const double a1 = kLinearWeight1 / sqr(eps + b[1]);
  const double a2 = kLinearWeight2 / sqr(eps + b[2]);
  return (a0 * c0 + a1 * c1 + a2 * c2) / (a0 + a1 + a2);
}

/* weno.hpp:78-80 */
double sgwo_weno5_flux_negative(const double* s, double eps, int mode) {
  const double r[5] = {s[4], s[3], s[2], s[1], s[0]};
  return sgwo_weno5_flux_positive(r, eps, mode);
}

/* weno.hpp:118-154 (generic) and 160-192 (advect fast path). */
int sgwo_weno_derivative_line(const double* u, int n, int flux_kind, double c, double alpha,
                              double dx, int bc, double eps, int mode, double* out) {
  if (bc == SGWO_PERIODIC && n < 6) return SGWO_EINVAL;
  if (n < 1) return SGWO_EINVAL;
  double* fp = (double*)malloc(sizeof(double) * (size_t)(n + 6));
  double* fm = (double*)malloc(sizeof(double) * (size_t)(n + 6));
  double* fhat = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  for (int j = -3; j < n + 3; ++j) {
    double uj;
    if (bc == SGWO_PERIODIC)
      uj = u[((j % n) + n) % n];
    else
      uj = (j >= 0 && j < n) ? u[j] : 0.0;
    if (flux_kind == 0) {
      fp[j + 3] = c * uj; /* weno.hpp:176 */
    } else {
      const double f = (flux_kind == 1) ? 0.5 * uj * uj : c * uj;
      const double fpj = 0.5 * (f + alpha * uj); /* weno.hpp:138-140 */
      fp[j + 3] = fpj;
      fm[j + 3] = f - fpj;
    }
  }
  const int downwind = (c < 0.0);
  const int nint = (bc == SGWO_PERIODIC) ? n : n + 1;
  const int k0 = (bc == SGWO_PERIODIC) ? 0 : -1;
  for (int k = k0; k < k0 + nint; ++k) {
    double v;
    if (flux_kind == 0)
      v = downwind ? sgwo_weno5_flux_negative(&fp[k + 2], eps, mode)
                   : sgwo_weno5_flux_positive(&fp[k + 1], eps, mode);
    else
      v = sgwo_weno5_flux_positive(&fp[k + 1], eps, mode) +
          sgwo_weno5_flux_negative(&fm[k + 2], eps, mode);
    fhat[k - k0] = v;
  }
  if (bc == SGWO_PERIODIC) {
    for (int i = 0; i < n; ++i) out[i] = (fhat[i] - fhat[(i + n - 1) % n]) / dx;
  } else {
    for (int i = 0; i < n; ++i) out[i] = (fhat[i + 1] - fhat[i]) / dx;
  }
  free(fp);
  free(fm);
  free(fhat);
  return SGWO_OK;
}

/* ------------------------------------------------------------------------ */
/* models.hpp                                                                */
/* ------------------------------------------------------------------------ */

typedef struct {
  int d;
  int points[4];
  double spacing[4];
  size_t strides[4];
  size_t total;
} geom_t;

static void make_geom(const sgwo_domain* dom, const int* level, geom_t* g) {
  g->d = dom->d;
  sgwo_member_geometry(dom, level, g->points, g->spacing);
  g->strides[dom->d - 1] = 1;
  for (int k = dom->d - 2; k >= 0; --k) g->strides[k] = g->strides[k + 1] * (size_t)g->points[k + 1];
  g->total = 1;
  for (int k = 0; k < dom->d; ++k) g->total *= (size_t)g->points[k];
}

/* models.hpp:110-114 */
static double max_abs(const double* v, size_t n) {
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double a = fabs(v[i]);
    m = (m < a) ? a : m; /* std::max(m, a) returns m unless m < a */
  }
  return m;
}

/* coordinate of dimension q of the line `which` along dimension k (line_at order,
 * grid.hpp:207-217); equivalently IndexExtractor (models.hpp:118-131). */
static int line_coord(const geom_t* g, int k, size_t which, int q) {
  size_t div = 1;
  for (int r = q + 1; r < g->d; ++r)
    if (r != k) div *= (size_t)g->points[r];
  return (int)((which / div) % (size_t)g->points[q]);
}

/* models.hpp:142-177: out -= d/dx_k (flux) along every line of dimension k.
 * coef: per-line coefficient callback data (advection) or NULL for Burgers. */
typedef double (*coef_fn)(const geom_t* g, int k, size_t which, const void* data);

static int sweep(const geom_t* g, int k, const double* state, int flux_kind, double alpha,
                 coef_fn coef, const void* cdata, int bc, double eps, int mode, double* out) {
  const int n = g->points[k];
  const double h = g->spacing[k];
  const size_t stride = g->strides[k];
  size_t inner = 1;
  for (int q = k + 1; q < g->d; ++q) inner *= (size_t)g->points[q];
  const size_t nlines = g->total / (size_t)n;
  double* bu = (double*)malloc(sizeof(double) * (size_t)n);
  double* bd = (double*)malloc(sizeof(double) * (size_t)n);
  int st = SGWO_OK;
  for (size_t which = 0; which < nlines && st == SGWO_OK; ++which) {
    const size_t o = which / inner, i = which % inner;
    const size_t base = o * (size_t)n * stride + i;
    for (int j = 0; j < n; ++j) bu[j] = state[base + (size_t)j * stride];
    double c = coef ? coef(g, k, which, cdata) : 0.0;
    st = sgwo_weno_derivative_line(bu, n, flux_kind, c, alpha, h, bc, eps, mode, bd);
    for (int j = 0; j < n; ++j) out[base + (size_t)j * stride] -= bd[j];
  }
  free(bu);
  free(bd);
  return st;
}

static double const_coef(const geom_t* g, int k, size_t which, const void* data) {
  (void)g;
  (void)which;
  return ((const double*)data)[k];
}

typedef struct {
  const double* coords[4]; /* grid coordinates per dimension */
  const double* field;     /* VP: E_j(x) component-major over the x-grid, else NULL */
  size_t nx;               /* x-grid size */
  int dx;                  /* space dim */
  int comp;                /* which component */
} kin_coef_t;

/* x_j lines: coefficient v_j (models.hpp:341-344) */
static double kin_x_coef(const geom_t* g, int k, size_t which, const void* data) {
  const kin_coef_t* kc = (const kin_coef_t*)data;
  int q = kc->dx + k;
  return kc->coords[q][line_coord(g, k, which, q)];
}

/* v_j lines: coefficient -x_j (VB, models.hpp:346-349) or -E_j(x) (VP). */
static double kin_v_coef(const geom_t* g, int k, size_t which, const void* data) {
  const kin_coef_t* kc = (const kin_coef_t*)data;
  int j = k - kc->dx;
  if (!kc->field) return -kc->coords[j][line_coord(g, k, which, j)];
  /* linear x index of the line */
  size_t xi = 0;
  for (int q = 0; q < kc->dx; ++q) xi = xi * (size_t)g->points[q] + (size_t)line_coord(g, k, which, q);
  return -kc->field[(size_t)kc->comp * kc->nx + xi];
}

/* models.hpp:64-71 */
static void trapezoid_weights_1d(const geom_t* g, int k, int bc, double* w) {
  for (int i = 0; i < g->points[k]; ++i) w[i] = g->spacing[k];
  if (bc == SGWO_ZERO) {
    w[0] *= 0.5;
    w[g->points[k] - 1] *= 0.5;
  }
}

/* models.hpp:240-257 */
static double* block_weights(const geom_t* g, const sgwo_domain* dom, int lo, int hi, size_t* nout) {
  double* w1[4];
  size_t n = 1;
  for (int k = lo; k < hi; ++k) {
    w1[k - lo] = (double*)malloc(sizeof(double) * (size_t)g->points[k]);
    trapezoid_weights_1d(g, k, dom->bc[k], w1[k - lo]);
    n *= (size_t)g->points[k];
  }
  double* out = (double*)malloc(sizeof(double) * n);
  int idx[4] = {0, 0, 0, 0};
  const int nd = hi - lo;
  for (size_t lin = 0; lin < n; ++lin) {
    double p = 1.0;
    for (int k = 0; k < nd; ++k) p *= w1[k][idx[k]];
    out[lin] = p;
    for (int k = nd - 1; k >= 0; --k) {
      if (++idx[k] < g->points[lo + k]) break;
      idx[k] = 0;
    }
  }
  for (int k = 0; k < nd; ++k) free(w1[k]);
  *nout = n;
  return out;
}

static double** make_coords(const sgwo_domain* dom, const geom_t* g) {
  double** c = (double**)malloc(sizeof(double*) * 4);
  for (int k = 0; k < g->d; ++k) {
    c[k] = (double*)malloc(sizeof(double) * (size_t)g->points[k]);
    for (int i = 0; i < g->points[k]; ++i) c[k][i] = dom->lower[k] + i * g->spacing[k];
  }
  return c;
}
static void free_coords(double** c, int d) {
  for (int k = 0; k < d; ++k) free(c[k]);
  free(c);
}

/* ---- Vlasov-Poisson field (NEW physics, unpinned; see header) ---- */

/* spectral periodic Poisson on an n1 x n2 grid (n2 = 1 for 1D).
 * rho_hat = DFT(rho); E_hat_j = -i kappa_j rho_hat / |kappa|^2; zero mean and
 * Nyquist modes dropped. */
static void spectral_poisson(int dxs, const int* n, const double* L, const double* rho, double* E) {
  const int n1 = n[0], n2 = (dxs == 2) ? n[1] : 1;
  const size_t N = (size_t)n1 * (size_t)n2;
  /* twiddle tables: the same cos, sin of 2 pi ph / n that the sums used inline */
  double* c1t = (double*)malloc(sizeof(double) * (size_t)n1);
  double* s1t = (double*)malloc(sizeof(double) * (size_t)n1);
  double* c2t = (double*)malloc(sizeof(double) * (size_t)n2);
  double* s2t = (double*)malloc(sizeof(double) * (size_t)n2);
  for (int ph = 0; ph < n1; ++ph) {
    const double th = 2.0 * M_PI * (double)ph / (double)n1;
    c1t[ph] = cos(th);
    s1t[ph] = sin(th);
  }
  for (int ph = 0; ph < n2; ++ph) {
    const double th = 2.0 * M_PI * (double)ph / (double)n2;
    c2t[ph] = cos(th);
    s2t[ph] = sin(th);
  }
  double* rr = (double*)calloc(N, sizeof(double));
  double* ri = (double*)calloc(N, sizeof(double));
  /* forward DFT, dimension 1 (fast) then dimension 0 */
  double* tr = (double*)calloc(N, sizeof(double));
  double* ti = (double*)calloc(N, sizeof(double));
  for (int a = 0; a < n1; ++a)
    for (int k2 = 0; k2 < n2; ++k2) {
      double sr = 0.0, si = 0.0;
      for (int b = 0; b < n2; ++b) {
        long ph = ((long)k2 * b) % n2;
        double v = rho[(size_t)a * n2 + b];
        sr += v * c2t[ph];
        si -= v * s2t[ph];
      }
      tr[(size_t)a * n2 + k2] = sr;
      ti[(size_t)a * n2 + k2] = si;
    }
  for (int k1 = 0; k1 < n1; ++k1)
    for (int k2 = 0; k2 < n2; ++k2) {
      double sr = 0.0, si = 0.0;
      for (int a = 0; a < n1; ++a) {
        long ph = ((long)k1 * a) % n1;
        double c = c1t[ph], s = -s1t[ph];
        double xr = tr[(size_t)a * n2 + k2], xi = ti[(size_t)a * n2 + k2];
        sr += xr * c - xi * s;
        si += xr * s + xi * c;
      }
      rr[(size_t)k1 * n2 + k2] = sr;
      ri[(size_t)k1 * n2 + k2] = si;
    }
  for (int comp = 0; comp < dxs; ++comp) {
    /* E_hat */
    for (int k1 = 0; k1 < n1; ++k1)
      for (int k2 = 0; k2 < n2; ++k2) {
        int s1 = (k1 <= n1 / 2) ? k1 : k1 - n1;
        int s2 = (k2 <= n2 / 2) ? k2 : k2 - n2;
        int nyq = ((n1 % 2 == 0) && k1 == n1 / 2 && n1 > 1) || ((n2 % 2 == 0) && k2 == n2 / 2 && n2 > 1);
        double kap1 = 2.0 * M_PI * (double)s1 / L[0];
        double kap2 = (dxs == 2) ? 2.0 * M_PI * (double)s2 / L[1] : 0.0;
        double k2s = kap1 * kap1 + kap2 * kap2;
        size_t id = (size_t)k1 * n2 + k2;
        if ((s1 == 0 && s2 == 0) || nyq) {
          tr[id] = 0.0;
          ti[id] = 0.0;
          continue;
        }
        double kc = (comp == 0) ? kap1 : kap2;
        /* -i kc (rr + i ri) / k2s = (kc ri - i kc rr)/k2s */
        tr[id] = kc * ri[id] / k2s;
        ti[id] = -kc * rr[id] / k2s;
      }
    /* inverse DFT (real part) */
    double* ur = (double*)calloc(N, sizeof(double));
    double* ui = (double*)calloc(N, sizeof(double));
    for (int k1 = 0; k1 < n1; ++k1)
      for (int b = 0; b < n2; ++b) {
        double sr = 0.0, si = 0.0;
        for (int k2 = 0; k2 < n2; ++k2) {
          long ph = ((long)k2 * b) % n2;
          double c = c2t[ph], s = s2t[ph];
          double xr = tr[(size_t)k1 * n2 + k2], xi = ti[(size_t)k1 * n2 + k2];
          sr += xr * c - xi * s;
          si += xr * s + xi * c;
        }
        ur[(size_t)k1 * n2 + b] = sr;
        ui[(size_t)k1 * n2 + b] = si;
      }
    for (int a = 0; a < n1; ++a)
      for (int b = 0; b < n2; ++b) {
        double sr = 0.0;
        for (int k1 = 0; k1 < n1; ++k1) {
          long ph = ((long)k1 * a) % n1;
          sr += ur[(size_t)k1 * n2 + b] * c1t[ph] - ui[(size_t)k1 * n2 + b] * s1t[ph];
        }
        E[(size_t)comp * N + (size_t)a * n2 + b] = sr / (double)N;
      }
    free(ur);
    free(ui);
  }
  free(rr);
  free(ri);
  free(tr);
  free(ti);
  free(c1t);
  free(s1t);
  free(c2t);
  free(s2t);
}

static int vp_field_geom(const sgwo_domain* dom, const geom_t* g, int dxs, const double* f,
                         double* rho, double* E) {
  size_t vn;
  double* vw = block_weights(g, dom, dxs, 2 * dxs, &vn);
  size_t nx = g->total / vn;
  for (size_t s = 0; s < nx; ++s) {
    /* moment_density (models.hpp:294-306): acc = sum_i w_i f_i, then rho = 1 - acc */
    double acc = 0.0;
    const double* block = f + s * vn;
    for (size_t i = 0; i < vn; ++i) acc += vw[i] * block[i];
    rho[s] = 1.0 - acc;
  }
  int n[2] = {g->points[0], dxs == 2 ? g->points[1] : 1};
  double L[2] = {dom->upper[0] - dom->lower[0], dxs == 2 ? dom->upper[1] - dom->lower[1] : 1.0};
  spectral_poisson(dxs, n, L, rho, E);
  free(vw);
  return SGWO_OK;
}

int sgwo_vp_field(const sgwo_domain* dom, const int* level, int space_dim, const double* f,
                  double* rho, double* E) {
  geom_t g;
  make_geom(dom, level, &g);
  if (dom->d != 2 * space_dim) return SGWO_EINVAL;
  for (int k = 0; k < space_dim; ++k)
    if (dom->bc[k] != SGWO_PERIODIC) return SGWO_EINVAL;
  return vp_field_geom(dom, &g, space_dim, f, rho, E);
}

/* models.hpp:184-198 (conservation law), 334-363 (VB), VP restatement. */
int sgwo_rhs(const sgwo_domain* dom, const int* level, const sgwo_model* model,
             const double* state, double* out) {
  geom_t g;
  make_geom(dom, level, &g);
  memset(out, 0, sizeof(double) * g.total);
  const double eps = model->epsilon;
  const int mode = model->weno_mode;
  int st = SGWO_OK;
  if (model->kind == SGWO_ADVECTION || model->kind == SGWO_BURGERS) {
    const double umax = (model->kind == SGWO_BURGERS) ? max_abs(state, g.total) : 0.0;
    for (int k = 0; k < g.d && st == SGWO_OK; ++k) {
      if (model->kind == SGWO_ADVECTION)
        st = sweep(&g, k, state, 0, 0.0, const_coef, model->speeds, dom->bc[k], eps, mode, out);
      else
        st = sweep(&g, k, state, 1, umax, NULL, NULL, dom->bc[k], eps, mode, out);
    }
    return st;
  }
  /* kinetic transport template (models.hpp:334-350) */
  const int dxs = model->space_dim;
  if (g.d != 2 * dxs) return SGWO_EINVAL;
  double** coords = make_coords(dom, &g);
  kin_coef_t kc;
  for (int k = 0; k < g.d; ++k) kc.coords[k] = coords[k];
  kc.dx = dxs;
  kc.field = NULL;
  kc.nx = 1;
  double* E = NULL;
  double* rho = NULL;
  size_t vn = 1;
  for (int k = dxs; k < g.d; ++k) vn *= (size_t)g.points[k];
  kc.nx = g.total / vn;
  if (model->kind == SGWO_VLASOV_POISSON) {
    E = (double*)malloc(sizeof(double) * kc.nx * (size_t)dxs);
    rho = (double*)malloc(sizeof(double) * kc.nx);
    vp_field_geom(dom, &g, dxs, state, rho, E);
    kc.field = E;
  }
  for (int j = 0; j < dxs && st == SGWO_OK; ++j) {
    st = sweep(&g, j, state, 0, 0.0, kin_x_coef, &kc, dom->bc[j], eps, mode, out);
    if (st != SGWO_OK) break;
    kc.comp = j;
    st = sweep(&g, dxs + j, state, 0, 0.0, kin_v_coef, &kc, dom->bc[dxs + j], eps, mode, out);
  }
  if (st == SGWO_OK && model->kind == SGWO_VLASOV_BOLTZMANN) {
    /* relaxation (models.hpp:351-362) with VbWorkspace (271-290) */
    size_t vn2;
    double* vw = block_weights(&g, dom, dxs, 2 * dxs, &vn2);
    /* maxwellian on the velocity sub-grid (models.hpp:213-224) */
    double* mu = (double*)malloc(sizeof(double) * vn2);
    const double norm = pow(2.0 * M_PI * model->theta, 0.5 * dxs);
    int idx[4] = {0, 0, 0, 0};
    for (size_t lin = 0; lin < vn2; ++lin) {
      double s = 0.0;
      for (int q = 0; q < dxs; ++q) {
        double c = dom->lower[dxs + q] + idx[q] * g.spacing[dxs + q];
        s += c * c;
      }
      mu[lin] = exp(-s / (2.0 * model->theta)) / norm;
      for (int q = dxs - 1; q >= 0; --q) {
        if (++idx[q] < g.points[dxs + q]) break;
        idx[q] = 0;
      }
    }
    double mass = 0.0;
    for (size_t i = 0; i < vn2; ++i) mass += vw[i] * mu[i];
    for (size_t i = 0; i < vn2; ++i) mu[i] /= mass;
    const size_t xn = g.total / vn2;
    const double inv_tau = 1.0 / model->tau;
    for (size_t s = 0; s < xn; ++s) {
      const double* block = state + s * vn2;
      double rho_s = 0.0;
      for (size_t i = 0; i < vn2; ++i) rho_s += vw[i] * block[i];
      double* o = out + s * vn2;
      for (size_t i = 0; i < vn2; ++i) o[i] += (mu[i] * rho_s - block[i]) * inv_tau;
    }
    free(vw);
    free(mu);
  }
  free(E);
  free(rho);
  free_coords(coords, g.d);
  return st;
}

/* ------------------------------------------------------------------------ */
/* timestep.hpp                                                              */
/* ------------------------------------------------------------------------ */

/* timestep.hpp:71-75 */
static int tendency_finite(const double* k, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += k[i];
  return isfinite(s);
}

/* timestep.hpp:83-108 */
int sgwo_rk3_step(const sgwo_domain* dom, const int* level, const sgwo_model* model,
                  double* u, double dt) {
  const size_t n = sgwo_member_points(dom, level);
  double* stage = (double*)malloc(sizeof(double) * n);
  double* k = (double*)malloc(sizeof(double) * n);
  int fail = 0;
  sgwo_rhs(dom, level, model, u, k);
  if (!tendency_finite(k, n)) { fail = 1; goto done; }
  for (size_t i = 0; i < n; ++i) stage[i] = u[i] + dt * k[i];
  sgwo_rhs(dom, level, model, stage, k);
  if (!tendency_finite(k, n)) { fail = 2; goto done; }
  for (size_t i = 0; i < n; ++i) stage[i] = 0.75 * u[i] + 0.25 * (stage[i] + dt * k[i]);
  sgwo_rhs(dom, level, model, stage, k);
  if (!tendency_finite(k, n)) { fail = 3; goto done; }
  for (size_t i = 0; i < n; ++i) u[i] = (1.0 / 3.0) * u[i] + (2.0 / 3.0) * (stage[i] + dt * k[i]);
done:
  free(stage);
  free(k);
  return fail;
}

/* timestep.hpp:47-67 (+ dt_scale: accuracy-mode multiplier, 1.0 = reference) */
double sgwo_compute_dt(const sgwo_policy* p, const double* speeds, const double* spacings, int d,
                       double remaining) {
  double dt;
  if (p->mode == SGWO_DT_CFL) {
    double inv = 0.0;
    for (int k = 0; k < d; ++k) inv += speeds[k] / spacings[k];
    if (inv == 0.0) return remaining;
    dt = p->cfl / inv;
  } else {
    dt = pow(p->reference_spacing, 5.0 / 3.0);
    if (p->dt_scale != 1.0) dt = p->dt_scale * dt;
  }
  return (remaining < dt) ? remaining : dt; /* std::min(dt, remaining) */
}

/* models.hpp:791-839 */
int sgwo_family_wave_speeds(const sgwo_domain* dom, const sgwo_model* model, const double* states,
                            double* speeds) {
  int* lv;
  int nm = family_levels(dom, &lv);
  const int d = dom->d;
  for (int k = 0; k < d; ++k) speeds[k] = 0.0;
  if (model->kind == SGWO_ADVECTION) {
    for (int k = 0; k < d; ++k) speeds[k] = fabs(model->speeds[k]);
  } else if (model->kind == SGWO_BURGERS) {
    double umax = 0.0;
    size_t off = 0;
    for (int m = 0; m < nm; ++m) {
      size_t n = sgwo_member_points(dom, lv + m * d);
      double a = max_abs(states + off, n);
      umax = (umax < a) ? a : umax;
      off += n;
    }
    for (int k = 0; k < d; ++k) speeds[k] = umax;
  } else {
    const int dxs = model->space_dim;
    for (int m = 0; m < nm; ++m)
      for (int j = 0; j < dxs; ++j) {
        double a = fmax(fabs(dom->lower[dxs + j]), fabs(dom->upper[dxs + j]));
        speeds[j] = (speeds[j] < a) ? a : speeds[j];
        if (model->kind == SGWO_VLASOV_BOLTZMANN) {
          double b = fmax(fabs(dom->lower[j]), fabs(dom->upper[j]));
          speeds[dxs + j] = (speeds[dxs + j] < b) ? b : speeds[dxs + j];
        }
      }
    if (model->kind == SGWO_VLASOV_POISSON) {
      /* family max |E_j| over members (new physics); per-member maxima in
       * parallel, folded in member order */
      size_t* offs = (size_t*)malloc(sizeof(size_t) * (size_t)nm);
      double* mx = (double*)calloc((size_t)nm * 4, sizeof(double));
      size_t off = 0;
      for (int m = 0; m < nm; ++m) {
        offs[m] = off;
        off += sgwo_member_points(dom, lv + m * d);
      }
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
      for (int m = 0; m < nm; ++m) {
        geom_t g;
        make_geom(dom, lv + m * d, &g);
        size_t vn = 1;
        for (int k = dxs; k < d; ++k) vn *= (size_t)g.points[k];
        size_t nx = g.total / vn;
        double* E = (double*)malloc(sizeof(double) * nx * (size_t)dxs);
        double* rho = (double*)malloc(sizeof(double) * nx);
        vp_field_geom(dom, &g, dxs, states + offs[m], rho, E);
        for (int j = 0; j < dxs; ++j) mx[m * 4 + j] = max_abs(E + (size_t)j * nx, nx);
        free(E);
        free(rho);
      }
      for (int m = 0; m < nm; ++m)
        for (int j = 0; j < dxs; ++j) {
          const double a = mx[m * 4 + j];
          speeds[dxs + j] = (speeds[dxs + j] < a) ? a : speeds[dxs + j];
        }
      free(offs);
      free(mx);
    }
  }
  free(lv);
  return SGWO_OK;
}

/* Per-step field-energy record of the Vlasov-Poisson evolve (new physics, the
 * device record sgwg_field_energy): ||E_c||_2 on the finest x-grid with
 * E_c = sum_m c_m I_m(E_m), I_m separable degree-4 Lagrange upsampling
 * (interp.hpp:36-53; dimension 1 first in 2D), members in order. */
double sgwo_field_energy(const sgwo_domain* dom, int space_dim, const double* states) {
  const int d = dom->d, dxs = space_dim;
  int* lv;
  int nm = family_levels(dom, &lv);
  long long coef[4];
  sgwo_combination_coefficients(d, dom->nl, coef);
  int nf[2] = {dom->root_cells[0] << dom->nl, dxs == 2 ? dom->root_cells[1] << dom->nl : 1};
  const size_t NF = (size_t)nf[0] * (size_t)nf[1];
  size_t* offs = (size_t*)malloc(sizeof(size_t) * (size_t)nm);
  size_t off = 0;
  for (int m = 0; m < nm; ++m) {
    offs[m] = off;
    off += sgwo_member_points(dom, lv + m * d);
  }
  double** fine = (double**)malloc(sizeof(double*) * (size_t)nm);
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
  for (int m = 0; m < nm; ++m) {
    geom_t g;
    make_geom(dom, lv + m * d, &g);
    size_t vn = 1;
    for (int k = dxs; k < d; ++k) vn *= (size_t)g.points[k];
    const size_t nx = g.total / vn;
    double* E = (double*)malloc(sizeof(double) * nx * (size_t)dxs);
    double* rho = (double*)malloc(sizeof(double) * nx);
    vp_field_geom(dom, &g, dxs, states + offs[m], rho, E);
    const int n0 = g.points[0], n1 = (dxs == 2) ? g.points[1] : 1;
    const int m0 = dom->nl - lv[m * d], m1 = (dxs == 2) ? dom->nl - lv[m * d + 1] : 0;
    double* out = (double*)malloc(sizeof(double) * NF * (size_t)dxs);
    double* rows = (double*)malloc(sizeof(double) * (size_t)n0 * (size_t)nf[1]);
    double* col = (double*)malloc(sizeof(double) * (size_t)(n0 > nf[0] ? n0 : nf[0]));
    double* col2 = (double*)malloc(sizeof(double) * (size_t)nf[0]);
    for (int c = 0; c < dxs; ++c) {
      const double* Ec = E + (size_t)c * nx;
      for (int i = 0; i < n0; ++i) {
        if (m1 > 0)
          sgwo_upsample_line(Ec + (size_t)i * n1, n1, rows + (size_t)i * nf[1], nf[1], m1,
                             SGWO_PERIODIC, SGWO_INTERP_LAGRANGE, 0.0);
        else
          memcpy(rows + (size_t)i * nf[1], Ec + (size_t)i * n1, sizeof(double) * (size_t)n1);
      }
      for (int j = 0; j < nf[1]; ++j) {
        for (int i = 0; i < n0; ++i) col[i] = rows[(size_t)i * nf[1] + j];
        if (m0 > 0)
          sgwo_upsample_line(col, n0, col2, nf[0], m0, SGWO_PERIODIC, SGWO_INTERP_LAGRANGE, 0.0);
        else
          memcpy(col2, col, sizeof(double) * (size_t)nf[0]);
        for (int i = 0; i < nf[0]; ++i) out[(size_t)c * NF + (size_t)i * nf[1] + j] = col2[i];
      }
    }
    free(rows);
    free(col);
    free(col2);
    free(E);
    free(rho);
    fine[m] = out;
  }
  double* acc = (double*)calloc(NF * (size_t)dxs, sizeof(double));
  for (int m = 0; m < nm; ++m) {
    int s = 0;
    for (int k = 0; k < d; ++k) s += lv[m * d + k];
    const double c = (double)coef[dom->nl - s];
    for (size_t i = 0; i < NF * (size_t)dxs; ++i) acc[i] += c * fine[m][i];
    free(fine[m]);
  }
  double hv = (dom->upper[0] - dom->lower[0]) / nf[0];
  if (dxs == 2) hv *= (dom->upper[1] - dom->lower[1]) / nf[1];
  double e = 0.0;
  for (size_t i = 0; i < NF * (size_t)dxs; ++i) e += acc[i] * acc[i];
  free(acc);
  free(fine);
  free(offs);
  free(lv);
  return sqrt(e * hv);
}

/* optional step limit of sgwo_evolve (0 = none): bounded CPU samples of a run */
static long g_max_steps = 0;
void sgwo_set_max_steps(long n) { g_max_steps = (n < 0) ? 0 : n; }

/* optional per-step energy record of sgwo_evolve (Vlasov-Poisson models) */
static double* g_energy = NULL;
static long g_energy_cap = 0;
void sgwo_set_energy_record(double* buf, long cap) {
  g_energy = buf;
  g_energy_cap = (buf != NULL) ? cap : 0;
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x < y) ? -1 : (x > y) ? 1 : 0;
}

/* timestep.hpp:126-174 */
int sgwo_evolve(const sgwo_domain* dom, const sgwo_model* model, const sgwo_policy* pol,
                double* states, double tfinal, const double* stops_in, int nstops, sgwo_stop_cb cb,
                void* user, double* dts, long cap, long* nsteps, int* fail_member,
                long* fail_step, int* fail_stage) {
  if (tfinal < 0.0) return SGWO_EINVAL;
  const int d = dom->d;
  int* lv;
  int nm = family_levels(dom, &lv);
  if (nm < 0) return SGWO_EINVAL;
  int fl[4];
  int fpts[4];
  double fsp[4];
  for (int k = 0; k < d; ++k) fl[k] = dom->nl;
  sgwo_member_geometry(dom, fl, fpts, fsp);

  const double eps_dedupe = 1e-12 * fmax(1.0, tfinal);
  double* stops = (double*)malloc(sizeof(double) * (size_t)(nstops + 1));
  int ns = 0;
  for (int i = 0; i < nstops; ++i) stops[ns++] = stops_in[i];
  stops[ns++] = tfinal;
  qsort(stops, (size_t)ns, sizeof(double), cmp_double);
  int w = 0;
  for (int i = 0; i < ns; ++i)
    if (!(stops[i] <= 0.0 || stops[i] > tfinal + eps_dedupe)) stops[w++] = stops[i];
  ns = w;
  if (ns > 0) { /* std::unique against the last kept element */
    int r = 0;
    for (int i = 1; i < ns; ++i)
      if (!(fabs(stops[r] - stops[i]) <= eps_dedupe)) stops[++r] = stops[i];
    ns = r + 1;
  }
  if (ns == 0) stops[ns++] = tfinal;

  size_t* off = (size_t*)malloc(sizeof(size_t) * (size_t)nm);
  size_t tot = 0;
  for (int m = 0; m < nm; ++m) {
    off[m] = tot;
    tot += sgwo_member_points(dom, lv + m * d);
  }
  double t = 0.0;
  long step_index = 0;
  const double eps_t = 1e-12 * fmax(1.0, tfinal);
  int status = SGWO_OK;
  for (int si = 0; si < ns && status == SGWO_OK; ++si) {
    const double stop = stops[si];
    if (stop > tfinal + eps_t) break;
    while (stop - t > eps_t) {
      if (g_max_steps > 0 && step_index >= g_max_steps) break;
      double speeds[4];
      if (g_energy != NULL && model->kind == SGWO_VLASOV_POISSON && step_index < g_energy_cap)
        g_energy[step_index] = sgwo_field_energy(dom, model->space_dim, states);
      sgwo_family_wave_speeds(dom, model, states, speeds);
      double dt = sgwo_compute_dt(pol, speeds, fsp, d, stop - t);
      if (stop - (t + dt) <= eps_t) dt = stop - t;
      int first_fail = nm, fail_code = 0;
      if (g_threads <= 1) {
        for (int m = 0; m < nm; ++m) {
          int f = sgwo_rk3_step(dom, lv + m * d, model, states + off[m], dt);
          if (f) {
            first_fail = m;
            fail_code = f;
            break;
          }
        }
      } else {
        /* members in parallel; the failure reported is the first member in
         * order (the serial loop's), later members' states are then unspecified
         * as after the reference's exception */
        int* codes = (int*)calloc((size_t)nm, sizeof(int));
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
        for (int m = 0; m < nm; ++m) codes[m] = sgwo_rk3_step(dom, lv + m * d, model, states + off[m], dt);
        for (int m = 0; m < nm; ++m)
          if (codes[m]) {
            first_fail = m;
            fail_code = codes[m];
            break;
          }
        free(codes);
      }
      if (first_fail < nm) {
        if (fail_member) *fail_member = first_fail;
        if (fail_step) *fail_step = step_index;
        if (fail_stage) *fail_stage = fail_code;
        status = SGWO_ENONFINITE;
        break;
      }
      t += dt;
      if (dts && step_index < cap) dts[step_index] = dt;
      ++step_index;
    }
    if (status != SGWO_OK) break;
    if (g_max_steps > 0 && step_index >= g_max_steps && stop - t > eps_t) break;
    t = stop;
    if (cb) cb(t, user);
  }
  if (nsteps) *nsteps = step_index;
  free(stops);
  free(off);
  free(lv);
  return status;
}

/* ------------------------------------------------------------------------ */
/* interp.hpp / combine.hpp                                                  */
/* ------------------------------------------------------------------------ */

/* interp.hpp:36-40 (and OffsetTable::cell_weights 119-122, same formulas) */
static void interp_weights(double t, double* c) {
  c[0] = (t - 1.0) * (t - 2.0) / 12.0;
  c[1] = (4.0 - t * t) / 6.0;
  c[2] = (t + 2.0) * (t + 1.0) / 12.0;
}

/* interp.hpp:45-53 */
static void substencil_values(const double* u, double t, double* p) {
  p[0] = u[0] * 0.5 * (t + 1.0) * t - u[1] * (t + 2.0) * t + u[2] * 0.5 * (t + 2.0) * (t + 1.0);
  p[1] = u[1] * 0.5 * t * (t - 1.0) - u[2] * (t + 1.0) * (t - 1.0) + u[3] * 0.5 * (t + 1.0) * t;
  p[2] = u[2] * 0.5 * (t - 1.0) * (t - 2.0) - u[3] * t * (t - 2.0) + u[4] * 0.5 * t * (t - 1.0);
}

/* interp.hpp:151-189 with OffsetTable::make (124-146) inlined */
int sgwo_upsample_line(const double* src, int n_src, double* dst, int n_dst, int m, int bc,
                       int mode, double eps) {
  const int f = 1 << m;
  int cached_i = INT32_MIN;
  double stencil[5] = {0, 0, 0, 0, 0};
  double beta[3] = {0, 0, 0};
  for (int j = 0; j < n_dst; ++j) {
    const int r = j & (f - 1);
    if (r == 0) {
      dst[j] = src[(j >> m) % n_src];
      continue;
    }
    int di;
    double t, c[3];
    if (mode == SGWO_INTERP_WENO) {
      di = (r >= f / 2) ? 1 : 0;
      t = (double)r / f - di;
    } else {
      di = 0;
      t = (double)r / f;
    }
    interp_weights(t, c);
    const int i = (j >> m) + di;
    if (i != cached_i) {
      cached_i = i;
      for (int s = 0; s < 5; ++s) {
        int q = i - 2 + s;
        if (bc == SGWO_PERIODIC)
          stencil[s] = src[((q % n_src) + n_src) % n_src];
        else
          stencil[s] = (q >= 0 && q < n_src) ? src[q] : 0.0;
      }
      if (mode == SGWO_INTERP_WENO) sgwo_smoothness_indicators(stencil, beta);
    }
    double p[3];
    substencil_values(stencil, t, p);
    if (mode == SGWO_INTERP_LAGRANGE) {
      dst[j] = c[0] * p[0] + c[1] * p[1] + c[2] * p[2];
    } else {
      const double a0 = c[0] / sqr(eps + beta[0]);
      const double a1 = c[1] / sqr(eps + beta[1]);
      const double a2 = c[2] / sqr(eps + beta[2]);
      dst[j] = (a0 * p[0] + a1 * p[1] + a2 * p[2]) / (a0 + a1 + a2);
    }
  }
  return SGWO_OK;
}

/* interp.hpp:197-250 */
int sgwo_prolong(const sgwo_domain* dom, const int* level, const double* src, int mode, double eps,
                 double* dst) {
  const int d = dom->d;
  int pts[4], tpts[4], tl[4];
  double sp[4], tsp[4];
  sgwo_member_geometry(dom, level, pts, sp);
  for (int k = 0; k < d; ++k) {
    if (level[k] > dom->nl) return SGWO_EINVAL;
    tl[k] = dom->nl;
  }
  sgwo_member_geometry(dom, tl, tpts, tsp);
  int lsum = 0;
  size_t n = 1, nt = 1;
  for (int k = 0; k < d; ++k) {
    lsum += level[k];
    n *= (size_t)pts[k];
    nt *= (size_t)tpts[k];
  }
  if (lsum == d * dom->nl) {
    memcpy(dst, src, sizeof(double) * n);
    return SGWO_OK;
  }
  int ext[4];
  for (int k = 0; k < d; ++k) ext[k] = pts[k];
  double* cur = (double*)malloc(sizeof(double) * nt);
  double* next = (double*)malloc(sizeof(double) * nt);
  memcpy(cur, src, sizeof(double) * n);
  double* sbuf = (double*)malloc(sizeof(double) * 65536);
  double* dbuf = (double*)malloc(sizeof(double) * 65536);
  for (int k = 0; k < d; ++k) {
    const int m = dom->nl - level[k];
    if (m == 0) continue;
    const int n_src = ext[k], n_dst = tpts[k];
    size_t outer = 1, inner = 1;
    for (int q = 0; q < k; ++q) outer *= (size_t)ext[q];
    for (int q = k + 1; q < d; ++q) inner *= (size_t)ext[q];
    for (size_t line = 0; line < outer * inner; ++line) {
      const size_t o = line / inner, in = line % inner;
      const double* sp2 = cur + (o * (size_t)n_src) * inner + in;
      for (int j = 0; j < n_src; ++j) sbuf[j] = sp2[(size_t)j * inner];
      sgwo_upsample_line(sbuf, n_src, dbuf, n_dst, m, dom->bc[k], mode, eps);
      double* dp = next + (o * (size_t)n_dst) * inner + in;
      for (int j = 0; j < n_dst; ++j) dp[(size_t)j * inner] = dbuf[j];
    }
    double* tmp = cur;
    cur = next;
    next = tmp;
    ext[k] = n_dst;
  }
  memcpy(dst, cur, sizeof(double) * nt);
  free(cur);
  free(next);
  free(sbuf);
  free(dbuf);
  return SGWO_OK;
}

/* One output point j of sgwo_upsample_line (interp.hpp:151-189): the same
 * OffsetTable offsets, stencil gather, smoothness indicators and expression
 * order, so the value is bitwise that of the whole-line routine. */
static double upsample_at(const double* src, int n_src, int j, int m, int bc, int mode,
                          double eps) {
  const int f = 1 << m;
  const int r = j & (f - 1);
  if (r == 0) return src[(j >> m) % n_src];
  int di;
  double t, c[3];
  if (mode == SGWO_INTERP_WENO) {
    di = (r >= f / 2) ? 1 : 0;
    t = (double)r / f - di;
  } else {
    di = 0;
    t = (double)r / f;
  }
  interp_weights(t, c);
  const int i = (j >> m) + di;
  double stencil[5], beta[3] = {0, 0, 0};
  for (int s = 0; s < 5; ++s) {
    int q = i - 2 + s;
    if (bc == SGWO_PERIODIC)
      stencil[s] = src[((q % n_src) + n_src) % n_src];
    else
      stencil[s] = (q >= 0 && q < n_src) ? src[q] : 0.0;
  }
  if (mode == SGWO_INTERP_WENO) sgwo_smoothness_indicators(stencil, beta);
  double p[3];
  substencil_values(stencil, t, p);
  if (mode == SGWO_INTERP_LAGRANGE) return c[0] * p[0] + c[1] * p[1] + c[2] * p[2];
  const double a0 = c[0] / sqr(eps + beta[0]);
  const double a1 = c[1] / sqr(eps + beta[1]);
  const double a2 = c[2] / sqr(eps + beta[2]);
  return (a0 * p[0] + a1 * p[1] + a2 * p[2]) / (a0 + a1 + a2);
}

/* source indices of a member line that the outputs [lo, hi) read (sorted, unique) */
static int needed_sources(int n_src, int m, int bc, int mode, int lo, int hi, int* out) {
  char* need = (char*)calloc((size_t)n_src, 1);
  const int f = 1 << m;
  for (int j = lo; j < hi; ++j) {
    const int r = j & (f - 1);
    if (r == 0) {
      need[(j >> m) % n_src] = 1;
      continue;
    }
    const int di = (mode == SGWO_INTERP_WENO && r >= f / 2) ? 1 : 0;
    const int i = (j >> m) + di;
    for (int s = 0; s < 5; ++s) {
      int q = i - 2 + s;
      if (bc == SGWO_PERIODIC)
        need[((q % n_src) + n_src) % n_src] = 1;
      else if (q >= 0 && q < n_src)
        need[q] = 1;
    }
  }
  int c = 0;
  for (int q = 0; q < n_src; ++q)
    if (need[q]) out[c++] = q;
  free(need);
  return c;
}

/* The combined solution (combine.hpp:95-122) on the finest-grid box
 * [lo_k, hi_k): each member prolonged (interp.hpp:197-250, dimensions in
 * order) only on the lines the box depends on, then acc += c * p in member
 * order -- bitwise the corresponding entries of sgwo_combine, at a cost
 * proportional to the box (cut planes of BASELINE C5, whose full finest grid
 * is 34.6 GB).  out: row-major over the box. */
int sgwo_combine_box(const sgwo_domain* dom, const double* states, int mode, double eps,
                     const int* lo, const int* hi, double* out) {
  const int d = dom->d;
  int* lv;
  int nm = family_levels(dom, &lv);
  if (nm <= 0) return SGWO_EINVAL;
  int fl[4], fpts[4];
  double fsp[4];
  for (int k = 0; k < d; ++k) fl[k] = dom->nl;
  sgwo_member_geometry(dom, fl, fpts, fsp);
  size_t nbox = 1;
  for (int k = 0; k < d; ++k) {
    if (lo[k] < 0 || hi[k] > fpts[k] || lo[k] >= hi[k]) {
      free(lv);
      return SGWO_EINVAL;
    }
    nbox *= (size_t)(hi[k] - lo[k]);
  }
  long long coef[4];
  sgwo_combination_coefficients(d, dom->nl, coef);
  size_t* offs = (size_t*)malloc(sizeof(size_t) * (size_t)nm);
  size_t off = 0;
  for (int m = 0; m < nm; ++m) {
    offs[m] = off;
    off += sgwo_member_points(dom, lv + m * d);
  }
  double** vals = (double**)malloc(sizeof(double*) * (size_t)nm);
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
  for (int mi = 0; mi < nm; ++mi) {
    const int* level = lv + mi * d;
    int pts[4];
    double sp[4];
    sgwo_member_geometry(dom, level, pts, sp);
    /* per dimension: the working index list (sources before the dimension is
     * processed, box outputs after) */
    int* idx[4];
    int ext[4], msh[4];
    for (int k = 0; k < d; ++k) {
      msh[k] = dom->nl - level[k];
      idx[k] = (int*)malloc(sizeof(int) * (size_t)(pts[k] > fpts[k] ? pts[k] : fpts[k]));
      ext[k] = needed_sources(pts[k], msh[k], dom->bc[k], mode, lo[k], hi[k], idx[k]);
    }
    /* gather the member sub-array */
    size_t n = 1;
    for (int k = 0; k < d; ++k) n *= (size_t)ext[k];
    double* cur = (double*)malloc(sizeof(double) * n);
    size_t mstr[4];
    mstr[d - 1] = 1;
    for (int k = d - 2; k >= 0; --k) mstr[k] = mstr[k + 1] * (size_t)pts[k + 1];
    {
      int it[4] = {0, 0, 0, 0};
      for (size_t lin = 0; lin < n; ++lin) {
        size_t src = 0;
        for (int k = 0; k < d; ++k) src += (size_t)idx[k][it[k]] * mstr[k];
        cur[lin] = states[offs[mi] + src];
        for (int k = d - 1; k >= 0; --k) {
          if (++it[k] < ext[k]) break;
          it[k] = 0;
        }
      }
    }
    int lmax = 1;
    for (int k = 0; k < d; ++k) lmax = (pts[k] > lmax) ? pts[k] : lmax;
    double* line = (double*)malloc(sizeof(double) * (size_t)lmax);
    for (int k = 0; k < d; ++k) {
      const int nb = hi[k] - lo[k];
      size_t outer = 1, inner = 1;
      for (int q = 0; q < k; ++q) outer *= (size_t)ext[q];
      for (int q = k + 1; q < d; ++q) inner *= (size_t)ext[q];
      double* next = (double*)malloc(sizeof(double) * outer * (size_t)nb * inner);
      for (size_t o = 0; o < outer; ++o)
        for (size_t in = 0; in < inner; ++in) {
          for (int q = 0; q < pts[k]; ++q) line[q] = 0.0; /* entries never read */
          for (int a = 0; a < ext[k]; ++a)
            line[idx[k][a]] = cur[(o * (size_t)ext[k] + (size_t)a) * inner + in];
          for (int b = 0; b < nb; ++b)
            next[(o * (size_t)nb + (size_t)b) * inner + in] =
                (msh[k] == 0) ? line[lo[k] + b]
                              : upsample_at(line, pts[k], lo[k] + b, msh[k], dom->bc[k], mode, eps);
        }
      free(cur);
      cur = next;
      ext[k] = nb;
    }
    vals[mi] = cur;
    free(line);
    for (int k = 0; k < d; ++k) free(idx[k]);
  }
  for (size_t i = 0; i < nbox; ++i) out[i] = 0.0;
  for (int mi = 0; mi < nm; ++mi) {
    int s = 0;
    for (int k = 0; k < d; ++k) s += lv[mi * d + k];
    const double c = (double)coef[dom->nl - s];
    for (size_t i = 0; i < nbox; ++i) out[i] += c * vals[mi][i];
    free(vals[mi]);
  }
  free(vals);
  free(offs);
  free(lv);
  return SGWO_OK;
}

/* combine.hpp:95-122 */
int sgwo_combine(const sgwo_domain* dom, const double* states, int mode, double eps, double* out) {
  const int d = dom->d;
  int* lv;
  int nm = family_levels(dom, &lv);
  if (nm <= 0) return SGWO_EINVAL;
  long long coef[4];
  sgwo_combination_coefficients(d, dom->nl, coef);
  const size_t nt = sgwo_finest_points(dom);
  memset(out, 0, sizeof(double) * nt);
  size_t* offs = (size_t*)malloc(sizeof(size_t) * (size_t)nm);
  double* cs = (double*)malloc(sizeof(double) * (size_t)nm);
  size_t off = 0;
  for (int m = 0; m < nm; ++m) {
    int s = 0;
    for (int k = 0; k < d; ++k) s += lv[m * d + k];
    cs[m] = (double)coef[dom->nl - s];
    offs[m] = off;
    off += sgwo_member_points(dom, lv + m * d);
  }
  /* batches of members prolonged in parallel, accumulated in member order
   * (acc += c * p, combine.hpp:115-120) */
  const int nb = (g_threads < nm) ? g_threads : nm;
  double** p = (double**)malloc(sizeof(double*) * (size_t)nb);
  for (int b = 0; b < nb; ++b) p[b] = (double*)malloc(sizeof(double) * nt);
  for (int m0 = 0; m0 < nm; m0 += nb) {
    const int cnt = (nm - m0 < nb) ? nm - m0 : nb;
#pragma omp parallel for schedule(dynamic, 1) num_threads(g_threads)
    for (int b = 0; b < cnt; ++b)
      sgwo_prolong(dom, lv + (m0 + b) * d, states + offs[m0 + b], mode, eps, p[b]);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (size_t i = 0; i < nt; ++i) {
      double acc = out[i];
      for (int b = 0; b < cnt; ++b) acc += cs[m0 + b] * p[b][i];
      out[i] = acc;
    }
  }
  for (int b = 0; b < nb; ++b) free(p[b]);
  free(p);
  free(offs);
  free(cs);
  free(lv);
  return SGWO_OK;
}

/* ------------------------------------------------------------------------ */
/* initial conditions: restrict_to_grid (grid.hpp:166-186)                   */
/* ------------------------------------------------------------------------ */

static double ic_eval(int preset, const double* x) {
  switch (preset) {
    case SGWO_IC_C1: return sin(M_PI * (x[0] + x[1]));
    case SGWO_IC_C2: return 0.5 + sin(M_PI * (x[0] + x[1]));
    case SGWO_IC_C3: return sin(M_PI * (x[0] + x[1] + x[2]));
    case SGWO_IC_C4:
      return (1.0 + 0.01 * cos(0.5 * x[0])) / sqrt(2.0 * M_PI) * exp(-0.5 * (x[1] * x[1]));
    case SGWO_IC_C5:
      return (1.0 + 0.05 * (cos(0.5 * x[0]) + cos(0.5 * x[1]))) / (2.0 * M_PI) *
             exp(-0.5 * (x[2] * x[2] + x[3] * x[3]));
    case SGWO_IC_EX1: return 0.3 + 0.7 * sin(0.5 * M_PI * (x[0] + x[1])); /* models.hpp:605-607 */
    case SGWO_IC_EX3: { /* models.hpp:647-651, d read from caller via x[4] sentinel */
      return 0.0;
    }
    case SGWO_IC_EX5A: { /* models.hpp:690-694 */
      const double xx = x[0], v = x[1];
      const double s = sin(0.5 * xx * xx);
      return s * s * exp(-0.5 * (xx * xx + v * v));
    }
    case SGWO_IC_EX5B: { /* models.hpp:709-714 */
      const double x1 = x[0], x2 = x[1], v1 = x[2], v2 = x[3];
      const double s = sin(0.5 * x1 * x1);
      const double c = cos(0.5 * x2 * x2);
      return s * s * c * c * exp(-0.5 * (x1 * x1 + x2 * x2 + v1 * v1 + v2 * v2));
    }
    case SGWO_IC_EX2: return 1.0 + 0.5 * sin(x[0] + x[1] + x[2]); /* models.hpp:625-627 */
  }
  return 0.0;
}

int sgwo_restrict_preset(int preset, const sgwo_domain* dom, const int* level, double* out) {
  geom_t g;
  make_geom(dom, level, &g);
  const int d = g.d;
  int idx[4] = {0, 0, 0, 0};
  double x[4];
  for (int k = 0; k < d; ++k) x[k] = dom->lower[k];
  for (size_t lin = 0; lin < g.total; ++lin) {
    double v;
    if (preset == SGWO_IC_EX3) {
      double s = 0.0;
      for (int k = 0; k < d; ++k) s += x[k];
      v = 1.0 + 0.5 * sin(s);
    } else {
      v = ic_eval(preset, x);
    }
    out[lin] = v;
    for (int k = d - 1; k >= 0; --k) {
      if (++idx[k] < g.points[k]) {
        x[k] = dom->lower[k] + idx[k] * g.spacing[k];
        break;
      }
      idx[k] = 0;
      x[k] = dom->lower[k];
    }
  }
  if (preset == SGWO_IC_EX5A || preset == SGWO_IC_EX5B) {
    /* normalize_initial (models.hpp:73-102): compensated trapezoid mass */
    double* w[4];
    for (int k = 0; k < d; ++k) {
      w[k] = (double*)malloc(sizeof(double) * (size_t)g.points[k]);
      trapezoid_weights_1d(&g, k, dom->bc[k], w[k]);
    }
    int id2[4] = {0, 0, 0, 0};
    double sum = 0.0, comp = 0.0;
    for (size_t lin = 0; lin < g.total; ++lin) {
      double wp = 1.0;
      for (int k = 0; k < d; ++k) wp *= w[k][id2[k]];
      const double term = wp * out[lin] - comp;
      const double next = sum + term;
      comp = (next - sum) - term;
      sum = next;
      for (int k = d - 1; k >= 0; --k) {
        if (++id2[k] < g.points[k]) break;
        id2[k] = 0;
      }
    }
    for (int k = 0; k < d; ++k) free(w[k]);
    if (!(sum > 0.0)) return SGWO_EINVAL;
    for (size_t lin = 0; lin < g.total; ++lin) out[lin] /= sum;
  }
  return SGWO_OK;
}

int sgwo_init_family(int preset, const sgwo_domain* dom, double* states) {
  int* lv;
  int nm = family_levels(dom, &lv);
  if (nm < 0) return SGWO_EINVAL;
  size_t off = 0;
  for (int m = 0; m < nm; ++m) {
    int st = sgwo_restrict_preset(preset, dom, lv + m * dom->d, states + off);
    if (st) {
      free(lv);
      return st;
    }
    off += sgwo_member_points(dom, lv + m * dom->d);
  }
  free(lv);
  return SGWO_OK;
}
