/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference MTNUFFT
 * path (see nus_oracle.h).  Reference paths are relative to
 * /root/reference/proj.  Compiled with -std=c11 (no FP contraction) so the
 * bin arithmetic follows the reference's IEEE operation order exactly.
 */
#include "nus_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;
#define kTwoPi (2.0 * 3.14159265358979323846)

/* ---- plan parameters ------------------------------------------------------ */

/* nufft.cpp:17-21,90-92: w = max(4, ceil(0.55 * -ln eps)) */
int64_t or_spread_width(double eps) {
  const double v = ceil(0.55 * (-log(eps)));
  int64_t w = (int64_t)v;
  return w < 4 ? 4 : w;
}

/* fft.cpp:10-14 */
int64_t or_next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

/* nufft.cpp:23-32 */
int or_centers_uniform(const double* c, int64_t n) {
  if (n < 2) return 0;
  const double df = c[1] - c[0];
  if (!(df > 0.0)) return 0;
  double max_dev = 0.0;
  for (int64_t i = 1; i < n; ++i) {
    const double d = fabs((c[i] - c[i - 1]) - df);
    if (d > max_dev) max_dev = d;
  }
  return max_dev <= 1e-9 * df;
}

/* nufft.cpp:71-89 (policy 0 auto, 1 force_fast, 2 force_direct) */
int or_select_path(int64_t n, const double* c, int64_t nc, int policy) {
  const int uni = or_centers_uniform(c, nc);
  if (policy == 1) return uni ? 1 : -1;
  if (policy == 2) return 0;
  return (uni && (uint64_t)n * (uint64_t)nc >= (1u << 14)) ? 1 : 0;
}

/* nufft.cpp:96-114 */
void or_plan_params(const double* c, int64_t nc, double eps, int oversampling, or_params* p) {
  p->n_centers = nc;
  p->spread_width = or_spread_width(eps);
  p->f0 = c[0];
  p->df = (c[nc - 1] - c[0]) / (double)(nc - 1);
  const int64_t w = p->spread_width;
  const int64_t a = (int64_t)oversampling * nc;
  const int64_t b = 4 * w + 4;
  p->mr = or_next_pow2(a > b ? a : b);
  const double ratio = (double)p->mr / (double)nc;
  p->tau = kPi * (double)w / ((double)nc * (double)nc * ratio * (ratio - 0.5));
  p->mode_offset = nc / 2;
  p->fshift = p->f0 + (double)p->mode_offset * p->df;
}

/* nufft.cpp:118-122 — the bit-exact bin contract */
void or_first_cells(const double* t, int64_t n, const or_params* p, int64_t* j0) {
  const double mr = (double)p->mr;
  for (int64_t i = 0; i < n; ++i) {
    double x = fmod(-kTwoPi * p->df * t[i], kTwoPi);
    if (x < 0.0) x += kTwoPi;
    const double cell = x * mr / kTwoPi;
    j0[i] = (int64_t)floor(cell) - p->spread_width + 1;
  }
}

/* nufft.cpp:114-117 */
void or_prephase(const double* t, int64_t n, const or_params* p, double* ph) {
  for (int64_t i = 0; i < n; ++i) {
    const double a = -kTwoPi * p->fshift * t[i];
    ph[2 * i] = cos(a);
    ph[2 * i + 1] = sin(a);
  }
}

/* ---- FFT: iterative radix-2 DIT, forward e^{-2 pi i jk/n} (fft.cpp:18-58) -- */

void or_fft(double* z, int64_t n, int inverse) {
  int64_t bits = 0;
  while (((int64_t)1 << bits) < n) ++bits;
  for (int64_t i = 0; i < n; ++i) {
    int64_t r = 0;
    for (int64_t b = 0; b < bits; ++b)
      if (i & ((int64_t)1 << b)) r |= (int64_t)1 << (bits - 1 - b);
    if (r > i) {
      double tr = z[2 * i], ti = z[2 * i + 1];
      z[2 * i] = z[2 * r];
      z[2 * i + 1] = z[2 * r + 1];
      z[2 * r] = tr;
      z[2 * r + 1] = ti;
    }
  }
  double* tw = (double*)malloc(sizeof(double) * (size_t)(n > 1 ? n : 2));
  for (int64_t j = 0; j < n / 2; ++j) {
    const double ang = -2.0 * kPi * (double)j / (double)n;
    tw[2 * j] = cos(ang);
    tw[2 * j + 1] = sin(ang);
  }
  for (int64_t len = 2; len <= n; len <<= 1) {
    const int64_t half = len >> 1, step = n / len;
    for (int64_t s = 0; s < n; s += len) {
      for (int64_t j = 0; j < half; ++j) {
        const double wr = tw[2 * j * step];
        const double wi = inverse ? -tw[2 * j * step + 1] : tw[2 * j * step + 1];
        double* u = z + 2 * (s + j);
        double* v = z + 2 * (s + j + half);
        const double vr = v[0] * wr - v[1] * wi;
        const double vi = v[0] * wi + v[1] * wr;
        v[0] = u[0] - vr;
        v[1] = u[1] - vi;
        u[0] += vr;
        u[1] += vi;
      }
    }
  }
  free(tw);
}

/* ---- NUFFT ----------------------------------------------------------------- */

/* nufft.cpp:96-166: Gaussian gridding onto Mr cells, FFT, deconvolve + crop */
void or_nufft_fast(const double* t, int64_t n, const double* c, int64_t nc, double eps,
                   int oversampling, const double* y, double* out) {
  or_params p;
  or_plan_params(c, nc, eps, oversampling, &p);
  const int64_t w = p.spread_width, w2 = 2 * w, mr = p.mr;
  double* b = (double*)calloc((size_t)(2 * mr), sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    const double a = -kTwoPi * p.fshift * t[i];
    const double pr = cos(a), pi = sin(a);
    double x = fmod(-kTwoPi * p.df * t[i], kTwoPi);
    if (x < 0.0) x += kTwoPi;
    const double cell = x * (double)mr / kTwoPi;
    const int64_t j0 = (int64_t)floor(cell) - w + 1;
    const double zr = y[2 * i] * pr - y[2 * i + 1] * pi;
    const double zi = y[2 * i] * pi + y[2 * i + 1] * pr;
    int64_t s = j0 % mr;
    if (s < 0) s += mr;
    for (int64_t q = 0; q < w2; ++q) {
      const double xi = kTwoPi * (double)(j0 + q) / (double)mr;
      const double dxr = x - xi;
      const double g = exp(-dxr * dxr / (4.0 * p.tau));
      int64_t cidx = s + q;
      if (cidx >= mr) cidx -= mr;
      b[2 * cidx] += g * zr;
      b[2 * cidx + 1] += g * zi;
    }
  }
  or_fft(b, mr, 0);
  const double norm = sqrt(kPi / p.tau) / (double)mr;
  for (int64_t i = 0; i < nc; ++i) {
    const int64_t m = i - p.mode_offset;
    int64_t bin = (-m) % mr;
    if (bin < 0) bin += mr;
    const double d = norm * exp(p.tau * (double)m * (double)m);
    out[2 * i] = d * b[2 * bin];
    out[2 * i + 1] = d * b[2 * bin + 1];
  }
  free(b);
}

/* nufft.cpp:36-54 */
void or_ndft_direct(const double* t, int64_t n, const double* y, const double* c, int64_t nc,
                    double* out) {
  for (int64_t i = 0; i < nc; ++i) {
    const double f = c[i];
    double ar = 0.0, ai = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double ph = -kTwoPi * f * t[k];
      const double cr = cos(ph), ci = sin(ph);
      ar += y[2 * k] * cr - y[2 * k + 1] * ci;
      ai += y[2 * k] * ci + y[2 * k + 1] * cr;
    }
    out[2 * i] = ar;
    out[2 * i + 1] = ai;
  }
}

/* nufft.cpp:194-227 (real tapers): row k = transform of w_k * x */
int or_eigencoefficients(const double* t, int64_t n, const double* w, int64_t k, const double* x,
                         const double* c, int64_t nc, double eps, int policy, double* out) {
  const int path = or_select_path(n, c, nc, policy);
  if (path < 0) return 1;
  double* y = (double*)malloc(sizeof(double) * (size_t)(2 * n));
  for (int64_t j = 0; j < k; ++j) {
    for (int64_t i = 0; i < n; ++i) {
      y[2 * i] = w[j * n + i] * x[i];
      y[2 * i + 1] = 0.0;
    }
    if (path == 1)
      or_nufft_fast(t, n, c, nc, eps, 2, y, out + 2 * j * nc);
    else
      or_ndft_direct(t, n, y, c, nc, out + 2 * j * nc);
  }
  free(y);
  return 0;
}

/* estimators.cpp:106-122: P_i = (1/K) sum_k |J_k(i)|^2, k-outer accumulation */
int or_mtnufft_power(const double* t, int64_t n, const double* w, int64_t k, const double* x,
                     const double* c, int64_t nc, double eps, int policy, double* power) {
  double* row = (double*)malloc(sizeof(double) * (size_t)(2 * nc));
  const int path = or_select_path(n, c, nc, policy);
  if (path < 0) {
    free(row);
    return 1;
  }
  double* y = (double*)malloc(sizeof(double) * (size_t)(2 * n));
  for (int64_t i = 0; i < nc; ++i) power[i] = 0.0;
  for (int64_t j = 0; j < k; ++j) {
    for (int64_t i = 0; i < n; ++i) {
      y[2 * i] = w[j * n + i] * x[i];
      y[2 * i + 1] = 0.0;
    }
    if (path == 1)
      or_nufft_fast(t, n, c, nc, eps, 2, y, row);
    else
      or_ndft_direct(t, n, y, c, nc, row);
    for (int64_t i = 0; i < nc; ++i) power[i] += row[2 * i] * row[2 * i] + row[2 * i + 1] * row[2 * i + 1];
  }
  for (int64_t i = 0; i < nc; ++i) power[i] /= (double)k;
  free(y);
  free(row);
  return 0;
}

/* ---- DPSS: top-K eigenpairs of the commuting tridiagonal ------------------
 * Matrix entries exactly as tapers.cpp:40-52 (fp64).  The eigen-solve is an
 * independent algorithm on purpose (the reference uses all-eigenvalue QL,
 * eig.cpp:21-91, which is O(N^2)): long-double Sturm bisection for the
 * eigenvalues, then long-double inverse iteration with partial pivoting (the
 * solve structure of eig.cpp:119-168).  Conventions follow eig.cpp:281-289
 * (largest-|v| entry positive) and unit 2-norm.
 */

typedef long double ld;

/* number of eigenvalues strictly below lam (Sturm count via LDL^T pivots) */
static int64_t sturm_count(const double* d, const ld* e2, int64_t n, ld lam, ld pivmin) {
  int64_t cnt = 0;
  ld q = (ld)d[0] - lam;
  if (fabsl(q) < pivmin) q = -pivmin;
  if (q < 0) ++cnt;
  for (int64_t i = 1; i < n; ++i) {
    q = ((ld)d[i] - lam) - e2[i - 1] / q;
    if (fabsl(q) < pivmin) q = -pivmin;
    if (q < 0) ++cnt;
  }
  return cnt;
}

static void tridiag_solve_ld(const double* d, const double* e, int64_t n, ld lam, ld* x, ld pivmin,
                             ld* u0, ld* u1, ld* u2) {
  if (n == 1) {
    ld p = (ld)d[0] - lam;
    if (fabsl(p) < pivmin) p = p < 0 ? -pivmin : pivmin;
    x[0] /= p;
    return;
  }
  ld c0 = (ld)d[0] - lam, c1 = (ld)e[0], c2 = 0;
  for (int64_t i = 0; i + 1 < n; ++i) {
    const ld sub = e[i];
    const ld dd = (ld)d[i + 1] - lam;
    const ld sup = (i + 2 < n) ? (ld)e[i + 1] : 0;
    if (fabsl(sub) > fabsl(c0)) {
      u0[i] = sub;
      u1[i] = dd;
      u2[i] = sup;
      const ld m = c0 / sub;
      const ld tmp = x[i];
      x[i] = x[i + 1];
      x[i + 1] = tmp - m * x[i];
      c0 = c1 - m * dd;
      c1 = c2 - m * sup;
      c2 = 0;
    } else {
      if (fabsl(c0) < pivmin) c0 = c0 < 0 ? -pivmin : pivmin;
      u0[i] = c0;
      u1[i] = c1;
      u2[i] = c2;
      const ld m = sub / c0;
      x[i + 1] -= m * x[i];
      c0 = dd - m * c1;
      c1 = sup - m * c2;
      c2 = 0;
    }
  }
  if (fabsl(c0) < pivmin) c0 = c0 < 0 ? -pivmin : pivmin;
  u0[n - 1] = c0;
  x[n - 1] /= u0[n - 1];
  x[n - 2] = (x[n - 2] - u1[n - 2] * x[n - 1]) / u0[n - 2];
  for (int64_t i = n - 2; i-- > 0;) x[i] = (x[i] - u1[i] * x[i + 1] - u2[i] * x[i + 2]) / u0[i];
}

typedef struct {
  const double* d;
  const double* e;
  const ld* e2;
  int64_t n, k, j;
  ld lo, hi, anorm;
  double* values;
  double* vectors;
} eig_job;

static void* eig_worker(void* arg) {
  eig_job* jb = (eig_job*)arg;
  const int64_t n = jb->n, j = jb->j;
  const ld pivmin = jb->anorm * (ld)LDBL_EPSILON * 1e-3L;
  /* eigenvalue with descending rank j == ascending index n-1-j */
  const int64_t idx = n - 1 - j;
  ld lo = jb->lo, hi = jb->hi;
  for (int it = 0; it < 400; ++it) {
    const ld mid = 0.5L * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(jb->d, jb->e2, n, mid, pivmin) > idx)
      hi = mid;
    else
      lo = mid;
  }
  const ld lam = 0.5L * (lo + hi);
  jb->values[j] = (double)lam;
  if (!jb->vectors) return NULL;
  ld* x = (ld*)malloc(sizeof(ld) * (size_t)n * 4);
  ld* u0 = x + n;
  ld* u1 = u0 + n;
  ld* u2 = u1 + n;
  uint64_t s = 0x9E3779B97F4A7C15ull * (uint64_t)(j + 1) + 0x2545F4914F6CDD1Dull;
  for (int64_t i = 0; i < n; ++i) {
    s ^= s >> 30;
    s *= 0xBF58476D1CE4E5B9ull;
    s ^= s >> 27;
    s *= 0x94D049BB133111EBull;
    s ^= s >> 31;
    x[i] = (ld)(s >> 11) / 9007199254740992.0L - 0.5L;
  }
  /* shift just outside the eigenvalue so the factorization stays nonsingular */
  const ld shift = lam + jb->anorm * (ld)LDBL_EPSILON * 4.0L;
  for (int it = 0; it < 4; ++it) {
    tridiag_solve_ld(jb->d, jb->e, n, shift, x, pivmin, u0, u1, u2);
    ld nrm = 0;
    for (int64_t i = 0; i < n; ++i) nrm += x[i] * x[i];
    nrm = sqrtl(nrm);
    for (int64_t i = 0; i < n; ++i) x[i] /= nrm;
  }
  int64_t imax = 0;
  for (int64_t i = 1; i < n; ++i)
    if (fabsl(x[i]) > fabsl(x[imax])) imax = i;
  const ld sg = x[imax] < 0 ? -1.0L : 1.0L;
  for (int64_t i = 0; i < n; ++i) jb->vectors[j * n + i] = (double)(sg * x[i]);
  free(x);
  return NULL;
}

int or_tridiag_top(const double* d, const double* e, int64_t n, int64_t k, double* values,
                   double* vectors, int threads) {
  if (k < 1 || k > n) return 1;
  ld* e2 = (ld*)malloc(sizeof(ld) * (size_t)(n > 1 ? n - 1 : 1));
  ld lo = 0, hi = 0, anorm = 0;
  for (int64_t i = 0; i < n; ++i) {
    ld r = fabsl((ld)d[i]);
    if (i > 0) r += fabsl((ld)e[i - 1]);
    if (i + 1 < n) r += fabsl((ld)e[i]);
    const ld a = (ld)d[i] - (r - fabsl((ld)d[i])), b = (ld)d[i] + (r - fabsl((ld)d[i]));
    if (i == 0 || a < lo) lo = a;
    if (i == 0 || b > hi) hi = b;
    if (r > anorm) anorm = r;
  }
  for (int64_t i = 0; i + 1 < n; ++i) e2[i] = (ld)e[i] * (ld)e[i];
  if (anorm <= 0) anorm = 1;
  lo -= anorm * 1e-12L + 1e-300L;
  hi += anorm * 1e-12L + 1e-300L;
  eig_job* jobs = (eig_job*)calloc((size_t)k, sizeof(eig_job));
  for (int64_t j = 0; j < k; ++j) {
    eig_job v = {d, e, e2, n, k, j, lo, hi, anorm, values, vectors};
    jobs[j] = v;
  }
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)calloc((size_t)k, sizeof(pthread_t));
  for (int64_t base = 0; base < k; base += threads) {
    int64_t end = base + threads < k ? base + threads : k;
    for (int64_t j = base; j < end; ++j) pthread_create(&th[j], NULL, eig_worker, &jobs[j]);
    for (int64_t j = base; j < end; ++j) pthread_join(th[j], NULL);
  }
  free(th);
  free(jobs);
  free(e2);
  return 0;
}

/* tapers.cpp:31-60: validation + commuting tridiagonal entries */
int or_dpss(int64_t n, double tw, int64_t k, double* tapers, double* eigenvalues, int threads) {
  if (n < 2) return 1;
  if (k < 1 || k > n) return 1;
  if (!(tw > 0.0) || !(tw < (double)n / 2.0)) return 1;
  const double w = tw / (double)n;
  double* d = (double*)malloc(sizeof(double) * (size_t)n);
  double* e = (double*)malloc(sizeof(double) * (size_t)n);
  const double c = cos(2.0 * kPi * w);
  for (int64_t m = 0; m < n; ++m) {
    const double half = ((double)n - 1.0 - 2.0 * (double)m) / 2.0;
    d[m] = half * half * c;
  }
  for (int64_t m = 1; m < n; ++m) e[m - 1] = (double)m * (double)(n - m) / 2.0;
  double* vals = eigenvalues ? eigenvalues : (double*)malloc(sizeof(double) * (size_t)k);
  const int rc = or_tridiag_top(d, e, n, k, vals, tapers, threads);
  if (!eigenvalues) free(vals);
  free(d);
  free(e);
  return rc;
}

/* ---- cubic spline, not-a-knot (eig.cpp:671-745) ---------------------------- */

typedef struct {
  const double* x;
  const double* y;
  double* m;
  int64_t n;
} spline_t;

static int spline_build(spline_t* s) {
  const int64_t n = s->n;
  if (n < 4) return 1;
  for (int64_t i = 1; i < n; ++i)
    if (!(s->x[i] > s->x[i - 1])) return 1;
  double* h = (double*)malloc(sizeof(double) * (size_t)(n - 1));
  for (int64_t i = 0; i + 1 < n; ++i) h[i] = s->x[i + 1] - s->x[i];
  const int64_t m = n - 2;
  double* sub = (double*)calloc((size_t)m, sizeof(double));
  double* dia = (double*)calloc((size_t)m, sizeof(double));
  double* sup = (double*)calloc((size_t)m, sizeof(double));
  double* rhs = (double*)calloc((size_t)m, sizeof(double));
  const double* y = s->y;
  for (int64_t i = 1; i + 1 < n; ++i) {
    const int64_t r = i - 1;
    sub[r] = h[i - 1] / 6.0;
    dia[r] = (h[i - 1] + h[i]) / 3.0;
    sup[r] = h[i] / 6.0;
    rhs[r] = (y[i + 1] - y[i]) / h[i] - (y[i] - y[i - 1]) / h[i - 1];
  }
  {
    const double r01 = h[0] / h[1];
    dia[0] += sub[0] * (1.0 + r01);
    sup[0] -= sub[0] * r01;
    sub[0] = 0.0;
  }
  {
    const double rr = h[n - 2] / h[n - 3];
    dia[m - 1] += sup[m - 1] * (1.0 + rr);
    sub[m - 1] -= sup[m - 1] * rr;
    sup[m - 1] = 0.0;
  }
  for (int64_t r = 1; r < m; ++r) {
    const double w = sub[r] / dia[r - 1];
    dia[r] -= w * sup[r - 1];
    rhs[r] -= w * rhs[r - 1];
  }
  double* mm = s->m;
  mm[m] = rhs[m - 1] / dia[m - 1];
  for (int64_t r = m - 1; r-- > 0;) mm[r + 1] = (rhs[r] - sup[r] * mm[r + 2]) / dia[r];
  mm[0] = mm[1] * (1.0 + h[0] / h[1]) - mm[2] * (h[0] / h[1]);
  mm[n - 1] = mm[n - 2] * (1.0 + h[n - 2] / h[n - 3]) - mm[n - 3] * (h[n - 2] / h[n - 3]);
  free(h);
  free(sub);
  free(dia);
  free(sup);
  free(rhs);
  return 0;
}

static int spline_eval(const spline_t* s, double xv, double* out) {
  const int64_t n = s->n;
  const double* x = s->x;
  const double glo = 0.5 * (x[1] - x[0]), ghi = 0.5 * (x[n - 1] - x[n - 2]);
  if (xv < x[0] - glo || xv > x[n - 1] + ghi) return 2;
  double xc = xv < x[0] ? x[0] : xv;
  if (xc > x[n - 1]) xc = x[n - 1];
  /* upper_bound */
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (x[mid] <= xc) lo = mid + 1; else hi = mid;
  }
  int64_t i = lo;
  if (i > 0) --i;
  if (i + 1 >= n) i = n - 2;
  const double hl = x[i + 1] - x[i];
  const double a = (x[i + 1] - xc) / hl;
  const double b = (xc - x[i]) / hl;
  *out = a * s->y[i] + b * s->y[i + 1] +
         ((a * a * a - a) * s->m[i] + (b * b * b - b) * s->m[i + 1]) * (hl * hl) / 6.0;
  return 0;
}

int or_spline(const double* xk, const double* yk, int64_t n, const double* xq, int64_t nq,
              double* out) {
  spline_t s = {xk, yk, NULL, n};
  if (n < 4) return 1;
  s.m = (double*)malloc(sizeof(double) * (size_t)n);
  int rc = spline_build(&s);
  for (int64_t i = 0; rc == 0 && i < nq; ++i) rc = spline_eval(&s, xq[i], out + i);
  free(s.m);
  return rc;
}

/* ---- R(B) quadratic form (kernels.cpp:16-19, 28-37, 100-115) --------------
 * q_k = sum_r w_r sum_c R_rc w_c with R_rc = sin(2 pi F d)/(pi d), d = t_r - t_c,
 * and 2F on the diagonal / at |d| < 1e-12 mean_dt.  Exact double sum without the
 * dense matrix; rows split across threads.
 */
typedef struct {
  const double* t;
  const double* w;
  int64_t n, k, r0, r1;
  double f_max, tol;
  double* acc;
} qf_job;

static void* qf_worker(void* arg) {
  qf_job* j = (qf_job*)arg;
  const double* t = j->t;
  for (int64_t kk = 0; kk < j->k; ++kk) j->acc[kk] = 0.0;
  double* row = (double*)malloc(sizeof(double) * (size_t)j->k);
  for (int64_t r = j->r0; r < j->r1; ++r) {
    for (int64_t kk = 0; kk < j->k; ++kk) row[kk] = 0.0;
    for (int64_t c = 0; c < j->n; ++c) {
      double v;
      if (c == r) {
        v = 2.0 * j->f_max;
      } else {
        const double d = t[r] - t[c];
        v = fabs(d) < j->tol ? 2.0 * j->f_max : sin(2.0 * kPi * j->f_max * d) / (kPi * d);
      }
      for (int64_t kk = 0; kk < j->k; ++kk) row[kk] += v * j->w[kk * j->n + c];
    }
    for (int64_t kk = 0; kk < j->k; ++kk) j->acc[kk] += j->w[kk * j->n + r] * row[kk];
  }
  free(row);
  return NULL;
}

void or_signal_band_quadform(const double* t, int64_t n, double f_max, const double* w, int64_t k,
                             double* q, int threads) {
  const double mean_dt = (t[n - 1] - t[0]) / (double)n;
  if (threads < 1) threads = 1;
  if (threads > n) threads = (int)n;
  qf_job* jobs = (qf_job*)calloc((size_t)threads, sizeof(qf_job));
  double* acc = (double*)calloc((size_t)threads * (size_t)k, sizeof(double));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int i = 0; i < threads; ++i) {
    qf_job v = {t, w, n, k, n * i / threads, n * (i + 1) / threads, f_max, 1e-12 * mean_dt,
                acc + (size_t)i * k};
    jobs[i] = v;
    pthread_create(&th[i], NULL, qf_worker, &jobs[i]);
  }
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  for (int64_t kk = 0; kk < k; ++kk) {
    double s = 0.0;
    for (int i = 0; i < threads; ++i) s += acc[(size_t)i * k + kk];
    q[kk] = s;
  }
  free(th);
  free(acc);
  free(jobs);
}

/* tapers.cpp:146-182: DPSS on span/(N-1) knots, spline to t_n, R(B) normalise.
 * Returns 3 for BandRangeError-type failures, 1 for invalid arguments. */
int or_gpss_interpolated(const double* t, int64_t n, double f_max, double f_w, int64_t k,
                         double* weights, double* q_out, int threads) {
  if (n < 8) return 1;
  if (!(f_w > 0.0)) return 1;
  if (!(f_w <= f_max + 1e-12 * f_max)) return 3;
  const double h = (t[n - 1] - t[0]) / (double)(n - 1);
  const double tw = f_w * h * (double)n;
  if (!(tw < (double)n / 2.0)) return 1;
  double* dp = (double*)malloc(sizeof(double) * (size_t)(n * k));
  int rc = or_dpss(n, tw, k, dp, NULL, threads);
  if (rc) {
    free(dp);
    return rc;
  }
  double* knots = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) knots[i] = t[0] + h * (double)i;
  for (int64_t j = 0; j < k && rc == 0; ++j) rc = or_spline(knots, dp + j * n, n, t, n, weights + j * n);
  double* q = (double*)malloc(sizeof(double) * (size_t)k);
  if (rc == 0) or_signal_band_quadform(t, n, f_max, weights, k, q, threads);
  for (int64_t j = 0; j < k && rc == 0; ++j) {
    if (!(q[j] > 0.0)) {
      rc = 5;
      break;
    }
    const double s = sqrt(2.0 * f_w / q[j]);
    for (int64_t i = 0; i < n; ++i) weights[j * n + i] *= s;
    if (q_out) q_out[j] = q[j];
  }
  free(q);
  free(knots);
  free(dp);
  return rc;
}
