/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference MTNUFFT path.
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load liboracle.so.  Every function
 * restates the reference algorithm and cites the reference file:line it follows
 * (paths relative to /root/reference/proj).  The restatement is pinned against
 * the reference itself (oracle/_ref/libnusref.so, compiled from the reference
 * sources) by tests/test_oracle_pin.py and against the committed golden
 * fixtures in tests/golden/.
 */
#ifndef NUS_ORACLE_H
#define NUS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n_centers;     /* I */
  int64_t spread_width;  /* w (nufft.cpp:90-92) */
  int64_t mr;            /* oversampled grid size (nufft.cpp:103-104) */
  int64_t mode_offset;   /* I/2 (nufft.cpp:109) */
  double f0, df, tau, fshift;
} or_params;

int64_t or_spread_width(double eps);
int64_t or_next_pow2(int64_t n);
int or_centers_uniform(const double* c, int64_t n);
/* 1 = fast, 0 = direct; -1 = force_fast on non-uniform centres (reference throws) */
int or_select_path(int64_t n, const double* c, int64_t nc, int policy);
void or_plan_params(const double* c, int64_t nc, double eps, int oversampling, or_params* p);
void or_first_cells(const double* t, int64_t n, const or_params* p, int64_t* j0);
void or_prephase(const double* t, int64_t n, const or_params* p, double* ph /* 2n */);
void or_fft(double* z, int64_t n, int inverse);
void or_nufft_fast(const double* t, int64_t n, const double* c, int64_t nc, double eps,
                   int oversampling, const double* y, double* out);
void or_ndft_direct(const double* t, int64_t n, const double* y, const double* c, int64_t nc,
                    double* out);
int or_eigencoefficients(const double* t, int64_t n, const double* w, int64_t k, const double* x,
                         const double* c, int64_t nc, double eps, int policy, double* out);
int or_mtnufft_power(const double* t, int64_t n, const double* w, int64_t k, const double* x,
                     const double* c, int64_t nc, double eps, int policy, double* power);
int or_dpss(int64_t n, double tw, int64_t k, double* tapers, double* eigenvalues, int threads);
int or_tridiag_top(const double* d, const double* e, int64_t n, int64_t k, double* values,
                   double* vectors, int threads);
int or_spline(const double* xk, const double* yk, int64_t n, const double* xq, int64_t nq,
              double* out);
void or_signal_band_quadform(const double* t, int64_t n, double f_max, const double* w, int64_t k,
                             double* q, int threads);
int or_gpss_interpolated(const double* t, int64_t n, double f_max, double f_w, int64_t k,
                         double* weights, double* q_out, int threads);

#ifdef __cplusplus
}
#endif
#endif
