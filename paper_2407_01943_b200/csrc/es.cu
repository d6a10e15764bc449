// Exponential-of-semicircle ("ES") spreading kernel: host-side parameters, the per-cell
// polynomial weights the spread evaluates, and the quadrature of its Fourier transform used
// for the deconvolution.  The reference spreads with a Gaussian of 2w cells
// (src/nufft.cpp:90-92, :122-126) and deconvolves by sqrt(pi/tau)/Mr e^{tau m^2}
// (src/nufft.cpp:139); this kernel keeps the reference's grid (Mr), bins (j0, nufft.cpp:118-121),
// phases and crop and only changes the window: phi(z) = exp(beta (sqrt(1 - z^2) - 1)) on
// ns cells, which reaches the reference's error contract max|fast - direct| <= eps ||y||_1
// (tests/test_nufft.cpp:81-96) with ns ~ log10(10/eps) instead of 2w ~ 1.1 ln(1/eps) cells.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "nus_internal.cuh"

namespace nus {

namespace {

int initial_kernel() {
  const char* e = std::getenv("NUS_KERNEL");
  if (e && std::strcmp(e, "gaussian") == 0) return NUS_KERNEL_GAUSSIAN;
  return NUS_KERNEL_ES;
}

std::atomic<int> g_kernel{initial_kernel()};

long double es_phi(long double z, long double beta) {
  if (std::fabs(z) > 1.0L) return 0.0L;
  return std::exp(beta * (std::sqrt(1.0L - z * z) - 1.0L));
}

}  // namespace

int default_kernel() { return g_kernel.load(); }
void set_default_kernel(int kind) { g_kernel.store(kind); }

int es_width(double eps) {
  // ns = ceil(log10(10 / eps)) rounded up to even (support centred on the bin: ns/2 cells
  // either side), 4 <= ns <= 16
  int ns = static_cast<int>(std::ceil(std::log10(10.0 / eps) - 1e-12));
  ns += ns & 1;
  return std::min(kEsMaxNs, std::max(kEsMinNs, ns));
}

void es_fit(int ns, double* out) {
  // Chebyshev interpolation at D + 1 Chebyshev points of s in [-1, 1] (fr = (s + 1) / 2), then
  // conversion to monomials in s; long double throughout.  Cell p of a point at cell position
  // b0 + fr (b0 = floor) is b0 - ns/2 + 1 + p, at distance u = p - ns/2 + 1 - fr.
  const int D = es_degree(ns);
  const long double beta = es_beta(ns);
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<long double> s(D + 1), cheb(D + 1), mono(D + 1);
  std::vector<std::vector<long double>> T(D + 1, std::vector<long double>(D + 1, 0.0L));
  T[0][0] = 1.0L;
  if (D >= 1) T[1][1] = 1.0L;
  for (int j = 2; j <= D; ++j)
    for (int d = 0; d <= j; ++d)
      T[j][d] = (d > 0 ? 2.0L * T[j - 1][d - 1] : 0.0L) - T[j - 2][d];
  for (int k = 0; k <= D; ++k) s[k] = std::cos(pi * (k + 0.5L) / (D + 1));
  for (int p = 0; p < ns; ++p) {
    std::vector<long double> f(D + 1);
    for (int k = 0; k <= D; ++k) {
      const long double fr = 0.5L * (s[k] + 1.0L);
      const long double u = static_cast<long double>(p) - 0.5L * ns + 1.0L - fr;
      f[k] = es_phi(2.0L * u / ns, beta);
    }
    for (int j = 0; j <= D; ++j) {
      long double a = 0.0L;
      for (int k = 0; k <= D; ++k) a += f[k] * std::cos(pi * j * (k + 0.5L) / (D + 1));
      cheb[j] = a * 2.0L / (D + 1) * (j == 0 ? 0.5L : 1.0L);
    }
    std::fill(mono.begin(), mono.end(), 0.0L);
    for (int j = 0; j <= D; ++j)
      for (int d = 0; d <= j; ++d) mono[d] += cheb[j] * T[j][d];
    for (int d = 0; d <= D; ++d) out[p * (D + 1) + d] = static_cast<double>(mono[d]);
  }
}

void es_quadrature(int ns, int nq, double* pairs) {
  // Gauss-Legendre nodes on [-1, 1] by Newton on P_nq, mapped to th in [0, pi/2]
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double beta = es_beta(ns);
  for (int i = 0; i < nq; ++i) {
    long double x = std::cos(pi * (i + 0.75L) / (nq + 0.5L)), dp = 1.0L;
    for (int it = 0; it < 100; ++it) {
      long double p0 = 1.0L, p1 = x;
      for (int k = 2; k <= nq; ++k) {
        const long double p2 = ((2.0L * k - 1.0L) * x * p1 - (k - 1.0L) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = nq * (x * p1 - p0) / (x * x - 1.0L);
      const long double dx = p1 / dp;
      x -= dx;
      if (std::fabs(dx) < 1e-19L) break;
    }
    long double p0 = 1.0L, p1 = x;
    for (int k = 2; k <= nq; ++k) {
      const long double p2 = ((2.0L * k - 1.0L) * x * p1 - (k - 1.0L) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    dp = nq * (x * p1 - p0) / (x * x - 1.0L);
    const long double w = 2.0L / ((1.0L - x * x) * dp * dp);
    const long double th = (x + 1.0L) * pi / 4.0L, wt = w * pi / 4.0L;
    pairs[2 * i] = static_cast<double>(std::sin(th));
    pairs[2 * i + 1] = static_cast<double>(wt * std::exp(beta * (std::cos(th) - 1.0L)) * std::cos(th));
  }
}

}  // namespace nus
