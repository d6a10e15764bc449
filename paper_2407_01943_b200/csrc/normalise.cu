// O(N log N) evaluation of the taper normalisation  q = w^T R(B) w  (src/tapers.cpp:167-179,
// src/kernels.cpp:16-19,28-37,100-115) for grids where the reference's dense O(N^2) form is
// out of reach (C4: N = 2^26).
//
//   q = sum_nm w_n w_m sin(2 pi F (t_n - t_m)) / (pi (t_n - t_m))      (diagonal 2F)
//     = int_{-F}^{F} |W(f)|^2 df,   W(f) = sum_n w_n e^{-2 pi i f t_n}.
//
// |W|^2 has Fourier support |tau| <= T1 = t_max - t_min, so the indicator of [-F, F] may be
// replaced by any window h whose transform equals the indicator's on [-T1, T1]:
//   h = 1_[-F,F] * psi,   psi(f) = sin(2 pi T' f) / (pi f) e^{-pi^2 s^2 f^2},
//   psi^(tau) = (erf((tau + T')/s) - erf((tau - T')/s)) / 2,   s = T1 / 12, T' = T1 + 6 s,
// (psi^ = 1 - O(e^{-36}) on [-T1, T1], support |tau| <~ 2 T1).  h is smooth, so by Poisson
// summation q = delta sum_j h(j delta) |W(j delta)|^2 exactly once 1/delta >= 3 T1 (no alias of
// the +-2 T1 support onto [-T1, T1]).  h(f) = S(f + F) - S(f - F) with S(x) = int_0^x psi, which
// is +-1/2 to 1e-17 beyond x0 = 6.2 / (pi s): h is 1 inside, 0 outside and tabulated (long
// double quadrature on the host) on the ~140 lattice points within x0 of the band edge.
//
// The lattice values W_k(j delta), j = 0 .. J, come from the path's own type-1 NUFFT: one plan
// with uniform centres i delta (i < Ic), chunk c of the lattice being the same plan applied to
// x_c(t) = e^{-2 pi i c Ic delta t} (phase in double-double), all K tapers per spread.
#include <algorithm>
#include <cmath>
#include <vector>

#include "nus_internal.cuh"

namespace nus {

namespace {

// x_c(t) = exp(-2 pi i F t) with the product F t formed exactly (two-product) and reduced mod 1
__global__ void chunk_phase_kernel(const double* __restrict__ t, int64_t n, double f, double2* __restrict__ x) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double p = f * t[i];
  const double e = fma(f, t[i], -p);
  const double r = (p - rint(p)) + e;  // cycles, |r| <= 1/2 + tiny
  double sn, cs;
  sincospi(2.0 * r, &sn, &cs);
  x[i] = double2{cs, -sn};
}

__global__ void permute_rows_kernel(const double* __restrict__ w_time, const int32_t* __restrict__ perm,
                                    int64_t n, int64_t k, double* __restrict__ w_sorted) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * k) return;
  const int64_t r = g / n, i = g - r * n;
  w_sorted[g] = w_time[r * n + perm[i]];
}

// per taper k: partial[k][block] = sum_i h(j0 + i) |J_k(i)|^2 (x2 for j > 0: |W(-f)| = |W(f)|)
constexpr int kRedThreads = 256;
__global__ void __launch_bounds__(kRedThreads) weighted_energy_kernel(
    const double2* __restrict__ jk, int64_t ic, int64_t j0, int64_t jmax, int64_t jlo,
    const double* __restrict__ edge, int64_t nedge, double* __restrict__ partial) {
  const int k = blockIdx.y;
  const double2* row = jk + static_cast<int64_t>(k) * ic;
  double acc = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRedThreads) + threadIdx.x; i < ic;
       i += static_cast<int64_t>(gridDim.x) * kRedThreads) {
    const int64_t j = j0 + i;
    if (j > jmax) break;
    const double h = j <= jlo ? 1.0 : (j - jlo - 1 < nedge ? edge[j - jlo - 1] : 0.0);
    const double2 v = row[i];
    acc += (j == 0 ? 1.0 : 2.0) * h * (v.x * v.x + v.y * v.y);
  }
  __shared__ double red[kRedThreads];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = kRedThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[static_cast<int64_t>(k) * gridDim.x + blockIdx.x] = red[0];
}

unsigned nblocks(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

// S(x) = int_0^x psi(u) du, psi(u) = sin(2 pi T' u) / (pi u) e^{-pi^2 s^2 u^2}; composite
// Gauss-Legendre (16 nodes per quarter period of the sine), +-1/2 beyond x0
long double window_cdf(long double x, long double tp, long double s, long double x0,
                       const std::vector<long double>& gx, const std::vector<long double>& gw) {
  if (x >= x0) return 0.5L;
  if (x <= -x0) return -0.5L;
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double ax = std::fabs(x);
  const long double panel = 1.0L / (4.0L * tp);
  const int64_t np = std::max<int64_t>(1, static_cast<int64_t>(std::ceil(ax / panel)));
  const long double hw = ax / (2.0L * np);
  long double sum = 0.0L;
  for (int64_t p = 0; p < np; ++p) {
    const long double mid = (2 * p + 1) * hw;
    for (size_t q = 0; q < gx.size(); ++q) {
      const long double u = mid + hw * gx[q];
      const long double v = u > 0 ? std::sin(2.0L * pi * tp * u) / (pi * u) : 2.0L * tp;
      sum += gw[q] * hw * v * std::exp(-pi * pi * s * s * u * u);
    }
  }
  return x < 0 ? -sum : sum;
}

void gauss_legendre(int m, std::vector<long double>& x, std::vector<long double>& w) {
  const long double pi = 3.141592653589793238462643383279502884L;
  x.resize(m);
  w.resize(m);
  for (int i = 0; i < m; ++i) {
    long double z = std::cos(pi * (i + 0.75L) / (m + 0.5L)), dp = 1.0L;
    for (int it = 0; it < 100; ++it) {
      long double p0 = 1.0L, p1 = z;
      for (int k = 2; k <= m; ++k) {
        const long double p2 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = m * (z * p1 - p0) / (z * z - 1.0L);
      const long double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-19L) break;
    }
    x[i] = z;
    w[i] = 2.0L / ((1.0L - z * z) * dp * dp);
  }
}

}  // namespace

void quadform_fast_device(const double* d_t, const double* h_t, int64_t n, double f_max, const double* d_w,
                          int64_t k, double* q_host, cudaStream_t s, int device) {
  require(k >= 1, "quadratic_form: need at least one weight row");
  require(n >= 2, "quadratic_form: need at least 2 samples");
  require(f_max > 0.0 && std::isfinite(f_max), "SignalBand: f_max must be positive");
  const long double T1 = static_cast<long double>(h_t[n - 1]) - h_t[0];
  require(T1 > 0.0L, "quadratic_form: degenerate grid span");
  const long double sw = T1 / 12.0L, tp = T1 + 6.0L * sw;
  const long double pi = 3.141592653589793238462643383279502884L;
  const long double x0 = 6.2L / (pi * sw);
  // lattice spacing: a power of two <= 1 / (3 T1), so j delta is exact
  const double delta = std::ldexp(1.0, static_cast<int>(std::floor(std::log2(1.0 / (3.0 * static_cast<double>(T1))))));
  const long double F = f_max;
  const int64_t jmax = static_cast<int64_t>(std::ceil((F + x0) / delta));
  const int64_t jlo = static_cast<int64_t>(std::floor((F - x0) / delta)) - 1;  // h == 1 for j <= jlo
  std::vector<long double> gx, gw;
  gauss_legendre(16, gx, gw);
  std::vector<double> edge;
  for (int64_t j = std::max<int64_t>(jlo + 1, 0); j <= jmax; ++j) {
    const long double f = static_cast<long double>(j) * delta;
    edge.push_back(static_cast<double>(window_cdf(f + F, tp, sw, x0, gx, gw) -
                                       window_cdf(f - F, tp, sw, x0, gx, gw)));
  }
  const int64_t jlo_eff = std::max<int64_t>(jlo, -1);
  // chunk plan: uniform centres i delta, i < ic
  // Every chunk spreads all N points, so fewer, larger chunks cost less: up to 2^25 centres per chunk
  // (Mr = 2^26) while the chunk's grid + coefficients take at most half the free device memory
  // (full C4: 32 chunks instead of 128, normalisation 4.9 -> ~1.5 s)
  const int64_t need = jmax + 1;
  size_t free_b = 0, total_b = 0;
  NUS_CUDA(cudaMemGetInfo(&free_b, &total_b));
  auto fits = [&](int64_t c) { return static_cast<double>(k) * (2.0 * c + c) * sizeof(double2) < 0.5 * free_b; };
  int64_t ic = 4096;
  while (ic < need && ic < (int64_t{1} << 25) && fits(2 * ic)) ic <<= 1;
  const int64_t chunks = (need + ic - 1) / ic;
  std::vector<double> centers(ic);
  for (int64_t i = 0; i < ic; ++i) centers[i] = static_cast<double>(i) * delta;
  auto plan = plan_create(h_t, 1, n, centers.data(), ic, 1e-13, NUS_FORCE_FAST, 2, NUS_F64, device);
  const int64_t kp = k;
  DeviceBuffer w_sorted(static_cast<size_t>(k) * n * sizeof(double));
  permute_rows_kernel<<<nblocks(n * k), 256, 0, s>>>(d_w, plan->tab.perm.as<int32_t>(), n, k, w_sorted.as<double>());
  note_launch();
  DeviceBuffer xc(static_cast<size_t>(n) * sizeof(double2));
  DeviceBuffer grid(static_cast<size_t>(kp) * plan->p.mr * sizeof(double2));
  DeviceBuffer jk(static_cast<size_t>(k) * ic * sizeof(double2));
  DeviceBuffer d_edge(std::max<size_t>(edge.size(), 1) * sizeof(double));
  if (!edge.empty())
    NUS_CUDA(cudaMemcpyAsync(d_edge.ptr, edge.data(), edge.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  const unsigned rblocks = 148;
  DeviceBuffer partial(static_cast<size_t>(chunks) * k * rblocks * sizeof(double));
  for (int64_t c = 0; c < chunks; ++c) {
    chunk_phase_kernel<<<nblocks(n), 256, 0, s>>>(plan->d_times.as<double>(), n,
                                                  static_cast<double>(c * ic) * delta, xc.as<double2>());
    note_launch();
    SpreadArgs a;
    a.x = xc.ptr;
    a.x_dtype = 0;
    a.x_complex = true;
    a.tapers = w_sorted.ptr;
    a.k = k;
    a.kpad = kp;
    a.grid = grid.ptr;
    launch_spread(*plan, a, s);
    run_fft(*plan, grid.ptr, k, kp, s);
    run_crop(*plan, grid.ptr, k, kp, jk.ptr, nullptr, true, 1.0, false, s);
    weighted_energy_kernel<<<dim3(rblocks, static_cast<unsigned>(k)), kRedThreads, 0, s>>>(
        jk.as<double2>(), ic, c * ic, jmax, jlo_eff, d_edge.as<double>(), static_cast<int64_t>(edge.size()),
        partial.as<double>() + c * k * rblocks);
    note_launch();
    check_launch("quadform_fast chunk");
  }
  std::vector<double> hp(static_cast<size_t>(chunks) * k * rblocks);
  NUS_CUDA(cudaMemcpyAsync(hp.data(), partial.ptr, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
  for (int64_t kk = 0; kk < k; ++kk) {
    long double acc = 0.0L;
    for (int64_t c = 0; c < chunks; ++c)
      for (unsigned b = 0; b < rblocks; ++b) acc += hp[(c * k + kk) * rblocks + b];
    q_host[kk] = static_cast<double>(acc * delta);
  }
}

}  // namespace nus
