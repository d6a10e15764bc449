// Harmonic F-test on the eigencoefficients (reference
// src/inference.cpp:132-186), on the device, reading J where the transform left it.
//
// Per band i:  num = sum_k J_k(i) conj(W0_k),  amp = num / E0,  E0 = sum_k |W0_k|^2,
//              resid = sum_k |J_k(i) - amp W0_k|^2,  F = |amp|^2 (K-1) E0 / resid,
// saturating at `cap` when resid < 1e-12 * numerator; bands with 2 f_c <= f_w are
// flagged (kFtestConditionViolated = 1), saturated ones kFtestSaturated = 2.
// f_quantile (F(d1,d2) upper-tail critical values, inference.cpp:94-130) is scalar
// host math: regularised incomplete beta by Lentz's continued fraction + Newton.
#include <cmath>
#include <limits>

#include "nus_estimator.cuh"

namespace nus {

namespace {

template <typename JT>
__global__ void ftest_kernel(const JT* __restrict__ j, int64_t k, int64_t nb, int64_t channels,
                             const double* __restrict__ w0, const double* __restrict__ e0,
                             const double* __restrict__ centers, double f_w, double cap,
                             double* __restrict__ f_out, double* __restrict__ amp_out,
                             uint8_t* __restrict__ flags) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= channels * nb) return;
  const int64_t c = g / nb, i = g - c * nb;
  const double* w = w0 + 2 * c * k;
  const double en = e0[c];
  double nr = 0.0, ni = 0.0;
  for (int64_t kk = 0; kk < k; ++kk) {  // J * conj(W0)
    const double jr = static_cast<double>(j[2 * ((c * k + kk) * nb + i)]);
    const double ji = static_cast<double>(j[2 * ((c * k + kk) * nb + i) + 1]);
    nr += jr * w[2 * kk] + ji * w[2 * kk + 1];
    ni += ji * w[2 * kk] - jr * w[2 * kk + 1];
  }
  const double ar = nr / en, ai = ni / en;
  double resid = 0.0;
  for (int64_t kk = 0; kk < k; ++kk) {
    const double jr = static_cast<double>(j[2 * ((c * k + kk) * nb + i)]);
    const double ji = static_cast<double>(j[2 * ((c * k + kk) * nb + i) + 1]);
    const double dr = jr - (ar * w[2 * kk] - ai * w[2 * kk + 1]);
    const double di = ji - (ar * w[2 * kk + 1] + ai * w[2 * kk]);
    resid += dr * dr + di * di;
  }
  const double numerator = (ar * ar + ai * ai) * static_cast<double>(k - 1) * en;
  uint8_t fl = 0;
  double f;
  if (resid < 1e-12 * numerator) {
    f = cap;
    fl |= 2;
  } else {
    f = numerator / resid;
  }
  if (!(2.0 * centers[i] > f_w)) fl |= 1;
  f_out[g] = f;
  amp_out[2 * g] = ar;
  amp_out[2 * g + 1] = ai;
  flags[g] = fl;
}

// zero-frequency responses W0_k = sum_n w_k(t_n) (tapers.cpp:110-116), one block per row
__global__ void row_sum_kernel(const double* __restrict__ w, int64_t n, double* __restrict__ out) {
  const int64_t r = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += w[r * n + i];
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[r] = red[0];
}

double log_gamma(double x) { return std::lgamma(x); }

// Regularised incomplete beta I_x(a, b), continued fraction (modified Lentz).
double betacf(double a, double b, double x) {
  const double tiny = 1e-300;
  double c = 1.0, d = 1.0 - (a + b) * x / (a + 1.0);
  if (std::fabs(d) < tiny) d = tiny;
  d = 1.0 / d;
  double h = d;
  for (int m = 1; m <= 400; ++m) {
    const double m2 = 2.0 * m;
    double aa = m * (b - m) * x / ((a + m2 - 1.0) * (a + m2));
    d = 1.0 + aa * d;
    if (std::fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c;
    if (std::fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    h *= d * c;
    aa = -(a + m) * (a + b + m) * x / ((a + m2) * (a + m2 + 1.0));
    d = 1.0 + aa * d;
    if (std::fabs(d) < tiny) d = tiny;
    c = 1.0 + aa / c;
    if (std::fabs(c) < tiny) c = tiny;
    d = 1.0 / d;
    const double del = d * c;
    h *= del;
    if (std::fabs(del - 1.0) < 1e-16) break;
  }
  return h;
}

double inc_beta(double a, double b, double x) {
  if (x <= 0.0) return 0.0;
  if (x >= 1.0) return 1.0;
  const double lbt = log_gamma(a + b) - log_gamma(a) - log_gamma(b) + a * std::log(x) + b * std::log1p(-x);
  const double bt = std::exp(lbt);
  if (x < (a + 1.0) / (a + b + 2.0)) return bt * betacf(a, b, x) / a;
  return 1.0 - bt * betacf(b, a, 1.0 - x) / b;
}

}  // namespace

double f_quantile_host(double p, int64_t d1, int64_t d2) {
  require(p > 0.0 && p < 1.0, "f_quantile: p must be in (0, 1)");
  require(d1 >= 1 && d2 >= 1, "f_quantile: degrees of freedom must be >= 1");
  const double a = 0.5 * static_cast<double>(d1), b = 0.5 * static_cast<double>(d2);
  const double target = 1.0 - p;  // P(F <= x) = I_z(a, b), z = d1 x / (d1 x + d2)
  const double lnorm = log_gamma(a + b) - log_gamma(a) - log_gamma(b);
  double lo = 0.0, hi = 1.0, z = a / (a + b);
  for (int it = 0; it < 300; ++it) {
    const double f = inc_beta(a, b, z) - target;
    if (f > 0.0) hi = z; else lo = z;
    const double pdf = std::exp(lnorm + (a - 1.0) * std::log(z) + (b - 1.0) * std::log1p(-z));
    double zn = z - f / pdf;
    if (!(zn > lo && zn < hi)) zn = 0.5 * (lo + hi);
    if (std::fabs(zn - z) <= 1e-16 * std::fmax(1.0, z)) {
      z = zn;
      break;
    }
    z = zn;
  }
  z = std::fmin(std::fmax(z, std::numeric_limits<double>::min()), 1.0 - 1e-16);
  return static_cast<double>(d2) * z / (static_cast<double>(d1) * (1.0 - z));
}

// J on the device ([C][K][nb] complex of the given precision), W0 host [C][K] complex.
void ftest_device(const void* j_dev, bool j_f32, int64_t k, int64_t nb, int64_t channels, const double* w0_host,
                  int64_t n_samples, const double* d_centers, double f_w, double cap, double* f_dev,
                  double* amp_dev, uint8_t* flags_dev, cudaStream_t s) {
  require(k >= 2, "f_test: need at least 2 tapers");
  std::vector<double> e0(channels);
  for (int64_t c = 0; c < channels; ++c) {
    double e = 0.0;
    for (int64_t kk = 0; kk < k; ++kk)
      e += w0_host[2 * (c * k + kk)] * w0_host[2 * (c * k + kk)] +
           w0_host[2 * (c * k + kk) + 1] * w0_host[2 * (c * k + kk) + 1];
    if (e <= 1e-14 * static_cast<double>(k) * static_cast<double>(n_samples))
      fail(NUS_ERR_DEGENERATE_TAPERS, "f_test: zero-frequency taper responses vanish");
    e0[c] = e;
  }
  DeviceBuffer dw(channels * k * 2 * sizeof(double)), de(channels * sizeof(double));
  NUS_CUDA(cudaMemcpyAsync(dw.ptr, w0_host, dw.bytes, cudaMemcpyHostToDevice, s));
  NUS_CUDA(cudaMemcpyAsync(de.ptr, e0.data(), de.bytes, cudaMemcpyHostToDevice, s));
  const unsigned blocks = static_cast<unsigned>((channels * nb + 255) / 256);
  if (j_f32)
    ftest_kernel<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(j_dev), k, nb, channels, dw.as<double>(),
                                               de.as<double>(), d_centers, f_w, cap, f_dev, amp_dev, flags_dev);
  else
    ftest_kernel<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(j_dev), k, nb, channels, dw.as<double>(),
                                                de.as<double>(), d_centers, f_w, cap, f_dev, amp_dev, flags_dev);
  note_launch();
  check_launch("ftest_kernel");
  NUS_CUDA(cudaStreamSynchronize(s));
}

void taper_zero_frequency(const Estimator& est, double* w0_host /* [C][K] complex */) {
  const int64_t rows = est.cfg.channels * est.cfg.k_tapers;
  DeviceBuffer sums(rows * sizeof(double));
  row_sum_kernel<<<static_cast<unsigned>(rows), 256>>>(est.tapers_time.as<double>(), est.cfg.n, sums.as<double>());
  note_launch();
  check_launch("row_sum_kernel");
  std::vector<double> h(rows);
  NUS_CUDA(cudaMemcpy(h.data(), sums.ptr, rows * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t r = 0; r < rows; ++r) {
    w0_host[2 * r] = h[r];
    w0_host[2 * r + 1] = 0.0;
  }
}

}  // namespace nus
