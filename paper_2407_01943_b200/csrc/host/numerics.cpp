// Eigen / spline / FFT / dense-kernel entry points of the drop-in.
// tridiagonal_eigen and Radix2Fft run on the device through the C-ABI; CubicSpline,
// KernelMatrix and detail::cholesky_lower are the reference interface's small host
// utilities (not on the MTNUFFT hot path, whose spline and R(B) sums are device kernels).
#include <algorithm>
#include <cmath>
#include <complex>
#include <stdexcept>
#include <utility>
#include <vector>

#include "nuspectral/eig.hpp"
#include "nuspectral/fft.hpp"
#include "nuspectral/kernels.hpp"
#include "status.hpp"

namespace nuspectral {

// ---- tridiagonal eigenpairs (eig.hpp:30-36) ---------------------------------------

EigenPairs tridiagonal_eigen(const std::vector<double>& diag, const std::vector<double>& offdiag,
                             std::size_t k_top) {
  const std::size_t n = diag.size();
  if (k_top == 0 || k_top > n) throw std::invalid_argument("tridiagonal_eigen: k_top out of range");
  if (offdiag.size() + 1 != n)
    throw std::invalid_argument("tridiagonal_eigenvalues: offdiag length must be n-1");
  EigenPairs out;
  out.values.resize(k_top);
  out.residuals.resize(k_top);
  std::vector<double> vec(k_top * n);
  const double dummy = 0.0;
  host::check(nus_tridiagonal_eigen(diag.data(), offdiag.empty() ? &dummy : offdiag.data(),
                                    static_cast<int64_t>(n), static_cast<int64_t>(k_top), host::device(),
                                    out.values.data(), vec.data(), out.residuals.data()));
  out.vectors.resize(k_top);
  for (std::size_t j = 0; j < k_top; ++j) {
    out.vectors[j].resize(n);
    for (std::size_t i = 0; i < n; ++i) out.vectors[j][i] = {vec[j * n + i], 0.0};
  }
  return out;
}

std::vector<double> tridiagonal_eigenvalues(const std::vector<double>& diag,
                                            const std::vector<double>& offdiag) {
  if (diag.empty()) throw std::invalid_argument("tridiagonal_eigenvalues: empty matrix");
  return tridiagonal_eigen(diag, offdiag, diag.size()).values;
}

// ---- cubic spline, not-a-knot (eig.hpp:68-84) --------------------------------------

CubicSpline::CubicSpline(std::vector<double> x_knots, std::vector<double> y_knots)
    : x_(std::move(x_knots)), y_(std::move(y_knots)) {
  const std::size_t n = x_.size();
  if (n < 4) throw std::invalid_argument("CubicSpline: need at least 4 knots");
  if (y_.size() != n) throw std::invalid_argument("CubicSpline: size mismatch");
  for (std::size_t i = 1; i < n; ++i)
    if (!(x_[i] > x_[i - 1])) throw std::invalid_argument("CubicSpline: knots must be strictly increasing");
  // Moment equations for M[1..n-2]; the not-a-knot conditions (third derivative
  // continuous at x_1 and x_{n-2}) eliminate M[0] and M[n-1].
  const std::size_t m = n - 2;
  std::vector<double> lo(m), di(m), up(m), rh(m);
  auto h = [&](std::size_t i) { return x_[i + 1] - x_[i]; };
  for (std::size_t r = 0; r < m; ++r) {
    const std::size_t i = r + 1;
    lo[r] = h(i - 1) / 6.0;
    di[r] = (h(i - 1) + h(i)) / 3.0;
    up[r] = h(i) / 6.0;
    rh[r] = (y_[i + 1] - y_[i]) / h(i) - (y_[i] - y_[i - 1]) / h(i - 1);
  }
  const double a0 = h(0) / h(1), an = h(n - 2) / h(n - 3);
  di[0] += lo[0] * (1.0 + a0);
  up[0] -= lo[0] * a0;
  lo[0] = 0.0;
  di[m - 1] += up[m - 1] * (1.0 + an);
  lo[m - 1] -= up[m - 1] * an;
  up[m - 1] = 0.0;
  for (std::size_t r = 1; r < m; ++r) {  // forward elimination
    const double f = lo[r] / di[r - 1];
    di[r] -= f * up[r - 1];
    rh[r] -= f * rh[r - 1];
  }
  m_.assign(n, 0.0);
  m_[m] = rh[m - 1] / di[m - 1];
  for (std::size_t r = m - 1; r-- > 0;) m_[r + 1] = (rh[r] - up[r] * m_[r + 2]) / di[r];
  m_[0] = m_[1] * (1.0 + a0) - m_[2] * a0;
  m_[n - 1] = m_[n - 2] * (1.0 + an) - m_[n - 3] * an;
}

double CubicSpline::operator()(double x) const {
  const std::size_t n = x_.size();
  if (x < x_[0] - 0.5 * (x_[1] - x_[0]) || x > x_[n - 1] + 0.5 * (x_[n - 1] - x_[n - 2]))
    throw ExtrapolationError("CubicSpline: evaluation outside knot span guard");
  const double xc = std::clamp(x, x_.front(), x_.back());
  std::size_t i = static_cast<std::size_t>(std::upper_bound(x_.begin(), x_.end(), xc) - x_.begin());
  if (i > 0) --i;
  if (i + 1 >= n) i = n - 2;
  const double hl = x_[i + 1] - x_[i];
  const double a = (x_[i + 1] - xc) / hl, b = (xc - x_[i]) / hl;
  return a * y_[i] + b * y_[i + 1] + ((a * a * a - a) * m_[i] + (b * b * b - b) * m_[i + 1]) * (hl * hl) / 6.0;
}

CubicSpline cubic_spline(std::vector<double> x_knots, std::vector<double> y_knots) {
  return CubicSpline(std::move(x_knots), std::move(y_knots));
}

namespace detail {
bool cholesky_lower(std::vector<double>& a, std::size_t n) {
  for (std::size_t j = 0; j < n; ++j) {
    double s = a[j * n + j];
    for (std::size_t q = 0; q < j; ++q) s -= a[j * n + q] * a[j * n + q];
    if (!(s > 0.0)) return false;
    const double d = std::sqrt(s);
    a[j * n + j] = d;
    for (std::size_t i = j + 1; i < n; ++i) {
      double v = a[i * n + j];
      for (std::size_t q = 0; q < j; ++q) v -= a[i * n + q] * a[j * n + q];
      a[i * n + j] = v / d;
    }
  }
  for (std::size_t r = 0; r < n; ++r)
    for (std::size_t c = r + 1; c < n; ++c) a[r * n + c] = 0.0;
  return true;
}
}  // namespace detail

// ---- FFT (fft.hpp:12-29) ------------------------------------------------------------

std::size_t Radix2Fft::next_power_of_two(std::size_t n) {
  std::size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

Radix2Fft::Radix2Fft(std::size_t n) : n_(n) {
  if (!is_power_of_two(n)) throw std::invalid_argument("Radix2Fft: size must be a power of two");
}

void Radix2Fft::forward(std::complex<double>* data) const {
  host::check(nus_fft_inplace(reinterpret_cast<double*>(data), static_cast<int64_t>(n_), 0, host::device()));
}

void Radix2Fft::inverse(std::complex<double>* data) const {
  host::check(nus_fft_inplace(reinterpret_cast<double*>(data), static_cast<int64_t>(n_), 1, host::device()));
}

// ---- dense kernels (kernels.hpp) ------------------------------------------------------

KernelMatrix::KernelMatrix(std::size_t n, bool is_real, std::string band_tag)
    : n_(n), real_(is_real), tag_(std::move(band_tag)), re_(n * n, 0.0) {
  if (!real_) im_.assign(n * n, 0.0);
}

double KernelMatrix::quadratic_form(const std::vector<double>& w) const {
  if (w.size() != n_) throw std::invalid_argument("quadratic_form: size mismatch");
  if (!real_) throw std::invalid_argument("quadratic_form: complex kernel, real vector");
  return bilinear_form(w, w);
}

double KernelMatrix::quadratic_form(const std::vector<std::complex<double>>& w) const {
  if (w.size() != n_) throw std::invalid_argument("quadratic_form: size mismatch");
  return bilinear_form(w, w).real();
}

double KernelMatrix::bilinear_form(const std::vector<double>& w, const std::vector<double>& v) const {
  if (w.size() != n_ || v.size() != n_) throw std::invalid_argument("bilinear_form: size mismatch");
  if (!real_) throw std::invalid_argument("bilinear_form: complex kernel, real vectors");
  double acc = 0.0;
  for (std::size_t r = 0; r < n_; ++r) {
    double row = 0.0;
    const double* m = re_.data() + r * n_;
    for (std::size_t c = 0; c < n_; ++c) row += m[c] * v[c];
    acc += w[r] * row;
  }
  return acc;
}

std::complex<double> KernelMatrix::bilinear_form(const std::vector<std::complex<double>>& w,
                                                 const std::vector<std::complex<double>>& v) const {
  if (w.size() != n_ || v.size() != n_) throw std::invalid_argument("bilinear_form: size mismatch");
  std::complex<double> acc{0.0, 0.0};
  for (std::size_t r = 0; r < n_; ++r) {
    std::complex<double> row{0.0, 0.0};
    for (std::size_t c = 0; c < n_; ++c) row += at(r, c) * v[c];
    acc += std::conj(w[r]) * row;
  }
  return acc;
}

double KernelMatrix::trace() const {
  double t = 0.0;
  for (std::size_t i = 0; i < n_; ++i) t += re_[i * n_ + i];
  return t;
}

KernelMatrix signal_band_kernel(const SamplingGrid& grid, const SignalBand& band) {
  const std::size_t n = grid.n_samples();
  KernelMatrix m(n, true, "B");
  host::check(nus_signal_band_matrix(grid.times().data(), static_cast<int64_t>(n), band.f_max, host::device(),
                                     m.re_data()));
  return m;
}

KernelMatrix analysis_band_kernel(const SamplingGrid& grid, const AnalysisBand& band) {
  const std::size_t n = grid.n_samples();
  const bool real = band.f_center == 0.0;
  KernelMatrix m(n, real, real ? "A0" : "A");
  host::check(nus_band_matrix(grid.times().data(), static_cast<int64_t>(n), band.half_width, band.f_center,
                              host::device(), m.re_data(), real ? nullptr : m.im_data()));
  return m;
}

namespace {
EigenPairs generalized(const KernelMatrix& A, const KernelMatrix& M, std::size_t k_top,
                       const GeneralizedEigenOptions& opts) {
  if (A.n() != M.n()) throw std::invalid_argument("generalized_hermitian_eigen: size mismatch");
  if (!M.is_real())
    throw std::invalid_argument("generalized_hermitian_eigen: metric must be the real signal-band kernel");
  if (k_top == 0) throw std::invalid_argument("generalized_hermitian_eigen: k_top must be >= 1");
  const std::size_t n = A.n(), k = std::min(k_top, n);
  std::vector<double> vals(k), vecs(opts.want_vectors ? 2 * k * n : 0), res(opts.want_vectors ? k : 0);
  host::check(nus_generalized_eigen(A.re_data(), A.is_real() ? nullptr : A.im_data(), M.re_data(),
                                    static_cast<int64_t>(n), static_cast<int64_t>(k), opts.ridge_first,
                                    opts.ridge_retry, opts.want_vectors ? 1 : 0, host::device(), vals.data(),
                                    opts.want_vectors ? vecs.data() : nullptr,
                                    opts.want_vectors ? res.data() : nullptr));
  EigenPairs out;
  out.metric = EigenMetric::rb_metric;
  out.values = std::move(vals);
  if (opts.want_vectors) {
    out.vectors.assign(k, std::vector<std::complex<double>>(n));
    for (std::size_t j = 0; j < k; ++j)
      for (std::size_t i = 0; i < n; ++i) out.vectors[j][i] = {vecs[2 * (j * n + i)], vecs[2 * (j * n + i) + 1]};
    out.residuals = std::move(res);
  }
  return out;
}
}  // namespace

EigenPairs generalized_hermitian_eigen(const KernelMatrix& A, const KernelMatrix& M, std::size_t k_top,
                                       const GeneralizedEigenOptions& opts) {
  return generalized(A, M, k_top, opts);
}

std::vector<double> generalized_hermitian_eigenvalues(const KernelMatrix& A, const KernelMatrix& M,
                                                      std::size_t k_top, const GeneralizedEigenOptions& opts) {
  GeneralizedEigenOptions o = opts;
  o.want_vectors = false;
  return generalized(A, M, k_top, o).values;
}

}  // namespace nuspectral
