// Symmetric tridiagonal eigenpairs and cubic splines (reference: include/nuspectral/eig.hpp).
// tridiagonal_eigen runs on the device (Sturm multisection + double-double inverse
// iteration); CubicSpline is the host utility class of the reference interface
// (the hot-path spline inside gpss_interpolated runs on the device).
#pragma once

#include <complex>
#include <cstddef>
#include <vector>

#include "nuspectral/errors.hpp"
#include "nuspectral/kernels.hpp"

namespace nuspectral {

enum class EigenMetric { identity, rb_metric };

struct EigenPairs {
  std::vector<double> values;                              // descending
  std::vector<std::vector<std::complex<double>>> vectors;  // unit norm, max-|v| entry positive
  EigenMetric metric = EigenMetric::identity;
  std::vector<double> residuals;  // ||T v - lambda v|| / ||T||_inf
  std::size_t count() const { return values.size(); }
};

EigenPairs tridiagonal_eigen(const std::vector<double>& diag, const std::vector<double>& offdiag,
                             std::size_t k_top);

struct GeneralizedEigenOptions {
  bool want_vectors = true;
  // Ridge factors tried in order, scaled by trace(M)/n, before Cholesky is declared failed.
  double ridge_first = 1e-12;
  double ridge_retry = 1e-9;
};

/// A w = lambda M w for Hermitian A and the real symmetric positive definite M (eig.hpp:46-56),
/// solved on the device (cuSOLVER / cuBLAS; MTNUFFT0): the k_top largest
/// pairs, values clamped into [0, 1] (SpectralRangeError beyond 1e-6), vectors normalised to
/// w^* M w = 1 with the canonical phase; ConditioningError when M + ridge is not positive definite.
EigenPairs generalized_hermitian_eigen(const KernelMatrix& A, const KernelMatrix& M, std::size_t k_top,
                                       const GeneralizedEigenOptions& opts = {});
std::vector<double> generalized_hermitian_eigenvalues(const KernelMatrix& A, const KernelMatrix& M,
                                                      std::size_t k_top,
                                                      const GeneralizedEigenOptions& opts = {});
std::vector<double> tridiagonal_eigenvalues(const std::vector<double>& diag,
                                            const std::vector<double>& offdiag);

/// Not-a-knot cubic interpolant; evaluation clamps within half an end interval and
/// throws ExtrapolationError beyond it.
class CubicSpline {
 public:
  CubicSpline(std::vector<double> x_knots, std::vector<double> y_knots);
  double operator()(double x) const;
  double front() const { return x_.front(); }
  double back() const { return x_.back(); }

 private:
  std::vector<double> x_, y_, m_;
};

CubicSpline cubic_spline(std::vector<double> x_knots, std::vector<double> y_knots);

namespace detail {
/// In-place lower Cholesky of a row-major n x n matrix (utility kept for the reference's
/// test support / simulators; not on the MTNUFFT path).
bool cholesky_lower(std::vector<double>& a, std::size_t n);
}  // namespace detail

}  // namespace nuspectral
