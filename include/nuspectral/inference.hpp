// Harmonic F-test on the MTNUFFT eigencoefficients (reference: include/nuspectral/inference.hpp:16-61).
// The regression runs on the device; f_quantile is host scalar math.  suboptimality (needs the
// Bronez GEP per band) is outside the B200 path and not declared here.
#pragma once

#include <complex>
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

#include "nuspectral/grid.hpp"
#include "nuspectral/nufft.hpp"
#include "nuspectral/tapers.hpp"

namespace nuspectral {

inline constexpr std::uint8_t kFtestConditionViolated = 1;  // 2 f_c <= f_w
inline constexpr std::uint8_t kFtestSaturated = 2;          // residual ~ 0

struct FTestResult {
  BandPlan plan;
  std::vector<double> f_stat;
  std::vector<std::complex<double>> amplitude;
  std::pair<std::size_t, std::size_t> dof;
  std::vector<std::pair<double, double>> critical_values;  // (p, threshold)
  std::vector<std::uint8_t> flags;
  double saturation_cap;
};

struct FTestOptions {
  std::vector<double> p_levels;  // empty -> {0.05, 0.01, 1/N}
  double saturation_cap = 1e12;
};

/// F(2, 2K-2) statistic per band from regressing the eigencoefficients on the tapers'
/// zero-frequency responses.  Throws DegenerateTapers when those responses vanish.
FTestResult f_test(const EigenCoefficients& eigencoeffs, const TaperSet& tapers, const BandPlan& plan,
                   const FTestOptions& opts = {});

/// x with P(F(d1, d2) > x) = p.
double f_quantile(double p, std::size_t d1, std::size_t d2);

}  // namespace nuspectral
