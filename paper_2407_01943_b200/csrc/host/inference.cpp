// F-test of the drop-in over the C-ABI (reference behaviour: src/inference.cpp:94-186).
#include "nuspectral/inference.hpp"

#include <stdexcept>

#include "status.hpp"

namespace nuspectral {

double f_quantile(double p, std::size_t d1, std::size_t d2) {
  double out = 0.0;
  host::check(nus_f_quantile(p, static_cast<int64_t>(d1), static_cast<int64_t>(d2), &out));
  return out;
}

FTestResult f_test(const EigenCoefficients& eigencoeffs, const TaperSet& tapers, const BandPlan& plan,
                   const FTestOptions& opts) {
  const std::size_t kk = tapers.k_tapers();
  if (kk < 2) throw std::invalid_argument("f_test: need at least 2 tapers");
  if (eigencoeffs.n_tapers != kk || eigencoeffs.n_bands != plan.size())
    throw std::invalid_argument("f_test: eigencoefficient shape mismatch");
  const std::vector<std::complex<double>> w0 = tapers.zero_frequency_responses();
  const std::vector<double> centers = plan.centers();
  const std::size_t nb = plan.size();
  FTestResult out{plan, std::vector<double>(nb), std::vector<std::complex<double>>(nb), {2, 2 * kk - 2}, {},
                  std::vector<std::uint8_t>(nb), opts.saturation_cap};
  host::check(nus_f_test(reinterpret_cast<const double*>(eigencoeffs.data.data()), static_cast<int64_t>(kk),
                         static_cast<int64_t>(nb), reinterpret_cast<const double*>(w0.data()),
                         static_cast<int64_t>(tapers.n_samples()), centers.data(), plan.half_width(),
                         opts.saturation_cap, host::device(), out.f_stat.data(),
                         reinterpret_cast<double*>(out.amplitude.data()), out.flags.data()));
  std::vector<double> levels = opts.p_levels;
  if (levels.empty()) levels = {0.05, 0.01, 1.0 / static_cast<double>(tapers.n_samples())};
  for (double p : levels) out.critical_values.emplace_back(p, f_quantile(p, 2, 2 * kk - 2));
  return out;
}

}  // namespace nuspectral
