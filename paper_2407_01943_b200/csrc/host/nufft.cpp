// NufftPlan / ndft_direct / eigencoefficients of the drop-in over the C-ABI
// (reference behaviour: src/nufft.cpp:36-227).
#include "nuspectral/nufft.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <utility>

#include "nuspectral/errors.hpp"
#include "status.hpp"

namespace nuspectral {

namespace {

std::vector<std::complex<double>> from_interleaved(const std::vector<double>& v) {
  std::vector<std::complex<double>> out(v.size() / 2);
  for (std::size_t i = 0; i < out.size(); ++i) out[i] = {v[2 * i], v[2 * i + 1]};
  return out;
}

int policy_code(NufftPathPolicy p) {
  switch (p) {
    case NufftPathPolicy::force_fast: return NUS_FORCE_FAST;
    case NufftPathPolicy::force_direct: return NUS_FORCE_DIRECT;
    default: return NUS_AUTO_SELECT;
  }
}

}  // namespace

std::vector<std::complex<double>> ndft_direct(const SamplingGrid& grid,
                                              const std::vector<std::complex<double>>& weighted_values,
                                              const std::vector<double>& freq_centers) {
  if (weighted_values.size() != grid.n_samples()) throw std::invalid_argument("ndft_direct: length mismatch");
  if (freq_centers.empty()) return {};
  std::vector<double> out(2 * freq_centers.size());
  host::check(nus_ndft_direct(grid.times().data(), static_cast<int64_t>(grid.n_samples()),
                              reinterpret_cast<const double*>(weighted_values.data()), freq_centers.data(),
                              static_cast<int64_t>(freq_centers.size()), host::device(), out.data()));
  return from_interleaved(out);
}

NufftPlan::NufftPlan(const SamplingGrid& grid, std::vector<double> freq_centers, double epsilon,
                     NufftPathPolicy policy, int oversampling)
    : times_(grid.times()), centers_(std::move(freq_centers)), epsilon_(epsilon), oversampling_(oversampling),
      policy_(policy) {
  nus_plan_t h = nullptr;
  host::check(nus_plan_create(times_.data(), static_cast<int64_t>(times_.size()),
                              centers_.empty() ? nullptr : centers_.data(), static_cast<int64_t>(centers_.size()),
                              epsilon_, policy_code(policy), oversampling, NUS_F64, host::device(), &h));
  handle_ = std::shared_ptr<nus_plan_s>(h, [](nus_plan_s* p) { nus_plan_destroy(p); });
  nus_plan_info_t info{};
  host::check(nus_plan_info(h, &info));
  spread_width_ = static_cast<std::size_t>(info.spread_width);
  path_ = info.path == NUS_PATH_FAST ? NufftPath::fast : NufftPath::direct;
  uniform_ = info.centers_uniform != 0;
}

std::vector<std::complex<double>> NufftPlan::execute(
    const std::vector<std::complex<double>>& weighted_values) const {
  if (weighted_values.size() != times_.size())
    throw PlanMismatch("NufftPlan: input length does not match plan grid");
  std::vector<double> out(2 * centers_.size());
  host::check(nus_plan_execute(handle_.get(), reinterpret_cast<const double*>(weighted_values.data()),
                               static_cast<int64_t>(weighted_values.size()), out.data()));
  return from_interleaved(out);
}

std::vector<long> NufftPlan::first_cells() const {
  std::vector<int64_t> j(times_.size());
  host::check(nus_plan_first_cells(handle_.get(), j.data()));
  return std::vector<long>(j.begin(), j.end());
}

std::vector<std::complex<double>> nufft_fast(const NufftPlan& plan,
                                             const std::vector<std::complex<double>>& weighted_values) {
  return plan.execute(weighted_values);
}

EigenCoefficients eigencoefficients(const TaperSet& tapers, const SignalSeries& series, const NufftPlan& plan) {
  const std::size_t n = series.grid.n_samples();
  if (tapers.n_samples() != n || plan.n_samples() != n)
    throw PlanMismatch("eigencoefficients: tapers, series and plan must share one grid");
  if (tapers.grid().times() != series.grid.times())
    throw PlanMismatch("eigencoefficients: taper grid differs from series grid");
  if (!tapers.is_real())
    throw std::invalid_argument("eigencoefficients: complex (shifted) tapers are outside the B200 path");
  const std::size_t kk = tapers.k_tapers();
  std::vector<double> w(kk * n);
  for (std::size_t k = 0; k < kk; ++k) std::copy(tapers.weights_real(k).begin(), tapers.weights_real(k).end(),
                                                 w.begin() + k * n);
  nus_mtnufft_config_t cfg{};
  cfg.channels = 1;
  cfg.n = static_cast<int64_t>(n);
  cfg.n_centers = static_cast<int64_t>(plan.n_centers());
  cfg.k_tapers = static_cast<int64_t>(kk);
  cfg.f_max = tapers.f_max();
  cfg.f_w = tapers.band().half_width;
  cfg.epsilon = plan.epsilon();
  cfg.policy = plan.path() == NufftPath::fast ? NUS_FORCE_FAST : NUS_FORCE_DIRECT;
  cfg.precision = NUS_F64;
  cfg.device = host::device();
  nus_mtnufft_t est = nullptr;
  host::check(nus_mtnufft_create(&cfg, series.grid.times().data(), plan.centers().data(), w.data(), &est));
  std::unique_ptr<nus_mtnufft_s, int (*)(nus_mtnufft_s*)> guard(est, nus_mtnufft_destroy);
  EigenCoefficients out;
  out.n_tapers = kk;
  out.n_bands = plan.n_centers();
  std::vector<double> j(2 * kk * out.n_bands);
  host::check(nus_mtnufft_eigencoefficients(est, series.values.data(), j.data()));
  out.data = from_interleaved(j);
  return out;
}

}  // namespace nuspectral
