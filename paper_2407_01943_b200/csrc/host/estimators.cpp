// MtnufftEstimator of the drop-in (reference behaviour: src/estimators.cpp:66-122,261-270).
#include "nuspectral/estimators.hpp"

#include <algorithm>
#include <stdexcept>
#include <utility>

#include "status.hpp"

namespace nuspectral {

std::string method_name(EstimatorMethod m) {
  switch (m) {
    case EstimatorMethod::mtnufft: return "mtnufft";
    case EstimatorMethod::mtnufft0: return "mtnufft0";
    case EstimatorMethod::bg_fixed: return "bg_fixed";
    case EstimatorMethod::bg_adaptive: return "bg_adaptive";
    case EstimatorMethod::baseline: return "baseline";
  }
  return "unknown";
}

std::optional<EstimatorMethod> method_from_name(const std::string& name) {
  for (auto m : {EstimatorMethod::mtnufft, EstimatorMethod::mtnufft0, EstimatorMethod::bg_fixed,
                 EstimatorMethod::bg_adaptive, EstimatorMethod::baseline})
    if (method_name(m) == name) return m;
  return std::nullopt;
}

SpectrumEstimate::SpectrumEstimate(BandPlan p, std::vector<double> pw, EstimatorMethod m,
                                   std::vector<std::size_t> k, std::vector<double> fw,
                                   std::vector<std::uint8_t> fl)
    : plan(std::move(p)), power(std::move(pw)), method(m), k_used(std::move(k)), f_w_used(std::move(fw)),
      flags(std::move(fl)) {
  const std::size_t n = plan.size();
  if (power.size() != n || k_used.size() != n || f_w_used.size() != n || flags.size() != n)
    throw std::invalid_argument("SpectrumEstimate: per-band field length mismatch");
  for (std::size_t i = 0; i < n; ++i)
    if (!(flags[i] & kBandFailed) && !(power[i] >= 0.0))
      throw std::invalid_argument("SpectrumEstimate: negative power");
}

struct MtnufftEstimator::Built {
  std::shared_ptr<nus_mtnufft_s> handle;
  TaperSet tapers;
  std::shared_ptr<nus_mtnufft_multi_s> multi;
};

namespace {

nus_mtnufft_config_t make_config(const SamplingGrid& grid, const SignalBand& band, const BandPlan& plan,
                                 const MtnufftEstimator::Options& o, std::size_t n_centers) {
  nus_mtnufft_config_t cfg{};
  cfg.channels = 1;
  cfg.n = static_cast<int64_t>(grid.n_samples());
  cfg.n_centers = static_cast<int64_t>(n_centers);
  cfg.k_tapers = static_cast<int64_t>(o.k_tapers);
  cfg.f_max = band.f_max;
  cfg.f_w = plan.half_width();
  cfg.epsilon = o.epsilon;
  cfg.policy = o.path_policy == NufftPathPolicy::force_fast     ? NUS_FORCE_FAST
               : o.path_policy == NufftPathPolicy::force_direct ? NUS_FORCE_DIRECT
                                                                : NUS_AUTO_SELECT;
  cfg.precision = NUS_F64;
  cfg.device = host::device();
  return cfg;
}

std::shared_ptr<nus_mtnufft_s> wrap(nus_mtnufft_t h) {
  return std::shared_ptr<nus_mtnufft_s>(h, [](nus_mtnufft_s* p) { nus_mtnufft_destroy(p); });
}

}  // namespace

// Tapers first, then the transform plan (estimators.cpp:91-104): interpolated prolates
// (MTNUFFT) are built inside the device estimator; the exact nominal-band tapers (MTNUFFT0)
// come from gpss_exact on the dense pencil and are handed to the estimator.
MtnufftEstimator::Built MtnufftEstimator::build(const SamplingGrid& grid, const SignalBand& band,
                                                const BandPlan& plan, const Options& o) {
  const std::vector<double> centers = plan.centers();
  const nus_mtnufft_config_t cfg = make_config(grid, band, plan, o, centers.size());
  const std::size_t n = grid.n_samples(), k = o.k_tapers;
  nus_mtnufft_t h = nullptr;
  if (o.taper_mode == TaperMode::exact_nominal) {
    TaperSet ts = gpss_exact(grid, band, AnalysisBand(0.0, plan.half_width()), k);
    std::vector<double> w(k * n);
    for (std::size_t j = 0; j < k; ++j) std::copy(ts.weights_real(j).begin(), ts.weights_real(j).end(), w.begin() + j * n);
    host::check(nus_mtnufft_create(&cfg, grid.times().data(), centers.data(), w.data(), &h));
    return {wrap(h), std::move(ts), nullptr};
  }
  if (k < 1 || k > n) throw std::invalid_argument("dpss_uniform: k_tapers out of range");
  if (o.devices.size() > 1) {  // one series over several GPUs (multi.cu)
    nus_mtnufft_multi_t mh = nullptr;
    const std::vector<int32_t> devs(o.devices.begin(), o.devices.end());
    host::check(nus_mtnufft_multi_create(&cfg, devs.data(), static_cast<int32_t>(devs.size()),
                                         o.sharding == Sharding::tapers ? NUS_SHARD_TAPERS : NUS_SHARD_SAMPLES,
                                         grid.times().data(), centers.data(), nullptr, nullptr, &mh));
    std::shared_ptr<nus_mtnufft_multi_s> multi(mh, [](nus_mtnufft_multi_s* p) { nus_mtnufft_multi_destroy(p); });
    std::vector<double> w(k * n);
    host::check(nus_mtnufft_multi_tapers(multi.get(), w.data()));
    std::vector<std::vector<std::complex<double>>> weights(k, std::vector<std::complex<double>>(n));
    for (std::size_t j = 0; j < k; ++j)
      for (std::size_t i = 0; i < n; ++i) weights[j][i] = {w[j * n + i], 0.0};
    return {nullptr, TaperSet(grid, AnalysisBand(0.0, plan.half_width()), band.f_max, std::move(weights), {}, true),
            std::move(multi)};
  }
  host::check(nus_mtnufft_create(&cfg, grid.times().data(), centers.data(), nullptr, &h));
  auto handle = wrap(h);
  std::vector<double> w(k * n);
  host::check(nus_mtnufft_tapers(handle.get(), w.data()));
  std::vector<std::vector<std::complex<double>>> weights(k, std::vector<std::complex<double>>(n));
  for (std::size_t j = 0; j < k; ++j)
    for (std::size_t i = 0; i < n; ++i) weights[j][i] = {w[j * n + i], 0.0};
  return {std::move(handle),
          TaperSet(grid, AnalysisBand(0.0, plan.half_width()), band.f_max, std::move(weights), {}, true), nullptr};
}

MtnufftEstimator::MtnufftEstimator(const SamplingGrid& grid, const SignalBand& signal_band, const BandPlan& plan,
                                   const Options& opts)
    : MtnufftEstimator(grid, plan, opts, build(grid, signal_band, plan, opts)) {}

MtnufftEstimator::MtnufftEstimator(const SamplingGrid& grid, const BandPlan& plan, const Options& opts,
                                   Built&& built)
    : grid_(grid),
      plan_(plan),
      opts_(opts),
      handle_(std::move(built.handle)),
      multi_(std::move(built.multi)),
      tapers_(std::move(built.tapers)) {}

SpectrumEstimate MtnufftEstimator::estimate(const std::vector<double>& values) const {
  if (values.size() != grid_.n_samples())
    throw std::invalid_argument("estimate: series length does not match grid");
  std::vector<double> power(plan_.size());
  if (multi_) host::check(nus_mtnufft_multi_estimate(multi_.get(), values.data(), power.data()));
  else host::check(nus_mtnufft_estimate(handle_.get(), values.data(), power.data()));
  const std::size_t bands = plan_.size();
  return SpectrumEstimate(plan_, std::move(power), method(),
                          std::vector<std::size_t>(bands, opts_.k_tapers),
                          std::vector<double>(bands, plan_.half_width()), plan_.flags());
}

const NufftPlan& MtnufftEstimator::transform_plan() const {
  std::call_once(plan_once_, [&] {
    nufft_plan_ = std::make_unique<NufftPlan>(grid_, plan_.centers(), opts_.epsilon, opts_.path_policy);
  });
  return *nufft_plan_;
}

SpectrumEstimate estimate_mtnufft(const SignalSeries& series, const SignalBand& signal_band, const BandPlan& plan,
                                  std::size_t k_tapers, double epsilon, TaperMode taper_mode) {
  MtnufftEstimator::Options o;
  o.k_tapers = k_tapers;
  o.epsilon = epsilon;
  o.taper_mode = taper_mode;
  return MtnufftEstimator(series.grid, signal_band, plan, o).estimate(series.values);
}

}  // namespace nuspectral
