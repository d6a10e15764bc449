// MTNUFFT multitaper estimator (reference: include/nuspectral/estimators.hpp:23-62,133-137).
// Setup (tapers, bins, sort, tables) and estimate() run on the device.  The Bronez
// GPSS estimators (BgFixed/BgAdaptive, O(N^4)) and the exact-GEP taper mode are outside
// the B200 hot path and not declared here.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "nuspectral/grid.hpp"
#include "nuspectral/nufft.hpp"
#include "nuspectral/tapers.hpp"

struct nus_mtnufft_s;
struct nus_mtnufft_multi_s;

namespace nuspectral {

enum class EstimatorMethod { mtnufft, mtnufft0, bg_fixed, bg_adaptive, baseline };
enum class TaperMode { interpolated, exact_nominal };
// B200 extension (not in the reference): how one estimator spreads over several GPUs.
enum class Sharding { tapers, samples };

std::string method_name(EstimatorMethod m);
std::optional<EstimatorMethod> method_from_name(const std::string& name);

struct SpectrumEstimate {
  BandPlan plan;
  std::vector<double> power;
  EstimatorMethod method;
  std::vector<std::size_t> k_used;
  std::vector<double> f_w_used;
  std::vector<std::uint8_t> flags;
  SpectrumEstimate(BandPlan p, std::vector<double> pw, EstimatorMethod m, std::vector<std::size_t> k,
                   std::vector<double> fw, std::vector<std::uint8_t> fl);
};

class MtnufftEstimator {
 public:
  struct Options {
    std::size_t k_tapers = 4;
    double epsilon = 1e-8;
    TaperMode taper_mode = TaperMode::interpolated;
    NufftPathPolicy path_policy = NufftPathPolicy::auto_select;
    // B200 extension (absent from the reference, defaulted so reference code compiles unchanged):
    // more than one device -> the series is sharded over these GPUs of this process
    // (nus_mtnufft_multi_*: tapers split, or the sample split with the grid exchange fused into the
    // spread over peer memory).  Empty or one entry: the current device only.
    std::vector<int> devices = {};
    Sharding sharding = Sharding::samples;
  };

  MtnufftEstimator(const SamplingGrid& grid, const SignalBand& signal_band, const BandPlan& plan,
                   const Options& opts);

  SpectrumEstimate estimate(const std::vector<double>& values) const;
  const TaperSet& tapers() const { return tapers_; }
  const NufftPlan& transform_plan() const;
  EstimatorMethod method() const {
    return opts_.taper_mode == TaperMode::exact_nominal ? EstimatorMethod::mtnufft0 : EstimatorMethod::mtnufft;
  }

 private:
  struct Built;  // device estimator + its tapers, built together (MTNUFFT0 tapers are O(N^3))
  static Built build(const SamplingGrid& grid, const SignalBand& signal_band, const BandPlan& plan,
                     const Options& opts);
  MtnufftEstimator(const SamplingGrid& grid, const BandPlan& plan, const Options& opts, Built&& built);
  SamplingGrid grid_;
  BandPlan plan_;
  Options opts_;
  std::shared_ptr<nus_mtnufft_s> handle_;
  std::shared_ptr<nus_mtnufft_multi_s> multi_;  // Options::devices with more than one entry
  TaperSet tapers_;
  mutable std::once_flag plan_once_;
  mutable std::unique_ptr<NufftPlan> nufft_plan_;
};

SpectrumEstimate estimate_mtnufft(const SignalSeries& series, const SignalBand& signal_band,
                                  const BandPlan& plan, std::size_t k_tapers, double epsilon,
                                  TaperMode taper_mode = TaperMode::interpolated);

}  // namespace nuspectral
