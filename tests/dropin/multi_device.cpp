// The C++ drop-in's multi-GPU extension (MtnufftEstimator::Options::devices / sharding) against
// the single-device estimator: the same P (to rounding) whether the series runs on one device,
// its tapers are split over devices, or its samples are split with the fused peer-slot exchange.
// Run on one GPU with the device repeated (emulated parts).  Prints "<n> failed" like doctest.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "nuspectral/estimators.hpp"

using namespace nuspectral;

static double rel_l2(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return std::sqrt(num / den);
}

int main() {
  const size_t n = size_t{1} << 18;
  std::mt19937_64 rng(20240702);
  std::uniform_real_distribution<double> jit(-0.4, 0.4);
  std::normal_distribution<double> gauss(0.0, 1.0);
  std::vector<double> t(n), x(n);
  for (size_t i = 0; i < n; ++i) t[i] = static_cast<double>(i) + jit(rng);
  for (size_t i = 0; i < n; ++i) x[i] = gauss(rng) + std::cos(0.6 * t[i]);
  const SamplingGrid grid(t);
  const double h = (t[n - 1] - t[0]) / static_cast<double>(n - 1);
  const double f_w = 4.0 / (h * static_cast<double>(n));
  const BandPlan plan = make_band_plan(0.5, f_w, 0.5 / static_cast<double>(n / 2 - 1));
  MtnufftEstimator::Options o;
  o.k_tapers = 7;
  o.epsilon = 1e-9;
  const MtnufftEstimator single(grid, SignalBand(0.5), plan, o);
  const std::vector<double> p1 = single.estimate(x).power;
  int failed = 0, checks = 0;
  for (Sharding sh : {Sharding::tapers, Sharding::samples}) {
    for (size_t parts : {2, 3}) {
      o.devices.assign(parts, 0);
      o.sharding = sh;
      const MtnufftEstimator multi(grid, SignalBand(0.5), plan, o);
      const double e = rel_l2(multi.estimate(x).power, p1);
      bool same_tapers = true;
      for (size_t k = 0; k < o.k_tapers; ++k)
        same_tapers = same_tapers && multi.tapers().weights_real(k) == single.tapers().weights_real(k);
      const bool ok = e < 1e-12 && same_tapers && multi.estimate(x).power == multi.estimate(x).power;
      std::printf("%s x%zu: relL2(P) vs one device = %.3e, tapers identical = %d -> %s\n",
                  sh == Sharding::tapers ? "tapers" : "samples", parts, e, same_tapers ? 1 : 0, ok ? "ok" : "FAIL");
      ++checks;
      failed += ok ? 0 : 1;
    }
  }
  std::printf("[multi_device] %d checks, %d failed\n", checks, failed);
  return failed == 0 ? 0 : 1;
}
