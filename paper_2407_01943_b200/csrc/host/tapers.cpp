// Taper entry points of the drop-in: DPSS and interpolated tapers computed on the device
// (nus_dpss, nus_gpss_interpolated); TaperSet is a host container (tapers.hpp:29-63).
#include "nuspectral/tapers.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <utility>

#include "status.hpp"

namespace nuspectral {

DpssSet dpss_uniform(std::size_t n, double time_half_bandwidth, std::size_t k_tapers) {
  if (n < 2) throw std::invalid_argument("dpss_uniform: n must be >= 2");
  if (k_tapers < 1 || k_tapers > n) throw std::invalid_argument("dpss_uniform: k_tapers out of range");
  if (!(time_half_bandwidth > 0.0) || !(time_half_bandwidth < n / 2.0))
    throw std::invalid_argument("dpss_uniform: need 0 < TW < n/2");
  std::vector<double> v(k_tapers * n), ev(k_tapers);
  DpssSet out;
  out.concentrations.resize(k_tapers);
  host::check(nus_dpss(static_cast<int64_t>(n), time_half_bandwidth, static_cast<int64_t>(k_tapers),
                       host::device(), v.data(), ev.data(), out.concentrations.data()));
  out.tapers.resize(k_tapers);
  for (std::size_t k = 0; k < k_tapers; ++k) out.tapers[k].assign(v.begin() + k * n, v.begin() + (k + 1) * n);
  return out;
}

TaperSet::TaperSet(SamplingGrid grid, AnalysisBand band, double f_max,
                   std::vector<std::vector<std::complex<double>>> weights, std::vector<double> eigenvalues,
                   bool is_real)
    : grid_(std::move(grid)), band_(band), f_max_(f_max), real_(is_real), w_(std::move(weights)),
      ev_(std::move(eigenvalues)) {
  if (w_.empty()) throw std::invalid_argument("TaperSet: no tapers");
  for (const auto& w : w_)
    if (w.size() != grid_.n_samples()) throw std::invalid_argument("TaperSet: taper length mismatch");
  if (!ev_.empty() && ev_.size() != w_.size()) throw std::invalid_argument("TaperSet: eigenvalue count mismatch");
  if (real_) {
    wr_.resize(w_.size());
    for (std::size_t k = 0; k < w_.size(); ++k) {
      wr_[k].resize(w_[k].size());
      for (std::size_t i = 0; i < w_[k].size(); ++i) wr_[k][i] = w_[k][i].real();
    }
  }
}

std::vector<std::complex<double>> TaperSet::zero_frequency_responses() const {
  std::vector<std::complex<double>> w0(w_.size(), {0.0, 0.0});
  for (std::size_t k = 0; k < w_.size(); ++k)
    for (const auto& v : w_[k]) w0[k] += v;
  return w0;
}

TaperSet gpss_interpolated(const SamplingGrid& grid, const SignalBand& signal_band, double f_w,
                           std::size_t k_tapers) {
  const std::size_t n = grid.n_samples();
  std::vector<double> w(std::max<std::size_t>(k_tapers, 1) * n);
  host::check(nus_gpss_interpolated(grid.times().data(), static_cast<int64_t>(n), signal_band.f_max, f_w,
                                    static_cast<int64_t>(k_tapers), host::device(), w.data()));
  std::vector<std::vector<std::complex<double>>> weights(k_tapers, std::vector<std::complex<double>>(n));
  for (std::size_t k = 0; k < k_tapers; ++k)
    for (std::size_t i = 0; i < n; ++i) weights[k][i] = {w[k * n + i], 0.0};
  return TaperSet(grid, AnalysisBand(0.0, f_w), signal_band.f_max, std::move(weights), {}, true);
}

TaperSet gpss_exact(const SamplingGrid& grid, const SignalBand& signal_band, const AnalysisBand& band,
                    std::size_t k_tapers, const GeneralizedEigenOptions& opts) {
  const std::size_t n = grid.n_samples();
  const std::size_t k = std::max<std::size_t>(k_tapers, 1);
  std::vector<double> w(2 * k * n), conc(k);
  host::check(nus_gpss_exact(grid.times().data(), static_cast<int64_t>(n), signal_band.f_max, band.f_center,
                             band.half_width, static_cast<int64_t>(k_tapers), opts.ridge_first, opts.ridge_retry,
                             host::device(), w.data(), conc.data()));
  std::vector<std::vector<std::complex<double>>> weights(k_tapers, std::vector<std::complex<double>>(n));
  for (std::size_t j = 0; j < k_tapers; ++j)
    for (std::size_t i = 0; i < n; ++i) weights[j][i] = {w[2 * (j * n + i)], w[2 * (j * n + i) + 1]};
  conc.resize(k_tapers);
  return TaperSet(grid, band, signal_band.f_max, std::move(weights), std::move(conc), band.f_center == 0.0);
}

std::size_t default_taper_count(double time_half_bandwidth) {
  const long k = std::lround(2.0 * time_half_bandwidth) - 1;
  return static_cast<std::size_t>(std::max(k, 1L));
}

}  // namespace nuspectral
