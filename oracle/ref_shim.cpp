// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the *unmodified* reference library (nuspectral, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It
// lets the Python tests, the golden-fixture generator and bench.py's
// cpu_baseline / --impl reference arm call the reference's own code paths
// through ctypes.  Only tests/, __graft_entry__.smoke() and bench.py's CPU arm
// may load the resulting oracle/_ref/libnusref.so.
//
// Every entry point is a thin adapter: it builds the reference's own objects
// (SamplingGrid, NufftPlan, TaperSet, MtnufftEstimator, ...) and calls their
// public methods.  The one exception is ref_plan_first_cells, which reads the
// plan's private first_cell_ table through an access-widening include (the
// class layout is unchanged, only the access check is relaxed) so the GPU
// bin computation can be compared bit-for-bit with the reference's
// (nufft.cpp:118-122).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#define private public
#include "nuspectral/nufft.hpp"
#undef private

#include "nuspectral/bench.hpp"
#include "nuspectral/eig.hpp"
#include "nuspectral/errors.hpp"
#include "nuspectral/estimators.hpp"
#include "nuspectral/fft.hpp"
#include "nuspectral/grid.hpp"
#include "nuspectral/inference.hpp"
#include "nuspectral/kernels.hpp"
#include "nuspectral/simkit.hpp"
#include "nuspectral/tapers.hpp"

using namespace nuspectral;
using cplx = std::complex<double>;

namespace {

thread_local std::string g_err;

// Error classes mapped to small integers so the Python side can assert the
// exact exception type the reference raised.
enum : int {
  kOk = 0,
  kInvalidArgument = 1,
  kPlanMismatch = 2,
  kBandRange = 3,
  kExtrapolation = 4,
  kNumeric = 5,
  kOther = 9,
};

int guard(const std::function<void()>& fn) {
  try {
    fn();
    return kOk;
  } catch (const PlanMismatch& e) {
    g_err = e.what();
    return kPlanMismatch;
  } catch (const BandRangeError& e) {
    g_err = e.what();
    return kBandRange;
  } catch (const ExtrapolationError& e) {
    g_err = e.what();
    return kExtrapolation;
  } catch (const Error& e) {
    g_err = e.what();
    return kNumeric;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalidArgument;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

std::vector<double> vec(const double* p, int64_t n) { return std::vector<double>(p, p + n); }

std::vector<cplx> cvec(const double* interleaved, int64_t n) {
  std::vector<cplx> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[i] = {interleaved[2 * i], interleaved[2 * i + 1]};
  return v;
}

void cout_(const std::vector<cplx>& v, double* out) {
  for (size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}

NufftPathPolicy policy_of(int p) {
  switch (p) {
    case 1: return NufftPathPolicy::force_fast;
    case 2: return NufftPathPolicy::force_direct;
    default: return NufftPathPolicy::auto_select;
  }
}

// Oracle-B: the reference's NufftPlan + eigencoefficients + power
// loop with injected (already normalised) taper weights, run one taper at a
// time so memory stays bounded; arithmetically identical to
// MtnufftEstimator::estimate (estimators.cpp:106-122).
struct InjectedEstimator {
  SamplingGrid grid;
  std::vector<std::vector<double>> weights;  // K x N
  NufftPlan plan;
  double f_max;
  double f_w;

  InjectedEstimator(SamplingGrid g, std::vector<std::vector<double>> w, std::vector<double> centers,
                    double eps, int policy, double fmax, double fw)
      : grid(std::move(g)),
        weights(std::move(w)),
        plan(grid, std::move(centers), eps, policy_of(policy)),
        f_max(fmax),
        f_w(fw) {}

  void power(const double* x, double* out) const {
    const SignalSeries series(grid, vec(x, grid.n_samples()));
    const size_t bands = plan.n_centers();
    std::vector<double> p(bands, 0.0);
    for (size_t k = 0; k < weights.size(); ++k) {
      std::vector<std::vector<cplx>> one(1, std::vector<cplx>(grid.n_samples()));
      for (size_t i = 0; i < grid.n_samples(); ++i) one[0][i] = {weights[k][i], 0.0};
      const TaperSet t(grid, AnalysisBand(0.0, f_w), f_max, std::move(one), {}, true);
      const EigenCoefficients j = eigencoefficients(t, series, plan);
      const cplx* row = j.row(0);
      for (size_t i = 0; i < bands; ++i) p[i] += std::norm(row[i]);
    }
    const double kk = static_cast<double>(weights.size());
    for (size_t i = 0; i < bands; ++i) out[i] = p[i] / kk;
  }
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- grid / bands ---------------------------------------------------------

int ref_grid_check(const double* t, int64_t n, double* mean_dt) {
  return guard([&] {
    SamplingGrid g(vec(t, n));
    if (mean_dt) *mean_dt = g.mean_dt();
  });
}

int ref_make_band_plan(double f_max, double f_w, double spacing, double margin, int64_t cap,
                       double* centers, uint8_t* flags, int64_t* count) {
  return guard([&] {
    const BandPlan p = margin > 0 ? make_band_plan(f_max, f_w, spacing, margin)
                                  : make_band_plan(f_max, f_w, spacing);
    *count = static_cast<int64_t>(p.size());
    for (size_t i = 0; i < p.size() && static_cast<int64_t>(i) < cap; ++i) {
      centers[i] = p.center(i);
      flags[i] = p.flags()[i];
    }
  });
}

// ---- NUFFT plan -----------------------------------------------------------

int ref_plan_info(const double* t, int64_t n, const double* c, int64_t nc, double eps, int policy,
                  int oversampling, int64_t* info /* path, width, uniform, mr */, double* tau) {
  return guard([&] {
    const NufftPlan p(SamplingGrid(vec(t, n)), vec(c, nc), eps, policy_of(policy), oversampling);
    info[0] = p.path() == NufftPath::fast ? 1 : 0;
    info[1] = static_cast<int64_t>(p.spread_width());
    info[2] = p.centers_uniform() ? 1 : 0;
    info[3] = static_cast<int64_t>(p.mr_);
    if (tau) *tau = p.tau_;
  });
}

// Private first_cell_ (j0 per sample, nufft.cpp:118-122) — the bit-exact bin contract.
int ref_plan_first_cells(const double* t, int64_t n, const double* c, int64_t nc, double eps,
                         int oversampling, int64_t* out) {
  return guard([&] {
    const NufftPlan p(SamplingGrid(vec(t, n)), vec(c, nc), eps, NufftPathPolicy::force_fast,
                      oversampling);
    for (int64_t i = 0; i < n; ++i) out[i] = p.first_cell_[i];
  });
}

int ref_plan_execute(const double* t, int64_t n, const double* c, int64_t nc, double eps, int policy,
                     int oversampling, const double* y, int64_t ny, double* out) {
  return guard([&] {
    const NufftPlan p(SamplingGrid(vec(t, n)), vec(c, nc), eps, policy_of(policy), oversampling);
    cout_(p.execute(cvec(y, ny)), out);
  });
}

int ref_ndft_direct(const double* t, int64_t n, const double* y, int64_t ny, const double* c,
                    int64_t nc, double* out) {
  return guard([&] { cout_(ndft_direct(SamplingGrid(vec(t, n)), cvec(y, ny), vec(c, nc)), out); });
}

int ref_fft_forward(double* data, int64_t n, int inverse) {
  return guard([&] {
    Radix2Fft f(static_cast<size_t>(n));
    auto* z = reinterpret_cast<cplx*>(data);
    if (inverse) f.inverse(z); else f.forward(z);
  });
}

// ---- tapers ---------------------------------------------------------------

int ref_dpss(int64_t n, double tw, int64_t k, double* tapers, double* conc) {
  return guard([&] {
    const DpssSet d = dpss_uniform(static_cast<size_t>(n), tw, static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) {
      std::copy(d.tapers[j].begin(), d.tapers[j].end(), tapers + j * n);
      if (conc) conc[j] = d.concentrations[j];
    }
  });
}

int ref_tridiagonal_eigen(const double* d, const double* e, int64_t n, int64_t ne, int64_t k,
                          double* values, double* vectors, double* residuals) {
  return guard([&] {
    const EigenPairs p = tridiagonal_eigen(vec(d, n), vec(e, ne), static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) {
      values[j] = p.values[j];
      if (residuals) residuals[j] = p.residuals[j];
      if (vectors)
        for (int64_t i = 0; i < n; ++i) vectors[j * n + i] = p.vectors[j][i].real();
    }
  });
}

int ref_spline(const double* xk, const double* yk, int64_t n, const double* xq, int64_t nq,
               double* out) {
  return guard([&] {
    const CubicSpline s(vec(xk, n), vec(yk, n));
    for (int64_t i = 0; i < nq; ++i) out[i] = s(xq[i]);
  });
}

int ref_signal_band_quadform(const double* t, int64_t n, double f_max, const double* w, int64_t k,
                             double* q) {
  return guard([&] {
    const KernelMatrix rb = signal_band_kernel(SamplingGrid(vec(t, n)), SignalBand(f_max));
    for (int64_t j = 0; j < k; ++j) q[j] = rb.quadratic_form(vec(w + j * n, n));
  });
}

int ref_gpss_interpolated(const double* t, int64_t n, double f_max, double f_w, int64_t k,
                          double* weights) {
  return guard([&] {
    const TaperSet s =
        gpss_interpolated(SamplingGrid(vec(t, n)), SignalBand(f_max), f_w, static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j)
      for (int64_t i = 0; i < n; ++i) weights[j * n + i] = s.weights_real(j)[i];
  });
}

int64_t ref_default_taper_count(double tw) { return static_cast<int64_t>(default_taper_count(tw)); }

// ---- eigencoefficients / estimator (Oracle-A and Oracle-B) -----------------

int ref_eigencoefficients(const double* t, int64_t n, const double* w /*K x N*/, int64_t k,
                          const double* x, const double* c, int64_t nc, double eps, int policy,
                          double f_max, double f_w, double* out /*K x I complex*/) {
  return guard([&] {
    SamplingGrid g(vec(t, n));
    std::vector<std::vector<cplx>> ws(static_cast<size_t>(k), std::vector<cplx>(n));
    for (int64_t j = 0; j < k; ++j)
      for (int64_t i = 0; i < n; ++i) ws[j][i] = {w[j * n + i], 0.0};
    const TaperSet ts(g, AnalysisBand(0.0, f_w), f_max, std::move(ws), {}, true);
    const NufftPlan p(g, vec(c, nc), eps, policy_of(policy));
    const EigenCoefficients j = eigencoefficients(ts, SignalSeries(g, vec(x, n)), p);
    cout_(j.data, out);
  });
}

// Oracle-A: the full reference MtnufftEstimator (setup + estimate).  Feasible
// for N up to ~2^15 (the reference's taper setup is O(N^2)).
int ref_mtnufft(const double* t, int64_t n, const double* x, double f_max, const double* c,
                int64_t nc, double f_w, double margin, int64_t k, double eps, int policy,
                double* power, double* weights /*K x N or null*/, uint8_t* flags) {
  return guard([&] {
    SamplingGrid g(vec(t, n));
    std::vector<AnalysisBand> bands;
    bands.reserve(nc);
    for (int64_t i = 0; i < nc; ++i) bands.emplace_back(c[i], f_w);
    const BandPlan plan(std::move(bands), f_max, margin);
    MtnufftEstimator::Options o;
    o.k_tapers = static_cast<size_t>(k);
    o.epsilon = eps;
    o.path_policy = policy_of(policy);
    const MtnufftEstimator est(g, SignalBand(f_max), plan, o);
    const SpectrumEstimate s = est.estimate(vec(x, n));
    std::copy(s.power.begin(), s.power.end(), power);
    if (flags) std::copy(s.flags.begin(), s.flags.end(), flags);
    if (weights)
      for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < n; ++i) weights[j * n + i] = est.tapers().weights_real(j)[i];
  });
}

// Oracle-B handle: plan built once, estimate many (the per-spectrum path the
// GPU replaces).  Used by the CPU baseline and by parity tests at large N.
void* ref_injected_create(const double* t, int64_t n, const double* w, int64_t k, const double* c,
                          int64_t nc, double eps, int policy, double f_max, double f_w) {
  InjectedEstimator* out = nullptr;
  const int rc = guard([&] {
    std::vector<std::vector<double>> ws(static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) ws[j] = vec(w + j * n, n);
    out = new InjectedEstimator(SamplingGrid(vec(t, n)), std::move(ws), vec(c, nc), eps, policy,
                                f_max, f_w);
  });
  return rc == kOk ? out : nullptr;
}

void ref_injected_destroy(void* h) { delete static_cast<InjectedEstimator*>(h); }

int ref_injected_power(void* h, const double* x, double* out) {
  return guard([&] { static_cast<InjectedEstimator*>(h)->power(x, out); });
}

// Many independent series on the same grid, spread over `threads` host
// threads (the reference path itself is serial per series, nufft.cpp:212-225).
int ref_injected_power_many(void* h, const double* x, int64_t count, int threads, double* out) {
  return guard([&] {
    auto* e = static_cast<InjectedEstimator*>(h);
    const int64_t n = static_cast<int64_t>(e->grid.n_samples());
    const int64_t bands = static_cast<int64_t>(e->plan.n_centers());
    std::atomic<int64_t> next{0};
    std::exception_ptr first;
    std::atomic<bool> failed{false};
    auto worker = [&] {
      for (;;) {
        const int64_t i = next.fetch_add(1);
        if (i >= count || failed.load()) return;
        try {
          e->power(x + i * n, out + i * bands);
        } catch (...) {
          if (!failed.exchange(true)) first = std::current_exception();
        }
      }
    };
    std::vector<std::thread> pool;
    const int nt = std::max(1, threads);
    for (int i = 0; i < nt; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    if (first) std::rethrow_exception(first);
  });
}

// One series, its K tapers spread over `threads` host threads (the plan is immutable and
// execute() is const, nufft.hpp:28-30): |J_k(i)|^2 per taper into out_k [K][bands].
int ref_injected_taper_powers(void* h, const double* x, int threads, double* out_k) {
  return guard([&] {
    auto* e = static_cast<InjectedEstimator*>(h);
    const size_t n = e->grid.n_samples(), bands = e->plan.n_centers(), K = e->weights.size();
    const SignalSeries series(e->grid, vec(x, static_cast<int64_t>(n)));
    std::atomic<size_t> next{0};
    std::exception_ptr first;
    std::atomic<bool> failed{false};
    auto worker = [&] {
      for (;;) {
        const size_t k = next.fetch_add(1);
        if (k >= K || failed.load()) return;
        try {
          std::vector<std::vector<cplx>> one(1, std::vector<cplx>(n));
          for (size_t i = 0; i < n; ++i) one[0][i] = {e->weights[k][i], 0.0};
          const TaperSet t(e->grid, AnalysisBand(0.0, e->f_w), e->f_max, std::move(one), {}, true);
          const EigenCoefficients j = eigencoefficients(t, series, e->plan);
          const cplx* row = j.row(0);
          double* dst = out_k + k * bands;
          for (size_t i = 0; i < bands; ++i) dst[i] = std::norm(row[i]);
        } catch (...) {
          if (!failed.exchange(true)) first = std::current_exception();
        }
      }
    };
    std::vector<std::thread> pool;
    const int nt = std::max(1, std::min<int>(threads, static_cast<int>(K)));
    for (int i = 0; i < nt; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    if (first) std::rethrow_exception(first);
  });
}

// P of one series with the tapers on `threads` threads: the per-taper |J_k|^2 summed over k in
// the serial loop's order (estimators.cpp:113-117), so the result is bit-identical to power().
int ref_injected_power_tapers(void* h, const double* x, int threads, double* out) {
  return guard([&] {
    auto* e = static_cast<InjectedEstimator*>(h);
    const size_t bands = e->plan.n_centers(), K = e->weights.size();
    std::vector<double> pk(K * bands);
    const int rc = ref_injected_taper_powers(h, x, threads, pk.data());
    if (rc != 0) throw std::runtime_error(g_err);
    std::vector<double> p(bands, 0.0);
    for (size_t k = 0; k < K; ++k)
      for (size_t i = 0; i < bands; ++i) p[i] += pk[k * bands + i];
    const double kk = static_cast<double>(K);
    for (size_t i = 0; i < bands; ++i) out[i] = p[i] / kk;
  });
}

// ---- inference: harmonic F-test on eigencoefficients ------

int ref_f_test(const double* t, int64_t n, const double* w, int64_t k, const double* x,
               const double* c, int64_t nc, double eps, int policy, double f_max, double f_w,
               double margin, double cap, double* f_out, double* amp_out, uint8_t* flags,
               double* crit /* 3 */) {
  return guard([&] {
    SamplingGrid g(vec(t, n));
    std::vector<std::vector<cplx>> ws(static_cast<size_t>(k), std::vector<cplx>(n));
    for (int64_t j = 0; j < k; ++j)
      for (int64_t i = 0; i < n; ++i) ws[j][i] = {w[j * n + i], 0.0};
    const TaperSet ts(g, AnalysisBand(0.0, f_w), f_max, std::move(ws), {}, true);
    const NufftPlan p(g, vec(c, nc), eps, policy_of(policy));
    const EigenCoefficients j = eigencoefficients(ts, SignalSeries(g, vec(x, n)), p);
    std::vector<AnalysisBand> bands;
    for (int64_t i = 0; i < nc; ++i) bands.emplace_back(c[i], f_w);
    const BandPlan plan(std::move(bands), f_max, margin);
    FTestOptions o;
    o.saturation_cap = cap;
    const FTestResult r = f_test(j, ts, plan, o);
    for (int64_t i = 0; i < nc; ++i) {
      f_out[i] = r.f_stat[i];
      amp_out[2 * i] = r.amplitude[i].real();
      amp_out[2 * i + 1] = r.amplitude[i].imag();
      flags[i] = r.flags[i];
    }
    for (size_t q = 0; q < r.critical_values.size() && q < 3; ++q) crit[q] = r.critical_values[q].second;
  });
}

int ref_f_quantile(double p, int64_t d1, int64_t d2, double* out) {
  return guard([&] { *out = f_quantile(p, static_cast<size_t>(d1), static_cast<size_t>(d2)); });
}

// ---- MTNUFFT0: exact nominal-band GPSS by the dense GEP ----------------

// generalized_hermitian_eigen (eig.cpp:612-659) on dense row-major host matrices
int ref_generalized_eigen(const double* a_re, const double* a_im /*null: real*/, const double* m, int64_t n,
                          int64_t k, double ridge_first, double ridge_retry, double* values,
                          double* vectors /*complex [k][n] or null*/, double* residuals) {
  return guard([&] {
    KernelMatrix A(static_cast<size_t>(n), a_im == nullptr, "A");
    KernelMatrix M(static_cast<size_t>(n), true, "B");
    std::copy(a_re, a_re + n * n, A.re_data());
    if (a_im) std::copy(a_im, a_im + n * n, A.im_data());
    std::copy(m, m + n * n, M.re_data());
    GeneralizedEigenOptions o;
    o.ridge_first = ridge_first;
    o.ridge_retry = ridge_retry;
    o.want_vectors = vectors != nullptr;
    const EigenPairs p = generalized_hermitian_eigen(A, M, static_cast<size_t>(k), o);
    for (size_t j = 0; j < p.count(); ++j) {
      values[j] = p.values[j];
      if (vectors) {
        for (int64_t i = 0; i < n; ++i) {
          vectors[2 * (j * n + i)] = p.vectors[j][i].real();
          vectors[2 * (j * n + i) + 1] = p.vectors[j][i].imag();
        }
        residuals[j] = p.residuals[j];
      }
    }
  });
}

// gpss_exact (tapers.cpp:118-144): normalised weights [k][n] complex + concentrations
int ref_gpss_exact(const double* t, int64_t n, double f_max, double f_c, double f_w, int64_t k, double* w,
                   double* conc) {
  return guard([&] {
    SamplingGrid g(vec(t, n));
    const TaperSet ts = gpss_exact(g, SignalBand(f_max), AnalysisBand(f_c, f_w), static_cast<size_t>(k));
    for (size_t j = 0; j < ts.k_tapers(); ++j) {
      const auto& wj = ts.weights(j);
      for (int64_t i = 0; i < n; ++i) {
        w[2 * (j * n + i)] = wj[i].real();
        w[2 * (j * n + i) + 1] = wj[i].imag();
      }
      conc[j] = ts.eigenvalues()[j];
    }
  });
}

// MtnufftEstimator with taper_mode = exact_nominal (estimators.cpp:91-104): MTNUFFT0 P(f)
int ref_mtnufft0(const double* t, int64_t n, const double* x, double f_max, const double* c, int64_t nc,
                 double f_w, double margin, int64_t k, double eps, double* power, double* weights /*k x n real*/,
                 int32_t* method) {
  return guard([&] {
    SamplingGrid g(vec(t, n));
    std::vector<AnalysisBand> bands;
    for (int64_t i = 0; i < nc; ++i) bands.emplace_back(c[i], f_w);
    const BandPlan plan(std::move(bands), f_max, margin);
    MtnufftEstimator::Options o;
    o.k_tapers = static_cast<size_t>(k);
    o.epsilon = eps;
    o.taper_mode = TaperMode::exact_nominal;
    const MtnufftEstimator est(g, SignalBand(f_max), plan, o);
    const SpectrumEstimate s = est.estimate(vec(x, n));
    std::copy(s.power.begin(), s.power.end(), power);
    if (weights)
      for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < n; ++i) weights[j * n + i] = est.tapers().weights_real(j)[i];
    *method = static_cast<int32_t>(est.method());
  });
}

// ---- speed / error harness (bench.cpp:130-275) -------------------------

// run_error_analysis: reports in (scheme-major, method-minor) order; per report the band
// centres, mse_db_mean, mse_db_sem and flags (bands entries each, NaN where failed)
int ref_run_error_analysis(const int32_t* methods, int64_t nm, const int32_t* schemes, int64_t ns, int64_t trials,
                           uint64_t base_seed, double f_max, double f_w, int64_t k, double spacing, int64_t n_samples,
                           double eps, int64_t cap_bands, double* centers, double* mean, double* sem,
                           uint8_t* flags, int64_t* bands_out, int64_t* failed_out) {
  return guard([&] {
    std::vector<EstimatorMethod> ms;
    for (int64_t i = 0; i < nm; ++i) ms.push_back(static_cast<EstimatorMethod>(methods[i]));
    std::vector<SamplingScheme> ss;
    for (int64_t i = 0; i < ns; ++i) ss.push_back(static_cast<SamplingScheme>(schemes[i]));
    BenchConfig cfg;
    cfg.f_max = f_max;
    cfg.f_w = f_w;
    cfg.k_tapers = static_cast<size_t>(k);
    cfg.spacing = spacing;
    cfg.n_samples = static_cast<size_t>(n_samples);
    cfg.epsilon = eps;
    const auto reps = run_error_analysis(ms, ss, static_cast<size_t>(trials), base_seed, cfg);
    for (size_t r = 0; r < reps.size(); ++r) {
      const auto& rep = reps[r];
      const int64_t b = static_cast<int64_t>(rep.centers.size());
      if (b > cap_bands) throw std::runtime_error("capacity");
      *bands_out = b;
      failed_out[r] = static_cast<int64_t>(rep.failed_bands);
      for (int64_t i = 0; i < b; ++i) {
        centers[r * cap_bands + i] = rep.centers[i];
        mean[r * cap_bands + i] = rep.mse_db_mean[i];
        sem[r * cap_bands + i] = rep.mse_db_sem[i];
        flags[r * cap_bands + i] = rep.flags[i];
      }
    }
  });
}

// ---- reference RNG / grids used by the reference's own tests ---------------

int ref_rng_gauss(uint64_t seed, int64_t count, double* out) {
  return guard([&] {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.next_gauss();
  });
}

int ref_rng_uniform(uint64_t seed, int64_t count, double* out) {
  return guard([&] {
    Rng r(seed);
    for (int64_t i = 0; i < count; ++i) out[i] = r.next_uniform();
  });
}

// scheme: 0 uniform, 1 jitter, 2 missing, 3 arithmetic (simkit.hpp SimConfig defaults otherwise)
int ref_generate_grid(int scheme, int64_t n, uint64_t seed, double jitter_sigma, double* out,
                      int64_t* count) {
  return guard([&] {
    SimConfig cfg;
    cfg.scheme = static_cast<SamplingScheme>(scheme);
    cfg.n = static_cast<size_t>(n);
    cfg.seed = seed;
    if (jitter_sigma >= 0) cfg.jitter_sigma = jitter_sigma;
    const SamplingGrid g = generate_grid(cfg);
    *count = static_cast<int64_t>(g.n_samples());
    std::copy(g.times().begin(), g.times().end(), out);
  });
}

int ref_line_plus_noise(const double* t, int64_t n, double freq, double amp, double phase,
                        double noise_var, uint64_t seed, double* out) {
  return guard([&] {
    const SignalSeries s = generate_line_plus_noise(SamplingGrid(vec(t, n)), freq, amp, phase,
                                                    noise_var, seed);
    std::copy(s.values.begin(), s.values.end(), out);
  });
}

}  // extern "C"
