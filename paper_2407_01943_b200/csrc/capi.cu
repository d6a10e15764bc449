#include <cstdio>
// extern "C" boundary (include/nus_c.h).  Every entry point converts internal
// failures into status codes + a thread-local message; nothing throws across
// the ABI.
#include <cmath>
#include <cstring>
#include <functional>
#include <string>

#include "nus_estimator.cuh"

struct nus_plan_s {
  std::unique_ptr<nus::Plan> plan;
};
struct nus_mtnufft_s {
  std::unique_ptr<nus::Estimator> est;
};

struct nus_mtnufft_multi_s {
  nus::MultiPtr m;
  std::mutex mu;
};

namespace {

thread_local std::string g_last_error;

int guarded(const std::function<void()>& fn) {
  try {
    fn();
    return NUS_OK;
  } catch (const nus::Failure& f) {
    g_last_error = f.what();
    return f.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return NUS_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return NUS_ERR_CUDA;
  } catch (...) {
    g_last_error = "unknown failure";
    return NUS_ERR_CUDA;
  }
}

__global__ void f32c_to_f64c(const float* __restrict__ a, int64_t n, double* __restrict__ b) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g < n) b[g] = static_cast<double>(a[g]);
}

void fill_info(const nus::Plan& pl, nus_plan_info_t* info) {
  const auto& p = pl.p;
  info->n_samples = p.n;
  info->n_centers = p.nc;
  info->epsilon = p.eps;
  info->oversampling = p.oversampling;
  info->path = p.path;
  info->centers_uniform = p.uniform ? 1 : 0;
  info->precision = p.precision;
  info->spread_width = p.w;
  info->mr = p.path == NUS_PATH_FAST ? p.mr : 0;
  info->tau = p.tau;
  info->df = p.df;
  info->fshift = p.fshift;
  info->kernel = p.kernel;
  info->support = p.sw;
}

// Execute the transform of one complex vector already on the device.
void plan_execute_one(nus::Plan& pl, const void* y_dev, bool y_f32, void* out_dev, cudaStream_t s) {
  const auto& p = pl.p;
  if (p.path == NUS_PATH_FAST) {
    const size_t rs = p.precision == NUS_F64 ? sizeof(double) : sizeof(float);
    if (pl.work.bytes < static_cast<size_t>(p.mr) * 2 * rs) pl.work.alloc(static_cast<size_t>(p.mr) * 2 * rs);
    nus::SpreadArgs a;
    a.x = y_dev;
    a.x_dtype = y_f32 ? 1 : 0;
    a.x_complex = true;
    a.k = 1;
    a.kpad = 1;
    a.grid = pl.work.ptr;
    nus::launch_spread(pl, a, s);
    nus::run_transform(pl, pl.work.ptr, 1, 1, out_dev, nullptr, false, 1.0, false, s);
  } else {
    nus::launch_ndft_direct(pl.d_times.as<double>(), p.n, y_dev, y_f32, pl.d_centers.as<double>(), p.nc,
                            out_dev, p.precision == NUS_F32, 1, s);
  }
}

}  // namespace

extern "C" {

const char* nus_last_error(void) { return g_last_error.c_str(); }

int64_t nus_kernel_launch_count(void) { return nus::g_launches.load(); }

int nus_set_spread_kernel(int32_t kind) {
  return guarded([&] {
    nus::require(kind == NUS_KERNEL_GAUSSIAN || kind == NUS_KERNEL_ES, "unknown spreading kernel");
    nus::set_default_kernel(kind);
  });
}

int nus_get_spread_kernel(int32_t* kind) {
  return guarded([&] {
    nus::require(kind != nullptr, "null output");
    *kind = nus::default_kernel();
  });
}

int nus_device_info(int device, int32_t* cc_major, int32_t* cc_minor, int32_t* sm_count,
                    int64_t* total_mem) {
  return guarded([&] {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      nus::fail(NUS_ERR_NO_DEVICE, "no CUDA device visible");
    }
    cudaDeviceProp prop;
    NUS_CUDA(cudaGetDeviceProperties(&prop, device));
    if (cc_major) *cc_major = prop.major;
    if (cc_minor) *cc_minor = prop.minor;
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (total_mem) *total_mem = static_cast<int64_t>(prop.totalGlobalMem);
  });
}

// ---- plan ---------------------------------------------------------------------

int nus_plan_create(const double* times, int64_t n, const double* centers, int64_t n_centers,
                    double epsilon, int32_t policy, int32_t oversampling, int32_t precision,
                    int32_t device, nus_plan_t* out) {
  return guarded([&] {
    nus::require(out != nullptr, "nus_plan_create: null output handle");
    auto h = new nus_plan_s;
    try {
      h->plan = nus::plan_create(times, 1, n, centers, n_centers, epsilon, policy, oversampling,
                                 precision, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int nus_plan_destroy(nus_plan_t plan) {
  return guarded([&] { delete plan; });
}

int nus_plan_info(nus_plan_t plan, nus_plan_info_t* info) {
  return guarded([&] {
    nus::require(plan && info, "nus_plan_info: null argument");
    fill_info(*plan->plan, info);
  });
}

int nus_plan_first_cells(nus_plan_t plan, int64_t* out_host) {
  return guarded([&] {
    nus::require(plan && out_host, "nus_plan_first_cells: null argument");
    auto& pl = *plan->plan;
    nus::require(pl.p.path == NUS_PATH_FAST, "nus_plan_first_cells: plan is on the direct path");
    nus::use_device(pl.device);
    NUS_CUDA(cudaMemcpy(out_host, pl.tab.first_cell.ptr, pl.p.n * pl.p.channels * sizeof(int64_t),
                        cudaMemcpyDeviceToHost));
  });
}

int nus_plan_sort_order(nus_plan_t plan, int32_t* perm_host) {
  return guarded([&] {
    nus::require(plan && perm_host, "nus_plan_sort_order: null argument");
    auto& pl = *plan->plan;
    nus::require(pl.p.path == NUS_PATH_FAST, "nus_plan_sort_order: plan is on the direct path");
    nus::use_device(pl.device);
    NUS_CUDA(cudaMemcpy(perm_host, pl.tab.perm.ptr, pl.p.n * pl.p.channels * sizeof(int32_t),
                        cudaMemcpyDeviceToHost));
  });
}

int nus_plan_execute(nus_plan_t plan, const double* y_host, int64_t n_y, double* out_host) {
  return guarded([&] {
    nus::require(plan && y_host && out_host, "nus_plan_execute: null argument");
    auto& pl = *plan->plan;
    if (n_y != pl.p.n) nus::fail(NUS_ERR_PLAN_MISMATCH, "NufftPlan: input length does not match plan grid");
    std::lock_guard<std::mutex> lock(pl.mu);
    nus::use_device(pl.device);
    const bool f32 = pl.p.precision == NUS_F32;
    nus::DeviceBuffer y(pl.p.n * 2 * sizeof(double));
    nus::DeviceBuffer out(pl.p.nc * 2 * (f32 ? sizeof(float) : sizeof(double)));
    NUS_CUDA(cudaMemcpy(y.ptr, y_host, y.bytes, cudaMemcpyHostToDevice));
    plan_execute_one(pl, y.ptr, false, out.ptr, 0);
    if (f32) {
      nus::DeviceBuffer o64(pl.p.nc * 2 * sizeof(double));
      f32c_to_f64c<<<static_cast<unsigned>((2 * pl.p.nc + 255) / 256), 256>>>(out.as<float>(), 2 * pl.p.nc,
                                                                             o64.as<double>());
      nus::note_launch();
      NUS_CUDA(cudaMemcpy(out_host, o64.ptr, o64.bytes, cudaMemcpyDeviceToHost));
    } else {
      NUS_CUDA(cudaMemcpy(out_host, out.ptr, out.bytes, cudaMemcpyDeviceToHost));
    }
  });
}

int nus_plan_execute_device(nus_plan_t plan, const void* y_dev, int64_t batch, void* out_dev,
                            void* stream) {
  return guarded([&] {
    nus::require(plan && y_dev && out_dev && batch >= 1, "nus_plan_execute_device: bad argument");
    auto& pl = *plan->plan;
    std::lock_guard<std::mutex> lock(pl.mu);
    nus::use_device(pl.device);
    const bool f32 = pl.p.precision == NUS_F32;
    const size_t rs = f32 ? sizeof(float) : sizeof(double);
    auto s = static_cast<cudaStream_t>(stream);
    for (int64_t b = 0; b < batch; ++b)
      plan_execute_one(pl, static_cast<const char*>(y_dev) + b * pl.p.n * 2 * rs, f32,
                       static_cast<char*>(out_dev) + b * pl.p.nc * 2 * rs, s);
  });
}

int nus_ndft_direct(const double* times, int64_t n, const double* y_host, const double* centers,
                    int64_t n_centers, int32_t device, double* out_host) {
  return guarded([&] {
    nus::require(times && y_host && centers && out_host, "ndft_direct: null argument");
    nus::require(n >= 1 && n_centers >= 1, "ndft_direct: empty input");
    nus::use_device(device);
    nus::DeviceBuffer t(n * sizeof(double)), y(n * 2 * sizeof(double)), c(n_centers * sizeof(double)),
        o(n_centers * 2 * sizeof(double));
    NUS_CUDA(cudaMemcpy(t.ptr, times, t.bytes, cudaMemcpyHostToDevice));
    NUS_CUDA(cudaMemcpy(y.ptr, y_host, y.bytes, cudaMemcpyHostToDevice));
    NUS_CUDA(cudaMemcpy(c.ptr, centers, c.bytes, cudaMemcpyHostToDevice));
    nus::launch_ndft_direct(t.as<double>(), n, y.ptr, false, c.as<double>(), n_centers, o.ptr, false, 1, 0);
    NUS_CUDA(cudaMemcpy(out_host, o.ptr, o.bytes, cudaMemcpyDeviceToHost));
  });
}

namespace {
__global__ void signal_band_matrix_kernel(const double* __restrict__ t, int64_t n, double f,
                                          double tol, double* __restrict__ m) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * n) return;
  const int64_t r = g / n, c = g - r * n;
  double v;
  if (r == c) {
    v = 2.0 * f;
  } else {
    const double d = t[r] - t[c];
    v = fabs(d) < tol ? 2.0 * f : sin(2.0 * nus::kPi * f * d) / (nus::kPi * d);  // kernels.cpp:16-19
  }
  m[g] = v;
}
}  // namespace

int nus_fft_inplace(double* data_host, int64_t n, int32_t inverse, int32_t device) {
  return guarded([&] {
    nus::require(data_host != nullptr, "Radix2Fft: null data");
    nus::require(n > 0 && (n & (n - 1)) == 0, "Radix2Fft: size must be a power of two");
    nus::use_device(device);
    nus::DeviceBuffer d(n * 2 * sizeof(double));
    NUS_CUDA(cudaMemcpy(d.ptr, data_host, d.bytes, cudaMemcpyHostToDevice));
    nus::fft_generic_inplace(d.ptr, n, 1, true, inverse != 0, 0);  // own kernels (fft.cu)
    NUS_CUDA(cudaMemcpy(data_host, d.ptr, d.bytes, cudaMemcpyDeviceToHost));
  });
}

int nus_signal_band_matrix(const double* times, int64_t n, double f_max, int32_t device,
                           double* out_host) {
  return guarded([&] {
    nus::require(times && out_host, "signal_band_kernel: null argument");
    nus::require(n >= 1, "signal_band_kernel: empty grid");
    nus::use_device(device);
    nus::DeviceBuffer t(n * sizeof(double)), m(static_cast<size_t>(n) * n * sizeof(double));
    NUS_CUDA(cudaMemcpy(t.ptr, times, t.bytes, cudaMemcpyHostToDevice));
    const double mean_dt = n > 0 ? (times[n - 1] - times[0]) / static_cast<double>(n) : 0.0;
    signal_band_matrix_kernel<<<static_cast<unsigned>((n * n + 255) / 256), 256>>>(
        t.as<double>(), n, f_max, 1e-12 * mean_dt, m.as<double>());
    nus::note_launch();
    nus::check_launch("signal_band_matrix_kernel");
    NUS_CUDA(cudaMemcpy(out_host, m.ptr, m.bytes, cudaMemcpyDeviceToHost));
  });
}

// ---- MTNUFFT0: exact nominal-band GPSS (gep.cu) -------------------------

int nus_generalized_eigen(const double* a_re, const double* a_im, const double* m, int64_t n, int64_t k,
                          double ridge_first, double ridge_retry, int32_t want_vectors, int32_t device,
                          double* values, double* vectors, double* residuals) {
  return guarded([&] {
    nus::require(a_re && m && values, "generalized_hermitian_eigen: null argument");
    nus::require(!want_vectors || (vectors && residuals), "generalized_hermitian_eigen: null vector output");
    nus::require(n >= 1 && k >= 1, "generalized_hermitian_eigen: k_top must be >= 1");
    nus::use_device(device);
    const size_t nn = static_cast<size_t>(n) * n;
    nus::DeviceBuffer dre(nn * sizeof(double)), dm(nn * sizeof(double)), dim(a_im ? nn * sizeof(double) : 0);
    NUS_CUDA(cudaMemcpy(dre.ptr, a_re, dre.bytes, cudaMemcpyHostToDevice));
    NUS_CUDA(cudaMemcpy(dm.ptr, m, dm.bytes, cudaMemcpyHostToDevice));
    if (a_im) {  // row-major Hermitian read column-major is conj(A): flip the imaginary part
      std::vector<double> neg(a_im, a_im + nn);
      for (double& v : neg) v = -v;
      NUS_CUDA(cudaMemcpy(dim.ptr, neg.data(), dim.bytes, cudaMemcpyHostToDevice));
    }
    nus::generalized_eigen_device(dre.as<double>(), a_im ? dim.as<double>() : nullptr, dm.as<double>(), n, k,
                                  ridge_first, ridge_retry, want_vectors != 0, values, vectors, residuals);
  });
}

int nus_band_matrix(const double* times, int64_t n, double f_w, double f_center, int32_t device, double* re_out,
                    double* im_out) {
  return guarded([&] {
    nus::require(times && re_out, "analysis_band_kernel: null argument");
    nus::require(n >= 1, "analysis_band_kernel: empty grid");
    nus::use_device(device);
    const size_t nn = static_cast<size_t>(n) * n;
    nus::DeviceBuffer t(n * sizeof(double)), re(nn * sizeof(double)), im(im_out ? nn * sizeof(double) : 0);
    NUS_CUDA(cudaMemcpy(t.ptr, times, t.bytes, cudaMemcpyHostToDevice));
    const double mean_dt = (times[n - 1] - times[0]) / static_cast<double>(n);
    nus::band_matrix_rowmajor(t.as<double>(), n, f_w, f_center, 1e-12 * mean_dt, re.as<double>(),
                              im_out ? im.as<double>() : nullptr);
    NUS_CUDA(cudaMemcpy(re_out, re.ptr, re.bytes, cudaMemcpyDeviceToHost));
    if (im_out) NUS_CUDA(cudaMemcpy(im_out, im.ptr, im.bytes, cudaMemcpyDeviceToHost));
  });
}

int nus_gpss_exact(const double* times, int64_t n, double f_max, double f_center, double f_w, int64_t k,
                   double ridge_first, double ridge_retry, int32_t device, double* w_out, double* concentrations) {
  return guarded([&] {
    nus::require(times && w_out && concentrations, "gpss_exact: null argument");
    nus::require(n >= 2, "gpss_exact: need at least 2 samples");
    nus::use_device(device);
    nus::gpss_exact_device(times, n, f_max, f_center, f_w, k, ridge_first, ridge_retry, w_out, concentrations);
  });
}

// ---- tapers -----------------------------------------------------------------------

int nus_dpss(int64_t n, double tw, int64_t k, int32_t device, double* tapers_host,
             double* eigenvalues_host, double* concentrations_host) {
  return guarded([&] {
    nus::use_device(device);
    nus::require(n >= 2, "dpss_uniform: n must be >= 2");
    nus::require(k >= 1 && k <= n, "dpss_uniform: k_tapers out of range");
    nus::DeviceBuffer v(static_cast<size_t>(k) * n * sizeof(double));
    const nus::DpssResult r = nus::dpss_device(n, tw, k, v.as<double>(), 0);
    if (eigenvalues_host) std::memcpy(eigenvalues_host, r.values.data(), k * sizeof(double));
    if (concentrations_host) nus::dpss_concentrations(n, tw, k, v.as<double>(), concentrations_host, 0);
    if (tapers_host) NUS_CUDA(cudaMemcpy(tapers_host, v.ptr, v.bytes, cudaMemcpyDeviceToHost));
  });
}

int nus_tridiagonal_eigen(const double* diag, const double* offdiag, int64_t n, int64_t k,
                          int32_t device, double* values, double* vectors, double* residuals) {
  return guarded([&] {
    nus::require(diag && offdiag && values, "tridiagonal_eigen: null argument");
    nus::require(n >= 1, "tridiagonal_eigenvalues: empty matrix");
    nus::require(k >= 1 && k <= n, "tridiagonal_eigen: k_top out of range");
    nus::use_device(device);
    nus::DeviceBuffer d(n * sizeof(double)), e(std::max<int64_t>(n - 1, 1) * sizeof(double)),
        v(static_cast<size_t>(k) * n * sizeof(double));
    NUS_CUDA(cudaMemcpy(d.ptr, diag, n * sizeof(double), cudaMemcpyHostToDevice));
    if (n > 1) NUS_CUDA(cudaMemcpy(e.ptr, offdiag, (n - 1) * sizeof(double), cudaMemcpyHostToDevice));
    const nus::DpssResult r = nus::tridiag_top_device(d.as<double>(), e.as<double>(), n, k, v.as<double>(), 0);
    std::memcpy(values, r.values.data(), k * sizeof(double));
    std::vector<double> hv(static_cast<size_t>(k) * n);
    NUS_CUDA(cudaMemcpy(hv.data(), v.ptr, v.bytes, cudaMemcpyDeviceToHost));
    if (vectors) std::memcpy(vectors, hv.data(), hv.size() * sizeof(double));
    if (residuals) {
      // ||T v - lambda v|| / ||T||_inf  (eig.cpp:602-606), host O(n k)
      double anorm = 0;
      for (int64_t i = 0; i < n; ++i) {
        double row = std::fabs(diag[i]);
        if (i > 0) row += std::fabs(offdiag[i - 1]);
        if (i + 1 < n) row += std::fabs(offdiag[i]);
        anorm = std::max(anorm, row);
      }
      anorm = std::max(anorm, 2.2250738585072014e-308);
      for (int64_t j = 0; j < k; ++j) {
        const double* x = hv.data() + j * n;
        double r2 = 0;
        for (int64_t i = 0; i < n; ++i) {
          double t = (diag[i] - r.values[j]) * x[i];
          if (i > 0) t += offdiag[i - 1] * x[i - 1];
          if (i + 1 < n) t += offdiag[i] * x[i + 1];
          r2 += t * t;
        }
        residuals[j] = std::sqrt(r2) / anorm;
      }
    }
  });
}

int nus_signal_band_quadform(const double* times, int64_t n, double f_max, const double* w_host,
                             int64_t k, int64_t row_begin, int64_t row_end, int32_t device,
                             double* q_host) {
  return guarded([&] {
    nus::require(times && w_host && q_host, "quadratic_form: null argument");
    nus::require(n >= 2, "SamplingGrid: need at least 2 samples");
    nus::require(f_max > 0.0 && std::isfinite(f_max), "SignalBand: f_max must be positive");
    nus::use_device(device);
    nus::DeviceBuffer t(n * sizeof(double)), w(static_cast<size_t>(k) * n * sizeof(double));
    NUS_CUDA(cudaMemcpy(t.ptr, times, t.bytes, cudaMemcpyHostToDevice));
    NUS_CUDA(cudaMemcpy(w.ptr, w_host, w.bytes, cudaMemcpyHostToDevice));
    for (int64_t k0 = 0; k0 < k; k0 += 8) {
      const int64_t kk = std::min<int64_t>(8, k - k0);
      nus::quadform_device(t.as<double>(), n, f_max, w.as<double>() + k0 * n, kk, row_begin, row_end,
                           q_host + k0, 0);
    }
  });
}

int nus_signal_band_quadform_fast(const double* times, int64_t n, double f_max, const double* w_host,
                                  int64_t k, int32_t device, double* q_host) {
  return guarded([&] {
    nus::require(times && w_host && q_host, "quadratic_form: null argument");
    nus::require(n >= 2, "SamplingGrid: need at least 2 samples");
    nus::require(f_max > 0.0 && std::isfinite(f_max), "SignalBand: f_max must be positive");
    nus::use_device(device);
    nus::DeviceBuffer t(n * sizeof(double)), w(static_cast<size_t>(k) * n * sizeof(double));
    NUS_CUDA(cudaMemcpy(t.ptr, times, t.bytes, cudaMemcpyHostToDevice));
    NUS_CUDA(cudaMemcpy(w.ptr, w_host, w.bytes, cudaMemcpyHostToDevice));
    nus::quadform_fast_device(t.as<double>(), times, n, f_max, w.as<double>(), k, q_host, 0, device);
  });
}

int nus_taper_spline(const double* times, int64_t n, double f_max, double f_w, int64_t k,
                     int32_t device, double* w_host) {
  return guarded([&] {
    nus::require(times && w_host, "taper_spline: null argument");
    nus::require(n >= 8, "gpss_interpolated: need at least 8 samples");
    nus::require(f_w > 0.0, "gpss_interpolated: f_w must be positive");
    if (!(f_w <= f_max + 1e-12 * f_max))
      nus::fail(NUS_ERR_BAND_RANGE, "gpss_interpolated: nominal band not inside signal band");
    const double h = (times[n - 1] - times[0]) / static_cast<double>(n - 1);
    const double tw = f_w * h * static_cast<double>(n);
    nus::require(tw < static_cast<double>(n) / 2.0, "gpss_interpolated: f_w too large for this grid");
    nus::use_device(device);
    nus::DeviceBuffer t(n * sizeof(double)), dp(static_cast<size_t>(k) * n * sizeof(double)),
        w(static_cast<size_t>(k) * n * sizeof(double));
    NUS_CUDA(cudaMemcpy(t.ptr, times, t.bytes, cudaMemcpyHostToDevice));
    nus::dpss_device(n, tw, k, dp.as<double>(), 0);
    nus::spline_uniform_device(t.as<double>(), n, dp.as<double>(), k, w.as<double>(), 0);
    NUS_CUDA(cudaMemcpy(w_host, w.ptr, w.bytes, cudaMemcpyDeviceToHost));
  });
}

int nus_gpss_interpolated(const double* times, int64_t n, double f_max, double f_w, int64_t k,
                          int32_t device, double* weights_host) {
  return guarded([&] {
    nus::require(times && weights_host, "gpss_interpolated: null argument");
    nus::require(n >= 2, "SamplingGrid: need at least 2 samples");
    nus::require(f_max > 0.0 && std::isfinite(f_max), "SignalBand: f_max must be positive");
    nus::use_device(device);
    nus::DeviceBuffer t(n * sizeof(double)), w(static_cast<size_t>(std::max<int64_t>(k, 1)) * n * sizeof(double));
    NUS_CUDA(cudaMemcpy(t.ptr, times, t.bytes, cudaMemcpyHostToDevice));
    nus::gpss_interpolated_device(t.as<double>(), times, n, f_max, f_w, k, w.as<double>(), 0);
    NUS_CUDA(cudaMemcpy(weights_host, w.ptr, static_cast<size_t>(k) * n * sizeof(double),
                        cudaMemcpyDeviceToHost));
  });
}

// ---- estimator --------------------------------------------------------------------

int nus_mtnufft_create(const nus_mtnufft_config_t* cfg, const double* times, const double* centers,
                       const double* tapers, nus_mtnufft_t* out) {
  return nus_mtnufft_create_channels(cfg, times, centers, nullptr, tapers, out);
}

int nus_mtnufft_create_channels(const nus_mtnufft_config_t* cfg, const double* times, const double* centers,
                                const double* f_w, const double* tapers, nus_mtnufft_t* out) {
  return guarded([&] {
    nus::require(cfg && out, "nus_mtnufft_create: null argument");
    auto h = new nus_mtnufft_s;
    try {
      h->est = nus::estimator_create(*cfg, times, centers, tapers, f_w);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int nus_mtnufft_multi_create(const nus_mtnufft_config_t* cfg, const int32_t* devices, int32_t n_devices,
                             int32_t sharding, const double* times, const double* centers, const double* f_w,
                             const double* tapers, nus_mtnufft_multi_t* out) {
  return guarded([&] {
    nus::require(cfg && out, "nus_mtnufft_multi_create: null argument");
    auto h = std::make_unique<nus_mtnufft_multi_s>();
    h->m = nus::multi_create(*cfg, devices, n_devices, sharding, times, centers, f_w, tapers);
    *out = h.release();
  });
}

int nus_mtnufft_multi_destroy(nus_mtnufft_multi_t est) {
  return guarded([&] { delete est; });
}

int nus_mtnufft_multi_estimate(nus_mtnufft_multi_t est, const double* x_host, double* power_host) {
  return guarded([&] {
    nus::require(est && x_host && power_host, "multi estimate: null argument");
    std::lock_guard<std::mutex> lock(est->mu);
    nus::multi_estimate(*est->m, x_host, power_host);
  });
}

int nus_mtnufft_multi_tapers(nus_mtnufft_multi_t est, double* out_host) {
  return guarded([&] {
    nus::require(est && out_host, "multi tapers: null argument");
    nus::multi_tapers(*est->m, out_host);
  });
}

int nus_mtnufft_multi_peer_bytes(nus_mtnufft_multi_t est, int64_t* bytes) {
  return guarded([&] {
    nus::require(est && bytes, "multi peer bytes: null argument");
    *bytes = nus::multi_peer_bytes(*est->m);
  });
}

int nus_mtnufft_destroy(nus_mtnufft_t est) {
  return guarded([&] { delete est; });
}

int nus_mtnufft_plan_info(nus_mtnufft_t est, nus_plan_info_t* info) {
  return guarded([&] {
    nus::require(est && info, "nus_mtnufft_plan_info: null argument");
    fill_info(*est->est->plan, info);
  });
}

int nus_mtnufft_tapers(nus_mtnufft_t est, double* out_host) {
  return guarded([&] {
    nus::require(est && out_host, "nus_mtnufft_tapers: null argument");
    auto& e = *est->est;
    nus::use_device(e.cfg.device);
    NUS_CUDA(cudaMemcpy(out_host, e.tapers_time.ptr, e.tapers_time.bytes, cudaMemcpyDeviceToHost));
  });
}

int nus_mtnufft_setup_ms(nus_mtnufft_t est, double* out5) {
  return guarded([&] {
    nus::require(est && out5, "nus_mtnufft_setup_ms: null argument");
    std::memcpy(out5, est->est->setup_ms, 5 * sizeof(double));
  });
}

int nus_mtnufft_estimate(nus_mtnufft_t est, const double* x_host, double* power_host) {
  return guarded([&] {
    nus::require(est && x_host && power_host, "estimate: null argument");
    nus::estimator_estimate_host(*est->est, x_host, power_host, nullptr);
  });
}

int nus_mtnufft_estimate_batch(nus_mtnufft_t est, const double* x_host, int64_t steps, double* power_host) {
  return guarded([&] {
    nus::require(est && x_host && power_host, "estimate_batch: null argument");
    nus::require(steps >= 1, "estimate_batch: steps must be >= 1");
    nus::estimator_estimate_batch_host(*est->est, x_host, steps, power_host);
  });
}

int nus_mtnufft_eigencoefficients(nus_mtnufft_t est, const double* x_host, double* j_host) {
  return guarded([&] {
    nus::require(est && x_host && j_host, "eigencoefficients: null argument");
    nus::estimator_estimate_host(*est->est, x_host, nullptr, j_host);
  });
}

int nus_mtnufft_estimate_device(nus_mtnufft_t est, const void* x_dev, int32_t x_dtype,
                                void* power_dev, void* j_dev, void* stream) {
  return guarded([&] {
    nus::require(est && x_dev, "estimate_device: null argument");
    auto& e = *est->est;
    std::lock_guard<std::mutex> lock(e.mu);
    nus::use_device(e.cfg.device);
    nus::estimator_run(e, x_dev, x_dtype, power_dev, false, j_dev, static_cast<cudaStream_t>(stream));
  });
}

int nus_mtnufft_spread_device(nus_mtnufft_t est, const void* x_dev, int32_t x_dtype, int64_t s0,
                              int64_t s1, void* grid_dev, int64_t k_pad, void* stream) {
  return guarded([&] {
    nus::require(est && x_dev && grid_dev, "spread_device: null argument");
    auto& e = *est->est;
    nus::require(e.plan->p.path == NUS_PATH_FAST, "spread_device: estimator is on the direct path");
    nus::require(k_pad >= e.cfg.k_tapers, "spread_device: k_pad < K");
    nus::require(0 <= s0 && s0 <= s1 && s1 <= e.cfg.n, "spread_device: bad sample range");
    nus::use_device(e.cfg.device);
    nus::SpreadArgs a;
    a.x = x_dev;
    a.x_dtype = x_dtype;
    a.tapers = e.tapers_sorted.ptr;
    a.k = e.cfg.k_tapers;
    a.kpad = k_pad;
    a.s0 = s0;
    a.s1 = s1;
    a.grid = grid_dev;
    nus::launch_spread(*e.plan, a, static_cast<cudaStream_t>(stream));
  });
}

int nus_mtnufft_transform_device(nus_mtnufft_t est, void* grid_dev, int64_t k0, int64_t k1,
                                 double divisor, int32_t accumulate, void* power_dev, void* stream) {
  return guarded([&] {
    nus::require(est && grid_dev && power_dev, "transform_device: null argument");
    auto& e = *est->est;
    nus::require(e.plan->p.path == NUS_PATH_FAST, "transform_device: estimator is on the direct path");
    nus::require(0 <= k0 && k0 <= k1, "transform_device: bad taper range");
    nus::require(divisor > 0.0, "transform_device: divisor must be positive");
    if (k1 == k0) return;
    std::lock_guard<std::mutex> lock(e.plan->mu);
    nus::use_device(e.cfg.device);
    nus::run_transform(*e.plan, grid_dev, k1 - k0, k1 - k0, nullptr, power_dev, false, divisor,
                       accumulate != 0, static_cast<cudaStream_t>(stream));
  });
}

int nus_mtnufft_spread_slots_device(nus_mtnufft_t est, const void* x_dev, int32_t x_dtype, int64_t s0,
                                    int64_t s1, const void* slot_ptrs_dev, int64_t per, void* stream) {
  return guarded([&] {
    nus::require(est && x_dev && slot_ptrs_dev, "spread_slots_device: null argument");
    auto& e = *est->est;
    nus::require(e.plan->p.path == NUS_PATH_FAST, "spread_slots_device: estimator is on the direct path");
    nus::require(e.cfg.channels == 1, "spread_slots_device: one channel");
    nus::require(per >= 1, "spread_slots_device: per must be >= 1");
    nus::require(0 <= s0 && s0 <= s1 && s1 <= e.cfg.n, "spread_slots_device: bad sample range");
    nus::use_device(e.cfg.device);
    nus::SpreadArgs a;
    a.x = x_dev;
    a.x_dtype = x_dtype;
    a.tapers = e.tapers_sorted.ptr;
    a.k = e.cfg.k_tapers;
    a.kpad = e.cfg.k_tapers;
    a.s0 = s0;
    a.s1 = s1;
    a.grid = nullptr;
    a.slots = static_cast<void* const*>(const_cast<void*>(slot_ptrs_dev));
    a.per = per;
    nus::launch_spread(*e.plan, a, static_cast<cudaStream_t>(stream));
  });
}

int nus_sum_slots_device(const void* base, int64_t nslots, int64_t slot_stride, int64_t count, void* out,
                         int32_t precision, void* stream) {
  return guarded([&] {
    nus::require(base && out && nslots >= 1 && count >= 0 && slot_stride >= count, "sum_slots: bad argument");
    nus::require(precision == NUS_F64 || precision == NUS_F32, "sum_slots: unknown precision");
    nus::sum_slots(base, nslots, slot_stride, count, out, precision == NUS_F64, static_cast<cudaStream_t>(stream));
  });
}

int nus_ipc_get_handle(const void* dev_ptr, void* handle64) {
  return guarded([&] {
    nus::require(dev_ptr && handle64, "ipc: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    NUS_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    std::memcpy(handle64, &h, sizeof(h));
  });
}

int nus_ipc_get_handle_offset(const void* dev_ptr, void* handle64, int64_t* offset) {
  return guarded([&] {
    nus::require(dev_ptr && handle64 && offset, "ipc: null argument");
    cudaIpcMemHandle_t h;
    NUS_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
    std::memcpy(handle64, &h, sizeof(h));
    // cudaIpcOpenMemHandle maps the base of the allocation holding dev_ptr: the peer needs the
    // byte offset of dev_ptr inside it (a caching allocator sub-allocates large segments)
    using AddrRange = int (*)(unsigned long long*, size_t*, unsigned long long);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    NUS_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    nus::require(fn != nullptr && q == cudaDriverEntryPointSuccess, "ipc: cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    const unsigned long long p = reinterpret_cast<unsigned long long>(dev_ptr);
    if (reinterpret_cast<AddrRange>(fn)(&base, &size, p) != 0)
      nus::fail(NUS_ERR_CUDA, "ipc: cuMemGetAddressRange failed");
    *offset = static_cast<int64_t>(p - base);
  });
}

int nus_ipc_open(const void* handle64, int32_t device, void** dev_ptr) {
  return guarded([&] {
    nus::require(handle64 && dev_ptr, "ipc: null argument");
    nus::use_device(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof(h));
    NUS_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int nus_ipc_close(void* dev_ptr) {
  return guarded([&] { NUS_CUDA(cudaIpcCloseMemHandle(dev_ptr)); });
}

int nus_mtnufft_grid_rows(nus_mtnufft_t est, int32_t* row_lo, int32_t* row_cnt, int32_t* nrows) {
  return guarded([&] {
    nus::require(est && row_lo && row_cnt && nrows, "grid_rows: null argument");
    const auto& f = est->est->plan->ffft;
    const bool blk = f.ready && f.blocked;
    *row_lo = blk ? f.row_lo : 0;
    *row_cnt = blk ? f.row_cnt : 0;
    *nrows = blk ? f.R : 0;
  });
}

int nus_mtnufft_set_grid_rows(nus_mtnufft_t est, int32_t row_lo, int32_t row_cnt) {
  return guarded([&] {
    nus::require(est != nullptr, "set_grid_rows: null argument");
    auto& f = est->est->plan->ffft;
    if (!(f.ready && f.blocked)) return;
    nus::require(row_lo >= 0 && row_lo < f.R && row_cnt >= 1 && row_cnt <= f.R, "set_grid_rows: bad interval");
    // every currently occupied row r (cyclic offset from row_lo < row_cnt) must stay inside
    for (int q = 0; q < f.row_cnt; ++q) {
      const int r = (f.row_lo + q) % f.R;
      nus::require(((r - row_lo) % f.R + f.R) % f.R < row_cnt,
                   "set_grid_rows: the interval must contain the estimator's occupied rows");
    }
    std::lock_guard<std::mutex> lock(est->est->plan->mu);
    f.row_lo = row_lo;
    f.row_cnt = row_cnt;
  });
}

int nus_mtnufft_timing(nus_mtnufft_t est, int64_t max_runs) {
  return guarded([&] {
    nus::require(est && max_runs >= 0, "nus_mtnufft_timing: bad argument");
    nus::use_device(est->est->cfg.device);
    nus::estimator_timing_enable(*est->est, static_cast<size_t>(max_runs));
  });
}

int nus_mtnufft_timing_read(nus_mtnufft_t est, double* stage_ms3, int64_t* runs) {
  return guarded([&] {
    nus::require(est && stage_ms3 && runs, "nus_mtnufft_timing_read: null argument");
    nus::use_device(est->est->cfg.device);
    nus::estimator_timing_read(*est->est, stage_ms3, runs);
  });
}

int nus_f_test(const double* j_host, int64_t k, int64_t n_bands, const double* w0_host, int64_t n_samples,
               const double* centers, double f_w, double cap, int32_t device, double* f_out, double* amp_out,
               uint8_t* flags_out) {
  return guarded([&] {
    nus::require(j_host && w0_host && centers && f_out && amp_out && flags_out, "f_test: null argument");
    nus::require(k >= 2, "f_test: need at least 2 tapers");
    nus::require(n_bands >= 1, "f_test: eigencoefficient shape mismatch");
    nus::use_device(device);
    nus::DeviceBuffer j(static_cast<size_t>(k) * n_bands * 2 * sizeof(double)), c(n_bands * sizeof(double)),
        f(n_bands * sizeof(double)), a(n_bands * 2 * sizeof(double)), fl(n_bands);
    NUS_CUDA(cudaMemcpy(j.ptr, j_host, j.bytes, cudaMemcpyHostToDevice));
    NUS_CUDA(cudaMemcpy(c.ptr, centers, c.bytes, cudaMemcpyHostToDevice));
    nus::ftest_device(j.ptr, false, k, n_bands, 1, w0_host, n_samples, c.as<double>(), f_w, cap, f.as<double>(),
                      a.as<double>(), fl.as<uint8_t>(), 0);
    NUS_CUDA(cudaMemcpy(f_out, f.ptr, f.bytes, cudaMemcpyDeviceToHost));
    NUS_CUDA(cudaMemcpy(amp_out, a.ptr, a.bytes, cudaMemcpyDeviceToHost));
    NUS_CUDA(cudaMemcpy(flags_out, fl.ptr, fl.bytes, cudaMemcpyDeviceToHost));
  });
}

int nus_mtnufft_f_test(nus_mtnufft_t est, const double* x_host, double cap, double* f_out, double* amp_out,
                       uint8_t* flags_out) {
  return guarded([&] {
    nus::require(est && x_host && f_out && amp_out && flags_out, "f_test: null argument");
    auto& e = *est->est;
    std::lock_guard<std::mutex> lock(e.mu);
    nus::use_device(e.cfg.device);
    const auto& p = e.plan->p;
    const int64_t C = e.cfg.channels, K = e.cfg.k_tapers, nb = p.nc;
    nus::require(K >= 2, "f_test: need at least 2 tapers");
    const bool f32 = p.precision == NUS_F32 && p.path == NUS_PATH_FAST;
    cudaStream_t s = e.stream();
    nus::DeviceBuffer x(static_cast<size_t>(C) * e.cfg.n * sizeof(double));
    nus::DeviceBuffer j(static_cast<size_t>(C) * K * nb * 2 * (f32 ? sizeof(float) : sizeof(double)));
    NUS_CUDA(cudaMemcpyAsync(x.ptr, x_host, x.bytes, cudaMemcpyHostToDevice, s));
    nus::estimator_run(e, x.ptr, 0, nullptr, false, j.ptr, s);  // J stays on the device
    std::vector<double> w0(C * K * 2);
    nus::taper_zero_frequency(e, w0.data());
    nus::DeviceBuffer f(C * nb * sizeof(double)), a(C * nb * 2 * sizeof(double)), fl(C * nb);
    bool uniform_fw = true;
    for (int64_t c = 1; c < C; ++c) uniform_fw = uniform_fw && e.f_w[c] == e.f_w[0];
    if (uniform_fw) {
      nus::ftest_device(j.ptr, f32, K, nb, C, w0.data(), e.cfg.n, e.plan->d_centers.as<double>(), e.f_w[0], cap,
                        f.as<double>(), a.as<double>(), fl.as<uint8_t>(), s);
    } else {  // each channel's band-edge flag uses its own half-bandwidth
      const size_t jb = static_cast<size_t>(K) * nb * 2 * (f32 ? sizeof(float) : sizeof(double));
      for (int64_t c = 0; c < C; ++c)
        nus::ftest_device(static_cast<const char*>(j.ptr) + c * jb, f32, K, nb, 1, w0.data() + c * K * 2, e.cfg.n,
                          e.plan->d_centers.as<double>(), e.f_w[c], cap, f.as<double>() + c * nb,
                          a.as<double>() + 2 * c * nb, fl.as<uint8_t>() + c * nb, s);
    }
    NUS_CUDA(cudaMemcpy(f_out, f.ptr, f.bytes, cudaMemcpyDeviceToHost));
    NUS_CUDA(cudaMemcpy(amp_out, a.ptr, a.bytes, cudaMemcpyDeviceToHost));
    NUS_CUDA(cudaMemcpy(flags_out, fl.ptr, fl.bytes, cudaMemcpyDeviceToHost));
  });
}

int nus_f_quantile(double p, int64_t d1, int64_t d2, double* out) {
  return guarded([&] {
    nus::require(out != nullptr, "f_quantile: null output");
    *out = nus::f_quantile_host(p, d1, d2);
  });
}

int nus_mtnufft_bytes_model(nus_mtnufft_t est, int32_t x_dtype, double* total, double* spread,
                            double* fft, double* crop) {
  return guarded([&] {
    nus::require(est != nullptr, "bytes_model: null estimator");
    nus::estimator_bytes(*est->est, x_dtype, total, spread, fft, crop);
  });
}

int nus_mtnufft_stage_kernels(nus_mtnufft_t est, char* out, int64_t len) {
  return guarded([&] {
    nus::require(est != nullptr && out != nullptr && len > 0, "stage_kernels: bad arguments");
    const char *a = nullptr, *b = nullptr;
    nus::fft_stage_names(*est->est->plan, &a, &b);
    const std::string names = nus::spread_kernel_names(*est->est->plan, est->est->cfg.k_tapers) + ";" + a + ";" + b;
    std::snprintf(out, static_cast<size_t>(len), "%s", names.c_str());
  });
}

}  // extern "C"
