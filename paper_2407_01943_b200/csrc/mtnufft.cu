// MtnufftEstimator on the device (src/estimators.cpp:91-122): taper setup
// (gpss_interpolated on the GPU, or injected weights), one NUFFT plan, and the
// per-spectrum pipeline  spread(all K) -> FFT pass A -> FFT pass B fused with crop+power.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "nus_estimator.cuh"

namespace nus {

namespace {

template <typename Real>
__global__ void permute_tapers_kernel(const double* __restrict__ w_time, const int32_t* __restrict__ perm,
                                      int64_t n, int64_t k, int64_t channels, Real* __restrict__ w_sorted) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= channels * k * n) return;
  const int64_t i = g % n;
  const int64_t ck = g / n;
  const int64_t c = ck / k;
  w_sorted[g] = static_cast<Real>(w_time[ck * n + perm[c * n + i]]);
}

// Direct path (N*I < 2^14 or non-uniform centres): y_k = w_k x (complex fp64)
__global__ void weight_series_kernel(const double* __restrict__ w, const void* __restrict__ x,
                                     int x_dtype, int64_t n, int64_t k, int64_t channels,
                                     double* __restrict__ y) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= channels * k * n) return;
  const int64_t i = g % n;
  const int64_t c = g / (k * n);
  const double xv = x_dtype == 0 ? static_cast<const double*>(x)[c * n + i]
                                 : static_cast<double>(static_cast<const float*>(x)[c * n + i]);
  y[2 * g] = w[g] * xv;
  y[2 * g + 1] = 0.0;
}

template <typename OutReal>
__global__ void power_from_j_kernel(const double* __restrict__ j, int64_t k, int64_t nc,
                                    int64_t channels, OutReal* __restrict__ power) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= channels * nc) return;
  const int64_t c = g / nc, i = g - c * nc;
  double acc = 0.0;
  for (int64_t kk = 0; kk < k; ++kk) {
    const double re = j[2 * ((c * k + kk) * nc + i)], im = j[2 * ((c * k + kk) * nc + i) + 1];
    acc += re * re + im * im;
  }
  power[g] = static_cast<OutReal>(acc / static_cast<double>(k));
}

__global__ void f32_to_f64_kernel(const float* __restrict__ a, int64_t n, double* __restrict__ b) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g < n) b[g] = static_cast<double>(a[g]);
}

unsigned nblk(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

void validate_grid(const double* times, int64_t channels, int64_t n) {
  require(n >= 2, "SamplingGrid: need at least 2 samples");
  for (int64_t c = 0; c < channels; ++c) {
    const double* t = times + c * n;
    for (int64_t i = 0; i < n; ++i) {
      require(std::isfinite(t[i]), "SamplingGrid: non-finite sample time");
      require(i == 0 || t[i] > t[i - 1], "SamplingGrid: times must be strictly increasing");
    }
  }
}

}  // namespace

std::unique_ptr<Estimator> estimator_create(const nus_mtnufft_config_t& cfg, const double* times,
                                            const double* centers, const double* tapers,
                                            const double* f_w_channels) {
  require(cfg.channels >= 1, "MtnufftEstimator: channels must be >= 1");
  require(cfg.k_tapers >= 1, "MtnufftEstimator: k_tapers must be >= 1");
  require(times && centers, "MtnufftEstimator: null input");
  validate_grid(times, cfg.channels, cfg.n);
  use_device(cfg.device);
  auto est = std::make_unique<Estimator>();
  est->cfg = cfg;
  est->f_w.assign(static_cast<size_t>(cfg.channels), cfg.f_w);
  if (f_w_channels) {
    for (int64_t c = 0; c < cfg.channels; ++c) est->f_w[c] = f_w_channels[c];
    est->cfg.f_w = f_w_channels[0];
  }
  const auto t_all = std::chrono::steady_clock::now();
  const int64_t C = cfg.channels, n = cfg.n, K = cfg.k_tapers;
  cudaStream_t s = 0;
  // tapers first, as the reference constructs them before the plan (estimators.cpp:95-100)
  est->tapers_time.alloc(static_cast<size_t>(C) * K * n * sizeof(double));
  if (tapers) {
    NUS_CUDA(cudaMemcpy(est->tapers_time.ptr, tapers, static_cast<size_t>(C) * K * n * sizeof(double),
                        cudaMemcpyHostToDevice));
  } else {
    require(cfg.f_max > 0.0 && std::isfinite(cfg.f_max), "SignalBand: f_max must be positive");
    DeviceBuffer dt(n * sizeof(double));
    DpssCache dpss_cache;  // channels whose f_w h N is the same double share one DPSS
    for (int64_t c = 0; c < C; ++c) {
      NUS_CUDA(cudaMemcpy(dt.ptr, times + c * n, n * sizeof(double), cudaMemcpyHostToDevice));
      double a = 0, b = 0, d = 0;
      gpss_interpolated_device(dt.as<double>(), times + c * n, n, cfg.f_max, est->f_w[c], K,
                               est->tapers_time.as<double>() + c * K * n, s, &a, &b, &d, &dpss_cache);
      est->setup_ms[0] += a;
      est->setup_ms[1] += b;
      est->setup_ms[2] += d;
    }
  }
  const auto t_plan = std::chrono::steady_clock::now();
  est->plan = plan_create(times, C, n, centers, cfg.n_centers, cfg.epsilon, cfg.policy, 2,
                          cfg.precision, cfg.device);
  const PlanParams& p = est->plan->p;
  if (p.path == NUS_PATH_FAST) {
    const size_t rs = p.precision == NUS_F64 ? sizeof(double) : sizeof(float);
    est->tapers_sorted.alloc(static_cast<size_t>(C) * K * n * rs);
    if (p.precision == NUS_F64)
      permute_tapers_kernel<double><<<nblk(C * K * n), 256, 0, s>>>(
          est->tapers_time.as<double>(), est->plan->tab.perm.as<int32_t>(), n, K, C,
          est->tapers_sorted.as<double>());
    else
      permute_tapers_kernel<float><<<nblk(C * K * n), 256, 0, s>>>(
          est->tapers_time.as<double>(), est->plan->tab.perm.as<int32_t>(), n, K, C,
          est->tapers_sorted.as<float>());
    note_launch();
    check_launch("permute_tapers_kernel");
    est->grid.alloc(static_cast<size_t>(C) * K * p.mr * 2 * rs);
  }
  NUS_CUDA(cudaDeviceSynchronize());
  const auto now = std::chrono::steady_clock::now();
  est->setup_ms[3] = std::chrono::duration<double, std::milli>(now - t_plan).count();
  est->setup_ms[4] = std::chrono::duration<double, std::milli>(now - t_all).count();
  return est;
}

void estimator_run(Estimator& est, const void* x_dev, int x_dtype, void* power_dev, bool power_f64,
                   void* j_dev, cudaStream_t s) {
  Plan& plan = *est.plan;
  const PlanParams& p = plan.p;
  const int64_t C = est.cfg.channels, n = est.cfg.n, K = est.cfg.k_tapers;
  require(x_dtype == 0 || x_dtype == 1, "estimate: x dtype must be 0 (f64) or 1 (f32)");
  if (p.path == NUS_PATH_FAST) {
    SpreadArgs a;
    a.x = x_dev;
    a.x_dtype = x_dtype;
    a.tapers = est.tapers_sorted.ptr;
    a.k = K;
    a.kpad = K;
    a.grid = est.grid.ptr;
    const bool timed = est.tslot < est.tcap;
    cudaEvent_t* ev = timed ? est.tev.data() + 4 * est.tslot : nullptr;
    if (timed) NUS_CUDA(cudaEventRecord(ev[0], s));
    launch_spread(plan, a, s);
    if (timed) NUS_CUDA(cudaEventRecord(ev[1], s));
    run_fft(plan, est.grid.ptr, K, K, s);
    if (timed) NUS_CUDA(cudaEventRecord(ev[2], s));
    run_crop(plan, est.grid.ptr, K, K, j_dev, power_dev, power_f64, static_cast<double>(K), false, s);
    if (timed) {
      NUS_CUDA(cudaEventRecord(ev[3], s));
      ++est.tslot;
    }
    return;
  }
  // direct path: exact sums in fp64 (nufft.cpp:174-186)
  DeviceBuffer y(static_cast<size_t>(C) * K * n * 2 * sizeof(double));
  DeviceBuffer jj(static_cast<size_t>(C) * K * p.nc * 2 * sizeof(double));
  weight_series_kernel<<<nblk(C * K * n), 256, 0, s>>>(est.tapers_time.as<double>(), x_dev, x_dtype, n,
                                                       K, C, y.as<double>());
  note_launch();
  // per channel: ndft over that channel's times, batch K
  for (int64_t c = 0; c < C; ++c)
    launch_ndft_direct(plan.d_times.as<double>() + c * n, n, y.as<double>() + 2 * c * K * n, false,
                       plan.d_centers.as<double>(), p.nc, jj.as<double>() + 2 * c * K * p.nc, false, K, s);
  if (power_dev) {
    if (power_f64 || p.precision == NUS_F64)
      power_from_j_kernel<double><<<nblk(C * p.nc), 256, 0, s>>>(jj.as<double>(), K, p.nc, C,
                                                                 static_cast<double*>(power_dev));
    else
      power_from_j_kernel<float><<<nblk(C * p.nc), 256, 0, s>>>(jj.as<double>(), K, p.nc, C,
                                                                static_cast<float*>(power_dev));
    note_launch();
  }
  if (j_dev) {
    if (p.precision == NUS_F64) {
      NUS_CUDA(cudaMemcpyAsync(j_dev, jj.ptr, jj.bytes, cudaMemcpyDeviceToDevice, s));
    } else {
      fail(NUS_ERR_INVALID_ARGUMENT, "eigencoefficients: f32 J on the direct path is not supported");
    }
  }
  check_launch("direct estimate");
  NUS_CUDA(cudaStreamSynchronize(s));
}

void estimator_estimate_host(Estimator& est, const double* x, double* power, double* j) {
  std::lock_guard<std::mutex> lock(est.mu);
  use_device(est.cfg.device);
  const PlanParams& p = est.plan->p;
  const int64_t C = est.cfg.channels, n = est.cfg.n, K = est.cfg.k_tapers;
  cudaStream_t s = est.stream();
  if (!est.x_stage.ptr) est.x_stage.alloc(static_cast<size_t>(C) * n * sizeof(double));
  if (power && !est.p_stage.ptr) est.p_stage.alloc(static_cast<size_t>(C) * p.nc * sizeof(double));
  const size_t jbytes = static_cast<size_t>(C) * K * p.nc * 2 *
                        (p.precision == NUS_F64 || p.path != NUS_PATH_FAST ? sizeof(double) : sizeof(float));
  if (j && est.j_stage.bytes < jbytes) est.j_stage.alloc(jbytes);
  NUS_CUDA(cudaMemcpyAsync(est.x_stage.ptr, x, static_cast<size_t>(C) * n * sizeof(double),
                           cudaMemcpyHostToDevice, s));
  estimator_run(est, est.x_stage.ptr, 0, power ? est.p_stage.ptr : nullptr, true,
                j ? est.j_stage.ptr : nullptr, s);
  if (power)
    NUS_CUDA(cudaMemcpyAsync(power, est.p_stage.ptr, static_cast<size_t>(C) * p.nc * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  if (j) {
    if (jbytes == static_cast<size_t>(C) * K * p.nc * 2 * sizeof(double)) {
      NUS_CUDA(cudaMemcpyAsync(j, est.j_stage.ptr, jbytes, cudaMemcpyDeviceToHost, s));
    } else {
      DeviceBuffer j64(static_cast<size_t>(C) * K * p.nc * 2 * sizeof(double));
      f32_to_f64_kernel<<<nblk(C * K * p.nc * 2), 256, 0, s>>>(est.j_stage.as<float>(), C * K * p.nc * 2,
                                                               j64.as<double>());
      note_launch();
      NUS_CUDA(cudaMemcpyAsync(j, j64.ptr, j64.bytes, cudaMemcpyDeviceToHost, s));
      NUS_CUDA(cudaStreamSynchronize(s));
    }
  }
  NUS_CUDA(cudaStreamSynchronize(s));
}

// Pipelined host estimate of `steps` series (x [steps][C][n], power [steps][C][I], host):
// step s's H2D copy, compute and D2H copy run on three streams with double-buffered device
// staging, so the copies of one step overlap the compute of its neighbours (copy engines in
// both directions at once).  Every step still moves its own input in and its own P out.
void estimator_estimate_batch_host(Estimator& est, const double* x, int64_t steps, double* power) {
  std::lock_guard<std::mutex> lock(est.mu);
  use_device(est.cfg.device);
  const PlanParams& p = est.plan->p;
  const int64_t C = est.cfg.channels, n = est.cfg.n;
  const size_t xbytes = static_cast<size_t>(C) * n * sizeof(double), pbytes = static_cast<size_t>(C) * p.nc * sizeof(double);
  cudaStream_t cs = est.stream();
  if (!est.h2d) {
    NUS_CUDA(cudaStreamCreateWithFlags(&est.h2d, cudaStreamNonBlocking));
    NUS_CUDA(cudaStreamCreateWithFlags(&est.d2h, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      NUS_CUDA(cudaEventCreateWithFlags(&est.ev_x[b], cudaEventDisableTiming));
      NUS_CUDA(cudaEventCreateWithFlags(&est.ev_c[b], cudaEventDisableTiming));
      NUS_CUDA(cudaEventCreateWithFlags(&est.ev_p[b], cudaEventDisableTiming));
    }
  }
  for (int b = 0; b < 2; ++b) {
    if (est.xb[b].bytes < xbytes) est.xb[b].alloc(xbytes);
    if (est.pb[b].bytes < pbytes) est.pb[b].alloc(pbytes);
  }
  for (int64_t st = 0; st < steps; ++st) {
    const int b = static_cast<int>(st & 1);
    if (st >= 2) NUS_CUDA(cudaStreamWaitEvent(est.h2d, est.ev_c[b], 0));  // x buffer consumed
    NUS_CUDA(cudaMemcpyAsync(est.xb[b].ptr, x + st * C * n, xbytes, cudaMemcpyHostToDevice, est.h2d));
    NUS_CUDA(cudaEventRecord(est.ev_x[b], est.h2d));
    NUS_CUDA(cudaStreamWaitEvent(cs, est.ev_x[b], 0));
    if (st >= 2) NUS_CUDA(cudaStreamWaitEvent(cs, est.ev_p[b], 0));  // P buffer drained
    estimator_run(est, est.xb[b].ptr, 0, est.pb[b].ptr, true, nullptr, cs);
    NUS_CUDA(cudaEventRecord(est.ev_c[b], cs));
    NUS_CUDA(cudaStreamWaitEvent(est.d2h, est.ev_c[b], 0));
    NUS_CUDA(cudaMemcpyAsync(power + st * C * p.nc, est.pb[b].ptr, pbytes, cudaMemcpyDeviceToHost, est.d2h));
    NUS_CUDA(cudaEventRecord(est.ev_p[b], est.d2h));
  }
  NUS_CUDA(cudaStreamSynchronize(est.d2h));
  NUS_CUDA(cudaStreamSynchronize(cs));
}

void estimator_timing_enable(Estimator& est, size_t max_runs) {
  for (auto e : est.tev) cudaEventDestroy(e);
  est.tev.assign(4 * max_runs, nullptr);
  for (auto& e : est.tev) NUS_CUDA(cudaEventCreate(&e));
  est.tslot = 0;
  est.tcap = max_runs;
}

void estimator_timing_read(Estimator& est, double* ms3, int64_t* runs) {
  ms3[0] = ms3[1] = ms3[2] = 0.0;
  for (size_t r = 0; r < est.tslot; ++r) {
    cudaEvent_t* ev = est.tev.data() + 4 * r;
    NUS_CUDA(cudaEventSynchronize(ev[3]));
    for (int q = 0; q < 3; ++q) {
      float ms = 0.f;
      NUS_CUDA(cudaEventElapsedTime(&ms, ev[q], ev[q + 1]));
      ms3[q] += ms;
    }
  }
  *runs = static_cast<int64_t>(est.tslot);
}

cudaStream_t Estimator::stream() {
  if (!own_stream) NUS_CUDA(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
  return own_stream;
}

Estimator::~Estimator() {
  for (auto e : tev) cudaEventDestroy(e);
  for (int b = 0; b < 2; ++b) {
    if (ev_x[b]) cudaEventDestroy(ev_x[b]);
    if (ev_c[b]) cudaEventDestroy(ev_c[b]);
    if (ev_p[b]) cudaEventDestroy(ev_p[b]);
  }
  if (h2d) cudaStreamDestroy(h2d);
  if (d2h) cudaStreamDestroy(d2h);
  if (own_stream) cudaStreamDestroy(own_stream);
}

void estimator_bytes(const Estimator& est, int x_dtype, double* total, double* spread, double* fft,
                     double* crop) {
  const PlanParams& p = est.plan->p;
  const double C = static_cast<double>(est.cfg.channels), N = static_cast<double>(est.cfg.n),
               K = static_cast<double>(est.cfg.k_tapers), I = static_cast<double>(p.nc),
               Mr = static_cast<double>(p.mr);
  const double r = p.precision == NUS_F64 ? 8.0 : 4.0;
  const double c = 2.0 * r;
  (void)x_dtype;
  // B = N(8+r) + K N r + 3 K Mr c + K I c + I r  (per channel)
  const double b_spread = N * (8.0 + r) + K * N * r + K * Mr * c;
  const double b_fft = 2.0 * K * Mr * c;
  const double b_crop = K * I * c + I * r;
  // per-stage figures are what each launched kernel must move: with the fused FFT the
  // crop/power epilogue lives in pass B, which reads the K rows-transformed grids once
  const double b_stage3 = est.plan->ffft.ready ? K * Mr * c + I * r : b_crop;
  const double b_stage2 = est.plan->ffft.ready && est.plan->ffft.R <= 1 ? 0.0 : b_fft;
  if (spread) *spread = C * b_spread;
  if (fft) *fft = C * b_stage2;
  if (crop) *crop = C * b_stage3;
  if (total) *total = C * (b_spread + b_fft + b_crop);  // SURVEY model (pipeline roofline)
}

}  // namespace nus
