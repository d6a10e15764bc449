// Estimator object shared by mtnufft.cu and capi.cu.
#pragma once

#include "nus_internal.cuh"

namespace nus {

struct Estimator {
  nus_mtnufft_config_t cfg{};
  std::vector<double> f_w;     // per-channel taper half-bandwidth (cfg.f_w unless given per channel)
  std::unique_ptr<Plan> plan;
  DeviceBuffer tapers_time;    // fp64 [C][K][n], time order (normalised)
  DeviceBuffer tapers_sorted;  // plan precision [C][K][n], start-cell order
  DeviceBuffer grid;           // [C][K][Mr] complex, plan precision
  DeviceBuffer x_stage, p_stage, j_stage;  // host-API staging
  // estimate_batch: double-buffered staging and the copy streams / events of the pipeline
  DeviceBuffer xb[2], pb[2];
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_x[2] = {nullptr, nullptr}, ev_c[2] = {nullptr, nullptr}, ev_p[2] = {nullptr, nullptr};
  double setup_ms[5] = {0, 0, 0, 0, 0};
  std::mutex mu;
  cudaStream_t own_stream = nullptr;
  // optional per-stage CUDA-event timing: 4 events per run (before spread,
  // after spread, after FFT, after crop) recorded on the caller's stream
  std::vector<cudaEvent_t> tev;
  size_t tslot = 0;         // runs recorded
  size_t tcap = 0;          // capacity in runs
  cudaStream_t stream();
  ~Estimator();
};

// f_w_channels: [channels] per-channel half-bandwidths, or null for cfg.f_w on every channel
std::unique_ptr<Estimator> estimator_create(const nus_mtnufft_config_t& cfg, const double* times,
                                            const double* centers, const double* tapers,
                                            const double* f_w_channels = nullptr);
void estimator_run(Estimator& est, const void* x_dev, int x_dtype, void* power_dev, bool power_f64,
                   void* j_dev, cudaStream_t s);
void estimator_estimate_batch_host(Estimator& est, const double* x, int64_t steps, double* power);
void estimator_estimate_host(Estimator& est, const double* x, double* power, double* j);
void estimator_timing_enable(Estimator& est, size_t max_runs);
void estimator_timing_read(Estimator& est, double* ms3, int64_t* runs);
void estimator_bytes(const Estimator& est, int x_dtype, double* total, double* spread, double* fft,
                     double* crop);

// Multi-GPU estimator in one process (multi.cu)
struct MultiEstimator;
struct MultiDeleter {
  void operator()(MultiEstimator* m) const;
};
using MultiPtr = std::unique_ptr<MultiEstimator, MultiDeleter>;
MultiPtr multi_create(const nus_mtnufft_config_t& cfg, const int32_t* devices, int32_t n_devices,
                                             int32_t sharding, const double* times, const double* centers,
                                             const double* f_w, const double* tapers);
void multi_estimate(MultiEstimator& m, const double* x_host, double* power_host);
int64_t multi_peer_bytes(const MultiEstimator& m);
void multi_tapers(const MultiEstimator& m, double* out_host);

double f_quantile_host(double p, int64_t d1, int64_t d2);
void ftest_device(const void* j_dev, bool j_f32, int64_t k, int64_t nb, int64_t channels, const double* w0_host,
                  int64_t n_samples, const double* d_centers, double f_w, double cap, double* f_dev,
                  double* amp_dev, uint8_t* flags_dev, cudaStream_t s);
void taper_zero_frequency(const Estimator& est, double* w0_host);

}  // namespace nus
