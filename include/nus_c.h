/* nus_c.h — C-ABI of the B200-native MTNUFFT hot path (libnus_b200.so).
 *
 * This is the drop-in boundary: plain pointers and sizes, opaque handles,
 * status codes, no C++ or torch types.  It replaces the reference's
 * in-process C++ calls on the MTNUFFT path (paths relative to
 * /root/reference/proj):
 *
 *   nus_plan_*            NufftPlan            include/nuspectral/nufft.hpp:31-76, src/nufft.cpp:56-187
 *   nus_ndft_direct       ndft_direct          include/nuspectral/nufft.hpp:16-18, src/nufft.cpp:36-54
 *   nus_dpss              dpss_uniform         include/nuspectral/tapers.hpp:22-23, src/tapers.cpp:31-79
 *   nus_tridiagonal_eigen tridiagonal_eigen    include/nuspectral/eig.hpp:30-32,     src/eig.cpp:572-610
 *   nus_signal_band_quadform  signal_band_kernel + KernelMatrix::quadratic_form
 *                                              include/nuspectral/kernels.hpp:38,60, src/kernels.cpp:28-37,100-115
 *   nus_gpss_interpolated gpss_interpolated    include/nuspectral/tapers.hpp:86-87, src/tapers.cpp:146-182
 *   nus_mtnufft_*         MtnufftEstimator / eigencoefficients / estimate_mtnufft
 *                                              include/nuspectral/estimators.hpp:39-62,133-137,
 *                                              src/estimators.cpp:91-122,261-270, src/nufft.cpp:194-227
 *
 * Conventions
 *  - Complex data is interleaved (re, im) in the plan's precision.
 *  - Host entry points take host pointers (std::vector semantics of the
 *    reference).  *_device entry points take device pointers plus a
 *    cudaStream_t passed as void* and never synchronise.
 *  - Every function returns a status; it never throws.  nus_last_error()
 *    returns the calling thread's last message.  The status codes map 1:1 to
 *    the reference's exception types (errors.hpp:9-49, std::invalid_argument).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with NUS_ERR_NO_DEVICE.
 */
#ifndef NUS_C_H
#define NUS_C_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum nus_status {
  NUS_OK = 0,
  NUS_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  NUS_ERR_PLAN_MISMATCH = 2,    /* nuspectral::PlanMismatch */
  NUS_ERR_BAND_RANGE = 3,       /* nuspectral::BandRangeError */
  NUS_ERR_EXTRAPOLATION = 4,    /* nuspectral::ExtrapolationError */
  NUS_ERR_NUMERIC = 5,          /* nuspectral::Error (numeric failure) */
  NUS_ERR_CUDA = 6,             /* CUDA runtime failure */
  NUS_ERR_OUT_OF_MEMORY = 7,
  NUS_ERR_NO_DEVICE = 8,
  NUS_ERR_DEGENERATE_TAPERS = 9, /* nuspectral::DegenerateTapers */
  NUS_ERR_CONDITIONING = 10,     /* nuspectral::ConditioningError (eig.cpp:497-499) */
  NUS_ERR_SPECTRAL_RANGE = 11    /* nuspectral::SpectralRangeError (eig.cpp:542-545) */
};

enum nus_path_policy { NUS_AUTO_SELECT = 0, NUS_FORCE_FAST = 1, NUS_FORCE_DIRECT = 2 };
enum nus_path { NUS_PATH_DIRECT = 0, NUS_PATH_FAST = 1 };
enum nus_precision { NUS_F64 = 0, NUS_F32 = 1 };
/* Spreading kernel of the fast path.  GAUSSIAN is the reference's own kernel (support 2w,
 * nufft.cpp:90-142): transforms replicate the reference to ~1e-12.  ES (exponential of
 * semicircle, exp(beta (sqrt(1 - z^2) - 1)), support ns = 2 ceil(log10(10/eps) / 2) cells,
 * beta = 2.30 ns) meets the same contract max|fast - direct| <= eps ||y||_1 with ~2.4x
 * narrower support; it is the default.  Bins (nus_plan_first_cells) are the reference's
 * either way. */
enum nus_kernel { NUS_KERNEL_GAUSSIAN = 0, NUS_KERNEL_ES = 1 };

typedef struct nus_plan_s* nus_plan_t;
typedef struct nus_mtnufft_s* nus_mtnufft_t;

typedef struct {
  int64_t n_samples;
  int64_t n_centers;
  double epsilon;
  int32_t oversampling;
  int32_t path;            /* enum nus_path */
  int32_t centers_uniform; /* nufft.cpp:23-32 */
  int32_t precision;       /* enum nus_precision */
  int64_t spread_width;    /* w; 2w cells per sample (nufft.cpp:90-92) */
  int64_t mr;              /* oversampled grid (nufft.cpp:103-104), 0 on the direct path */
  double tau;              /* Gaussian width (nufft.cpp:105-108) */
  double df;               /* centre spacing */
  double fshift;           /* f0 + (I/2) df */
  int32_t kernel;          /* enum nus_kernel (fast path) */
  int32_t support;         /* cells per sample actually spread: 2w (Gaussian) or ns (ES) */
} nus_plan_info_t;

const char* nus_last_error(void);
/* Library/device facts: device count, compute capability, build string. */
int nus_device_info(int device, int32_t* cc_major, int32_t* cc_minor, int32_t* sm_count,
                    int64_t* total_mem);
/* Number of this library's kernels launched so far (process-wide). */
int64_t nus_kernel_launch_count(void);
/* Process-wide spreading kernel for plans created afterwards (enum nus_kernel).  The initial
 * value is NUS_KERNEL_ES, or the NUS_KERNEL environment variable ("gaussian" / "es"). */
int nus_set_spread_kernel(int32_t kind);
int nus_get_spread_kernel(int32_t* kind);

/* ---- NufftPlan (nufft.hpp:31-76) ---------------------------------------- */
int nus_plan_create(const double* times, int64_t n, const double* centers, int64_t n_centers,
                    double epsilon, int32_t policy, int32_t oversampling, int32_t precision,
                    int32_t device, nus_plan_t* out);
int nus_plan_destroy(nus_plan_t plan);
int nus_plan_info(nus_plan_t plan, nus_plan_info_t* info);
/* Reference first_cell_ (j0 = floor(x*Mr/2pi) - w + 1 per sample, nufft.cpp:118-122), bit-exact. */
int nus_plan_first_cells(nus_plan_t plan, int64_t* out_host);
/* Stable order of samples by start cell (j0 mod Mr) used by the spreading kernel. */
int nus_plan_sort_order(nus_plan_t plan, int32_t* perm_host);
/* NufftPlan::execute on one complex vector (host in/out, interleaved fp64). */
int nus_plan_execute(nus_plan_t plan, const double* y_host, int64_t n_y, double* out_host);
/* Batched device execute: y_dev [batch][n] complex, out_dev [batch][I] complex (plan precision). */
int nus_plan_execute_device(nus_plan_t plan, const void* y_dev, int64_t batch, void* out_dev,
                            void* stream);

/* Direct NUDFT oracle path (nufft.cpp:36-54) on the device, fp64. */
int nus_ndft_direct(const double* times, int64_t n, const double* y_host, const double* centers,
                    int64_t n_centers, int32_t device, double* out_host);

/* In-place forward (inverse != 0: unscaled inverse) complex FFT of n (power of two)
 * interleaved fp64 values on the device (Radix2Fft, fft.hpp:12-29 / fft.cpp:39-58). */
int nus_fft_inplace(double* data_host, int64_t n, int32_t inverse, int32_t device);
/* Dense R(B) (n x n row-major) filled on the device (signal_band_kernel, kernels.cpp:100-115). */
int nus_signal_band_matrix(const double* times, int64_t n, double f_max, int32_t device,
                           double* out_host);

/* ---- MTNUFFT0: exact nominal-band tapers ----------------
 * Generalized Hermitian eigenproblem A w = lambda M w (eig.cpp:612-659) on the device:
 * Cholesky of M + ridge * trace(M)/n * I (ridge_first, then ridge_retry; else
 * NUS_ERR_CONDITIONING), C = L^-1 A L^-T, the k largest eigenpairs, values descending
 * clamped into [0, 1] (NUS_ERR_SPECTRAL_RANGE beyond 1e-6), vectors w = L^-T y normalised to
 * w^H M w = 1 with the canonical phase (largest |w_i| real positive), residuals
 * ||A w - lambda M w|| / (||A||_F ||w||).  A: n x n row-major (a_im null when real),
 * M: n x n row-major real symmetric; vectors: [k][n] complex. */
int nus_generalized_eigen(const double* a_re, const double* a_im, const double* m, int64_t n, int64_t k,
                          double ridge_first, double ridge_retry, int32_t want_vectors, int32_t device,
                          double* values, double* vectors, double* residuals);
/* Dense analysis-band kernel R(A) (n x n row-major; im_out null for a band centred at 0),
 * filled on the device (analysis_band_kernel, kernels.cpp:117-153). */
int nus_band_matrix(const double* times, int64_t n, double f_w, double f_center, int32_t device, double* re_out,
                    double* im_out);
/* gpss_exact (tapers.cpp:118-144): R(B) and R(A) (band f_center +- f_w) built on the device,
 * the GEP above, each vector scaled to w^H R(B) w = 2 f_w.  w_out [k][n] complex. */
int nus_gpss_exact(const double* times, int64_t n, double f_max, double f_center, double f_w, int64_t k,
                   double ridge_first, double ridge_retry, int32_t device, double* w_out, double* concentrations);

/* ---- tapers (tapers.hpp) -------------------------------------------------- */
/* Top-k eigenpairs of the commuting tridiagonal (tapers.cpp:40-52); vectors K x n unit norm,
 * largest-|v| entry positive (eig.cpp:281-289).  eigenvalues / concentrations may be NULL. */
int nus_dpss(int64_t n, double time_half_bandwidth, int64_t k, int32_t device, double* tapers_host,
             double* eigenvalues_host, double* concentrations_host);
int nus_tridiagonal_eigen(const double* diag, const double* offdiag, int64_t n, int64_t k,
                          int32_t device, double* values, double* vectors, double* residuals);
/* q_k = w_k^T R(B) w_k for K weight rows over rows [row_begin,row_end) of R(B) (pass 0,n for all). */
int nus_signal_band_quadform(const double* times, int64_t n, double f_max, const double* w_host,
                             int64_t k, int64_t row_begin, int64_t row_end, int32_t device,
                             double* q_host);
/* The same q_k in O(N log N) (normalise.cu): q = int_{-F}^{F} |W_k(f)|^2 df as a windowed lattice
 * sum of the path's own type-1 NUFFT.  gpss_interpolated uses it above NUS_QUADFORM_EXACT_MAX
 * samples (default 2^18; NUS_NORMALISE=exact|fast forces one form). */
int nus_signal_band_quadform_fast(const double* times, int64_t n, double f_max, const double* w_host,
                                  int64_t k, int32_t device, double* q_host);
/* Un-normalised interpolated DPSS: spline of dpss_uniform(n, f_w*h*n, k) at t (tapers.cpp:156-174). */
int nus_taper_spline(const double* times, int64_t n, double f_max, double f_w, int64_t k,
                     int32_t device, double* w_host);
/* Full gpss_interpolated: spline + R(B) normalisation to w^T R(B) w = 2 f_w. */
int nus_gpss_interpolated(const double* times, int64_t n, double f_max, double f_w, int64_t k,
                          int32_t device, double* weights_host);

/* ---- MtnufftEstimator (estimators.hpp:39-62) -------------------------------
 * channels independent series share n, the centres, K and epsilon.
 * times: [channels][n].  tapers: NULL -> computed on the GPU (gpss_interpolated per
 * channel), else injected normalised weights [channels][K][n] (Oracle-B style).
 * The setup (DPSS, spline, R(B) norm, bins, sort) runs on the device. */
typedef struct {
  int64_t channels;
  int64_t n;
  int64_t n_centers;
  int64_t k_tapers;
  double f_max;
  double f_w;
  double epsilon;
  int32_t policy;
  int32_t precision;
  int32_t device;
  int32_t reserved;
} nus_mtnufft_config_t;

int nus_mtnufft_create(const nus_mtnufft_config_t* cfg, const double* times, const double* centers,
                       const double* tapers, nus_mtnufft_t* out);
/* Same with a per-channel taper half-bandwidth f_w [channels] (NULL -> cfg->f_w for all): each
 * channel's tapers are gpss_interpolated(grid_c, SignalBand(f_max), f_w[c], K) as the reference
 * builds one MtnufftEstimator per channel (estimators.cpp:91-104). */
int nus_mtnufft_create_channels(const nus_mtnufft_config_t* cfg, const double* times, const double* centers,
                                const double* f_w, const double* tapers, nus_mtnufft_t* out);
int nus_mtnufft_destroy(nus_mtnufft_t est);
int nus_mtnufft_plan_info(nus_mtnufft_t est, nus_plan_info_t* info);
/* ---- Multi-GPU MtnufftEstimator in one process ----------------
 * A device list; one estimator part per device; exchanges over peer memory (NVLink) ordered by
 * CUDA events.  cfg->device is ignored.  Replaces the serial loops of nufft.cpp:194-227 /
 * estimators.cpp:106-122 for one series (tapers / samples) or many (channels):
 *   NUS_SHARD_CHANNELS  channels split over the devices, no exchange;
 *   NUS_SHARD_TAPERS    one series, tapers split, partial spectra summed on devices[0];
 *   NUS_SHARD_SAMPLES   one series, contiguous sample chunks; the spread stores every taper's
 *                       grid straight into its owner device's receive slot (peer stores fused into
 *                       the spread), owners sum slots in device order and transform their tapers.
 * Results equal the single-device estimator's to rounding (deterministic order).  A device may be
 * listed more than once (emulated parts on one GPU). */
typedef struct nus_mtnufft_multi_s* nus_mtnufft_multi_t;
enum { NUS_SHARD_CHANNELS = 0, NUS_SHARD_TAPERS = 1, NUS_SHARD_SAMPLES = 2 };
int nus_mtnufft_multi_create(const nus_mtnufft_config_t* cfg, const int32_t* devices, int32_t n_devices,
                             int32_t sharding, const double* times, const double* centers, const double* f_w,
                             const double* tapers, nus_mtnufft_multi_t* out);
int nus_mtnufft_multi_destroy(nus_mtnufft_multi_t est);
/* x [channels][n] host -> P [channels][I] host. */
int nus_mtnufft_multi_estimate(nus_mtnufft_multi_t est, const double* x_host, double* power_host);
/* Normalised tapers [channels][K][n] (time order). */
int nus_mtnufft_multi_tapers(nus_mtnufft_multi_t est, double* out_host);
/* Bytes each spectrum moves between devices (peer slot stores + partial spectra). */
int nus_mtnufft_multi_peer_bytes(nus_mtnufft_multi_t est, int64_t* bytes);

/* Normalised taper weights [channels][K][n] (fp64, time order). */
int nus_mtnufft_tapers(nus_mtnufft_t est, double* out_host);
/* Setup timings in ms: [dpss, spline, normalise, plan(bins+sort+tables), total]. */
int nus_mtnufft_setup_ms(nus_mtnufft_t est, double* out5);
/* estimate(): x [channels][n] fp64 host -> power [channels][I] fp64 host. */
int nus_mtnufft_estimate(nus_mtnufft_t est, const double* x_host, double* power_host);
/* estimate() of `steps` series in one call: x [steps][channels][n] -> power [steps][channels][I]
 * (host, fp64; pinned memory lets the copies run asynchronously).  Copies of one step overlap
 * the compute of its neighbours (double-buffered device staging, separate H2D / D2H streams). */
int nus_mtnufft_estimate_batch(nus_mtnufft_t est, const double* x_host, int64_t steps, double* power_host);
/* eigencoefficients(): -> J [channels][K][I] complex fp64 host (nufft.cpp:194-227). */
int nus_mtnufft_eigencoefficients(nus_mtnufft_t est, const double* x_host, double* j_host);
/* Device-resident estimate.  x_dev: [channels][n] of x_dtype (0 f64, 1 f32); power_dev:
 * [channels][I] in the plan precision; j_dev optional [channels][K][I] complex. */
int nus_mtnufft_estimate_device(nus_mtnufft_t est, const void* x_dev, int32_t x_dtype,
                                void* power_dev, void* j_dev, void* stream);
/* Sample-split building blocks.  spread: samples [s0,s1) (time order) of every
 * channel into grid_dev [channels][k_pad][Mr] complex (tapers >= K left untouched);
 * transform: FFT + deconvolve/crop + sum_k |J|^2 / divisor of tapers [k0,k1) held in grid_dev
 * rows 0..k1-k0-1 (one channel), written to (or added into, accumulate != 0) power_dev. */
int nus_mtnufft_spread_device(nus_mtnufft_t est, const void* x_dev, int32_t x_dtype, int64_t s0,
                              int64_t s1, void* grid_dev, int64_t k_pad, void* stream);
int nus_mtnufft_transform_device(nus_mtnufft_t est, void* grid_dev, int64_t k0, int64_t k1,
                                 double divisor, int32_t accumulate, void* power_dev, void* stream);
/* Occupied pass-A rows of the fused FFT's blocked grid: the spread writes and pass A reads only
 * rows [row_lo, row_lo + row_cnt) (cyclic, of nrows) that this estimator's own samples touch.
 * A sample split must widen every rank's interval to the union over ranks before grids are
 * summed (set: the new interval must contain the current one; nrows = 0 when not blocked). */
/* The sample split's spread fused with its exchange: samples [s0,s1) are spread and taper k is
 * stored straight into slot_ptrs_dev[k / per] + (k % per) * Mr (a device array of G pointers
 * to the owners' receive slots for this rank; peer NVLink addresses from nus_ipc_open_handle on
 * a multi-GPU box), so the transfer overlaps the spread segment by segment instead of following
 * it as a reduce-scatter.  One channel. */
int nus_mtnufft_spread_slots_device(nus_mtnufft_t est, const void* x_dev, int32_t x_dtype, int64_t s0,
                                    int64_t s1, const void* slot_ptrs_dev, int64_t per, void* stream);
/* out = sum over nslots slots (slot q at base + q * slot_stride complex elements) of count complex
 * elements, in slot order (deterministic); precision = enum nus_precision. */
int nus_sum_slots_device(const void* base, int64_t nslots, int64_t slot_stride, int64_t count, void* out,
                         int32_t precision, void* stream);
/* CUDA IPC for the receive slots: 64-byte handle of a device allocation, and a peer mapping of
 * another process's handle (close with nus_ipc_close). */
int nus_ipc_get_handle(const void* dev_ptr, void* handle64);
/* Same, plus the byte offset of dev_ptr inside its allocation (peers add it to the mapped base). */
int nus_ipc_get_handle_offset(const void* dev_ptr, void* handle64, int64_t* offset);
int nus_ipc_open(const void* handle64, int32_t device, void** dev_ptr);
int nus_ipc_close(void* dev_ptr);
int nus_mtnufft_grid_rows(nus_mtnufft_t est, int32_t* row_lo, int32_t* row_cnt, int32_t* nrows);
int nus_mtnufft_set_grid_rows(nus_mtnufft_t est, int32_t row_lo, int32_t row_cnt);
/* Per-stage CUDA-event timing of the fast path: record (on the caller's stream) the
 * next max_runs estimate calls; _read syncs and returns summed ms for
 * [spread, fft, crop+power] and the number of runs recorded. */
int nus_mtnufft_timing(nus_mtnufft_t est, int64_t max_runs);
int nus_mtnufft_timing_read(nus_mtnufft_t est, double* stage_ms3, int64_t* runs);
/* Names of the kernels behind the three timed stages ("spread;fft;crop+power"), ';'-separated. */
int nus_mtnufft_stage_kernels(nus_mtnufft_t est, char* out, int64_t len);
/* ---- inference (inference.hpp:16-48) -------------------------------------
 * Harmonic F-test (inference.cpp:132-186) on host eigencoefficients j [K][I] complex with
 * zero-frequency responses w0 [K] complex; outputs F [I], amplitude [I] complex, flags [I]
 * (1 = 2 f_c <= f_w, 2 = saturated at cap).  Computed on the device. */
int nus_f_test(const double* j_host, int64_t k, int64_t n_bands, const double* w0_host, int64_t n_samples,
               const double* centers, double f_w, double cap, int32_t device, double* f_out, double* amp_out,
               uint8_t* flags_out);
/* F-test of one estimate with J kept on the device: x [channels][n] -> [channels][I] outputs. */
int nus_mtnufft_f_test(nus_mtnufft_t est, const double* x_host, double cap, double* f_out, double* amp_out,
                       uint8_t* flags_out);
/* Upper-tail F(d1, d2) critical value: x with P(F > x) = p (inference.cpp:94-130). Host scalar math. */
int nus_f_quantile(double p, int64_t d1, int64_t d2, double* out);

/* Algorithmic bytes of one estimate (SURVEY §8d model) and of its spreading kernel. */
int nus_mtnufft_bytes_model(nus_mtnufft_t est, int32_t x_dtype, double* total, double* spread,
                            double* fft, double* crop);

#ifdef __cplusplus
}
#endif
#endif /* NUS_C_H */
