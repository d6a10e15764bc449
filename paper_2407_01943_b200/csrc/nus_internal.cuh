// Internal declarations shared by the libnus_b200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <utility>

#include <atomic>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "nus_c.h"

namespace nus {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * 3.14159265358979323846;

// Status-carrying exception used inside the library; converted to a status
// code at the C-ABI boundary (capi.cu) and never crosses it.
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }
inline void require(bool ok, const std::string& msg) {
  if (!ok) fail(NUS_ERR_INVALID_ARGUMENT, msg);
}

void cuda_check(cudaError_t e, const char* what);
#define NUS_CUDA(x) ::nus::cuda_check((x), #x)

// Count of our own kernel launches (the bench reports it as gpu_launches).
extern std::atomic<int64_t> g_launches;
inline void note_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }
void check_launch(const char* what);

// Selects `device` for the calling thread and verifies it is an sm_100 part.
void use_device(int device);

// RAII device buffer.
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t b) { alloc(b); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr(o.ptr), bytes(o.bytes) { o.ptr = nullptr; o.bytes = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) { release(); ptr = o.ptr; bytes = o.bytes; o.ptr = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DeviceBuffer() { release(); }
  void alloc(size_t b);
  void release();
  template <class T> T* as() const { return static_cast<T*>(ptr); }
};

// ---- plan ------------------------------------------------------------------

// Per-grid NUFFT tables on the device, all indexed in start-cell-sorted order.
struct PlanParams {
  int64_t n = 0;          // samples per channel
  int64_t nc = 0;         // centres I
  int64_t channels = 1;
  double eps = 0;
  int oversampling = 2;
  int path = NUS_PATH_FAST;
  bool uniform = false;
  int precision = NUS_F64;
  int w = 0;              // spread width; support is 2w cells
  int64_t mr = 0;
  double tau = 0, f0 = 0, df = 0, fshift = 0;
  int64_t mode_offset = 0;
  double beta = 0;        // Gaussian exponent per cell^2: (2pi/Mr)^2 / (4 tau)
  double deconv_norm = 0; // sqrt(pi/tau)/Mr
  // spreading kernel (fast path): NUS_KERNEL_GAUSSIAN (the reference's, sw = 2w) or
  // NUS_KERNEL_ES (sw = ns cells); a point's support starts at cell j0 + sshift, j0 being
  // the reference bin (nufft.cpp:118-121), sshift = w - ns/2 for ES, 0 for the Gaussian
  int kernel = NUS_KERNEL_GAUSSIAN;
  int sw = 0;
  int sshift = 0;
  double es_beta = 0;
};

// ---- exponential-of-semicircle kernel (es.cu) ----------------------------------------
// phi(z) = exp(beta (sqrt(1 - z^2) - 1)) on |z| <= 1, z = 2 (cell - position) / ns.
constexpr int kEsMinNs = 4, kEsMaxNs = 16;
int default_kernel();
void set_default_kernel(int kind);
int es_width(double eps);                 // ns: even, 4 .. 16
inline double es_beta(int ns) { return 2.30 * ns; }
// Degree of the window polynomials per even ns: the lowest whose max error over a cell is
// <= ~eps_min(ns)/10 (eps_min = 10^(1-ns); the fit error plateaus at ~5% of e^-beta, the
// square-root edge of the window)
__host__ __device__ constexpr int es_degree(int ns) {
  return ns <= 6 ? ns + 1 : ns == 8 ? 8 : ns <= 14 ? ns - 1 : 13;
}
// Monomial coefficients (in s = 2 fr - 1, degree es_degree(ns)) of the weight of cell
// p = 0..ns-1 of a point at fractional offset fr in [0, 1): out[p * (es_degree(ns) + 1) + d].
void es_fit(int ns, double* out);
// Offset of ns's block in the packed table of all even ns in [kEsMinNs, kEsMaxNs].
__host__ __device__ constexpr int es_table_offset(int ns) {
  int o = 0;
  for (int q = kEsMinNs; q < ns; q += 2) o += q * (es_degree(q) + 1);
  return o;
}
constexpr int kEsTableSize = es_table_offset(kEsMaxNs + 2);
// Gauss-Legendre rule for Phi(m) = ns int_0^{pi/2} e^{beta (cos th - 1)} cos(a sin th) cos th dth:
// node pairs (sin th_q, w_q e^{beta (cos th_q - 1)} cos th_q), q < nq.
void es_quadrature(int ns, int nq, double* pairs);

struct SpreadTables {
  int tile = 128;               // cells per spreading tile (= spread.cu kTile)
  int64_t ntiles = 0;
  DeviceBuffer start;           // int32 [C][n] start cell s = j0 mod Mr (sorted)
  DeviceBuffer perm;            // int32 [C][n] original sample index of sorted point
  DeviceBuffer gauss;           // Gaussian: real2 [C][n] (A, g), W_p = A g^p C_p for the point's 2w cells;
                                // ES: real [C][n] fr, the window polynomials' argument (compact)
  DeviceBuffer prephase;        // real2 [C][n] e^{-i 2pi fshift t}
  int64_t nseg = 0;             // 32-cell segments (tensor-core spread)
  DeviceBuffer seg_range;       // int32 [C][nseg][4]: own lo, own hi, wrap lo, 0
  std::vector<int32_t> h_seg_range;  // host copy (the streaming spread's work partition)
  // Work units of the streaming spread (spread.cu): contiguous cell ranges of equal work, one per
  // resident warp; built on first use per (warps, occupied rows) and cached.
  struct Units {
    int64_t nwarps = 0, count = 0, ilv = 0;
    int row_lo = 0, row_cnt = 0;
    DeviceBuffer buf;             // int32 [count][8]: channel, first segment, segments, own lo, own hi, wrap lo, 0, 0
  };
  mutable std::deque<Units> units;  // deque: references stay valid as entries are added
  mutable std::mutex units_mu;
  DeviceBuffer tile_range;      // int32 [C][ntiles+1][2]: point range of tile (lo, hi)
  DeviceBuffer wrap_lo;         // int32 [C]: first sorted point whose support wraps into tile 0
  DeviceBuffer deconv;          // real  [I]
  DeviceBuffer first_cell;      // int64 [C][n] reference j0, time order (kept for parity queries)
};

// Tables of the fused two-pass FFT (fft.cu): Mr = R * C, twiddles e^{-2 pi i m / L}.
struct FusedFft {
  bool ready = false;
  int R = 1, C = 1, RPC = 1, CW = 0, lo_bits = 0;
  // blocked: the spread writes cell j1*C + j2 at (j2/CW)*R*CW + j1*CW + j2%CW so that every
  // pass-A column block (tile, 2^lgT = R*CW cells) is contiguous; lgC/lgCW/lgT are its shifts
  bool blocked = false;
  int lgC = 0, lgCW = 0, lgT = 12;
  // lw: the layout's column blocks are 2^lw pass-A tiles wide (lgCW, lgT describe the layout; CW the
  // tile): a tile is then a CW-column slice of a wider block, whose rows the spread stores in one piece
  int lw = 0;
  // pass A over the blocked grid: 1 = register-loading tiles of 4096 (256 threads, default),
  // 0 = tiles of 2048 (128 threads), 2 = bulk-copy pipeline (NUS_FFT_COLS=reg128 / async)
  int cols_mode = 1;
  DeviceBuffer scratch;  // pass-A output (natural layout) when blocked: [C][kpad][Mr]
  // Occupied rows (blocked only): every cell any point's support touches lies in rows
  // j1 in [row_lo, row_lo + row_cnt) (cyclic, union over channels).  The spread writes only
  // those rows and pass A loads only them; the other rows are exact zeros of the grid.
  int row_lo = 0, row_cnt = 1;
  DeviceBuffer tw_r, tw_c, tw_hi, tw_lo;
  DeviceBuffer zeros;  // 16 KB of zeros (bulk-copy source)
};

struct Plan {
  PlanParams p;
  FusedFft ffft;
  int device = 0;
  std::vector<double> times;    // host copy, time order [C][n]
  std::vector<double> centers;
  DeviceBuffer d_times;         // fp64 [C][n]
  DeviceBuffer d_centers;       // fp64 [I]
  SpreadTables tab;
  std::mutex mu;                // serialises use of the default workspace
  DeviceBuffer work;            // default grid workspace
};

void plan_validate_and_select(PlanParams& p, const double* centers, int64_t nc, double eps,
                              int policy, int oversampling);
void plan_build_tables(Plan& plan, cudaStream_t s);
std::unique_ptr<Plan> plan_create(const double* times, int64_t channels, int64_t n,
                                  const double* centers, int64_t nc, double eps, int policy,
                                  int oversampling, int precision, int device);

// Spreads K taper-weighted copies of x (sorted-order tapers; nullptr tapers = weight 1 and
// x complex) onto grid [C][kpad][Mr].  Samples [s0, s1) in time order only.
struct SpreadArgs {
  const void* x = nullptr;   // [C][n] real (x_dtype) or complex when x_complex
  int x_dtype = 0;           // 0 f64, 1 f32
  bool x_complex = false;
  const void* tapers = nullptr;  // [C][K][n] sorted-order real (plan precision)
  int64_t k = 1;
  int64_t kpad = 1;
  int64_t s0 = 0, s1 = -1;
  void* grid = nullptr;
  // sample split fused with its exchange (one channel): taper k is written to
  // slots[k / per] + (k % per) * Mr instead of grid + k * Mr -- the owner's receive slot for
  // this rank, a peer (NVLink) address on a multi-GPU box.  Device array of pointers.
  void* const* slots = nullptr;
  int64_t per = 0;
};
void launch_spread(const Plan& plan, const SpreadArgs& a, cudaStream_t s);
// out[i] = sum_{s < nslots} slots[s][i] over `count` complex elements (fixed order: deterministic)
void sum_slots(const void* base, int64_t nslots, int64_t slot_stride, int64_t count, void* out, bool f64,
               cudaStream_t s);

// FFT of rows [C][kpad][Mr] (first k rows per channel are transformed), then crop:
// optional J [C][k][I] = deconv * B[bin] and power [C][I] (+)= sum_k |J|^2 / divisor.
void run_transform(Plan& plan, void* grid, int64_t k, int64_t kpad, void* j_out, void* power,
                   bool power_f64, double divisor, bool accumulate, cudaStream_t s);

void run_fft(Plan& plan, void* grid, int64_t k, int64_t kpad, cudaStream_t s);
void run_crop(Plan& plan, void* grid, int64_t k, int64_t kpad, void* j_out, void* power,
              bool power_f64, double divisor, bool accumulate, cudaStream_t s);

// Fused two-pass FFT + crop/power (fft.cu); 512 <= Mr <= 2^26 (else the generic radix-2 kernels).
bool fused_fft_supported(const PlanParams& p);
// Generic radix-2 Stockham FFT (fft.cu), one launch per stage: `rows` rows of length n (power of
// two), row r at ((r / k) kpad + r % k) n, transformed in place (forward e^{-2 pi i jk/n}, inverse
// the conjugate transform without 1/n, as Radix2Fft); scratch holds rows * n complex elements.
void fft_generic_rows(void* data, int64_t n, int64_t rows, int64_t k, int64_t kpad, bool f64, bool inverse,
                      void* scratch, cudaStream_t s);
// Same for `batch` contiguous rows, allocating its own scratch (synchronises s).
void fft_generic_inplace(void* data, int64_t n, int64_t batch, bool f64, bool inverse, cudaStream_t s);
// MTNUFFT0 (gep.cu)
void generalized_eigen_device(const double* d_are, const double* d_aim, const double* d_m, int64_t n, int64_t k,
                              double ridge_first, double ridge_retry, bool want_vectors, double* values,
                              double* vectors, double* residuals);
void band_matrix_rowmajor(const double* d_t, int64_t n, double f, double fc, double tol, double* d_re,
                          double* d_im);
void gpss_exact_device(const double* h_t, int64_t n, double f_max, double f_c, double f_w, int64_t k,
                       double ridge_first, double ridge_retry, double* w_out, double* conc);
const char* spread_kernel_name();
void fft_stage_names(const Plan& plan, const char** pass_a, const char** pass_b);
void fused_fft_prepare(Plan& plan);
void run_fused_pass_a(Plan& plan, void* grid, int64_t k, int64_t kpad, cudaStream_t s);
// Spread kernel(s) a spectrum of k tapers launches (bench / tests)
std::string spread_kernel_names(const Plan& plan, int64_t k);
void run_fused_pass_b(Plan& plan, void* grid, int64_t k, int64_t kpad, void* j_out, void* power, bool power_f64,
                      double divisor, bool accumulate, cudaStream_t s);

void launch_ndft_direct(const double* d_t, int64_t n, const void* d_y, bool y_f32,
                        const double* d_c, int64_t nc, void* d_out, bool out_f32, int64_t batch,
                        cudaStream_t s);

// ---- tapers ----------------------------------------------------------------

struct DpssResult {
  std::vector<double> values;  // K descending
};
// vectors on device: d_vec [K][n] fp64
DpssResult dpss_device(int64_t n, double tw, int64_t k, double* d_vec, cudaStream_t s);
DpssResult dpss_from_coarse(const double* d_diag, const double* d_off, int64_t n, double tw, int64_t k,
                            double* d_vec, cudaStream_t s);
DpssResult tridiag_top_device(const double* d_diag, const double* d_off, int64_t n, int64_t k,
                              double* d_vec, cudaStream_t s);
void dpss_concentrations(int64_t n, double tw, int64_t k, const double* d_vec, double* conc,
                         cudaStream_t s);
// Interpolates K DPSS rows (knots t0 + h i) at times d_t -> d_w [K][n].
void spline_uniform_device(const double* d_t, int64_t n, const double* d_y, int64_t k,
                           double* d_w, cudaStream_t s);
void quadform_device(const double* d_t, int64_t n, double f_max, const double* d_w, int64_t k,
                     int64_t row0, int64_t row1, double* q_host, cudaStream_t s);
// q_k = w_k^T R(B) w_k in O(N log N) (normalise.cu); h_t = host copy of the times
void quadform_fast_device(const double* d_t, const double* h_t, int64_t n, double f_max, const double* d_w,
                          int64_t k, double* q_host, cudaStream_t s, int device);
// exact O(N^2) form for n <= this (NUS_QUADFORM_EXACT_MAX, default 2^16) unless NUS_NORMALISE
bool normalise_exact(int64_t n);
// Uniform-grid DPSS kept across the channels of one estimator: the vectors depend only on
// (n, time-bandwidth product, k), and channels of one recording share them whenever f_w h N
// rounds to the same double (C3: 256 channels, 2-3 distinct values).  Exact-key match only.
struct DpssCache {
  struct Entry {
    int64_t n = 0, k = 0;
    double tw = 0.0;
    DeviceBuffer dp;  // [k][n]
  };
  std::vector<Entry> entries;
  int64_t hits = 0;
};
// Full gpss_interpolated for one grid: d_w [K][n] normalised; timings optional.
void gpss_interpolated_device(const double* d_t, const double* h_t, int64_t n, double f_max,
                              double f_w, int64_t k, double* d_w, cudaStream_t s,
                              double* ms_dpss = nullptr, double* ms_spline = nullptr,
                              double* ms_norm = nullptr, DpssCache* cache = nullptr);

__host__ __device__ inline int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---- programmatic dependent launch ---------------------------------------------------
// The per-spectrum kernels are launched with programmatic stream serialisation: a kernel's
// CTAs may be dispatched while its predecessor drains, and each waits (griddepcontrol.wait:
// predecessor complete, memory visible) before its first dependent read.  Disabled (see
// pdl_enabled in fft.cu): slower on C2, and a programmatic launch was seen to overlap an H2D
// copy queued before it on the same stream.
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  NUS_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ---- double-double helpers ---------------------------------------------------

struct dd { double hi, lo; };

__host__ __device__ inline dd dd_two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__host__ __device__ inline dd dd_quick(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ inline dd dd_add(dd a, dd b) {
  dd s = dd_two_sum(a.hi, b.hi);
  dd t = dd_two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = dd_quick(s.hi, s.lo);
  s.lo += t.lo;
  return dd_quick(s.hi, s.lo);
}
__device__ inline dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ inline dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }
__device__ inline dd dd_mul(dd a, dd b) {
  double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return dd_quick(p, e);
}
__device__ inline dd dd_mul_d(dd a, double b) {
  double p = a.hi * b;
  double e = fma(a.hi, b, -p);
  e = fma(a.lo, b, e);
  return dd_quick(p, e);
}
__device__ inline dd dd_div(dd a, dd b) {
  double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul_d(b, q1));
  double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul_d(b, q2));
  double q3 = r.hi / b.hi;
  dd q = dd_quick(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}
// 1 / b to ~2^-104 relative with ONE fp64 divide: r = 1/b.hi, then r (1 + e) with the
// residual e = 1 - b r formed exactly by fma (dd_div's three dependent divides cost ~4x more)
__device__ inline dd dd_recip(dd b) {
  const double r = 1.0 / b.hi;
  const double e = fma(-b.hi, r, 1.0) - b.lo * r;
  return dd_quick(r, r * e);
}
__device__ inline dd dd_from(double a) { return {a, 0.0}; }
__device__ inline double dd_abs_hi(dd a) { return fabs(a.hi); }

}  // namespace nus
