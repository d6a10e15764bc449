// NufftPlan on the device: parameter selection (host, identical to the
// reference), per-sample bin/phase tables (one fused kernel), a stable radix
// sort of samples by start cell, per-tile point ranges and the deconvolution
// table.  Reference: src/nufft.cpp:23-32 (uniform check), :56-94 (validation,
// path, spread width), :96-142 (tables).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "nus_internal.cuh"

namespace nus {

std::atomic<int64_t> g_launches{0};

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    fail(NUS_ERR_OUT_OF_MEMORY, std::string("out of device memory: ") + what);
  }
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    fail(NUS_ERR_NO_DEVICE, std::string("no usable CUDA device: ") + cudaGetErrorString(e));
  fail(NUS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void check_launch(const char* what) { cuda_check(cudaGetLastError(), what); }

void use_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(NUS_ERR_NO_DEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= count) fail(NUS_ERR_INVALID_ARGUMENT, "device index out of range");
  NUS_CUDA(cudaSetDevice(device));
  int major = 0;
  NUS_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major < 10)
    fail(NUS_ERR_NO_DEVICE, "device is not sm_100-class; libnus_b200 is built for sm_100a only");
}

void DeviceBuffer::alloc(size_t b) {
  release();
  if (b == 0) return;
  NUS_CUDA(cudaMalloc(&ptr, b));
  bytes = b;
}

void DeviceBuffer::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

// ---- parameter selection (host; must reproduce the reference exactly) -------

namespace {

bool uniform_spacing(const double* c, int64_t n) {  // nufft.cpp:23-32
  if (n < 2) return false;
  const double df = c[1] - c[0];
  if (!(df > 0.0)) return false;
  double max_dev = 0.0;
  for (int64_t i = 1; i < n; ++i) max_dev = std::max(max_dev, std::abs((c[i] - c[i - 1]) - df));
  return max_dev <= 1e-9 * df;
}

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace

void plan_validate_and_select(PlanParams& p, const double* centers, int64_t nc, double eps,
                              int policy, int oversampling) {
  require(nc > 0, "NufftPlan: no frequency centers");
  require(eps > 0.0 && !(eps > 1e-2), "NufftPlan: epsilon must be in (0, 1e-2]");
  require(oversampling >= 2, "NufftPlan: oversampling must be >= 2");
  p.nc = nc;
  p.eps = eps;
  p.oversampling = oversampling;
  p.uniform = uniform_spacing(centers, nc);
  switch (policy) {
    case NUS_FORCE_FAST:
      require(p.uniform, "NufftPlan: fast path requires uniformly spaced centers");
      p.path = NUS_PATH_FAST;
      break;
    case NUS_FORCE_DIRECT:
      p.path = NUS_PATH_DIRECT;
      break;
    default:
      p.path = (p.uniform && static_cast<uint64_t>(p.n) * static_cast<uint64_t>(nc) >= (1u << 14))
                   ? NUS_PATH_FAST
                   : NUS_PATH_DIRECT;
  }
  p.w = static_cast<int>(std::max<int64_t>(4, static_cast<int64_t>(std::ceil(0.55 * (-std::log(eps))))));
  p.kernel = default_kernel();
  if (p.kernel == NUS_KERNEL_ES) {
    p.sw = es_width(eps);
    p.sshift = p.w - p.sw / 2;
    p.es_beta = es_beta(p.sw);
  } else {
    p.sw = 2 * p.w;
    p.sshift = 0;
  }
  if (p.path != NUS_PATH_FAST) return;
  // nufft.cpp:96-114, same operation order
  p.f0 = centers[0];
  p.df = (centers[nc - 1] - centers[0]) / static_cast<double>(nc - 1);
  p.mr = next_pow2(std::max<int64_t>(static_cast<int64_t>(oversampling) * nc, 4 * p.w + 4));
  const double ratio = static_cast<double>(p.mr) / static_cast<double>(nc);
  p.tau = kPi * static_cast<double>(p.w) /
          (static_cast<double>(nc) * static_cast<double>(nc) * ratio * (ratio - 0.5));
  p.mode_offset = nc / 2;
  p.fshift = p.f0 + static_cast<double>(p.mode_offset) * p.df;
  const double h = kTwoPi / static_cast<double>(p.mr);
  p.beta = h * h / (4.0 * p.tau);
  p.deconv_norm = std::sqrt(kPi / p.tau) / static_cast<double>(p.mr);
}

// ---- table kernels -----------------------------------------------------------

namespace {

// Per sample (time order): reference j0 (bit-exact, nufft.cpp:118-121) and the
// radix-sort key/value.  Explicit _rn intrinsics forbid FMA contraction so the
// IEEE operation order matches the reference TU (compiled without -mfma).
__global__ void bins_kernel(const double* __restrict__ t, int64_t n, int64_t total, double neg2pi_df,
                            double mr_d, int64_t mr, int w, int sshift, int mr_bits, int64_t* __restrict__ j0_out,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= total) return;
  const int64_t c = g / n;
  const int64_t i = g - c * n;
  double x = fmod(__dmul_rn(neg2pi_df, t[g]), kTwoPi);
  if (x < 0.0) x = __dadd_rn(x, kTwoPi);
  const double cell = __ddiv_rn(__dmul_rn(x, mr_d), kTwoPi);
  const int64_t j0 = static_cast<int64_t>(floor(cell)) - w + 1;
  j0_out[g] = j0;
  int64_t s = (j0 + sshift) % mr;  // the spreading window's first cell
  if (s < 0) s += mr;
  keys[g] = (static_cast<uint64_t>(c) << mr_bits) | static_cast<uint64_t>(s);
  vals[g] = static_cast<int32_t>(i);
}

// Sorted order: start cell, fractional offset and prephase for each point.
template <typename Real>
__global__ void sorted_tables_kernel(const double* __restrict__ t, int64_t n, int64_t total,
                                     const uint64_t* __restrict__ keys_sorted,
                                     const int32_t* __restrict__ perm, int mr_bits,
                                     double neg2pi_df, double neg2pi_fshift, double mr_d,
                                     double beta, int w2, int es, int32_t* __restrict__ start,
                                     Real* __restrict__ gauss, Real* __restrict__ prephase) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= total) return;
  const int64_t c = g / n;
  const double tv = t[c * n + perm[g]];
  double x = fmod(__dmul_rn(neg2pi_df, tv), kTwoPi);
  if (x < 0.0) x = __dadd_rn(x, kTwoPi);
  const double cell = __ddiv_rn(__dmul_rn(x, mr_d), kTwoPi);
  const double fr = cell - floor(cell);
  const uint64_t mask = (static_cast<uint64_t>(1) << mr_bits) - 1;
  start[g] = static_cast<int32_t>(keys_sorted[g] & mask);
  // Gaussian factors around the support centre, fr' = frac - 1/2:
  //   exp(-beta (frac + w - 1 - p)^2) = A g^p C_p,  g = e^{2 beta fr'},
  //   A = e^{-beta fr' (fr' + 2w - 1)},  C_p = e^{-beta (p - w + 1/2)^2}
  if (es) {  // ES: the spread evaluates the window polynomials at fr (compact table, one real per point)
    gauss[g] = static_cast<Real>(fr);
  } else {
  const double frc = fr - 0.5;
  gauss[2 * g] = static_cast<Real>(exp(-beta * frc * (frc + static_cast<double>(w2 - 1))));
  gauss[2 * g + 1] = static_cast<Real>(exp(2.0 * beta * frc));
  }
  double sn, cs;
  sincos(__dmul_rn(neg2pi_fshift, tv), &sn, &cs);  // nufft.cpp:116-117
  prephase[2 * g] = static_cast<Real>(cs);
  prephase[2 * g + 1] = static_cast<Real>(sn);
}

__device__ inline int32_t lower_bound_i32(const int32_t* a, int32_t n, int64_t v) {
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Point range of each spreading tile: samples whose 2w-cell support
// [s, s+2w-1] meets [c0, c0+T).  Tile 0 additionally takes the wrapping
// samples s >= Mr-2w+1 (wrap_lo .. n).
__global__ void tile_ranges_kernel(const int32_t* __restrict__ start, int64_t n, int64_t channels,
                                   int64_t ntiles, int tile, int w2, int64_t mr,
                                   int32_t* __restrict__ ranges, int32_t* __restrict__ wrap_lo) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= channels * (ntiles + 1)) return;
  const int64_t c = g / (ntiles + 1);
  const int64_t tl = g - c * (ntiles + 1);
  const int32_t* s = start + c * n;
  if (tl == ntiles) {
    wrap_lo[c] = lower_bound_i32(s, static_cast<int32_t>(n), mr - (w2 - 1));
    return;
  }
  const int64_t c0 = tl * tile;
  ranges[2 * g] = lower_bound_i32(s, static_cast<int32_t>(n), c0 - (w2 - 1));
  ranges[2 * g + 1] = lower_bound_i32(s, static_cast<int32_t>(n), c0 + tile);
}

// Point ranges of the 32-cell segments of the tensor-core spread: int32 [C][nseg][4] =
// (own lo, own hi, wrap lo, 0): own points start in [s0-(w2-1), s0+32), wrapping points
// (segments with s0 < w2-1 only) start in [Mr+s0-(w2-1), Mr) and run to the channel's end.
__global__ void seg_ranges_kernel(const int32_t* __restrict__ start, int64_t n, int64_t channels, int64_t nseg,
                                  int w2, int64_t mr, int32_t* __restrict__ ranges) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= channels * nseg) return;
  const int64_t c = g / nseg, sg = g - c * nseg;
  const int32_t* s = start + c * n;
  const int64_t s0 = sg * 32;
  ranges[4 * g] = lower_bound_i32(s, static_cast<int32_t>(n), s0 - (w2 - 1));
  ranges[4 * g + 1] = lower_bound_i32(s, static_cast<int32_t>(n), s0 + 32);
  ranges[4 * g + 2] = s0 < w2 - 1 ? lower_bound_i32(s, static_cast<int32_t>(n), mr + s0 - (w2 - 1))
                                  : static_cast<int32_t>(n);
  ranges[4 * g + 3] = 0;
}

// Rows j1 = cell >> lgC touched by a point's support [start, start + w2) mod Mr (<= 2 rows).
__global__ void row_occupancy_kernel(const int32_t* __restrict__ start, int64_t total, int w2, int64_t mr,
                                     int lgC, uint8_t* __restrict__ occ) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= total) return;
  const int64_t s = start[g];
  occ[s >> lgC] = 1;
  occ[((s + w2 - 1) & (mr - 1)) >> lgC] = 1;
}

template <typename Real>
__global__ void deconv_kernel(int64_t nc, int64_t mode_offset, double tau, double norm,
                              Real* __restrict__ out) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nc) return;
  const double m = static_cast<double>(i - mode_offset);
  out[i] = static_cast<Real>(norm * exp(tau * m * m));  // nufft.cpp:139
}

// ES deconvolution: 1 / Phi(m), Phi(m) = int phi(2u/ns) cos(2 pi u m / Mr) du over the support
// (cell units), by the Gauss-Legendre rule of es_quadrature (pairs (sin th_q, weight_q)).
constexpr int kEsQuad = 100;
template <typename Real>
__global__ void deconv_es_kernel(int64_t nc, int64_t mode_offset, double a_per_mode, double ns,
                                 const double* __restrict__ pairs, Real* __restrict__ out) {
  __shared__ double sq[2 * kEsQuad];
  for (int q = threadIdx.x; q < 2 * kEsQuad; q += blockDim.x) sq[q] = pairs[q];
  __syncthreads();
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= nc) return;
  const double a = a_per_mode * static_cast<double>(i - mode_offset);
  double phi = 0.0;
  for (int q = 0; q < kEsQuad; ++q) phi += sq[2 * q + 1] * cos(a * sq[2 * q]);
  out[i] = static_cast<Real>(1.0 / (ns * phi));
}

int log2_exact(int64_t v) {
  int b = 0;
  while ((int64_t{1} << b) < v) ++b;
  return b;
}

}  // namespace

void plan_build_tables(Plan& plan, cudaStream_t st) {
  PlanParams& p = plan.p;
  SpreadTables& tb = plan.tab;
  const int64_t total = p.channels * p.n;
  require(total < (int64_t{1} << 31), "NufftPlan: channels * samples must be < 2^31");
  const size_t rs = p.precision == NUS_F64 ? sizeof(double) : sizeof(float);
  const int mr_bits = log2_exact(p.mr);
  const int ch_bits = log2_exact(p.channels);
  require(mr_bits + ch_bits <= 63, "NufftPlan: grid too large");

  tb.first_cell.alloc(total * sizeof(int64_t));
  tb.start.alloc(total * sizeof(int32_t));
  tb.perm.alloc(total * sizeof(int32_t));
  tb.gauss.alloc(total * 2 * rs);
  tb.prephase.alloc(total * 2 * rs);

  DeviceBuffer keys(total * sizeof(uint64_t)), keys_sorted(total * sizeof(uint64_t));
  DeviceBuffer vals(total * sizeof(int32_t));
  const double neg2pi_df = -kTwoPi * p.df;
  const double neg2pi_fshift = -kTwoPi * p.fshift;
  const double mr_d = static_cast<double>(p.mr);
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>((total + threads - 1) / threads);
  bins_kernel<<<blocks, threads, 0, st>>>(plan.d_times.as<double>(), p.n, total, neg2pi_df, mr_d,
                                          p.mr, p.w, p.sshift, mr_bits, tb.first_cell.as<int64_t>(),
                                          keys.as<uint64_t>(), vals.as<int32_t>());
  note_launch();
  check_launch("bins_kernel");

  size_t temp = 0;
  const int end_bit = mr_bits + ch_bits;
  NUS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys.as<uint64_t>(),
                                           keys_sorted.as<uint64_t>(), vals.as<int32_t>(),
                                           tb.perm.as<int32_t>(), static_cast<int>(total), 0,
                                           std::max(end_bit, 1), st));
  DeviceBuffer tmp(std::max<size_t>(temp, 16));
  NUS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.ptr, temp, keys.as<uint64_t>(),
                                           keys_sorted.as<uint64_t>(), vals.as<int32_t>(),
                                           tb.perm.as<int32_t>(), static_cast<int>(total), 0,
                                           std::max(end_bit, 1), st));
  note_launch(4);

  if (p.precision == NUS_F64)
    sorted_tables_kernel<double><<<blocks, threads, 0, st>>>(
        plan.d_times.as<double>(), p.n, total, keys_sorted.as<uint64_t>(), tb.perm.as<int32_t>(),
        mr_bits, neg2pi_df, neg2pi_fshift, mr_d, p.beta, p.sw, p.kernel == NUS_KERNEL_ES, tb.start.as<int32_t>(),
        tb.gauss.as<double>(), tb.prephase.as<double>());
  else
    sorted_tables_kernel<float><<<blocks, threads, 0, st>>>(
        plan.d_times.as<double>(), p.n, total, keys_sorted.as<uint64_t>(), tb.perm.as<int32_t>(),
        mr_bits, neg2pi_df, neg2pi_fshift, mr_d, p.beta, p.sw, p.kernel == NUS_KERNEL_ES, tb.start.as<int32_t>(),
        tb.gauss.as<float>(), tb.prephase.as<float>());
  note_launch();
  check_launch("sorted_tables_kernel");

  tb.tile = static_cast<int>(std::min<int64_t>(128, p.mr));  // = spread.cu kTile
  require(tb.tile >= p.sw, "NufftPlan: spread width exceeds the tile size");
  tb.ntiles = p.mr / tb.tile;
  tb.tile_range.alloc(p.channels * (tb.ntiles + 1) * 2 * sizeof(int32_t));
  tb.wrap_lo.alloc(p.channels * sizeof(int32_t));
  {
    const int64_t cnt = p.channels * (tb.ntiles + 1);
    tile_ranges_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(
        tb.start.as<int32_t>(), p.n, p.channels, tb.ntiles, tb.tile, p.sw, p.mr,
        tb.tile_range.as<int32_t>(), tb.wrap_lo.as<int32_t>());
    note_launch();
    check_launch("tile_ranges_kernel");
  }
  tb.nseg = p.mr / 32;
  tb.seg_range.alloc(p.channels * tb.nseg * 4 * sizeof(int32_t));
  {
    const int64_t cnt = p.channels * tb.nseg;
    seg_ranges_kernel<<<static_cast<unsigned>((cnt + 255) / 256), 256, 0, st>>>(
        tb.start.as<int32_t>(), p.n, p.channels, tb.nseg, p.sw, p.mr, tb.seg_range.as<int32_t>());
    note_launch();
    check_launch("seg_ranges_kernel");
    tb.h_seg_range.resize(static_cast<size_t>(cnt) * 4);
    NUS_CUDA(cudaMemcpyAsync(tb.h_seg_range.data(), tb.seg_range.ptr, tb.seg_range.bytes, cudaMemcpyDeviceToHost, st));
  }
  tb.deconv.alloc(p.nc * rs);
  if (p.kernel == NUS_KERNEL_ES) {
    std::vector<double> pairs(2 * kEsQuad);
    es_quadrature(p.sw, kEsQuad, pairs.data());
    DeviceBuffer dq(pairs.size() * sizeof(double));
    NUS_CUDA(cudaMemcpyAsync(dq.ptr, pairs.data(), dq.bytes, cudaMemcpyHostToDevice, st));
    const double a_per_mode = kPi * static_cast<double>(p.sw) / static_cast<double>(p.mr);
    if (p.precision == NUS_F64)
      deconv_es_kernel<double><<<static_cast<unsigned>((p.nc + 255) / 256), 256, 0, st>>>(
          p.nc, p.mode_offset, a_per_mode, static_cast<double>(p.sw), dq.as<double>(), tb.deconv.as<double>());
    else
      deconv_es_kernel<float><<<static_cast<unsigned>((p.nc + 255) / 256), 256, 0, st>>>(
          p.nc, p.mode_offset, a_per_mode, static_cast<double>(p.sw), dq.as<double>(), tb.deconv.as<float>());
    note_launch();
    check_launch("deconv_es_kernel");
    NUS_CUDA(cudaStreamSynchronize(st));  // dq is released at scope end
  } else if (p.precision == NUS_F64)
    deconv_kernel<double><<<static_cast<unsigned>((p.nc + 255) / 256), 256, 0, st>>>(
        p.nc, p.mode_offset, p.tau, p.deconv_norm, tb.deconv.as<double>());
  else
    deconv_kernel<float><<<static_cast<unsigned>((p.nc + 255) / 256), 256, 0, st>>>(
        p.nc, p.mode_offset, p.tau, p.deconv_norm, tb.deconv.as<float>());
  note_launch();
  check_launch("deconv_kernel");
  NUS_CUDA(cudaStreamSynchronize(st));
  // NUS_FFT=generic forces the generic radix-2 kernels (test hook for every grid size)
  const char* fft_env = std::getenv("NUS_FFT");
  if (!(fft_env && std::strcmp(fft_env, "generic") == 0)) fused_fft_prepare(plan);
  FusedFft& ff = plan.ffft;
  ff.row_lo = 0;
  ff.row_cnt = ff.R;
  if (ff.ready && ff.blocked && p.n > 0) {
    // minimal cyclic row interval covering every occupied row: complement of the largest gap
    DeviceBuffer occ(static_cast<size_t>(ff.R));
    NUS_CUDA(cudaMemsetAsync(occ.ptr, 0, occ.bytes, st));
    const int64_t total = p.channels * p.n;
    row_occupancy_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        tb.start.as<int32_t>(), total, p.sw, p.mr, ff.lgC, occ.as<uint8_t>());
    note_launch();
    check_launch("row_occupancy_kernel");
    std::vector<uint8_t> h(ff.R);
    NUS_CUDA(cudaMemcpyAsync(h.data(), occ.ptr, ff.R, cudaMemcpyDeviceToHost, st));
    NUS_CUDA(cudaStreamSynchronize(st));
    int best_len = 0, best_end = 0;  // largest run of empty rows, cyclic
    for (int start_row = 0; start_row < ff.R; ++start_row) {
      if (h[start_row] || h[(start_row + ff.R - 1) % ff.R] == 0) continue;  // runs start after an occupied row
      int len = 0;
      while (len < ff.R && h[(start_row + len) % ff.R] == 0) ++len;
      if (len > best_len) {
        best_len = len;
        best_end = (start_row + len) % ff.R;
      }
    }
    if (best_len > 0 && best_len < ff.R) {
      ff.row_lo = best_end;
      ff.row_cnt = ff.R - best_len;
    }
  }
}

std::unique_ptr<Plan> plan_create(const double* times, int64_t channels, int64_t n,
                                  const double* centers, int64_t nc, double eps, int policy,
                                  int oversampling, int precision, int device) {
  require(times != nullptr && centers != nullptr, "NufftPlan: null input");
  require(channels >= 1, "NufftPlan: channels must be >= 1");
  require(precision == NUS_F64 || precision == NUS_F32, "NufftPlan: unknown precision");
  // SamplingGrid invariants (grid.cpp:9-22), per channel.
  require(n >= 2, "SamplingGrid: need at least 2 samples");
  for (int64_t c = 0; c < channels; ++c) {
    const double* t = times + c * n;
    for (int64_t i = 0; i < n; ++i) {
      require(std::isfinite(t[i]), "SamplingGrid: non-finite sample time");
      require(i == 0 || t[i] > t[i - 1], "SamplingGrid: times must be strictly increasing");
    }
  }
  use_device(device);
  auto plan = std::make_unique<Plan>();
  plan->device = device;
  plan->p.n = n;
  plan->p.channels = channels;
  plan->p.precision = precision;
  plan_validate_and_select(plan->p, centers, nc, eps, policy, oversampling);
  plan->times.assign(times, times + channels * n);
  plan->centers.assign(centers, centers + nc);
  plan->d_times.alloc(channels * n * sizeof(double));
  plan->d_centers.alloc(nc * sizeof(double));
  NUS_CUDA(cudaMemcpy(plan->d_times.ptr, times, channels * n * sizeof(double), cudaMemcpyHostToDevice));
  NUS_CUDA(cudaMemcpy(plan->d_centers.ptr, centers, nc * sizeof(double), cudaMemcpyHostToDevice));
  if (plan->p.path == NUS_PATH_FAST) plan_build_tables(*plan, 0);
  return plan;
}

// ---- direct NUDFT (nufft.cpp:36-54, :174-186) --------------------------------

namespace {

template <typename YT, typename OT>
__global__ void ndft_kernel(const double* __restrict__ t, int64_t n, const YT* __restrict__ y,
                            const double* __restrict__ c, int64_t nc, OT* __restrict__ out) {
  const int64_t i = blockIdx.x;
  const int64_t b = blockIdx.y;
  const double a = __dmul_rn(-kTwoPi, c[i]);
  const YT* yb = y + 2 * b * n;
  double ar = 0.0, ai = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    double sn, cs;
    sincos(__dmul_rn(a, t[k]), &sn, &cs);
    const double yr = static_cast<double>(yb[2 * k]), yi = static_cast<double>(yb[2 * k + 1]);
    ar += yr * cs - yi * sn;
    ai += yr * sn + yi * cs;
  }
  __shared__ double sr[32], si[32];
  for (int off = 16; off > 0; off >>= 1) {
    ar += __shfl_down_sync(0xffffffffu, ar, off);
    ai += __shfl_down_sync(0xffffffffu, ai, off);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sr[wid] = ar; si[wid] = ai; }
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    ar = lane < nw ? sr[lane] : 0.0;
    ai = lane < nw ? si[lane] : 0.0;
    for (int off = 16; off > 0; off >>= 1) {
      ar += __shfl_down_sync(0xffffffffu, ar, off);
      ai += __shfl_down_sync(0xffffffffu, ai, off);
    }
    if (lane == 0) {
      out[2 * (b * nc + i)] = static_cast<OT>(ar);
      out[2 * (b * nc + i) + 1] = static_cast<OT>(ai);
    }
  }
}

}  // namespace

void launch_ndft_direct(const double* d_t, int64_t n, const void* d_y, bool y_f32,
                        const double* d_c, int64_t nc, void* d_out, bool out_f32, int64_t batch,
                        cudaStream_t s) {
  const dim3 grid(static_cast<unsigned>(nc), static_cast<unsigned>(batch));
  const int threads = n >= 256 ? 256 : 32 * static_cast<int>((n + 31) / 32);
  if (!y_f32 && !out_f32)
    ndft_kernel<double, double><<<grid, threads, 0, s>>>(d_t, n, static_cast<const double*>(d_y), d_c, nc,
                                                          static_cast<double*>(d_out));
  else if (y_f32 && out_f32)
    ndft_kernel<float, float><<<grid, threads, 0, s>>>(d_t, n, static_cast<const float*>(d_y), d_c, nc,
                                                        static_cast<float*>(d_out));
  else if (!y_f32 && out_f32)
    ndft_kernel<double, float><<<grid, threads, 0, s>>>(d_t, n, static_cast<const double*>(d_y), d_c, nc,
                                                         static_cast<float*>(d_out));
  else
    ndft_kernel<float, double><<<grid, threads, 0, s>>>(d_t, n, static_cast<const float*>(d_y), d_c, nc,
                                                         static_cast<double*>(d_out));
  note_launch();
  check_launch("ndft_kernel");
}

}  // namespace nus
