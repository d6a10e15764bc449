// The FFT + crop entry points of the path (run_fft / run_crop / run_transform).
//
// Fused path (fft.cu, 512 <= Mr <= 2^26): pass A here, pass B fused with the crop and the
// eigenspectrum reduction.  Other grid sizes: the generic radix-2 Stockham kernels
// (e^{-2 pi i jk/Mr} as Radix2Fft::forward, src/fft.cpp:39-58) followed by one fused
// deconvolve / crop / eigenspectrum kernel:
//     J_k(i) = deconv_i * B_k[(-m_i) mod Mr],  m_i = i - I/2   (src/nufft.cpp:131-140,161-164)
//     P(i)   = (sum_k |J_k(i)|^2) / K                           (src/estimators.cpp:113-117)
// The power reduction over tapers happens in registers, so J never has to be
// written unless the caller asks for eigencoefficients.
#include "nus_internal.cuh"

namespace nus {

namespace {

template <typename Real> struct V2;
template <> struct V2<double> { using T = double2; };
template <> struct V2<float> { using T = float2; };

template <typename Real, typename PReal>
__global__ void crop_power_kernel(const typename V2<Real>::T* __restrict__ grid, int64_t kpad,
                                  int64_t k, int64_t mr, int64_t nc, int64_t mode_offset,
                                  const Real* __restrict__ deconv, typename V2<Real>::T* __restrict__ j_out,
                                  PReal* __restrict__ power, double divisor, int accumulate) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (i >= nc) return;
  const int64_t m = i - mode_offset;
  int64_t bin = (-m) % mr;
  if (bin < 0) bin += mr;
  const Real d = deconv[i];
  const typename V2<Real>::T* g = grid + c * kpad * mr + bin;
  Real acc = Real(0);
  for (int64_t kk = 0; kk < k; ++kk) {
    const typename V2<Real>::T b = g[kk * mr];
    const Real jr = d * b.x, ji = d * b.y;
    if (j_out) j_out[(c * k + kk) * nc + i] = typename V2<Real>::T{jr, ji};
    acc += jr * jr + ji * ji;
  }
  if (power) {
    const PReal v = static_cast<PReal>(static_cast<double>(acc) / divisor);
    PReal* dst = power + c * nc + i;
    *dst = accumulate ? *dst + v : v;
  }
}

}  // namespace

void run_fft(Plan& plan, void* grid, int64_t k, int64_t kpad, cudaStream_t s) {
  if (plan.ffft.ready) {  // fused two-pass FFT: pass A here, pass B fused with the crop
    run_fused_pass_a(plan, grid, k, kpad, s);
    return;
  }
  const PlanParams& p = plan.p;
  const bool f64 = p.precision == NUS_F64;
  const size_t need = static_cast<size_t>(p.channels * k * p.mr) * (f64 ? sizeof(double2) : sizeof(float2));
  if (plan.ffft.scratch.bytes < need) {
    NUS_CUDA(cudaStreamSynchronize(s));
    plan.ffft.scratch.alloc(need);
  }
  fft_generic_rows(grid, p.mr, p.channels * k, k, kpad, f64, false, plan.ffft.scratch.ptr, s);
}

void run_crop(Plan& plan, void* grid, int64_t k, int64_t kpad, void* j_out, void* power,
              bool power_f64, double divisor, bool accumulate, cudaStream_t s) {
  if (plan.ffft.ready) {
    run_fused_pass_b(plan, grid, k, kpad, j_out, power, power_f64, divisor, accumulate, s);
    return;
  }
  const PlanParams& p = plan.p;
  const bool f64 = p.precision == NUS_F64;
  const dim3 gridd(static_cast<unsigned>((p.nc + 255) / 256), static_cast<unsigned>(p.channels));
  const int acc = accumulate ? 1 : 0;
  if (f64)
    crop_power_kernel<double, double><<<gridd, 256, 0, s>>>(
        static_cast<const double2*>(grid), kpad, k, p.mr, p.nc, p.mode_offset,
        plan.tab.deconv.as<double>(), static_cast<double2*>(j_out), static_cast<double*>(power),
        divisor, acc);
  else if (power_f64)
    crop_power_kernel<float, double><<<gridd, 256, 0, s>>>(
        static_cast<const float2*>(grid), kpad, k, p.mr, p.nc, p.mode_offset,
        plan.tab.deconv.as<float>(), static_cast<float2*>(j_out), static_cast<double*>(power),
        divisor, acc);
  else
    crop_power_kernel<float, float><<<gridd, 256, 0, s>>>(
        static_cast<const float2*>(grid), kpad, k, p.mr, p.nc, p.mode_offset,
        plan.tab.deconv.as<float>(), static_cast<float2*>(j_out), static_cast<float*>(power),
        divisor, acc);
  note_launch();
  check_launch("crop_power_kernel");
}

void run_transform(Plan& plan, void* grid, int64_t k, int64_t kpad, void* j_out, void* power,
                   bool power_f64, double divisor, bool accumulate, cudaStream_t s) {
  run_fft(plan, grid, k, kpad, s);
  run_crop(plan, grid, k, kpad, j_out, power, power_f64, divisor, accumulate, s);
}

}  // namespace nus
