// Gaussian-gridding spread of K taper-weighted series onto the oversampled
// grid, as a deterministic, atomic-free GATHER over start-cell-sorted points.
//
// Replaces the reference's per-taper serial scatter (src/nufft.cpp:150-159
// with simd::spread_accum, src/simd_avx2.cpp:158-171) and the taper x signal
// product (src/nufft.cpp:213-216, simd::mul_real): one pass over the samples
// produces all K grids.
//
// Each CTA owns a tile of T consecutive cells for one channel and one group
// of up to KG tapers.  It walks the (contiguous, pre-computed) range of
// sorted points whose 2w-cell support meets the tile, staging batches of
// points in shared memory:
//     rel  = start cell - tile origin           (ascending inside a batch)
//     z_k  = w_k(t) * x * e^{-i 2 pi fshift t}  (k < KG)
//     W_p  = exp(-beta (d - p)^2),  p < 2w,  d = frac + w - 1
// where W_p uses one exp pair per point (Greengard-Lee style factorisation
// around the support centre).  Each thread then owns R consecutive cells and
// sums the contributions of the points covering them (binary search in the
// staged batch), accumulating K complex values per cell in registers.  Every
// cell of the grid is written exactly once (zeros included), so no memset.
#include <algorithm>

#include "nus_internal.cuh"

namespace nus {

namespace {

constexpr int kThreads = 256;
constexpr int kCellsPerThread = 2;   // R
constexpr int kBatch = 128;          // points staged per pass
constexpr int kMaxW2 = 64;

template <typename Real> struct Vec2;
template <> struct Vec2<double> { using T = double2; };
template <> struct Vec2<float> { using T = float2; };

template <typename Real>
struct SpreadParams {
  const int32_t* start;
  const int32_t* perm;
  const Real* frac;
  const Real* prephase;
  const int32_t* ranges;
  const int32_t* wrap_lo;
  const Real* tapers;     // sorted-order [C][K][n] or null
  const void* x;          // [C][n] time order
  typename Vec2<Real>::T* grid;  // [C][kpad][mr]
  int64_t n, mr, ntiles, kpad, k_total;
  int64_t s0, s1;
  int tile, w, w2, k0, kg, x_dtype, x_complex;
  Real beta, cq[kMaxW2];
};

__device__ inline int lower_bound_smem(const int* a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <typename Real, int KG>
__global__ void __launch_bounds__(kThreads) spread_gather_kernel(const SpreadParams<Real> P) {
  using R2 = typename Vec2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R2* sm_z = reinterpret_cast<R2*>(smem_raw);                         // [kBatch][KG]
  Real* sm_w = reinterpret_cast<Real*>(sm_z + kBatch * KG);          // [kBatch][w2s]
  const int w2s = P.w2 | 1;
  int* sm_rel = reinterpret_cast<int*>(sm_w + kBatch * w2s);         // [kBatch]

  const int64_t tile_id = blockIdx.x;
  const int64_t c = blockIdx.y;
  const int kg = P.kg;
  const int64_t c0 = tile_id * P.tile;
  const int64_t base = c * P.n;
  const int r0 = threadIdx.x * kCellsPerThread;

  R2 acc[kCellsPerThread][KG];
#pragma unroll
  for (int j = 0; j < kCellsPerThread; ++j)
#pragma unroll
    for (int k = 0; k < KG; ++k) acc[j][k] = R2{Real(0), Real(0)};

  const int32_t* rng = P.ranges + 2 * (c * (P.ntiles + 1) + tile_id);
  // segment 0: wrapping points (tile 0 only); segment 1: the tile's own range
  const int seg_lo[2] = {tile_id == 0 ? P.wrap_lo[c] : 0, rng[0]};
  const int seg_hi[2] = {tile_id == 0 ? static_cast<int>(P.n) : 0, rng[1]};
  const int64_t seg_shift[2] = {c0 + P.mr, c0};

  for (int seg = 0; seg < 2; ++seg) {
    for (int b0 = seg_lo[seg]; b0 < seg_hi[seg]; b0 += kBatch) {
      const int nb = min(kBatch, seg_hi[seg] - b0);
      __syncthreads();
      for (int j = threadIdx.x; j < nb; j += kThreads) {
        const int64_t gi = base + b0 + j;
        const int32_t ti = P.perm[gi];
        sm_rel[j] = static_cast<int>(static_cast<int64_t>(P.start[gi]) - seg_shift[seg]);
        // sample value times prephase
        Real xr, xi;
        if (P.x_complex) {
          if (P.x_dtype == 0) {
            const double* xv = static_cast<const double*>(P.x) + 2 * (base + ti);
            xr = static_cast<Real>(xv[0]); xi = static_cast<Real>(xv[1]);
          } else {
            const float* xv = static_cast<const float*>(P.x) + 2 * (base + ti);
            xr = static_cast<Real>(xv[0]); xi = static_cast<Real>(xv[1]);
          }
        } else {
          xr = P.x_dtype == 0 ? static_cast<Real>(static_cast<const double*>(P.x)[base + ti])
                              : static_cast<Real>(static_cast<const float*>(P.x)[base + ti]);
          xi = Real(0);
        }
        if (ti < P.s0 || ti >= P.s1) { xr = Real(0); xi = Real(0); }
        const Real pr = P.prephase[2 * gi], pi = P.prephase[2 * gi + 1];
        const Real yr = xr * pr - xi * pi;
        const Real yi = xr * pi + xi * pr;
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          Real wk = Real(1);
          if (P.tapers != nullptr && k < kg)
            wk = P.tapers[(c * P.k_total + P.k0 + k) * P.n + (b0 + j)];
          if (k >= kg) wk = Real(0);
          sm_z[j * KG + k] = R2{wk * yr, wk * yi};
        }
        // Gaussian weights W_p = A g^p C_p, fr' = frac - 1/2
        const Real fr = P.frac[gi] - Real(0.5);
        Real gval = exp(Real(2) * P.beta * fr);
        Real a = exp(-P.beta * fr * (fr + Real(P.w2 - 1)));
        Real* wrow = sm_w + j * w2s;
        for (int p = 0; p < P.w2; ++p) {
          wrow[p] = a * P.cq[p];
          a *= gval;
        }
      }
      __syncthreads();
      const int lo = lower_bound_smem(sm_rel, nb, r0 - (P.w2 - 1));
      const int hi = lower_bound_smem(sm_rel, nb, r0 + kCellsPerThread);
      for (int i = lo; i < hi; ++i) {
        const int p0 = r0 - sm_rel[i];
        R2 z[KG];
#pragma unroll
        for (int k = 0; k < KG; ++k) z[k] = sm_z[i * KG + k];
        const Real* wrow = sm_w + i * w2s;
#pragma unroll
        for (int j = 0; j < kCellsPerThread; ++j) {
          const int p = p0 + j;
          if (p >= 0 && p < P.w2) {
            const Real wt = wrow[p];
#pragma unroll
            for (int k = 0; k < KG; ++k) {
              acc[j][k].x = fma(wt, z[k].x, acc[j][k].x);
              acc[j][k].y = fma(wt, z[k].y, acc[j][k].y);
            }
          }
        }
      }
    }
  }
  // write every cell of the tile (zeros included)
  if (r0 >= P.tile) return;
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    if (k < kg) {
      R2* row = P.grid + (c * P.kpad + P.k0 + k) * P.mr + c0 + r0;
#pragma unroll
      for (int j = 0; j < kCellsPerThread; ++j) row[j] = acc[j][k];
    }
  }
}

template <typename Real, int KG>
void launch_group(const SpreadParams<Real>& P, int64_t channels, cudaStream_t s) {
  const size_t smem = kBatch * KG * sizeof(typename Vec2<Real>::T) +
                      kBatch * static_cast<size_t>(P.w2 | 1) * sizeof(Real) + kBatch * sizeof(int);
  static bool configured = false;
  if (!configured) {
    NUS_CUDA(cudaFuncSetAttribute(spread_gather_kernel<Real, KG>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    configured = true;
  }
  const dim3 grid(static_cast<unsigned>(P.ntiles), static_cast<unsigned>(channels));
  spread_gather_kernel<Real, KG><<<grid, kThreads, smem, s>>>(P);
  note_launch();
  check_launch("spread_gather_kernel");
}

template <typename Real>
void spread_typed(const Plan& plan, const SpreadArgs& a, cudaStream_t s) {
  const PlanParams& p = plan.p;
  const SpreadTables& tb = plan.tab;
  require(tb.tile == kThreads * kCellsPerThread || p.mr < kThreads * kCellsPerThread,
          "spread: unexpected tile size");
  require(2 * p.w <= kMaxW2, "spread: spread width too large");
  SpreadParams<Real> P{};
  P.start = tb.start.as<int32_t>();
  P.perm = tb.perm.as<int32_t>();
  P.frac = tb.frac.as<Real>();
  P.prephase = tb.prephase.as<Real>();
  P.ranges = tb.tile_range.as<int32_t>();
  P.wrap_lo = tb.wrap_lo.as<int32_t>();
  P.tapers = static_cast<const Real*>(a.tapers);
  P.x = a.x;
  P.grid = static_cast<typename Vec2<Real>::T*>(a.grid);
  P.n = p.n;
  P.mr = p.mr;
  P.ntiles = tb.ntiles;
  P.kpad = a.kpad;
  P.k_total = a.k;
  P.s0 = a.s0;
  P.s1 = a.s1 < 0 ? p.n : a.s1;
  P.tile = tb.tile;
  P.w = p.w;
  P.w2 = 2 * p.w;
  P.x_dtype = a.x_dtype;
  P.x_complex = a.x_complex ? 1 : 0;
  P.beta = static_cast<Real>(p.beta);
  for (int q = 0; q < P.w2; ++q) {
    const double qc = static_cast<double>(q) - (static_cast<double>(p.w) - 0.5);
    P.cq[q] = static_cast<Real>(std::exp(-p.beta * qc * qc));
  }
  // taper groups of at most 8, balanced
  const int64_t k = a.tapers ? a.k : 1;
  const int64_t groups = (k + 7) / 8;
  int64_t k0 = 0;
  for (int64_t gidx = 0; gidx < groups; ++gidx) {
    const int64_t kg = (k - k0 + (groups - gidx) - 1) / (groups - gidx);
    P.k0 = static_cast<int>(k0);
    P.kg = static_cast<int>(kg);
    switch (kg) {
      case 1: launch_group<Real, 1>(P, p.channels, s); break;
      case 2: launch_group<Real, 2>(P, p.channels, s); break;
      case 3: launch_group<Real, 3>(P, p.channels, s); break;
      case 4: launch_group<Real, 4>(P, p.channels, s); break;
      case 5: launch_group<Real, 5>(P, p.channels, s); break;
      case 6: launch_group<Real, 6>(P, p.channels, s); break;
      case 7: launch_group<Real, 7>(P, p.channels, s); break;
      default: launch_group<Real, 8>(P, p.channels, s); break;
    }
    k0 += kg;
  }
}

}  // namespace

void launch_spread(const Plan& plan, const SpreadArgs& a, cudaStream_t s) {
  if (plan.p.precision == NUS_F64)
    spread_typed<double>(plan, a, s);
  else
    spread_typed<float>(plan, a, s);
}

}  // namespace nus
