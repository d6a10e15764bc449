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
// around the support centre).  Each WARP then owns 32 consecutive cells (one
// per lane) and walks, in lock-step, the staged points whose support meets
// them: the point's z_k are warp-wide shared-memory broadcasts (one
// wavefront per 16 B) and only the Gaussian weight is a per-lane read, so
// there is no per-lane search and no trip-count divergence.  K complex
// accumulators per cell live in registers.  Every cell of the grid is written
// exactly once (zeros included), so no memset.
#include <algorithm>

#include "nus_internal.cuh"

namespace nus {

namespace {

constexpr int kThreads = 128;
constexpr int kTile = kThreads;      // one cell per thread, 32 per warp
constexpr int kBatch = 128;          // points staged per pass (a C2 tile holds ~76)
constexpr int kMaxW2 = 64;

template <typename Real> struct Vec2;
template <> struct Vec2<double> { using T = double2; };
template <> struct Vec2<float> { using T = float2; };

template <typename Real>
struct SpreadParams {
  const int32_t* start;
  const int32_t* perm;
  const typename Vec2<Real>::T* gauss;  // per point (A, g): W_p = A g^p C_p
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

template <typename Real, int KG>
__global__ void __launch_bounds__(kThreads, 5) spread_gather_kernel(const SpreadParams<Real> P) {
  using R2 = typename Vec2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R2* sm_z = reinterpret_cast<R2*>(smem_raw);                         // [kBatch][KG]
  Real* sm_w = reinterpret_cast<Real*>(sm_z + kBatch * KG);          // [kBatch][w2s]
  const int w2s = P.w2 + 1;  // odd stride (w2 is even) spreads rows over banks
  int* sm_rel = reinterpret_cast<int*>(sm_w + kBatch * w2s);         // [kBatch]

  const int64_t tile_id = blockIdx.x;
  const int64_t c = blockIdx.y;
  const int64_t c0 = tile_id * P.tile;
  const int64_t base = c * P.n;
  const int lane = threadIdx.x & 31;
  const int wcell = threadIdx.x & ~31;        // warp's first cell inside the tile
  const int cell = threadIdx.x;               // this lane's cell inside the tile
  const bool warp_live = wcell < P.tile;

  R2 acc[KG];
#pragma unroll
  for (int k = 0; k < KG; ++k) acc[k] = R2{Real(0), Real(0)};

  const int32_t* rng = P.ranges + 2 * (c * (P.ntiles + 1) + tile_id);
  // segment 0: wrapping points (tile 0 only); segment 1: the tile's own range
  const int wrap_lo = tile_id == 0 ? P.wrap_lo[c] : 0;
  const int wrap_hi = tile_id == 0 ? static_cast<int>(P.n) : 0;
  const int own_lo = rng[0], own_hi = rng[1];

  for (int seg = 0; seg < 2; ++seg) {
    const int lo_s = seg == 0 ? wrap_lo : own_lo;
    const int hi_s = seg == 0 ? wrap_hi : own_hi;
    const int64_t shift = seg == 0 ? c0 + P.mr : c0;
    for (int b0 = lo_s; b0 < hi_s; b0 += kBatch) {
      const int nb = min(kBatch, hi_s - b0);
      __syncthreads();
      for (int j = threadIdx.x; j < nb; j += kThreads) {
        const int64_t gi = base + b0 + j;
        const int32_t ti = P.perm[gi];
        sm_rel[j] = static_cast<int>(static_cast<int64_t>(P.start[gi]) - shift);
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
        const R2 ph = reinterpret_cast<const R2*>(P.prephase)[gi];
        const Real yr = xr * ph.x - xi * ph.y;
        const Real yi = xr * ph.y + xi * ph.x;
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          Real wk = Real(1);
          if (P.tapers != nullptr) wk = P.tapers[(c * P.k_total + P.k0 + k) * P.n + (b0 + j)];
          sm_z[j * KG + k] = R2{wk * yr, wk * yi};
        }
        // Gaussian weights W_p = A g^p C_p (A, g precomputed per point at plan time);
        // two interleaved recurrences (even / odd p) halve the dependent chain.
        const R2 ag = P.gauss[gi];
        const Real g2 = ag.y * ag.y;
        Real ae = ag.x;
        Real ao = ag.x * ag.y;
        Real* wrow = sm_w + j * w2s;
        for (int p = 0; p < P.w2; p += 2) {
          wrow[p] = ae * P.cq[p];
          wrow[p + 1] = ao * P.cq[p + 1];
          ae *= g2;
          ao *= g2;
        }
      }
      __syncthreads();
      if (!warp_live) continue;
      // points of this batch meeting the warp's cells [wcell, wcell+32): count the staged
      // rel values below each bound with ballots (no serial search)
      int lo = 0, hi = 0;
      for (int j0 = 0; j0 < nb; j0 += 32) {
        const int j = j0 + lane;
        const int r = j < nb ? sm_rel[j] : 0x7fffffff;
        lo += __popc(__ballot_sync(0xffffffffu, r < wcell - (P.w2 - 1)));
        hi += __popc(__ballot_sync(0xffffffffu, r < wcell + 32));
      }
      for (int i = lo; i < hi; ++i) {
        const int p = cell - sm_rel[i];            // broadcast read
        const bool in = p >= 0 && p < P.w2;
        const Real wt = in ? sm_w[i * w2s + (in ? p : 0)] : Real(0);
        const R2* zr = sm_z + i * KG;
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          const R2 z = zr[k];                      // broadcast read
          acc[k].x = fma(wt, z.x, acc[k].x);
          acc[k].y = fma(wt, z.y, acc[k].y);
        }
      }
    }
  }
  // write every cell of the tile (zeros included): 32 consecutive cells per warp and row
  if (cell >= P.tile) return;
#pragma unroll
  for (int k = 0; k < KG; ++k)
    P.grid[(c * P.kpad + P.k0 + k) * P.mr + c0 + cell] = acc[k];
  (void)lane;
}

template <typename Real, int KG>
void launch_group(const SpreadParams<Real>& P, int64_t channels, cudaStream_t s) {
  const size_t smem = kBatch * KG * sizeof(typename Vec2<Real>::T) +
                      kBatch * static_cast<size_t>(P.w2 + 1) * sizeof(Real) + kBatch * sizeof(int);
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
  require(tb.tile == kTile || p.mr < kTile, "spread: unexpected tile size");
  require(2 * p.w <= kMaxW2, "spread: spread width too large");
  SpreadParams<Real> P{};
  P.start = tb.start.as<int32_t>();
  P.perm = tb.perm.as<int32_t>();
  P.gauss = tb.gauss.as<typename Vec2<Real>::T>();
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
