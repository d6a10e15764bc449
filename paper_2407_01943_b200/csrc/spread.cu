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
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

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
  int64_t channels, nseg;
  int blocked, lgC, lgCW, lgT;  // blocked grid layout of the fused FFT (FusedFft::blocked)
  int lg_nseg;
  // items = channels * nseg_used segments: rows (of 2^lg_spr segments) row_lo .. row_lo+row_cnt-1
  // (cyclic mod nrows) of each channel; other rows are never written (FusedFft::row_lo)
  int lg_spr, row_lo, nrows;
  int64_t nseg_used;
  const Real* taper_base;  // tapers, or a device constant 1 with zero strides
  int64_t tstride_k, tstride_j;
  const int32_t* seg_ranges;
  typename Vec2<Real>::T* const* slots;  // fused sample-split exchange (SpreadArgs::slots) or null
  int64_t per;
  const int32_t* units;  // streaming spread: work units (SpreadTables::Units)
  const int32_t* warp_first;  // warp w runs units [warp_first[w], warp_first[w + 1])
  int nunits;
  int tile, w, w2, k0, kg, x_dtype, x_complex;
  Real beta, cq[kMaxW2];
  // tensor-core staging: W_{p+2} = W_p * q_p, q_{p+2} = q_p * ve (even / odd chains)
  double c0, c1, qe0, qo0, ve;
};

// Grid address of cell j: natural, or the fused FFT's blocked layout (j = j1 C + j2 stored
// at (j2 / CW) * 2^lgT + j1 * CW + j2 % CW, so each pass-A column block is contiguous).
__device__ inline int64_t cell_addr(int64_t j, int blocked, int lgC, int lgCW, int lgT) {
  if (!blocked) return j;
  const int64_t j1 = j >> lgC, j2 = j & ((int64_t{1} << lgC) - 1);
  return ((j2 >> lgCW) << lgT) | (j1 << lgCW) | (j2 & ((int64_t{1} << lgCW) - 1));
}

__device__ inline int cell_addr32(int j, int blocked, int lgC, int lgCW, int lgT) {
  if (!blocked) return j;
  const int j1 = j >> lgC, j2 = j & ((1 << lgC) - 1);
  return ((j2 >> lgCW) << lgT) | (j1 << lgCW) | (j2 & ((1 << lgCW) - 1));
}

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
    P.grid[(c * P.kpad + P.k0 + k) * P.mr + cell_addr(c0 + cell, P.blocked, P.lgC, P.lgCW, P.lgT)] = acc[k];
  (void)lane;
}

// ---- persistent, warp-independent FP64 tensor-core spread (default) ---------------------
// The banded product of spread_gather_kernel on mma.sync m8n8k4 f64 (DMMA): per 8-cell
// block, G(8 cells x 8 tapers) += W(8 cells x 4 points) Z(4 points x 8 tapers); lane
// (g, t) holds a = W(cell g, point t), b = z(point t, taper g) and accumulates G(cell g,
// tapers 2t, 2t+1) (layout checked by tests/micro/dmma_layout.cu); one MMA for Re z, one
// for Im z.  That is 256 complex MACs per ~11 instructions against the gather's 224 per 31,
// so what remains is staging latency, which is hidden by making every WARP an independent,
// persistent worker: it owns 32-cell segments (4 blocks), stages up to 32 points per round
// (one per lane) into its private shared rows, and finds each block's point range with two
// ballots; no CTA barrier anywhere.  The global loads of round n+1 (and the perm index of
// round n+2, so the x gather never waits on a dependent load) are in flight while round n
// runs on the tensor cores.
//
// Private tables (row stride kTcRows = 36 = 4 mod 16): Z[taper][point] = (re, im) and
// W[point][slot] with slot = cell mod 32, holding W(cell - rel) on the point's support only
// (never cleared: off-support slots are masked by a range test on cell - rel).  Lane (g, t)
// reads Z[g][p0+t] and W[p0+t][8b+g]: bank-conflict free for any rel.  rel of an absent
// point is a far sentinel; points 32..35 absorb the last 4-point step's overrun.
constexpr int kTcWarps = 3;       // warps per CTA (each an independent worker)
constexpr int kTcRows = 36;       // row stride of the private tables (= 4 mod 16)
// staged point rows: 32 + the last 4-point step's overrun (p <= 34); with two taper groups the
// overrun rows read row 31 instead (masked by their sentinel rel), so 4 CTAs/SM fit
__host__ __device__ constexpr int tc_pts(int groups) { return groups == 1 ? 35 : 32; }
constexpr int kTcCtasPerSm = 5;

__device__ inline void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// A warp's walk over its rounds: item = channel * nseg_used + s (s indexes the channel's used
// segments); each segment visits its wrapping points (part 0, segments with s0 < w2-1) then
// its own (part 1), 32 at a time; a segment without points still yields one empty round so
// that its cells are written.  Only the furthest cursor advances; the segment range it will
// need next is prefetched one item ahead (`pre`, at position `pp`), so no cursor step waits on
// a global load.  Items are carried as (channel, s) and stepped by the stride with a wrap, so
// the walk has no integer division.
struct TcCursor {
  int64_t seg, shift;
  int c, part, b0, hi, nb, own_lo, own_hi;
  bool valid, last;
};
struct TcPos {
  int c, s;
};

template <typename Real>
__device__ inline void tc_step(TcPos& p, int stride, const SpreadParams<Real>& P) {
  p.s += stride;
  while (p.s >= static_cast<int>(P.nseg_used)) {
    p.s -= static_cast<int>(P.nseg_used);
    ++p.c;
  }
}

// used-segment index -> segment: rows row_lo .. row_lo + row_cnt - 1 (cyclic) of the channel
template <typename Real>
__device__ inline int64_t tc_seg(int s, const SpreadParams<Real>& P) {
  const int64_t row = ((s >> P.lg_spr) + P.row_lo) & (P.nrows - 1);
  return (row << P.lg_spr) | (s & ((1 << P.lg_spr) - 1));
}

template <typename Real>
__device__ inline int4 tc_range(TcPos p, const SpreadParams<Real>& P) {
  // unconditional (clamped) load: a conditional one merges with a default and the merge
  // waits on the load; past-the-end items are never settled (valid = false)
  const bool ok = p.c < static_cast<int>(P.channels);
  const int c = ok ? p.c : static_cast<int>(P.channels) - 1;
  const int s = ok ? p.s : static_cast<int>(P.nseg_used) - 1;
  return reinterpret_cast<const int4*>(P.seg_ranges)[static_cast<int64_t>(c) * P.nseg + tc_seg(s, P)];
}

template <typename Real>
__device__ inline void tc_settle(TcCursor& u, TcPos p, int4 r, const SpreadParams<Real>& P) {
  if (p.c >= static_cast<int>(P.channels)) {
    u.valid = false;
    u.nb = 0;
    u.last = false;
    return;
  }
  u.valid = true;
  u.c = p.c;
  u.seg = tc_seg(p.s, P);
  u.own_lo = r.x;
  u.own_hi = r.y;
  if (r.z < static_cast<int>(P.n)) {
    u.part = 0;
    u.b0 = r.z;
    u.hi = static_cast<int>(P.n);
    u.shift = u.seg * 32 + P.mr;
  } else {
    u.part = 1;
    u.b0 = r.x;
    u.hi = r.y;
    u.shift = u.seg * 32;
  }
  u.nb = max(0, min(32, u.hi - u.b0));
  u.last = u.b0 + 32 >= u.hi && (u.part == 1 || u.own_hi <= u.own_lo);
}

template <typename Real>
__device__ inline void tc_advance(TcCursor& u, int4& pre, TcPos& pp, const SpreadParams<Real>& P, int stride) {
  if (!u.valid) return;
  if (u.b0 + 32 < u.hi) {
    u.b0 += 32;
  } else if (u.part == 0 && u.own_hi > u.own_lo) {
    u.part = 1;
    u.b0 = u.own_lo;
    u.hi = u.own_hi;
    u.shift = u.seg * 32;
  } else {
    const TcPos next = pp;  // its range is `pre`, loaded one item ago
    const int4 r = pre;
    tc_step(pp, stride, P);
    pre = tc_range(pp, P);
    tc_settle(u, next, r, P);
    return;
  }
  u.nb = min(32, u.hi - u.b0);
  // the segment's final round: the last of part 1, or of part 0 when it has no own points
  // (a multi-round part 0 of an own-empty segment must still write its cells)
  u.last = u.b0 + 32 >= u.hi && (u.part == 1 || u.own_hi <= u.own_lo);
}

// x kinds (template XK): 0 f64 real, 1 f64 complex, 2 f32 real, 3 f32 complex
template <typename Real, int G>
struct TcPoint {  // this lane's prefetched point of the next round: raw loads only, so the
                  // loads stay in flight until the round is staged
  int start, ti;
  unsigned long long xa, xb;  // x bits (f64 re/im, or f32 pair / scalar in xa)
  typename Vec2<Real>::T ph, ag;
  Real w[8 * G];
};

// Every load is unconditional (clamped point index, clamped taper row): lanes past the
// round's points read a real point with ti = -1, which the staging masks to x = 0; rows
// k >= kg are read but never staged.  No lane-divergent branch, no use of loaded values.
template <typename Real, int XK, int G, int NS>
__device__ inline void tc_load(TcPoint<Real, G>& q, int ti, const TcCursor& u, int lane, const SpreadParams<Real>& P) {
  using R2 = typename Vec2<Real>::T;
  if (!u.valid || u.nb == 0) return;  // warp-uniform
  const bool has = lane < u.nb;
  const int j = has ? lane : u.nb - 1;
  const int64_t base = static_cast<int64_t>(u.c) * P.n;
  const int64_t gi = base + u.b0 + j;
  q.ti = has ? ti : -1;
  const int64_t xi = base + (has ? ti : 0);
  q.start = P.start[gi];
  if constexpr (XK == 1) {
    const ulonglong2 xv = reinterpret_cast<const ulonglong2*>(P.x)[xi];
    q.xa = xv.x;
    q.xb = xv.y;
  } else if constexpr (XK == 0 || XK == 3) {
    q.xa = reinterpret_cast<const unsigned long long*>(P.x)[xi];
  } else {
    q.xa = reinterpret_cast<const unsigned int*>(P.x)[xi];
  }
  q.ph = reinterpret_cast<const R2*>(P.prephase)[gi];
  if constexpr (NS > 0) q.ag.x = reinterpret_cast<const Real*>(P.gauss)[gi];  // ES: compact fr table
  else q.ag = P.gauss[gi];
  const Real* tp =
      P.taper_base + (static_cast<int64_t>(u.c) * P.k_total + P.k0) * P.tstride_k + (u.b0 + j) * P.tstride_j;
  // rows k >= kg re-read row kg - 1 (never staged): the pointer stops advancing there
  const int64_t stride = P.tstride_k;
  if constexpr (G == 1) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      q.w[k] = *tp;
      if (k + 1 < P.kg) tp += stride;
    }
  } else {  // independent addresses: the 16 loads issue back to back
#pragma unroll
    for (int k = 0; k < 8 * G; ++k) q.w[k] = tp[min(k, P.kg - 1) * stride];
  }
}

// Unconditional (clamped) load, like the other prefetches: a conditional load with a default
// value put the default's register write behind the round's just-issued prefetch loads (one
// instruction held 19 % of the kernel's stall samples on the long scoreboard)
template <typename Real>
__device__ inline int tc_perm(const TcCursor& u, int lane, const SpreadParams<Real>& P) {
  const int j = lane < u.nb ? lane : 0;
  const int64_t i = u.valid ? static_cast<int64_t>(u.c) * P.n + min(static_cast<int64_t>(u.b0 + j), P.n - 1) : 0;
  return P.perm[i];
}

// ES window polynomials of every even ns (es.cu es_fit), uploaded once per device: with ns a
// template parameter every coefficient is a constant-bank operand of its DFMA.
__constant__ double c_es[kEsTableSize];

// NS = 0: the reference's Gaussian (support P.w2, geometric chains); NS > 0: the ES window on NS
// cells, weight of cell p = Horner(c_es[ns block][p], 2 fr - 1).
// G taper groups of 8 share one staging of the points (K = 9..16 with G = 2: Z rows 8 G,
// accumulators per group; 3 CTAs / SM instead of 5)
template <typename Real, int XK, int NS, int G = 1>
__global__ void __launch_bounds__(kTcWarps * 32, G == 1 ? (sizeof(Real) == 8 ? 4 : kTcCtasPerSm) : 4) spread_tc_kernel(const SpreadParams<Real> P) {
  using R2 = typename Vec2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int RS = kTcRows;
  constexpr int PTS = tc_pts(G);
  constexpr size_t kWarpBytes = (8 * G * RS) * sizeof(double2) + (PTS * RS) * sizeof(double) + RS * sizeof(int);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* scq = reinterpret_cast<double*>(smem_raw);     // C_p
  unsigned char* mine = smem_raw + kMaxW2 * sizeof(double) + warp * kWarpBytes;
  double2* sz = reinterpret_cast<double2*>(mine);        // Z [8 tapers][RS points] (rows >= KG stay 0)
  double* sw = reinterpret_cast<double*>(sz + 8 * G * RS);  // W [PTS points][RS], slot = cell mod 32
  int* srel = reinterpret_cast<int*>(sw + PTS * RS);  // rel [RS points]

  const int w2 = NS > 0 ? NS : P.w2;
  if constexpr (NS == 0)
    for (int i = threadIdx.x; i < P.w2; i += blockDim.x) scq[i] = static_cast<double>(P.cq[i]);
  for (int i = lane; i < static_cast<int>((kWarpBytes - RS * sizeof(int)) / 16); i += 32)
    reinterpret_cast<double2*>(mine)[i] = double2{0.0, 0.0};
  for (int i = lane; i < RS; i += 32) srel[i] = 1 << 20;  // absent points: outside every block
  __syncthreads();
  pdl_launch_dependents();
  pdl_wait();  // x (and the grid's previous reader) before any load or store

  const int stride = static_cast<int>(gridDim.x) * kTcWarps;
  TcPos p0{0, static_cast<int>(blockIdx.x) * kTcWarps + warp};
  tc_step(p0, 0, P);  // normalise (fewer used segments than warps)
  TcPos pp = p0;
  tc_step(pp, stride, P);
  // D2 (fp64, one taper group): loads two rounds ahead (a second prefetched point set, 150
  // registers at 4 CTAs/SM), perm three rounds ahead: C2 fp64 spread 90.6 -> 88.1 us; in fp32 the
  // one-round prefetch at 5 CTAs/SM stays faster (73.3 vs 77.5 us)
  constexpr bool D2 = sizeof(Real) == 8 && G == 1;
  TcCursor cur, n1, n2, n3;
  int4 pre = tc_range(pp, P);
  tc_settle(cur, p0, tc_range(p0, P), P);
  n1 = cur;
  tc_advance(n1, pre, pp, P, stride);
  n2 = n1;
  tc_advance(n2, pre, pp, P, stride);
  if constexpr (D2) {
    n3 = n2;
    tc_advance(n3, pre, pp, P, stride);
  }
  TcPoint<Real, G> pt, pt1;
  pt.ti = -1;
  pt1.ti = -1;
  tc_load<Real, XK, G, NS>(pt, tc_perm(cur, lane, P), cur, lane, P);
  if constexpr (D2) tc_load<Real, XK, G, NS>(pt1, tc_perm(n1, lane, P), n1, lane, P);
  int perm_next = tc_perm(D2 ? n2 : n1, lane, P);

  double cr[G][4][2], ci[G][4][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int b = 0; b < 4; ++b) cr[gg][b][0] = cr[gg][b][1] = ci[gg][b][0] = ci[gg][b][1] = 0.0;

  const int64_t off_h0 = static_cast<int64_t>(2 * t) * P.mr, off_h1 = off_h0 + P.mr;  // tapers 2t, 2t+1
  while (cur.valid) {
    // ---- stage round `cur`: lane = point; z column, rel, and the W row (support only)
    const bool has = lane < cur.nb;
    const bool busy = cur.nb > 0;  // empty segments only write their zeros
    const int rel = has ? static_cast<int>(static_cast<int64_t>(pt.start) - cur.shift) : (1 << 20);
    if (busy) {
      double xr = 0.0, xi = 0.0;
      if constexpr (XK == 1) {
        xr = __longlong_as_double(static_cast<long long>(pt.xa));
        xi = __longlong_as_double(static_cast<long long>(pt.xb));
      } else if constexpr (XK == 3) {
        xr = __uint_as_float(static_cast<unsigned>(pt.xa));
        xi = __uint_as_float(static_cast<unsigned>(pt.xa >> 32));
      } else if constexpr (XK == 0) {
        xr = __longlong_as_double(static_cast<long long>(pt.xa));
      } else {
        xr = __uint_as_float(static_cast<unsigned>(pt.xa));
      }
      if (pt.ti < P.s0 || pt.ti >= P.s1) { xr = 0.0; xi = 0.0; }  // absent lanes: ti = -1
      const double pr = static_cast<double>(pt.ph.x), pi = static_cast<double>(pt.ph.y);
      const double yr = xr * pr - xi * pi, yi = xr * pi + xi * pr;
#pragma unroll
      for (int k = 0; k < 8 * G; ++k) {  // rows k >= kg are never written: they stay zero
        const double wk = static_cast<double>(pt.w[k]);
        if (k < P.kg) sz[k * RS + lane] = double2{wk * yr, wk * yi};
      }
      srel[lane] = rel;
      if constexpr (NS > 0) {
        if (has) {
          const double sv = 2.0 * static_cast<double>(pt.ag.x) - 1.0;
          double* row = sw + lane * RS;
          // the window is even: cell ns-1-p at s is cell p at -s, so each pair of cells is
          // E(s^2) +- s O(s^2) from cell p's even / odd coefficients (half the Horner steps)
          const double s2 = sv * sv;
#pragma unroll
          for (int p = 0; p < NS / 2; ++p) {
            constexpr int D = es_degree(NS);
            const double* cf = c_es + es_table_offset(NS) + p * (D + 1);
            constexpr int de = D & ~1, dod = (D - 1) | 1;  // highest even / odd degree
            double ev = cf[de], od = cf[dod];
#pragma unroll
            for (int d = de - 2; d >= 0; d -= 2) ev = fma(ev, s2, cf[d]);
#pragma unroll
            for (int d = dod - 2; d >= 1; d -= 2) od = fma(od, s2, cf[d]);
            row[(rel + p) & 31] = fma(sv, od, ev);
            row[(rel + NS - 1 - p) & 31] = fma(-sv, od, ev);
          }
        }
      } else if (has) {  // W_p = A g^p C_p stored at slot (rel + p) mod 32 of the point's row;
                  // C_{p+2}/C_p = e^{-4 beta (p - w + 1.5)} is a geometric chain too
        const double gg = static_cast<double>(pt.ag.y), g2 = gg * gg, A = static_cast<double>(pt.ag.x);
        double ae = A * P.c0, ao = A * gg * P.c1, qe = g2 * P.qe0, qo = g2 * P.qo0;
        double* row = sw + lane * RS;
        for (int p = 0; p < P.w2; p += 2) {
          row[(rel + p) & 31] = ae;
          row[(rel + p + 1) & 31] = ao;
          ae *= qe;
          ao *= qo;
          qe *= P.ve;
          qo *= P.ve;
        }
      }
    }
    __syncwarp();
    // ---- prefetch round n1 (its perm is in hand) and the perm of round n2
    if constexpr (D2) {
      pt = pt1;
      tc_load<Real, XK, G, NS>(pt1, perm_next, n2, lane, P);
      perm_next = tc_perm(n3, lane, P);
    } else {
      tc_load<Real, XK, G, NS>(pt, perm_next, n1, lane, P);
      perm_next = tc_perm(n2, lane, P);
    }
    // ---- per block: its point range by ballot (rel ascends over the lanes), then exact
    // 4-point steps on the tensor cores; a = W(cell - rel) masked to the support
    const double* wrow = sw + g;               // + min(p0 + t, 31)*RS (point row) + 8b (slot of cell 8b + g)
    const double2* zcol = sz + g * RS + t;     // + p0
    const int* rcol = srel + t;
#pragma unroll
    for (int b = 0; b < 4 && busy; ++b) {
      const int lo = __popc(__ballot_sync(0xffffffffu, rel < 8 * b - (w2 - 1)));
      const int hi = __popc(__ballot_sync(0xffffffffu, rel < 8 * b + 8));
      for (int p0 = lo; p0 < hi; p0 += 4) {  // rows up to hi + 3 <= 34: absent ones are masked
        const int pp = 8 * b + g - rcol[p0];
        const double wv = wrow[(PTS > 32 ? p0 + t : min(p0 + t, PTS - 1)) * RS + 8 * b];
        const double a = static_cast<unsigned>(pp) < static_cast<unsigned>(w2) ? wv : 0.0;
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {  // taper group gg: Z rows 8 gg .. 8 gg + 7
          const double2 zb = zcol[gg * 8 * RS + p0];
          dmma_8x8x4(cr[gg][b][0], cr[gg][b][1], a, zb.x);
          dmma_8x8x4(ci[gg][b][0], ci[gg][b][1], a, zb.y);
        }
      }
    }
    if (cur.last) {
      R2* out = P.grid + (static_cast<int64_t>(cur.c) * P.kpad + P.k0) * P.mr;
      const int cell0 = static_cast<int>(cur.seg) * 32 + g;
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        R2* out0 = out + off_h0 + static_cast<int64_t>(8 * gg) * P.mr;
        R2* out1 = out + off_h1 + static_cast<int64_t>(8 * gg) * P.mr;
        const bool k0ok = 8 * gg + 2 * t < P.kg, k1ok = 8 * gg + 2 * t + 1 < P.kg;
        if (P.slots) {  // taper k -> owner k / per, its slot row k % per (possibly a peer GPU);
                        // padding lanes (k >= kg, never stored) read the table at k0 only
          const int64_t ka = P.k0 + (k0ok ? 8 * gg + 2 * t : 0), kb = P.k0 + (k1ok ? 8 * gg + 2 * t + 1 : 0);
          out0 = P.slots[ka / P.per] + (ka % P.per) * P.mr;
          out1 = P.slots[kb / P.per] + (kb % P.per) * P.mr;
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int addr = cell_addr32(cell0 + 8 * b, P.blocked, P.lgC, P.lgCW, P.lgT);
          if (k0ok) out0[addr] = R2{static_cast<Real>(cr[gg][b][0]), static_cast<Real>(ci[gg][b][0])};
          if (k1ok) out1[addr] = R2{static_cast<Real>(cr[gg][b][1]), static_cast<Real>(ci[gg][b][1])};
          cr[gg][b][0] = cr[gg][b][1] = ci[gg][b][0] = ci[gg][b][1] = 0.0;
        }
      }
    }
    __syncwarp();  // private tables are restaged next
    cur = n1;
    n1 = n2;
    if constexpr (D2) {
      n2 = n3;
      tc_advance(n3, pre, pp, P, stride);
    } else {
      tc_advance(n2, pre, pp, P, stride);
    }
  }
  if (P.slots) __threadfence_system();  // peer-slot stores ordered before the caller's barrier
}


// ---- streaming FP64 tensor-core spread (default) -----------------------------------------
// The same banded product on DMMA as spread_tc_kernel, but every warp STREAMS one contiguous
// cell range (a work unit: equal numbers of points per warp, cut at plan time from the segment
// point counts) instead of restaging the points of each 32-cell segment: batches of 32
// consecutive sorted points are staged once (lane = point) and accumulated into a sliding
// window of 64 cells (8 DMMA blocks of 8 cells x 8 tapers, accumulators in registers).  A point
// is processed once its support [rel, rel + w2) lies inside the window; when the next point's
// support does not, the lower 32 cells are complete (points arrive in start order), are stored,
// and the window slides by 32 cells (upper half -> lower half, a register move).  At C2's
// density (one point per cell, 10-cell support) this stages each point once instead of ~1.3
// times and halves the staging rounds of the per-segment kernel (one partial batch per unit
// instead of one per segment).  Cells without points are written as zeros by the slides.
constexpr int kStWarps = 3;

struct StUnit {  // one work unit: its cells and its point stream
  int c, cell0, ncell;             // channel, first cell, cells
  int wrap_lo, len0, own_lo, len;  // stream = wrapping points [wrap_lo, n) then own [own_lo, own_hi)
};

template <typename Real>
__device__ inline StUnit st_unit(int unit, const SpreadParams<Real>& P) {
  const int4 a = reinterpret_cast<const int4*>(P.units)[2 * unit];
  const int4 b = reinterpret_cast<const int4*>(P.units)[2 * unit + 1];
  StUnit u;
  u.c = a.x;
  u.cell0 = a.y * 32;
  u.ncell = a.z * 32;
  u.own_lo = a.w;
  u.wrap_lo = b.y;
  u.len0 = static_cast<int>(P.n) - b.y;
  u.len = u.len0 + (b.x - a.w);
  return u;
}

// stream position q of unit u -> sorted point index (channel-relative)
__device__ inline int st_point(const StUnit& u, int q) { return q < u.len0 ? u.wrap_lo + q : u.own_lo + (q - u.len0); }

template <typename Real, int KG>
struct StPoint {  // this lane's prefetched point: raw loads only
  int start, ti, q;
  unsigned long long xa, xb;
  typename Vec2<Real>::T ph;
  Real fr;  // ES: fr; Gaussian: A (with g in fg)
  Real fg;
  Real w[KG];
};

// Loads of batch [b0, b0 + nb) of unit u (nb >= 1): every load unconditional (clamped index), so
// no merge waits on HBM; lanes past the batch get ti = -1 (x masked to 0 at staging).  `base` is the
// channel's first point (u.c * n) and `tp0` its first taper row at point 0, both fixed per unit.
template <typename Real, int XK, int KG, int NS>
__device__ inline void st_load(StPoint<Real, KG>& q, int ti, const StUnit& u, int64_t base, const Real* tp0, int b0,
                               int nb, int lane, const SpreadParams<Real>& P) {
  using R2 = typename Vec2<Real>::T;
  const bool has = lane < nb;
  const int qq = b0 + (has ? lane : nb - 1);
  const int pi = st_point(u, qq);
  const int64_t gi = base + pi;
  q.q = qq;
  q.ti = has ? ti : -1;
  const int64_t xi = base + (has ? ti : 0);
  if constexpr (XK == 1) {
    const ulonglong2 xv = reinterpret_cast<const ulonglong2*>(P.x)[xi];
    q.xa = xv.x;
    q.xb = xv.y;
  } else if constexpr (XK == 0 || XK == 3) {
    q.xa = reinterpret_cast<const unsigned long long*>(P.x)[xi];
  } else {
    q.xa = reinterpret_cast<const unsigned int*>(P.x)[xi];
  }
  q.start = P.start[gi];
  q.ph = reinterpret_cast<const R2*>(P.prephase)[gi];
  if constexpr (NS > 0) {
    q.fr = reinterpret_cast<const Real*>(P.gauss)[gi];
  } else {
    const R2 ag = P.gauss[gi];
    q.fr = ag.x;
    q.fg = ag.y;
  }
  // rows k >= kg re-read row kg - 1 (never staged): the pointer stops advancing there
  const Real* tp = tp0 + static_cast<int64_t>(pi) * P.tstride_j;
#pragma unroll
  for (int k = 0; k < KG; ++k) {
    q.w[k] = *tp;
    tp += (k + 1 < P.kg) ? P.tstride_k : 0;
  }
}

// perm index of this lane's point of batch b0 (clamped into the stream)
template <typename Real>
__device__ inline int st_perm(const StUnit& u, int b0, int lane, const SpreadParams<Real>& P) {
  const int q = min(b0 + lane, max(u.len - 1, 0));
  return P.perm[static_cast<int64_t>(u.c) * P.n + (u.len > 0 ? st_point(u, q) : 0)];
}

// Where a lane's two tapers (2t, 2t + 1 of the launch's group) of channel c go: fixed per unit.
template <typename Real>
struct StOut {
  typename Vec2<Real>::T *p0, *p1;
  bool ok0, ok1;
};
template <typename Real>
__device__ inline StOut<Real> st_out(int c, int t, const SpreadParams<Real>& P) {
  using R2 = typename Vec2<Real>::T;
  StOut<Real> o;
  o.ok0 = 2 * t < P.kg;
  o.ok1 = 2 * t + 1 < P.kg;
  if (P.slots) {  // taper k -> owner k / per, its slot row k % per (possibly a peer GPU)
    const int64_t ka = P.k0 + (o.ok0 ? 2 * t : 0), kb = P.k0 + (o.ok1 ? 2 * t + 1 : 0);
    o.p0 = P.slots[ka / P.per] + (ka % P.per) * P.mr;
    o.p1 = P.slots[kb / P.per] + (kb % P.per) * P.mr;
  } else {
    R2* out = P.grid + (static_cast<int64_t>(c) * P.kpad + P.k0) * P.mr;
    o.p0 = out + static_cast<int64_t>(2 * t) * P.mr;
    o.p1 = o.p0 + P.mr;
  }
  return o;
}

// Store window blocks PH .. PH + 3 of the accumulator ring (cells `cell` .. + 31, cell a multiple
// of 32) and clear them for reuse as the window's upper half.  In the blocked layout the 32 cells
// share their row j1, so block b sits at a fixed offset from block 0: d1 for b = 1, d2 for b = 2,
// d1 + d2 for b = 3 (8 b cells on: ((8b) >> lgCW) tiles + (8b) mod CW; natural layout: 8 b).
template <int PH, typename Real>
__device__ __forceinline__ void st_flush(double (&cr)[8][2], double (&ci)[8][2], const StOut<Real>& o, int cell,
                                         int g, int d1, int d2, const SpreadParams<Real>& P) {
  using R2 = typename Vec2<Real>::T;
  const int a0 = cell_addr32(cell + g, P.blocked, P.lgC, P.lgCW, P.lgT);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int addr = a0 + ((b & 1) ? d1 : 0) + ((b & 2) ? d2 : 0);
    if (o.ok0) o.p0[addr] = R2{static_cast<Real>(cr[PH + b][0]), static_cast<Real>(ci[PH + b][0])};
    if (o.ok1) o.p1[addr] = R2{static_cast<Real>(cr[PH + b][1]), static_cast<Real>(ci[PH + b][1])};
    cr[PH + b][0] = cr[PH + b][1] = ci[PH + b][0] = ci[PH + b][1] = 0.0;
  }
}

// One accumulation pass over the staged points [pst, pend) for the 8 window blocks.  The window is
// a RING over the accumulator registers: register block r holds window block (r + 4 ph) & 7, ph the
// ring phase, so a slide is a store + clear of the old lower half and a phase flip, never a register
// move -- and because a W row's slot of cell 8 b + g is 8 (r & 3) + g in either phase, both phases
// run the same code (only the blocks' point ranges are picked by ph).  Per block its point range
// [lo, hi) comes from byte-packed counts summed over the warp (rel ascends over the lanes:
// lo = #points whose support ends below the block, hi = #points that start at or below its last
// cell; one 32-bit warp sum yields four blocks' counts), then exact 4-point steps on the tensor
// cores.  ES (NS > 0): the W rows are zero off the point's support and an ns <= 16 support cannot
// alias a block cell mod 32 for a point of [lo, hi), so a = W[point][cell mod 32] as stored, masked
// only past hi; the Gaussian (NS = 0, up to 32 cells, rows not cleared) also masks cells outside
// the point's support.
template <int NS, int RS>
__device__ __forceinline__ void st_pass(double (&cr)[8][2], double (&ci)[8][2], int rel, int wb, int ph, int w2,
                                        int pst, int pend, const double* sw, const double2* sz, const int* srel,
                                        int g, int t) {
  const double* wrow = sw + g;            // + point row * RS + slot base
  const double2* zcol = sz + g * RS + t;  // + p0
  const int* rcol = srel + t;
  // first block at or past this lane's point start / first block past its support, clamped to 0..8
  const int d = rel - wb;
  const int sf = min(max(d >> 3, 0), 8);
  const int sl = min(max(((d + w2 - 1) >> 3) + 1, 0), 8);
  const unsigned long long ones = 0x0101010101010101ull;
  const unsigned long long vf = sf < 8 ? ones << (8 * sf) : 0ull, vl = sl < 8 ? ones << (8 * sl) : 0ull;
  const unsigned hi03 = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(vf));
  const unsigned hi47 = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(vf >> 32));
  const unsigned lo03 = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(vl));
  const unsigned lo47 = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(vl >> 32));
  // counts of register blocks 0..3 (A) and 4..7 (B): window blocks 0..3 / 4..7, swapped in phase 1
  const unsigned hiA = ph ? hi47 : hi03, hiB = ph ? hi03 : hi47;
  const unsigned loA = ph ? lo47 : lo03, loB = ph ? lo03 : lo47;
  const int wbA = wb + (ph ? 32 : 0), wbB = wb + (ph ? 0 : 32);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int cb = (r < 4 ? wbA : wbB) + 8 * (r & 3);  // block's first cell
    const int lo = max(pst, static_cast<int>(((r < 4 ? loA : loB) >> (8 * (r & 3))) & 0xffu));
    const int hi = min(pend, static_cast<int>(((r < 4 ? hiA : hiB) >> (8 * (r & 3))) & 0xffu));
    for (int p0 = lo; p0 < hi; p0 += 4) {
      const int pi = p0 + t;  // rows up to hi + 3 <= 34 < 35: the overrun rows are zero
      double a = wrow[pi * RS + 8 * (r & 3)];
      bool keep = pi < hi;
      if constexpr (NS == 0) keep = keep && static_cast<unsigned>(cb + g - rcol[p0]) < static_cast<unsigned>(w2);
      a = keep ? a : 0.0;
      const double2 zb = zcol[p0];
      dmma_8x8x4(cr[r][0], cr[r][1], a, zb.x);
      dmma_8x8x4(ci[r][0], ci[r][1], a, zb.y);
    }
  }
}

// KG: taper rows loaded per point (8: up to 8 tapers, P.kg of them real; 1: one taper / untapered)
template <typename Real, int XK, int NS, int KG>
#ifndef NUS_ST_CTAS
#define NUS_ST_CTAS 4
#endif
__global__ void __launch_bounds__(kStWarps * 32, NUS_ST_CTAS) spread_stream_kernel(const SpreadParams<Real> P) {
  using R2 = typename Vec2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int RS = kTcRows;
  constexpr int PTS = 35;  // 32 staged points + the last 4-point step's overrun rows (zero)
  constexpr int RELS = (PTS + 3) & ~3;  // rel entries, rounded so every warp's tables stay 16-byte aligned
  constexpr size_t kWarpBytes = (8 * RS) * sizeof(double2) + (PTS * RS) * sizeof(double) + RELS * sizeof(int);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  unsigned char* mine = smem_raw + warp * kWarpBytes;
  double2* sz = reinterpret_cast<double2*>(mine);        // Z [8 tapers][RS points] (rows >= kg and columns >= 32 stay 0)
  double* sw = reinterpret_cast<double*>(sz + 8 * RS);   // W [PTS points][RS], slot = cell mod 32 (ES: 0 off support)
  int* srel = reinterpret_cast<int*>(sw + PTS * RS);     // rel [PTS points]
  for (int i = lane; i < static_cast<int>((kWarpBytes - RELS * sizeof(int)) / 16); i += 32)
    reinterpret_cast<double2*>(mine)[i] = double2{0.0, 0.0};
  for (int i = lane; i < RELS; i += 32) srel[i] = 1 << 20;  // absent points: outside every block
  __syncwarp();
  pdl_launch_dependents();
  pdl_wait();

  const int w2 = NS > 0 ? NS : P.w2;
  double cr[8][2], ci[8][2];
#pragma unroll
  for (int b = 0; b < 8; ++b) cr[b][0] = cr[b][1] = ci[b][0] = ci[b][1] = 0.0;
  StPoint<Real, KG> pt;
  const int gw = static_cast<int>(blockIdx.x) * kStWarps + warp;
  const int unit_end = P.warp_first[gw + 1];
  int erase_rel = 1 << 20;  // ES: support of this lane's previous point, cleared before restaging
  int ph = 0;               // ring phase of the accumulator window (st_pass)
  // offsets of window blocks 1 and 2 from block 0 in the grid layout (st_flush)
  const int d1 = P.blocked ? ((8 >> P.lgCW) << P.lgT) + (8 & ((1 << P.lgCW) - 1)) : 8;
  const int d2 = P.blocked ? ((16 >> P.lgCW) << P.lgT) + (16 & ((1 << P.lgCW) - 1)) : 16;
  for (int unit = P.warp_first[gw]; unit < unit_end; ++unit) {
    const StUnit u = st_unit(unit, P);
    const StOut<Real> out = st_out<Real>(u.c, t, P);
    const int64_t base = static_cast<int64_t>(u.c) * P.n;
    const Real* tp0 = P.taper_base + (static_cast<int64_t>(u.c) * P.k_total + P.k0) * P.tstride_k;
    int wb = 0;  // window base, cells relative to the unit's first cell
    if (u.len > 0) st_load<Real, XK, KG, NS>(pt, st_perm(u, 0, lane, P), u, base, tp0, 0, min(32, u.len), lane, P);
    int perm_next = st_perm(u, 32, lane, P);
    for (int b0 = 0; b0 < u.len; b0 += 32) {
      // ---- stage batch [b0, b0 + nb): lane = point; z column, rel, and the W row (support only)
      const int nb = min(32, u.len - b0);
      const bool has = lane < nb;
      const int rel = has ? pt.start - u.cell0 - (pt.q < u.len0 ? static_cast<int>(P.mr) : 0) : (1 << 20);
      {
        double xr = 0.0, xi = 0.0;
        if constexpr (XK == 1) {
          xr = __longlong_as_double(static_cast<long long>(pt.xa));
          xi = __longlong_as_double(static_cast<long long>(pt.xb));
        } else if constexpr (XK == 3) {
          xr = __uint_as_float(static_cast<unsigned>(pt.xa));
          xi = __uint_as_float(static_cast<unsigned>(pt.xa >> 32));
        } else if constexpr (XK == 0) {
          xr = __longlong_as_double(static_cast<long long>(pt.xa));
        } else {
          xr = __uint_as_float(static_cast<unsigned>(pt.xa));
        }
        if (pt.ti < P.s0 || pt.ti >= P.s1) { xr = 0.0; xi = 0.0; }  // absent lanes: ti = -1
        const double pr = static_cast<double>(pt.ph.x), pim = static_cast<double>(pt.ph.y);
        const double yr = xr * pr - xi * pim, yi = xr * pim + xi * pr;
#pragma unroll
        for (int k = 0; k < KG; ++k) {  // rows k >= kg are never written: they stay zero
          const double wk = static_cast<double>(pt.w[k]);
          if (KG == 1 || k < P.kg) sz[k * RS + lane] = double2{wk * yr, wk * yi};
        }
        srel[lane] = rel;
        double* row = sw + lane * RS;
        if constexpr (NS > 0) {
          // clear the previous point's support (the rows are zero off the support), then write this one's
#pragma unroll
          for (int q = 0; q < NS; ++q) row[(erase_rel + q) & 31] = 0.0;
          erase_rel = rel;
          if (has) {
            const double sv = 2.0 * static_cast<double>(pt.fr) - 1.0;
            const double s2 = sv * sv;
#pragma unroll
            for (int q = 0; q < NS / 2; ++q) {  // even window: cells q and ns-1-q from one E/O pair
              constexpr int D = es_degree(NS);
              const double* cf = c_es + es_table_offset(NS) + q * (D + 1);
              constexpr int de = D & ~1, dod = (D - 1) | 1;
              double ev = cf[de], od = cf[dod];
#pragma unroll
              for (int d = de - 2; d >= 0; d -= 2) ev = fma(ev, s2, cf[d]);
#pragma unroll
              for (int d = dod - 2; d >= 1; d -= 2) od = fma(od, s2, cf[d]);
              row[(rel + q) & 31] = fma(sv, od, ev);
              row[(rel + NS - 1 - q) & 31] = fma(-sv, od, ev);
            }
          } else {
            erase_rel = 0;  // nothing written: clearing slots 0 .. ns-1 next time is harmless
          }
        } else if (has) {  // W_p = A g^p C_p, two geometric chains (spread_tc_kernel)
          const double gg = static_cast<double>(pt.fg), g2 = gg * gg, A = static_cast<double>(pt.fr);
          double ae = A * P.c0, ao = A * gg * P.c1, qe = g2 * P.qe0, qo = g2 * P.qo0;
          for (int q = 0; q < P.w2; q += 2) {
            row[(rel + q) & 31] = ae;
            row[(rel + q + 1) & 31] = ao;
            ae *= qe;
            ao *= qo;
            qe *= P.ve;
            qo *= P.ve;
          }
        }
      }
      __syncwarp();
      // ---- prefetch the next batch (its perm is in hand) and the perm of the one after
      if (b0 + 32 < u.len) {
        st_load<Real, XK, KG, NS>(pt, perm_next, u, base, tp0, b0 + 32, min(32, u.len - b0 - 32), lane, P);
        perm_next = st_perm(u, b0 + 64, lane, P);
      }
      // ---- accumulate the prefix of the batch whose supports fit the window; when the next point's
      // support leaves it, the lower 32 cells are complete (points arrive in start order): store
      // them, slide the window by 32 cells, repeat
      int pst = 0;
      for (;;) {
        const int pend = __popc(__ballot_sync(0xffffffffu, has && rel + (w2 - 1) < wb + 64));
        if (pend > pst) {
          st_pass<NS, RS>(cr, ci, rel, wb, ph, w2, pst, pend, sw, sz, srel, g, t);
          pst = pend;
        }
        if (pst >= nb) break;
        // the lower 32 cells are complete: store and clear them (they become the upper half)
        if (ph == 0) st_flush<0, Real>(cr, ci, out, u.cell0 + wb, g, d1, d2, P);
        else st_flush<4, Real>(cr, ci, out, u.cell0 + wb, g, d1, d2, P);
        ph ^= 1;
        wb += 32;
      }
      __syncwarp();  // private tables are restaged next
    }
    // end of the unit: store the rest of its cells (zeros past the last point)
    while (wb < u.ncell) {
      if (ph == 0) st_flush<0, Real>(cr, ci, out, u.cell0 + wb, g, d1, d2, P);
      else st_flush<4, Real>(cr, ci, out, u.cell0 + wb, g, d1, d2, P);
      ph ^= 1;
      wb += 32;
    }
    // what is left holds contributions past the unit's last cell: discard them
#pragma unroll
    for (int b = 0; b < 8; ++b) cr[b][0] = cr[b][1] = ci[b][0] = ci[b][1] = 0.0;
    ph = 0;
  }
  if (P.slots) __threadfence_system();  // peer-slot stores ordered before the caller's barrier
}

void es_upload() {  // once per device
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  NUS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && done[dev]) return;
  std::vector<double> tab(kEsTableSize);
  for (int ns = kEsMinNs; ns <= kEsMaxNs; ns += 2) es_fit(ns, tab.data() + es_table_offset(ns));
  NUS_CUDA(cudaMemcpyToSymbol(c_es, tab.data(), tab.size() * sizeof(double)));
  if (dev < 64) done[dev] = true;
}

template <typename Real, int XK, int NS, int G = 1>
void launch_tc(const SpreadParams<Real>& P, cudaStream_t s) {
  const size_t warp_bytes =
      (8 * G * kTcRows) * sizeof(double2) + (tc_pts(G) * kTcRows) * sizeof(double) + kTcRows * sizeof(int);
  const size_t smem = kMaxW2 * sizeof(double) + kTcWarps * warp_bytes;
  // kernel attributes are per device: configured once for every device the process uses
  static std::mutex mu;
  static int bps[64] = {}, sm_of[64] = {};
  int dev = 0;
  NUS_CUDA(cudaGetDevice(&dev));
  require(dev < 64, "spread: device ordinal out of range");
  int blocks_per_sm = 0, sms = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (bps[dev] == 0) {
      NUS_CUDA(cudaFuncSetAttribute(spread_tc_kernel<Real, XK, NS, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
      NUS_CUDA(cudaDeviceGetAttribute(&sm_of[dev], cudaDevAttrMultiProcessorCount, dev));
      NUS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[dev], spread_tc_kernel<Real, XK, NS, G>,
                                                             kTcWarps * 32, smem));
      require(bps[dev] > 0, "spread: tensor-core kernel does not fit on an SM");
    }
    blocks_per_sm = bps[dev];
    sms = sm_of[dev];
  }
  const int64_t warps = P.nseg_used * P.channels;
  const int64_t grid = std::min<int64_t>((warps + kTcWarps - 1) / kTcWarps, static_cast<int64_t>(blocks_per_sm) * sms);
  if constexpr (NS > 0) es_upload();
  launch_pdl(spread_tc_kernel<Real, XK, NS, G>, dim3(static_cast<unsigned>(grid)), dim3(kTcWarps * 32), smem, s, P);
  note_launch();
  check_launch("spread_tc_kernel");
}

__device__ double g_one_f64 = 1.0;
__device__ float g_one_f32 = 1.0f;

template <typename Real, int XK, int G = 1>
void launch_tc_ns(const SpreadParams<Real>& P, int ns, cudaStream_t s) {
  switch (ns) {
    case 0: launch_tc<Real, XK, 0, G>(P, s); break;
    case 4: launch_tc<Real, XK, 4, G>(P, s); break;
    case 6: launch_tc<Real, XK, 6, G>(P, s); break;
    case 8: launch_tc<Real, XK, 8, G>(P, s); break;
    case 10: launch_tc<Real, XK, 10, G>(P, s); break;
    case 12: launch_tc<Real, XK, 12, G>(P, s); break;
    case 14: launch_tc<Real, XK, 14, G>(P, s); break;
    case 16: launch_tc<Real, XK, 16, G>(P, s); break;
    default: fail(NUS_ERR_INVALID_ARGUMENT, "spread: unsupported ES width");
  }
}

template <typename Real>
void set_taper_base(SpreadParams<Real>& P) {
  if (P.tapers) {
    P.taper_base = P.tapers;
    P.tstride_k = P.n;
    P.tstride_j = 1;
  } else {  // untapered: every weight reads one device constant 1
    void* one = nullptr;
    if constexpr (sizeof(Real) == 8) NUS_CUDA(cudaGetSymbolAddress(&one, g_one_f64));
    else NUS_CUDA(cudaGetSymbolAddress(&one, g_one_f32));
    P.taper_base = static_cast<const Real*>(one);
    P.tstride_k = 0;
    P.tstride_j = 0;
  }
}

template <typename Real>
void launch_tc_x(SpreadParams<Real> P, int ns, cudaStream_t s, bool two_groups = false) {
  set_taper_base(P);
  const int xk = P.x_dtype == 0 ? (P.x_complex ? 1 : 0) : (P.x_complex ? 3 : 2);
  if (two_groups) {  // real x only (the estimator's spectra)
    require(xk == 0 || xk == 2, "spread: two taper groups need real x");
    if (xk == 0) launch_tc_ns<Real, 0, 2>(P, ns, s);
    else launch_tc_ns<Real, 2, 2>(P, ns, s);
    return;
  }
  switch (xk) {
    case 0: launch_tc_ns<Real, 0>(P, ns, s); break;
    case 1: launch_tc_ns<Real, 1>(P, ns, s); break;
    case 2: launch_tc_ns<Real, 2>(P, ns, s); break;
    default: launch_tc_ns<Real, 3>(P, ns, s); break;
  }
}


// Work units of the streaming spread: the occupied segments of all channels (each channel's in
// the pass-A row order) weighted by the points whose start cell they hold plus a charge for their
// cells, cut into one contiguous range of equal weight per resident warp.  A warp's range is
// split into units where it crosses a channel boundary or the cyclic wrap of the occupied rows
// past cell Mr - 1, so each unit's cells are consecutive; warp w runs units
// [first[w], first[w + 1]).
const SpreadTables::Units& stream_units(const Plan& plan, int64_t nwarps, int64_t nseg_used, int lg_spr, int row_lo,
                                        int nrows) {
  const SpreadTables& tb = plan.tab;
  std::lock_guard<std::mutex> lk(tb.units_mu);
  const int row_cnt = static_cast<int>(nseg_used >> lg_spr);
  const int64_t C = plan.p.channels, nseg = tb.nseg;
  // nparts = nwarps * ilv equal-weight parts; part j runs on warp j mod nwarps, so with ilv > 1 the
  // parts in flight at any time are neighbours in memory.  Measured (K = 7, fp64): C2 (2^20 points,
  // point tables ~100 MB, largely L2-resident across spectra) is fastest with one part per warp
  // (87.4 us; 2 parts 90.1, 4 parts 94.9); C5 (2^22 points, ~370 MB of tables streamed from HBM)
  // with ~300 points per part (1/2/4/8/16/32 parts per warp: 471/431/381/329/339/394 us; the
  // per-segment kernel 386 us): the DRAM pages of the neighbouring parts are then open together.
  // NUS_SPREAD_ILV overrides.
  const int64_t total_points = C * plan.p.n;
  const int64_t ilv = [&] {
    const char* e = std::getenv("NUS_SPREAD_ILV");
    if (e) return std::max<int64_t>(1, std::atoll(e));
    if (total_points <= (int64_t{1} << 21)) return int64_t{1};
    return std::min<int64_t>(32, std::max<int64_t>(1, (total_points / nwarps + 150) / 300));
  }();
  for (const auto& u : tb.units)
    if (u.nwarps == nwarps && u.ilv == ilv && u.row_lo == row_lo && u.row_cnt == row_cnt) return u;
  const int32_t* hs = tb.h_seg_range.data();
  require(static_cast<int64_t>(tb.h_seg_range.size()) == C * nseg * 4, "spread: segment ranges missing");
  constexpr int64_t kSegCharge = 2;  // ~ the cost of two points: one slide + store of 32 cells
  auto abs_seg = [&](int64_t u) {
    const int64_t row = ((u >> lg_spr) + row_lo) & (nrows - 1);
    return (row << lg_spr) | (u & ((int64_t{1} << lg_spr) - 1));
  };
  // cumulative weight over (channel, used segment)
  const int64_t total_segs = C * nseg_used;
  std::vector<int64_t> cum(static_cast<size_t>(total_segs) + 1, 0);
  for (int64_t c = 0; c < C; ++c) {
    const int32_t* h = hs + c * nseg * 4;
    for (int64_t u = 0; u < nseg_used; ++u) {
      const int64_t a = abs_seg(u);
      const int64_t own = h[4 * a + 1] - (a > 0 ? h[4 * (a - 1) + 1] : 0);
      const int64_t gidx = c * nseg_used + u;
      cum[gidx + 1] = cum[gidx] + own + kSegCharge;
    }
  }
  const int64_t total = cum[total_segs];
  const int64_t nparts = nwarps * ilv;
  std::vector<std::vector<int32_t>> parts(static_cast<size_t>(nparts));
  int64_t g0 = 0;
  for (int64_t w = 0; w < nparts; ++w) {
    std::vector<int32_t>& units = parts[w];
    int64_t g1 = total_segs;
    if (w + 1 < nparts) {
      const int64_t target = static_cast<int64_t>((static_cast<__int128>(total) * (w + 1)) / nparts);
      g1 = std::lower_bound(cum.begin() + g0, cum.end(), target) - cum.begin();
      g1 = std::min(std::max(g1, g0), total_segs);
    }
    // pieces of [g0, g1): cut at channel boundaries and at the cyclic wrap (absolute segment 0)
    for (int64_t lo = g0; lo < g1;) {
      const int64_t c = lo / nseg_used;
      int64_t hi = std::min(g1, (c + 1) * nseg_used);
      for (int64_t q = lo + 1; q < hi; ++q)
        if (abs_seg(q - c * nseg_used) == 0) { hi = q; break; }
      const int32_t* h = hs + c * nseg * 4;
      const int64_t a0 = abs_seg(lo - c * nseg_used), na = hi - lo;
      units.insert(units.end(), {static_cast<int32_t>(c), static_cast<int32_t>(a0), static_cast<int32_t>(na),
                                 h[4 * a0], h[4 * (a0 + na - 1) + 1], h[4 * a0 + 2], 0, 0});
      lo = hi;
    }
    g0 = g1;
  }
  std::vector<int32_t> units, first(static_cast<size_t>(nwarps) + 1, 0);
  for (int64_t w = 0; w < nwarps; ++w) {
    first[w] = static_cast<int32_t>(units.size() / 8);
    for (int64_t j = 0; j < ilv; ++j) {
      const std::vector<int32_t>& pu = parts[j * nwarps + w];
      units.insert(units.end(), pu.begin(), pu.end());
    }
  }
  first[nwarps] = static_cast<int32_t>(units.size() / 8);
  SpreadTables::Units nu;
  nu.nwarps = nwarps;
  nu.ilv = ilv;
  nu.row_lo = row_lo;
  nu.row_cnt = row_cnt;
  nu.count = static_cast<int64_t>(units.size() / 8);
  std::vector<int32_t> all(units);
  all.insert(all.end(), first.begin(), first.end());
  nu.buf.alloc(all.size() * sizeof(int32_t));
  NUS_CUDA(cudaMemcpy(nu.buf.ptr, all.data(), all.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  tb.units.push_back(std::move(nu));
  return tb.units.back();
}

template <typename Real, int XK, int NS, int KG>
void launch_stream(SpreadParams<Real> P, const Plan& plan, cudaStream_t s) {
  const size_t smem = kStWarps * ((8 * kTcRows) * sizeof(double2) + (35 * kTcRows) * sizeof(double) +
                                  36 * sizeof(int));  // = kStWarps * kWarpBytes of the kernel
  static std::mutex mu;
  static int bps[64] = {}, sm_of[64] = {};
  int dev = 0;
  NUS_CUDA(cudaGetDevice(&dev));
  require(dev < 64, "spread: device ordinal out of range");
  int blocks_per_sm = 0, sms = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (bps[dev] == 0) {
      NUS_CUDA(cudaFuncSetAttribute(spread_stream_kernel<Real, XK, NS, KG>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      NUS_CUDA(cudaDeviceGetAttribute(&sm_of[dev], cudaDevAttrMultiProcessorCount, dev));
      NUS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps[dev], spread_stream_kernel<Real, XK, NS, KG>,
                                                             kStWarps * 32, smem));
      require(bps[dev] > 0, "spread: streaming kernel does not fit on an SM");
    }
    blocks_per_sm = bps[dev];
    sms = sm_of[dev];
  }
  const int64_t grid = static_cast<int64_t>(blocks_per_sm) * sms;
  const auto& units = stream_units(plan, grid * kStWarps, P.nseg_used, P.lg_spr, P.row_lo, P.nrows);
  P.units = static_cast<const int32_t*>(units.buf.ptr);
  P.nunits = static_cast<int>(units.count);
  P.warp_first = P.units + 8 * units.count;
  if constexpr (NS > 0) es_upload();
  launch_pdl(spread_stream_kernel<Real, XK, NS, KG>, dim3(static_cast<unsigned>(grid)), dim3(kStWarps * 32), smem, s,
             P);
  note_launch();
  check_launch("spread_stream_kernel");
}

template <typename Real, int XK, int KG>
void launch_stream_ns(const SpreadParams<Real>& P, const Plan& plan, int ns, cudaStream_t s) {
  switch (ns) {
    case 0: launch_stream<Real, XK, 0, KG>(P, plan, s); break;
    case 4: launch_stream<Real, XK, 4, KG>(P, plan, s); break;
    case 6: launch_stream<Real, XK, 6, KG>(P, plan, s); break;
    case 8: launch_stream<Real, XK, 8, KG>(P, plan, s); break;
    case 10: launch_stream<Real, XK, 10, KG>(P, plan, s); break;
    case 12: launch_stream<Real, XK, 12, KG>(P, plan, s); break;
    case 14: launch_stream<Real, XK, 14, KG>(P, plan, s); break;
    case 16: launch_stream<Real, XK, 16, KG>(P, plan, s); break;
    default: fail(NUS_ERR_INVALID_ARGUMENT, "spread: unsupported ES width");
  }
}

// one taper group (kg <= 8) on the streaming kernel
template <typename Real>
void launch_stream_x(SpreadParams<Real> P, const Plan& plan, int ns, cudaStream_t s) {
  set_taper_base(P);
  const int xk = P.x_dtype == 0 ? (P.x_complex ? 1 : 0) : (P.x_complex ? 3 : 2);
  if (P.kg == 1) {
    switch (xk) {
      case 0: launch_stream_ns<Real, 0, 1>(P, plan, ns, s); break;
      case 1: launch_stream_ns<Real, 1, 1>(P, plan, ns, s); break;
      case 2: launch_stream_ns<Real, 2, 1>(P, plan, ns, s); break;
      default: launch_stream_ns<Real, 3, 1>(P, plan, ns, s); break;
    }
    return;
  }
  switch (xk) {  // complex x with tapers: the O(N log N) normalisation's lattice chunks (normalise.cu)
    case 0: launch_stream_ns<Real, 0, 8>(P, plan, ns, s); break;
    case 1: launch_stream_ns<Real, 1, 8>(P, plan, ns, s); break;
    case 2: launch_stream_ns<Real, 2, 8>(P, plan, ns, s); break;
    default: launch_stream_ns<Real, 3, 8>(P, plan, ns, s); break;
  }
}

template <typename Real, int KG>
void launch_group(const SpreadParams<Real>& P, int64_t channels, cudaStream_t s) {
  const size_t smem = kBatch * KG * sizeof(typename Vec2<Real>::T) +
                      kBatch * static_cast<size_t>(P.w2 + 1) * sizeof(Real) + kBatch * sizeof(int);
  static std::mutex mu;
  static bool configured[64] = {};
  int dev = 0;
  NUS_CUDA(cudaGetDevice(&dev));
  require(dev < 64, "spread: device ordinal out of range");
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!configured[dev]) {
      NUS_CUDA(cudaFuncSetAttribute(spread_gather_kernel<Real, KG>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
      configured[dev] = true;
    }
  }
  const dim3 grid(static_cast<unsigned>(P.ntiles), static_cast<unsigned>(channels));
  spread_gather_kernel<Real, KG><<<grid, kThreads, smem, s>>>(P);
  note_launch();
  check_launch("spread_gather_kernel");
}


struct SpreadLaunch {
  enum Kind { kStream, kSegment, kSegment2, kGather } kind;
  int64_t k0, kg;
};

// Which spread kernel(s) a spectrum of k tapers launches, and their taper ranges.
//   spread_stream_kernel (default): one launch per group of <= 8 tapers, balanced;
//   spread_tc_kernel with two taper groups per staging: 9..16 tapers of a real series on dense data
//     (C3, C4), NUS_SPREAD_GROUPS=1 turns it off;
//   NUS_SPREAD=segment: the per-segment spread_tc_kernel for single groups; NUS_SPREAD=gather: the
//   CUDA-core broadcast gather (Gaussian only), which also takes Gaussians wider than 32 cells.
std::vector<SpreadLaunch> spread_schedule(const Plan& plan, int64_t k, bool x_complex, bool slots) {
  const PlanParams& p = plan.p;
  static const bool use_tc = [] {
    const char* e = std::getenv("NUS_SPREAD");
    return !(e && std::strcmp(e, "gather") == 0);
  }();
  static const bool use_stream = [] {
    const char* e = std::getenv("NUS_SPREAD");
    return !(e && (std::strcmp(e, "gather") == 0 || std::strcmp(e, "segment") == 0));
  }();
  require(use_tc || p.kernel == NUS_KERNEL_GAUSSIAN, "spread: the gather kernel implements the Gaussian only");
  // the tensor-core kernels' weight rows hold one 32-cell window: wider Gaussians (eps < ~2e-13,
  // 2w > 32) take the gather kernel; the ES window is at most 16 cells
  const bool tc = use_tc && p.sw <= 32;
  require(!slots || tc, "spread: slot output needs the tensor-core kernel");
  static const bool two_ok = [] {
    const char* e = std::getenv("NUS_SPREAD_GROUPS");
    return !(e && std::strcmp(e, "1") == 0);
  }();
  static const bool two_forced = [] {
    const char* e = std::getenv("NUS_SPREAD_GROUPS");
    return e && std::strcmp(e, "2") == 0;
  }();
  // two groups per staging: C3 (fp32, K = 9, ns = 6) 781 vs 1085 us against two per-segment
  // single-group launches, C4's structure 543 vs 623 us; slower with the narrowest window (ns = 4)
  // unless the data is dense
  static const int64_t dense_min = [] {
    const char* e = std::getenv("NUS_SPREAD_DENSE_MIN");
    return e ? static_cast<int64_t>(std::atoll(e)) : int64_t{48};
  }();
  const FusedFft& f = plan.ffft;
  const int64_t nseg_used = (f.ready && f.blocked) ? static_cast<int64_t>(f.row_cnt) << (f.lgC - 5) : plan.tab.nseg;
  const bool dense = p.n >= dense_min * nseg_used || p.sw >= 6;
  const SpreadLaunch::Kind single = !tc ? SpreadLaunch::kGather : use_stream ? SpreadLaunch::kStream : SpreadLaunch::kSegment;
  std::vector<SpreadLaunch> out;
  // fp32 plans take streaming launches instead (C3, 32 channels x 2^18, K = 9, ns = 6: two streaming
  // launches 789 us vs 937 us for the two-group kernel, whose 41-point segments need two staging
  // rounds each); in fp64 the two-group kernel stays ahead on HBM-streamed tables (C4's structure
  // 4.72 vs 5.98 ms, C5 at K = 15 703 vs 739 us).  NUS_SPREAD_GROUPS=2 forces it, =1 turns it off.
  const bool two_pref = two_forced || !(use_stream && p.precision == NUS_F32);
  if (tc && two_ok && two_pref && dense && k > 8 && !x_complex) {  // launches of <= 16 tapers, balanced
    const int64_t launches = (k + 15) / 16;
    int64_t kb = 0;
    for (int64_t li = 0; li < launches; ++li) {
      const int64_t kn = (k - kb + (launches - li) - 1) / (launches - li);
      out.push_back({kn > 8 ? SpreadLaunch::kSegment2 : single, kb, kn});
      kb += kn;
    }
    return out;
  }
  const int64_t groups = (k + 7) / 8;  // taper groups of at most 8, balanced
  int64_t k0 = 0;
  for (int64_t gi = 0; gi < groups; ++gi) {
    const int64_t kg = (k - k0 + (groups - gi) - 1) / (groups - gi);
    out.push_back({single, k0, kg});
    k0 += kg;
  }
  return out;
}

template <typename Real>
void spread_typed(const Plan& plan, const SpreadArgs& a, cudaStream_t s) {
  const PlanParams& p = plan.p;
  const SpreadTables& tb = plan.tab;
  require(tb.tile == kTile || p.mr < kTile, "spread: unexpected tile size");
  require(p.sw <= kMaxW2, "spread: spread width too large");
  SpreadParams<Real> P{};
  P.start = tb.start.as<int32_t>();
  P.perm = tb.perm.as<int32_t>();
  P.gauss = tb.gauss.as<typename Vec2<Real>::T>();
  P.prephase = tb.prephase.as<Real>();
  P.ranges = tb.tile_range.as<int32_t>();
  P.seg_ranges = tb.seg_range.as<int32_t>();
  P.nseg = tb.nseg;
  P.lg_nseg = 0;
  while ((int64_t{1} << P.lg_nseg) < tb.nseg) ++P.lg_nseg;
  P.channels = p.channels;
  P.blocked = plan.ffft.ready && plan.ffft.blocked ? 1 : 0;
  if (P.blocked) {  // only the occupied rows of pass A (the others stay unwritten zeros)
    P.lg_spr = plan.ffft.lgC - 5;
    P.row_lo = plan.ffft.row_lo;
    P.nrows = plan.ffft.R;
    P.nseg_used = static_cast<int64_t>(plan.ffft.row_cnt) << P.lg_spr;
  } else {
    P.lg_spr = P.lg_nseg;
    P.row_lo = 0;
    P.nrows = 1;
    P.nseg_used = tb.nseg;
  }
  P.lgC = plan.ffft.lgC;
  P.lgCW = plan.ffft.lgCW;
  P.lgT = plan.ffft.lgT;
  P.wrap_lo = tb.wrap_lo.as<int32_t>();
  P.tapers = static_cast<const Real*>(a.tapers);
  P.x = a.x;
  P.grid = static_cast<typename Vec2<Real>::T*>(a.grid);
  P.slots = reinterpret_cast<typename Vec2<Real>::T* const*>(a.slots);
  P.per = a.per;
  require(!a.slots || (p.channels == 1 && a.per >= 1), "spread: slot output needs one channel and per >= 1");
  P.n = p.n;
  P.mr = p.mr;
  P.ntiles = tb.ntiles;
  P.kpad = a.kpad;
  P.k_total = a.k;
  P.s0 = a.s0;
  P.s1 = a.s1 < 0 ? p.n : a.s1;
  P.tile = tb.tile;
  P.w = p.w;
  P.w2 = p.sw;
  P.x_dtype = a.x_dtype;
  P.x_complex = a.x_complex ? 1 : 0;
  P.beta = static_cast<Real>(p.beta);
  for (int q = 0; q < P.w2; ++q) {
    const double qc = static_cast<double>(q) - (static_cast<double>(p.w) - 0.5);
    P.cq[q] = static_cast<Real>(std::exp(-p.beta * qc * qc));
  }
  {
    auto cexp = [&](double q) {
      const double qc = q - (static_cast<double>(p.w) - 0.5);
      return std::exp(-p.beta * qc * qc);
    };
    P.c0 = cexp(0.0);
    P.c1 = cexp(1.0);
    P.qe0 = std::exp(-4.0 * p.beta * (1.5 - static_cast<double>(p.w)));  // C_2 / C_0
    P.qo0 = std::exp(-4.0 * p.beta * (2.5 - static_cast<double>(p.w)));  // C_3 / C_1
    P.ve = std::exp(-8.0 * p.beta);
  }
  const int ns = p.kernel == NUS_KERNEL_ES ? p.sw : 0;
  const auto sched = spread_schedule(plan, a.tapers ? a.k : 1, a.x_complex, a.slots != nullptr);
  for (const SpreadLaunch& l : sched) {
    P.k0 = static_cast<int>(l.k0);
    P.kg = static_cast<int>(l.kg);
    switch (l.kind) {
      case SpreadLaunch::kStream: launch_stream_x<Real>(P, plan, ns, s); break;
      case SpreadLaunch::kSegment: launch_tc_x<Real>(P, ns, s); break;
      case SpreadLaunch::kSegment2: launch_tc_x<Real>(P, ns, s, true); break;
      default:
        switch (l.kg) {
          case 1: launch_group<Real, 1>(P, p.channels, s); break;
          case 2: launch_group<Real, 2>(P, p.channels, s); break;
          case 3: launch_group<Real, 3>(P, p.channels, s); break;
          case 4: launch_group<Real, 4>(P, p.channels, s); break;
          case 5: launch_group<Real, 5>(P, p.channels, s); break;
          case 6: launch_group<Real, 6>(P, p.channels, s); break;
          case 7: launch_group<Real, 7>(P, p.channels, s); break;
          default: launch_group<Real, 8>(P, p.channels, s); break;
        }
    }
  }
}

}  // namespace

const char* spread_kernel_name() {
  const char* e = std::getenv("NUS_SPREAD");
  return (e && std::strcmp(e, "gather") == 0) ? "spread_gather_kernel"
         : (e && std::strcmp(e, "segment") == 0) ? "spread_tc_kernel"
                                                 : "spread_stream_kernel";
}

std::string spread_kernel_names(const Plan& plan, int64_t k) {
  std::string names;
  for (const SpreadLaunch& l : spread_schedule(plan, k, false, false)) {
    const char* n = l.kind == SpreadLaunch::kStream ? "spread_stream_kernel"
                    : l.kind == SpreadLaunch::kGather ? "spread_gather_kernel"
                                                      : "spread_tc_kernel";
    if (names.find(n) == std::string::npos) names += (names.empty() ? "" : "+") + std::string(n);
  }
  return names;
}

namespace {

template <typename T2>
__global__ void sum_slots_kernel(const T2* __restrict__ base, int64_t nslots, int64_t stride, int64_t count,
                                 T2* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    T2 acc = base[i];
    for (int64_t q = 1; q < nslots; ++q) {
      const T2 v = base[q * stride + i];
      acc.x += v.x;
      acc.y += v.y;
    }
    out[i] = acc;
  }
}

}  // namespace

void sum_slots(const void* base, int64_t nslots, int64_t slot_stride, int64_t count, void* out, bool f64,
               cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, 148 * 8));
  if (f64)
    sum_slots_kernel<double2><<<blocks, 256, 0, s>>>(static_cast<const double2*>(base), nslots, slot_stride, count,
                                                     static_cast<double2*>(out));
  else
    sum_slots_kernel<float2><<<blocks, 256, 0, s>>>(static_cast<const float2*>(base), nslots, slot_stride, count,
                                                    static_cast<float2*>(out));
  note_launch();
  check_launch("sum_slots_kernel");
}


void launch_spread(const Plan& plan, const SpreadArgs& a, cudaStream_t s) {
  if (plan.p.precision == NUS_F64)
    spread_typed<double>(plan, a, s);
  else
    spread_typed<float>(plan, a, s);
}

}  // namespace nus
