// The uniform FFT of the K oversampled grids (every power-of-two Mr), with the deconvolve /
// crop / eigenspectrum reduction fused into its last pass.  No library FFT anywhere.
//
// Replaces Radix2Fft::forward (src/fft.cpp:39-58) + the crop of
// src/nufft.cpp:161-164 + the power loop of src/estimators.cpp:113-117.
//
//   Mr = R * C, j = j1 C + j2, k = k1 + R k2:
//   X[k1 + R k2] = sum_j2 w_C^{j2 k2} [ w_Mr^{j2 k1} sum_j1 x[j1 C + j2] w_R^{j1 k1} ]
//
// Pass A (fft_cols_blk_kernel; fft_cols_small_kernel for R <= 16): each CTA loads one tile of
//   columns (CW consecutive j2, all R rows; contiguous in the spread's blocked layout), runs
//   the length-R FFTs, applies the inter-pass twiddle w_Mr^{j2 k1} (two-level table) and
//   stores the result out of place in the natural layout (row k1).
// Pass B (fft_rows_crop_kernel): each CTA owns one row k1 and loops over the K tapers:
//   length-C FFT in shared memory, then for every output bin k = k1 + R k2 that the crop
//   keeps (m = (-k) mod Mr in [-I/2, I/2)) it adds |X|^2 into a per-thread register
//   accumulator; after the last taper it writes P(i) = d_i^2 * sum_k |X_k|^2 / K.  The
//   transformed grid is never written back.
//
// Sizes: 512 <= Mr <= 8192 is pass B alone (R = 1, C = Mr, NT = Mr / 16 threads); 2^14 .. 2^23
// two passes with C = 2048; 2^24 with C = 4096; 2^25 and 2^26 with C = 8192 (512 threads).
// Grids below 512 cells or above 2^26 (no config comes near either) use the generic radix-2
// Stockham kernels (one launch per stage) + crop_power_kernel; those also serve the Radix2Fft
// drop-in and the DPSS concentration convolution.
//
// In-CTA FFTs are Stockham autosort stages in shared memory with radix-16/8/4/2
// register butterflies; every thread handles 16 elements per stage.  Twiddles come from a
// per-plan table of e^{-2 pi i m / L} built with sincospi (exact argument).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "nus_internal.cuh"

namespace nus {

bool fused_pass_b_async();

namespace {

constexpr int kFftThreads = 256;
constexpr int kFftElems = 4096;  // complex elements resident per CTA

template <typename Real> struct C2;
template <> struct C2<double> { using T = double2; };
template <> struct C2<float> { using T = float2; };

template <typename T2>
__device__ inline T2 cmul(T2 a, T2 b) {
  return T2{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T2>
__device__ inline T2 cadd(T2 a, T2 b) { return T2{a.x + b.x, a.y + b.y}; }
template <typename T2>
__device__ inline T2 csub(T2 a, T2 b) { return T2{a.x - b.x, a.y - b.y}; }

// e^{-2 pi i q / 16}, q = 0..7 (cos, -sin): twiddles of the in-register butterflies
__device__ constexpr double kW16re[8] = {1.0, 0.92387953251128674, 0.70710678118654752, 0.38268343236508977,
                                         0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674};
__device__ constexpr double kW16im[8] = {-0.0, -0.38268343236508977, -0.70710678118654752, -0.92387953251128674,
                                         -1.0, -0.92387953251128674, -0.70710678118654752, -0.38268343236508977};

template <int R>
__host__ __device__ constexpr int bitrev_c(int i) {
  return R <= 1 ? 0 : ((i & 1) * (R >> 1)) | bitrev_c<(R > 1 ? R / 2 : 1)>(i >> 1);
}

// Radix-2 DIT butterflies of span LEN over R registers, then the next span (template
// recursion keeps every index a compile-time constant: no local-memory arrays).
template <int R, int LEN, typename T2>
__device__ inline void dit_stages(T2* v) {
  if constexpr (LEN <= R) {
    using Real = decltype(v[0].x);
    constexpr int half = LEN / 2;
#pragma unroll
    for (int s = 0; s < R; s += LEN) {
#pragma unroll
      for (int q = 0; q < half; ++q) {
        const T2 u = v[s + q];
        T2 t = v[s + q + half];
        constexpr int kStep = 16 / LEN;
        const int wi = q * kStep;  // e^{-2 pi i q / LEN} = W16[wi]
        if (wi == 4) {             // -i
          t = T2{t.y, -t.x};
        } else if (wi == 2) {      // (1 - i) / sqrt(2)
          const Real c = static_cast<Real>(kW16re[2]);
          t = T2{(t.x + t.y) * c, (t.y - t.x) * c};
        } else if (wi == 6) {      // (-1 - i) / sqrt(2)
          const Real c = static_cast<Real>(kW16re[2]);
          t = T2{(t.y - t.x) * c, -(t.x + t.y) * c};
        } else if (wi != 0) {
          t = cmul(t, T2{static_cast<Real>(kW16re[wi]), static_cast<Real>(kW16im[wi])});
        }
        v[s + q] = cadd(u, t);
        v[s + q + half] = csub(u, t);
      }
    }
    dit_stages<R, LEN * 2>(v);
  }
}

// In-register forward DFT of size R (R = 2, 4, 8, 16): natural-order in and out.
template <int R, typename T2>
__device__ inline void dft_reg(T2* v) {
  using Real = decltype(v[0].x);
  // bit-reverse permutation: swap pairs (i, bitrev(i)), indices are compile-time constants
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int j = bitrev_c<R>(i);
    if (j > i) {
      const T2 t = v[i];
      v[i] = v[j];
      v[j] = t;
    }
  }
  dit_stages<R, 2>(v);
}

// Shared-memory index of logical element e: an XOR swizzle chosen per buffer kind, element size and
// exchange so that each wavefront's W lanes (8 lanes of 16-byte elements, 16 of 8-byte ones) meet
// distinct banks in both the stores of one stage and the loads of the next (lanes j' = consecutive
// elements: any XOR of the low lg W bits by higher bits keeps the loads conflict-free).
//   Row buffers (pass B, SWZ).  First exchange: the radix-R0 stage 0 stores lane j at R0 j + q, so the
//   low bits take j's: (e >> lg R0) & (W - 1) when R0 >= W, else (e >> lg W) & (R0 - 1).  Later
//   exchanges: stage stores of stride >= 16 (and the Ns = R0 < W store, whose lanes j, j + Ns sit
//   16 Ns apart) are spread by (e >> 4) & (W - 1).
//   Column buffers (pass A): element (column f, row) at f + CW row, lanes column-fastest; with fewer
//   columns than lanes per wavefront (CW = 4: Mr = 2^21, 2^22) the wavefront spans n = W / CW rows,
//   which the radix-R0 stage-0 stores put CW R0 apart: the row's bits [lg R0, lg R0 + lg n) are
//   XORed into the index bits [lg CW, lg W) (needs R0 >= n, which keeps every later stage's store and
//   load conflict-free too).
// `first`: the exchange between stage 0 and stage 1.
template <bool SWZ, int R0, int ESZ>
__device__ __forceinline__ int sidx(int e, bool first, int lgNfft) {
  constexpr int lgW = ESZ == 16 ? 3 : 4;
  constexpr int W = 1 << lgW;
  constexpr int lgR0 = R0 == 16 ? 4 : R0 == 8 ? 3 : R0 == 4 ? 2 : 1;
  if constexpr (SWZ) {
    const int h0 = R0 >= W ? (e >> lgR0) & (W - 1) : (e >> lgW) & (R0 - 1);
    const int h1 = (e >> 4) & (W - 1);
    return e ^ (first ? h0 : h1);
  } else {
    const int lgn = lgW - lgNfft;
    if (lgn <= 0 || lgR0 < lgn) return e;
    return e ^ (((e >> (lgNfft + lgR0)) & ((1 << lgn) - 1)) << lgNfft);
  }
}

// Register-resident FFT: the thread holds 16 elements.  Stage 0 (radix R0 in {2,4,8,16},
// Ns = 1, no twiddles) runs on values the caller loaded straight from global memory;
// stages 1.. are radix 16 through shared memory; the last stage's outputs stay in
// registers for the caller's epilogue.  Thread -> butterfly mapping is column-fastest
// (u = f + nfft * j).  On entry v[bb*R0 + q] = element (f, j + q*L/R0) of butterfly
// u = tid + bb*256; on exit v[q] = output element (f_out, out0 + q*Ns_last).
// Barrier over the kFftThreads threads that share one in-CTA FFT: id 0 with a 256-thread CTA
// is __syncthreads(); the grouped kernels run two such groups per CTA on ids 1 and 2.
template <int NT = kFftThreads>
__device__ inline void group_bar(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NT) : "memory");
}

template <int R0, bool SWZ, typename T2, int NT = kFftThreads>
__device__ __forceinline__ void fft16_regs(T2 (&v)[16], T2* buf, int lgL, int lgNfft, int es, int fs,
                                  const T2* __restrict__ tw, int& f_out, int& out0, int& step_out, int bar = 0,
                                  int tid = -1) {
  if (tid < 0) tid = threadIdx.x;
  constexpr int B0 = 16 / R0;
  constexpr int lgR0 = R0 == 16 ? 4 : R0 == 8 ? 3 : R0 == 4 ? 2 : 1;
  const int nfm = (1 << lgNfft) - 1;
  // the first radix-16 stage's twiddle, loaded before stage 0 so that its latency hides
  T2 w_next = tw[(((tid >> lgNfft) & ((1 << (lgL - 4)) - 1)) & ((1 << lgR0) - 1)) << (lgL - lgR0 - 4)];
  // ---- stage 0 (registers -> shared)
  {
    const int lgNb = lgL - lgR0;
#pragma unroll
    for (int bb = 0; bb < B0; ++bb) {
      T2* g = v + bb * R0;
      dft_reg<R0>(g);
      const int u = tid + bb * NT;
      const int f = u & nfm, j = (u >> lgNfft) & ((1 << lgNb) - 1);
      const int base = f * fs + (j << lgR0) * es;  // Ns = 1: out = j*R0 + q
#pragma unroll
      for (int q = 0; q < R0; ++q) buf[sidx<SWZ, R0, sizeof(T2)>(base + q * es, true, lgNfft)] = g[q];
    }
  }
  group_bar<NT>(bar);
  // ---- radix-16 stages; the last keeps its outputs in registers
  const int lgNb = lgL - 4;
  const int u = tid;
  const int f = u & nfm, j = (u >> lgNfft) & ((1 << lgNb) - 1);
  const int in0 = f * fs + j * es;
  // each later stage's twiddle is loaded one stage ahead (its latency hides behind a stage)
  for (int lgNs = lgR0; lgNs < lgL; lgNs += 4) {
    const int Ns = 1 << lgNs;
    const int jm = j & (Ns - 1);
    const T2 w1 = w_next;
    if (lgNs + 4 < lgL) w_next = tw[(j & ((Ns << 4) - 1)) << (lgL - lgNs - 8)];
    T2 wq = w1;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      T2 x = buf[sidx<SWZ, R0, sizeof(T2)>(in0 + (q << lgNb) * es, lgNs == lgR0, lgNfft)];
      if (q) {
        x = cmul(x, wq);
        wq = cmul(wq, w1);
      }
      v[q] = x;
    }
    dft_reg<16>(v);
    const int outb = f * fs + (((j - jm) << 4) + jm) * es;
    if (lgNs + 4 < lgL) {
      group_bar<NT>(bar);
#pragma unroll
      for (int q = 0; q < 16; ++q) buf[sidx<SWZ, R0, sizeof(T2)>(outb + (q << lgNs) * es, false, lgNfft)] = v[q];
      group_bar<NT>(bar);
    } else {
      f_out = f;
      out0 = ((j - jm) << 4) + jm;
      step_out = Ns;
    }
  }
}

// Stage-0 input index of register slot (bb, q) for this thread: element j + q*L/R0 of FFT f.
template <int R0, int NT = kFftThreads>
__device__ __forceinline__ void stage0_index(int slot, int lgL, int lgNfft, int& f, int& e, int tid = -1) {
  if (tid < 0) tid = threadIdx.x;
  constexpr int lgR0 = R0 == 16 ? 4 : R0 == 8 ? 3 : R0 == 4 ? 2 : 1;
  const int bb = slot / R0, q = slot % R0;
  const int lgNb = lgL - lgR0;
  const int u = tid + bb * NT;
  f = u & ((1 << lgNfft) - 1);
  const int j = (u >> lgNfft) & ((1 << lgNb) - 1);
  e = j + (q << lgNb);
}

// Output placement of fft16_regs' last (register-resident) radix-16 stage, known before the
// transform: FFT f = tid mod Nfft, outputs out0 + q*st with out0 = j, st = L/16.
__device__ inline void last_stage_out(int tid, int lgL, int lgNfft, int& f, int& out0, int& st) {
  f = tid & ((1 << lgNfft) - 1);
  out0 = (tid >> lgNfft) & ((1 << (lgL - 4)) - 1);
  st = 1 << (lgL - 4);
}

// Inter-pass twiddle pair for w_Mr^{j2 (out0 + q st)}: base w^{j2 out0} and step w^{j2 st}, each
// a product of the two-level table entries (hi, lo).
template <typename T2>
struct PassATwiddles {
  T2 b_hi, b_lo, s_hi, s_lo;
};
template <typename T2>
__device__ inline PassATwiddles<T2> pass_a_twiddles(int64_t j2, int out0, int st, int64_t mr, int lo_bits,
                                                    const T2* __restrict__ tw_hi, const T2* __restrict__ tw_lo) {
  const int64_t lo_mask = (int64_t{1} << lo_bits) - 1;
  const int64_t a0 = (j2 * out0) & (mr - 1), as = (j2 * st) & (mr - 1);
  return PassATwiddles<T2>{tw_hi[a0 >> lo_bits], tw_lo[a0 & lo_mask], tw_hi[as >> lo_bits], tw_lo[as & lo_mask]};
}

// ---- pass A ----------------------------------------------------------------------------

// Pass A over the blocked grid with register loads: one tile (R rows x CW columns, contiguous,
// NT * 16 elements) per CTA, several CTAs per SM in flight instead of a persistent bulk-copy
// pipeline.  Rows outside the occupied interval are zeros and are not read.
// LGR > 0: the column length R = 2^LGR is a compile-time constant (every shared-memory and
// register-slot index of the in-CTA FFT folds to an immediate); 0 = runtime R.
template <typename Real, int R0, int NT, int LGR = 0, int LW = 0>
__global__ void __launch_bounds__(NT, NT == 128 ? 4 : NT == 256 ? (sizeof(Real) == 4 ? 3 : 2) : 1) fft_cols_blk_kernel(
    const typename C2<Real>::T* __restrict__ grid, typename C2<Real>::T* __restrict__ out, int64_t mr, int R, int C,
    int CW, int k, int kpad, const typename C2<Real>::T* __restrict__ tw_r,
    const typename C2<Real>::T* __restrict__ tw_hi, const typename C2<Real>::T* __restrict__ tw_lo, int lo_bits,
    int row_lo, int row_cnt) {
  using T2 = typename C2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* const buf = reinterpret_cast<T2*>(smem_raw);  // [R][CW]
  constexpr int lw = LW;  // FusedFft::lw, compile-time
  constexpr int kLgTile = NT == 128 ? 11 : NT == 256 ? 12 : 13;
  if constexpr (LGR > 0) {
    R = 1 << LGR;
    CW = 1 << (kLgTile - LGR);
  }
  const int lgR = LGR > 0 ? LGR : __ffs(R) - 1;
  const int lgCW = LGR > 0 ? kLgTile - LGR : __ffs(CW) - 1;
  const int lg_nblk = __ffs(C) - 1 - lgCW;
  const int t = blockIdx.x;
  const int blk = t & ((1 << lg_nblk) - 1), ck = t >> lg_nblk;
  const int ch = ck / k, kk = ck - ch * k;
  // tile blk is columns [(blk mod 2^lw) CW, +CW) of layout block blk >> lw, whose rows hold CW << lw cells
  const T2* src = grid + (static_cast<int64_t>(ch) * kpad + kk) * mr +
                  (static_cast<int64_t>(blk >> lw) << (lgR + lgCW + lw)) + ((blk & ((1 << lw) - 1)) << lgCW);
  pdl_launch_dependents();
  pdl_wait();  // the spread's grid
  T2 v[16];
#pragma unroll
  for (int sl = 0; sl < 16; ++sl) {
    int f, e;
    stage0_index<R0, NT>(sl, lgR, lgCW, f, e);
    const bool occ = static_cast<unsigned>((e - row_lo) & (R - 1)) < static_cast<unsigned>(row_cnt);
    v[sl] = occ ? src[((e * CW) << lw) + f] : T2{Real(0), Real(0)};
  }
  int f, out0, st;
  fft16_regs<R0, false, T2, NT>(v, buf, lgR, lgCW, CW, 1, tw_r, f, out0, st);
  T2* g = out + (static_cast<int64_t>(ch) * kpad + kk) * mr;
  const int j2 = blk * CW + f;
  const PassATwiddles<T2> tw2 = pass_a_twiddles(static_cast<int64_t>(j2), out0, st, mr, lo_bits, tw_hi, tw_lo);
  T2 w = cmul(tw2.b_hi, tw2.b_lo);
  const T2 wstep = cmul(tw2.s_hi, tw2.s_lo);
  T2* gr = g + j2 + static_cast<int64_t>(out0) * C;
  const int64_t rstep = static_cast<int64_t>(st) * C;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    gr[q * rstep] = cmul(v[q], w);
    if (q < 15) w = cmul(w, wstep);
  }
}

// Pass A for short columns (R = 2..16: Mr = 2^14, 2^15 with C = 2048): a column's R cells fit in
// one thread's registers, so the length-R DFT runs there with no shared memory.  One blocked tile
// (R rows x CW columns, contiguous) per CTA, each thread taking columns f = tid, tid + 256, ...;
// loads and stores are coalesced across the columns.
template <typename Real, int R>
__global__ void __launch_bounds__(kFftThreads) fft_cols_small_kernel(
    const typename C2<Real>::T* __restrict__ grid, typename C2<Real>::T* __restrict__ out, int64_t mr, int C, int CW,
    int lg_nblk, int k, int kpad, const typename C2<Real>::T* __restrict__ tw_hi,
    const typename C2<Real>::T* __restrict__ tw_lo, int lo_bits, int row_lo, int row_cnt) {
  using T2 = typename C2<Real>::T;
  const int t = blockIdx.x;
  const int blk = t & ((1 << lg_nblk) - 1), ck = t >> lg_nblk;
  const int ch = ck / k, kk = ck - ch * k;
  const T2* src = grid + (static_cast<int64_t>(ch) * kpad + kk) * mr + static_cast<int64_t>(blk) * R * CW;
  T2* g = out + (static_cast<int64_t>(ch) * kpad + kk) * mr;
  for (int f = threadIdx.x; f < CW; f += kFftThreads) {
    T2 v[R];
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const bool occ = static_cast<unsigned>((e - row_lo) & (R - 1)) < static_cast<unsigned>(row_cnt);
      v[e] = occ ? src[e * CW + f] : T2{Real(0), Real(0)};
    }
    dft_reg<R>(v);
    const int j2 = blk * CW + f;
    // w_Mr^{j2 k1}, k1 = 0..R-1: base 1, step w_Mr^{j2} (two-level table)
    const PassATwiddles<T2> tw2 = pass_a_twiddles(static_cast<int64_t>(j2), 0, 1, mr, lo_bits, tw_hi, tw_lo);
    const T2 wstep = cmul(tw2.s_hi, tw2.s_lo);
    T2 w = wstep;
    g[j2] = v[0];
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) {
      g[static_cast<int64_t>(k1) * C + j2] = cmul(v[k1], w);
      if (k1 + 1 < R) w = cmul(w, wstep);
    }
  }
}

// ---- generic radix-2 Stockham FFT (any power of two; one launch per stage) ---------------
// For grids outside the fused passes (Mr < 512, Mr > 2^26), the Radix2Fft drop-in and the DPSS
// concentration convolution.  Stage with half-span ns: y[2(j - k) + k] = a + w b,
// y[2(j - k) + k + ns] = a - w b with a = x[j], b = x[j + n/2], k = j mod ns,
// w = e^{-+ i pi k / ns} (sincospi, exact argument).  Rows r < rows of length n live at
// ((r / kin) kpad_in + r % kin) n on input and ((r / kin) kpad_out + r % kin) n on output.
template <typename T2>
__global__ void stockham_r2_kernel(const T2* __restrict__ x, T2* __restrict__ y, int64_t n, int64_t ns,
                                   int64_t rows, int64_t kin, int64_t kpad_in, int64_t kpad_out, int inverse) {
  using Real = decltype(T2{}.x);
  const int64_t half = n >> 1;
  const int64_t total = rows * half;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = g / half, j = g - r * half;
    const int64_t rc = r / kin, rk = r - rc * kin;
    const T2* xr = x + (rc * kpad_in + rk) * n;
    T2* yr = y + (rc * kpad_out + rk) * n;
    const int64_t k = j & (ns - 1);
    double sn, cs;
    sincospi((inverse ? 1.0 : -1.0) * static_cast<double>(k) / static_cast<double>(ns), &sn, &cs);
    const T2 a = xr[j], b = xr[j + half];
    const Real c = static_cast<Real>(cs), s = static_cast<Real>(sn);
    const T2 bw{b.x * c - b.y * s, b.x * s + b.y * c};
    const int64_t o = ((j - k) << 1) + k;
    yr[o] = T2{a.x + bw.x, a.y + bw.y};
    yr[o + ns] = T2{a.x - bw.x, a.y - bw.y};
  }
}

template <typename T2>
__global__ void copy_rows_kernel(const T2* __restrict__ x, T2* __restrict__ y, int64_t n, int64_t rows, int64_t kin,
                                 int64_t kpad_in, int64_t kpad_out) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < rows * n;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = g / n, i = g - r * n;
    const int64_t rc = r / kin, rk = r - rc * kin;
    y[(rc * kpad_out + rk) * n + i] = x[(rc * kpad_in + rk) * n + i];
  }
}

// ---- pass B + crop / power ---------------------------------------------------------------

constexpr int kCropN = 9;  // last-stage outputs q the crop can keep (pass B, Mr >= 2 nc)
__host__ __device__ constexpr int crop_q(int c) { return c < 5 ? c : c + 7; }

// NT threads per row: 256 for C = 4096 (2 CTAs / SM), 128 for C = 2048 (4 CTAs / SM, twice the
// rows in flight to cover the row loads).
// C = NT * 16 is fixed by NT, so every index of the in-CTA FFT is a compile-time constant
__host__ __device__ constexpr int lg_threads(int nt) { return nt <= 1 ? 0 : 1 + lg_threads(nt / 2); }

// NT = 32 / 64 (C = 512 / 1024): single-pass transforms of small grids (R = 1), several rows per SM.
#ifndef NUS_ROWS_F32_CTAS
#define NUS_ROWS_F32_CTAS 7
#endif
template <typename Real, typename PReal, int R0, int NT = kFftThreads>
__global__ void __launch_bounds__(NT, NT <= 64 ? 8 : NT == 128 ? (sizeof(Real) == 4 ? NUS_ROWS_F32_CTAS : 4) : NT == 256 ? (sizeof(Real) == 4 ? 3 : 2) : 1) fft_rows_crop_kernel(
    const typename C2<Real>::T* __restrict__ grid, int64_t mr, int R, int C, int RPC, int64_t kpad,
    int k_count, int64_t nc, int64_t mode_offset, const Real* __restrict__ deconv,
    const typename C2<Real>::T* __restrict__ tw_c, typename C2<Real>::T* __restrict__ j_out,
    PReal* __restrict__ power, double divisor, int accumulate) {
  using T2 = typename C2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* const buf = reinterpret_cast<T2*>(smem_raw);  // [C] (swizzled)
  const int k1 = blockIdx.x;                        // one row per CTA
  const int64_t ch = blockIdx.y;
  constexpr int lgC = lg_threads(NT) + 4;  // NT threads x 16 registers
  C = 1 << lgC;
  // Mr >= 2 nc, so the crop keeps k2 <= C/4 or k2 >= 3C/4 only: of this thread's outputs
  // k2 = out0 + q C/16 that is q in {0..4, 12..15} (kCropQ); the other seven are never formed
  Real acc[kCropN];
#pragma unroll
  for (int c = 0; c < kCropN; ++c) acc[c] = Real(0);
  int f = 0, out0 = 0, step = 1;
  pdl_launch_dependents();
  pdl_wait();  // pass A's output (and, for power, the previous reader of P)
  // tapers in reverse: pass A wrote them in order, so the last ones are still in L2 for the
  // first wave of rows
  for (int kk = k_count - 1; kk >= 0; --kk) {
    const T2* g = grid + (ch * kpad + kk) * mr + static_cast<int64_t>(k1) * C;
    T2 v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      int ff, e;
      stage0_index<R0, NT>(s, lgC, 0, ff, e);
      v[s] = g[e];
    }
    fft16_regs<R0, true, T2, NT>(v, buf, lgC, 0, 1, C, tw_c, f, out0, step);
#pragma unroll
    for (int c = 0; c < kCropN; ++c) {
      const int q = crop_q(c);
      const T2 x = v[q];
      acc[c] += x.x * x.x + x.y * x.y;
      if (j_out) {
        const int64_t k = static_cast<int64_t>(k1) + static_cast<int64_t>(R) * (out0 + q * step);
        int64_t i = -1;
        if (k <= mode_offset) i = mode_offset - k;
        else if (mr - k < nc - mode_offset) i = mode_offset + (mr - k);
        if (i >= 0 && i < nc) {
          const Real d = deconv[i];
          j_out[(ch * k_count + kk) * nc + i] = T2{d * x.x, d * x.y};
        }
      }
    }
    __syncthreads();  // buf reused by the next taper
  }
  if (!power) return;
  // crop (nufft.cpp:131-140): bin k = k1 + R k2 keeps i = m + I/2 for m in [-I/2, I - I/2), (-m) mod Mr = k.
  // All nine deconvolution factors are loaded (clamped index) before the first is used, so their
  // latencies overlap instead of queueing behind nine branches.
  int64_t iv[kCropN];
  Real dv[kCropN];
#pragma unroll
  for (int c = 0; c < kCropN; ++c) {
    const int64_t k = static_cast<int64_t>(k1) + static_cast<int64_t>(R) * (out0 + crop_q(c) * step);
    int64_t i = -1;
    if (k <= mode_offset) i = mode_offset - k;
    else if (mr - k < nc - mode_offset) i = mode_offset + (mr - k);
    iv[c] = i;
    dv[c] = deconv[i < 0 ? 0 : (i < nc ? i : nc - 1)];
  }
#pragma unroll
  for (int c = 0; c < kCropN; ++c) {
    const int64_t i = iv[c];
    if (i >= 0 && i < nc) {
      const double d = static_cast<double>(dv[c]);
      const PReal val = static_cast<PReal>(d * d * static_cast<double>(acc[c]) / divisor);
      PReal* dst = power + ch * nc + i;
      *dst = accumulate ? *dst + val : val;
    }
  }
  (void)f;
  (void)RPC;
}

// ---- asynchronous (bulk-copy, double-buffered) variants ----------------------------------
// Persistent CTAs, one per SM: each tile (pass A: R rows x CW columns of one taper; pass B:
// one C-element row of one taper) is bulk-copied global -> shared (cp.async.bulk, completion
// on an mbarrier) into one of two buffers while the previous tile is transformed in place in
// the other, so HBM reads overlap the in-CTA FFT instead of stalling its first stage.

__device__ inline uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ inline void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ inline void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ inline void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ inline void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "NUS_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra NUS_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ inline void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ inline void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ inline void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Tile loads: `count` contiguous complex elements -> shared, in 16 KB bulk copies.
template <typename T2>
__device__ inline void issue_tile(T2* dst, const T2* src, int count, uint64_t* bar) {
  const uint32_t bytes = static_cast<uint32_t>(count * sizeof(T2));
  fence_proxy_async();
  mbar_expect_tx(bar, bytes);
  constexpr uint32_t kChunk = 16384;
  for (uint32_t o = 0; o < bytes; o += kChunk)
    bulk_g2s(reinterpret_cast<unsigned char*>(dst) + o, reinterpret_cast<const unsigned char*>(src) + o,
             min(kChunk, bytes - o), bar);
}

// Three tile buffers, two compute groups of kFftThreads threads (named barriers 1, 2): the
// CTA's tiles i = 0, 1, 2, ... go to group i % 2 and buffer i % 3; when a group finishes
// tile i it refills that buffer with tile i + 3, so two tiles are in the FFT and one is in
// flight from HBM at any time.
constexpr int kGroups = 2;
constexpr int kBufs = 3;

// Pass-A tile load restricted to the occupied rows [row_lo, row_lo + row_cnt) (cyclic): one
// or two contiguous runs of the tile (row j1 at offset j1 * CW); the rest is zero-filled at
// stage 0.
// The other rows are copied from a zero buffer (L2-resident), so the tile is complete and
// stage 0 reads it unconditionally.
template <typename T2>
__device__ inline void issue_cols_tile(T2* dst, const T2* src, const T2* zeros, int R, int CW, int row_lo,
                                       int row_cnt, uint64_t* bar) {
  const uint32_t row_bytes = static_cast<uint32_t>(CW * sizeof(T2));
  fence_proxy_async();
  mbar_expect_tx(bar, row_bytes * static_cast<uint32_t>(R));
  constexpr uint32_t kChunk = 16384;
  auto copy = [&](int r0, int rows, bool zero) {
    const uint32_t bytes = row_bytes * static_cast<uint32_t>(rows);
    unsigned char* d = reinterpret_cast<unsigned char*>(dst + r0 * CW);
    const unsigned char* s = reinterpret_cast<const unsigned char*>(zero ? zeros : src + r0 * CW);
    for (uint32_t o = 0; o < bytes; o += kChunk)
      bulk_g2s(d + o, zero ? s : s + o, min(kChunk, bytes - o), bar);
  };
  const int end = row_lo + row_cnt;  // occupied: [row_lo, end) mod R
  if (end <= R) {
    if (row_lo > 0) copy(0, row_lo, true);
    copy(row_lo, row_cnt, false);
    if (end < R) copy(end, R - end, true);
  } else {
    copy(0, end - R, false);
    copy(end - R, row_lo - (end - R), true);
    copy(row_lo, R - row_lo, false);
  }
}

// pass A: tile t = ((ch * k) + kk) * nblk + blk is the contiguous column block blk of the
// blocked grid layout (spread.cu writes cell j1 C + j2 at blk*R*CW + j1*CW + (j2 % CW)).
template <typename T2>
__device__ inline const T2* cols_tile_src(const T2* grid, int64_t t, int64_t nblk, int k, int kpad, int64_t mr) {
  const int64_t blk = t % nblk, ck = t / nblk;
  const int64_t ch = ck / k, kk = ck - ch * k;
  return grid + (ch * kpad + kk) * mr + blk * kFftElems;  // bulk-copy pass A: tiles of 4096 (cols_mode 2)
}

template <typename Real, int R0>
__global__ void __launch_bounds__(kFftThreads * kGroups, 1) fft_cols_async_kernel(
    const typename C2<Real>::T* __restrict__ grid, typename C2<Real>::T* __restrict__ out, int64_t mr, int R, int C,
    int CW, int64_t ntiles, int k, int kpad,
    const typename C2<Real>::T* __restrict__ tw_r, const typename C2<Real>::T* __restrict__ tw_hi,
    const typename C2<Real>::T* __restrict__ tw_lo, int lo_bits, int row_lo, int row_cnt,
    const typename C2<Real>::T* __restrict__ zeros) {
  using T2 = typename C2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* const bufs = reinterpret_cast<T2*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(bufs + kBufs * kFftElems);
  const int64_t nblk = C / CW;
  const int lgR = __ffs(R) - 1, lgCW = __ffs(CW) - 1;
  const int grp = threadIdx.x / kFftThreads, gt = threadIdx.x % kFftThreads;
  const int64_t step = gridDim.x;
  const int64_t nmine = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / step + 1 : 0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < kBufs; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
    for (int b = 0; b < kBufs && b < nmine; ++b)
      issue_cols_tile(bufs + b * kFftElems, cols_tile_src(grid, blockIdx.x + b * step, nblk, k, kpad, mr), zeros, R,
                      CW, row_lo, row_cnt, &bars[b]);
  }
  __syncthreads();
  // 32-bit tile bookkeeping (ntiles < 2^31; nblk = C / CW is a power of two)
  const int lg_nblk = __ffs(static_cast<int>(nblk)) - 1;
  const int nm = static_cast<int>(nmine), st32 = static_cast<int>(step);
  for (int i = grp; i < nm; i += kGroups) {
    const int b = i % kBufs;
    T2* const buf = bufs + b * kFftElems;
    const int t = static_cast<int>(blockIdx.x) + i * st32;
    const int blk = t & ((1 << lg_nblk) - 1), ck = t >> lg_nblk;
    // fp32: the base/step twiddles are loaded before the FFT (they land during it); fp64 has
    // no registers to spare across the transform and loads them after it (one L1 latency)
    PassATwiddles<T2> tw2;
    if constexpr (sizeof(Real) == 4) {
      int fl, out0l, stl;
      last_stage_out(gt, lgR, lgCW, fl, out0l, stl);
      tw2 = pass_a_twiddles(static_cast<int64_t>(blk * CW + fl), out0l, stl, mr, lo_bits, tw_hi, tw_lo);
    }
    mbar_wait(&bars[b], static_cast<uint32_t>((i / kBufs) & 1));
    T2 v[16];
#pragma unroll
    for (int sl = 0; sl < 16; ++sl) {
      int f, e;
      stage0_index<R0>(sl, lgR, lgCW, f, e, gt);
      v[sl] = buf[e * CW + f];
    }
    group_bar(1 + grp);  // stage 0 runs in place
    int f, out0, st;
    fft16_regs<R0, false>(v, buf, lgR, lgCW, CW, 1, tw_r, f, out0, st, 1 + grp, gt);
    const int ch = ck / k, kk = ck - ch * k;
    T2* g = out + (static_cast<int64_t>(ch) * kpad + kk) * mr;  // out of place: the blocked input is still being read
    const int j2 = blk * CW + f;
    if constexpr (sizeof(Real) == 8) tw2 = pass_a_twiddles(static_cast<int64_t>(j2), out0, st, mr, lo_bits, tw_hi, tw_lo);
    // inter-pass twiddles w_Mr^{j2 k1}, k1 = out0 + q st: w_base * w_step^q (base and step were
    // loaded from the two-level table before the FFT; 15 complex products instead of 30 loads)
    T2 w = cmul(tw2.b_hi, tw2.b_lo);
    const T2 wstep = cmul(tw2.s_hi, tw2.s_lo);
    T2* gr = g + j2 + static_cast<int64_t>(out0) * C;
    const int64_t rstep = static_cast<int64_t>(st) * C;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      gr[q * rstep] = cmul(v[q], w);  // natural row-major layout for pass B
      if (q < 15) w = cmul(w, wstep);
    }
    group_bar(1 + grp);  // buf consumed: refill it with tile i + 3
    if (gt == 0 && i + kBufs < nm)
      issue_cols_tile(buf, cols_tile_src(grid, blockIdx.x + static_cast<int64_t>(i + kBufs) * step, nblk, k, kpad, mr),
                      zeros, R, CW, row_lo, row_cnt, &bars[b]);
  }
}

// pass B: CTA unit i = 2 m + g is group g's m-th unit, row rl = blockIdx.x + (2 (m / K) + g) gridDim.x,
// taper kk = m % K (each group keeps a row's K tapers to itself for the |X|^2 sum).
__device__ inline bool rows_unit(int64_t i, int k_count, int64_t nrows, int64_t& row, int64_t& kk) {
  const int64_t g = i % kGroups, m = i / kGroups;
  const int64_t rl = kGroups * (m / k_count) + g;
  kk = m % k_count;
  row = blockIdx.x + rl * static_cast<int64_t>(gridDim.x);
  return row < nrows;
}

template <typename Real, typename PReal, int R0>
__global__ void __launch_bounds__(kFftThreads * kGroups, 1) fft_rows_crop_async_kernel(
    const typename C2<Real>::T* __restrict__ grid, int64_t mr, int R, int C, int64_t nrows, int64_t kpad,
    int k_count, int64_t nc, int64_t mode_offset, const Real* __restrict__ deconv,
    const typename C2<Real>::T* __restrict__ tw_c, typename C2<Real>::T* __restrict__ j_out,
    PReal* __restrict__ power, double divisor, int accumulate) {
  using T2 = typename C2<Real>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T2* const bufs = reinterpret_cast<T2*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(bufs + kBufs * kFftElems);
  const int lgC = __ffs(C) - 1;
  const int grp = threadIdx.x / kFftThreads, gt = threadIdx.x % kFftThreads;
  // units run to the end of the longer group: m < ceil(my_rows / 2) * K per group
  const int64_t my_rows = nrows > blockIdx.x ? (nrows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nunits = ((my_rows + kGroups - 1) / kGroups) * k_count * kGroups;
  auto src_of = [&](int64_t row, int64_t kk) {
    const int64_t ch = row / R, k1 = row - ch * R;
    return grid + (ch * kpad + kk) * mr + k1 * C;
  };
  auto issue = [&](int64_t i, int b) {
    int64_t row, kk;
    if (rows_unit(i, k_count, nrows, row, kk))
      issue_tile(bufs + b * kFftElems, src_of(row, kk), C, &bars[b]);
    else
      mbar_arrive(&bars[b]);  // missing row (odd row count): complete the phase without data
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < kBufs; ++b) mbar_init(&bars[b], 1);
    fence_mbar_init();
    for (int b = 0; b < kBufs && b < nunits; ++b) issue(b, b);
  }
  __syncthreads();
  Real acc[kCropN];
#pragma unroll
  for (int c = 0; c < kCropN; ++c) acc[c] = Real(0);
  const int nu = static_cast<int>(nunits);
  for (int i = grp; i < nu; i += kGroups) {
    const int b = i % kBufs;
    T2* const buf = bufs + b * kFftElems;
    // unit i = 2 m + g: group g's m-th unit, row rl = 2 (m / K) + g of this CTA, taper m % K
    const int m = i >> 1, mq = m / k_count, kk = m - mq * k_count;
    const int row = static_cast<int>(blockIdx.x) + (kGroups * mq + grp) * static_cast<int>(gridDim.x);
    const bool live = row < static_cast<int>(nrows);  // uniform over the group
    // every unit waits for its phase, live or not: a group must never run ahead and refill a
    // buffer (unit i + 3) before that buffer's current unit has been issued and consumed
    mbar_wait(&bars[b], static_cast<uint32_t>((i / kBufs) & 1));
    if (live) {
      const int ch = row / R, k1 = row - ch * R;
      T2 v[16];
#pragma unroll
      for (int sl = 0; sl < 16; ++sl) {
        int ff, e;
        stage0_index<R0>(sl, lgC, 0, ff, e, gt);
        v[sl] = buf[e];
      }
      group_bar(1 + grp);  // stage 0 runs in place
      int f = 0, out0 = 0, st = 1;
      fft16_regs<R0, true>(v, buf, lgC, 0, 1, C, tw_c, f, out0, st, 1 + grp, gt);
#pragma unroll
      for (int c = 0; c < kCropN; ++c) {
        const int q = crop_q(c);
        const T2 x = v[q];
        acc[c] += x.x * x.x + x.y * x.y;
        if (j_out) {
          const int64_t kb = k1 + static_cast<int64_t>(R) * (out0 + q * st);
          int64_t ii = -1;
          if (kb <= mode_offset) ii = mode_offset - kb;
          else if (mr - kb < nc - mode_offset) ii = mode_offset + (mr - kb);
          if (ii >= 0 && ii < nc) {
            const Real d = deconv[ii];
            j_out[(static_cast<int64_t>(ch) * k_count + kk) * nc + ii] = T2{d * x.x, d * x.y};
          }
        }
      }
      if (kk == k_count - 1) {
        if (power) {
          int64_t iv[kCropN];
          Real dv[kCropN];
#pragma unroll
          for (int c = 0; c < kCropN; ++c) {  // all nine loads in flight before the first use
            const int64_t kb = k1 + static_cast<int64_t>(R) * (out0 + crop_q(c) * st);
            int64_t ii = -1;
            if (kb <= mode_offset) ii = mode_offset - kb;
            else if (mr - kb < nc - mode_offset) ii = mode_offset + (mr - kb);
            iv[c] = ii;
            dv[c] = deconv[ii < 0 ? 0 : (ii < nc ? ii : nc - 1)];
          }
#pragma unroll
          for (int c = 0; c < kCropN; ++c) {
            const int64_t ii = iv[c];
            if (ii >= 0 && ii < nc) {
              const double d = static_cast<double>(dv[c]);
              const PReal val = static_cast<PReal>(d * d * static_cast<double>(acc[c]) / divisor);
              PReal* dst = power + static_cast<int64_t>(ch) * nc + ii;
              *dst = accumulate ? *dst + val : val;
            }
          }
        }
#pragma unroll
        for (int c = 0; c < kCropN; ++c) acc[c] = Real(0);
      }
    }
    group_bar(1 + grp);  // buf consumed: refill it with unit i + 3
    if (gt == 0 && i + kBufs < nu) issue(i + kBufs, b);
  }
}


template <typename Real>
__global__ void twiddle_table_kernel(typename C2<Real>::T* __restrict__ out, int64_t count, int64_t stride,
                                     int64_t denom) {
  const int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (m >= count) return;
  // e^{-2 pi i (m * stride) / denom}, argument reduced exactly (powers of two)
  const int64_t a = (m * stride) & (denom - 1);
  double sn, cs;
  sincospi(-2.0 * static_cast<double>(a) / static_cast<double>(denom), &sn, &cs);
  out[m] = typename C2<Real>::T{static_cast<Real>(cs), static_cast<Real>(sn)};
}

int ilog2(int64_t v) {
  int b = 0;
  while ((int64_t{1} << b) < v) ++b;
  return b;
}

}  // namespace

bool pdl_enabled() {
  // Programmatic dependent launch stays off.  Measured on C2 (ES window): 0.288 ms per spectrum
  // with it against 0.264 without, also with last-wave-only triggers and with the spread not
  // waiting on pass B.  It is also unsafe here: a programmatic launch overlapped a preceding
  // H2D copy on the same stream (the host estimate read the previous x), so the launch attribute
  // is never set; the griddepcontrol instructions in the kernels are then no-ops.
  return false;
}

bool fused_fft_supported(const PlanParams& p) {
  // single pass (R = 1) for 512 <= Mr <= 8192: one C = Mr row per CTA, NT = Mr / 16 threads;
  // two passes above: C = 2048 up to 2^23 (R = 8 .. 4096), 4096 at 2^24, 8192 at 2^25 / 2^26.
  // Smaller and larger grids take the generic radix-2 kernels (fft_generic_rows).
  return p.mr >= 512 && p.mr <= (int64_t{1} << 26);
}

namespace {
// Kernel attributes are per device: configured once for every device a process uses.
void configure_fft_kernels() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  NUS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && done[dev]) return;
  const int smem = kFftElems * static_cast<int>(sizeof(double2));
#define NUS_ATTR(KERN) NUS_CUDA(cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))
  NUS_ATTR((fft_rows_crop_kernel<double, double, 16>));
  NUS_ATTR((fft_cols_blk_kernel<double, 16, kFftThreads>));
  NUS_ATTR((fft_cols_blk_kernel<double, 8, kFftThreads>));
  NUS_ATTR((fft_cols_blk_kernel<double, 4, kFftThreads>));
  NUS_ATTR((fft_cols_blk_kernel<double, 2, kFftThreads>));
  NUS_ATTR((fft_cols_blk_kernel<double, 4, kFftThreads, 6>));
  NUS_ATTR((fft_cols_blk_kernel<double, 8, kFftThreads, 7>));
  NUS_ATTR((fft_cols_blk_kernel<double, 16, kFftThreads, 8>));
  NUS_ATTR((fft_cols_blk_kernel<double, 2, kFftThreads, 9>));
  NUS_ATTR((fft_cols_blk_kernel<double, 4, kFftThreads, 10>));
  NUS_ATTR((fft_cols_blk_kernel<double, 8, kFftThreads, 11>));
  NUS_ATTR((fft_cols_blk_kernel<double, 16, kFftThreads, 12>));
  NUS_ATTR((fft_cols_blk_kernel<double, 4, kFftThreads, 10, 1>));
  NUS_ATTR((fft_cols_blk_kernel<double, 8, kFftThreads, 11, 1>));
  NUS_ATTR((fft_cols_blk_kernel<double, 8, kFftThreads, 11, 2>));
  NUS_ATTR((fft_cols_blk_kernel<double, 16, kFftThreads, 12, 1>));
  NUS_ATTR((fft_cols_blk_kernel<double, 16, kFftThreads, 12, 2>));
  NUS_ATTR((fft_cols_blk_kernel<double, 16, kFftThreads, 12, 3>));
#undef NUS_ATTR
  const int smem_w = 2 * kFftElems * static_cast<int>(sizeof(double2));
#define NUS_ATTRW(KERN) NUS_CUDA(cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_w))
  NUS_ATTRW((fft_cols_blk_kernel<double, 16, 512>));
  NUS_ATTRW((fft_cols_blk_kernel<float, 16, 512>));
  NUS_ATTRW((fft_cols_blk_kernel<double, 2, 512>));
  NUS_ATTRW((fft_cols_blk_kernel<double, 16, 512, 0, 1>));
  NUS_ATTRW((fft_cols_blk_kernel<double, 16, 512, 0, 2>));
  NUS_ATTRW((fft_cols_blk_kernel<double, 2, 512, 0, 1>));
  NUS_ATTRW((fft_cols_blk_kernel<double, 2, 512, 0, 2>));
  NUS_ATTRW((fft_cols_blk_kernel<double, 4, 512>));
  NUS_ATTRW((fft_cols_blk_kernel<double, 8, 512>));
  NUS_ATTRW((fft_cols_blk_kernel<float, 4, 512>));
  NUS_ATTRW((fft_cols_blk_kernel<float, 8, 512>));
  NUS_ATTRW((fft_cols_blk_kernel<float, 2, 512>));
  NUS_ATTRW((fft_rows_crop_kernel<double, double, 2, 512>));
  NUS_ATTRW((fft_rows_crop_kernel<float, float, 2, 512>));
  NUS_ATTRW((fft_rows_crop_kernel<float, double, 2, 512>));
#undef NUS_ATTRW
  const int smem2 = kBufs * kFftElems * static_cast<int>(sizeof(double2)) + kBufs * 8;
#define NUS_ATTR2(KERN) NUS_CUDA(cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2))
  NUS_ATTR2((fft_cols_async_kernel<double, 16>));
  NUS_ATTR2((fft_cols_async_kernel<double, 8>));
  NUS_ATTR2((fft_cols_async_kernel<double, 4>));
  NUS_ATTR2((fft_cols_async_kernel<double, 2>));
  NUS_ATTR2((fft_cols_async_kernel<float, 16>));
  NUS_ATTR2((fft_cols_async_kernel<float, 8>));
  NUS_ATTR2((fft_cols_async_kernel<float, 4>));
  NUS_ATTR2((fft_cols_async_kernel<float, 2>));
  NUS_ATTR2((fft_rows_crop_async_kernel<double, double, 16>));
  NUS_ATTR2((fft_rows_crop_async_kernel<float, double, 16>));
  NUS_ATTR2((fft_rows_crop_async_kernel<float, float, 16>));
#undef NUS_ATTR2
  if (dev < 64) done[dev] = true;
}
}  // namespace

void fused_fft_prepare(Plan& plan) {
  PlanParams& p = plan.p;
  FusedFft& f = plan.ffft;
  if (!fused_fft_supported(p) || f.ready) return;
  configure_fft_kernels();
  const int lg = ilog2(p.mr);
  // Rows (pass B, one row per CTA): NT threads x 16 registers = C elements.  C = Mr for
  // Mr <= 8192 (single pass, no pass A); 2048-point rows (4 CTAs / SM) for 2^14 <= Mr <= 2^23
  // (NUS_FFT_C=4096 keeps 4096-point rows from 2^17); 4096 at 2^24; 8192 (512 threads) at 2^25, 2^26.
  // Columns (pass A): R = Mr / C, one R x CW tile (contiguous in the blocked layout) per CTA.
  {
    const char* e = std::getenv("NUS_FFT_C");
    const bool c4096 = e && std::strcmp(e, "4096") == 0;
    if (p.mr <= 2 * kFftElems) f.C = static_cast<int>(p.mr);
    else if (p.mr <= (int64_t{1} << 23)) f.C = (c4096 && p.mr >= (int64_t{1} << 17)) ? kFftElems : kFftElems / 2;
    else if (p.mr == (int64_t{1} << 24)) f.C = kFftElems;
    else f.C = 2 * kFftElems;
  }
  const bool wide = f.C == 2 * kFftElems && p.mr > f.C;  // 8192-element tiles
  f.R = static_cast<int>(p.mr / f.C);
  f.RPC = 1;
  {  // pass A: register-loading 4096-cell tiles (default; 96.4 vs 107.4 us for the bulk-copy
     // pipeline and 114 us for 2048-cell tiles, whose 32-byte row segments coalesce poorly)
    const char* e = std::getenv("NUS_FFT_COLS");
    f.cols_mode = (e && std::strcmp(e, "async") == 0) ? 2 : (e && std::strcmp(e, "reg128") == 0) ? 0 : 1;
  }
  if (f.cols_mode == 0 && (f.R > kFftElems / 2 || f.R < 32)) f.cols_mode = 1;  // a 2048-cell tile must hold >= 1 column
  if (f.cols_mode == 2 && f.R < 32) f.cols_mode = 1;
  if (wide) f.cols_mode = 3;  // R = 4096 / 8192 rows x CW = 2 / 1 columns per 8192-cell tile
  {  // NUS_FFT_COLS=wide: 8192-cell tiles (512 threads, 1 CTA/SM) at any R >= 32: twice the columns per tile
    const char* e = std::getenv("NUS_FFT_COLS");
    if (e && std::strcmp(e, "wide") == 0 && f.R >= 32) f.cols_mode = 3;
  }
  if (f.R > 1 && f.R <= 16) f.cols_mode = 4;  // short columns: register DFTs (fft_cols_small_kernel)
  const int tile = f.cols_mode == 0 ? kFftElems / 2 : f.cols_mode == 3 ? 2 * kFftElems : kFftElems;
  f.CW = f.R > 1 ? tile / f.R : 0;
  f.lo_bits = lg / 2;
  // blocked grid layout whenever there is a pass A (every pass-A tile contiguous)
  f.blocked = f.R > 1;
  f.lgC = ilog2(f.C);
  // fp64 grids with narrow tiles (CW <= 4 columns: R >= 1024): the layout's column blocks are 2^lw = 2
  // tiles wide, so that the spread's 8-cell stores land in pieces twice as long (CW = 4: one 128-byte
  // row instead of two 64-byte ones); a pass-A CTA then reads its CW-column slice of the block's rows.
  // Measured (NUS_FFT_LW = 0 / 1 / 2): C2 spread 74.7 / 71.3 / 71.3 us; C5 spread 333 / 272 / 264 with
  // pass A 220 / 240 / 258; C4's structure at 2^24 (CW = 1) spread 4.60 / 2.15 / 1.99 ms with pass A
  // 1.94 / 1.86 / 2.00; full C4 (8192-cell tiles) 17.5 / 16.7 / 16.7 ms per spectrum.
  f.lw = 0;
  const bool env_wide = [] {
    const char* e = std::getenv("NUS_FFT_COLS");
    return e && std::strcmp(e, "wide") == 0;
  }();
  if (p.precision == NUS_F64 && !env_wide &&
      ((f.cols_mode == 1 && f.R >= 1024 && f.R <= 4096) || (f.cols_mode == 3 && f.R >= 4096))) {
    const char* e = std::getenv("NUS_FFT_LW");
    int lw = e ? std::atoi(e) : 1;
    lw = std::max(0, std::min(lw, f.cols_mode == 3 ? 2 : 3));
    while (lw > 0 && (f.CW << lw) > 8) --lw;  // instantiated up to 8-column blocks
    f.lw = lw;
  }
  f.lgCW = (f.CW > 0 ? ilog2(f.CW) : 0) + f.lw;
  f.lgT = ilog2(f.R) + f.lgCW;
  const bool f64 = p.precision == NUS_F64;
  const size_t cb = f64 ? sizeof(double2) : sizeof(float2);
  const int64_t hi_count = (p.mr >> f.lo_bits), lo_count = int64_t{1} << f.lo_bits;
  f.zeros.alloc(16384);  // bulk-copy source for the unoccupied rows of pass-A tiles
  NUS_CUDA(cudaMemset(f.zeros.ptr, 0, f.zeros.bytes));
  f.tw_r.alloc(std::max(f.R, 2) * cb);
  f.tw_c.alloc(f.C * cb);
  f.tw_hi.alloc(hi_count * cb);
  f.tw_lo.alloc(lo_count * cb);
  auto build = [&](DeviceBuffer& b, int64_t count, int64_t stride, int64_t denom) {
    if (f64)
      twiddle_table_kernel<double><<<static_cast<unsigned>((count + 255) / 256), 256>>>(b.as<double2>(), count,
                                                                                          stride, denom);
    else
      twiddle_table_kernel<float><<<static_cast<unsigned>((count + 255) / 256), 256>>>(b.as<float2>(), count,
                                                                                        stride, denom);
    note_launch();
    check_launch("twiddle_table_kernel");
  };
  build(f.tw_r, std::max(f.R, 2), 1, std::max(f.R, 2));
  build(f.tw_c, f.C, 1, f.C);
  build(f.tw_hi, hi_count, lo_count, p.mr);
  build(f.tw_lo, lo_count, 1, p.mr);
  NUS_CUDA(cudaDeviceSynchronize());
  f.ready = true;
}

namespace {

// first-stage radix so that the remaining stages are all radix 16: L = R0 * 16^m
int first_radix(int L) {
  int lg = 0;
  while ((1 << lg) < L) ++lg;
  const int r = lg % 4;
  return r == 0 ? 16 : (1 << r);
}


int sm_count() {
  static int sms = [] {
    int dev = 0, n = 0;
    NUS_CUDA(cudaGetDevice(&dev));
    NUS_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
  }();
  return sms;
}

template <typename Real>
void launch_cols(const Plan& plan, void* grid, void* scratch, int64_t k, int64_t kpad, cudaStream_t s) {
  const PlanParams& p = plan.p;
  const FusedFft& f = plan.ffft;
  using T2 = typename C2<Real>::T;
  auto* g = static_cast<T2*>(grid);
  auto* out = static_cast<T2*>(scratch);
  const T2 *tr = f.tw_r.as<T2>(), *th = f.tw_hi.as<T2>(), *tl = f.tw_lo.as<T2>();
  const int r0 = first_radix(f.R);
  const int64_t ntiles = p.channels * k * (f.C / f.CW);
  if (f.cols_mode == 4) {  // R <= 16: register DFTs per column
    const int lg_nblk = ilog2(f.C / f.CW);
#define NUS_COLS_SMALL(RR)                                                                                     \
  fft_cols_small_kernel<Real, RR><<<static_cast<unsigned>(ntiles), kFftThreads, 0, s>>>(                      \
      static_cast<const T2*>(g), out, p.mr, f.C, f.CW, lg_nblk, static_cast<int>(k), static_cast<int>(kpad), th, \
      tl, f.lo_bits, f.row_lo, f.row_cnt)
    switch (f.R) {
      case 2: NUS_COLS_SMALL(2); break;
      case 4: NUS_COLS_SMALL(4); break;
      case 8: NUS_COLS_SMALL(8); break;
      case 16: NUS_COLS_SMALL(16); break;
      default: fail(NUS_ERR_INVALID_ARGUMENT, "fft: unsupported short column length");
    }
#undef NUS_COLS_SMALL
    return;
  }
  if (f.cols_mode != 2) {
#define NUS_COLS_REG(R0, NT) NUS_COLS_REGL(R0, NT, 0)
#define NUS_COLS_REGL(R0, NT, LG) NUS_COLS_REGW(R0, NT, LG, 0)
#define NUS_COLS_REGW(R0, NT, LG, LWV)                                                                       \
  launch_pdl(fft_cols_blk_kernel<Real, R0, NT, LG, LWV>, dim3(static_cast<unsigned>(ntiles)), dim3(NT),       \
             static_cast<size_t>(NT) * 16 * sizeof(T2), s, static_cast<const T2*>(g), out, p.mr, f.R, f.C, f.CW, \
             static_cast<int>(k), static_cast<int>(kpad), tr, th, tl, f.lo_bits, f.row_lo, f.row_cnt)
    if (f.cols_mode == 3 && f.lw > 0) {  // fp64, R = 4096 / 8192 (fused_fft_prepare)
      if constexpr (std::is_same_v<Real, double>) {
        if (r0 == 16 && f.lw == 1) NUS_COLS_REGW(16, 512, 0, 1);
        else if (r0 == 16 && f.lw == 2) NUS_COLS_REGW(16, 512, 0, 2);
        else if (r0 == 2 && f.lw == 1) NUS_COLS_REGW(2, 512, 0, 1);
        else if (r0 == 2 && f.lw == 2) NUS_COLS_REGW(2, 512, 0, 2);
        else fail(NUS_ERR_INVALID_ARGUMENT, "fft: unsupported layout block width for 8192-element tiles");
      } else {
        fail(NUS_ERR_INVALID_ARGUMENT, "fft: wide layout blocks are fp64 only");
      }
    } else if (f.cols_mode == 3) {  // R = 4096 (Mr = 2^25) or 8192 (2^26)
      if (r0 == 16) NUS_COLS_REG(16, 512);
      else if (r0 == 2) NUS_COLS_REG(2, 512);
      else if (r0 == 4) NUS_COLS_REG(4, 512);
      else if (r0 == 8) NUS_COLS_REG(8, 512);
      else fail(NUS_ERR_INVALID_ARGUMENT, "fft: unexpected first radix for 8192-element tiles");
    } else if (f.cols_mode == 0) {
      if (r0 == 16) NUS_COLS_REG(16, 128);
      else if (r0 == 8) NUS_COLS_REG(8, 128);
      else if (r0 == 4) NUS_COLS_REG(4, 128);
      else NUS_COLS_REG(2, 128);
    } else if (f.lw > 0) {  // fp64 only (fused_fft_prepare): layout blocks of 2^lw tiles
      if constexpr (std::is_same_v<Real, double>) {
        const int key = f.R * 4 + f.lw;
        switch (key) {
          case 1024 * 4 + 1: NUS_COLS_REGW(4, kFftThreads, 10, 1); break;
          case 2048 * 4 + 1: NUS_COLS_REGW(8, kFftThreads, 11, 1); break;
          case 2048 * 4 + 2: NUS_COLS_REGW(8, kFftThreads, 11, 2); break;
          case 4096 * 4 + 1: NUS_COLS_REGW(16, kFftThreads, 12, 1); break;
          case 4096 * 4 + 2: NUS_COLS_REGW(16, kFftThreads, 12, 2); break;
          case 4096 * 4 + 3: NUS_COLS_REGW(16, kFftThreads, 12, 3); break;
          default: fail(NUS_ERR_INVALID_ARGUMENT, "fft: unsupported layout block width");
        }
      } else {
        fail(NUS_ERR_INVALID_ARGUMENT, "fft: wide layout blocks are fp64 only");
      }
    } else {
      switch (f.R) {  // the column lengths of the configs (Mr = 2^17 .. 2^24), compile-time shapes
        case 64: NUS_COLS_REGL(4, kFftThreads, 6); break;
        case 128: NUS_COLS_REGL(8, kFftThreads, 7); break;
        case 256: NUS_COLS_REGL(16, kFftThreads, 8); break;
        case 512: NUS_COLS_REGL(2, kFftThreads, 9); break;
        case 1024: NUS_COLS_REGL(4, kFftThreads, 10); break;
        case 2048: NUS_COLS_REGL(8, kFftThreads, 11); break;
        case 4096: NUS_COLS_REGL(16, kFftThreads, 12); break;
        default:
          if (r0 == 16) NUS_COLS_REG(16, kFftThreads);
          else if (r0 == 8) NUS_COLS_REG(8, kFftThreads);
          else if (r0 == 4) NUS_COLS_REG(4, kFftThreads);
          else NUS_COLS_REG(2, kFftThreads);
      }
    }
#undef NUS_COLS_REG
#undef NUS_COLS_REGL
#undef NUS_COLS_REGW
    return;
  }
  const unsigned grid_x = static_cast<unsigned>(std::min<int64_t>(ntiles, sm_count()));
  const size_t smem = kBufs * static_cast<size_t>(kFftElems) * sizeof(T2) + kBufs * sizeof(uint64_t);
#define NUS_COLS_ASYNC(R0)                                                                                   \
  fft_cols_async_kernel<Real, R0><<<grid_x, kFftThreads * kGroups, smem, s>>>(g, out, p.mr, f.R, f.C, f.CW, ntiles, \
                                                                    static_cast<int>(k), static_cast<int>(kpad), \
                                                                    tr, th, tl, f.lo_bits, f.row_lo, f.row_cnt, \
                                                                    f.zeros.as<T2>())
  if (r0 == 16) NUS_COLS_ASYNC(16);
  else if (r0 == 8) NUS_COLS_ASYNC(8);
  else if (r0 == 4) NUS_COLS_ASYNC(4);
  else NUS_COLS_ASYNC(2);
#undef NUS_COLS_ASYNC
}

template <typename Real, typename PReal>
void launch_rows(const Plan& plan, void* grid, int64_t k, int64_t kpad, void* j_out, void* power, double divisor,
                 int acc, cudaStream_t s) {
  const PlanParams& p = plan.p;
  const FusedFft& f = plan.ffft;
  using T2 = typename C2<Real>::T;
  const dim3 gb(static_cast<unsigned>(f.R), static_cast<unsigned>(p.channels));
  const size_t smem = static_cast<size_t>(f.C) * sizeof(T2);
  auto* g = static_cast<const T2*>(grid);
  const int r0 = first_radix(f.C);
  // The bulk-copy pass B is correct but measured slower than the register-loading kernel
  // on C2 (0.102 vs 0.097 ms): opt in with NUS_FFT_ASYNC_B=1.
  static const bool async_b = fused_pass_b_async();
  if (f.blocked && r0 == 16 && f.C == kFftElems && async_b) {
    const int64_t nrows = p.channels * f.R;
    const unsigned grid_x = static_cast<unsigned>(std::min<int64_t>(nrows, sm_count()));
    const size_t smem_a = kBufs * static_cast<size_t>(kFftElems) * sizeof(T2) + kBufs * sizeof(uint64_t);
    fft_rows_crop_async_kernel<Real, PReal, 16><<<grid_x, kFftThreads * kGroups, smem_a, s>>>(
        g, p.mr, f.R, f.C, nrows, kpad, static_cast<int>(k), p.nc, p.mode_offset, plan.tab.deconv.as<Real>(),
        f.tw_c.as<T2>(), static_cast<T2*>(j_out), static_cast<PReal*>(power), divisor, acc);
    return;
  }
#define NUS_ROWS(R0, NT)                                                                                  \
  launch_pdl(fft_rows_crop_kernel<Real, PReal, R0, NT>, gb, dim3(NT), smem, s, g, p.mr, f.R, f.C, 1, kpad, \
             static_cast<int>(k), p.nc, p.mode_offset, plan.tab.deconv.as<Real>(), f.tw_c.as<T2>(),       \
             static_cast<T2*>(j_out), static_cast<PReal*>(power), divisor, acc)
  switch (f.C) {  // C = NT * 16; the first radix makes the remaining stages radix 16
    case 512: NUS_ROWS(2, 32); break;
    case 1024: NUS_ROWS(4, 64); break;
    case 2048: NUS_ROWS(8, 128); break;
    case 4096: NUS_ROWS(16, kFftThreads); break;
    case 8192: NUS_ROWS(2, 512); break;
    default: fail(NUS_ERR_INVALID_ARGUMENT, "fft: unsupported row length");
  }
#undef NUS_ROWS
}

}  // namespace

bool fused_pass_b_async() {
  const char* e = std::getenv("NUS_FFT_ASYNC_B");
  return e && std::strcmp(e, "1") == 0;
}

void fft_stage_names(const Plan& plan, const char** a, const char** b) {
  if (!plan.ffft.ready) {
    *a = "stockham_r2_kernel";
    *b = "crop_power_kernel";
    return;
  }
  *a = plan.ffft.R <= 1            ? "(none: single pass)"
       : plan.ffft.cols_mode == 4  ? "fft_cols_small_kernel"
       : plan.ffft.cols_mode == 2  ? "fft_cols_async_kernel"
                                   : "fft_cols_blk_kernel";
  *b = (plan.ffft.blocked && fused_pass_b_async()) ? "fft_rows_crop_async_kernel" : "fft_rows_crop_kernel";
}

void fft_generic_rows(void* data, int64_t n, int64_t rows, int64_t k, int64_t kpad, bool f64, bool inverse,
                      void* scratch, cudaStream_t s) {
  require(n >= 1 && (n & (n - 1)) == 0, "fft: size must be a power of two");
  if (n == 1 || rows == 0) return;
  const int stages = ilog2(n);
  const int64_t work = rows * (n / 2);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((work + 255) / 256, int64_t{148} * 16));
  void* bufs[2] = {data, scratch};
  const int64_t kp[2] = {kpad, k};  // data: [C][kpad][n] (first k rows per channel); scratch dense
  for (int st = 0; st < stages; ++st) {
    const int in = st & 1, out = in ^ 1;
    const int64_t ns = int64_t{1} << st;
    if (f64)
      stockham_r2_kernel<double2><<<blocks, 256, 0, s>>>(static_cast<const double2*>(bufs[in]),
                                                         static_cast<double2*>(bufs[out]), n, ns, rows, k, kp[in],
                                                         kp[out], inverse ? 1 : 0);
    else
      stockham_r2_kernel<float2><<<blocks, 256, 0, s>>>(static_cast<const float2*>(bufs[in]),
                                                        static_cast<float2*>(bufs[out]), n, ns, rows, k, kp[in],
                                                        kp[out], inverse ? 1 : 0);
    note_launch();
    check_launch("stockham_r2_kernel");
  }
  if (stages & 1) {  // the result is in the scratch: back to the caller's layout
    const unsigned cb = static_cast<unsigned>(std::min<int64_t>((rows * n + 255) / 256, int64_t{148} * 16));
    if (f64)
      copy_rows_kernel<double2><<<cb, 256, 0, s>>>(static_cast<const double2*>(scratch), static_cast<double2*>(data),
                                                   n, rows, k, k, kpad);
    else
      copy_rows_kernel<float2><<<cb, 256, 0, s>>>(static_cast<const float2*>(scratch), static_cast<float2*>(data), n,
                                                  rows, k, k, kpad);
    note_launch();
    check_launch("copy_rows_kernel");
  }
}

void fft_generic_inplace(void* data, int64_t n, int64_t batch, bool f64, bool inverse, cudaStream_t s) {
  DeviceBuffer scratch(static_cast<size_t>(n) * batch * (f64 ? sizeof(double2) : sizeof(float2)));
  fft_generic_rows(data, n, batch, batch, batch, f64, inverse, scratch.ptr, s);
  NUS_CUDA(cudaStreamSynchronize(s));  // scratch is released at scope end
}


void run_fused_pass_a(Plan& plan, void* grid, int64_t k, int64_t kpad, cudaStream_t s) {
  if (plan.ffft.R <= 1) return;
  void* scratch = nullptr;
  {  // pass A writes the natural layout out of place; pass B reads it there
    const size_t need = static_cast<size_t>(plan.p.channels * kpad * plan.p.mr) *
                        (plan.p.precision == NUS_F64 ? sizeof(double2) : sizeof(float2));
    if (plan.ffft.scratch.bytes < need) {
      NUS_CUDA(cudaStreamSynchronize(s));
      plan.ffft.scratch.alloc(need);
    }
    scratch = plan.ffft.scratch.ptr;
  }
  if (plan.p.precision == NUS_F64) launch_cols<double>(plan, grid, scratch, k, kpad, s);
  else launch_cols<float>(plan, grid, scratch, k, kpad, s);
  note_launch();
  check_launch("fft pass A");
}

void run_fused_pass_b(Plan& plan, void* grid, int64_t k, int64_t kpad, void* j_out, void* power, bool power_f64,
                      double divisor, bool accumulate, cudaStream_t s) {
  if (plan.ffft.R > 1) grid = plan.ffft.scratch.ptr;  // pass A's output
  const int acc = accumulate ? 1 : 0;
  if (plan.p.precision == NUS_F64) launch_rows<double, double>(plan, grid, k, kpad, j_out, power, divisor, acc, s);
  else if (power_f64) launch_rows<float, double>(plan, grid, k, kpad, j_out, power, divisor, acc, s);
  else launch_rows<float, float>(plan, grid, k, kpad, j_out, power, divisor, acc, s);
  note_launch();
  check_launch("fft_rows_crop_kernel");
}

}  // namespace nus
