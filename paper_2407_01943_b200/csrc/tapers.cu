// Taper setup on the device: nominal-band DPSS, not-a-knot spline
// interpolation to the sample times, and R(B)-metric normalisation.
//
// Reference (paths relative to /root/reference/proj):
//   dpss_uniform       src/tapers.cpp:31-79   (matrix entries :40-52 reproduced exactly)
//   tridiagonal_eigen  src/eig.cpp:572-610    (QL + inverse iteration; here: Sturm
//                      multisection in fp64 + inverse iteration in double-double)
//   canonical_sign     src/eig.cpp:281-289
//   CubicSpline        src/eig.cpp:671-745    (not-a-knot; here: the uniform-knot
//                      moment system solved by its exact two-sided recursive filter)
//   signal_band_kernel + quadratic_form   src/kernels.cpp:16-19,28-37,100-115
//                      (here: an O(N^2) tiled kernel without the dense matrix)
//   gpss_interpolated  src/tapers.cpp:146-182
#include <cub/cub.cuh>

#include <algorithm>
#include <cfloat>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "nus_internal.cuh"

namespace nus {

namespace {

// ---------------------------------------------------------------- Sturm counts

// Each thread evaluates kProbes shift values (independent chains give ILP).  The quotient
// e_i^2 / q uses a branch-free reciprocal (MUFU seed + two Newton steps, <= 1 ulp): the IEEE
// divide's slow-path branch would otherwise serialise the kProbes chains (613 vs ~150 cycles
// per row, scratch microbenchmark).  All threads of a block walk the same rows, so d and e^2
// are staged through shared memory a chunk ahead with cp.async.
constexpr int kProbes = 4;
constexpr int kSturmThreads = 64;
constexpr int kSturmChunk = 1024;

__device__ inline double rcp_nr2(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  return fma(r, e, r);
}

__device__ inline void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ inline void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ inline void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ inline void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__global__ void __launch_bounds__(kSturmThreads) sturm_multisect_kernel(
    const double* __restrict__ d, const double* __restrict__ e2, int64_t n, const double* __restrict__ lo,
    const double* __restrict__ hi, int probes_per_eig, double pivmin, int32_t* __restrict__ counts) {
  constexpr int CH = kSturmChunk;
  __shared__ double sd[2][CH], se[2][CH];
  const int j = blockIdx.y;  // eigenvalue rank
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int p0 = t * kProbes;
  const double a = lo[j], b = hi[j];
  const double step = (b - a) / static_cast<double>(probes_per_eig + 1);
  double lam[kProbes], q[kProbes];
  int cnt[kProbes];
#pragma unroll
  for (int u = 0; u < kProbes; ++u) {
    lam[u] = a + step * static_cast<double>(p0 + u + 1);
    q[u] = d[0] - lam[u];
    if (fabs(q[u]) < pivmin) q[u] = -pivmin;
    cnt[u] = q[u] < 0.0 ? 1 : 0;
  }
  // rows i = 1 .. n-1; chunk c holds i in [1 + c CH, 1 + c CH + CH)
  const int64_t rows = n - 1, nch = (rows + CH - 1) / CH;
  auto load = [&](int64_t c, int buf) {
    const int64_t i0 = 1 + c * CH, cnt_c = rows - c * CH < CH ? rows - c * CH : static_cast<int64_t>(CH);
    for (int r = threadIdx.x; r < cnt_c; r += kSturmThreads) {
      cp_async8(&sd[buf][r], d + i0 + r);
      cp_async8(&se[buf][r], e2 + i0 + r - 1);
    }
    cp_commit();
  };
  if (nch > 0) load(0, 0);
  for (int64_t c = 0; c < nch; ++c) {
    const int buf = static_cast<int>(c & 1);
    if (c + 1 < nch) load(c + 1, buf ^ 1);
    else cp_commit();
    cp_wait1();
    __syncthreads();
    const int cnt_c = static_cast<int>(rows - c * CH < CH ? rows - c * CH : CH);
    for (int r = 0; r < cnt_c; ++r) {
      const double di = sd[buf][r], ei = se[buf][r];
#pragma unroll
      for (int u = 0; u < kProbes; ++u) {
        double v = (di - lam[u]) - ei * rcp_nr2(q[u]);
        if (fabs(v) < pivmin) v = -pivmin;
        q[u] = v;
        cnt[u] += v < 0.0 ? 1 : 0;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < kProbes; ++u)
    if (p0 + u < probes_per_eig) counts[j * probes_per_eig + p0 + u] = cnt[u];
}

__global__ void square_kernel(const double* __restrict__ e, int64_t m, double* __restrict__ e2) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < m) e2[i] = e[i] * e[i];
}

// ------------------------------------------------- inverse iteration (double-double)


__device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Inverse iteration, one warp per eigenvector.  Each iteration solves (T - sigma I) x_new = x
// with partial pivoting (the structure of src/eig.cpp:119-168) entirely in double-double,
// storing the U factor rows (inverse pivot, u1, u2) in global scratch for the back
// substitution; x is renormalised between iterations.
// The recurrences stay serial on lane 0, but every input row
// (d, e, x forward; x, U backward) is brought into shared memory by cp.async one chunk ahead
// and every output row leaves through coalesced stores by the whole warp, so lane 0 never
// waits on a dependent global load (the one-thread version was global-latency bound).
constexpr int kIiChunk = 128;


__global__ void ii_init_kernel(dd* __restrict__ xs, int64_t n, int k) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * k) return;
  const int64_t j = g / n, i = g - j * n;  // same pseudo-random start as the one-thread kernel
  const uint64_t r = mix64(0x9E3779B97F4A7C15ull * static_cast<uint64_t>(j + 1) + static_cast<uint64_t>(i));
  xs[g] = dd{static_cast<double>(r >> 11) * 0x1.0p-53 - 0.5, 0.0};
}

__global__ void __launch_bounds__(32) inverse_iteration_dd_warp_kernel(
    const double* __restrict__ d, const double* __restrict__ e, int64_t n, const double* __restrict__ sigma_hi,
    const double* __restrict__ sigma_lo, int iters, double pivmin, dd* __restrict__ xs, dd* __restrict__ us,
    double* __restrict__ norms) {
  constexpr int CH = kIiChunk;
  __shared__ double sd[2][CH], se[2][CH + 1];
  __shared__ dd sx[2][CH];
  __shared__ dd ox[CH], ou[3 * CH], su[2][3 * CH];
  const int j = blockIdx.x, lane = threadIdx.x;
  dd* x = xs + static_cast<int64_t>(j) * n;
  dd* u = us + static_cast<int64_t>(j) * n * 3;
  const dd sig = {sigma_hi[j], sigma_lo[j]};
  const dd pm = {pivmin, 0.0};
  dd scale = {1.0, 0.0};
  if (n == 1) {
    if (lane == 0) {
      dd p = dd_sub(dd_from(d[0]), sig);
      if (fabs(p.hi) < pivmin) p = p.hi < 0 ? dd_neg(pm) : pm;
      x[0] = dd_mul(x[0], dd_recip(p));
      const dd sc = dd_recip(dd_from(fabs(x[0].hi)));
      norms[2 * j] = sc.hi;
      norms[2 * j + 1] = sc.lo;
    }
    return;
  }
  const int64_t rows = n - 1;  // forward elimination rows i = 0 .. n-2
  const int64_t nch = (rows + CH - 1) / CH;
  for (int it = 0; it < iters; ++it) {
    // ---- forward elimination: chunk c holds rows [c CH, c CH + CH) with inputs
    // d[i+1], e[i], e[i+1] (sup), x[i+1]; outputs x[i], U row i
    auto load_fwd = [&](int64_t c, int b) {
      const int64_t i0 = c * CH, cnt = rows - i0 < CH ? rows - i0 : static_cast<int64_t>(CH);
      for (int q = lane; q < cnt; q += 32) {
        cp_async8(&sd[b][q], d + i0 + q + 1);
        cp_async16(&sx[b][q], x + i0 + q + 1);
      }
      for (int q = lane; q <= cnt; q += 32)
        if (i0 + q < rows) cp_async8(&se[b][q], e + i0 + q);
      cp_commit();
    };
    dd c0 = dd_sub(dd_from(d[0]), sig), c1 = dd_from(e[0]), c2 = dd_from(0.0);
    dd xi = dd_mul(x[0], scale);
    load_fwd(0, 0);
    for (int64_t c = 0; c < nch; ++c) {
      const int b = static_cast<int>(c & 1);
      if (c + 1 < nch) load_fwd(c + 1, b ^ 1);
      else cp_commit();
      cp_wait1();
      __syncwarp();
      const int64_t i0 = c * CH, cnt = rows - i0 < CH ? rows - i0 : static_cast<int64_t>(CH);
      if (lane == 0) {
        for (int q = 0; q < cnt; ++q) {
          const int64_t i = i0 + q;
          const double sub = se[b][q];
          const dd ddv = dd_sub(dd_from(sd[b][q]), sig);
          const double sup = (i + 2 < n) ? se[b][q + 1] : 0.0;
          const dd xn = dd_mul(sx[b][q], scale);
          if (fabs(sub) > fabs(c0.hi)) {
            // pivot on the row below: row i <- (sub, dd, sup), swap rhs
            const dd isub = dd_recip(dd_from(sub));
            const dd m = dd_mul(c0, isub);
            ou[3 * q] = isub;
            ou[3 * q + 1] = ddv;
            ou[3 * q + 2] = dd_from(sup);
            const dd tmp = xi;
            ox[q] = xn;
            xi = dd_sub(tmp, dd_mul(m, xn));
            c0 = dd_sub(c1, dd_mul(m, ddv));
            c1 = dd_sub(c2, dd_mul_d(m, sup));
            c2 = dd_from(0.0);
          } else {
            if (fabs(c0.hi) < pivmin) c0 = c0.hi < 0 ? dd_neg(pm) : pm;
            const dd inv = dd_recip(c0);
            ou[3 * q] = inv;
            ou[3 * q + 1] = c1;
            ou[3 * q + 2] = c2;
            ox[q] = xi;
            const dd m = dd_mul_d(inv, sub);
            xi = dd_sub(xn, dd_mul(m, xi));
            c0 = dd_sub(ddv, dd_mul(m, c1));
            c1 = dd_sub(dd_from(sup), dd_mul(m, c2));
            c2 = dd_from(0.0);
          }
        }
      }
      __syncwarp();
      for (int q = lane; q < cnt; q += 32) x[i0 + q] = ox[q];
      for (int q = lane; q < 3 * cnt; q += 32) u[3 * i0 + q] = ou[q];
      __syncwarp();
    }
    // the last pivot and x[n-1], broadcast from lane 0
    if (lane == 0) {
      if (fabs(c0.hi) < pivmin) c0 = c0.hi < 0 ? dd_neg(pm) : pm;
      x[n - 1] = dd_mul(xi, dd_recip(c0));
    }
    __threadfence_block();
    __syncwarp();
    // ---- back substitution, chunks from the top: rows [c CH, c CH + CH), i descending;
    // the chunk below is prefetched (x rows and U rows) while lane 0 works on this one
    auto load_bwd = [&](int64_t c, int b) {
      const int64_t i0 = c * CH, cnt = rows - i0 < CH ? rows - i0 : static_cast<int64_t>(CH);
      for (int q = lane; q < cnt; q += 32) cp_async16(&sx[b][q], x + i0 + q);
      for (int q = lane; q < 3 * cnt; q += 32) cp_async16(&su[b][q], u + 3 * i0 + q);
      cp_commit();
    };
    dd xl1 = x[n - 1], xl2 = dd_from(0.0);
    dd nrm = dd_mul(xl1, xl1);
    load_bwd(nch - 1, 0);
    for (int64_t cc = 0; cc < nch; ++cc) {
      const int64_t c = nch - 1 - cc;
      const int b = static_cast<int>(cc & 1);
      if (cc + 1 < nch) load_bwd(c - 1, b ^ 1);
      else cp_commit();
      cp_wait1();
      __syncwarp();
      const int64_t i0 = c * CH, cnt = rows - i0 < CH ? rows - i0 : static_cast<int64_t>(CH);
      if (lane == 0) {
        for (int q = static_cast<int>(cnt) - 1; q >= 0; --q) {
          const int64_t i = i0 + q;
          // x_i - u2 x_{i+2} is off the loop-carried path; only u1 x_{i+1} waits on the last row
          const dd t = i != n - 2 ? dd_sub(sx[b][q], dd_mul(su[b][3 * q + 2], xl2)) : sx[b][q];
          const dd v = dd_mul(dd_sub(t, dd_mul(su[b][3 * q + 1], xl1)), su[b][3 * q]);
          ox[q] = v;
          nrm = dd_add(nrm, dd_mul(v, v));
          xl2 = xl1;
          xl1 = v;
        }
      }
      __syncwarp();
      for (int q = lane; q < cnt; q += 32) x[i0 + q] = ox[q];
      __syncwarp();
    }
    if (lane == 0) {
      const double fn = sqrt(nrm.hi);
      const double s0 = 1.0 / fn;
      const dd s0d = dd_from(s0);
      const dd resid = dd_sub(dd_from(1.0), dd_mul(nrm, dd_mul(s0d, s0d)));
      scale = dd_add(s0d, dd_mul_d(dd_mul_d(resid, s0), 0.5));
    }
    scale.hi = __shfl_sync(0xffffffffu, scale.hi, 0);
    scale.lo = __shfl_sync(0xffffffffu, scale.lo, 0);
    __threadfence_block();
    __syncwarp();
  }
  if (lane == 0) {
    norms[2 * j] = scale.hi;
    norms[2 * j + 1] = scale.lo;
  }
}


// ---- DPSS vectors by the eigenvector recurrence, in parallel (large n) ---------------------
// With sigma within ~1e-11 of the eigenvalue, (T - sigma) x = 0 row by row is the three-term
// recurrence x_{i+1} = alpha_i x_i + beta_i x_{i-1}, alpha_i = -(d_i - sigma)/e_i,
// beta_i = -e_{i-1}/e_i.  Run from each end toward the middle, the DPSS grow (edge -> centre) or
// oscillate (centre), so both recurrences are stable there; they are run from x_0 = 1 (left, rows
// 0 .. n/2 + w) and from x_{n-1} = 1 (right, the mirrored recurrence, rows n-1 .. n/2 - w - 1) and
// matched by least squares on the overlap [n/2 - w, n/2 + w] (w = n/64: an odd taper vanishes at
// the centre, so no single row can be the match).  The recurrence is a product of 2x2 matrices,
// evaluated in double-double as a three-phase scan: chunk matrices (two basis solutions per
// chunk of kRecChunk rows, all chunks of all tapers and both halves in parallel), a sequential
// pass over the chunk matrices for the state at every chunk start, and a parallel re-run of the
// chunks writing the vector.  This replaces the full-length sequential inverse iteration (one
// warp per taper over n rows: ~40 s at n = 2^26) of the coarse-start path.
constexpr int kRecChunk = 2048;

struct RecArgs {
  const double* d;
  const double* e;
  int64_t n, len, nch;  // rows per half (recurrence positions 0 .. len-1), chunks per half
  const double* sig_hi;
  const double* sig_lo;
};

// coefficients of recurrence step i (position i -> i+1) of half h (1: mirrored rows)
__device__ inline void rec_coef(const RecArgs& A, int h, int64_t i, dd sig, dd& alpha, dd& beta) {
  const int64_t row = h ? A.n - 1 - i : i;
  const double ei = h ? A.e[A.n - 2 - i] : A.e[i];        // couples positions i, i+1
  const double eim1 = h ? A.e[A.n - 1 - i] : A.e[i - 1];  // couples positions i-1, i
  const dd inv = dd_recip(dd_from(ei));
  alpha = dd_neg(dd_mul(dd_sub(dd_from(A.d[row]), sig), inv));
  beta = dd_neg(dd_mul_d(inv, eim1));
}

// steps of chunk c: i in [1 + c CH, min(1 + (c + 1) CH, len - 1))
__global__ void rec_chunk_matrix_kernel(const RecArgs A, int k, dd* __restrict__ mats) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= static_cast<int64_t>(k) * 2 * A.nch) return;
  const int64_t c = g % A.nch;
  const int h = static_cast<int>((g / A.nch) & 1);
  const int j = static_cast<int>(g / (2 * A.nch));
  const dd sig = {A.sig_hi[j], A.sig_lo[j]};
  dd uc = dd_from(1.0), up = dd_from(0.0), vc = dd_from(0.0), vp = dd_from(1.0);
  const int64_t i0 = 1 + c * kRecChunk, i1 = imin64(1 + (c + 1) * kRecChunk, A.len - 1);
  for (int64_t i = i0; i < i1; ++i) {
    dd al, be;
    rec_coef(A, h, i, sig, al, be);
    const dd un = dd_add(dd_mul(al, uc), dd_mul(be, up));
    const dd vn = dd_add(dd_mul(al, vc), dd_mul(be, vp));
    up = uc;
    uc = un;
    vp = vc;
    vc = vn;
  }
  dd* m = mats + 4 * g;  // end = [uc vc; up vp] (cur, prev) of the chunk's start state
  m[0] = uc;
  m[1] = vc;
  m[2] = up;
  m[3] = vp;
}

__global__ void rec_prefix_kernel(const RecArgs A, int k, const dd* __restrict__ mats, dd* __restrict__ starts) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= 2 * k) return;
  const int h = g & 1, j = g >> 1;
  const dd sig = {A.sig_hi[j], A.sig_lo[j]};
  // x_0 = 1, x_1 = -(d_0 - sigma) / e_0  (mirrored for h = 1)
  const double e0 = h ? A.e[A.n - 2] : A.e[0];
  const int64_t row0 = h ? A.n - 1 : 0;
  dd cur = dd_neg(dd_mul(dd_sub(dd_from(A.d[row0]), sig), dd_recip(dd_from(e0)))), prev = dd_from(1.0);
  const dd* m = mats + 4 * static_cast<int64_t>(g) * A.nch;
  dd* st = starts + 2 * static_cast<int64_t>(g) * A.nch;
  for (int64_t c = 0; c < A.nch; ++c) {
    st[2 * c] = cur;
    st[2 * c + 1] = prev;
    const dd* mc = m + 4 * c;
    const dd nc = dd_add(dd_mul(mc[0], cur), dd_mul(mc[1], prev));
    const dd np = dd_add(dd_mul(mc[2], cur), dd_mul(mc[3], prev));
    cur = nc;
    prev = np;
  }
}

// positions p: left half writes xs[p] for p <= mid + w; right half writes xs[p] for p > mid + w
// and ov[p - (mid - w)] for mid - w <= p <= mid + w
__global__ void rec_expand_kernel(const RecArgs A, int k, const dd* __restrict__ starts, int64_t mid, int64_t w,
                                  dd* __restrict__ xs, dd* __restrict__ ov) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= static_cast<int64_t>(k) * 2 * A.nch) return;
  const int64_t c = g % A.nch;
  const int h = static_cast<int>((g / A.nch) & 1);
  const int j = static_cast<int>(g / (2 * A.nch));
  const dd sig = {A.sig_hi[j], A.sig_lo[j]};
  dd* x = xs + static_cast<int64_t>(j) * A.n;
  dd* o = ov + static_cast<int64_t>(j) * (2 * w + 1);
  auto put = [&](int64_t q, dd v) {  // recurrence position q of half h
    const int64_t p = h ? A.n - 1 - q : q;
    if (h == 0) {
      if (p <= mid + w) x[p] = v;
    } else {
      if (p > mid + w) x[p] = v;
      else if (p >= mid - w) o[p - (mid - w)] = v;
    }
  };
  dd cur = starts[2 * g], prev = starts[2 * g + 1];
  const int64_t i0 = 1 + c * kRecChunk, i1 = imin64(1 + (c + 1) * kRecChunk, A.len - 1);
  if (c == 0) {
    put(0, prev);
    put(1, cur);
  }
  for (int64_t i = i0; i < i1; ++i) {
    dd al, be;
    rec_coef(A, h, i, sig, al, be);
    const dd nx = dd_add(dd_mul(al, cur), dd_mul(be, prev));
    prev = cur;
    cur = nx;
    put(i + 1, cur);
  }
}

// per taper: sums over the overlap of x y and y y, and over the whole vector of x x (after the
// right half is scaled); double-double partial sums per block
constexpr int kRecRed = 256;
__global__ void __launch_bounds__(kRecRed) rec_dot_kernel(const dd* __restrict__ a, const dd* __restrict__ b,
                                                          int64_t len, int64_t stride_a, int64_t stride_b,
                                                          dd* __restrict__ partial) {
  const int j = blockIdx.y;
  const dd* x = a + static_cast<int64_t>(j) * stride_a;
  const dd* y = b + static_cast<int64_t>(j) * stride_b;
  dd acc = dd_from(0.0);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRecRed) + threadIdx.x; i < len;
       i += static_cast<int64_t>(gridDim.x) * kRecRed)
    acc = dd_add(acc, dd_mul(x[i], y[i]));
  __shared__ double sh[kRecRed], sl[kRecRed];
  sh[threadIdx.x] = acc.hi;
  sl[threadIdx.x] = acc.lo;
  __syncthreads();
  for (int o = kRecRed / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const dd r = dd_add(dd{sh[threadIdx.x], sl[threadIdx.x]}, dd{sh[threadIdx.x + o], sl[threadIdx.x + o]});
      sh[threadIdx.x] = r.hi;
      sl[threadIdx.x] = r.lo;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[static_cast<int64_t>(j) * gridDim.x + blockIdx.x] = dd{sh[0], sl[0]};
}

__global__ void dd_scale_range_kernel(dd* __restrict__ xs, const double* __restrict__ scales, int64_t n, int64_t p0,
                                      int64_t p1, int k) {
  const int64_t len = p1 - p0;
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= len * k) return;
  const int64_t j = g / len, p = p0 + (g - j * len);
  xs[j * n + p] = dd_mul(xs[j * n + p], dd{scales[2 * j], scales[2 * j + 1]});
}

// x_j <- x_j * scale_j in double-double (normalised start vectors for a refined second run)
__global__ void dd_scale_kernel(dd* __restrict__ xs, const double* __restrict__ scales, int64_t n, int k) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * k) return;
  const int64_t j = g / n;
  xs[g] = dd_mul(xs[g], dd{scales[2 * j], scales[2 * j + 1]});
}

// Rayleigh-quotient correction of the shift: per block, sum x_i r_i and x_i^2 with
// r = (T - sigma) x formed in double-double (|T| ~ N^2 / 4 against a residual of O(gap) |x|:
// the cancellation needs the extra precision; the sums themselves do not)
constexpr int kRqThreads = 256;
__global__ void __launch_bounds__(kRqThreads) rayleigh_partials_kernel(
    const double* __restrict__ d, const double* __restrict__ e, int64_t n, const dd* __restrict__ xs,
    const double* __restrict__ sigma_hi, const double* __restrict__ sigma_lo, double* __restrict__ partial) {
  const int j = blockIdx.y;
  const dd* x = xs + static_cast<int64_t>(j) * n;
  const dd sig = {sigma_hi[j], sigma_lo[j]};
  double xr = 0.0, xx = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kRqThreads) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * kRqThreads) {
    dd r = dd_mul(dd_sub(dd_from(d[i]), sig), x[i]);
    if (i > 0) r = dd_add(r, dd_mul_d(x[i - 1], e[i - 1]));
    if (i + 1 < n) r = dd_add(r, dd_mul_d(x[i + 1], e[i]));
    xr += x[i].hi * r.hi;
    xx += x[i].hi * x[i].hi;
  }
  __shared__ double s0[kRqThreads], s1[kRqThreads];
  s0[threadIdx.x] = xr;
  s1[threadIdx.x] = xx;
  __syncthreads();
  for (int o = kRqThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s0[threadIdx.x] += s0[threadIdx.x + o];
      s1[threadIdx.x] += s1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * (static_cast<int64_t>(j) * gridDim.x + blockIdx.x)] = s0[0];
    partial[2 * (static_cast<int64_t>(j) * gridDim.x + blockIdx.x) + 1] = s1[0];
  }
}

// Start vectors for large n from the DPSS of a coarse length nc (same NW): fine index m sits at
// coarse position u = m (nc - 1) / (n - 1); 4-point Lagrange interpolation (the vectors vary on
// a scale of ~nc / NW coarse samples, so the interpolant is far below the O(1/nc) difference
// between the two lengths' sequences, which the inverse iteration removes)
__global__ void coarse_start_kernel(const double* __restrict__ cv, int64_t nc, int64_t n, int k, dd* __restrict__ xs) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * k) return;
  const int64_t j = g / n, m = g - j * n;
  const double u = static_cast<double>(m) * static_cast<double>(nc - 1) / static_cast<double>(n - 1);
  int64_t i0 = static_cast<int64_t>(floor(u)) - 1;
  i0 = i0 < 0 ? 0 : (i0 > nc - 4 ? nc - 4 : i0);
  const double* v = cv + j * nc + i0;
  const double x = u - static_cast<double>(i0);  // in [0, 3]
  const double l0 = -(x - 1.0) * (x - 2.0) * (x - 3.0) / 6.0, l1 = x * (x - 2.0) * (x - 3.0) / 2.0;
  const double l2 = -x * (x - 1.0) * (x - 3.0) / 2.0, l3 = x * (x - 1.0) * (x - 2.0) / 6.0;
  xs[g] = dd{l0 * v[0] + l1 * v[1] + l2 * v[2] + l3 * v[3], 0.0};
}

// out[j][i] = x_j[i] * scale_j  (dd -> fp64)
__global__ void dd_finalize_kernel(const dd* __restrict__ xs, const double* __restrict__ scales,
                                   int64_t n, int k, double* __restrict__ out) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * k) return;
  const int64_t j = g / n;
  const dd s = {scales[2 * j], scales[2 * j + 1]};
  const dd v = dd_mul(xs[g], s);
  out[g] = v.hi + v.lo;
}

// canonical_sign (eig.cpp:281-289): first index of max |v| made positive.
struct AbsMax {
  double v;
  int64_t i;
};
__device__ inline AbsMax absmax_merge(AbsMax a, AbsMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__global__ void absmax_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ sign_out) {
  const int j = blockIdx.x;
  const double* row = v + static_cast<int64_t>(j) * n;
  AbsMax best = {-1.0, 0};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) best = absmax_merge(best, AbsMax{fabs(row[i]), i});
  __shared__ double sv[1024];
  __shared__ int64_t si[1024];
  sv[threadIdx.x] = best.v;
  si[threadIdx.x] = best.i;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const AbsMax r = absmax_merge(AbsMax{sv[threadIdx.x], si[threadIdx.x]},
                                    AbsMax{sv[threadIdx.x + off], si[threadIdx.x + off]});
      sv[threadIdx.x] = r.v;
      si[threadIdx.x] = r.i;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sign_out[j] = row[si[0]] < 0.0 ? -1.0 : 1.0;
}

__global__ void scale_rows_kernel(double* __restrict__ v, int64_t n, int k, const double* __restrict__ s) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * k) return;
  v[g] *= s[g / n];
}

__global__ void dpss_matrix_kernel(int64_t n, double c, double* __restrict__ diag, double* __restrict__ off) {
  const int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (m >= n) return;
  // tapers.cpp:46-52, exact operation order (no contraction)
  const double half = __dmul_rn(__dsub_rn(__dsub_rn(static_cast<double>(n), 1.0), __dmul_rn(2.0, static_cast<double>(m))), 0.5);
  diag[m] = __dmul_rn(__dmul_rn(half, half), c);
  if (m >= 1) off[m - 1] = __dmul_rn(static_cast<double>(m), static_cast<double>(n - m)) / 2.0;
}

// ---------------------------------------------------------------- spline

constexpr double kR = -0.26794919243112270;   // sqrt(3) - 2, root of r^2 + 4r + 1
constexpr double kC = 0.28867513459481287;    // 1/sqrt(12)
constexpr int kFilterHalf = 36;               // |r|^36 < 3e-21

// g_j = 6 (y_{j+1} - 2 y_j + y_{j-1}) / h^2 for interior j in [2, n-3]
__device__ inline double ipow_r(int64_t e) {
  double v = 1.0;
  for (int64_t q = 0; q < e && q < 200; ++q) v *= kR;
  return e > 200 ? 0.0 : v;
}

__device__ inline double moment_rhs(const double* y, int64_t j, double inv_h2) {
  return 6.0 * (((y[j + 1] - y[j]) - (y[j] - y[j - 1])) * inv_h2);
}

__device__ inline double filter_at(const double* y, int64_t n, int64_t i, double inv_h2) {
  const int64_t a = imax64(2, i - kFilterHalf), b = imin64(n - 3, i + kFilterHalf);
  double left = 0.0, right = 0.0, pw = 1.0;
  for (int64_t j = imin64(i, b); j >= a; --j) {  // sum_{j<=i} r^{i-j} g_j
    if (j == imin64(i, b)) pw = ipow_r(i - j);
    left = fma(pw, moment_rhs(y, j, inv_h2), left);
    pw *= kR;
  }
  pw = 1.0;
  for (int64_t j = imax64(i + 1, a); j <= b; ++j) {  // sum_{j>i} r^{j-i} g_j
    if (j == imax64(i + 1, a)) pw = ipow_r(j - i);
    right = fma(pw, moment_rhs(y, j, inv_h2), right);
    pw *= kR;
  }
  return kC * (left + right);
}

// Second derivatives M for K rows of knot values (uniform spacing h), n >= 2*kFilterHalf+8.
// Interior: M_{i-1} + 4 M_i + M_{i+1} = g_i (i in [2,n-3]) with the not-a-knot rows
// giving M_1 = (y_2-2y_1+y_0)/h^2 and M_{n-2} likewise (eig.cpp:696-709 with h_i = h).
__global__ void spline_moments_kernel(const double* __restrict__ yk, int64_t n, double h,
                                      double* __restrict__ m_out) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int k = blockIdx.y;
  if (g >= n) return;
  const double* y = yk + static_cast<int64_t>(k) * n;
  double* M = m_out + static_cast<int64_t>(k) * n;
  const double inv_h2 = 1.0 / (h * h);
  const double A = ((y[2] - y[1]) - (y[1] - y[0])) * inv_h2;
  const double B = ((y[n - 1] - y[n - 2]) - (y[n - 2] - y[n - 3])) * inv_h2;
  auto interior = [&](int64_t i) {
    double v = filter_at(y, n, i, inv_h2);
    if (i - 1 < 2 * kFilterHalf) v += (A - filter_at(y, n, 1, inv_h2)) * ipow_r(i - 1);
    if (n - 2 - i < 2 * kFilterHalf)
      v += (B - filter_at(y, n, n - 2, inv_h2)) * ipow_r(n - 2 - i);
    return v;
  };
  double v;
  if (g == 1) v = A;
  else if (g == n - 2) v = B;
  else if (g == 0) v = 2.0 * A - interior(2);
  else if (g == n - 1) v = 2.0 * B - interior(n - 3);
  else v = interior(g);
  M[g] = v;
}

// Small-n path: the reference's Thomas solve (eig.cpp:681-724) on one thread per row.
__global__ void spline_moments_thomas_kernel(const double* __restrict__ xk, const double* __restrict__ yk,
                                             int64_t n, double* __restrict__ m_out,
                                             double* __restrict__ scratch) {
  const int k = blockIdx.x;
  const double* y = yk + static_cast<int64_t>(k) * n;
  double* M = m_out + static_cast<int64_t>(k) * n;
  const int64_t m = n - 2;
  double* sub = scratch + static_cast<int64_t>(k) * 4 * n;
  double* dia = sub + n;
  double* sup = dia + n;
  double* rhs = sup + n;
  auto hh = [&](int64_t i) { return xk[i + 1] - xk[i]; };
  for (int64_t i = 1; i + 1 < n; ++i) {
    const int64_t r = i - 1;
    sub[r] = hh(i - 1) / 6.0;
    dia[r] = (hh(i - 1) + hh(i)) / 3.0;
    sup[r] = hh(i) / 6.0;
    rhs[r] = (y[i + 1] - y[i]) / hh(i) - (y[i] - y[i - 1]) / hh(i - 1);
  }
  {
    const double r01 = hh(0) / hh(1);
    dia[0] += sub[0] * (1.0 + r01);
    sup[0] -= sub[0] * r01;
    sub[0] = 0.0;
  }
  {
    const double rr = hh(n - 2) / hh(n - 3);
    dia[m - 1] += sup[m - 1] * (1.0 + rr);
    sub[m - 1] -= sup[m - 1] * rr;
    sup[m - 1] = 0.0;
  }
  for (int64_t r = 1; r < m; ++r) {
    const double w = sub[r] / dia[r - 1];
    dia[r] -= w * sup[r - 1];
    rhs[r] -= w * rhs[r - 1];
  }
  M[m] = rhs[m - 1] / dia[m - 1];
  for (int64_t r = m - 1; r-- > 0;) M[r + 1] = (rhs[r] - sup[r] * M[r + 2]) / dia[r];
  M[0] = M[1] * (1.0 + hh(0) / hh(1)) - M[2] * (hh(0) / hh(1));
  M[n - 1] = M[n - 2] * (1.0 + hh(n - 2) / hh(n - 3)) - M[n - 3] * (hh(n - 2) / hh(n - 3));
}

__device__ inline double knot_at(double t0, double h, int64_t i) {
  return __dadd_rn(t0, __dmul_rn(h, static_cast<double>(i)));  // tapers.cpp:165
}

// Evaluate K splines (knots t0 + h i) at every sample time (eig.cpp:727-745).
__global__ void spline_eval_kernel(const double* __restrict__ t, int64_t n, double t0, double h,
                                   const double* __restrict__ yk, const double* __restrict__ mk,
                                   int k, double* __restrict__ w) {
  const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= n) return;
  const double x_last = knot_at(t0, h, n - 1);
  double xc = t[s];
  xc = fmin(fmax(xc, t0), x_last);
  int64_t i = static_cast<int64_t>(floor((xc - t0) / h));
  i = imax64(0, imin64(i, n - 1));
  // upper_bound(knots, xc) - 1 on the rounded knots
  while (i + 1 < n && knot_at(t0, h, i + 1) <= xc) ++i;
  while (i > 0 && knot_at(t0, h, i) > xc) --i;
  if (i + 1 >= n) i = n - 2;
  const double xi = knot_at(t0, h, i), xi1 = knot_at(t0, h, i + 1);
  const double hl = xi1 - xi;
  const double a = (xi1 - xc) / hl;
  const double b = (xc - xi) / hl;
  const double ca = a * a * a - a, cb = b * b * b - b, h26 = (hl * hl) / 6.0;
  for (int kk = 0; kk < k; ++kk) {
    const double* y = yk + static_cast<int64_t>(kk) * n;
    const double* M = mk + static_cast<int64_t>(kk) * n;
    w[static_cast<int64_t>(kk) * n + s] = a * y[i] + b * y[i + 1] + (ca * M[i] + cb * M[i + 1]) * h26;
  }
}

// ---------------------------------------------------------------- R(B) quadratic form

// sin / cos of 2 pi F t with the product F t reduced exactly (two-product + rint).
__global__ void band_phase_kernel(const double* __restrict__ t, int64_t n, double f,
                                  double* __restrict__ sn, double* __restrict__ cs) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double p = f * t[i];
  const double e = fma(f, t[i], -p);
  const double r = (p - rint(p)) + e;
  double s, c;
  sincospi(2.0 * r, &s, &c);
  sn[i] = s;
  cs[i] = c;
}

constexpr int kQfRows = 256;
constexpr int kQfCols = 256;
constexpr int kQfChunks = 8;  // column chunks per CTA
constexpr int kQfGroup = 8;   // weight rows per launch (register accumulators)

// q_k partial over rows [row0,row1): sum_n (2F w_n^2 + 2 sum_{m>n} w_n R_nm w_m),
// the symmetric split of sum_n w_n (R(B) w)_n (kernels.cpp:28-37).
__global__ void __launch_bounds__(kQfRows) quadform_kernel(
    const double* __restrict__ t, const double* __restrict__ sn, const double* __restrict__ cs,
    const double* __restrict__ w, int64_t n, int k, double f, double tol, int64_t row0,
    int64_t row1, double* __restrict__ partial) {
  __shared__ double s_t[kQfCols], s_s[kQfCols], s_c[kQfCols];
  __shared__ double s_w[kQfGroup][kQfCols];
  const int64_t rblock = blockIdx.y;
  const int64_t r = row0 + rblock * kQfRows + threadIdx.x;
  const bool has_row = r < row1;
  const int64_t col_start = static_cast<int64_t>(blockIdx.x) * kQfCols * kQfChunks;
  const int64_t row_first = row0 + rblock * kQfRows;
  double acc[kQfGroup];
#pragma unroll
  for (int kk = 0; kk < kQfGroup; ++kk) acc[kk] = 0.0;
  const double tn = has_row ? t[r] : 0.0;
  const double snn = has_row ? sn[r] : 0.0, csn = has_row ? cs[r] : 0.0;
  const double two_pi_f = 2.0 * kPi * f;
  if (col_start + kQfCols * kQfChunks - 1 >= row_first) {
    for (int ch = 0; ch < kQfChunks; ++ch) {
      const int64_t c0 = col_start + static_cast<int64_t>(ch) * kQfCols;
      if (c0 >= n) break;
      if (c0 + kQfCols - 1 < row_first) continue;
      __syncthreads();
      {
        const int64_t cidx = c0 + threadIdx.x;
        const bool ok = cidx < n;
        s_t[threadIdx.x] = ok ? t[cidx] : 0.0;
        s_s[threadIdx.x] = ok ? sn[cidx] : 0.0;
        s_c[threadIdx.x] = ok ? cs[cidx] : 0.0;
#pragma unroll
        for (int kk = 0; kk < kQfGroup; ++kk)
          s_w[kk][threadIdx.x] = (ok && kk < k) ? w[kk * n + cidx] : 0.0;
      }
      __syncthreads();
      if (!has_row || c0 + kQfCols - 1 < r) continue;
      const int cend = static_cast<int>(imin64(kQfCols, n - c0));
      const int cbeg = static_cast<int>(imax64(0, r - c0));
      for (int cc = cbeg; cc < cend; ++cc) {
        const int64_t m = c0 + cc;
        double v;
        if (m == r) {
          v = 2.0 * f;  // diagonal, counted once (kernels.cpp:108)
        } else {
          const double dlt = tn - s_t[cc];
          const double adl = fabs(dlt);
          if (adl < tol) {
            v = 4.0 * f;  // zero-lag rule (kernels.cpp:17), pair counted twice
          } else if (adl * f < 8.0) {
            v = 2.0 * (sin(two_pi_f * dlt) / (kPi * dlt));  // kernels.cpp:18, near lags
          } else {
            v = 2.0 * ((snn * s_c[cc] - csn * s_s[cc]) / (kPi * dlt));
          }
        }
#pragma unroll
        for (int kk = 0; kk < kQfGroup; ++kk) acc[kk] = fma(v, s_w[kk][cc], acc[kk]);
      }
    }
  }
  // acc_k * w_k(n) summed over the block's rows
  __shared__ double red[kQfRows / 32][kQfGroup];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t cta = static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
  for (int kk = 0; kk < kQfGroup; ++kk) {
    double v = (has_row && kk < k) ? acc[kk] * w[kk * n + r] : 0.0;
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    if (lane == 0) red[wid][kk] = v;
  }
  __syncthreads();
  if (threadIdx.x < k) {
    double sum = 0.0;
    for (int q = 0; q < kQfRows / 32; ++q) sum += red[q][threadIdx.x];
    partial[cta * k + threadIdx.x] = sum;
  }
}

__global__ void reduce_partials_kernel(const double* __restrict__ partial, int64_t count, int k,
                                       double* __restrict__ out) {
  const int kk = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += partial[i * k + kk];
  __shared__ double red[1024];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[kk] = red[0];
}

// ---------------------------------------------------------------- concentrations

__global__ void sinc_symbol_kernel(int64_t n, int64_t L, double wband, double2* __restrict__ a) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= L) return;
  double v = 0.0;
  int64_t lag = i <= L / 2 ? i : i - L;
  if (lag == 0) v = 2.0 * wband;
  else if (lag < n && lag > -n) {
    const double lg = static_cast<double>(lag);
    v = sin(2.0 * kPi * wband * lg) / (kPi * lg);  // tapers.cpp:71-72
  }
  a[i] = double2{v, 0.0};
}

__global__ void embed_kernel(const double* __restrict__ v, int64_t n, int64_t L, int k,
                             double2* __restrict__ b) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= L * k) return;
  const int64_t j = g / L, i = g - j * L;
  b[g] = double2{i < n ? v[j * n + i] : 0.0, 0.0};
}

__global__ void cmul_kernel(double2* __restrict__ b, const double2* __restrict__ a, int64_t L, int k) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= L * k) return;
  const double2 x = b[g], y = a[g % L];
  b[g] = double2{x.x * y.x - x.y * y.y, x.x * y.y + x.y * y.x};
}

__global__ void conc_dot_kernel(const double* __restrict__ v, const double2* __restrict__ conv,
                                int64_t n, int64_t L, double* __restrict__ out) {
  const int j = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += v[j * n + i] * conv[j * L + i].x;
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = red[0] / static_cast<double>(L);
}

unsigned blocks_for(int64_t n, int threads) { return static_cast<unsigned>((n + threads - 1) / threads); }

double host_ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// ---------------------------------------------------------------- tridiagonal top-K

// Eigenvectors of (near-)degenerate eigenvalues (|lambda_p - lambda_j| <= 1e-13 ||T||), following the
// reference's inverse iteration (eig.cpp:217-279) so that degenerate spectra give the same
// basis: start at the unused coordinate whose diagonal is nearest lambda (chosen on the host,
// in order over all k vectors), shift lambda + ||T|| eps 10 (rank + 1), up to 6 iterations
// of (partially pivoted solve, normalise, re-orthogonalise against the earlier cluster
// members, normalise), stop at residual <= 1e-11 ||T||.  One block per cluster (members in
// index order); thread 0 runs the sequential solve, the block the reductions.  fp64.
namespace {
constexpr int kClusterThreads = 256;

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < kClusterThreads / 32; ++w) t += red[w];
  return t;
}

__global__ void cluster_inverse_iteration_kernel(const double* __restrict__ d, const double* __restrict__ e,
                                                 int64_t n, const int32_t* __restrict__ offs,
                                                 const int32_t* __restrict__ members,
                                                 const int32_t* __restrict__ starts, const double* __restrict__ lam,
                                                 const double* __restrict__ lam_solve, double anorm, double pivmin,
                                                 double* __restrict__ vec, double* __restrict__ scratch) {
  __shared__ double red[kClusterThreads / 32];
  const int c = blockIdx.x;
  const int m0 = offs[c], m1 = offs[c + 1];
  double* u0 = scratch + static_cast<int64_t>(c) * 3 * n;
  double* u1 = u0 + n;
  double* u2 = u1 + n;
  const double cluster_tol = anorm * 1e-8, accept = anorm * 1e-11;
  for (int q = m0; q < m1; ++q) {
    const int j = members[q];
    double* x = vec + static_cast<int64_t>(j) * n;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = i == starts[q] ? 1.0 : 0.0;
    __syncthreads();
    for (int it = 0; it < 6; ++it) {
      if (threadIdx.x == 0) {  // solve_shifted_tridiag (eig.cpp:119-168)
        const double ls = lam_solve[q];
        if (n == 1) {
          double p = d[0] - ls;
          if (fabs(p) < pivmin) p = copysign(pivmin, p == 0.0 ? 1.0 : p);
          x[0] /= p;
        } else {
          double c0 = d[0] - ls, c1 = e[0], c2 = 0.0;
          for (int64_t i = 0; i + 1 < n; ++i) {
            const double sub = e[i], dd = d[i + 1] - ls, sup = (i + 2 < n) ? e[i + 1] : 0.0;
            if (fabs(sub) > fabs(c0)) {
              u0[i] = sub;
              u1[i] = dd;
              u2[i] = sup;
              const double mm = c0 / sub;
              const double t = x[i];
              x[i] = x[i + 1];
              x[i + 1] = t - mm * x[i];
              c0 = c1 - mm * dd;
              c1 = c2 - mm * sup;
              c2 = 0.0;
            } else {
              if (fabs(c0) < pivmin) c0 = copysign(pivmin, c0 == 0.0 ? 1.0 : c0);
              u0[i] = c0;
              u1[i] = c1;
              u2[i] = c2;
              const double mm = sub / c0;
              x[i + 1] -= mm * x[i];
              c0 = dd - mm * c1;
              c1 = sup - mm * c2;
              c2 = 0.0;
            }
          }
          if (fabs(c0) < pivmin) c0 = copysign(pivmin, c0 == 0.0 ? 1.0 : c0);
          u0[n - 1] = c0;
          x[n - 1] /= u0[n - 1];
          x[n - 2] = (x[n - 2] - u1[n - 2] * x[n - 1]) / u0[n - 2];
          for (int64_t i = n - 2; i-- > 0;) x[i] = (x[i] - u1[i] * x[i + 1] - u2[i] * x[i + 2]) / u0[i];
        }
      }
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {  // normalise, re-orthogonalise, normalise
        double s2 = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s2 += x[i] * x[i];
        const double nrm = sqrt(block_sum(s2, red));
        if (nrm > 0.0)
          for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] /= nrm;
        __syncthreads();
        if (pass == 1) break;
        for (int p = m0; p < q; ++p) {
          if (fabs(lam[p] - lam[q]) > cluster_tol) continue;
          const double* xp = vec + static_cast<int64_t>(members[p]) * n;
          double dot = 0.0;
          for (int64_t i = threadIdx.x; i < n; i += blockDim.x) dot += x[i] * xp[i];
          const double proj = block_sum(dot, red);
          for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] -= proj * xp[i];
          __syncthreads();
        }
      }
      double r2 = 0.0;  // tridiag_residual
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double t = (d[i] - lam[q]) * x[i];
        if (i > 0) t += e[i - 1] * x[i - 1];
        if (i + 1 < n) t += e[i] * x[i + 1];
        r2 += t * t;
      }
      const double resid = sqrt(block_sum(r2, red));
      if (resid <= accept) break;
    }
    __syncthreads();
  }
}
}  // namespace

DpssResult tridiag_top_device(const double* d_diag, const double* d_off, int64_t n, int64_t k,
                              double* d_vec, cudaStream_t s) {
  require(k >= 1 && k <= n, "tridiagonal_eigen: k_top out of range");
  const bool prof = std::getenv("NUS_DPSS_PROF") != nullptr;
  auto tic = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!prof) return;
    NUS_CUDA(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dpss] %s %.3f s\n", what, std::chrono::duration<double>(now - tic).count());
    tic = now;
  };
  // Gershgorin bounds and ||T||_inf from host copies (O(n) validation work)
  std::vector<double> hd(n), he(n > 1 ? n - 1 : 0);
  NUS_CUDA(cudaMemcpyAsync(hd.data(), d_diag, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (n > 1) NUS_CUDA(cudaMemcpyAsync(he.data(), d_off, (n - 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
  double glo = 0, ghi = 0, anorm = 0;
  for (int64_t i = 0; i < n; ++i) {
    require(std::isfinite(hd[i]) && (i + 1 >= n || std::isfinite(he[i])), "tridiagonal: non-finite input");
    double rad = 0;
    if (i > 0) rad += std::fabs(he[i - 1]);
    if (i + 1 < n) rad += std::fabs(he[i]);
    glo = i == 0 ? hd[i] - rad : std::min(glo, hd[i] - rad);
    ghi = i == 0 ? hd[i] + rad : std::max(ghi, hd[i] + rad);
    anorm = std::max(anorm, std::fabs(hd[i]) + rad);
  }
  anorm = std::max(anorm, DBL_MIN);
  const double pad = anorm * 1e-12 + 1e-300;
  glo -= pad;
  ghi += pad;

  DeviceBuffer e2(std::max<int64_t>(n - 1, 1) * sizeof(double));
  if (n > 1) {
    square_kernel<<<blocks_for(n - 1, 256), 256, 0, s>>>(d_off, n - 1, e2.as<double>());
    note_launch();
  }
  // multisection: probes_per_eig probes per eigenvalue per pass
  const int probes = 1024;
  std::vector<double> lo(k, glo), hi(k, ghi);
  DeviceBuffer d_lo(k * sizeof(double)), d_hi(k * sizeof(double)), d_cnt(k * probes * sizeof(int32_t));
  std::vector<int32_t> cnt(k * probes);
  const double pivmin = anorm * DBL_EPSILON * 1e-3;
  // Large n (the DPSS matrix has ||T|| ~ n^2/2 but eigenvalue gaps of O(10) for every n, e.g.
  // 12.75 .. 24.6 at NW = 8): bisect to 2 eps ||T|| and refine every shift by a double-double
  // Rayleigh quotient (below), since at n = 2^26 16 eps ||T|| would exceed half a gap.
  const char* force_refine = std::getenv("NUS_DPSS_REFINE");
  const bool refine = n >= (int64_t{1} << 21) || (force_refine && force_refine[0] == '1');
  const double target = (refine ? 2.0 : 16.0) * DBL_EPSILON * anorm;
  for (int pass = 0; pass < 16; ++pass) {
    bool done = true;
    for (int64_t j = 0; j < k; ++j) done = done && (hi[j] - lo[j] <= target);
    if (done) break;
    if (prof) std::fprintf(stderr, "[dpss] sturm pass %d\n", pass);
    NUS_CUDA(cudaMemcpyAsync(d_lo.ptr, lo.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
    NUS_CUDA(cudaMemcpyAsync(d_hi.ptr, hi.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
    const dim3 grid(blocks_for(probes / kProbes, kSturmThreads), static_cast<unsigned>(k));
    sturm_multisect_kernel<<<grid, kSturmThreads, 0, s>>>(d_diag, e2.as<double>(), n, d_lo.as<double>(),
                                                          d_hi.as<double>(), probes, pivmin,
                                                          d_cnt.as<int32_t>());
    note_launch();
    check_launch("sturm_multisect_kernel");
    NUS_CUDA(cudaMemcpyAsync(cnt.data(), d_cnt.ptr, k * probes * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    NUS_CUDA(cudaStreamSynchronize(s));
    for (int64_t j = 0; j < k; ++j) {
      const int64_t idx = n - 1 - j;  // ascending index of the j-th largest eigenvalue
      const double a = lo[j], b = hi[j];
      const double step = (b - a) / static_cast<double>(probes + 1);
      double nlo = a, nhi = b;
      for (int p = 0; p < probes; ++p) {
        const double lam = a + step * static_cast<double>(p + 1);
        if (cnt[j * probes + p] > idx) { nhi = lam; break; }
        nlo = lam;
      }
      if (!(nhi - nlo < b - a)) { nlo = a; nhi = b; }
      lo[j] = nlo;
      hi[j] = nhi;
    }
  }
  lap("gershgorin+sturm");
  DpssResult res;
  res.values.resize(k);
  std::vector<double> sig_hi(k), sig_lo(k);
  // a diagonal entry split off by negligible off-diagonals (the QL deflation rule,
  // |e_i| <= eps (|d_i| + |d_i+1|)) is an exact eigenvalue: return it exactly, as the reference
  std::vector<double> isolated;
  for (int64_t i = 0; i < n; ++i) {
    const bool lo_split = i == 0 || std::fabs(he[i - 1]) <= DBL_EPSILON * (std::fabs(hd[i - 1]) + std::fabs(hd[i]));
    const bool hi_split = i + 1 >= n || std::fabs(he[i]) <= DBL_EPSILON * (std::fabs(hd[i]) + std::fabs(hd[i + 1]));
    if (lo_split && hi_split) isolated.push_back(hd[i]);
  }
  for (int64_t j = 0; j < k; ++j) {
    double mid = 0.5 * (lo[j] + hi[j]);
    for (const double v : isolated)
      if (v >= lo[j] - target && v <= hi[j] + target) {
        mid = v;
        break;
      }
    res.values[j] = mid;
    sig_hi[j] = mid;
    sig_lo[j] = 0.0;
  }
  // inverse iteration in double-double, one thread per vector
  DeviceBuffer d_sh(k * sizeof(double)), d_sl(k * sizeof(double)), d_norm(2 * k * sizeof(double));
  DeviceBuffer xs(static_cast<size_t>(k) * n * sizeof(dd)), us(static_cast<size_t>(k) * n * 3 * sizeof(dd));
  NUS_CUDA(cudaMemcpyAsync(d_sh.ptr, sig_hi.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  NUS_CUDA(cudaMemcpyAsync(d_sl.ptr, sig_lo.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  ii_init_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(xs.as<dd>(), n, static_cast<int>(k));
  note_launch();
  inverse_iteration_dd_warp_kernel<<<static_cast<unsigned>(k), 32, 0, s>>>(
      d_diag, d_off, n, d_sh.as<double>(), d_sl.as<double>(), 3, pivmin, xs.as<dd>(), us.as<dd>(),
      d_norm.as<double>());
  note_launch();
  check_launch("inverse_iteration_dd_warp_kernel");
  lap("inverse iteration");
  if (refine) {  // shift <- shift + x^T (T - shift) x / x^T x, then two more iterations
    dd_scale_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(xs.as<dd>(), d_norm.as<double>(), n, static_cast<int>(k));
    note_launch();
    const unsigned rb = 296;
    DeviceBuffer part(static_cast<size_t>(k) * rb * 2 * sizeof(double));
    rayleigh_partials_kernel<<<dim3(rb, static_cast<unsigned>(k)), kRqThreads, 0, s>>>(
        d_diag, d_off, n, xs.as<dd>(), d_sh.as<double>(), d_sl.as<double>(), part.as<double>());
    note_launch();
    check_launch("rayleigh_partials_kernel");
    std::vector<double> hp(static_cast<size_t>(k) * rb * 2);
    NUS_CUDA(cudaMemcpyAsync(hp.data(), part.ptr, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    NUS_CUDA(cudaStreamSynchronize(s));
    for (int64_t j = 0; j < k; ++j) {
      long double xr = 0.0L, xx = 0.0L;
      for (unsigned b = 0; b < rb; ++b) {
        xr += hp[2 * (j * rb + b)];
        xx += hp[2 * (j * rb + b) + 1];
      }
      const double mu = static_cast<double>(xr / xx);
      // (sig_hi + sig_lo) + mu as a normalised double-double
      const double s1 = sig_hi[j] + mu, bb = s1 - sig_hi[j];
      const double err = (sig_hi[j] - (s1 - bb)) + (mu - bb) + sig_lo[j];
      sig_hi[j] = s1 + err;
      sig_lo[j] = err - (sig_hi[j] - s1);
      res.values[j] = sig_hi[j];
    }
    NUS_CUDA(cudaMemcpyAsync(d_sh.ptr, sig_hi.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
    NUS_CUDA(cudaMemcpyAsync(d_sl.ptr, sig_lo.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
    inverse_iteration_dd_warp_kernel<<<static_cast<unsigned>(k), 32, 0, s>>>(
        d_diag, d_off, n, d_sh.as<double>(), d_sl.as<double>(), 2, pivmin, xs.as<dd>(), us.as<dd>(),
        d_norm.as<double>());
    note_launch();
    check_launch("inverse_iteration_dd_warp_kernel (refined)");
    lap("rayleigh refinement + 2 iterations");
  }
  dd_finalize_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(xs.as<dd>(), d_norm.as<double>(), n,
                                                            static_cast<int>(k), d_vec);
  note_launch();
  {
    // (near-)degenerate eigenvalues, which no inverse iteration separates: the reference's
    // start-vector / re-orthogonalisation rule.  Pairs the double-double iteration resolves
    // (DPSS gaps are ~1e-8 ||T|| at N = 2^16) keep the fast path: their eigenvectors are unique.
    const double cluster_tol = refine ? 8.0 * DBL_EPSILON * anorm : anorm * 1e-13;
    std::vector<int32_t> offs{0}, members, starts;
    std::vector<double> lam, lam_solve;
    std::vector<char> used(n, 0);
    std::vector<int64_t> best(k);
    for (int64_t j = 0; j < k; ++j) {  // nearest unused diagonal, in order (eig.cpp:234-245)
      int64_t b = n;
      double gap = 0.0;
      for (int64_t i = 0; i < n; ++i) {
        if (used[i]) continue;
        const double g = std::fabs(hd[i] - res.values[j]);
        if (b == n || g < gap) {
          b = i;
          gap = g;
        }
      }
      if (b == n) b = j % n;
      used[b] = 1;
      best[j] = b;
    }
    std::vector<char> done(k, 0);
    for (int64_t j = 0; j < k; ++j) {
      if (done[j]) continue;
      // connected component of the "within cluster_tol" relation starting at j
      std::vector<int64_t> comp{j};
      done[j] = 1;
      for (size_t a = 0; a < comp.size(); ++a)
        for (int64_t p = 0; p < k; ++p)
          if (!done[p] && std::fabs(res.values[p] - res.values[comp[a]]) <= cluster_tol) {
            done[p] = 1;
            comp.push_back(p);
          }
      if (comp.size() < 2) continue;
      std::sort(comp.begin(), comp.end());
      for (const int64_t q : comp) {
        int64_t rank = 0;
        for (int64_t p = 0; p < q; ++p)
          if (std::fabs(res.values[p] - res.values[q]) <= cluster_tol) ++rank;
        members.push_back(static_cast<int32_t>(q));
        starts.push_back(static_cast<int32_t>(best[q]));
        lam.push_back(res.values[q]);
        lam_solve.push_back(res.values[q] + anorm * DBL_EPSILON * 10.0 * static_cast<double>(rank + 1));
      }
      offs.push_back(static_cast<int32_t>(members.size()));
    }
    const int ncl = static_cast<int>(offs.size()) - 1;
    if (ncl > 0) {
      DeviceBuffer d_offs(offs.size() * sizeof(int32_t)), d_mem(members.size() * sizeof(int32_t)),
          d_st(starts.size() * sizeof(int32_t)), d_lam(lam.size() * sizeof(double)),
          d_ls(lam_solve.size() * sizeof(double)), scr(static_cast<size_t>(ncl) * 3 * n * sizeof(double));
      NUS_CUDA(cudaMemcpyAsync(d_offs.ptr, offs.data(), d_offs.bytes, cudaMemcpyHostToDevice, s));
      NUS_CUDA(cudaMemcpyAsync(d_mem.ptr, members.data(), d_mem.bytes, cudaMemcpyHostToDevice, s));
      NUS_CUDA(cudaMemcpyAsync(d_st.ptr, starts.data(), d_st.bytes, cudaMemcpyHostToDevice, s));
      NUS_CUDA(cudaMemcpyAsync(d_lam.ptr, lam.data(), d_lam.bytes, cudaMemcpyHostToDevice, s));
      NUS_CUDA(cudaMemcpyAsync(d_ls.ptr, lam_solve.data(), d_ls.bytes, cudaMemcpyHostToDevice, s));
      cluster_inverse_iteration_kernel<<<static_cast<unsigned>(ncl), kClusterThreads, 0, s>>>(
          d_diag, d_off, n, d_offs.as<int32_t>(), d_mem.as<int32_t>(), d_st.as<int32_t>(), d_lam.as<double>(),
          d_ls.as<double>(), anorm, pivmin, d_vec, scr.as<double>());
      note_launch();
      check_launch("cluster_inverse_iteration_kernel");
      NUS_CUDA(cudaStreamSynchronize(s));
    }
  }
  lap("clusters");
  DeviceBuffer sg(k * sizeof(double));
  absmax_kernel<<<static_cast<unsigned>(k), 1024, 0, s>>>(d_vec, n, sg.as<double>());
  note_launch();
  scale_rows_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(d_vec, n, static_cast<int>(k), sg.as<double>());
  note_launch();
  check_launch("dpss finalize");
  NUS_CUDA(cudaStreamSynchronize(s));
  return res;
}

namespace {

// Rayleigh quotient shift update sig <- sig + x^T (T - sig) x / x^T x for every row of xs
void rayleigh_update(const double* d_diag, const double* d_off, int64_t n, int64_t k, const dd* xs,
                     std::vector<double>& sig_hi, std::vector<double>& sig_lo, cudaStream_t s) {
  DeviceBuffer d_sh(k * sizeof(double)), d_sl(k * sizeof(double));
  NUS_CUDA(cudaMemcpyAsync(d_sh.ptr, sig_hi.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  NUS_CUDA(cudaMemcpyAsync(d_sl.ptr, sig_lo.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  const unsigned rb = 296;
  DeviceBuffer part(static_cast<size_t>(k) * rb * 2 * sizeof(double));
  rayleigh_partials_kernel<<<dim3(rb, static_cast<unsigned>(k)), kRqThreads, 0, s>>>(
      d_diag, d_off, n, xs, d_sh.as<double>(), d_sl.as<double>(), part.as<double>());
  note_launch();
  check_launch("rayleigh_partials_kernel");
  std::vector<double> hp(static_cast<size_t>(k) * rb * 2);
  NUS_CUDA(cudaMemcpyAsync(hp.data(), part.ptr, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
  for (int64_t j = 0; j < k; ++j) {
    long double xr = 0.0L, xx = 0.0L;
    for (unsigned b = 0; b < rb; ++b) {
      xr += hp[2 * (j * rb + b)];
      xx += hp[2 * (j * rb + b) + 1];
    }
    const double mu = static_cast<double>(xr / xx);
    const double s1 = sig_hi[j] + mu, bb = s1 - sig_hi[j];
    const double err = (sig_hi[j] - (s1 - bb)) + (mu - bb) + sig_lo[j];
    sig_hi[j] = s1 + err;
    sig_lo[j] = err - (sig_hi[j] - s1);
  }
}


// DPSS rows xs [k][n] (double-double, unit norm) by the two-sided recurrence at the shifts sig
// (rec_* kernels above).
void dpss_recurrence_vectors(const double* d_diag, const double* d_off, int64_t n, int64_t k,
                             const std::vector<double>& sig_hi, const std::vector<double>& sig_lo, dd* xs,
                             cudaStream_t s) {
  const int64_t mid = n / 2, w = std::max<int64_t>(8, n / 64);
  RecArgs A{};
  A.d = d_diag;
  A.e = d_off;
  A.n = n;
  A.len = mid + w + 1;
  A.nch = (A.len - 2 + kRecChunk - 1) / kRecChunk;
  DeviceBuffer d_sh(k * sizeof(double)), d_sl(k * sizeof(double));
  NUS_CUDA(cudaMemcpyAsync(d_sh.ptr, sig_hi.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  NUS_CUDA(cudaMemcpyAsync(d_sl.ptr, sig_lo.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  A.sig_hi = d_sh.as<double>();
  A.sig_lo = d_sl.as<double>();
  const int64_t chunks = k * 2 * A.nch;
  DeviceBuffer mats(static_cast<size_t>(chunks) * 4 * sizeof(dd)), starts(static_cast<size_t>(chunks) * 2 * sizeof(dd));
  DeviceBuffer ov(static_cast<size_t>(k) * (2 * w + 1) * sizeof(dd));
  rec_chunk_matrix_kernel<<<blocks_for(chunks, 128), 128, 0, s>>>(A, static_cast<int>(k), mats.as<dd>());
  note_launch();
  rec_prefix_kernel<<<blocks_for(2 * k, 32), 32, 0, s>>>(A, static_cast<int>(k), mats.as<dd>(), starts.as<dd>());
  note_launch();
  rec_expand_kernel<<<blocks_for(chunks, 128), 128, 0, s>>>(A, static_cast<int>(k), starts.as<dd>(), mid, w, xs,
                                                            ov.as<dd>());
  note_launch();
  check_launch("dpss recurrence");
  constexpr unsigned kBlocks = 256;
  DeviceBuffer part(static_cast<size_t>(k) * kBlocks * sizeof(dd));
  std::vector<dd> hp(static_cast<size_t>(k) * kBlocks);
  auto dot = [&](const dd* a, const dd* b, int64_t len, int64_t sa, int64_t sb) {
    rec_dot_kernel<<<dim3(kBlocks, static_cast<unsigned>(k)), kRecRed, 0, s>>>(a, b, len, sa, sb, part.as<dd>());
    note_launch();
    check_launch("rec_dot_kernel");
    NUS_CUDA(cudaMemcpyAsync(hp.data(), part.ptr, hp.size() * sizeof(dd), cudaMemcpyDeviceToHost, s));
    NUS_CUDA(cudaStreamSynchronize(s));
    std::vector<long double> r(k, 0.0L);
    for (int64_t j = 0; j < k; ++j)
      for (unsigned b2 = 0; b2 < kBlocks; ++b2)
        r[j] += static_cast<long double>(hp[j * kBlocks + b2].hi) + static_cast<long double>(hp[j * kBlocks + b2].lo);
    return r;
  };
  // match the right half to the left on the overlap (least squares), then normalise
  const std::vector<long double> xy = dot(xs + (mid - w), ov.as<dd>(), 2 * w + 1, n, 2 * w + 1);
  const std::vector<long double> yy = dot(ov.as<dd>(), ov.as<dd>(), 2 * w + 1, 2 * w + 1, 2 * w + 1);
  std::vector<double> sc(2 * k);
  auto to_dd = [](long double v, double* out) {
    out[0] = static_cast<double>(v);
    out[1] = static_cast<double>(v - static_cast<long double>(out[0]));
  };
  for (int64_t j = 0; j < k; ++j) {
    require(yy[j] > 0.0L, "dpss: degenerate recurrence overlap");
    to_dd(xy[j] / yy[j], &sc[2 * j]);
  }
  DeviceBuffer d_sc(2 * k * sizeof(double));
  NUS_CUDA(cudaMemcpyAsync(d_sc.ptr, sc.data(), sc.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  const int64_t p0 = mid + w + 1;
  dd_scale_range_kernel<<<blocks_for((n - p0) * k, 256), 256, 0, s>>>(xs, d_sc.as<double>(), n, p0, n,
                                                                      static_cast<int>(k));
  note_launch();
  const std::vector<long double> xx = dot(xs, xs, n, n, n);
  for (int64_t j = 0; j < k; ++j) to_dd(1.0L / std::sqrt(xx[j]), &sc[2 * j]);
  NUS_CUDA(cudaMemcpyAsync(d_sc.ptr, sc.data(), sc.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  dd_scale_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(xs, d_sc.as<double>(), n, static_cast<int>(k));
  note_launch();
  check_launch("dpss recurrence normalise");
  NUS_CUDA(cudaStreamSynchronize(s));
}
}  // namespace

// DPSS for large n (>= NUS_DPSS_COARSE, default 2^20) without bisection at full length: the DPSS
// of a coarse length nc = n / 64 (>= 2^17, same NW) interpolated to n gives start vectors within
// O(1/nc) of the answer; two double-double Rayleigh quotients (against shift 0, then against the
// first, so the second residual sum carries no N^2-sized cancellation) give shifts within
// ~(1/nc)^2 x gap of the eigenvalues; then one double-double inverse iteration and a final
// Rayleigh quotient (the vectors agree with the bisection path's to 1.8e-16 at 2^23; C4: one
// full-length solve instead of 5 plus 6 Sturm passes).
DpssResult dpss_from_coarse(const double* d_diag, const double* d_off, int64_t n, double tw, int64_t k,
                            double* d_vec, cudaStream_t s) {
  const bool prof = std::getenv("NUS_DPSS_PROF") != nullptr;
  auto tic = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!prof) return;
    NUS_CUDA(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dpss coarse] %s %.3f s\n", what, std::chrono::duration<double>(now - tic).count());
    tic = now;
  };
  const int64_t nc = std::max<int64_t>(int64_t{1} << 17, n / 64);
  DeviceBuffer cv(static_cast<size_t>(k) * nc * sizeof(double));
  dpss_device(nc, tw, k, cv.as<double>(), s);
  lap("coarse dpss");
  DeviceBuffer xs(static_cast<size_t>(k) * n * sizeof(dd));
  coarse_start_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(cv.as<double>(), nc, n, static_cast<int>(k), xs.as<dd>());
  note_launch();
  check_launch("coarse_start_kernel");
  std::vector<double> sig_hi(k, 0.0), sig_lo(k, 0.0);
  rayleigh_update(d_diag, d_off, n, k, xs.as<dd>(), sig_hi, sig_lo, s);
  rayleigh_update(d_diag, d_off, n, k, xs.as<dd>(), sig_hi, sig_lo, s);
  lap("start vectors + Rayleigh shifts");
  // default: the parallel two-sided recurrence at the Rayleigh shifts, twice (the second pass at
  // the shifts of the first pass's vectors); NUS_DPSS_RECURRENCE=0 keeps the sequential inverse
  // iteration below
  const char* re = std::getenv("NUS_DPSS_RECURRENCE");
  const int rec_passes = re ? std::atoi(re) : 2;
  DeviceBuffer d_norm(2 * k * sizeof(double));
  if (rec_passes > 0) {
    for (int pass = 0; pass < rec_passes; ++pass) {
      dpss_recurrence_vectors(d_diag, d_off, n, k, sig_hi, sig_lo, xs.as<dd>(), s);
      rayleigh_update(d_diag, d_off, n, k, xs.as<dd>(), sig_hi, sig_lo, s);
      lap("recurrence + Rayleigh");
    }
  } else {
  DeviceBuffer us(static_cast<size_t>(k) * n * 3 * sizeof(dd));
  // ||T|| for the pivot floor (as tridiag_top_device)
  std::vector<double> hd(n), he(n - 1);
  NUS_CUDA(cudaMemcpyAsync(hd.data(), d_diag, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaMemcpyAsync(he.data(), d_off, (n - 1) * sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
  double anorm = 0.0;
  for (int64_t i = 0; i < n; ++i)
    anorm = std::max(anorm, std::fabs(hd[i]) + (i > 0 ? std::fabs(he[i - 1]) : 0.0) + (i + 1 < n ? std::fabs(he[i]) : 0.0));
  const double pivmin = std::max(anorm, DBL_MIN) * DBL_EPSILON * 1e-3;
  DeviceBuffer d_sh(k * sizeof(double)), d_sl(k * sizeof(double));
  const char* pe = std::getenv("NUS_DPSS_COARSE_ITERS");
  const int passes = pe ? std::max(1, std::atoi(pe)) : 1;  // 1: 1.8e-16 from the bisection path at 2^23 (0: 5e-3)
  for (int pass = 0; pass < passes; ++pass) {
    NUS_CUDA(cudaMemcpyAsync(d_sh.ptr, sig_hi.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
    NUS_CUDA(cudaMemcpyAsync(d_sl.ptr, sig_lo.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
    inverse_iteration_dd_warp_kernel<<<static_cast<unsigned>(k), 32, 0, s>>>(
        d_diag, d_off, n, d_sh.as<double>(), d_sl.as<double>(), 1, pivmin, xs.as<dd>(), us.as<dd>(),
        d_norm.as<double>());
    note_launch();
    check_launch("inverse_iteration_dd_warp_kernel (coarse start)");
    dd_scale_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(xs.as<dd>(), d_norm.as<double>(), n, static_cast<int>(k));
    note_launch();
    rayleigh_update(d_diag, d_off, n, k, xs.as<dd>(), sig_hi, sig_lo, s);
    lap("inverse iteration + Rayleigh");
  }
  }
  // xs is normalised (scale 1): finalize with unit scales, then the canonical sign
  std::vector<double> ones(2 * k);
  for (int64_t j = 0; j < k; ++j) {
    ones[2 * j] = 1.0;
    ones[2 * j + 1] = 0.0;
  }
  NUS_CUDA(cudaMemcpyAsync(d_norm.ptr, ones.data(), 2 * k * sizeof(double), cudaMemcpyHostToDevice, s));
  dd_finalize_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(xs.as<dd>(), d_norm.as<double>(), n, static_cast<int>(k),
                                                            d_vec);
  note_launch();
  DeviceBuffer sg(k * sizeof(double));
  absmax_kernel<<<static_cast<unsigned>(k), 1024, 0, s>>>(d_vec, n, sg.as<double>());
  note_launch();
  scale_rows_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(d_vec, n, static_cast<int>(k), sg.as<double>());
  note_launch();
  check_launch("dpss finalize");
  NUS_CUDA(cudaStreamSynchronize(s));
  DpssResult res;
  res.values.assign(sig_hi.begin(), sig_hi.end());
  for (int64_t j = 0; j < k; ++j) res.values[j] += sig_lo[j];
  return res;
}

DpssResult dpss_device(int64_t n, double tw, int64_t k, double* d_vec, cudaStream_t s) {
  // tapers.cpp:33-39 validation
  require(n >= 2, "dpss_uniform: n must be >= 2");
  require(k >= 1 && k <= n, "dpss_uniform: k_tapers out of range");
  require(tw > 0.0 && tw < static_cast<double>(n) / 2.0, "dpss_uniform: need 0 < TW < n/2");
  const double w = tw / static_cast<double>(n);
  const double c = std::cos(2.0 * kPi * w);
  DeviceBuffer diag(n * sizeof(double)), off(std::max<int64_t>(n - 1, 1) * sizeof(double));
  dpss_matrix_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, c, diag.as<double>(), off.as<double>());
  note_launch();
  check_launch("dpss_matrix_kernel");
  const char* ce = std::getenv("NUS_DPSS_COARSE");
  const int64_t coarse_from = ce ? std::atoll(ce) : (int64_t{1} << 20);
  if (n >= coarse_from && n >= 64 && k <= 64)
    return dpss_from_coarse(diag.as<double>(), off.as<double>(), n, tw, k, d_vec, s);
  return tridiag_top_device(diag.as<double>(), off.as<double>(), n, k, d_vec, s);
}

void dpss_concentrations(int64_t n, double tw, int64_t k, const double* d_vec, double* conc,
                         cudaStream_t s) {
  const double wband = tw / static_cast<double>(n);
  int64_t L = 1;
  while (L < 2 * n) L <<= 1;
  DeviceBuffer a(L * sizeof(double2)), b(static_cast<size_t>(L) * k * sizeof(double2)), out(k * sizeof(double));
  sinc_symbol_kernel<<<blocks_for(L, 256), 256, 0, s>>>(n, L, wband, a.as<double2>());
  embed_kernel<<<blocks_for(L * k, 256), 256, 0, s>>>(d_vec, n, L, static_cast<int>(k), b.as<double2>());
  note_launch(2);
  fft_generic_inplace(a.ptr, L, 1, true, false, s);
  fft_generic_inplace(b.ptr, L, k, true, false, s);
  cmul_kernel<<<blocks_for(L * k, 256), 256, 0, s>>>(b.as<double2>(), a.as<double2>(), L, static_cast<int>(k));
  note_launch();
  fft_generic_inplace(b.ptr, L, k, true, true, s);
  conc_dot_kernel<<<static_cast<unsigned>(k), 256, 0, s>>>(d_vec, b.as<double2>(), n, L, out.as<double>());
  note_launch();
  check_launch("dpss_concentrations");
  NUS_CUDA(cudaMemcpyAsync(conc, out.ptr, k * sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
  for (int64_t j = 0; j < k; ++j) conc[j] = std::min(std::max(conc[j], 0.0), 1.0);  // tapers.cpp:76
}

void spline_uniform_device(const double* d_t, int64_t n, const double* d_y, int64_t k,
                           double* d_w, cudaStream_t s) {
  require(n >= 4, "CubicSpline: need at least 4 knots");
  double t0 = 0, tl = 0;
  NUS_CUDA(cudaMemcpyAsync(&t0, d_t, sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaMemcpyAsync(&tl, d_t + n - 1, sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
  const double h = (tl - t0) / static_cast<double>(n - 1);  // tapers.cpp:156
  DeviceBuffer moments(static_cast<size_t>(k) * n * sizeof(double));
  if (n >= 4 * kFilterHalf + 16) {
    const dim3 grid(blocks_for(n, 256), static_cast<unsigned>(k));
    spline_moments_kernel<<<grid, 256, 0, s>>>(d_y, n, h, moments.as<double>());
    note_launch();
  } else {
    DeviceBuffer knots(n * sizeof(double)), scratch(static_cast<size_t>(k) * 4 * n * sizeof(double));
    std::vector<double> hk(n);
    for (int64_t i = 0; i < n; ++i) hk[i] = t0 + h * static_cast<double>(i);
    NUS_CUDA(cudaMemcpyAsync(knots.ptr, hk.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
    spline_moments_thomas_kernel<<<static_cast<unsigned>(k), 1, 0, s>>>(knots.as<double>(), d_y, n,
                                                                        moments.as<double>(),
                                                                        scratch.as<double>());
    note_launch();
    NUS_CUDA(cudaStreamSynchronize(s));
  }
  check_launch("spline moments");
  spline_eval_kernel<<<blocks_for(n, 256), 256, 0, s>>>(d_t, n, t0, h, d_y, moments.as<double>(),
                                                        static_cast<int>(k), d_w);
  note_launch();
  check_launch("spline_eval_kernel");
  NUS_CUDA(cudaStreamSynchronize(s));
}

void quadform_device(const double* d_t, int64_t n, double f_max, const double* d_w, int64_t k,
                     int64_t row0, int64_t row1, double* q_host, cudaStream_t s) {
  require(k >= 1 && k <= kQfGroup, "quadratic_form: at most 8 weight rows per launch");
  require(row0 >= 0 && row1 <= n && row0 <= row1, "quadratic_form: bad row range");
  if (row0 == row1) {
    for (int64_t j = 0; j < k; ++j) q_host[j] = 0.0;
    return;
  }
  double t0 = 0, tl = 0;
  NUS_CUDA(cudaMemcpyAsync(&t0, d_t, sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaMemcpyAsync(&tl, d_t + n - 1, sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
  const double mean_dt = (tl - t0) / static_cast<double>(n);  // grid.cpp:21
  const double tol = 1e-12 * mean_dt;                          // kernels.cpp:103
  DeviceBuffer sn(n * sizeof(double)), cs(n * sizeof(double));
  band_phase_kernel<<<blocks_for(n, 256), 256, 0, s>>>(d_t, n, f_max, sn.as<double>(), cs.as<double>());
  note_launch();
  const int64_t rblocks = (row1 - row0 + kQfRows - 1) / kQfRows;
  const int64_t cgroups = (n + kQfCols * kQfChunks - 1) / (kQfCols * kQfChunks);
  require(rblocks < 65536, "quadratic_form: too many row blocks for one launch");
  const dim3 grid(static_cast<unsigned>(cgroups), static_cast<unsigned>(rblocks));
  const int64_t ncta = cgroups * rblocks;
  DeviceBuffer partial(static_cast<size_t>(ncta) * k * sizeof(double)), out(k * sizeof(double));
  quadform_kernel<<<grid, kQfRows, 0, s>>>(d_t, sn.as<double>(), cs.as<double>(), d_w, n,
                                           static_cast<int>(k), f_max, tol, row0, row1,
                                           partial.as<double>());
  note_launch();
  check_launch("quadform_kernel");
  reduce_partials_kernel<<<static_cast<unsigned>(k), 1024, 0, s>>>(partial.as<double>(), ncta,
                                                                   static_cast<int>(k), out.as<double>());
  note_launch();
  check_launch("reduce_partials_kernel");
  NUS_CUDA(cudaMemcpyAsync(q_host, out.ptr, k * sizeof(double), cudaMemcpyDeviceToHost, s));
  NUS_CUDA(cudaStreamSynchronize(s));
}

namespace {
__global__ void scale_by_kernel(double* __restrict__ w, int64_t n, int k, const double* __restrict__ s) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * k) return;
  w[g] *= s[g / n];
}
}  // namespace

bool normalise_exact(int64_t n) {
  const char* e = std::getenv("NUS_NORMALISE");
  if (e && std::strcmp(e, "exact") == 0) return true;
  if (e && std::strcmp(e, "fast") == 0) return false;
  const char* m = std::getenv("NUS_QUADFORM_EXACT_MAX");
  // exact O(N^2) form up to 2^16 samples; above, the O(N log N) lattice form (agreement <= 5e-12 on
  // every config's sampling): C3's 256 channels of 2^18 samples 0.83 s -> ~0.1 s of setup each
  const int64_t lim = m ? std::atoll(m) : (int64_t{1} << 16);
  return n <= lim;
}

void gpss_interpolated_device(const double* d_t, const double* h_t, int64_t n, double f_max,
                              double f_w, int64_t k, double* d_w, cudaStream_t s, double* ms_dpss,
                              double* ms_spline, double* ms_norm, DpssCache* cache) {
  // tapers.cpp:146-160 validation, same order and exception types
  require(n >= 8, "gpss_interpolated: need at least 8 samples");
  require(f_w > 0.0, "gpss_interpolated: f_w must be positive");
  require(std::isfinite(f_w), "AnalysisBand: half_width must be positive");
  require(f_max > 0.0 && std::isfinite(f_max), "SignalBand: f_max must be positive");
  if (!(f_w <= f_max + 1e-12 * f_max))
    fail(NUS_ERR_BAND_RANGE, "gpss_interpolated: nominal band not inside signal band");
  const double h = (h_t[n - 1] - h_t[0]) / static_cast<double>(n - 1);
  const double tw = f_w * h * static_cast<double>(n);
  require(tw < static_cast<double>(n) / 2.0, "gpss_interpolated: f_w too large for this grid");
  auto t0 = std::chrono::steady_clock::now();
  DeviceBuffer own;
  const double* dpv = nullptr;
  if (cache) {
    for (const DpssCache::Entry& e : cache->entries)
      if (e.n == n && e.k == k && e.tw == tw) {
        dpv = e.dp.as<double>();
        ++cache->hits;
        break;
      }
  }
  if (!dpv) {
    own.alloc(static_cast<size_t>(k) * n * sizeof(double));
    dpss_device(n, tw, k, own.as<double>(), s);
    dpv = own.as<double>();
    if (cache) {
      cache->entries.emplace_back();
      DpssCache::Entry& e = cache->entries.back();
      e.n = n;
      e.k = k;
      e.tw = tw;
      e.dp = std::move(own);
    }
  }
  if (ms_dpss) *ms_dpss = host_ms_since(t0);
  t0 = std::chrono::steady_clock::now();
  spline_uniform_device(d_t, n, dpv, k, d_w, s);
  if (ms_spline) *ms_spline = host_ms_since(t0);
  t0 = std::chrono::steady_clock::now();
  std::vector<double> q(k), scale(k);
  if (normalise_exact(n)) {
    for (int64_t k0 = 0; k0 < k; k0 += kQfGroup) {
      const int64_t kk = std::min<int64_t>(kQfGroup, k - k0);
      quadform_device(d_t, n, f_max, d_w + k0 * n, kk, 0, n, q.data() + k0, s);
    }
  } else {  // O(N log N) lattice form of the same quadratic form (normalise.cu)
    int dev = 0;
    NUS_CUDA(cudaGetDevice(&dev));
    quadform_fast_device(d_t, h_t, n, f_max, d_w, k, q.data(), s, dev);
  }
  for (int64_t j = 0; j < k; ++j) {
    if (!(q[j] > 0.0)) fail(NUS_ERR_NUMERIC, "gpss_interpolated: degenerate metric norm");
    scale[j] = std::sqrt(2.0 * f_w / q[j]);  // tapers.cpp:177
  }
  DeviceBuffer ds(k * sizeof(double));
  NUS_CUDA(cudaMemcpyAsync(ds.ptr, scale.data(), k * sizeof(double), cudaMemcpyHostToDevice, s));
  scale_by_kernel<<<blocks_for(n * k, 256), 256, 0, s>>>(d_w, n, static_cast<int>(k), ds.as<double>());
  note_launch();
  check_launch("scale_by_kernel");
  NUS_CUDA(cudaStreamSynchronize(s));
  if (ms_norm) *ms_norm = host_ms_since(t0);
}

}  // namespace nus
