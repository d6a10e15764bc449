// MTNUFFT0 tapers: the exact nominal-band GPSS by the dense generalized
// Hermitian eigenproblem R(A) w = lambda R(B) w, on the device.
//
// Reference: generalized_hermitian_eigen (src/eig.cpp:612-659; cholesky_with_ridge :485-500,
// reduced_matrix :515-537, enforce_spectral_range :539-548, canonical_phase :291-300) and
// gpss_exact (src/tapers.cpp:118-144), kernels signal_band_kernel / analysis_band_kernel
// (src/kernels.cpp:100-153).  Library dense linear algebra (cuSOLVER potrf + syevdx/heevdx,
// cuBLAS trsm/gemm) replaces the reference's Householder + implicit-QL solver; the kernel
// matrices are built on the device with the reference's entry formulas.  Dense O(N^2) memory
// and O(N^3) work: the reference itself limits this path to N <~ 2^15.
//
// All matrices are column-major n x n.  A Hermitian (real when the band is centred at 0),
// M real symmetric positive definite.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "nus_internal.cuh"

namespace nus {

namespace {

#define NUS_CUSOLVER(x)                                                                            \
  do {                                                                                             \
    const cusolverStatus_t st_ = (x);                                                              \
    if (st_ != CUSOLVER_STATUS_SUCCESS) fail(NUS_ERR_CUDA, std::string("cusolver: ") + #x);        \
  } while (0)
#define NUS_CUBLAS(x)                                                                              \
  do {                                                                                             \
    const cublasStatus_t st_ = (x);                                                                \
    if (st_ != CUBLAS_STATUS_SUCCESS) fail(NUS_ERR_CUDA, std::string("cublas: ") + #x);            \
  } while (0)

struct Handles {
  cusolverDnHandle_t sol = nullptr;
  cublasHandle_t blas = nullptr;
  cudaStream_t s = nullptr;
  Handles() {
    NUS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    NUS_CUSOLVER(cusolverDnCreate(&sol));
    NUS_CUSOLVER(cusolverDnSetStream(sol, s));
    NUS_CUBLAS(cublasCreate(&blas));
    NUS_CUBLAS(cublasSetStream(blas, s));
  }
  ~Handles() {
    if (blas) cublasDestroy(blas);
    if (sol) cusolverDnDestroy(sol);
    if (s) cudaStreamDestroy(s);
  }
};

constexpr double kPi = 3.14159265358979323846;

// band_sinc (kernels.cpp:15-18) times e^{2 pi i fc d}: entry (r, c), d = t_r - t_c, stored at r + c n
__global__ void band_matrix_kernel(const double* __restrict__ t, int64_t n, double f, double fc, double tol,
                                   double* __restrict__ re, double* __restrict__ im) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * n) return;
  const int64_t r = g % n, c = g / n;
  if (r == c) {
    re[g] = 2.0 * f;
    if (im) im[g] = 0.0;
    return;
  }
  const double d = t[r] - t[c];
  const double env = fabs(d) < tol ? 2.0 * f : sin(2.0 * kPi * f * d) / (kPi * d);
  if (!im) {
    re[g] = env;
    return;
  }
  double sn, cs;
  sincos(2.0 * kPi * fc * d, &sn, &cs);
  re[g] = env * cs;
  im[g] = env * sn;
}

__global__ void add_diag_kernel(double* a, int64_t n, double v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) a[i + i * n] += v;
}

// C <- (C + C^H) / 2 with a real diagonal (reduced_matrix, eig.cpp:527-535); interleave into z
__global__ void hermitize_kernel(const double* __restrict__ cre, const double* __restrict__ cim, int64_t n,
                                 double2* __restrict__ z, double* __restrict__ dre) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= n * n) return;
  const int64_t r = g % n, c = g / n, gt = c + r * n;
  const double vr = 0.5 * (cre[g] + cre[gt]);
  const double vi = cim ? (r == c ? 0.0 : 0.5 * (cim[g] - cim[gt])) : 0.0;
  if (z) z[g] = double2{vr, vi};
  if (dre) dre[g] = vr;
}

template <class F>
void for_ridges(double r1, double r2, F&& try_factor) {
  for (const double f : {r1, r2})
    if (try_factor(f)) return;
  fail(NUS_ERR_CONDITIONING,
       "generalized_hermitian_eigen: metric matrix not positive definite after ridge regularization");
}

unsigned blocks(int64_t count, int threads) { return static_cast<unsigned>((count + threads - 1) / threads); }

}  // namespace

// Dense band kernel, row-major, on the device: entry (r, c) = env(t_r - t_c) e^{2 pi i fc (t_r - t_c)}
// (kernels.cpp:100-153).  The column-major fill with -fc is exactly the row-major matrix.
void band_matrix_rowmajor(const double* d_t, int64_t n, double f, double fc, double tol, double* d_re,
                          double* d_im) {
  const int64_t nn = n * n;
  band_matrix_kernel<<<blocks(nn, 256), 256>>>(d_t, n, f, -fc, tol, d_re, d_im);
  note_launch();
  check_launch("band_matrix_kernel");
}

// Solves on device copies of A (re, im nullable) and M; outputs on the host.
void generalized_eigen_device(const double* d_are, const double* d_aim, const double* d_m, int64_t n, int64_t k,
                              double ridge_first, double ridge_retry, bool want_vectors, double* values,
                              double* vectors /* [k][n] complex, row per pair */, double* residuals) {
  require(n >= 1, "generalized_hermitian_eigen: empty pencil");
  require(k >= 1, "generalized_hermitian_eigen: k_top must be >= 1");
  k = std::min(k, n);
  Handles h;
  const bool cplx = d_aim != nullptr;
  const size_t nn = static_cast<size_t>(n) * n;
  // trace(M) / n (eig.cpp:487)
  std::vector<double> diag(n);
  NUS_CUDA(cudaMemcpy2DAsync(diag.data(), sizeof(double), d_m, (n + 1) * sizeof(double), sizeof(double), n,
                             cudaMemcpyDeviceToHost, h.s));
  NUS_CUDA(cudaStreamSynchronize(h.s));
  double tr = 0.0;
  for (double v : diag) tr += v;
  const double unit = tr / static_cast<double>(n);

  // Cholesky with ridge: L L^T = M + ridge * unit * I
  DeviceBuffer L(nn * sizeof(double)), info(sizeof(int));
  int lwork = 0;
  NUS_CUSOLVER(cusolverDnDpotrf_bufferSize(h.sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), L.as<double>(),
                                           static_cast<int>(n), &lwork));
  DeviceBuffer work(static_cast<size_t>(std::max(lwork, 1)) * sizeof(double));
  for_ridges(ridge_first, ridge_retry, [&](double f) {
    NUS_CUDA(cudaMemcpyAsync(L.ptr, d_m, nn * sizeof(double), cudaMemcpyDeviceToDevice, h.s));
    add_diag_kernel<<<blocks(n, 256), 256, 0, h.s>>>(L.as<double>(), n, f * unit);
    note_launch();
    NUS_CUSOLVER(cusolverDnDpotrf(h.sol, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n), L.as<double>(),
                                  static_cast<int>(n), work.as<double>(), lwork, info.as<int>()));
    int hinfo = 0;
    NUS_CUDA(cudaMemcpyAsync(&hinfo, info.ptr, sizeof(int), cudaMemcpyDeviceToHost, h.s));
    NUS_CUDA(cudaStreamSynchronize(h.s));
    return hinfo == 0;
  });

  // C = L^{-1} A L^{-T}, real and imaginary parts separately (L is real)
  const double one = 1.0;
  DeviceBuffer cre(nn * sizeof(double)), cim(cplx ? nn * sizeof(double) : 0);
  auto reduce = [&](const double* src, DeviceBuffer& dst) {
    NUS_CUDA(cudaMemcpyAsync(dst.ptr, src, nn * sizeof(double), cudaMemcpyDeviceToDevice, h.s));
    NUS_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                           static_cast<int>(n), static_cast<int>(n), &one, L.as<double>(), static_cast<int>(n),
                           dst.as<double>(), static_cast<int>(n)));
    NUS_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                           static_cast<int>(n), static_cast<int>(n), &one, L.as<double>(), static_cast<int>(n),
                           dst.as<double>(), static_cast<int>(n)));
  };
  reduce(d_are, cre);
  if (cplx) reduce(d_aim, cim);

  // dense Hermitian eigenproblem, the k largest (ascending from cuSOLVER)
  const int il = static_cast<int>(n - k + 1), iu = static_cast<int>(n);
  int meig = 0;
  std::vector<double> w_asc(n);
  DeviceBuffer dW(n * sizeof(double));
  DeviceBuffer Y;  // eigenvectors of C (first k columns), complex or real
  const cusolverEigMode_t jobz = want_vectors ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
  if (cplx) {
    Y.alloc(nn * sizeof(double2));
    hermitize_kernel<<<blocks(static_cast<int64_t>(nn), 256), 256, 0, h.s>>>(cre.as<double>(), cim.as<double>(),
                                                                            n, Y.as<double2>(), nullptr);
    note_launch();
    NUS_CUSOLVER(cusolverDnZheevdx_bufferSize(h.sol, jobz, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER,
                                              static_cast<int>(n), Y.as<cuDoubleComplex>(), static_cast<int>(n), 0.0,
                                              0.0, il, iu, &meig, dW.as<double>(), &lwork));
    DeviceBuffer zw(static_cast<size_t>(std::max(lwork, 1)) * sizeof(double2));
    NUS_CUSOLVER(cusolverDnZheevdx(h.sol, jobz, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n),
                                   Y.as<cuDoubleComplex>(), static_cast<int>(n), 0.0, 0.0, il, iu, &meig,
                                   dW.as<double>(), zw.as<cuDoubleComplex>(), lwork, info.as<int>()));
    NUS_CUDA(cudaStreamSynchronize(h.s));
  } else {
    Y.alloc(nn * sizeof(double));
    hermitize_kernel<<<blocks(static_cast<int64_t>(nn), 256), 256, 0, h.s>>>(cre.as<double>(), nullptr, n,
                                                                            nullptr, Y.as<double>());
    note_launch();
    NUS_CUSOLVER(cusolverDnDsyevdx_bufferSize(h.sol, jobz, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER,
                                              static_cast<int>(n), Y.as<double>(), static_cast<int>(n), 0.0, 0.0, il,
                                              iu, &meig, dW.as<double>(), &lwork));
    DeviceBuffer dw(static_cast<size_t>(std::max(lwork, 1)) * sizeof(double));
    NUS_CUSOLVER(cusolverDnDsyevdx(h.sol, jobz, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, static_cast<int>(n),
                                   Y.as<double>(), static_cast<int>(n), 0.0, 0.0, il, iu, &meig, dW.as<double>(),
                                   dw.as<double>(), lwork, info.as<int>()));
    NUS_CUDA(cudaStreamSynchronize(h.s));
  }
  int hinfo = 0;
  NUS_CUDA(cudaMemcpy(&hinfo, info.ptr, sizeof(int), cudaMemcpyDeviceToHost));
  if (hinfo != 0 || meig != k) fail(NUS_ERR_NUMERIC, "generalized_hermitian_eigen: dense eigensolver failed");
  NUS_CUDA(cudaMemcpy(w_asc.data(), dW.ptr, k * sizeof(double), cudaMemcpyDeviceToHost));
  // descending, range-checked and clamped into [0, 1] (eig.cpp:539-548)
  for (int64_t j = 0; j < k; ++j) {
    double v = w_asc[k - 1 - j];
    if (v < -1e-6 || v > 1.0 + 1e-6)
      fail(NUS_ERR_SPECTRAL_RANGE, "generalized eigenvalue outside [0,1] beyond tolerance: " + std::to_string(v));
    values[j] = std::min(std::max(v, 0.0), 1.0);
  }
  if (!want_vectors) return;

  // w = L^{-T} y for the k selected columns (descending order), re and im parts
  DeviceBuffer wre(static_cast<size_t>(n) * k * sizeof(double)), wim(static_cast<size_t>(n) * k * sizeof(double));
  {
    std::vector<double> hy(static_cast<size_t>(n) * k * (cplx ? 2 : 1));
    NUS_CUDA(cudaMemcpy(hy.data(), Y.ptr, hy.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<double> hre(static_cast<size_t>(n) * k), him(static_cast<size_t>(n) * k, 0.0);
    for (int64_t j = 0; j < k; ++j) {
      const int64_t src = k - 1 - j;  // column of the j-th largest
      for (int64_t i = 0; i < n; ++i) {
        if (cplx) {
          hre[j * n + i] = hy[2 * (src * n + i)];
          him[j * n + i] = hy[2 * (src * n + i) + 1];
        } else {
          hre[j * n + i] = hy[src * n + i];
        }
      }
    }
    NUS_CUDA(cudaMemcpy(wre.ptr, hre.data(), hre.size() * sizeof(double), cudaMemcpyHostToDevice));
    NUS_CUDA(cudaMemcpy(wim.ptr, him.data(), him.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  for (DeviceBuffer* b : {&wre, &wim})
    NUS_CUBLAS(cublasDtrsm(h.blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                           static_cast<int>(n), static_cast<int>(k), &one, L.as<double>(), static_cast<int>(n),
                           b->as<double>(), static_cast<int>(n)));
  // M w and A w (A = Are + i Aim): (Are wre - Aim wim) + i (Are wim + Aim wre)
  const double zero = 0.0, mone = -1.0;
  DeviceBuffer mwr(static_cast<size_t>(n) * k * sizeof(double)), mwi(static_cast<size_t>(n) * k * sizeof(double));
  DeviceBuffer awr(static_cast<size_t>(n) * k * sizeof(double)), awi(static_cast<size_t>(n) * k * sizeof(double));
  auto gemm = [&](const double* a, const DeviceBuffer& x, double beta, DeviceBuffer& y, double alpha) {
    NUS_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(k),
                           static_cast<int>(n), &alpha, a, static_cast<int>(n), x.as<double>(), static_cast<int>(n),
                           &beta, y.as<double>(), static_cast<int>(n)));
  };
  gemm(d_m, wre, zero, mwr, one);
  gemm(d_m, wim, zero, mwi, one);
  gemm(d_are, wre, zero, awr, one);
  gemm(d_are, wim, zero, awi, one);
  if (cplx) {
    gemm(d_aim, wim, one, awr, mone);
    gemm(d_aim, wre, one, awi, one);
  }
  double afro2 = 0.0;
  {
    double v = 0.0;
    NUS_CUBLAS(cublasDnrm2(h.blas, static_cast<int>(nn), d_are, 1, &v));
    afro2 += v * v;
    if (cplx) {
      NUS_CUBLAS(cublasDnrm2(h.blas, static_cast<int>(nn), d_aim, 1, &v));
      afro2 += v * v;
    }
  }
  const size_t nk = static_cast<size_t>(n) * k;
  std::vector<double> hwr(nk), hwi(nk), hmr(nk), hmi(nk), har(nk), hai(nk);
  NUS_CUDA(cudaStreamSynchronize(h.s));
  NUS_CUDA(cudaMemcpy(hwr.data(), wre.ptr, nk * sizeof(double), cudaMemcpyDeviceToHost));
  NUS_CUDA(cudaMemcpy(hwi.data(), wim.ptr, nk * sizeof(double), cudaMemcpyDeviceToHost));
  NUS_CUDA(cudaMemcpy(hmr.data(), mwr.ptr, nk * sizeof(double), cudaMemcpyDeviceToHost));
  NUS_CUDA(cudaMemcpy(hmi.data(), mwi.ptr, nk * sizeof(double), cudaMemcpyDeviceToHost));
  NUS_CUDA(cudaMemcpy(har.data(), awr.ptr, nk * sizeof(double), cudaMemcpyDeviceToHost));
  NUS_CUDA(cudaMemcpy(hai.data(), awi.ptr, nk * sizeof(double), cudaMemcpyDeviceToHost));
  const double anorm = std::sqrt(afro2);
  for (int64_t j = 0; j < k; ++j) {
    const size_t o = static_cast<size_t>(j) * n;
    // metric norm w^H M w (M real symmetric): sum conj(w) (M w), real part
    double q = 0.0;
    for (int64_t i = 0; i < n; ++i) q += hwr[o + i] * hmr[o + i] + hwi[o + i] * hmi[o + i];
    const double inv = q > 0.0 ? 1.0 / std::sqrt(q) : 1.0;
    // canonical_phase (eig.cpp:291-300): the first entry of largest |w|^2 made real positive;
    // final w = w_raw * c with c = inv * conj(w_imax) / |w_imax|
    int64_t imax = 0;
    double best = hwr[o] * hwr[o] + hwi[o] * hwi[o];
    for (int64_t i = 1; i < n; ++i) {
      const double m2 = hwr[o + i] * hwr[o + i] + hwi[o + i] * hwi[o + i];
      if (m2 > best) {
        best = m2;
        imax = i;
      }
    }
    double sr = inv, si = 0.0;
    if (best > 0.0) {
      const double mag = std::sqrt(best);
      sr = inv * hwr[o + imax] / mag;
      si = -inv * hwi[o + imax] / mag;
    }
    // residual || A w - lambda M w || / (||A||_F ||w||) with the final w (eig.cpp:641-655)
    const double lam = w_asc[k - 1 - j];  // unclamped value, as the reference
    double r2 = 0.0, w2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double rr = har[o + i] - lam * hmr[o + i], ri = hai[o + i] - lam * hmi[o + i];
      r2 += (rr * rr + ri * ri) * (sr * sr + si * si);
      const double xr = hwr[o + i] * sr - hwi[o + i] * si, xi = hwr[o + i] * si + hwi[o + i] * sr;
      w2 += xr * xr + xi * xi;
      vectors[2 * (o + i)] = xr;
      vectors[2 * (o + i) + 1] = xi;
    }
    residuals[j] = std::sqrt(r2) / (anorm * std::sqrt(w2));
  }
}

// gpss_exact (tapers.cpp:118-144): kernels from the times on the device, GEP, then each
// vector scaled to w^H R(B) w = 2 f_w.  Output: weights [k][n] complex, concentrations [k].
void gpss_exact_device(const double* h_t, int64_t n, double f_max, double f_c, double f_w, int64_t k,
                       double ridge_first, double ridge_retry, double* w_out, double* conc) {
  if (!(f_c + f_w <= f_max + 1e-12 * f_max))  // band_inside (tapers.cpp:18-21)
    fail(NUS_ERR_BAND_RANGE, "gpss_exact: analysis band not inside signal band");
  require(k >= 1 && k <= n, "gpss_exact: k_tapers out of range");
  const double mean_dt = (h_t[n - 1] - h_t[0]) / static_cast<double>(n);  // grid.cpp:21
  const double tol = 1e-12 * mean_dt;
  const size_t nn = static_cast<size_t>(n) * n;
  DeviceBuffer dt(n * sizeof(double)), M(nn * sizeof(double)), Are(nn * sizeof(double));
  DeviceBuffer Aim(f_c != 0.0 ? nn * sizeof(double) : 0);
  NUS_CUDA(cudaMemcpy(dt.ptr, h_t, n * sizeof(double), cudaMemcpyHostToDevice));
  band_matrix_kernel<<<blocks(static_cast<int64_t>(nn), 256), 256>>>(dt.as<double>(), n, f_max, 0.0, tol,
                                                                     M.as<double>(), nullptr);
  note_launch();
  band_matrix_kernel<<<blocks(static_cast<int64_t>(nn), 256), 256>>>(dt.as<double>(), n, f_w, f_c, tol,
                                                                     Are.as<double>(),
                                                                     f_c != 0.0 ? Aim.as<double>() : nullptr);
  note_launch();
  check_launch("band_matrix_kernel");
  NUS_CUDA(cudaDeviceSynchronize());
  std::vector<double> vec(2 * static_cast<size_t>(k) * n), res(k);
  generalized_eigen_device(Are.as<double>(), f_c != 0.0 ? Aim.as<double>() : nullptr, M.as<double>(), n, k,
                           ridge_first, ridge_retry, true, conc, vec.data(), res.data());
  // w^H R(B) w of the metric-normalised vectors (about 1) and the taper scale sqrt(2 f_w / q)
  DeviceBuffer wr(static_cast<size_t>(n) * k * sizeof(double)), wi(static_cast<size_t>(n) * k * sizeof(double));
  DeviceBuffer mr(static_cast<size_t>(n) * k * sizeof(double)), mi(static_cast<size_t>(n) * k * sizeof(double));
  std::vector<double> hre(static_cast<size_t>(n) * k), him(static_cast<size_t>(n) * k);
  for (size_t i = 0; i < hre.size(); ++i) {
    hre[i] = vec[2 * i];
    him[i] = vec[2 * i + 1];
  }
  NUS_CUDA(cudaMemcpy(wr.ptr, hre.data(), hre.size() * sizeof(double), cudaMemcpyHostToDevice));
  NUS_CUDA(cudaMemcpy(wi.ptr, him.data(), him.size() * sizeof(double), cudaMemcpyHostToDevice));
  {
    Handles h;
    const double one = 1.0, zero = 0.0;
    NUS_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(k),
                           static_cast<int>(n), &one, M.as<double>(), static_cast<int>(n), wr.as<double>(),
                           static_cast<int>(n), &zero, mr.as<double>(), static_cast<int>(n)));
    NUS_CUBLAS(cublasDgemm(h.blas, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), static_cast<int>(k),
                           static_cast<int>(n), &one, M.as<double>(), static_cast<int>(n), wi.as<double>(),
                           static_cast<int>(n), &zero, mi.as<double>(), static_cast<int>(n)));
    NUS_CUDA(cudaStreamSynchronize(h.s));
  }
  std::vector<double> hmr(hre.size()), hmi(him.size());
  NUS_CUDA(cudaMemcpy(hmr.data(), mr.ptr, hmr.size() * sizeof(double), cudaMemcpyDeviceToHost));
  NUS_CUDA(cudaMemcpy(hmi.data(), mi.ptr, hmi.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t j = 0; j < k; ++j) {
    double q = 0.0;
    for (int64_t i = 0; i < n; ++i) q += hre[j * n + i] * hmr[j * n + i] + him[j * n + i] * hmi[j * n + i];
    if (!(q > 0.0)) fail(NUS_ERR_NUMERIC, "gpss_exact: degenerate metric norm");
    const double s = std::sqrt(2.0 * f_w / q);
    for (int64_t i = 0; i < n; ++i) {
      w_out[2 * (j * n + i)] = hre[j * n + i] * s;
      w_out[2 * (j * n + i) + 1] = him[j * n + i] * s;
    }
  }
}

}  // namespace nus
