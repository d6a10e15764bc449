"""GPU parity at the BASELINE configs' FULL sizes against the live reference (Oracle-B).

Oracle-B is the reference library itself (oracle/_ref/libnusref.so, compiled from
/root/reference/proj/src): its NufftPlan + eigencoefficients + power loop
(nufft.cpp:56-227, estimators.cpp:106-122) fed the GPU's normalised tapers, the K tapers of one
series on the box's host threads (bit-identical to the serial loop).  The reference's own taper
setup is O(N^2) (hours at these N), so the taper stage is checked separately against the
long-double restatement (oracle/nus_oracle.c: bisection + inverse iteration on the matrix of
tapers.cpp:40-52, then the not-a-knot spline of eig.cpp:671-745).

Tolerances (BASELINE.json north_star): relL2(P) <= 1e-6 in fp64 at eps = 1e-9, <= 1e-4 in fp32;
bins and the sample sort bit-exact.  The C5 lattice uses max(10 eps, 1e-9) in fp64 and
max(10 eps, 1e-4) in fp32 (the transform contract is eps ||y||_1; at eps = 1e-12 the two windows'
fp64 rounding floors -- C5's f t reaches 1e6 -- sit near 1e-10).
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from conftest import rel_l2, sign_align
from oracle import C, Injected, ref_available

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = max(1, min(os.cpu_count() or 1, 16))


def _need_ref():
    if not ref_available():
        pytest.skip("oracle/_ref (the compiled reference) is not built")


def _shape_check(w, t, nw, k, tol_dpss, threads=THREADS):
    """Taper stage in three links, each against an independent computation:
    (1) the GPU DPSS (double-double inverse iteration) against the long-double bisection + inverse
        iteration restatement (tapers.cpp:40-52 matrix), absolute on unit vectors -- the long-double
        solve carries ~eps_ld ||T|| / gap ~ 1e-19 N^2 / 50 of rounding, so its agreement with the
        double-double vectors is ~1e-11 at 2^24 and ~7e-11 at 2^26 (tol_dpss);
    (2) the GPU spline of those DPSS rows against the C not-a-knot spline (eig.cpp:671-745) at the
        sample times, relative to the taper's peak (1e-12);
    (3) the estimator's tapers = (2) up to the R(B) scale (checked separately)."""
    n = t.size
    h = (t[-1] - t[0]) / (n - 1)
    dg = nus.dpss_uniform(n, nw, k, concentrations=False).tapers  # tw = f_w h N = NW by construction
    dp, _ = C.dpss(n, nw, k, threads=threads)
    err_dpss = float(np.abs(sign_align(dg, dp) - dp).max())
    assert err_dpss < tol_dpss, err_dpss
    knots = t[0] + h * np.arange(n)
    worst = 0.0
    for j in range(k):
        r = C.spline(knots, dg[j], t)
        r /= np.linalg.norm(r)
        g = w[j] / np.linalg.norm(w[j])
        g = g * np.sign(np.dot(g, r))
        worst = max(worst, float(np.abs(g - r).max() / np.abs(r).max()))
    assert worst < 1e-12, worst
    return err_dpss, worst


@pytest.mark.parametrize("kern", ["es"])
def test_c3_256x2e18_channels_fp32_vs_reference(kern):
    """C3: 256 channels x N = 2^18 (fp32, eps 1e-5, NW 5, K 9, I = 2^17 -> Mr = 2^18: the own two-pass
    FFT, the nine tapers as two streaming spread launches), each channel with its own gaps and its own f_w, against the
    reference per channel (host threads across channels)."""
    _need_ref()
    wl = W.c3(channels=256)
    est = nus.api._Estimator(wl.times, wl.centers, wl.f_max, wl.f_w, wl.k, wl.eps, 1, "f32", 0)
    assert est.info.mr == 1 << 18
    # K = 9 in fp32: two streaming spread launches (8 + 1 tapers)
    assert est.stage_kernels() == ["spread_stream_kernel", "fft_cols_blk_kernel", "fft_rows_crop_kernel"]
    p = est.power(wl.values)
    w = est.tapers()

    def ref(c):
        h = Injected(wl.times[c], w[c], wl.centers, wl.eps, wl.f_max, float(wl.f_w[c]), policy=1)
        try:
            return h.power(wl.values[c])
        finally:
            h.close()

    with ThreadPoolExecutor(THREADS) as ex:
        refs = list(ex.map(ref, range(wl.channels)))
    errs = [rel_l2(p[c], refs[c]) for c in range(wl.channels)]
    print(f"C3 256 channels: max relL2(P) = {max(errs):.3e}")
    assert max(errs) <= 1e-4
    # every channel's tapers were built on its own grid with its own half-bandwidth
    for c in (0, 97, 255):
        _shape_check(w[c], wl.times[c], 5.0, 9, 1e-12)
        q = nus.signal_band_quadform_fast(nus.SamplingGrid(wl.times[c]), nus.SignalBand(wl.f_max), w[c])
        np.testing.assert_allclose(q, 2 * wl.f_w[c], rtol=1e-9)


@pytest.mark.parametrize("kern", ["es"])
def test_c4_full_2e26_vs_reference(kern):
    """C4 at full size: N = 2^26 clustered samples, I = 2^24 dyadic centres (Mr = 2^25: 8192-element
    tiles and rows), NW 8, K 15, eps 1e-9, fp64.  GPU setup (coarse-start DPSS at 2^26, spline,
    O(N log N) normalisation) + spectrum; P against the reference's NufftPlan + power loop with the
    same tapers; bins and sort bit-exact against the restatement; the taper shapes against the
    long-double DPSS + spline at 2^26."""
    _need_ref()
    wl = W.c4()
    g = nus.SamplingGrid(wl.times)
    plan = nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max)
    est = nus.MtnufftEstimator(g, nus.SignalBand(wl.f_max), plan,
                               nus.MtnufftEstimator.Options(k_tapers=15, epsilon=1e-9))
    assert est.transform_info().mr == 1 << 25
    p = est.estimate(wl.values).power
    w = est.tapers().weights_matrix()
    del est
    h = Injected(wl.times, w, wl.centers, 1e-9, wl.f_max, float(wl.f_w[0]), policy=1)
    try:
        pref = h.power_tapers(wl.values, min(THREADS, 8))
    finally:
        h.close()
    err = rel_l2(p, pref)
    print(f"C4 full: relL2(P) = {err:.3e}")
    assert err <= 1e-6
    # bins (nufft.cpp:118-122) and the stable start-cell sort, bit-exact at 2^26
    with nus.spread_kernel("gaussian"):
        bp = nus.NufftPlan(g, wl.centers, 1e-9, nus.NufftPathPolicy.force_fast)
    j0 = bp.first_cells()
    assert np.array_equal(j0, C.first_cells(wl.times, wl.centers, 1e-9))
    assert np.array_equal(bp.sort_order(), np.argsort(np.mod(j0, bp.grid_size()), kind="stable"))
    del bp
    e_dpss, e_shape = _shape_check(w, wl.times, 8.0, 15, 2e-10, threads=15)
    print(f"C4 full: DPSS vs long double {e_dpss:.3e} (unit vectors), tapers vs C spline {e_shape:.3e}")


@pytest.mark.parametrize("kern", ["es"])
def test_c5_2e22_eps_k_precision_lattice_vs_reference(kern):
    """C5 at full size: N = 2^22 jittered samples, I = 2^21; eps in {1e-3, 1e-6, 1e-9, 1e-12} x
    K in {1, 3, 7, 15, 31} (NW = (K+1)/2) x {fp32, fp64}, every point against the reference
    transform at the same eps with the same tapers (not GPU against GPU)."""
    _need_ref()
    base = W.c5()
    t, x, c = base.times, base.values, base.centers
    g = nus.SamplingGrid(t)
    ks = (1, 3, 7, 15, 31)
    tapers, fws = {}, {}
    for k in ks:
        nw = (k + 1) / 2.0
        fw = W.half_width_for(t, nw)
        plan = nus.BandPlan.from_centers(c, fw, base.f_max)
        est = nus.MtnufftEstimator(g, nus.SignalBand(base.f_max), plan,
                                   nus.MtnufftEstimator.Options(k_tapers=k, epsilon=1e-9))
        tapers[k], fws[k] = est.tapers().weights_matrix(), fw
        del est
    allw = np.concatenate([tapers[k] for k in ks])
    offs = np.cumsum((0,) + ks)
    worst = {}
    for eps in (1e-3, 1e-6, 1e-9, 1e-12):
        h = Injected(t, allw, c, eps, base.f_max, fws[7], policy=1)
        try:
            pk = h.taper_powers(x, THREADS)
        finally:
            h.close()
        for i, k in enumerate(ks):
            pref = np.zeros(c.size)
            for j in range(offs[i], offs[i + 1]):  # the reference's k-outer accumulation order
                pref += pk[j]
            pref /= k
            for prec in ("f64", "f32"):
                e = nus.api._Estimator(t, c, base.f_max, fws[k], k, eps, 1, prec, 0, tapers=tapers[k])
                pw = e.power(x)[0]
                del e
                err = rel_l2(pw, pref)
                worst[(eps, k, prec)] = err
    print("C5 lattice relL2(P) vs reference:", {f"{e:g}/K{k}/{p}": f"{v:.2e}" for (e, k, p), v in worst.items()})
    for (eps, k, prec), err in worst.items():
        tol = max(10 * eps, 1e-9) if prec == "f64" else max(10 * eps, 1e-4)
        assert err <= tol, (eps, k, prec, err)
    # the spec's anchor point
    assert max(v for (e, k, p), v in worst.items() if e == 1e-9 and p == "f64") <= 1e-6


@pytest.mark.parametrize("lg", [23, 24])
def test_dpss_coarse_start_2e23_2e24_vs_long_double(lg):
    """The default large-N DPSS (coarse start + the parallel two-sided recurrence, no full-length
    bisection or solve) at 2^23 and 2^24, NW 8, K 15 (C4's band), against the long-double bisection
    + inverse iteration restatement."""
    n = 1 << lg
    d = nus.dpss_uniform(n, 8.0, 15, concentrations=False)
    tc, ev = C.dpss(n, 8.0, 15, threads=THREADS)
    err = float(np.abs(sign_align(d.tapers, tc) - tc).max())
    print(f"DPSS 2^{lg}: max |gpu - long double| = {err:.3e}")
    assert err < 1e-10
    np.testing.assert_allclose(d.eigenvalues, ev, rtol=1e-13)
