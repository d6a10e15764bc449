"""GPU parity: DPSS, tridiagonal eigenpairs, interpolated tapers and the R(B)
normalisation (ports of test_tapers.cpp / test_eig.cpp cases + oracle checks)."""
import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from conftest import golden, rel_l2, sign_align
from oracle import C

pytestmark = pytest.mark.gpu


def test_dpss_concentrations_n50():  # test_tapers.cpp:40-50
    d = nus.dpss_uniform(50, 2.5, 4)
    assert d.concentrations[0] > 0.999
    assert np.all(d.concentrations > 0.9) and np.all(d.concentrations <= 1.0)
    assert np.all(np.diff(d.concentrations) < 0)
    g = golden("dpss.npz")
    np.testing.assert_allclose(d.concentrations, g["conc50"], rtol=1e-9)


def test_dpss_parity_of_first_two_tapers():  # test_tapers.cpp:52-58
    d = nus.dpss_uniform(50, 2.5, 2)
    np.testing.assert_allclose(d.tapers[0], d.tapers[0][::-1], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(d.tapers[1], -d.tapers[1][::-1], rtol=1e-9, atol=1e-12)


def test_dpss_orthonormal():  # test_tapers.cpp:60-69
    d = nus.dpss_uniform(32, 3.0, 5)
    assert np.abs(d.tapers @ d.tapers.T - np.eye(5)).max() < 1e-10


def test_dpss_input_validation():  # test_tapers.cpp:71-75
    for args in ((10, 2.5, 11), (10, 5.0, 2), (10, 0.0, 2)):
        with pytest.raises(nus.InvalidArgument):
            nus.dpss_uniform(*args)


def test_dpss_matches_reference_and_oracle():
    g = golden("dpss.npz")
    d = nus.dpss_uniform(512, 4.0, 7)
    assert np.abs(sign_align(d.tapers, g["tap512"]) - g["tap512"]).max() < 1e-8  # reference fp64 error
    tc, ev = C.dpss(512, 4.0, 7)
    assert np.abs(sign_align(d.tapers, tc) - tc).max() < 1e-13
    np.testing.assert_allclose(d.eigenvalues, ev, rtol=1e-13)
    np.testing.assert_allclose(d.concentrations, g["conc512"], rtol=1e-9)


@pytest.mark.parametrize("n,tw,k", [(4096, 4.0, 7), (1 << 16, 5.0, 9), (1 << 16, 16.0, 31)])
def test_dpss_large_vs_extended_precision_oracle(n, tw, k):
    d = nus.dpss_uniform(n, tw, k, concentrations=False)
    tc, ev = C.dpss(n, tw, k)
    # the GPU solve is double-double inverse iteration; the oracle long-double bisection
    assert np.abs(sign_align(d.tapers, tc) - tc).max() < (1e-11 if n <= 4096 else 1e-10)
    np.testing.assert_allclose(d.eigenvalues, ev, rtol=1e-12)


def test_tridiagonal_closed_form():  # test_eig.cpp:71-79
    p = nus.tridiagonal_eigen([2.0, 2.0, 2.0], [-1.0, -1.0], 3)
    s2 = np.sqrt(2.0)
    np.testing.assert_allclose(p.values, [2 + s2, 2.0, 2 - s2], rtol=1e-13)
    assert np.all(p.residuals < 1e-12)


def test_tridiagonal_random_vs_dense():  # test_eig.cpp:92-109
    r = np.random.default_rng(99)
    d, e = r.standard_normal(8), r.standard_normal(7)
    p = nus.tridiagonal_eigen(d, e, 8)
    dense = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    lam = np.sort(np.linalg.eigvalsh(dense))[::-1]
    np.testing.assert_allclose(p.values, lam, rtol=1e-10, atol=1e-12)
    assert np.all(p.residuals < 1e-10)


def test_tridiagonal_validation():  # test_eig.cpp:111-116
    with pytest.raises(nus.InvalidArgument):
        nus.tridiagonal_eigen([1.0, 2.0], [0.5, 0.5], 1)
    with pytest.raises(nus.InvalidArgument):
        nus.tridiagonal_eigen([1.0, np.nan], [0.5], 1)
    with pytest.raises(nus.InvalidArgument):
        nus.tridiagonal_eigen([1.0, 2.0], [0.5], 3)


def test_gpss_interpolated_uniform_grid_is_rescaled_dpss():  # test_tapers.cpp:138-156
    grid = nus.SamplingGrid(np.arange(1.0, 51.0))
    s = nus.gpss_interpolated(grid, nus.SignalBand(0.5), 0.05, 4)
    assert not s.has_eigenvalues() and s.is_real()
    d = nus.dpss_uniform(50, 2.5, 4)
    w = sign_align(s.weights_matrix(), d.tapers)
    assert np.abs(w - np.sqrt(0.1) * d.tapers).max() < 1e-10


@pytest.mark.parametrize("name", ["uniform", "jitter", "arithmetic"])
def test_gpss_normalisation_and_reference(name):  # test_tapers.cpp:158-166
    g = golden("gpss.npz")
    t = g[f"t_{name}"]
    s = nus.gpss_interpolated(nus.SamplingGrid(t), nus.SignalBand(0.5), 0.05, 4)
    w = s.weights_matrix()
    np.testing.assert_allclose(C.quadform(t, 0.5, w), 0.1, rtol=1e-8)
    assert np.abs(sign_align(w, g[f"w_{name}"]) - g[f"w_{name}"]).max() < 1e-9


def test_gpss_band_range_error():
    grid = nus.SamplingGrid(np.arange(1.0, 51.0))
    with pytest.raises(nus.BandRangeError):
        nus.gpss_interpolated(grid, nus.SignalBand(0.5), 0.6, 2)
    with pytest.raises(nus.InvalidArgument):
        nus.gpss_interpolated(nus.SamplingGrid(np.arange(1.0, 6.0)), nus.SignalBand(0.5), 0.05, 2)


def test_quadform_kernel_vs_oracle_and_row_split():
    from paper_2407_01943_b200 import workloads as W
    wl = W.small(n=6000, k=3)
    w = C.gpss_interpolated(wl.times, wl.f_max, float(wl.f_w[0]), 3)[0]
    grid = nus.SamplingGrid(wl.times)
    band = nus.SignalBand(wl.f_max)
    q = nus.signal_band_quadform(grid, band, w)
    qc = C.quadform(wl.times, wl.f_max, w)
    np.testing.assert_allclose(q, qc, rtol=1e-11)
    # row partition (multi-GPU normalisation): partial sums over row blocks add up
    parts = [nus.signal_band_quadform(grid, band, w, rows=(a, b))
             for a, b in ((0, 1000), (1000, 3500), (3500, 6000))]
    np.testing.assert_allclose(np.sum(parts, axis=0), q, rtol=1e-12)


def test_spline_taper_matches_oracle_c1():
    g = golden("c1.npz")
    t = g["t"]
    grid = nus.SamplingGrid(t)
    w = nus.api.taper_spline(grid, nus.SignalBand(float(g["f_max"])), float(g["f_w"]), 7)
    n = t.size
    h = (t[-1] - t[0]) / (n - 1)
    dp, _ = C.dpss(n, float(g["f_w"]) * h * n, 7)
    knots = t[0] + h * np.arange(n)
    ref = np.stack([C.spline(knots, dp[j], t) for j in range(7)])
    assert np.abs(sign_align(w, ref) - ref).max() < 1e-12


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5", "small"])
def test_fast_normalisation_matches_exact_quadform(cfg):
    """normalise.cu: q = int_{-F}^{F} |W(f)|^2 df as a windowed lattice sum of the type-1 NUFFT
    agrees with the reference's dense form w^T R(B) w (kernels.cpp:28-37,100-115) to ~1e-12 on
    every config's sampling (F*T from 2e3 to 4e4 band-widths, gaps, many wraps)."""
    wl = {"c1": lambda: W.c1(), "c2": lambda: W.c2(n=1 << 15), "c3": lambda: W.c3(channels=1, n=1 << 15),
          "c4": lambda: W.c4(n=1 << 15, n_centers=1 << 12, windows=20), "c5": lambda: W.c5(n=1 << 15),
          "small": lambda: W.small(n=3000)}[cfg]()
    t = wl.times if wl.times.ndim == 1 else wl.times[0]
    g = nus.SamplingGrid(t)
    band = nus.SignalBand(wl.f_max)
    w = nus.api.taper_spline(g, band, float(wl.f_w[0]), 5)
    qe = nus.signal_band_quadform(g, band, w)
    qf = nus.signal_band_quadform_fast(g, band, w)
    assert np.abs(qf / qe - 1).max() < 1e-10


@pytest.mark.parametrize("n,tw,k,force", [(1 << 16, 8.0, 15, True), (1 << 18, 8.0, 15, True), (1 << 21, 8.0, 15, False)])
def test_dpss_rayleigh_refined_vs_extended_precision_oracle(n, tw, k, force, monkeypatch):
    """Large-n DPSS path (n >= 2^21, or NUS_DPSS_REFINE=1): bisection to 2 eps ||T||, double-double
    inverse iteration, a double-double Rayleigh-quotient shift and two more iterations; the gaps of
    the commuting tridiagonal stay O(10) while ||T|| ~ n^2/2, the regime of C4 (NW=8, K=15)."""
    if force:
        monkeypatch.setenv("NUS_DPSS_REFINE", "1")
    d = nus.dpss_uniform(n, tw, k, concentrations=False)
    tc, ev = C.dpss(n, tw, k)
    assert np.abs(sign_align(d.tapers, tc) - tc).max() < 1e-10
    np.testing.assert_allclose(d.eigenvalues, ev, rtol=1e-13)


@pytest.mark.parametrize("n,tw,k", [(1 << 20, 8.0, 15), (1 << 21, 4.0, 7)])
def test_dpss_from_coarse_start_vs_extended_precision_oracle(n, tw, k, monkeypatch):
    """Large-n DPSS without full-length bisection (default from 2^23, forced here): the coarse
    DPSS (n/64, >= 2^17) interpolated to n, double-double Rayleigh shifts, one inverse
    iteration and a final Rayleigh quotient."""
    monkeypatch.setenv("NUS_DPSS_COARSE", str(n))
    d = nus.dpss_uniform(n, tw, k, concentrations=False)
    tc, ev = C.dpss(n, tw, k)
    assert np.abs(sign_align(d.tapers, tc) - tc).max() < 1e-10
    np.testing.assert_allclose(d.eigenvalues, ev, rtol=1e-13)


@pytest.mark.parametrize("n,tw,k", [(1 << 20, 8.0, 15), (1 << 21, 4.0, 7), (1 << 22, 8.0, 15)])
def test_dpss_recurrence_vs_inverse_iteration(n, tw, k, monkeypatch):
    """The large-n vectors (coarse start, default from 2^20) by the parallel two-sided eigenvector
    recurrence (tapers.cu rec_* kernels, the default) against the sequential double-double inverse
    iteration they replace (NUS_DPSS_RECURRENCE=0), and both against the long-double restatement."""
    d_rec = nus.dpss_uniform(n, tw, k, concentrations=False)
    monkeypatch.setenv("NUS_DPSS_RECURRENCE", "0")
    d_ii = nus.dpss_uniform(n, tw, k, concentrations=False)
    monkeypatch.delenv("NUS_DPSS_RECURRENCE")
    assert np.abs(sign_align(d_rec.tapers, d_ii.tapers) - d_ii.tapers).max() < 1e-14
    np.testing.assert_allclose(d_rec.eigenvalues, d_ii.eigenvalues, rtol=1e-15)
    tc, ev = C.dpss(n, tw, k)
    assert np.abs(sign_align(d_rec.tapers, tc) - tc).max() < 1e-10
    np.testing.assert_allclose(d_rec.eigenvalues, ev, rtol=1e-13)
