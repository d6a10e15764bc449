"""GPU parity for the MTNUFFT estimator on the BASELINE configs.

Tolerances (BASELINE.json north_star): relL2(P) <= 1e-6 in fp64 at eps=1e-9,
<= 1e-4 in fp32 at eps=1e-5; bins bit-exact.  The CPU side is the reference
itself (Oracle-A, full MtnufftEstimator: golden fixture / live oracle/_ref)
where its O(N^2) setup is feasible, else the C restatement with the same
injected tapers (Oracle-B).
"""
import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from conftest import KERNELS, golden, kernel_tol, rel_l2, sign_align
from oracle import C, REF, ref_available

pytestmark = pytest.mark.gpu


def estimator(wl, tapers=None, precision=None, k=None, eps=None, policy=nus.NufftPathPolicy.auto_select):
    t = wl.times if wl.times.ndim == 1 else wl.times[0]
    plan = nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max)
    opts = nus.MtnufftEstimator.Options(k_tapers=k or wl.k, epsilon=eps or wl.eps,
                                        precision=precision or wl.precision, path_policy=policy)
    return nus.MtnufftEstimator(nus.SamplingGrid(t), nus.SignalBand(wl.f_max), plan, opts, tapers=tapers)


@pytest.mark.parametrize("kern", KERNELS)
def test_c1_full_pipeline_vs_reference_oracle_a(kern):
    """Config C1 end to end (GPU DPSS + spline + R(B) + NUFFT) vs the full reference estimator,
    under the reference's Gaussian window and under the ES window."""
    g = golden("c1.npz")
    wl = W.c1()
    assert np.array_equal(wl.times, g["t"]) and np.array_equal(wl.values, g["x"])
    est = estimator(wl)
    p = est.estimate(wl.values).power
    assert rel_l2(p, g["power"]) <= 1e-6
    w = est.tapers().weights_matrix()
    assert np.abs(sign_align(w, g["tapers"]) - g["tapers"]).max() < 1e-6 * np.abs(g["tapers"]).max()
    # with the reference's own tapers injected, the NUFFT stage agrees to ~1e-12 (Gaussian, the
    # reference's own window) / ~eps (ES: a different window meeting the same eps contract)
    p_inj = estimator(wl, tapers=g["tapers"]).estimate(wl.values).power
    assert rel_l2(p_inj, g["power"]) < kernel_tol(kern, 1e-11, 1e-8)
    assert np.array_equal(est.estimate(wl.values).flags, g["flags"])


@pytest.mark.parametrize("kern", KERNELS)
def test_c1_fp32_mode(kern):
    g = golden("c1.npz")
    wl = W.c1()
    p = estimator(wl, tapers=g["tapers"], precision="f32", eps=1e-5).estimate(wl.values).power
    assert rel_l2(p, g["power"]) <= 1e-4


@pytest.fixture(scope="module", params=KERNELS)
def c2_case(request):
    wl = W.c2()
    with nus.spread_kernel(request.param):
        est = estimator(wl)
    assert nus.SpreadKernel(est.transform_info().kernel).name == request.param
    w = est.tapers().weights_matrix()
    ref = C.mtnufft_power(wl.times, w, wl.values, wl.centers, 1e-9)  # Oracle-B (restatement)
    return wl, est, w, ref


def test_c2_fp64_vs_oracle(c2_case):
    wl, est, w, ref = c2_case
    p = est.estimate(wl.values).power
    assert rel_l2(p, ref) <= 1e-6
    kern = nus.SpreadKernel(est.transform_info().kernel).name
    assert rel_l2(p, ref) < kernel_tol(kern, 1e-8, 2e-8)  # the NUFFT stage is far tighter than the spec


def test_c2_fp32_vs_fp64_oracle(c2_case):
    wl, est, w, ref = c2_case
    with nus.spread_kernel(nus.SpreadKernel(est.transform_info().kernel)):
        est32 = estimator(wl, tapers=w, precision="f32", eps=1e-5)
    p = est32.estimate(wl.values).power
    assert rel_l2(p, ref) <= 1e-4


def test_c2_tapers_vs_extended_precision_oracle(c2_case):
    wl, _, w, _ = c2_case
    n = wl.n
    h = (wl.times[-1] - wl.times[0]) / (n - 1)
    dp, _ = C.dpss(n, float(wl.f_w[0]) * h * n, 7)
    knots = wl.times[0] + h * np.arange(n)
    ref = np.stack([C.spline(knots, dp[j], wl.times) for j in range(7)])
    # normalisation differs only by the per-taper scale; compare shapes
    ws = w / np.linalg.norm(w, axis=1, keepdims=True)
    rs = ref / np.linalg.norm(ref, axis=1, keepdims=True)
    assert np.abs(sign_align(ws, rs) - rs).max() < 1e-8 * np.abs(rs).max()
    # R(B) normalisation: w^T R(B) w = 2 f_w, checked on a row block with the oracle's exact sum
    q = nus.signal_band_quadform(nus.SamplingGrid(wl.times), nus.SignalBand(wl.f_max), w[:2])
    np.testing.assert_allclose(q, 2 * wl.f_w[0], rtol=1e-9)


def test_c2_linearity_and_power_properties_full_size(c2_case):
    """Size-independent properties at the full C2 size: J linear in x, P >= 0, P(a x) = a^2 P."""
    wl, est, w, ref = c2_case
    x, z = wl.values, np.roll(wl.values, 1234)
    jx = est.eigencoefficients(x).data
    jz = est.eigencoefficients(z).data
    jc = est.eigencoefficients(2 * x - 3 * z).data
    assert rel_l2(jc, 2 * jx - 3 * jz) < 1e-12
    p = est.estimate(x).power
    assert np.all(p >= 0)
    assert rel_l2(est.estimate(3 * x).power, 9 * p) < 1e-13
    np.testing.assert_allclose(np.mean(np.abs(jx) ** 2, axis=0), p, rtol=1e-12)


@pytest.mark.parametrize("kern", KERNELS)
def test_c3_channels_batch_fp32(kern):
    wl = W.c3(channels=4, n=1 << 16)
    pl = nus.api._Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), wl.k, wl.eps, 0, "f32", 0)
    # per-channel tapers: the batch estimator builds each channel's tapers on its own grid
    p = pl.power(wl.values)
    w = pl.tapers()
    for c in range(4):
        ref = C.mtnufft_power(wl.times[c], w[c], wl.values[c], wl.centers, wl.eps)
        assert rel_l2(p[c], ref) <= 1e-4
        single = nus.api._Estimator(wl.times[c], wl.centers, wl.f_max, float(wl.f_w[c]), wl.k, 1e-9, 0,
                                    "f64", 0, tapers=w[c])
        assert rel_l2(p[c], single.power(wl.values[c])[0]) <= 1e-4


@pytest.mark.parametrize("kern", KERNELS)
def test_c5_subset_vs_direct_nudft(kern):
    """C5 check: N=2^14 subset as its own grid, MTNUFFT P vs exact direct-sum P."""
    full = W.c5(n=1 << 16)
    t, x = full.times[: 1 << 14], full.values[: 1 << 14]
    wl = W.Workload("c5sub", t, x, 0.5 * np.arange(1 << 13) / ((1 << 13) - 1), 0.5, 4.0, 7, 1e-9, "f64")
    wl.f_w = np.array([W.half_width_for(t, 4.0)])
    est = estimator(wl)
    p = est.estimate(x).power
    w = est.tapers().weights_matrix()
    jd = np.stack([nus.ndft_direct(nus.SamplingGrid(t), w[k] * x, wl.centers) for k in range(7)])
    pd = np.mean(np.abs(jd) ** 2, axis=0)
    assert rel_l2(p, pd) <= 1e-6
    # and the GPU direct kernel agrees with the CPU reference direct sum on a strided subset
    sub = wl.centers[::64]
    jc = C.ndft_direct(t, w[0] * x, sub)
    assert rel_l2(jd[0][::64], jc) < 1e-12


@pytest.mark.parametrize("kern", KERNELS)
@pytest.mark.parametrize("k,eps", [(1, 1e-3), (3, 1e-6), (15, 1e-9), (31, 1e-12)])
def test_taper_count_and_width_sweep(k, eps, kern):
    """C5-style lattice over K (1..31, taper groups of 8) and eps (w = 4..16; ES ns = 4..14).
    Gaussian: the reference's transform replicated; ES: P within the eps contract of the
    exact direct-sum P (and of the reference's Gaussian P)."""
    wl = W.small(n=6000, n_centers=4096, k=k, nw=(k + 1) / 2, eps=eps, seed=k)
    est = estimator(wl)
    p = est.estimate(wl.values).power
    w = est.tapers().weights_matrix()
    ref = C.mtnufft_power(wl.times, w, wl.values, wl.centers, eps)
    if kern == "gaussian":
        assert rel_l2(p, ref) < 1e-10
    else:
        exact = C.mtnufft_power(wl.times, w, wl.values, wl.centers, eps, policy=2)
        assert rel_l2(p, exact) < 10 * eps
        assert rel_l2(p, ref) < 10 * eps


def test_direct_path_estimator_small_problem():
    """N*I < 2^14: the auto policy takes the exact direct sum (nufft.cpp:82-88)."""
    t = np.cumsum(np.random.default_rng(2).uniform(0.5, 1.5, 50))
    wl = W.Workload("tiny", t, np.random.default_rng(3).standard_normal(50), np.arange(51) * 0.01, 0.5,
                    2.5, 4, 1e-8, "f64")
    wl.f_w = np.array([W.half_width_for(t, 2.5)])
    est = estimator(wl)
    assert est.transform_info().path == 0
    p = est.estimate(wl.values).power
    w = est.tapers().weights_matrix()
    assert rel_l2(p, C.mtnufft_power(t, w, wl.values, wl.centers, 1e-8, policy=2)) < 1e-12
    if ref_available():
        pr, wr, _ = REF.mtnufft(t, wl.values, 0.5, wl.centers, float(wl.f_w[0]), 4, 1e-8)
        assert rel_l2(p, pr) <= 1e-6


def test_estimate_rejects_wrong_length():
    wl = W.small(n=2048, k=2)
    est = estimator(wl)
    with pytest.raises(nus.InvalidArgument):
        est.estimate(np.zeros(2047))


def test_estimate_mtnufft_one_shot_matches_estimator():
    wl = W.small(n=2048, k=3)
    series = nus.SignalSeries(nus.SamplingGrid(wl.times), wl.values)
    plan = nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max)
    a = nus.estimate_mtnufft(series, nus.SignalBand(wl.f_max), plan, 3, 1e-9).power
    b = estimator(wl, k=3).estimate(wl.values).power
    assert rel_l2(a, b) < 1e-14


def test_estimate_many_equals_estimate(c2_case):
    """The pipelined batch entry (copies overlapped across steps) returns exactly estimate()'s P."""
    wl, est, _, _ = c2_case
    xs = np.stack([np.roll(wl.values, 101 * i) for i in range(5)])
    many = est.estimate_many(xs)
    assert len(many) == 5
    for i in (0, 3, 4):
        assert np.array_equal(many[i].power, est.estimate(xs[i]).power)


@pytest.mark.parametrize("kern", KERNELS)
def test_c4_structure_fp64_vs_oracle(kern):
    """C4 structure (400 lognormal observing windows, Poisson inside, dyadic centres i/32, df*T ~
    12.5 wraps of the grid, NW=8, K=15, eps=1e-9) at N=2^20, I=2^18: GPU setup (DPSS, spline,
    O(N log N) normalisation) + NUFFT vs Oracle-B with the same tapers."""
    wl = W.c4(n=1 << 20, n_centers=1 << 18)
    est = estimator(wl)
    p = est.estimate(wl.values).power
    w = est.tapers().weights_matrix()
    ref = C.mtnufft_power(wl.times, w, wl.values, wl.centers, 1e-9)
    assert rel_l2(p, ref) <= 1e-6
    assert rel_l2(p, ref) < kernel_tol(kern, 1e-9, 2e-8)
    # the normalisation reached w^T R(B) w = 2 f_w (checked with the dense form on two rows)
    q = nus.signal_band_quadform(nus.SamplingGrid(wl.times), nus.SignalBand(wl.f_max), w[[0, 14]])
    np.testing.assert_allclose(q, 2 * wl.f_w[0], rtol=1e-9)


def test_c4_tapers_vs_extended_precision_oracle():
    """C4 tapers (K=15, NW=8) at N=2^18 against the long-double DPSS + spline restatement."""
    wl = W.c4(n=1 << 18, n_centers=1 << 16)
    est = estimator(wl)
    w = est.tapers().weights_matrix()
    n = wl.n
    h = (wl.times[-1] - wl.times[0]) / (n - 1)
    dp, _ = C.dpss(n, float(wl.f_w[0]) * h * n, 15)
    knots = wl.times[0] + h * np.arange(n)
    ref = np.stack([C.spline(knots, dp[j], wl.times) for j in range(15)])
    ws = w / np.linalg.norm(w, axis=1, keepdims=True)
    rs = ref / np.linalg.norm(ref, axis=1, keepdims=True)
    assert np.abs(sign_align(ws, rs) - rs).max() < 1e-8 * np.abs(rs).max()
