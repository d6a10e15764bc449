"""GPU: the exponential-of-semicircle (ES) window of the fast path (es.cu, the default).

The reference spreads with a Gaussian of 2w cells (nufft.cpp:90-142).  The ES window keeps
the reference's grid size, bins, phases, FFT sign and crop and changes only the window and
its deconvolution, so the parity bar is the reference's own NUFFT contract
max|fast - direct| <= eps ||y||_1 (test_nufft.cpp:81-96, golden lattice from the reference),
bit-exact bins, and the BASELINE P tolerances (1e-6 fp64 at eps=1e-9, 1e-4 fp32 at eps=1e-5)
against the reference's Gaussian result; those end-to-end cases run in test_gpu_mtnufft.py
(kern="es").
"""
import math

import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from conftest import golden, rel_l2
from oracle import C

pytestmark = pytest.mark.gpu

FAST = nus.NufftPathPolicy.force_fast


def es_width(eps):
    ns = math.ceil(math.log10(10.0 / eps) - 1e-12)
    ns += ns & 1
    return min(16, max(4, ns))


@pytest.mark.parametrize("kern", ["es"])
@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-5, 1e-6, 1e-9, 1e-12, 1e-14])
def test_es_plan_parameters(kern, eps):
    """Support ns from eps; the reference's w, Mr, tau and bins are unchanged."""
    wl = W.small(n=4000, n_centers=2048, k=1, eps=eps)
    plan = nus.NufftPlan(nus.SamplingGrid(wl.times), wl.centers, eps, FAST)
    assert plan.spread_kernel() == nus.SpreadKernel.es
    assert plan.support() == es_width(eps)
    w = max(4, math.ceil(0.55 * -math.log(eps)))
    assert plan.spread_width() == w
    assert plan.grid_size() == max(2 * 2048, 1 << math.ceil(math.log2(4 * w + 4)))
    assert np.array_equal(plan.first_cells(), C.first_cells(wl.times, wl.centers, eps))


@pytest.mark.parametrize("kern", ["es"])
def test_es_fast_path_contract_on_reference_lattice(kern):  # test_nufft.cpp:81-96
    gd = golden("nufft_lattice.npz")
    for i in range(int(gd["ncases"])):
        eps, t, y, c = float(gd[f"case{i}_eps"]), gd[f"case{i}_t"], gd[f"case{i}_y"], gd[f"case{i}_c"]
        plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
        assert plan.spread_kernel() == nus.SpreadKernel.es
        assert np.array_equal(plan.first_cells(), gd[f"case{i}_j0"])  # bins bit-exact either way
        fast = plan.execute(y)
        direct = gd[f"case{i}_direct"]
        assert np.abs(fast - direct).max() <= eps * np.abs(y).sum()
        # and it agrees with the reference's own (Gaussian) fast path to within that contract
        assert np.abs(fast - gd[f"case{i}_fast"]).max() <= 2 * eps * np.abs(y).sum()


@pytest.mark.parametrize("kern", ["es"])
def test_es_error_scales_with_precision(kern):  # test_nufft.cpp:98-111
    gd = golden("nufft_small.npz")
    g = nus.SamplingGrid(gd["t200"])
    y, c, direct = gd["y200"], gd["c256"], gd["direct200"]
    loose = nus.NufftPlan(g, c, 1e-4, FAST).execute(y)
    tight = nus.NufftPlan(g, c, 1e-10, FAST).execute(y)
    err_l, err_t = np.abs(loose - direct).max(), np.abs(tight - direct).max()
    assert err_t * 1e4 <= err_l + 1e-300
    assert err_t <= 1e-10 * np.abs(y).sum()
    assert err_l <= 1e-4 * np.abs(y).sum()


@pytest.mark.parametrize("kern", ["es"])
@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9, 1e-12])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_es_many_wrap_grid_vs_direct_sum(kern, eps, precision):
    """C4-like many-wrap grid (df*T >> 1) with clustered times: complex y, fast vs the direct
    sum on the CPU oracle; fp32 plans are checked at their own floor (1e-5 relative)."""
    if precision == "f32" and eps < 1e-6:
        pytest.skip("fp32 plans: eps below fp32 resolution")
    rng = np.random.default_rng(17)
    n = 20000
    t = np.sort(np.concatenate([d + rng.uniform(0, 0.3, n // 40) for d in range(40)]))
    t = np.unique(t)
    y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
    c = np.arange(4096) / 8.0  # df*T ~ 5 wraps
    plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST, precision=precision)
    got = plan.execute(y)
    sub = np.arange(0, c.size, 7)
    direct = C.ndft_direct(t, y, c[sub])
    err = np.abs(got[sub] - direct).max() / np.abs(y).sum()
    assert err <= max(eps, 2e-6 if precision == "f32" else 0.0)
    assert rel_l2(got[sub], direct) <= 5 * max(eps, 1e-6 if precision == "f32" else 0.0)


@pytest.mark.parametrize("kern", ["es"])
def test_es_eigencoefficients_linear_and_zero_frequency(kern):
    """Linearity of J (test_nufft.cpp:192-213) and J(f=0) = sum_n w_k(t_n) x_n (:154-190) on
    the fast path (N * I >= 2^14), to the eps contract."""
    wl = W.small(n=3000, n_centers=1024, k=4, eps=1e-10)
    grid = nus.SamplingGrid(wl.times)
    plan = nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max)
    est = nus.MtnufftEstimator(grid, nus.SignalBand(wl.f_max), plan,
                               nus.MtnufftEstimator.Options(k_tapers=4, epsilon=1e-10))
    assert nus.SpreadKernel(est.transform_info().kernel) == nus.SpreadKernel.es
    x = wl.values
    z = np.random.default_rng(3).standard_normal(x.size)
    jx, jz = est.eigencoefficients(x).data, est.eigencoefficients(z).data
    jc = est.eigencoefficients(2 * x - 3 * z).data
    assert rel_l2(jc, 2 * jx - 3 * jz) < 1e-12
    w = est.tapers().weights_matrix()
    j1 = est.eigencoefficients(np.ones_like(x)).data
    assert wl.centers[0] == 0.0
    w0 = w.sum(axis=1)
    assert np.all(np.abs(j1[:, 0] - w0) <= 1e-10 * np.abs(w).sum(axis=1))


def test_default_window_is_es_and_switchable():
    """Process default: ES; nus_set_spread_kernel switches plans created afterwards."""
    assert nus.get_spread_kernel() == nus.SpreadKernel.gaussian  # the autouse fixture's choice
    wl = W.small(n=3000, n_centers=1024, k=1, eps=1e-9)
    g = nus.SamplingGrid(wl.times)
    with nus.spread_kernel("es"):
        a = nus.NufftPlan(g, wl.centers, 1e-9, FAST)
    b = nus.NufftPlan(g, wl.centers, 1e-9, FAST)
    assert a.spread_kernel() == nus.SpreadKernel.es and a.support() == 10
    assert b.spread_kernel() == nus.SpreadKernel.gaussian and b.support() == 24
    y = np.random.default_rng(1).standard_normal(wl.times.size) + 0j
    d = C.ndft_direct(wl.times, y, wl.centers)
    for p in (a, b):
        assert np.abs(p.execute(y) - d).max() <= 1e-9 * np.abs(y).sum()


@pytest.mark.parametrize("kern", ["gaussian", "es"])
@pytest.mark.parametrize("ncl,n", [(1, 2000), (4, 20000), (40, 20000), (40, 50000)])
def test_dense_clusters_wrapping_into_empty_first_segment(kern, ncl, n):
    """Regression: > 32 points whose support wraps past Mr into a first segment with no points
    of its own (multi-round wrap part) — dense clusters starting at t = 0, 3-100 points/cell."""
    rng = np.random.default_rng(n + ncl)
    t = np.unique(np.sort(np.concatenate([d + rng.uniform(0, 0.3, n // ncl) for d in range(ncl)])))
    y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
    c = np.arange(4096) / 64.0
    plan = nus.NufftPlan(nus.SamplingGrid(t), c, 1e-6, FAST)
    got = plan.execute(y)
    if kern == "gaussian":
        assert rel_l2(got, C.nufft_fast(t, c, 1e-6, y)) < 1e-11
    else:
        sub = np.arange(0, c.size, 5)
        assert np.abs(got[sub] - C.ndft_direct(t, y, c[sub])).max() <= 1e-6 * np.abs(y).sum()


@pytest.mark.parametrize("kern", ["gaussian", "es"])
def test_random_problems_meet_the_eps_contract(kern):
    """30 seeded random problems across the plan's regimes (Mr from 4096 to 2^17: single- and
    two-pass fused FFTs; uniform / jittered / clustered / Poisson times; wraps from < 1 to ~20;
    complex y; eps from 1e-2 to 1e-12): max|fast - direct| <= eps ||y||_1 (test_nufft.cpp:81-96)."""
    rng = np.random.default_rng(2407)
    for case in range(30):
        n = int(rng.integers(200, 6000))
        nc = int(2 ** rng.integers(7, 16))
        eps = float(10 ** -rng.uniform(2, 12))
        kind = case % 4
        if kind == 0:
            t = np.sort(rng.uniform(0, 100, n))
        elif kind == 1:
            t = np.arange(n) + rng.uniform(-0.4, 0.4, n)
        elif kind == 2:
            t = np.sort(np.concatenate([c + rng.uniform(0, 0.2, n // 10) for c in rng.uniform(0, 50, 10)]))
        else:
            t = np.cumsum(rng.exponential(1.0, n))
        t = np.unique(t)
        span = t[-1] - t[0]
        df = rng.uniform(0.05, 20.0) / span  # 0.05 .. 20 wraps of the grid period
        c = rng.uniform(-5, 5) * df + df * np.arange(nc)
        y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
        plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
        got = plan.execute(y)
        d = C.ndft_direct(t, y, c)
        err = np.abs(got - d).max() / np.abs(y).sum()
        # fp64 phases 2 pi f t carry ~1e-16 relative rounding in both sums: the contract's floor
        floor = 4e-16 * 2 * np.pi * np.abs(c).max() * np.abs(t).max()
        assert err <= max(eps, floor), (case, n, nc, eps, kind, err, floor)
