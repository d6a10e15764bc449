"""GPU parity: NufftPlan / ndft_direct / eigencoefficients through the C-ABI.

Ports of /root/reference/proj/tests/test_nufft.cpp (case by case, same
tolerances) plus the bit-exact bin contract and J parity against the oracle.
"""
import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from conftest import golden, rel_l2
from oracle import C

pytestmark = pytest.mark.gpu

FAST = nus.NufftPathPolicy.force_fast


def test_ndft_direct_single_sample_and_zero_frequency():  # test_nufft.cpp:52-62
    g = nus.SamplingGrid([3.0, 4.0])
    out = nus.ndft_direct(g, [1.0, 0.0], [0.25])
    assert abs(out[0].real) < 1e-15 and out[0].imag == pytest.approx(1.0)
    out = nus.ndft_direct(g, [1.5, 2.5], [0.0])
    assert out[0].real == pytest.approx(4.0) and abs(out[0].imag) < 1e-15


def test_ndft_direct_integer_grid_matches_dft():  # test_nufft.cpp:64-79
    gd = golden("nufft_small.npz")
    got = nus.ndft_direct(nus.SamplingGrid(gd["t16"]), gd["x16"], gd["c16"])
    expect = np.fft.fft(gd["x16"])
    assert np.all(np.abs(got - expect) < 1e-12 * (1 + np.abs(expect)))
    assert rel_l2(got, gd["dft16"]) < 1e-14


def test_fast_path_accuracy_lattice_against_reference():  # test_nufft.cpp:81-96
    gd = golden("nufft_lattice.npz")
    for i in range(int(gd["ncases"])):
        eps, t, y, c = float(gd[f"case{i}_eps"]), gd[f"case{i}_t"], gd[f"case{i}_y"], gd[f"case{i}_c"]
        plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
        assert plan.path() == nus.NufftPath.fast
        assert np.array_equal(plan.first_cells(), gd[f"case{i}_j0"])  # bit-exact bins
        fast = plan.execute(y)
        assert np.abs(fast - gd[f"case{i}_direct"]).max() <= eps * np.abs(y).sum()
        assert rel_l2(fast, gd[f"case{i}_fast"]) < 1e-11  # vs the reference's own fast path


def test_fast_path_error_scales_with_precision():  # test_nufft.cpp:98-111
    gd = golden("nufft_small.npz")
    g = nus.SamplingGrid(gd["t200"])
    y, c, direct = gd["y200"], gd["c256"], gd["direct200"]
    loose = nus.NufftPlan(g, c, 1e-4, FAST).execute(y)
    tight = nus.NufftPlan(g, c, 1e-10, FAST).execute(y)
    err_l, err_t = np.abs(loose - direct).max(), np.abs(tight - direct).max()
    assert err_t * 1e4 <= err_l + 1e-300
    assert err_t <= 1e-10 * np.abs(y).sum()
    assert rel_l2(loose, gd["loose200"]) < 1e-11 and rel_l2(tight, gd["tight200"]) < 1e-11


def test_uniform_grid_agrees_with_fft():  # test_nufft.cpp:113-129
    gd = golden("nufft_small.npz")
    fast = nus.NufftPlan(nus.SamplingGrid(gd["t64"]), gd["c64"], 1e-8, FAST).execute(gd["x64"])
    expect = np.fft.fft(gd["x64"])
    assert np.abs(fast - expect).max() <= 1e-8 * np.abs(gd["x64"]).sum()


def test_plan_path_selection_and_mismatches():  # test_nufft.cpp:131-152
    gd = golden("nufft_small.npz")
    small = nus.SamplingGrid(gd["grid50"])
    centers = np.arange(51) * 0.01
    plan = nus.NufftPlan(small, centers, 1e-8)
    assert plan.path() == nus.NufftPath.direct
    big = nus.NufftPlan(nus.SamplingGrid(gd["grid500"]), np.arange(64) * (0.5 / 64), 1e-8)
    assert big.path() == nus.NufftPath.fast
    ragged = [0.0, 0.1, 0.15, 0.4]
    pr = nus.NufftPlan(small, ragged, 1e-8)
    assert pr.path() == nus.NufftPath.direct and not pr.centers_uniform()
    with pytest.raises(nus.InvalidArgument):
        nus.NufftPlan(small, ragged, 1e-8, FAST)
    with pytest.raises(nus.PlanMismatch):
        plan.execute(np.ones(49, complex))
    with pytest.raises(nus.InvalidArgument):
        nus.NufftPlan(small, centers, 0.5)
    with pytest.raises(nus.InvalidArgument):
        nus.NufftPlan(small, [], 1e-8)
    with pytest.raises(nus.InvalidArgument):
        nus.NufftPlan(small, centers, 1e-8, oversampling=1)
    # direct path result == exact sum
    y = np.random.default_rng(1).standard_normal(50) + 0j
    assert rel_l2(plan.execute(y), C.ndft_direct(gd["grid50"], y, centers)) < 1e-13


def test_single_center_is_direct_path():
    g = nus.SamplingGrid(np.arange(20000.0))
    p = nus.NufftPlan(g, [0.25], 1e-8)
    assert p.path() == nus.NufftPath.direct and not p.centers_uniform()


def _uniform_grid(n):
    return nus.SamplingGrid(np.arange(1.0, n + 1.0))


def test_eigencoefficients_zero_constant_line():  # test_nufft.cpp:154-190
    grid = _uniform_grid(50)
    band = nus.SignalBand(0.5)
    tapers = nus.gpss_interpolated(grid, band, 0.05, 4)
    plan = nus.make_band_plan(0.5, 0.05, 0.01)
    nplan = nus.NufftPlan(grid, plan.centers(), 1e-8)
    jz = nus.eigencoefficients(tapers, nus.SignalSeries(grid, np.zeros(50)), nplan)
    assert np.all(np.abs(jz.data) == 0.0)
    j1 = nus.eigencoefficients(tapers, nus.SignalSeries(grid, np.ones(50)), nplan)
    w0 = tapers.zero_frequency_responses()
    assert np.all(np.abs(j1.data[:, 0] - w0) < 1e-10)
    t = grid.times()
    line = np.cos(2 * np.pi * 0.25 * t + 0.3)
    jl = nus.eigencoefficients(tapers, nus.SignalSeries(grid, line), nplan)
    best = int(np.argmax(np.abs(jl.data[0])))
    assert plan.center(best) == pytest.approx(0.25, rel=0.021)


def test_eigencoefficients_linear_in_series():  # test_nufft.cpp:192-213
    from oracle import REF, ref_available
    t = golden("nufft_small.npz")["grid50"][:40] if not ref_available() else REF.generate_grid(1, 40, seed=31)
    grid = nus.SamplingGrid(t)
    tapers = nus.gpss_interpolated(grid, nus.SignalBand(0.5), 0.05, 3)
    plan = nus.make_band_plan(0.5, 0.05, 0.01)
    nplan = nus.NufftPlan(grid, plan.centers(), 1e-8)
    r = np.random.default_rng(8)
    x, z = r.standard_normal(40), r.standard_normal(40)
    jx = nus.eigencoefficients(tapers, nus.SignalSeries(grid, x), nplan).data
    jz = nus.eigencoefficients(tapers, nus.SignalSeries(grid, z), nplan).data
    jc = nus.eigencoefficients(tapers, nus.SignalSeries(grid, 2 * x - 3 * z), nplan).data
    expect = 2 * jx - 3 * jz
    assert np.all(np.abs(jc - expect) < 1e-10 * (1 + np.abs(expect)))


def test_plan_mismatch_when_grids_differ():  # test_nufft.cpp:215-223
    g1 = nus.SamplingGrid(np.cumsum(np.full(30, 1.0)))
    g2 = nus.SamplingGrid(np.cumsum(np.full(30, 1.0)) + 0.01)
    tapers = nus.gpss_interpolated(g1, nus.SignalBand(0.5), 0.05, 2)
    nplan = nus.NufftPlan(g2, nus.make_band_plan(0.5, 0.05, 0.05).centers(), 1e-8)
    with pytest.raises(nus.PlanMismatch):
        nus.eigencoefficients(tapers, nus.SignalSeries(g2, np.ones(30)), nplan)


# ---------------------------------------------------------------- bins / sort contract

@pytest.mark.parametrize("name", ["c1", "many_wrap"])
def test_bins_bit_exact_golden(name):
    gd = golden("c1.npz" if name == "c1" else "bins_many_wrap.npz")
    eps = float(gd["eps"])
    plan = nus.NufftPlan(nus.SamplingGrid(gd["t"]), gd["centers"], eps, FAST)
    assert np.array_equal(plan.first_cells(), gd["first_cells"])


def test_bins_bit_exact_c2_full_size_and_sort_is_stable():
    wl = W.c2()
    plan = nus.NufftPlan(nus.SamplingGrid(wl.times), wl.centers, 1e-9, FAST)
    j0 = plan.first_cells()
    assert np.array_equal(j0, C.first_cells(wl.times, wl.centers, 1e-9))
    mr = plan.grid_size()
    s = np.mod(j0, mr)
    perm = plan.sort_order()
    assert np.array_equal(perm, np.argsort(s, kind="stable"))  # stable: ties keep time order


def test_fp64_transform_matches_oracle_at_c1_size():
    gd = golden("c1.npz")
    y = gd["x"] * gd["tapers"][0]
    plan = nus.NufftPlan(nus.SamplingGrid(gd["t"]), gd["centers"], 1e-9, FAST)
    got = plan.execute(y)
    ref = C.nufft_fast(gd["t"], gd["centers"], 1e-9, y)
    assert rel_l2(got, ref) < 1e-12


def test_fp32_transform_accuracy():
    wl = W.small(n=4096, eps=1e-5)
    y = np.random.default_rng(3).standard_normal(wl.n) + 1j * np.random.default_rng(4).standard_normal(wl.n)
    plan = nus.NufftPlan(nus.SamplingGrid(wl.times), wl.centers, 1e-5, FAST, precision="f32")
    got = plan.execute(y)
    direct = C.ndft_direct(wl.times, y, wl.centers)
    assert np.abs(got - direct).max() <= 1e-5 * np.abs(y).sum()
    assert rel_l2(got, direct) < 1e-4


@pytest.mark.parametrize("eps", [1e-3, 1e-6, 1e-9, 1e-12])
def test_accuracy_sweep_against_direct(eps):
    wl = W.small(n=3000, n_centers=2048, eps=eps, seed=7)
    y = np.random.default_rng(5).standard_normal(wl.n) + 0j
    plan = nus.NufftPlan(nus.SamplingGrid(wl.times), wl.centers, eps, FAST)
    got = plan.execute(y)
    assert np.abs(got - C.ndft_direct(wl.times, y, wl.centers)).max() <= eps * np.abs(y).sum()
    assert rel_l2(got, C.nufft_fast(wl.times, wl.centers, eps, y)) < 1e-11


def test_clustered_dense_tiles_spill_over_batches():
    """Many points per spreading tile (clustered sampling): several staging batches per tile."""
    r = np.random.default_rng(11)
    t = np.sort(np.concatenate([r.uniform(0, 1, 20000), r.uniform(50, 50.01, 5000)]))
    t = np.unique(t)
    c = np.arange(256) * (10.0 / 255)
    y = r.standard_normal(t.size) + 0j
    plan = nus.NufftPlan(nus.SamplingGrid(t), c, 1e-9, FAST)
    assert np.array_equal(plan.first_cells(), C.first_cells(t, c, 1e-9))
    assert rel_l2(plan.execute(y), C.nufft_fast(t, c, 1e-9, y)) < 1e-11


@pytest.mark.parametrize("kern", ["gaussian", "es"])
def test_fused_fft_at_mr_2_25_matches_generic_path(kern, monkeypatch):
    """C4's grid (I = 2^24 dyadic centres, Mr = 2^25): the fused two-pass FFT with 8192-element
    tiles and rows agrees with the generic radix-2 + crop path on the same spread grid."""
    wl = W.c4(n=1 << 18, n_centers=1 << 24, windows=100)
    g = nus.SamplingGrid(wl.times)
    y = wl.values.astype(np.complex128)
    fused = nus.NufftPlan(g, wl.centers, 1e-9, FAST)
    assert fused.grid_size() == 1 << 25
    a = fused.execute(y)
    monkeypatch.setenv("NUS_FFT", "generic")
    b = nus.NufftPlan(g, wl.centers, 1e-9, FAST).execute(y)
    assert rel_l2(a, b) < 1e-13
    sub = np.arange(0, 1 << 24, 4099)
    d = C.ndft_direct(wl.times, y, wl.centers[sub])
    assert np.abs(a[sub] - d).max() <= 1e-9 * np.abs(y).sum()
