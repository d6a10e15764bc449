"""GPU parity for the harmonic F-test (reference src/inference.cpp:132-186)."""
import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from conftest import KERNELS, golden, kernel_tol, rel_l2
from oracle import REF, ref_available

pytestmark = pytest.mark.gpu


def _c1_plan(g):
    return nus.BandPlan.from_centers(g["centers"], float(g["f_w"]), float(g["f_max"]))


@pytest.mark.parametrize("kern", KERNELS)
def test_f_test_on_reference_tapers_matches_reference_golden(kern):
    g, gf = golden("c1.npz"), golden("ftest_c1.npz")
    grid = nus.SamplingGrid(g["t"])
    plan = _c1_plan(g)
    tapers = nus.TaperSet(grid, nus.AnalysisBand(0.0, float(g["f_w"])), float(g["f_max"]), g["tapers"])
    nplan = nus.NufftPlan(grid, g["centers"], float(g["eps"]))
    j = nus.eigencoefficients(tapers, nus.SignalSeries(grid, g["x"]), nplan)
    r = nus.f_test(j, tapers, plan)
    tol = kernel_tol(kern, 1e-9, 1e-7)  # ES: a different window within the same eps contract
    assert rel_l2(r.f_stat, gf["f"]) < tol
    assert rel_l2(r.amplitude, gf["amp"]) < tol
    assert np.array_equal(r.flags, gf["flags"])
    np.testing.assert_allclose([c for _, c in r.critical_values], gf["crit"], rtol=1e-10)
    assert r.dof == (2, 12)
    # the 10 Hz line of C1 is the most significant band
    assert abs(plan.center(int(np.argmax(r.f_stat))) - 10.0) < 0.1


@pytest.mark.parametrize("kern", KERNELS)
def test_estimator_f_test_with_device_resident_j(kern):
    g = golden("c1.npz")
    wl = W.c1()
    plan = _c1_plan(g)
    est = nus.MtnufftEstimator(nus.SamplingGrid(wl.times), nus.SignalBand(wl.f_max), plan,
                               nus.MtnufftEstimator.Options(k_tapers=7, epsilon=1e-9))
    r = est.f_test(wl.values)
    w = est.tapers().weights_matrix()
    if ref_available():
        f, amp, flags, crit = REF.f_test(wl.times, w, wl.values, wl.centers, wl.eps, wl.f_max, float(wl.f_w[0]))
        assert rel_l2(r.f_stat, f) < kernel_tol(kern, 1e-9, 1e-7) and np.array_equal(r.flags, flags)
    # vs the reference's own tapers: F is taper-sign invariant and within the DPSS accuracy
    gf = golden("ftest_c1.npz")
    assert rel_l2(r.f_stat, gf["f"]) < 1e-5


def test_f_test_saturation_and_condition_flags():
    t = np.arange(1.0, 257.0)
    x = np.cos(2 * np.pi * 0.125 * t)  # exact line on a uniform grid
    plan = nus.BandPlan.from_centers(np.arange(129) / 256.0, 0.02, 0.5)
    est = nus.MtnufftEstimator(nus.SamplingGrid(t), nus.SignalBand(0.5), plan,
                               nus.MtnufftEstimator.Options(k_tapers=3, epsilon=1e-9))
    r = est.f_test(x, nus.FTestOptions(saturation_cap=1e9))
    assert r.flags[0] & nus.kFtestConditionViolated          # 2 f_c <= f_w at f_c = 0
    assert not (r.flags[64] & nus.kFtestConditionViolated)
    assert r.f_stat.max() <= 1e9
    with pytest.raises(nus.InvalidArgument):
        nus.MtnufftEstimator(nus.SamplingGrid(t), nus.SignalBand(0.5), plan,
                             nus.MtnufftEstimator.Options(k_tapers=1, epsilon=1e-9)).f_test(x)


def test_f_test_degenerate_tapers():
    g = golden("c1.npz")
    grid = nus.SamplingGrid(g["t"])
    w = np.zeros((3, g["t"].size))
    w[:, 0], w[:, 1] = 1.0, -1.0  # zero-frequency responses vanish
    tapers = nus.TaperSet(grid, nus.AnalysisBand(0.0, float(g["f_w"])), float(g["f_max"]), w)
    j = nus.EigenCoefficients(3, g["centers"].size, np.zeros((3, g["centers"].size), complex))
    with pytest.raises(nus.DegenerateTapers):
        nus.f_test(j, tapers, _c1_plan(g))
