"""GPU parity of the path's own FFT at every grid size (no library FFT anywhere).

The uniform FFT replaces Radix2Fft::forward (/root/reference/proj/src/fft.cpp:39-58) inside
NufftPlan::execute (nufft.cpp:144-166) and the estimator.  fft.cu covers 512 <= Mr <= 2^26 with
the fused passes (single pass up to 8192, register-column pass A for R <= 16, tiled pass A
above) and every other power of two with the generic radix-2 Stockham kernels; the Radix2Fft
drop-in runs on the latter.  Checks: against the C restatement of the reference's gridding
(oracle/nus_oracle.c, which uses the reference's radix-2 FFT), against the generic path
(NUS_FFT=generic) on the same spread grid, and the eps contract against the direct sum.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from conftest import ROOT, rel_l2
from oracle import C, REF, ref_available

pytestmark = pytest.mark.gpu

FAST = nus.NufftPathPolicy.force_fast


@pytest.mark.parametrize("lg", list(range(0, 21)))
def test_radix2fft_dropin_matches_numpy(lg):
    """Radix2Fft forward / inverse (fft.hpp:12-29): forward e^{-2 pi i jk/n}, inverse unscaled."""
    n = 1 << lg
    rng = np.random.default_rng(lg)
    z = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    f = nus.Radix2Fft(n)
    fw = f.forward(z)
    assert rel_l2(fw, np.fft.fft(z)) < 1e-14 * max(lg, 1)
    assert rel_l2(f.inverse(z), n * np.fft.ifft(z)) < 1e-14 * max(lg, 1)
    assert rel_l2(f.inverse(fw) / n, z) < 1e-14 * max(lg, 1)


def test_radix2fft_dropin_matches_reference_and_rejects_bad_sizes():
    rng = np.random.default_rng(7)
    for n in (1, 2, 8, 1024, 1 << 16):
        z = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        if ref_available():
            assert rel_l2(nus.Radix2Fft(n).forward(z), REF.fft(z)) < 1e-14 * 17
            assert rel_l2(nus.Radix2Fft(n).inverse(z), REF.fft(z, inverse=True)) < 1e-14 * 17
        assert rel_l2(nus.Radix2Fft(n).forward(z), C.fft(z)) < 1e-14 * 17
    for bad in (0, 3, 12, 1000):
        with pytest.raises(nus.InvalidArgument):
            nus.Radix2Fft(bad)


def _case(lg_mr, seed):
    """Random times and I = Mr / 2 uniform centres, eps picked so that Mr = 2I (nufft.cpp:103-104)."""
    mr = 1 << lg_mr
    nc = mr // 2
    eps = 1e-2 if mr <= 32 else 1e-5 if mr <= 64 else 1e-9
    rng = np.random.default_rng(seed)
    n = 3000
    t = np.sort(rng.uniform(0, 50, n))
    t = np.unique(t)
    df = rng.uniform(0.3, 3.0) / (t[-1] - t[0])
    c = df * np.arange(nc)
    y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
    return t, c, eps, y


@pytest.mark.parametrize("lg_mr", list(range(5, 23)))
def test_plan_execute_at_every_grid_size(lg_mr, monkeypatch):
    """NufftPlan::execute for Mr = 2^5 .. 2^22: the own FFT (fused or generic) reproduces the
    reference's gridding (Gaussian window) to within their common rounding floor, equals the generic
    radix-2 path on the same spread grid, and meets the eps contract against the direct sum
    (test_nufft.cpp:81-96).  The floor grows with Mr: both evaluate each Gaussian weight from a
    difference x - 2 pi (j0 + p) / Mr of two O(1) numbers whose result is O(w / Mr) (nufft.cpp:
    122-126), i.e. a relative rounding of ~1e-16 Mr in the weights, not in the FFT."""
    t, c, eps, y = _case(lg_mr, lg_mr)
    plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
    assert plan.grid_size() == 1 << lg_mr
    got = plan.execute(y)
    assert rel_l2(got, C.nufft_fast(t, c, eps, y)) < max(3e-11, 2e-16 * (1 << lg_mr))
    sub = np.arange(0, c.size, max(1, c.size // 512))
    assert np.abs(got[sub] - C.ndft_direct(t, y, c[sub])).max() <= eps * np.abs(y).sum()
    monkeypatch.setenv("NUS_FFT", "generic")
    gen = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST).execute(y)
    assert rel_l2(got, gen) < 1e-13


@pytest.mark.parametrize("lg_mr", [9, 10, 11, 12, 13, 14, 15, 16, 17])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_estimator_power_at_every_fused_row_length(lg_mr, precision):
    """P(f) = sum_k |J_k|^2 / K accumulated in pass B for every row length C = 512 .. 8192 (single
    pass) and the two-pass grids with short (R <= 16) and tiled columns, several channels."""
    mr = 1 << lg_mr
    nc = mr // 2
    rng = np.random.default_rng(100 + lg_mr)
    chans, n, k = 3, 4000, 3
    ts = np.stack([np.sort(rng.uniform(0, 40, n)) + 1e-9 * np.arange(n) for _ in range(chans)])
    df = 1.7 / 40.0
    c = df * np.arange(nc)
    x = rng.standard_normal((chans, n))
    w = rng.uniform(0.5, 1.5, (chans, k, n)) / np.sqrt(n)
    eps = 1e-9 if precision == "f64" else 1e-5
    est = nus.api._Estimator(ts, c, 10.0, 0.1, k, eps, 1, precision, 0, tapers=w)
    assert est.info.mr == mr
    names = est.stage_kernels()
    assert names[0] == "spread_stream_kernel"
    assert names[2] == "fft_rows_crop_kernel"
    assert names[1] == ("(none: single pass)" if mr <= 8192 else
                        "fft_cols_small_kernel" if mr <= 1 << 15 else "fft_cols_blk_kernel")
    p = est.power(x)
    tol = 1e-10 if precision == "f64" else 1e-4
    for ch in range(chans):
        ref = C.mtnufft_power(ts[ch], w[ch], x[ch], c, eps)
        assert rel_l2(p[ch], ref) < tol


def test_c1_uses_only_own_kernels():
    """BASELINE C1 (I = 4096 -> Mr = 8192): one spread + one single-pass FFT/crop kernel."""
    wl = W.c1()
    plan = nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max)
    est = nus.MtnufftEstimator(nus.SamplingGrid(wl.times), nus.SignalBand(wl.f_max), plan,
                               nus.MtnufftEstimator.Options(k_tapers=wl.k, epsilon=wl.eps))
    assert est.transform_info().mr == 8192
    assert est.stage_kernels() == ["spread_stream_kernel", "(none: single pass)", "fft_rows_crop_kernel"]
    before = nus._capi.launch_count()
    est.estimate(wl.values)
    assert nus._capi.launch_count() - before == 2  # our kernels only: spread + fused FFT/crop


@pytest.mark.slow
@pytest.mark.parametrize("lg_mr", [26, 27])
def test_largest_grids_own_fft(lg_mr, monkeypatch):
    """Mr = 2^26 (the fused passes' largest: 8192-element tiles and rows, one column per tile) and
    2^27 (generic radix-2): eps contract against the direct sum on a strided subset, up to the
    fp64 phase floor of both sums (f t reaches 2^26 here)."""
    nc = 1 << (lg_mr - 1)
    rng = np.random.default_rng(lg_mr)
    t = np.sort(rng.uniform(0, 64, 1 << 16))
    t = np.unique(t)
    c = np.arange(nc) / 32.0
    y = rng.standard_normal(t.size) + 0j
    plan = nus.NufftPlan(nus.SamplingGrid(t), c, 1e-9, FAST)
    assert plan.grid_size() == 1 << lg_mr
    got = plan.execute(y)
    sub = np.arange(0, nc, 65537)
    err = np.abs(got[sub] - C.ndft_direct(t, y, c[sub])).max() / np.abs(y).sum()
    floor = 4e-16 * 2 * np.pi * np.abs(c).max() * np.abs(t).max()  # as test_gpu_es
    assert err <= max(1e-9, floor), (err, floor)
    if lg_mr == 26:
        monkeypatch.setenv("NUS_FFT", "generic")
        gen = nus.NufftPlan(nus.SamplingGrid(t), c, 1e-9, FAST).execute(y)
        assert rel_l2(got, gen) < 1e-12

