"""CPU: host-side logic of the drop-in (validation, band plans, error mapping), the
C-ABI library loading with every declared symbol exported, and the synthetic
workload generators.  No GPU compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import _capi, workloads as W
from conftest import ROOT


def declared_symbols(header):
    txt = open(header).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int64_t|int)\s+(nus_\w+)\s*\(", txt, re.M)))


def test_c_abi_library_exports_every_declared_symbol():
    lib = _capi.lib()
    syms = declared_symbols(os.path.join(ROOT, "include", "nus_c.h"))
    assert len(syms) >= 29
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _capi._SIGS, f"{s} missing from the ctypes signature table"


def test_cpp_dropin_library_exports_reference_symbols():
    path = os.path.join(ROOT, "paper_2407_01943_b200", "lib", "libnuspectral_b200.so")
    if not os.path.exists(path):
        pytest.skip("C++ drop-in library not built")
    lib = ctypes.CDLL(path)
    # mangled names of a few reference entry points (nufft.hpp, estimators.hpp)
    out = os.popen(f"nm -DC {path}").read()
    for name in ("nuspectral::NufftPlan::NufftPlan", "nuspectral::NufftPlan::execute",
                 "nuspectral::eigencoefficients", "nuspectral::MtnufftEstimator::estimate",
                 "nuspectral::gpss_interpolated", "nuspectral::dpss_uniform", "nuspectral::ndft_direct"):
        assert name in out, name
    del lib


def test_library_links_no_fft_library():
    """Every FFT of the path (and of the Radix2Fft drop-in) is the library's own kernel: the
    shared object does not even link cuFFT (its DT_NEEDED entries)."""
    path = os.path.join(ROOT, "paper_2407_01943_b200", "lib", "libnus_b200.so")
    out = os.popen(f"readelf -d {path}").read()
    needed = re.findall(r"\(NEEDED\)\s+Shared library: \[([^\]]+)\]", out)
    assert needed, "readelf found no dynamic section"
    assert not [n for n in needed if "cufft" in n], needed
    syms = os.popen(f"nm -D --undefined-only {path}").read()
    assert "cufft" not in syms


def test_no_device_fails_loudly_without_cpu_fallback():
    try:
        info = _capi.device_info()
    except _capi.NoDeviceError:
        g = nus.SamplingGrid([0.0, 1.0, 2.5, 3.0])
        with pytest.raises(_capi.NoDeviceError):
            nus.NufftPlan(g, [0.0, 0.1, 0.2], 1e-8)
        return
    assert info["cc"][0] >= 10


def test_sampling_grid_validation():
    with pytest.raises(nus.InvalidArgument):
        nus.SamplingGrid([1.0])
    with pytest.raises(nus.InvalidArgument):
        nus.SamplingGrid([0.0, 1.0, 1.0])
    with pytest.raises(nus.InvalidArgument):
        nus.SamplingGrid([0.0, np.nan])
    g = nus.SamplingGrid([0.0, 1.0, 3.0])
    assert g.mean_dt == pytest.approx(1.0)  # (t_N - t_1)/N, grid.cpp:21


def test_band_plans_match_reference_grid_tests():
    # test_grid.cpp:19-42: sizes 51 / 3 / 241
    assert nus.make_band_plan(0.5, 0.05, 0.01).size() == 51
    assert nus.make_band_plan(0.5, 0.25, 0.25).size() == 3
    p = nus.make_band_plan(0.5, 0.05, 0.01)
    assert p.flagged(0) and not p.flagged(25) and p.flagged(50)
    with pytest.raises(nus.InvalidArgument):
        nus.make_band_plan(0.5, 0.3, 0.01)
    with pytest.raises(nus.InvalidArgument):
        nus.make_band_plan(0.5, 0.05, 0.2)
    with pytest.raises(nus.InvalidArgument):
        nus.BandPlan([nus.AnalysisBand(0.1, 0.05), nus.AnalysisBand(0.1, 0.05)], 0.5, 0.1)
    with pytest.raises(nus.InvalidArgument):
        nus.AnalysisBand(-0.1, 0.05)


def test_vectorised_band_plan_equals_object_plan():
    a = nus.make_band_plan(0.5, 0.05, 0.01)
    b = nus.BandPlan.from_centers(a.centers(), 0.05, 0.5)
    assert np.array_equal(a.centers(), b.centers()) and np.array_equal(a.flags(), b.flags())


def test_default_taper_count():
    # tapers.cpp:219-222 and the BASELINE configs: NW 4 -> 7, 5 -> 9, 8 -> 15
    for tw, k in ((4, 7), (5, 9), (8, 15), (0.5, 1), (2.5, 4), (16, 31)):
        assert nus.default_taper_count(tw) == k


def test_error_hierarchy_mirrors_reference():
    assert issubclass(nus.PlanMismatch, nus.NusError)
    assert issubclass(nus.InvalidArgument, ValueError)
    assert issubclass(nus.BandRangeError, nus.NusError)


@pytest.mark.parametrize("gen", [W.c1, lambda: W.c2(n=1 << 14), lambda: W.c3(channels=2, n=1 << 12),
                                 lambda: W.c4(n=1 << 14, n_centers=1 << 12, windows=20),
                                 lambda: W.c5(n=1 << 14)])
def test_workloads_are_valid_grids(gen):
    wl = gen()
    t = np.atleast_2d(wl.times)
    assert np.all(np.diff(t, axis=1) > 0)
    assert t.shape == np.atleast_2d(wl.values).shape
    # tw = f_w h N == NW (tapers.cpp:156-157)
    h = (t[0, -1] - t[0, 0]) / (t.shape[1] - 1)
    assert wl.f_w[0] * h * t.shape[1] == pytest.approx(wl.nw, rel=1e-12)
    from oracle import C
    assert C.centers_uniform(wl.centers)


def test_workloads_are_seeded():
    a, b = W.c2(n=4096), W.c2(n=4096)
    assert np.array_equal(a.times, b.times) and np.array_equal(a.values, b.values)


def test_f_quantile_matches_reference_and_scipy():
    from scipy.stats import f as fdist
    from oracle import REF, ref_available
    for p, d1, d2 in ((0.05, 2, 12), (0.01, 2, 12), (1 / 4096, 2, 12), (0.05, 2, 60), (0.3, 3, 7)):
        v = nus.f_quantile(p, d1, d2)
        assert v == pytest.approx(fdist.isf(p, d1, d2), rel=1e-9)
        if ref_available():
            assert v == pytest.approx(REF.f_quantile(p, d1, d2), rel=1e-10)
    with pytest.raises(nus.InvalidArgument):
        nus.f_quantile(1.5, 2, 3)
