"""MTNUFFT0: the exact nominal-band GPSS by the dense generalized Hermitian
eigenproblem on the device (cuSOLVER/cuBLAS), against the reference's own gpss_exact,
generalized_hermitian_eigen and MtnufftEstimator(exact_nominal) (golden fixtures from
tests/golden/make_golden_gep.py; the reference is O(N^3), so N <= 1024 here).

Eigenvectors are compared up to the phase the canonical-phase rule leaves ambiguous when two
entries tie in magnitude (symmetric / antisymmetric tapers on near-symmetric grids).
"""
import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu


def _align(w, ref):
    """Rotate each row of w by the unit phase that best matches ref (least squares)."""
    out = np.empty_like(ref, dtype=np.complex128)
    for j in range(ref.shape[0]):
        ip = np.vdot(w[j], ref[j])
        out[j] = w[j] * (ip / abs(ip) if abs(ip) > 0 else 1.0)
    return out


@pytest.mark.parametrize("n", [256, 512, 1024])
def test_gpss_exact_real_band_matches_reference(n):
    g = golden("gep_gpss.npz")
    grid = nus.SamplingGrid(g[f"t{n}"])
    ts = nus.gpss_exact(grid, nus.SignalBand(float(g[f"fmax{n}"])), nus.AnalysisBand(0.0, float(g[f"fw{n}"])), 7)
    assert ts.is_real()
    ref_w, ref_c = g[f"w{n}"], g[f"conc{n}"]
    assert np.abs(ts.eigenvalues() - ref_c).max() < 1e-9
    w = _align(ts.weights_matrix().astype(np.complex128), ref_w)
    assert np.abs(w - ref_w).max() < 1e-6 * np.abs(ref_w).max()
    # normalisation w^T R(B) w = 2 f_w (tapers.cpp:134-140)
    q = nus.signal_band_quadform(grid, nus.SignalBand(float(g[f"fmax{n}"])), ts.weights_matrix())
    assert np.allclose(q, 2 * float(g[f"fw{n}"]), rtol=1e-10)


def test_gpss_exact_complex_band_matches_reference():
    g = golden("gep_gpss.npz")
    grid = nus.SamplingGrid(g["tc"])
    ts = nus.gpss_exact(grid, nus.SignalBand(float(g["fmaxc"])), nus.AnalysisBand(float(g["fcc"]), float(g["fwc"])), 5)
    assert not ts.is_real()
    assert np.abs(ts.eigenvalues() - g["concc"]).max() < 1e-9
    w = _align(ts.weights_matrix(), g["wc"])
    assert np.abs(w - g["wc"]).max() < 1e-6 * np.abs(g["wc"]).max()


def test_generalized_eigen_pencil_matches_reference():
    g = golden("gep_pencil.npz")
    pairs = nus.generalized_hermitian_eigen(g["a"], g["m"], 6)
    assert np.abs(pairs.values - g["values"]).max() < 1e-11
    w = _align(pairs.vectors, g["vectors"])
    assert np.abs(w - g["vectors"]).max() < 1e-9 * np.abs(g["vectors"]).max()
    assert np.all(pairs.residuals < 1e-12) and np.all(g["residuals"] < 1e-12)
    # the canonical phase: the largest-magnitude entry is real positive
    for v in pairs.vectors:
        i = int(np.argmax(np.abs(v)))
        assert abs(v[i].imag) < 1e-14 * abs(v[i]) and v[i].real > 0
    # values only
    vals = nus.generalized_hermitian_eigen(g["a"], g["m"], 6, nus.GeneralizedEigenOptions(want_vectors=False)).values
    assert np.abs(vals - g["values"]).max() < 1e-11


def test_generalized_eigen_errors():
    n = 16
    m = -np.eye(n)  # not positive definite even after both ridges
    with pytest.raises(nus.ConditioningError):
        nus.generalized_hermitian_eigen(np.eye(n), m, 2)
    with pytest.raises(nus.SpectralRangeError):  # lambda = 2 is outside [0, 1]
        nus.generalized_hermitian_eigen(2.0 * np.eye(n), np.eye(n), 2)
    with pytest.raises(nus.BandRangeError):
        t = np.arange(64.0)
        nus.gpss_exact(nus.SamplingGrid(t), nus.SignalBand(0.5), nus.AnalysisBand(0.45, 0.1), 3)


@pytest.mark.parametrize("kern", ["gaussian", "es"])
def test_mtnufft0_estimator_matches_reference(kern):
    g = golden("gep_mtnufft0.npz")
    grid = nus.SamplingGrid(g["t"])
    f_w = float(g["f_w"])
    plan = nus.BandPlan.from_centers(g["centers"], f_w, float(g["f_max"]))
    opts = nus.MtnufftEstimator.Options(k_tapers=7, epsilon=1e-9, taper_mode="exact_nominal")
    est = nus.MtnufftEstimator(grid, nus.SignalBand(float(g["f_max"])), plan, opts)
    assert est.method() == "mtnufft0"
    r = est.estimate(g["x"])
    assert r.method == "mtnufft0" and int(g["method"]) == 1
    assert rel_l2(r.power, g["power"]) <= 1e-6
    print("MTNUFFT0 relL2(P) =", rel_l2(r.power, g["power"]))
