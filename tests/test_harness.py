"""Speed / error harness and its input generators.

CPU: the simkit restatement (paper_2407_01943_b200/simkit.py) reproduces the reference's own
Rng and the paper's four sampling grids bit for bit (simkit.cpp:19-141).
GPU: run_error_analysis for mtnufft / mtnufft0 against the reference's run_error_analysis
(bench.cpp:130-204, live through oracle/_ref/libnusref.so) on the same seeds.
"""
import json

import numpy as np
import pytest

from oracle import REF, ref_available


def _simkit():
    from paper_2407_01943_b200 import simkit
    return simkit


@pytest.mark.skipif(not ref_available(), reason="reference library not built")
def test_rng_matches_reference():
    sk = _simkit()
    for seed in (0, 1, 20240702, 2 ** 63 + 5):
        r = sk.Rng(seed)
        assert np.array_equal(np.array([r.next_gauss() for _ in range(101)]), REF.rng_gauss(seed, 101))
        r = sk.Rng(seed)
        assert np.array_equal(np.array([r.next_uniform() for _ in range(64)]), REF.rng_uniform(seed, 64))


@pytest.mark.skipif(not ref_available(), reason="reference library not built")
@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_generate_grid_matches_reference(scheme):
    sk = _simkit()
    for seed in (0, 7, sk.Rng.substream(20240702, scheme)):
        g = sk.generate_grid(sk.SimConfig(scheme=scheme, n=50, seed=seed))
        assert np.array_equal(np.asarray(g.times()), REF.generate_grid(scheme, 50, seed=seed))


def test_harness_rejects_out_of_scope_methods():
    from paper_2407_01943_b200 import api, harness
    with pytest.raises(api.InvalidArgument, match="outside the MTNUFFT path"):
        harness.run_error_analysis(["bg_fixed"], [0], 4, 1)
    with pytest.raises(api.InvalidArgument):
        harness.run_error_analysis(["mtnufft"], [0], 1, 1)  # trials >= 2
    with pytest.raises(api.InvalidArgument):
        harness.run_speed_analysis(["mtnufft"], [0], 5)  # reps >= 10


@pytest.mark.gpu
@pytest.mark.skipif(not ref_available(), reason="reference library not built")
def test_error_analysis_matches_reference():
    from paper_2407_01943_b200 import harness
    methods, schemes, trials, seed = ["mtnufft", "mtnufft0"], [0, 1, 2, 3], 4, 20240702
    ours = harness.run_error_analysis(methods, schemes, trials, seed)
    ref = REF.run_error_analysis([0, 1], schemes, trials, seed)
    assert len(ours) == len(ref) == 8
    for o, r in zip(ours, ref):
        assert np.array_equal(o.centers, r["centers"]) and np.array_equal(o.flags, r["flags"])
        ok = ~np.isnan(r["mean"])
        assert np.array_equal(ok, ~np.isnan(o.mse_db_mean))
        # squared dB errors of the same estimates: agree to the taper / NUFFT accuracy
        assert np.abs(o.mse_db_mean[ok] - r["mean"][ok]).max() <= 1e-6 * max(1.0, np.abs(r["mean"][ok]).max())
        assert np.abs(o.mse_db_sem[ok] - r["sem"][ok]).max() <= 1e-6 * max(1.0, np.abs(r["sem"][ok]).max())
    doc = json.loads(harness.write_error_reports_json(ours, "h"))
    assert doc["kind"] == "error_analysis" and len(doc["reports"]) == 8


@pytest.mark.gpu
def test_speed_analysis_reports():
    from paper_2407_01943_b200 import harness
    cfg = harness.SpeedConfig(min_batch_seconds=0.01, max_cell_seconds=5.0)
    reps = harness.run_speed_analysis(["mtnufft"], [0, 1], 10, cfg)
    assert len(reps) == 2
    for r in reps:
        assert r.spectra_per_second_mean > 0 and r.calls >= 10 and r.batches >= 2
    doc = json.loads(harness.write_speed_reports_json(reps, "h"))
    assert doc["kind"] == "speed_analysis" and doc["reports"][0]["method"] == "mtnufft"
