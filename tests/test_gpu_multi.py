"""The multi-GPU estimator in one process (C-ABI nus_mtnufft_multi_*, multi.cu) against the
single-GPU estimator: channel, taper and sample sharding (the sample split's spread storing into
the owners' peer slots, double-buffered).  This box has one GPU, so the device list repeats
device 0: every part is a separate estimator with its own stream, slots and events, and every
cross-part order is an event wait (no kernel waits on another), exactly the multi-GPU code path
minus the NVLink hop.  Reference behaviour: the serial loops of nufft.cpp:194-227 and
estimators.cpp:106-122 -- P must not depend on how the work is split.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from paper_2407_01943_b200.api import MultiDeviceEstimator, _Estimator
from conftest import ROOT, rel_l2
from oracle import C

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("parts", [2, 3])
def test_channel_sharding_equals_single_device(parts):
    wl = W.c3(channels=5, n=1 << 15)
    centers = 2500.0 * np.arange(1 << 14) / ((1 << 14) - 1)
    single = _Estimator(wl.times, centers, wl.f_max, wl.f_w, 9, 1e-5, 1, "f32", 0)
    multi = MultiDeviceEstimator(wl.times, centers, wl.f_max, wl.f_w, 9, 1e-5, [0] * parts, "channels", "f32",
                                 policy=nus.NufftPathPolicy.force_fast)
    assert np.array_equal(multi.tapers(), single.tapers())
    p1, pm = single.power(wl.values), multi.estimate(wl.values)
    assert max(rel_l2(pm[c], p1[c]) for c in range(5)) < 1e-12
    assert multi.peer_bytes() == 0


@pytest.mark.parametrize("kern", ["gaussian", "es"])
@pytest.mark.parametrize("parts", [2, 3])
def test_taper_sharding_equals_single_device(parts, kern):
    wl = W.c2(n=1 << 18)
    single = _Estimator(wl.times, wl.centers, wl.f_max, wl.f_w, 7, 1e-9, 1, "f64", 0)
    multi = MultiDeviceEstimator(wl.times, wl.centers, wl.f_max, wl.f_w, 7, 1e-9, [0] * parts, "tapers")
    assert np.array_equal(multi.tapers()[0], single.tapers()[0])  # one taper build on devices[0]
    p1, pm = single.power(wl.values)[0], multi.estimate(wl.values)[0]
    assert rel_l2(pm, p1) < 1e-13
    assert multi.peer_bytes() == (parts - 1) * wl.centers.size * 8


@pytest.mark.parametrize("kern", ["gaussian", "es"])
@pytest.mark.parametrize("parts,k,cfg", [(2, 7, "c2"), (3, 7, "c2"), (2, 15, "c4"), (4, 15, "c4")])
def test_sample_sharding_fused_peer_slots_equals_single_device(parts, k, cfg, kern):
    """C2 structure (< 1 wrap) and C4 structure (400 windows, ~12 wraps, K = 15 padded to a multiple
    of the parts): P equals the single-device P; consecutive spectra alternate the slot parities
    and stay exact (x1, x2, x1 -> the first and third identical)."""
    if cfg == "c2":
        wl = W.c2(n=1 << 18)
    else:
        wl = W.c4(n=1 << 18, n_centers=1 << 16)
    single = _Estimator(wl.times, wl.centers, wl.f_max, wl.f_w, k, 1e-9, 1, "f64", 0)
    tap = single.tapers()[0]
    multi = MultiDeviceEstimator(wl.times, wl.centers, wl.f_max, wl.f_w, k, 1e-9, [0] * parts, "samples", tapers=tap)
    x1, x2 = wl.values, np.roll(wl.values, 777)
    a = multi.estimate(x1)[0]
    b = multi.estimate(x2)[0]
    c = multi.estimate(x1)[0]
    assert np.array_equal(a, c)
    assert rel_l2(a, single.power(x1)[0]) < 1e-12
    assert rel_l2(b, single.power(x2)[0]) < 1e-12
    ref = C.mtnufft_power(wl.times, tap, x1, wl.centers, 1e-9)
    assert rel_l2(a, ref) < (1e-8 if kern == "gaussian" else 2e-8)
    assert multi.peer_bytes() > 0


def test_sample_sharding_builds_the_full_grid_tapers():
    """Without injected tapers the multi estimator builds the full grid's tapers once (devices[0]):
    identical to the single-device estimator's."""
    wl = W.c2(n=1 << 17)
    single = _Estimator(wl.times, wl.centers, wl.f_max, wl.f_w, 7, 1e-9, 1, "f64", 0)
    multi = MultiDeviceEstimator(wl.times, wl.centers, wl.f_max, wl.f_w, 7, 1e-9, [0, 0], "samples")
    assert np.array_equal(multi.tapers()[0], single.tapers()[0])
    assert rel_l2(multi.estimate(wl.values)[0], single.power(wl.values)[0]) < 1e-12


def test_multi_rejects_bad_arguments():
    wl = W.c2(n=1 << 14)
    with pytest.raises(nus.InvalidArgument):
        MultiDeviceEstimator(wl.times, wl.centers, wl.f_max, wl.f_w, 7, 1e-9, [], "samples")
    with pytest.raises(nus.InvalidArgument):  # more parts than tapers
        MultiDeviceEstimator(wl.times, wl.centers, wl.f_max, wl.f_w, 2, 1e-9, [0, 0, 0], "tapers")
    with pytest.raises(nus.InvalidArgument):
        MultiDeviceEstimator(wl.times, wl.centers, wl.f_max, wl.f_w, 7, 1e-9, [0, 99], "samples")


def test_cpp_dropin_options_devices():
    """C++: MtnufftEstimator::Options::devices / sharding (tests/dropin/multi_device.cpp, `make
    dropin_multi`): taper and sample sharding over 2 and 3 parts equal the one-device estimator."""
    exe = os.path.join(ROOT, "tests", "dropin", "multi_device")
    assert os.path.exists(exe), "make dropin_multi"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
