"""Diagnose the full-C4 taper shape check: the estimator's normalised tapers vs the GPU DPSS +
spline alone (isolates the normalisation stage), at C4's structure for the given log2 N."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_01943_b200 as nus  # noqa: E402
from paper_2407_01943_b200 import workloads as W  # noqa: E402


def shape(a):
    return a / np.linalg.norm(a)


for lg in [int(v) for v in sys.argv[1:]]:
    wl = W.c4(n=1 << lg, n_centers=1 << (lg - 2))
    t = wl.times
    g = nus.SamplingGrid(t)
    plan = nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max)
    est = nus.MtnufftEstimator(g, nus.SignalBand(wl.f_max), plan,
                               nus.MtnufftEstimator.Options(k_tapers=15, epsilon=1e-9))
    we = est.tapers().weights_matrix()
    del est
    ws = nus.api.taper_spline(g, nus.SignalBand(wl.f_max), float(wl.f_w[0]), 15)
    out = []
    for j in range(15):
        a, b = shape(we[j]), shape(ws[j])
        b = b * np.sign(np.dot(a, b))
        d = np.abs(a - b)
        out.append(f"{j}:{d.max() / np.abs(b).max():.1e}@{int(d.argmax())}")
    print(f"2^{lg}: estimator vs dpss+spline shapes: {' '.join(out)}", flush=True)
