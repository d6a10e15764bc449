"""Diagnose the C4 taper shape difference: GPU DPSS -> GPU spline vs GPU DPSS -> C spline at the
C4 sample times (separates the spline stage from the DPSS stage)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_01943_b200 as nus  # noqa: E402
from paper_2407_01943_b200 import workloads as W  # noqa: E402
from oracle import C  # noqa: E402

for lg in [int(v) for v in sys.argv[1:]]:
    wl = W.c4(n=1 << lg, n_centers=1 << (lg - 2))
    t = wl.times
    n = t.size
    h = (t[-1] - t[0]) / (n - 1)
    d = nus.dpss_uniform(n, 8.0, 15, concentrations=False).tapers
    g = nus.SamplingGrid(t)
    ws = nus.api.taper_spline(g, nus.SignalBand(wl.f_max), float(wl.f_w[0]), 15)
    knots = t[0] + h * np.arange(n)
    worst = []
    for j in (0, 7, 14):
        r = C.spline(knots, d[j], t)
        a = ws[j] * np.sign(np.dot(ws[j], r))
        diff = np.abs(a - r)
        i = int(diff.argmax())
        worst.append((j, float(diff.max() / np.abs(r).max()), i, float(t[i]), float((t[i] - t[0]) / h)))
    print(f"2^{lg}: (taper, max|gpu spline - C spline| / max, index, t, knot pos) {worst}", flush=True)
