"""Re-run the full-C4 taper shape check of tests/test_gpu_fullsize.py per taper: the estimator's
tapers vs the long-double DPSS + C spline, and the GPU DPSS + C spline vs the same."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_01943_b200 as nus  # noqa: E402
from paper_2407_01943_b200 import workloads as W  # noqa: E402
from oracle import C  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
threads = int(sys.argv[2]) if len(sys.argv) > 2 else 15
wl = W.c4(n=1 << lg, n_centers=1 << (lg - 2))
t = wl.times
n = t.size
g = nus.SamplingGrid(t)
plan = nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max)
est = nus.MtnufftEstimator(g, nus.SignalBand(wl.f_max), plan, nus.MtnufftEstimator.Options(k_tapers=15, epsilon=1e-9))
w = est.tapers().weights_matrix().copy()
del est
h = (t[-1] - t[0]) / (n - 1)
knots = t[0] + h * np.arange(n)
t0 = time.time()
dp, ev = C.dpss(n, 8.0, 15, threads=threads)
print(f"long-double dpss {time.time() - t0:.1f}s", flush=True)
dg = nus.dpss_uniform(n, 8.0, 15, concentrations=False).tapers
for j in range(15):
    r = C.spline(knots, dp[j], t)
    r /= np.linalg.norm(r)
    a = w[j] / np.linalg.norm(w[j])
    a = a * np.sign(np.dot(a, r))
    d = np.abs(a - r)
    e_dp = np.abs(dg[j] * np.sign(np.dot(dg[j], dp[j])) - dp[j])
    print(f"taper {j}: shape {d.max() / np.abs(r).max():.2e} at {int(d.argmax())} (t={t[int(d.argmax())]:.6f}); "
          f"dpss gpu-ld {e_dp.max():.2e} at {int(e_dp.argmax())}; max|r| {np.abs(r).max():.3e} ev {ev[j]:.6e}", flush=True)
