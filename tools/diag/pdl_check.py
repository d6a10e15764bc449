import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
from paper_2407_01943_b200.api import _Estimator
wl = W.c2()
est = _Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), wl.k, wl.eps, 1, "f64", 0)
x = wl.values
p1 = est.power(x)[0]; p2 = est.power(x)[0]
xs = np.stack([np.roll(x, 17 * i) for i in range(6)] + [x])
pb = est.power_batch(xs)
print(os.environ.get("NUS_PDL"), os.environ.get("NUS_KERNEL"), "repeat equal", np.array_equal(p1, p2), "batch-last vs single maxrel",
      np.abs(pb[-1, 0] - p1).max() / p1.max(), [float(np.abs(pb[i,0]-est.power(xs[i])[0]).max()/p1.max()) for i in range(len(xs))], flush=True)
