import sys, time, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
n = 1 << 23
os.environ["NUS_DPSS_COARSE"] = str(1 << 30)
e = nus.dpss_uniform(n, 8.0, 15, concentrations=False)
del os.environ["NUS_DPSS_COARSE"]
for it in ["1", "2"]:
    os.environ["NUS_DPSS_COARSE_ITERS"] = it
    t0 = time.time(); d = nus.dpss_uniform(n, 8.0, 15, concentrations=False); t1 = time.time()
    s = np.sign(np.sum(d.tapers * e.tapers, axis=1, keepdims=True))
    print("iters", it, "%.1fs" % (t1 - t0), "maxdiff vs bisection", np.abs(d.tapers * s - e.tapers).max(), "ev", np.abs(d.eigenvalues / e.eigenvalues - 1).max(), flush=True)
