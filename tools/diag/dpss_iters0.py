import sys, time, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
for lg in [21, 23]:
    n = 1 << lg
    os.environ["NUS_DPSS_COARSE"] = str(1 << 30)
    e = nus.dpss_uniform(n, 8.0, 15, concentrations=False)
    os.environ["NUS_DPSS_COARSE"] = str(1 << 20)
    for it in ["0", "1"]:
        os.environ["NUS_DPSS_COARSE_ITERS"] = it
        t0 = time.time(); d = nus.dpss_uniform(n, 8.0, 15, concentrations=False); t1 = time.time()
        s = np.sign(np.sum(d.tapers * e.tapers, axis=1, keepdims=True))
        print(lg, "iters", it, "%.1fs" % (t1 - t0), "maxdiff", np.abs(d.tapers * s - e.tapers).max(), "rel ev", np.abs(d.eigenvalues / e.eigenvalues - 1).max(), flush=True)
