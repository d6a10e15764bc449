import sys, time, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
for lg in [23, 24]:
    n = 1 << lg
    t0 = time.time(); d = nus.dpss_uniform(n, 8.0, 15, concentrations=False); t1 = time.time()
    os.environ["NUS_DPSS_COARSE"] = str(1 << 30)
    t2 = time.time(); e = nus.dpss_uniform(n, 8.0, 15, concentrations=False); t3 = time.time()
    del os.environ["NUS_DPSS_COARSE"]
    s = np.sign(np.sum(d.tapers * e.tapers, axis=1, keepdims=True))
    print(lg, "coarse-start %.1fs bisection %.1fs" % (t1 - t0, t3 - t2), "maxdiff", np.abs(d.tapers * s - e.tapers).max(),
          "ev rel", np.abs(d.eigenvalues / e.eigenvalues - 1).max(), flush=True)
