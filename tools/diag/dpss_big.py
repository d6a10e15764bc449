import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from oracle import C
for lg in [21, 22]:
    n = 1 << lg
    t0 = time.time(); d = nus.dpss_uniform(n, 8.0, 15, concentrations=False); t1 = time.time()
    if lg == 21:
        tc, ev = C.dpss(n, 8.0, 15); t2 = time.time()
        s = np.sign(np.sum(d.tapers * tc, axis=1, keepdims=True))
        print(lg, "gpu %.1fs oracle %.1fs" % (t1 - t0, t2 - t1), "maxdiff", np.abs(d.tapers * s - tc).max(), "ev rel", np.abs(d.eigenvalues / ev - 1).max(), flush=True)
    else:
        print(lg, "gpu %.1fs" % (t1 - t0), flush=True)
