import sys, time, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from oracle import C
for n, tw, k in [(1 << 20, 4.0, 7), (1 << 20, 8.0, 15), (1 << 21, 5.0, 9), (1 << 22, 2.0, 3)]:
    t0 = time.time(); d = nus.dpss_uniform(n, tw, k, concentrations=False); t1 = time.time()
    tc, ev = C.dpss(n, tw, k); t2 = time.time()
    s = np.sign(np.sum(d.tapers * tc, axis=1, keepdims=True))
    print(n, tw, k, "gpu %.2fs oracle %.2fs" % (t1 - t0, t2 - t1), "maxdiff", np.abs(d.tapers * s - tc).max(), "ev rel", np.abs(d.eigenvalues / ev - 1).max(), flush=True)
