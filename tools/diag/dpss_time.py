import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
for lg, nw, k in [(20, 4, 7), (22, 8, 15), (24, 8, 15)]:
    t0 = time.time()
    d = nus.dpss_uniform(1 << lg, nw, k)
    print("n 2^%d K %d: %.2f s" % (lg, k, time.time() - t0), d.eigenvalues[:3] if hasattr(d, "eigenvalues") else "", flush=True)
