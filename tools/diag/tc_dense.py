import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from oracle import C
FAST = nus.NufftPathPolicy.force_fast
c = np.arange(4096) / 64.0
for width in [0.5, 0.2, 0.05, 0.01]:
    for n in [20, 33, 40, 64, 100, 200, 500, 2000]:
        rng = np.random.default_rng(n)
        t = np.unique(np.sort(10 + rng.uniform(0, width, n)))
        y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
        ok = True
        for eps in [1e-3, 1e-6]:
            plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
            got = plan.execute(y)
            ref = C.nufft_fast(t, c, eps, y)
            r = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            if r > 1e-10:
                print("width", width, "n", n, "eps", eps, "relL2", r, "cells", (t[-1]-t[0])/64*8192, flush=True)
print("done")
