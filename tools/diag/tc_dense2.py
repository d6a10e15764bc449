import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from oracle import C
FAST = nus.NufftPathPolicy.force_fast
c = np.arange(4096) / 64.0
for ncl in [1, 4, 10, 40]:
    for n in [2000, 5000, 10000, 20000, 50000]:
        rng = np.random.default_rng(n + ncl)
        t = np.unique(np.sort(np.concatenate([d + rng.uniform(0, 0.3, n // ncl) for d in range(ncl)])))
        y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
        for eps in [1e-6]:
            plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
            got = plan.execute(y)
            ref = C.nufft_fast(t, c, eps, y)
            r = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            print("clusters", ncl, "n", t.size, "relL2", r, flush=True)
