import sys, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from oracle import C
FAST = nus.NufftPathPolicy.force_fast
rng = np.random.default_rng(17)
n = 20000
t = np.unique(np.sort(np.concatenate([d + rng.uniform(0, 0.3, n // 40) for d in range(40)])))
y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
for name, c in [("wrap5", np.arange(4096) / 8.0), ("wrap0.6", np.arange(4096) / 64.0), ("big", np.arange(1 << 17) / 8.0)]:
    sub = np.arange(0, c.size, max(1, c.size // 600))
    direct = C.ndft_direct(t, y, c[sub])
    for kern in ["gaussian", "es"]:
        for eps in [1e-3, 1e-6, 1e-9, 1e-12]:
            with nus.spread_kernel(kern):
                plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
            got = plan.execute(y)
            err = np.abs(got[sub] - direct).max() / np.abs(y).sum()
            print(name, kern, eps, "mr", plan.grid_size(), "support", plan.support(), "err/eps", err / eps, flush=True)
