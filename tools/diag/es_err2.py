import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from oracle import C
FAST = nus.NufftPathPolicy.force_fast
rng = np.random.default_rng(17)
for n in [2000, 5000, 20000]:
    t = np.unique(np.sort(np.concatenate([d + rng.uniform(0, 0.3, n // 40) for d in range(40)])))
    y = rng.standard_normal(t.size) + 1j * rng.standard_normal(t.size)
    c = np.arange(4096) / 64.0
    sub = np.arange(0, c.size, 7)
    direct = C.ndft_direct(t, y, c[sub])
    for eps in [1e-3, 1e-6]:
        plan = nus.NufftPlan(nus.SamplingGrid(t), c, eps, FAST)
        got = plan.execute(y)
        ref = C.nufft_fast(t, c, eps, y)
        err = np.abs(got[sub] - direct).max() / np.abs(y).sum()
        print(os.environ.get("NUS_SPREAD", "tc"), n, eps, "err/eps", err / eps, "vs C gaussian fast relL2",
              np.linalg.norm(got - ref) / np.linalg.norm(ref), "C fast vs direct", np.abs(ref[sub]-direct).max()/np.abs(y).sum()/eps, flush=True)
