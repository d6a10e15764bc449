import sys, os, numpy as np
sys.path.insert(0, '.')
import torch
from paper_2407_01943_b200 import _capi as CAPI, workloads as W
from paper_2407_01943_b200.api import _Estimator
wl = W.c5(n=1 << 22, k=15)
rng = np.random.default_rng(0)
tap = rng.standard_normal((1, 15, wl.n)) * 1e-3
for eps in (1e-6, 1e-9):
    est = _Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), 15, eps, 1, "f64", 0, tapers=tap)
    x = torch.tensor(wl.values, device="cuda"); pw = torch.empty(wl.centers.size, dtype=torch.float64, device="cuda")
    for _ in range(3):
        CAPI.check(CAPI.lib().nus_mtnufft_estimate_device(est.h, x.data_ptr(), 0, pw.data_ptr(), None, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
