"""DPSS at large N: the parallel two-sided recurrence (default) vs the sequential double-double
inverse iteration (NUS_DPSS_RECURRENCE=0) vs the long-double restatement; NW 8, K 15."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2407_01943_b200 as nus  # noqa: E402
from oracle import C  # noqa: E402


def align(a, b):
    s = np.sign(np.sum(a * b, axis=-1, keepdims=True))
    s[s == 0] = 1
    return a * s


ld = "--ld" in sys.argv
for lg in [int(v) for v in sys.argv[1:] if v.isdigit()]:
    n = 1 << lg
    os.environ.pop("NUS_DPSS_RECURRENCE", None)
    nus.dpss_uniform(1 << 20, 8.0, 15, concentrations=False)  # warm-up
    t0 = time.time()
    dr = nus.dpss_uniform(n, 8.0, 15, concentrations=False)
    t1 = time.time()
    os.environ["NUS_DPSS_RECURRENCE"] = "0"
    di = nus.dpss_uniform(n, 8.0, 15, concentrations=False)
    t2 = time.time()
    os.environ.pop("NUS_DPSS_RECURRENCE", None)
    d = np.abs(align(dr.tapers, di.tapers) - di.tapers).max(axis=1)
    print(f"2^{lg}: recurrence {t1 - t0:.2f}s, inverse iteration {t2 - t1:.2f}s; max|rec - ii| per taper "
          f"{np.array2string(d, precision=1)}; eig rel {np.abs(dr.eigenvalues / di.eigenvalues - 1).max():.1e}",
          flush=True)
    if ld:
        tl, el = C.dpss(n, 8.0, 15, threads=15)
        e1 = np.abs(align(dr.tapers, tl) - tl).max()
        e2 = np.abs(align(di.tapers, tl) - tl).max()
        print(f"  vs long double: recurrence {e1:.2e}, inverse iteration {e2:.2e}", flush=True)
