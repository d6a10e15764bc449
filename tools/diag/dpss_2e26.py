"""Diagnose DPSS accuracy at 2^25 / 2^26 (NW 8, K 15): GPU coarse-start path vs GPU full
bisection path vs the long-double restatement."""
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


for lg in [int(v) for v in sys.argv[1:]]:
    n = 1 << lg
    t0 = time.time()
    dc = nus.dpss_uniform(n, 8.0, 15, concentrations=False)
    t1 = time.time()
    os.environ["NUS_DPSS_COARSE"] = str(1 << 40)
    db = nus.dpss_uniform(n, 8.0, 15, concentrations=False)
    del os.environ["NUS_DPSS_COARSE"]
    t2 = time.time()
    tl, el = C.dpss(n, 8.0, 15, threads=15)
    t3 = time.time()
    print(f"2^{lg}: coarse {t1 - t0:.1f}s bisection {t2 - t1:.1f}s long-double {t3 - t2:.1f}s", flush=True)
    for name, a, b in (("coarse-bisect", dc.tapers, db.tapers), ("coarse-ld", dc.tapers, tl),
                       ("bisect-ld", db.tapers, tl)):
        d = np.abs(align(a, b) - b)
        per = d.max(axis=1)
        arg = d.argmax(axis=1) / n
        print(f"  {name}: max {per.max():.3e}  per taper {np.array2string(per, precision=1)}  at {np.array2string(arg, precision=3)}")
    print(f"  eig coarse-ld rel {np.abs(dc.eigenvalues / el - 1).max():.2e}  bisect-ld {np.abs(db.eigenvalues / el - 1).max():.2e}"
          f"  gaps {np.array2string(-np.diff(el), precision=3)}", flush=True)
