"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container (where /root/reference exists and oracle/_ref is
compiled from its sources):  python tests/golden/make_golden.py
The outputs (tests/golden/*.npz) are small and committed; the GPU box never
needs the reference tree.

Every case mirrors a reference test or a BASELINE config:
  nufft_lattice.npz  test_nufft.cpp:81-96  (fast vs direct over eps x N x I) on the
                     reference's own jitter grids (simkit generate_grid) and Rng draws
  nufft_small.npz    test_nufft.cpp:52-79,113-152 known answers / DFT / path selection
  dpss.npz           dpss_uniform(512, 4.0, 7) and (50, 2.5, 4) from the reference
  spline.npz         test_eig.cpp:252-270 sin case (max error 3.855517e-3)
  gpss.npz           gpss_interpolated on jitter / arithmetic / uniform grids (N=50)
  c1.npz             BASELINE config C1 through the full reference MtnufftEstimator (Oracle-A)
  ftest_c1.npz       the reference f_test on C1's eigencoefficients
  bins_many_wrap.npz first_cell_ on a clustered, many-wrap grid (C4-like, 2^15 samples)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import REF, build  # noqa: E402
from paper_2407_01943_b200 import workloads as W  # noqa: E402


def rng_complex(n, seed):
    g = REF.rng_gauss(seed, 2 * n)
    return g[0::2] + 1j * g[1::2]


def main():
    build(ref=True)
    out = {}
    # test_nufft.cpp:81-96 lattice
    cases = []
    for eps in (1e-4, 1e-6, 1e-8):
        for n in (50, 500):
            for count in (64, 1024):
                t = REF.generate_grid(1, n, seed=n + count)
                c = np.arange(count) * (0.5 / count)
                y = rng_complex(n, count + 7)
                fast = REF.plan_execute(t, c, eps, y, policy=1)
                direct = REF.ndft_direct(t, y, c)
                j0 = REF.first_cells(t, c, eps)
                cases.append((eps, n, count, t, y, c, fast, direct, j0))
    np.savez_compressed(
        os.path.join(HERE, "nufft_lattice.npz"),
        **{f"case{i}_{k}": v for i, cs in enumerate(cases)
           for k, v in zip(["eps", "n", "count", "t", "y", "c", "fast", "direct", "j0"], cs)},
        ncases=len(cases))

    # small known answers
    t16 = np.arange(16.0)
    x16 = rng_complex(16, 3)
    c16 = np.arange(16) / 16.0
    t64 = np.arange(64.0)
    x64 = rng_complex(64, 21)
    c64 = np.arange(64) / 64.0
    t200 = REF.generate_grid(1, 200, seed=5)
    c256 = np.arange(256) * (0.5 / 256.0)
    y200 = rng_complex(200, 11)
    np.savez_compressed(
        os.path.join(HERE, "nufft_small.npz"),
        t16=t16, x16=x16, c16=c16, dft16=REF.ndft_direct(t16, x16, c16),
        t64=t64, x64=x64, c64=c64, fast64=REF.plan_execute(t64, c64, 1e-8, x64, policy=1),
        t200=t200, c256=c256, y200=y200,
        loose200=REF.plan_execute(t200, c256, 1e-4, y200, policy=1),
        tight200=REF.plan_execute(t200, c256, 1e-10, y200, policy=1),
        direct200=REF.ndft_direct(t200, y200, c256),
        info_small=np.array([REF.plan_info(REF.generate_grid(1, 50, seed=1), np.arange(51) * 0.01, 1e-8)["path"] == "fast"]),
        info_big=np.array([REF.plan_info(REF.generate_grid(1, 500, seed=2), np.arange(64) * (0.5 / 64), 1e-8)["path"] == "fast"]),
        grid50=REF.generate_grid(1, 50, seed=1), grid500=REF.generate_grid(1, 500, seed=2))

    # DPSS
    t512, c512 = REF.dpss(512, 4.0, 7)
    t50, c50 = REF.dpss(50, 2.5, 4)
    np.savez_compressed(os.path.join(HERE, "dpss.npz"), tap512=t512, conc512=c512, tap50=t50, conc50=c50)

    # spline sin case
    xs = np.arange(50.0)
    ys = np.sin(2 * np.pi * xs / 10.0)
    xq = xs[:-1] + 0.5
    np.savez_compressed(os.path.join(HERE, "spline.npz"), xs=xs, ys=ys, xq=xq, ref=REF.spline(xs, ys, xq))

    # gpss on the paper's N=50 schemes
    gp = {}
    for scheme, name in ((0, "uniform"), (1, "jitter"), (3, "arithmetic")):
        t = REF.generate_grid(scheme, 50, seed=4)
        gp[f"t_{name}"] = t
        gp[f"w_{name}"] = REF.gpss_interpolated(t, 0.5, 0.05, 4)
        gp[f"q_{name}"] = REF.quadform(t, 0.5, gp[f"w_{name}"])
    np.savez_compressed(os.path.join(HERE, "gpss.npz"), **gp)

    # C1 through the full reference estimator (Oracle-A)
    wl = W.c1()
    p, w, flags = REF.mtnufft(wl.times, wl.values, wl.f_max, wl.centers, float(wl.f_w[0]), wl.k, wl.eps)
    j0 = REF.first_cells(wl.times, wl.centers, wl.eps)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), t=wl.times, x=wl.values, centers=wl.centers,
                        f_max=wl.f_max, f_w=wl.f_w[0], k=wl.k, eps=wl.eps, power=p, tapers=w,
                        flags=flags, first_cells=j0)
    # harmonic F-test on the C1 eigencoefficients (inference.cpp:132-186), reference tapers
    f, amp, fflags, crit = REF.f_test(wl.times, w, wl.values, wl.centers, wl.eps, wl.f_max, float(wl.f_w[0]))
    np.savez_compressed(os.path.join(HERE, "ftest_c1.npz"), f=f, amp=amp, flags=fflags, crit=crit)

    # many-wrap clustered grid (C4-like at 2^15 samples, 2^13 dyadic centres)
    c4 = W.c4(n=1 << 15, n_centers=1 << 13, windows=50)
    np.savez_compressed(os.path.join(HERE, "bins_many_wrap.npz"), t=c4.times, centers=c4.centers,
                        eps=1e-9, first_cells=REF.first_cells(c4.times, c4.centers, 1e-9))
    total = sum(os.path.getsize(os.path.join(HERE, f)) for f in os.listdir(HERE) if f.endswith(".npz"))
    print(f"golden fixtures written ({total / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
