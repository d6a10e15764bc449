"""Quick end-to-end GPU sanity run (development aid; the real checks are the pytest suite)."""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])

import paper_2407_01943_b200 as nus  # noqa: E402
from paper_2407_01943_b200 import workloads as W  # noqa: E402
from oracle import C, REF, ref_available  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def step(name, fn):
    t0 = time.time()
    try:
        out = fn()
        print(f"[ok] {name} ({time.time() - t0:.2f}s): {out}", flush=True)
    except Exception:
        print(f"[FAIL] {name} ({time.time() - t0:.2f}s)", flush=True)
        traceback.print_exc()


print(nus._capi.device_info())

wl = W.small(n=2000, k=4)
g = nus.SamplingGrid(wl.times)


def bins():
    p = nus.NufftPlan(g, wl.centers, 1e-9, nus.NufftPathPolicy.force_fast)
    a = p.first_cells()
    b = C.first_cells(wl.times, wl.centers, 1e-9)
    return dict(equal=bool(np.array_equal(a, b)), path=int(p.path()), mr=p.grid_size())


step("bins small", bins)


def execute():
    rng = np.random.default_rng(1)
    y = rng.standard_normal(g.n_samples()) + 1j * rng.standard_normal(g.n_samples())
    p = nus.NufftPlan(g, wl.centers, 1e-9, nus.NufftPathPolicy.force_fast)
    a = p.execute(y)
    b = C.nufft_fast(wl.times, wl.centers, 1e-9, y)
    d = C.ndft_direct(wl.times, y, wl.centers)
    return dict(rel_vs_oracle=rel(a, b), maxdev_direct=float(np.abs(a - d).max()),
                bound=1e-9 * float(np.abs(y).sum()))


step("execute small", execute)


def direct():
    rng = np.random.default_rng(2)
    y = rng.standard_normal(g.n_samples()) + 1j * rng.standard_normal(g.n_samples())
    a = nus.ndft_direct(g, y, wl.centers[:64])
    b = C.ndft_direct(wl.times, y, wl.centers[:64])
    return rel(a, b)


step("ndft direct", direct)


def dpss():
    d = nus.dpss_uniform(4096, 4.0, 7)
    tc, ev = C.dpss(4096, 4.0, 7)
    s = np.sign(np.sum(d.tapers * tc, axis=1))[:, None]
    return dict(maxdiff=float(np.abs(d.tapers - s * tc).max()), ev_rel=rel(d.eigenvalues, ev),
                conc=d.concentrations.tolist())


step("dpss 4096", dpss)


def gpss():
    w = nus.gpss_interpolated(g, nus.SignalBand(wl.f_max), float(wl.f_w[0]), 4).weights_matrix()
    wc, q = C.gpss_interpolated(wl.times, wl.f_max, float(wl.f_w[0]), 4)
    s = np.sign(np.sum(w * wc, axis=1))[:, None]
    return dict(maxdiff=float(np.abs(w - s * wc).max()), scale=float(np.abs(wc).max()))


step("gpss small", gpss)


def mt_injected():
    wc, _ = C.gpss_interpolated(wl.times, wl.f_max, float(wl.f_w[0]), 4)
    est = nus.MtnufftEstimator(g, nus.SignalBand(wl.f_max),
                               nus.BandPlan.from_centers(wl.centers, float(wl.f_w[0]), wl.f_max),
                               nus.MtnufftEstimator.Options(k_tapers=4, epsilon=1e-9), tapers=wc)
    p = est.estimate(wl.values).power
    pc = C.mtnufft_power(wl.times, wc, wl.values, wl.centers, 1e-9)
    return rel(p, pc)


step("mtnufft injected small", mt_injected)


def c1_full():
    wl1 = W.c1()
    g1 = nus.SamplingGrid(wl1.times)
    plan = nus.BandPlan.from_centers(wl1.centers, float(wl1.f_w[0]), wl1.f_max)
    est = nus.MtnufftEstimator(g1, nus.SignalBand(wl1.f_max), plan,
                               nus.MtnufftEstimator.Options(k_tapers=7, epsilon=1e-9))
    p = est.estimate(wl1.values).power
    out = dict(setup=est.setup_ms())
    if ref_available():
        pr, wr, _ = REF.mtnufft(wl1.times, wl1.values, wl1.f_max, wl1.centers, float(wl1.f_w[0]), 7, 1e-9)
        out["rel_vs_reference"] = rel(p, pr)
    return out


step("c1 full vs reference", c1_full)


def c2_f64():
    wl2 = W.c2()
    g2 = nus.SamplingGrid(wl2.times)
    plan = nus.BandPlan.from_centers(wl2.centers, float(wl2.f_w[0]), wl2.f_max)
    t0 = time.time()
    est = nus.MtnufftEstimator(g2, nus.SignalBand(wl2.f_max), plan,
                               nus.MtnufftEstimator.Options(k_tapers=7, epsilon=1e-9))
    t1 = time.time()
    p = est.estimate(wl2.values).power
    t2 = time.time()
    for _ in range(3):
        est.estimate(wl2.values)
    t3 = time.time()
    return dict(setup_s=t1 - t0, setup=est.setup_ms(), first_est_s=t2 - t1, est_s=(t3 - t2) / 3,
                pmax=float(p.max()))


step("c2 f64", c2_f64)
print("launches", nus._capi.launch_count())
