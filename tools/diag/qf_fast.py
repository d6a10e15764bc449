import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2407_01943_b200 as nus
from paper_2407_01943_b200 import workloads as W
cases = [("c1", W.c1()), ("c2_2^16", W.c2(n=1 << 16)), ("c4_2^16", W.c4(n=1 << 16, n_centers=1 << 12, windows=20)),
         ("c3_2^16", W.c3(channels=1, n=1 << 16)), ("c5_2^16", W.c5(n=1 << 16)), ("small", W.small(n=3000))]
for name, wl in cases:
    t = wl.times if wl.times.ndim == 1 else wl.times[0]
    g = nus.SamplingGrid(t)
    fw = float(wl.f_w[0])
    w = nus.api.taper_spline(g, nus.SignalBand(wl.f_max), fw, 5)
    t0 = time.time(); qe = nus.signal_band_quadform(g, nus.SignalBand(wl.f_max), w); t1 = time.time()
    qf = nus.signal_band_quadform_fast(g, nus.SignalBand(wl.f_max), w); t2 = time.time()
    print(name, "n", t.size, "F*T", wl.f_max * (t[-1] - t[0]), "rel", np.abs(qf / qe - 1).max(), "exact s", round(t1 - t0, 3), "fast s", round(t2 - t1, 3), flush=True)
for lg in [20, 22]:
    wl = W.c2(n=1 << lg)
    t = wl.times; g = nus.SamplingGrid(t)
    w = nus.api.taper_spline(g, nus.SignalBand(wl.f_max), float(wl.f_w[0]), 7)
    t1 = time.time(); qf = nus.signal_band_quadform_fast(g, nus.SignalBand(wl.f_max), w); t2 = time.time()
    if lg == 20:
        qe = nus.signal_band_quadform(g, nus.SignalBand(wl.f_max), w); t3 = time.time()
        print("c2 2^20 rel", np.abs(qf / qe - 1).max(), "fast s", t2 - t1, "exact s", t3 - t2, flush=True)
    else:
        print("c2 2^22 fast s", t2 - t1, flush=True)
