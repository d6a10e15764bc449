"""C5 accuracy / throughput sweep (BASELINE.json config 5) on one B200.

N = 2^22 jittered-uniform times (+-0.4/fs, 10% dropouts), unit white noise, I = 2^21 centres;
eps in {1e-3, 1e-6, 1e-9, 1e-12} x K in {1, 3, 7, 15, 31} (NW = (K+1)/2), fp64 and fp32.
Per K the tapers are built once on the device (DPSS + spline + O(N log N) normalisation) and
injected into every (eps, precision) estimator.  Accuracy: relL2(P) against the fp64 eps=1e-12
estimate with the reference's Gaussian window (the tightest transform available at this size;
the reference's own CPU path would need ~1 min per taper here).  Throughput: CUDA-event time of
`steps` spectra with x resident in HBM, as bench.py.

    python tools/c5_sweep.py [--steps 20] [--out profiles/c5_sweep.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--log2n", type=int, default=22)
    ap.add_argument("--out", default="profiles/c5_sweep.json")
    ap.add_argument("--k", type=int, nargs="+", default=[1, 3, 7, 15, 31])
    args = ap.parse_args()
    import torch

    import paper_2407_01943_b200 as nus
    from paper_2407_01943_b200 import _capi as CAPI
    from paper_2407_01943_b200 import workloads as W
    from paper_2407_01943_b200.api import _Estimator

    L = CAPI.lib()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = []
    for k in args.k:
        wl = W.c5(n=1 << args.log2n, k=k)
        t0 = time.time()
        base = _Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), k, 1e-12, 1, "f64", 0)
        setup = base.setup_ms()
        tapers = base.tapers()
        with nus.spread_kernel("gaussian"):
            ref_est = _Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), k, 1e-12, 1, "f64", 0,
                                 tapers=tapers)
        ref = ref_est.power(wl.values)[0]
        del ref_est
        print(f"K={k}: tapers {time.time() - t0:.1f} s", flush=True)
        for prec in ("f64", "f32"):
            for eps in (1e-3, 1e-6, 1e-9, 1e-12):
                if prec == "f32" and eps < 1e-6:
                    continue  # below fp32 resolution
                est = _Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), k, eps, 1, prec, 0,
                                 tapers=tapers)
                p = est.power(wl.values)[0]
                err = float(np.linalg.norm(p - ref) / np.linalg.norm(ref))
                xdt = torch.float32 if prec == "f32" else torch.float64
                x = torch.tensor(wl.values, dtype=xdt, device=dev)
                pw = torch.empty(wl.centers.size, dtype=xdt, device=dev)
                f32 = 1 if prec == "f32" else 0

                def step():
                    CAPI.check(L.nus_mtnufft_estimate_device(est.h, x.data_ptr(), f32, pw.data_ptr(), None,
                                                             stream.cuda_stream))

                for _ in range(3):
                    step()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.steps):
                    step()
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / args.steps
                CAPI.check(L.nus_mtnufft_timing(est.h, 5))
                for _ in range(5):
                    step()
                torch.cuda.synchronize()
                st = np.zeros(3)
                runs = CAPI._i64()
                CAPI.check(L.nus_mtnufft_timing_read(est.h, CAPI.dptr(st), runs))
                CAPI.check(L.nus_mtnufft_timing(est.h, 0))
                stages = (st / max(runs.value, 1)).tolist()
                bm = est.bytes_model(f32)
                info = est.info
                row = {"K": k, "eps": eps, "precision": prec, "window": "es" if info.kernel == 1 else "gaussian",
                       "support": int(info.support), "mr": int(info.mr), "ms_per_spectrum": ms,
                       "points_tapers_per_s": wl.n * k / (ms / 1e3), "hbm_frac": bm["total"] / (ms / 1e3) / 1e9 / peak,
                       "relL2_vs_fp64_eps1e-12": err, "stage_ms": stages}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del est
        rows.append({"K": k, "setup_ms": setup})
    out = {"config": f"C5: jittered N=2^{args.log2n}, I=2^{args.log2n - 1}, white noise", "peak_gbs": peak,
           "reference": "fp64, eps=1e-12, Gaussian window, same tapers", "rows": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
