#!/usr/bin/env python
"""MTNUFFT benchmark (BASELINE.json metric: NUFFT points x tapers / s, spectra/s, %HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c2|c2f32|c3|c4|c5] [--impl ours|reference]
                    [--shard replicas|channels|tapers|samples]

One step = one multitaper spectrum estimate (spread of all K tapers -> the own two-pass FFT
with the deconvolve/crop/eigenspectrum fused into its second pass) of one synthetic series of the workload, with
the inputs already resident in HBM (``value``); ``e2e`` is the same metric
through the host C-ABI entry point nus_mtnufft_estimate with pinned host
buffers, so each step includes the H2D copy of x and the D2H copy of P(f).

Multi-GPU (torchrun, one process per GPU, NCCL): every rank estimates its own
independent series (seed offset = rank) — channel/series sharding has no
data-path collective, so scaling is "weak"; the timed region is bracketed by a
barrier + synchronize and the max over ranks is reported.

``--impl reference`` times the reference's own CPU implementation of the path
(oracle/_ref, compiled from /root/reference sources) on this host's cores:
rank 0 only, same metric/config, each step = one taper NUFFT of the workload
per host thread (the reference path is serial per series, nufft.cpp:212-225).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "NUFFT points*tapers/sec (MTNUFFT multitaper spectrum)"
UNIT = "points*tapers/s"


def load_peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def make_workload(name, rank):
    from paper_2407_01943_b200 import workloads as W
    if name == "c2":
        return W.c2(precision="f64", seed_offset=rank)
    if name == "c2f32":
        return W.c2(precision="f32", seed_offset=rank)
    if name == "c3":  # BASELINE C3: 256 channels per replica (NUS_C3_CHANNELS overrides)
        ch = int(os.environ.get("NUS_C3_CHANNELS", "256"))
        return W.c3(channels=ch, first_channel=ch * rank)
    if name == "c5":
        return W.c5(k=int(os.environ.get("NUS_C5_K", "7")))
    if name == "c4":  # C4's structure; N defaults to 2^22 (DPSS setup at 2^26)
        lg = int(os.environ.get("NUS_C4_LOG2N", "22"))
        return W.c4(n=1 << lg, n_centers=1 << (lg - 2))
    if name == "c1":
        return W.c1()
    raise SystemExit(f"unknown workload {name}")


def describe(wl, name):
    n, i = wl.n, wl.centers.size
    desc = {
        "c2": f"c2: Poisson times N=2^{int(np.log2(n))}, I=2^{int(np.log2(i))}, K={wl.k} (NW={wl.nw:g}), eps={wl.eps:g}, {wl.precision}",
        "c2f32": f"c2 fp32: Poisson times N=2^{int(np.log2(n))}, I=2^{int(np.log2(i))}, K={wl.k} (NW={wl.nw:g}), eps={wl.eps:g}",
        "c3": f"c3: {wl.channels} channels x N=2^{int(np.log2(n))}, I=2^{int(np.log2(i))}, K={wl.k}, eps={wl.eps:g}, fp32",
        "c5": f"c5: jittered N=2^{int(np.log2(n))}, I=2^{int(np.log2(i))}, K={wl.k}, eps={wl.eps:g}, {wl.precision}",
        "c1": f"c1: N={n}, I={i}, K={wl.k}, eps={wl.eps:g}",
        "c4": f"c4: clustered N=2^{int(np.log2(n))} (400 windows), I=2^{int(np.log2(i))}, K={wl.k} (NW={wl.nw:g}), eps={wl.eps:g}, {wl.precision}, all samples on one GPU (BASELINE C4 is N=2^26, I=2^24)",
    }[name]
    return desc


def bench_config(wl, name):
    """The workload keys both arms print (identical dicts: the driver compares them)."""
    n = wl.times.shape[-1]
    return {"workload": describe(wl, name), "N": int(n), "I": int(wl.centers.size), "K": int(wl.k),
            "channels_per_gpu": int(wl.times.shape[0]) if wl.times.ndim == 2 else 1, "eps": wl.eps,
            "precision": wl.precision}


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock"}

    def __init__(self, index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = str(e)
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def reference_tapers(wl):
    """Interpolated DPSS from the oracle restatement (CPU), for the reference arm's inputs."""
    from oracle import C as OC
    t = wl.times if wl.times.ndim == 1 else wl.times[0]
    n = t.size
    h = (t[-1] - t[0]) / (n - 1)
    tw = float(wl.f_w[0]) * h * n
    dp, _ = OC.dpss(n, tw, wl.k, threads=os.cpu_count() or 1)
    knots = t[0] + h * np.arange(n)
    return np.stack([OC.spline(knots, dp[j], t) for j in range(wl.k)])


def cpu_reference_leg(wl, tapers, threads, spectra_steps, taper_per_step=False):
    """Time the reference CPU path (oracle/_ref) on this host: returns (value, sample string, steps)."""
    from oracle import Injected, ref_available
    if not ref_available():
        return None
    t = wl.times if wl.times.ndim == 1 else wl.times[0]
    x = wl.values if wl.values.ndim == 1 else wl.values[0]
    w = tapers[:1] if taper_per_step else tapers
    est = Injected(t, w, wl.centers, wl.eps, wl.f_max, float(wl.f_w[0]), policy=0)
    xs = np.tile(x, (threads, 1))
    est.power_many(xs[:threads], threads)  # warm-up (page-in, caches)
    times = []
    for _ in range(spectra_steps):
        t0 = time.perf_counter()
        est.power_many(xs, threads)
        times.append(time.perf_counter() - t0)
    est.close()
    per_step_units = threads * t.size * w.shape[0]
    return per_step_units / (sum(times) / len(times)), times, per_step_units


def cpu_reference_channels(wl, tapers, threads, steps, warmup=1):
    """The reference CPU path on independent channels (channels in parallel, as the
    reference's parallel_for): one Injected handle (NufftPlan + eigencoefficients + power loop,
    oracle/_ref) per channel for `threads` channels, each step = those channels' full K-taper spectra
    on `threads` host threads.  Returns (points*tapers/s, seconds per step)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import Injected
    cnt = min(threads, wl.times.shape[0])
    hs = [Injected(wl.times[c], tapers[c], wl.centers, wl.eps, wl.f_max, float(wl.f_w[c]), policy=0)
          for c in range(cnt)]
    try:
        with ThreadPoolExecutor(cnt) as ex:
            def one():
                list(ex.map(lambda c: hs[c].power(wl.values[c]), range(cnt)))
            for _ in range(warmup):
                one()
            times = []
            for _ in range(steps):
                t0 = time.perf_counter()
                one()
                times.append(time.perf_counter() - t0)
    finally:
        for h in hs:
            h.close()
    units = cnt * wl.times.shape[1] * tapers.shape[1]
    return units / (sum(times) / len(times)), times, cnt


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = make_workload(args.workload, 0)
    try:
        from oracle import ref_available
        if not ref_available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libnusref.so not built"}))
            return 0
    except Exception as e:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle import failed: {e}"}))
        return 0
    threads = max(1, min(os.cpu_count() or 1, 32))
    if wl.times.ndim == 2:  # independent channels (C3): channels in parallel on the host threads
        from oracle import C as OC
        cnt = min(threads, wl.times.shape[0])
        taps = []
        for c in range(cnt):  # interpolated DPSS per channel from the restatement, R(B)-normalised
            t = wl.times[c]
            n = t.size
            h = (t[-1] - t[0]) / (n - 1)
            dp, _ = OC.dpss(n, float(wl.f_w[c]) * h * n, wl.k, threads=threads)
            knots = t[0] + h * np.arange(n)
            w = np.stack([OC.spline(knots, dp[j], t) for j in range(wl.k)])
            taps.append(w)
        value, ts, cnt = cpu_reference_channels(wl, np.stack(taps), threads, args.steps, args.warmup)
        line = {
            "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(ts) / len(ts),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": bench_config(wl, args.workload),
            "parallelism": f"{cnt} channels on {cnt} host threads (rank 0 only)",
            "window": "Gaussian (the reference's own gridding kernel)",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cnt, "kind": "reference",
                             "sample": f"per step: {cnt} channels x one full {wl.k}-taper spectrum each "
                                       f"(N={wl.times.shape[1]}, I={wl.centers.size}) through the reference "
                                       "NufftPlan + eigencoefficients + power loop, tapers injected"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0
    tapers = reference_tapers(wl)
    from oracle import Injected
    t = wl.times if wl.times.ndim == 1 else wl.times[0]
    x = wl.values if wl.values.ndim == 1 else wl.values[0]
    est = Injected(t, tapers[:1], wl.centers, wl.eps, wl.f_max, float(wl.f_w[0]), policy=0)
    xs = np.tile(x, (threads, 1))
    for _ in range(args.warmup):
        est.power_many(xs, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        est.power_many(xs, threads)
    dt = time.perf_counter() - t0
    est.close()
    units = threads * t.size * 1 * args.steps
    value = units / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": bench_config(wl, args.workload),
        "parallelism": f"{threads} host threads (rank 0 only)",
        "window": "Gaussian (the reference's own gridding kernel)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"per step: {threads} threads x one taper NUFFT (N={t.size}, "
                                   f"I={wl.centers.size}) through the reference NufftPlan + "
                                   "eigencoefficients + power loop, tapers injected"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0



def run_sharded(args):
    """One workload partitioned over the ranks (distributed.py), one process per GPU:

    * ``--shard channels`` (C3: 256 channels x 2^18, fp32): rank r estimates channels
      [r C/G, (r+1) C/G) with their own tapers and plans; no data-path collective.
    * ``--shard tapers`` (C2): every rank spreads all samples for its taper subset; one NCCL
      ``reduce`` of the I partial powers per spectrum.
    * ``--shard samples`` (C4: N = 2^NUS_C4_LOG2N, default 26): rank r owns a contiguous sample chunk;
      its spread stores every taper's 32-cell segments straight into the owner rank's receive slot
      over CUDA IPC peer memory (NVLink), one stream-ordered NCCL all_reduce flag, the owners sum
      their slots, FFT + crop their tapers, and one NCCL ``reduce`` of P.

    The total work is fixed as G grows ("strong" scaling); value = all points x tapers / max over
    ranks of the device-timed region."""
    import torch
    import torch.distributed as dist
    from paper_2407_01943_b200 import _capi as CAPI
    from paper_2407_01943_b200 import distributed as D
    from paper_2407_01943_b200 import workloads as W
    from paper_2407_01943_b200.api import _Estimator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    eng = D.DeviceEngine(local)
    stream = torch.cuda.current_stream(dev)
    t_setup = time.perf_counter()
    nvlink_bytes = 0
    if args.shard == "channels":
        total_ch = int(os.environ.get("NUS_C3_CHANNELS", "256"))
        c0, c1 = D.split_range(total_ch, world, rank)
        wl = W.c3(channels=c1 - c0, first_channel=c0)
        est = _Estimator(wl.times, wl.centers, wl.f_max, wl.f_w, wl.k, wl.eps, 1, wl.precision, local)
        xdt = torch.float32
        x_host = np.asarray(wl.values, dtype=np.float64).reshape(c1 - c0, -1)
        p_dev = torch.empty((c1 - c0, wl.centers.size), dtype=xdt, device=dev)

        def run(x_dev):
            eng.estimate(est, x_dev, p_dev)
        units_rank = (c1 - c0) * wl.times.shape[-1] * wl.k
        units_total = total_ch * wl.times.shape[-1] * wl.k
        workload = (f"c3 channel shard: {total_ch} channels x N=2^{int(np.log2(wl.times.shape[-1]))}, "
                    f"I=2^{int(np.log2(wl.centers.size))}, K={wl.k}, eps={wl.eps:g}, fp32, {world} rank(s)")
        bm = est.bytes_model(0)["total"] / (c1 - c0) * total_ch
        parallelism = f"channels split over {world} GPU(s), no data-path collective"
    elif args.shard == "tapers":
        wl = W.c2()
        one = _Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), wl.k, wl.eps, 1, wl.precision, local)
        tapers = one.tapers()[0]
        del one
        ts = D.TaperShard(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), tapers, wl.eps, wl.precision, engine=eng)
        xdt = torch.float64
        x_host = np.asarray(wl.values, dtype=np.float64).reshape(1, -1)
        p_dev = torch.empty(wl.centers.size, dtype=xdt, device=dev)

        def run(x_dev):
            ts.estimate(x_dev[0], p_dev)
        units_rank = wl.n * (ts.k1 - ts.k0)
        units_total = wl.n * wl.k
        workload = (f"c2 taper shard: N=2^20, I=2^20, K={wl.k}, eps={wl.eps:g}, fp64, {world} rank(s)")
        bm = None
        parallelism = f"tapers split over {world} GPU(s), NCCL reduce of I partial powers"
    else:  # samples
        lg = int(os.environ.get("NUS_C4_LOG2N", "26"))
        wl = W.c4(n=1 << lg, n_centers=1 << (lg - 2))
        ss = D.SampleSplit(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), wl.k, wl.eps, wl.precision, engine=eng)
        xdt = torch.float64
        x_host = np.asarray(wl.values[ss.s0:ss.s1], dtype=np.float64).reshape(1, -1)
        p_dev = torch.empty(wl.centers.size, dtype=xdt, device=dev)

        def run(x_dev):
            ss.estimate(x_dev[0], p_dev)
        units_rank = (ss.s1 - ss.s0) * wl.k
        units_total = wl.n * wl.k
        # each rank's spread stores the tapers other ranks own into their slots: (G-1)/G of K_pad grids
        nvlink_bytes = (world - 1) * ss.per_rank * ss.mr * 16 if world > 1 else 0
        workload = (f"c4 sample split: clustered N=2^{lg} (400 windows), I=2^{lg - 2}, K={wl.k} (NW=8), "
                    f"eps={wl.eps:g}, fp64, {world} rank(s)")
        bm = None
        parallelism = (f"samples split over {world} GPU(s): spread -> peer receive slots (CUDA IPC over NVLink), "
                       "NCCL all_reduce flag, owner slot sums, FFT + crop of owned tapers, NCCL reduce of P")
    setup_s = time.perf_counter() - t_setup
    x_dev = torch.tensor(x_host, dtype=xdt, device=dev)
    for _ in range(args.warmup):
        run(x_dev)
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = CAPI.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            run(x_dev)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    launches = CAPI.launch_count() - l0
    dist.barrier()
    ms_t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    # e2e: every step copies this rank's x in from pinned host memory and its P out, in the timed region
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 20))
    xh = torch.tensor(x_host, dtype=xdt).pin_memory()
    ph = torch.empty(tuple(p_dev.shape), dtype=p_dev.dtype).pin_memory()
    xd = torch.empty_like(x_dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        xd.copy_(xh, non_blocking=True)
        run(xd)
        ph.copy_(p_dev, non_blocking=True)
    torch.cuda.synchronize(dev)
    e2e_t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())
    value = units_total * args.steps / (ms_max / 1e3)
    step_ms = ms_max / args.steps
    peak, peak_src = load_peaks()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if xdt == torch.float32 else "f64", "data": "synthetic",
        "config": {"workload": workload, "N": int(wl.times.shape[-1]), "I": int(wl.centers.size), "K": int(wl.k),
                   "eps": wl.eps, "precision": wl.precision, "shard": args.shard},
        "parallelism": parallelism,
        "l2": "inputs larger than L2 (per-step grids and tables exceed 126 MB)",
        "e2e": {"value": units_total * e2e_steps / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(xh.numel() * xh.element_size()),
                "d2h_bytes_per_step": int(ph.numel() * ph.element_size()), "steps": e2e_steps,
                "api": "distributed.py shard estimate, torch pinned-buffer copies on the compute stream"},
        "gpu_launches": int(launches),
        "nvlink_bytes_per_step_per_rank": int(nvlink_bytes),
        "units_per_step_this_rank": int(units_rank),
        "setup_s": setup_s,
    }
    if bm is not None:
        ach = bm / (step_ms / 1e3) / 1e9
        line["roofline"] = {"bound": "hbm", "kernel": "pipeline (all ranks' algorithmic bytes / step)",
                            "achieved": ach, "peak": peak * world, "unit": "GB/s", "frac": ach / (peak * world),
                            "traffic": None, "peak_source": peak_src}
    if rank == 0:
        line["clocks"] = clk.summary()
        print(json.dumps(line), flush=True)
    if args.shard == "samples":
        ss.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c2f32", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--eps", type=float, default=None, help="override the workload's NUFFT tolerance")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "channels", "tapers", "samples"],
                    help="replicas (default): an independent series per GPU; channels (C3) / tapers (C2) / "
                         "samples (C4): one workload partitioned over the GPUs (run_sharded)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.shard != "replicas":
        return run_sharded(args)

    import torch
    import torch.distributed as dist
    from paper_2407_01943_b200 import _capi as CAPI
    from paper_2407_01943_b200.api import _Estimator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    wl = make_workload(args.workload, rank)
    if args.eps is not None:
        wl.eps = args.eps
    # independent channels (C3): each channel's tapers on its own grid with its own half-bandwidth
    # (same time-bandwidth product, so the channels share one DPSS)
    fw = wl.f_w if np.ndim(wl.times) == 2 and np.size(wl.f_w) == np.shape(wl.times)[0] else float(wl.f_w[0])
    est = _Estimator(wl.times, wl.centers, wl.f_max, fw, wl.k, wl.eps, 1,
                     wl.precision, local)
    setup = est.setup_ms()
    C_, n, k, nc = est.channels, est.n, est.k, est.nc
    f32 = wl.precision == "f32"
    xdt = torch.float32 if f32 else torch.float64
    vals = np.asarray(wl.values, dtype=np.float64).reshape(C_, n)
    nrot = 4  # rotate x over resident series (per-step footprint already exceeds L2)
    xs = [torch.tensor(np.roll(vals, 17 * r, axis=1), dtype=xdt, device=dev) for r in range(nrot)]
    pw = torch.empty((C_, nc), dtype=xdt, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    L = CAPI.lib()

    def step(i):
        CAPI.check(L.nus_mtnufft_estimate_device(est.h, xs[i % nrot].data_ptr(), 1 if f32 else 0,
                                                 pw.data_ptr(), None, sptr))

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    # the timed region carries no per-stage events: events between the kernels would serialise
    # the programmatic dependent launches (each kernel's CTAs dispatched while its predecessor
    # drains); the stage breakdown comes from a separate pass below
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = CAPI.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    launches = CAPI.launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    # stage breakdown: CUDA events around each kernel, a separate pass of the same steps
    stage_steps = max(1, min(args.steps, 20))
    CAPI.check(L.nus_mtnufft_timing(est.h, stage_steps))
    for i in range(stage_steps):
        step(i)
    torch.cuda.synchronize(dev)
    stage = np.zeros(3)
    runs = CAPI._i64()
    CAPI.check(L.nus_mtnufft_timing_read(est.h, CAPI.dptr(stage), runs))
    stage_ms = stage / max(runs.value, 1)
    CAPI.check(L.nus_mtnufft_timing(est.h, 0))

    # ---- e2e through the host C-ABI with pinned buffers: nus_mtnufft_estimate_batch moves every
    # step's own input in (H2D) and its own P out (D2H) inside the timed region; the copies of one
    # step overlap the compute of its neighbours (the same rotation of 4 series as the device leg)
    # up to 100 steps (pipeline fill / drain amortised), host buffers capped at ~2 GB
    step_bytes = C_ * (n + nc) * 8
    e2e_steps = args.e2e_steps or max(3, min(100, int(2e9 // step_bytes)))
    xh = torch.empty((e2e_steps, C_, n), dtype=torch.float64, pin_memory=True).numpy()
    for i in range(e2e_steps):
        xh[i] = np.roll(vals, 17 * (i % nrot), axis=1)
    ph = torch.empty((e2e_steps, C_, nc), dtype=torch.float64, pin_memory=True).numpy()
    CAPI.check(L.nus_mtnufft_estimate_batch(est.h, CAPI.dptr(xh), min(2, e2e_steps), CAPI.dptr(ph)))  # warm-up
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # three repetitions of the whole batch, the median reported (one wall-clock sample of ~25 ms is
    # at the mercy of a single host hiccup)
    e2e_runs = []
    for _ in range(3):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        CAPI.check(L.nus_mtnufft_estimate_batch(est.h, CAPI.dptr(xh), e2e_steps, CAPI.dptr(ph)))
        e2e_runs.append(time.perf_counter() - t0)
    e2e_s = sorted(e2e_runs)[1]
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_t.item())
    # the batch result equals the one-shot host estimate (same API, same kernels)
    p1 = np.empty((C_, nc))
    CAPI.check(L.nus_mtnufft_estimate(est.h, CAPI.dptr(np.ascontiguousarray(xh[e2e_steps - 1])), CAPI.dptr(p1)))
    if not np.array_equal(p1, ph[e2e_steps - 1]):
        raise RuntimeError("estimate_batch and estimate disagree")

    units_per_step = C_ * n * k  # points x tapers, per rank
    value = world * units_per_step * args.steps / (ms_max / 1e3)
    e2e_value = world * units_per_step * e2e_steps / e2e_s

    bm = est.bytes_model(1 if f32 else 0)
    peak, peak_src = load_peaks()
    buf = ctypes.create_string_buffer(256)
    CAPI.check(L.nus_mtnufft_stage_kernels(est.h, buf, 256))
    stage_names = buf.value.decode().split(";")
    stage_bytes = [bm["spread"], bm["fft"], bm["crop"]]
    own = [q for q in range(3) if "library" not in stage_names[q] and stage_bytes[q] > 0]
    dom_own = max(own, key=lambda q: stage_ms[q])
    traffic = None
    tpath = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.workload, {}).get(stage_names[dom_own])
        except Exception:
            traffic = None
    ach = stage_bytes[dom_own] / (stage_ms[dom_own] / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": stage_names[dom_own], "achieved": ach, "peak": peak,
            "unit": "GB/s", "frac": ach / peak, "traffic": traffic, "peak_source": peak_src,
            "bytes_per_launch": stage_bytes[dom_own], "avg_launch_ms": stage_ms[dom_own]}
    step_ms = ms_max / args.steps
    pipe_ach = bm["total"] / (step_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if f32 else "f64", "data": "synthetic",
        "config": bench_config(wl, args.workload),
        "window": ("exponential of semicircle" if est.info.kernel == 1 else "Gaussian (the reference's)")
                  + f", {int(est.info.support)} cells per sample",
        "parallelism": f"{world} GPU(s), independent series per GPU (no data-path collective)",
        "l2": "inputs larger than L2: per-step grid K*Mr complex + tables exceed 126 MB; x rotated over 4 resident series",
        "spectra_per_s": world * C_ * args.steps / (ms_max / 1e3),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(xh[0].nbytes),
                "d2h_bytes_per_step": int(ph[0].nbytes), "steps": e2e_steps,
                "repeats": 3, "seconds": [round(t, 6) for t in e2e_runs],
                "api": "nus_mtnufft_estimate_batch (host C-ABI, pinned buffers, copies overlapped across steps)"},
        "gpu_launches": int(launches),
        "gpu_launches_note": "our kernels per timed region: " + " + ".join(n for n in stage_names if "library" not in n)
                             + " per step",
        "roofline": roof,
        "pipeline_roofline": {"bound": "hbm", "achieved": pipe_ach, "peak": peak, "unit": "GB/s",
                              "frac": pipe_ach / peak, "algorithmic_bytes_per_step": bm["total"],
                              "model": "SURVEY §8(d): N(8+r)+KNr+3K*Mr*c+KIc+Ir per channel"},
        "stages_ms": {stage_names[q]: stage_ms[q] for q in range(3)},
        "stage_bytes": {stage_names[q]: stage_bytes[q] for q in range(3)},
        "setup_ms": setup,
    }
    if rank == 0:
        line["clocks"] = clk.summary()
    # ---- cpu baseline (rank 0, N=1 only)
    if rank == 0 and world == 1 and not args.no_cpu and wl.times.ndim == 2:
        try:  # independent channels: the reference on `threads` channels in parallel
            threads = max(1, min(os.cpu_count() or 1, 32))
            v, ts, cnt = cpu_reference_channels(wl, est.tapers(), threads, 1)
            line["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": cnt, "kind": "reference",
                "sample": f"{cnt} channels x one full {k}-taper spectrum each (N={n}, I={nc}) on {cnt} host "
                          "threads through the reference's NufftPlan + eigencoefficients + power loop "
                          "(oracle/_ref), the GPU's tapers injected, 1 timed batch after 1 warm-up",
                "seconds": ts}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0 and world == 1 and not args.no_cpu and wl.times.ndim == 1:
        try:
            threads = max(1, min(os.cpu_count() or 1, 32))
            tap = est.tapers()[0]
            res = cpu_reference_leg(wl, tap, threads, 1)
            if res is not None:
                v, ts, per = res
                line["cpu_baseline"] = {
                    "value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                    "sample": f"{threads} host threads x one full {k}-taper spectrum each "
                              f"(N={n}, I={nc}) through the reference's NufftPlan + "
                              "eigencoefficients + power loop (oracle/_ref), 1 timed batch after 1 warm-up",
                    "seconds": ts}
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
