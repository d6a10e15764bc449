"""CPU, world_size 2 over gloo: the multi-GPU orchestration of distributed.py
(channel shard, taper shard, sample split with reduce-scatter of fine grids and
row-split R(B) normalisation) reproduces the single-process result.

The per-rank device work is replaced by a numpy engine restating the same
stages (Gaussian gridding of a sample subset, FFT + crop + power of owned taper
rows) on CPU tensors; the collectives, partitioning and padding logic are the
product code.  On the GPU box the same classes run with DeviceEngine over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import rel_l2
from oracle import C
from paper_2407_01943_b200 import distributed as D
from paper_2407_01943_b200 import workloads as W

TWO_PI = 2.0 * np.pi


class NumpyEngine:
    """CPU stand-in for DeviceEngine (same interface), built on the oracle restatement."""

    class Est:
        pass

    def taper_spline(self, times, f_max, f_w, k):
        n = times.size
        h = (times[-1] - times[0]) / (n - 1)
        dp, _ = C.dpss(n, f_w * h * n, k, threads=1)
        knots = times[0] + h * np.arange(n)
        return np.stack([C.spline(knots, dp[j], times) for j in range(k)])

    def quadform_rows(self, times, f_max, w, row0, row1):
        tol = 1e-12 * (times[-1] - times[0]) / times.size
        q = np.zeros(w.shape[0])
        for r in range(row0, row1):
            d = times[r] - times[r + 1:]
            v = np.where(np.abs(d) < tol, 2 * f_max, np.sin(2 * np.pi * f_max * d) / (np.pi * d))
            q += w[:, r] * (2 * f_max * w[:, r] + 2 * (w[:, r + 1:] @ v))
        return q

    def create(self, times, centers, f_max, f_w, k, eps, precision, tapers):
        e = self.Est()
        e.t = np.atleast_2d(times)
        e.c = np.asarray(centers)
        e.k = k
        e.eps = eps
        e.w = None if tapers is None else np.asarray(tapers).reshape(e.t.shape[0], k, -1)
        if e.w is None:  # per-channel normalised tapers (ChannelShard), each with its own f_w
            fw = np.broadcast_to(np.asarray(f_w, dtype=np.float64), (e.t.shape[0],))
            e.fw = fw.copy()
            e.w = np.stack([C.gpss_interpolated(e.t[ch], f_max, float(fw[ch]), k, threads=1)[0]
                            for ch in range(e.t.shape[0])])
        e.p, _ = C.plan_params(e.c, eps)
        return e

    def quadform_fast(self, times, f_max, w):  # the O(N log N) engine call; dense here
        return self.quadform_rows(times, f_max, w, 0, times.size)

    def real_dtype(self, est):
        return torch.float64

    def zeros(self, shape, dtype):
        return torch.zeros(shape, dtype=dtype)

    def to_device(self, a, dtype):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype)

    def mr(self, est):
        return int(est.p["mr"])

    def _grid(self, est, ch, x, s0, s1):
        p = est.p
        mr, w = int(p["mr"]), int(p["spread_width"])
        t = est.t[ch][s0:s1]
        xs = x[s0:s1]
        pre = np.exp(1j * (-TWO_PI * p["fshift"] * t))
        xx = np.fmod(-TWO_PI * p["df"] * t, TWO_PI)
        xx = np.where(xx < 0, xx + TWO_PI, xx)
        j0 = np.floor(xx * mr / TWO_PI).astype(np.int64) - w + 1
        grids = np.zeros((est.k, mr), complex)
        for q in range(2 * w):
            xi = TWO_PI * (j0 + q) / mr
            g = np.exp(-(xx - xi) ** 2 / (4 * p["tau"]))
            cells = np.mod(j0 + q, mr)
            for kk in range(est.k):
                np.add.at(grids[kk], cells, g * est.w[ch, kk, s0:s1] * xs * pre)
        return grids

    def _power(self, est, grids):
        p = est.p
        mr, nc = int(p["mr"]), est.c.size
        b = np.fft.fft(grids, axis=-1)
        m = np.arange(nc) - int(p["mode_offset"])
        d = np.sqrt(np.pi / p["tau"]) / mr * np.exp(p["tau"] * m * m)
        return np.sum(np.abs(d * b[:, np.mod(-m, mr)]) ** 2, axis=0)

    def estimate(self, est, x, power):
        xs = np.atleast_2d(x.numpy())
        out = np.stack([self._power(est, self._grid(est, ch, xs[ch], 0, xs.shape[1])) / est.k
                        for ch in range(xs.shape[0])])
        power.copy_(torch.as_tensor(out.reshape(power.shape)))

    def spread(self, est, x, s0, s1, grid, kpad):
        g = self._grid(est, 0, x.numpy(), s0, s1)
        view = grid.view(kpad, -1, 2)
        view[: est.k, :, 0] = torch.as_tensor(g.real)
        view[: est.k, :, 1] = torch.as_tensor(g.imag)

    def transform(self, est, rows, k0, k1, divisor, power):
        v = rows.view(rows.shape[0], -1, 2).numpy()
        g = v[: k1 - k0, :, 0] + 1j * v[: k1 - k0, :, 1]
        power.copy_(torch.as_tensor(self._power(est, g) / divisor))


class SlotEngine(NumpyEngine):
    """NumpyEngine plus the fused exchange's device interface, with file-backed shared mappings
    standing in for CUDA IPC: a receive buffer is a memmap whose "handle" is its path, and a
    "device pointer" is (registered base + byte offset), so the ranks' slot pointer arithmetic,
    handle exchange, barrier and slot sums run exactly as SampleSplit drives them."""

    def __init__(self, tmpdir, rank):
        self.tmpdir, self.rank = tmpdir, rank
        self.maps = {}  # base address -> float64 array (flat)

    def synchronize(self):
        for arr in self.maps.values():
            if isinstance(arr, np.memmap):
                arr.flush()

    def _register(self, arr):
        base = (len(self.maps) + 1) << 40
        self.maps[base] = arr
        return base

    def alloc_slots(self, shape, dtype):
        path = os.path.join(self.tmpdir, f"recv{self.rank}.bin")
        mm = np.memmap(path, dtype=np.float64, mode="w+", shape=tuple(shape))
        mm[:] = 0.0
        mm.flush()
        t = torch.from_numpy(mm)
        self.own = (t, self._register(mm.reshape(-1)))
        return t

    def ipc_handle(self, t):
        path = os.path.join(self.tmpdir, f"recv{self.rank}.bin").encode()
        return path + b"\0" * (64 - len(path)), 0

    def ipc_open(self, handle):
        raw, offset = handle
        path = raw.rstrip(b"\0").decode()
        return self._register(np.memmap(path, dtype=np.float64, mode="r+").reshape(-1)) + offset

    def _resolve(self, ptr):
        if self.own[0].data_ptr() <= ptr < self.own[0].data_ptr() + self.own[0].numel() * 8:
            return self.maps[self.own[1]], (ptr - self.own[0].data_ptr()) // 8
        base = max(b for b in self.maps if b <= ptr)
        return self.maps[base], (ptr - base) // 8

    def spread_slots(self, est, x, s0, s1, slot_ptrs, per):
        g = self._grid(est, 0, x.numpy(), s0, s1)
        mr = g.shape[1]
        for k in range(est.k):
            arr, off = self._resolve(int(slot_ptrs[k // per]))
            row = off + (k % per) * 2 * mr
            arr[row:row + 2 * mr:2] = g[k].real
            arr[row + 1:row + 2 * mr:2] = g[k].imag

    def sum_slots(self, base, nslots, slot_stride, count, out):
        flat = base.reshape(-1)
        acc = torch.zeros(2 * count, dtype=torch.float64)
        for q in range(nslots):
            acc += flat[2 * q * slot_stride:2 * q * slot_stride + 2 * count]
        out.view(-1).copy_(acc)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = W.small(n=700, n_centers=256, k=3, nw=3.0, eps=1e-9, seed=5)
        eng = NumpyEngine()
        fw = float(wl.f_w[0])
        if kind in ("sample", "sample_fused", "sample_fast_norm"):
            if kind == "sample_fused":
                eng = SlotEngine(os.environ["NUS_TEST_SLOTDIR"], rank)
            if kind == "sample_fast_norm":  # the N > 2^18 branch: rank 0's forms, broadcast
                D.SampleSplit.fast_normalise_min = 100
            ss = D.SampleSplit(wl.times, wl.centers, wl.f_max, fw, 3, 1e-9, engine=eng)
            assert ss.fused == (kind == "sample_fused")
            xl = torch.as_tensor(wl.values[ss.s0:ss.s1].copy())
            pw = torch.zeros(wl.centers.size, dtype=torch.float64)
            ss.estimate(xl, pw)
            if kind == "sample_fused":  # three more spectra: the two slot parities alternate
                for _ in range(3):
                    p2 = torch.zeros_like(pw)
                    ss.estimate(xl, p2)
                    if rank == 0:
                        assert torch.equal(p2, pw)
            res = (pw.numpy(), ss.tapers, ss.kpad)
        elif kind == "taper":
            w, _ = C.gpss_interpolated(wl.times, wl.f_max, fw, 3, threads=1)
            ts = D.TaperShard(wl.times, wl.centers, wl.f_max, fw, w, 1e-9, engine=eng)
            pw = torch.zeros(wl.centers.size, dtype=torch.float64)
            ts.estimate(torch.as_tensor(wl.values), pw)
            res = (pw.numpy(), w, None)
        else:
            c3 = W.c3(channels=3, n=512)
            cs = D.ChannelShard(c3.times, np.arange(128) * (2500.0 / 127), 2500.0, c3.f_w, 2, 1e-9,
                                precision="f64", engine=eng)
            xl = torch.as_tensor(c3.values[cs.c0:cs.c1].copy())
            pl = torch.zeros((cs.c1 - cs.c0, 128), dtype=torch.float64)
            cs.estimate_local(xl, pl)
            res = (cs.gather(pl).numpy(), None, (cs.c0, cs.c1))
        if rank == 0:
            q.put(res)
    except Exception as e:  # surface worker failures instead of waiting for the timeout
        q.put(e)
        raise
    finally:
        dist.destroy_process_group()


def _run(kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    if isinstance(res, Exception):
        for p in procs:
            p.join(timeout=30)
        raise res
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return res


def test_sample_split_reduce_scatter_matches_single_process():
    p, tapers, kpad = _run("sample")
    assert kpad == 4  # K=3 padded to a multiple of G=2
    wl = W.small(n=700, n_centers=256, k=3, nw=3.0, eps=1e-9, seed=5)
    # row-split normalisation == full normalisation
    w_full, _ = C.gpss_interpolated(wl.times, wl.f_max, float(wl.f_w[0]), 3, threads=1)
    np.testing.assert_allclose(np.abs(tapers), np.abs(w_full), rtol=1e-9, atol=1e-15)
    ref = C.mtnufft_power(wl.times, tapers, wl.values, wl.centers, 1e-9)
    assert rel_l2(p, ref) < 1e-12


def test_sample_split_fused_slot_exchange_matches_single_process(tmp_path, monkeypatch):
    """World 2 (gloo): the fused exchange's host logic -- receive slots, handle exchange
    (all_gather_object), per-owner slot pointers, the barrier, slot sums in rank order."""
    monkeypatch.setenv("NUS_TEST_SLOTDIR", str(tmp_path))
    p, tapers, kpad = _run("sample_fused")
    assert kpad == 4
    wl = W.small(n=700, n_centers=256, k=3, nw=3.0, eps=1e-9, seed=5)
    ref = C.mtnufft_power(wl.times, tapers, wl.values, wl.centers, 1e-9)
    assert rel_l2(p, ref) < 1e-12


def test_sample_split_fast_normalisation_broadcast_matches_full():
    """N above SampleSplit.fast_normalise_min: rank 0's forms broadcast, identical on every rank."""
    p, tapers, kpad = _run("sample_fast_norm")
    wl = W.small(n=700, n_centers=256, k=3, nw=3.0, eps=1e-9, seed=5)
    w_full, _ = C.gpss_interpolated(wl.times, wl.f_max, float(wl.f_w[0]), 3, threads=1)
    np.testing.assert_allclose(np.abs(tapers), np.abs(w_full), rtol=1e-9, atol=1e-15)
    ref = C.mtnufft_power(wl.times, tapers, wl.values, wl.centers, 1e-9)
    assert rel_l2(p, ref) < 1e-12


def test_taper_shard_reduce_matches_single_process():
    p, w, _ = _run("taper")
    wl = W.small(n=700, n_centers=256, k=3, nw=3.0, eps=1e-9, seed=5)
    assert rel_l2(p, C.mtnufft_power(wl.times, w, wl.values, wl.centers, 1e-9)) < 1e-12


def test_channel_shard_gather_matches_per_channel():
    p, _, _ = _run("channel")
    c3 = W.c3(channels=3, n=512)
    centers = np.arange(128) * (2500.0 / 127)
    assert np.ptp(c3.f_w) > 0  # the channels' half-bandwidths differ: each must keep its own
    for ch in range(3):
        w, _ = C.gpss_interpolated(c3.times[ch], 2500.0, float(c3.f_w[ch]), 2, threads=1)
        ref = C.mtnufft_power(c3.times[ch], w, c3.values[ch], centers, 1e-9)
        assert rel_l2(p[ch], ref) < 1e-12


def test_balanced_triangle_rows_partition():
    for n, g in ((1000, 2), (4096, 8), (17, 3)):
        b = D.balanced_triangle_rows(n, g)
        assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))
        work = [sum(n - i for i in range(b[r], b[r + 1])) for r in range(g)]
        assert max(work) - min(work) <= n + 1


def test_covering_interval_cyclic():
    occ = np.zeros(16, dtype=bool)
    occ[[3, 4, 5, 9]] = True
    assert D.covering_interval(occ) == (3, 7)
    occ = np.zeros(16, dtype=bool)
    occ[[0, 1, 14, 15]] = True  # wraps
    assert D.covering_interval(occ) == (14, 4)
    assert D.covering_interval(np.ones(8, dtype=bool)) == (0, 8)
