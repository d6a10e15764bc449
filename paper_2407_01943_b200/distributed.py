"""Multi-GPU partitioning of the MTNUFFT path, one process per GPU.

Three shardings, all driven by ``torch.distributed`` (NCCL over NVLink/NVSwitch on
the B200 box; ``gloo`` in the CPU tests):

* :class:`ChannelShard` — independent channels (config C3): rank r owns channels
  [r C/G, (r+1) C/G) with their own tapers, plans and grids.  No data-path
  collective; P can optionally be all-gathered.
* :class:`TaperShard` — independent tapers of one series: rank r spreads all N
  samples for its taper subset and reduces sum_k |J_k|^2 (one ``reduce`` of I reals).
* :class:`SampleSplit` — one very long series (config C4): rank r owns a
  contiguous chunk of the time-sorted samples, spreads it into a FULL local
  fine grid for all K tapers (K padded to a multiple of G), then one in-place
  ``reduce_scatter`` (sum) hands rank r the complete grids of tapers
  [r K_pad/G, (r+1) K_pad/G); it FFTs + crops those and a final ``reduce``
  sums the partial spectra.  Taper normalisation is row-split too: each rank
  computes its rows of w^T R(B) w and the K partial sums are all-reduced.

The device work goes through an *engine* (``DeviceEngine`` = the C-ABI on this
rank's GPU); the orchestration only moves torch tensors through collectives.
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional, Sequence

import numpy as np

from . import _capi as C


def split_range(n: int, world: int, rank: int):
    """Contiguous near-equal split of [0, n)."""
    return n * rank // world, n * (rank + 1) // world


def host_collectives(dist, group=None) -> bool:
    """gloo (CPU tests, or ranks sharing one GPU): collectives on host tensors and a host
    barrier after a device synchronise instead of stream-ordered NCCL calls."""
    try:
        return dist.is_initialized() and dist.get_backend(group) == "gloo"
    except Exception:  # pragma: no cover
        return False


def covering_interval(occupied) -> tuple:
    """Smallest cyclic interval (start, length) holding every True of ``occupied``: the
    complement of its longest cyclic run of False (plan.cu's rule for one estimator)."""
    occ = np.asarray(occupied, dtype=bool)
    nr = occ.size
    if occ.all() or not occ.any():
        return 0, nr
    best_len, best_end = 0, 0
    for start in range(nr):
        if occ[start] or not occ[(start - 1) % nr]:
            continue
        length = 0
        while length < nr and not occ[(start + length) % nr]:
            length += 1
        if length > best_len:
            best_len, best_end = length, (start + length) % nr
    return best_end, nr - best_len


def balanced_triangle_rows(n: int, world: int):
    """Row boundaries so each rank gets ~equal work in the upper-triangle sum
    sum_n (2F w_n^2 + 2 sum_{m>n} ...): row n costs (n_total - n) pairs."""
    total = n * (n + 1) / 2.0
    bounds = [0]
    for g in range(1, world):
        # solve sum_{i<r} (n - i) = g/world * total  ->  r n - r(r-1)/2 = target
        target = total * g / world
        r = (2 * n + 1 - math.sqrt((2 * n + 1) ** 2 - 8 * target)) / 2
        bounds.append(int(min(max(round(r), bounds[-1]), n)))
    bounds.append(n)
    return bounds


# --------------------------------------------------------------------------- engine

class DeviceEngine:
    """One rank's GPU work through the C-ABI (libnus_b200.so)."""

    def __init__(self, device: int = 0):
        self.device = device
        import torch
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self._mapped = {}  # peer pointer (with allocation offset) -> mapped base, for nus_ipc_close

    # taper setup -------------------------------------------------------------
    def taper_spline(self, times, f_max, f_w, k):
        t = C.f64(times)
        w = np.empty((k, t.size))
        C.check(C.lib().nus_taper_spline(C.dptr(t), t.size, f_max, f_w, k, self.device, C.dptr(w)))
        return w

    def quadform_rows(self, times, f_max, w, row0, row1):
        t, w = C.f64(times), C.f64(w)
        q = np.empty(w.shape[0])
        C.check(C.lib().nus_signal_band_quadform(C.dptr(t), t.size, f_max, C.dptr(w), w.shape[0], row0,
                                                 row1, self.device, C.dptr(q)))
        return q

    def quadform_fast(self, times, f_max, w):
        """All K forms w^T R(B) w in O(N log N) (normalise.cu), the single-GPU setup's method."""
        t, w = C.f64(times), C.f64(w)
        q = np.empty(w.shape[0])
        C.check(C.lib().nus_signal_band_quadform_fast(C.dptr(t), t.size, f_max, C.dptr(w), w.shape[0],
                                                      self.device, C.dptr(q)))
        return q

    # estimator ---------------------------------------------------------------
    def create(self, times, centers, f_max, f_w, k, eps, precision, tapers):
        from .api import _Estimator
        return _Estimator(times, centers, f_max, f_w, k, eps, 1, precision, self.device, tapers=tapers)

    def real_dtype(self, est):
        return self.torch.float32 if est.info.precision == C.F32 else self.torch.float64

    def zeros(self, shape, dtype):
        return self.torch.zeros(shape, dtype=dtype, device=self.dev)

    def to_device(self, a, dtype):
        return self.torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=self.dev)

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def estimate(self, est, x, power):
        C.check(C.lib().nus_mtnufft_estimate_device(est.h, x.data_ptr(), 1 if x.dtype == self.torch.float32 else 0,
                                                    power.data_ptr(), None, self._stream()))

    def spread(self, est, x, s0, s1, grid, kpad):
        C.check(C.lib().nus_mtnufft_spread_device(est.h, x.data_ptr(), 1 if x.dtype == self.torch.float32 else 0,
                                                  s0, s1, grid.data_ptr(), kpad, self._stream()))

    def transform(self, est, grid_rows, k0, k1, divisor, power):
        C.check(C.lib().nus_mtnufft_transform_device(est.h, grid_rows.data_ptr(), k0, k1, divisor, 0,
                                                     power.data_ptr(), self._stream()))

    def spread_slots(self, est, x, s0, s1, slot_ptrs, per):
        C.check(C.lib().nus_mtnufft_spread_slots_device(est.h, x.data_ptr(), 1 if x.dtype == self.torch.float32 else 0,
                                                        s0, s1, slot_ptrs.data_ptr(), per, self._stream()))

    def sum_slots(self, base, nslots, slot_stride, count, out):
        prec = 1 if base.dtype == self.torch.float32 else 0
        C.check(C.lib().nus_sum_slots_device(base.data_ptr(), nslots, slot_stride, count, out.data_ptr(), prec,
                                             self._stream()))

    def ipc_handle(self, t):
        """(64-byte CUDA IPC handle of the allocation holding t, byte offset of t in it).  The
        caching allocator may place t inside a larger cudaMalloc segment and cudaIpcOpenMemHandle
        maps the segment base, so the offset is part of the handle (cuMemGetAddressRange)."""
        buf = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        C.check(C.lib().nus_ipc_get_handle_offset(t.data_ptr(), buf, ctypes.byref(off)))
        return buf.raw, int(off.value)

    def ipc_open(self, handle) -> int:
        raw, offset = handle
        p = ctypes.c_void_p()
        C.check(C.lib().nus_ipc_open(ctypes.create_string_buffer(raw, 64), self.device, ctypes.byref(p)))
        self._mapped[int(p.value) + offset] = int(p.value)
        return int(p.value) + offset

    def ipc_close(self, ptr: int) -> None:
        base = self._mapped.pop(ptr, None)
        if base is not None:
            C.check(C.lib().nus_ipc_close(ctypes.c_void_p(base)))

    def synchronize(self):
        self.torch.cuda.synchronize(self.dev)

    def grid_rows(self, est):
        lo, cnt, nr = C._i32(), C._i32(), C._i32()
        C.check(C.lib().nus_mtnufft_grid_rows(est.h, ctypes.byref(lo), ctypes.byref(cnt), ctypes.byref(nr)))
        return lo.value, cnt.value, nr.value

    def set_grid_rows(self, est, lo, cnt):
        C.check(C.lib().nus_mtnufft_set_grid_rows(est.h, int(lo), int(cnt)))

    def mr(self, est):
        return int(est.info.mr)


# --------------------------------------------------------------------------- shardings

class ChannelShard:
    """Config C3: channels sharded across ranks, no data-path collective."""

    def __init__(self, times, centers, f_max, f_w, k, eps, precision="f32", engine=None, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        times = np.atleast_2d(times)
        self.channels = times.shape[0]
        self.c0, self.c1 = split_range(self.channels, self.world, self.rank)
        self.engine = engine or DeviceEngine()
        f_w = np.broadcast_to(np.asarray(f_w, dtype=np.float64), (self.channels,))
        self.est = None
        if self.c1 > self.c0:
            # one batch estimator per rank: channels share n, centres, K, eps; each channel's tapers
            # are built on its own grid with its OWN half-bandwidth (P must not depend on the rank)
            self.est = self.engine.create(times[self.c0:self.c1], centers, f_max,
                                          np.ascontiguousarray(f_w[self.c0:self.c1]), k, eps, precision, None)
        self.nc = len(centers)

    def estimate_local(self, x_local, power_local):
        """x_local: this rank's channels [c1-c0][n] on the device."""
        if self.est is not None:
            self.engine.estimate(self.est, x_local, power_local)

    def gather(self, power_local):
        """All-gather P of every channel (optional; the throughput path never calls it)."""
        import torch
        counts = [split_range(self.channels, self.world, r) for r in range(self.world)]
        width = max(b - a for a, b in counts)  # collectives need equal shapes: pad, then trim
        padded = torch.zeros((width, self.nc), dtype=power_local.dtype, device=power_local.device)
        padded[: power_local.shape[0]] = power_local
        bufs = [torch.empty_like(padded) for _ in counts]
        self.dist.all_gather(bufs, padded, group=self.group)
        return torch.cat([buf[: b - a] for buf, (a, b) in zip(bufs, counts)], dim=0)


class TaperShard:
    """One series, tapers sharded: rank r spreads all samples for its tapers, then reduce(P)."""

    def __init__(self, times, centers, f_max, f_w, tapers, eps, precision="f64", engine=None, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        self.k = tapers.shape[0]
        self.k0, self.k1 = split_range(self.k, self.world, self.rank)
        self.engine = engine or DeviceEngine()
        self.est = None
        if self.k1 > self.k0:
            self.est = self.engine.create(times, centers, f_max, f_w, self.k1 - self.k0, eps, precision,
                                          tapers[self.k0:self.k1])
        self.nc = len(centers)

    def estimate(self, x, power):
        """x: full series on the device; power: [I] buffer; rank 0 receives P (sum / K)."""
        if self.est is not None:
            self.engine.estimate(self.est, x, power)  # mean over local tapers
            power.mul_(float(self.k1 - self.k0))
        else:
            power.zero_()
        if host_collectives(self.dist, self.group) and power.is_cuda:
            host = power.cpu()
            self.dist.reduce(host, dst=0, op=self.dist.ReduceOp.SUM, group=self.group)
            power.copy_(host)
        else:
            self.dist.reduce(power, dst=0, op=self.dist.ReduceOp.SUM, group=self.group)
        if self.rank == 0:
            power.div_(float(self.k))
        return power


class SampleSplit:
    """Config C4: one long series, samples split across ranks, reduce-scatter of fine grids."""

    fast_normalise_min = 1 << 16  # above this N the R(B) forms use the O(N log N) method (as tapers.cu)

    def __init__(self, times, centers, f_max, f_w, k, eps, precision="f64", engine=None, group=None,
                 tapers: Optional[np.ndarray] = None, fused: Optional[bool] = None):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.group = group
        self.engine = engine or DeviceEngine()
        times = np.asarray(times, dtype=np.float64)
        n = times.size
        self.n, self.k = n, k
        self.s0, self.s1 = split_range(n, self.world, self.rank)
        if tapers is None:
            tapers = self._normalised_tapers(times, f_max, f_w, k)
        self.tapers = tapers
        self.est = self.engine.create(times[self.s0:self.s1], centers, f_max, f_w, k, eps, precision,
                                      tapers[:, self.s0:self.s1])
        if self.world > 1:  # partial grids are summed: every rank covers the union of occupied rows
            self._widen_rows()
        self.kpad = int(math.ceil(k / self.world)) * self.world
        self.per_rank = self.kpad // self.world
        self.mr = self.engine.mr(self.est)
        self.real = self.engine.real_dtype(self.est)
        self.nc = len(centers)
        self.owned = self.engine.zeros((self.per_rank, self.mr * 2), self.real)
        # fused (default with the device engine): the spread stores each taper straight into its
        # owner's receive slot for this rank over peer memory; else a full local grid and NCCL's
        # reduce-scatter (the baseline, and the CPU test engine's path)
        self.fused = hasattr(self.engine, "spread_slots") if fused is None else fused
        if self.fused:
            self._setup_slots()
        else:
            # full local grid [kpad][Mr] complex as interleaved reals; padding rows stay zero
            self.grid = self.engine.zeros((self.kpad, self.mr * 2), self.real)

    def _setup_slots(self):
        """Receive slots [2][G][per][Mr] on every rank (two parities, alternated per spectrum);
        this rank's slot pointer in every owner's buffer for each parity (CUDA IPC peer mappings,
        exchanged with all_gather_object).

        Double buffering closes the write-after-read window: spectrum i+1 stores into the other
        parity, and spectrum i+2 (same parity as i) starts only after the flag all_reduce of
        spectrum i+1, which every owner reaches after its sum_slots of spectrum i (stream order)."""
        import torch
        g, r, per, mr = self.world, self.rank, self.per_rank, self.mr
        alloc = getattr(self.engine, "alloc_slots", self.engine.zeros)
        self.recv = alloc((2, g, per, mr * 2), self.real)
        csize = 2 * self.recv.element_size()
        if g > 1:
            handles = [None] * g
            self.dist.all_gather_object(handles, self.engine.ipc_handle(self.recv), group=self.group)
            self.peers = {o: self.engine.ipc_open(handles[o]) for o in range(g) if o != r}
            bases = [self.recv.data_ptr() if o == r else self.peers[o] for o in range(g)]
        else:
            self.peers = {}
            bases = [self.recv.data_ptr()]
        ptrs = [[b + (par * g + r) * per * mr * csize for b in bases] for par in range(2)]
        self.slot_ptrs = torch.tensor(ptrs, dtype=torch.int64, device=self.recv.device)
        self.parity = 0
        self.flag = torch.zeros(1, dtype=self.real, device=self.recv.device)

    def close(self):
        """Unmap the peer receive slots (CUDA IPC); the estimator's buffers go with the object."""
        if getattr(self, "peers", None) and hasattr(self.engine, "ipc_close"):
            if self.world > 1 and self.dist.is_initialized():
                self.dist.barrier(group=self.group)  # no rank still writes into a peer's slots
            for ptr in self.peers.values():
                self.engine.ipc_close(ptr)
            self.peers = {}

    def _widen_rows(self):
        """Union of the ranks' occupied pass-A rows (a cyclic interval each) -> every rank."""
        if not hasattr(self.engine, "grid_rows"):
            return
        import torch
        lo, cnt, nr = self.engine.grid_rows(self.est)
        if nr == 0:
            return
        occ = torch.zeros(nr, dtype=torch.float64)
        occ[(lo + np.arange(cnt)) % nr] = 1.0
        if self.engine.__class__.__name__ == "DeviceEngine" and not host_collectives(self.dist, self.group):
            occ = occ.to(self.engine.dev)
        self.dist.all_reduce(occ, op=self.dist.ReduceOp.MAX, group=self.group)
        new_lo, new_cnt = covering_interval(occ.cpu().numpy() > 0)
        self.engine.set_grid_rows(self.est, new_lo, new_cnt)

    def _normalised_tapers(self, times, f_max, f_w, k):
        """Interpolated DPSS on the full grid + the R(B) normalisation w^T R(B) w = 2 f_w.

        N > 2^18 (C4): the O(N log N) form (normalise.cu, as the single-GPU setup) on rank 0,
        broadcast so every rank holds bit-identical tapers.  Smaller N: the dense form, row-split
        over the ranks (balanced triangle rows) + an all_reduce of the K partial sums."""
        import torch
        w = self.engine.taper_spline(times, f_max, f_w, k)
        on_device = self.engine.__class__.__name__ == "DeviceEngine" and not host_collectives(self.dist, self.group)
        if times.size > self.fast_normalise_min and hasattr(self.engine, "quadform_fast"):
            q = self.engine.quadform_fast(times, f_max, w) if self.rank == 0 else np.zeros(k)
            qt = torch.tensor(q, dtype=torch.float64)
            if on_device:
                qt = qt.to(self.engine.dev)
            self.dist.broadcast(qt, src=0, group=self.group)
        else:
            rows = balanced_triangle_rows(times.size, self.world)
            q = np.zeros(k)
            for k0 in range(0, k, 8):
                q[k0:k0 + 8] = self.engine.quadform_rows(times, f_max, w[k0:k0 + 8], rows[self.rank],
                                                         rows[self.rank + 1])
            qt = torch.tensor(q, dtype=torch.float64)
            if on_device:
                qt = qt.to(self.engine.dev)
            self.dist.all_reduce(qt, op=self.dist.ReduceOp.SUM, group=self.group)
        q = qt.cpu().numpy()
        if not np.all(q > 0):
            raise C.NumericError("gpss_interpolated: degenerate metric norm")
        return w * np.sqrt(2.0 * f_w / q)[:, None]

    def estimate(self, x_local, power):
        """x_local: this rank's samples [s1-s0] on the device; rank 0 receives P in ``power``."""
        if self.fused:
            par = self.parity
            self.parity ^= 1
            self.engine.spread_slots(self.est, x_local, 0, self.s1 - self.s0, self.slot_ptrs[par], self.per_rank)
            if self.world > 1:  # every rank's slot stores have landed before any owner sums
                if host_collectives(self.dist, self.group):
                    self.engine.synchronize()
                    self.dist.barrier(group=self.group)
                else:  # stream-ordered (NCCL)
                    self.dist.all_reduce(self.flag, op=self.dist.ReduceOp.SUM, group=self.group)
            count = self.per_rank * self.mr
            self.engine.sum_slots(self.recv[par], self.world, count, count, self.owned)
        else:
            self.engine.spread(self.est, x_local, 0, self.s1 - self.s0, self.grid, self.kpad)
            self.dist.reduce_scatter_tensor(self.owned, self.grid, op=self.dist.ReduceOp.SUM, group=self.group)
        k0 = self.rank * self.per_rank
        k1 = min(self.k, k0 + self.per_rank)
        if k1 > k0:
            self.engine.transform(self.est, self.owned, k0, k1, 1.0, power)
        else:
            power.zero_()
        if host_collectives(self.dist, self.group) and power.is_cuda:
            host = power.cpu()
            self.dist.reduce(host, dst=0, op=self.dist.ReduceOp.SUM, group=self.group)
            power.copy_(host)
        else:
            self.dist.reduce(power, dst=0, op=self.dist.ReduceOp.SUM, group=self.group)
        if self.rank == 0:
            power.div_(float(self.k))
        return power
