"""GPU: the distributed shardings through the real DeviceEngine (C-ABI spread/transform
building blocks + NCCL collectives) in a world-size-1 NCCL group (gpurun gives one GPU).
The multi-rank partitioning itself is covered by tests/test_distributed.py (gloo, world 2)."""
import os
import socket

import numpy as np
import pytest

from conftest import rel_l2
from oracle import C
from paper_2407_01943_b200 import distributed as D
from paper_2407_01943_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("fused", [True, False])
def test_sample_split_device_engine(nccl_group, fused):
    """World-1 NCCL group: the fused path (spread into receive slots + slot sum) and the
    baseline (full local grid + reduce_scatter)."""
    import torch
    wl = W.small(n=20000, n_centers=8192, k=5, nw=3.0, eps=1e-9, seed=3)
    ss = D.SampleSplit(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), 5, 1e-9, fused=fused)
    assert ss.fused == fused
    x = torch.as_tensor(wl.values, device="cuda")
    p = torch.zeros(wl.centers.size, dtype=torch.float64, device="cuda")
    ss.estimate(x, p)
    ref = C.mtnufft_power(wl.times, ss.tapers, wl.values, wl.centers, 1e-9)
    assert rel_l2(p.cpu().numpy(), ref) < 1e-10
    w_ref, _ = C.gpss_interpolated(wl.times, wl.f_max, float(wl.f_w[0]), 5)
    assert np.abs(np.abs(ss.tapers) - np.abs(w_ref)).max() < 1e-9 * np.abs(w_ref).max()


def test_taper_and_channel_shard_device_engine(nccl_group):
    import torch
    wl = W.small(n=20000, n_centers=8192, k=4, nw=2.5, eps=1e-9, seed=4)
    w, _ = C.gpss_interpolated(wl.times, wl.f_max, float(wl.f_w[0]), 4)
    ts = D.TaperShard(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), w, 1e-9)
    p = torch.zeros(wl.centers.size, dtype=torch.float64, device="cuda")
    ts.estimate(torch.as_tensor(wl.values, device="cuda"), p)
    assert rel_l2(p.cpu().numpy(), C.mtnufft_power(wl.times, w, wl.values, wl.centers, 1e-9)) < 1e-10
    c3 = W.c3(channels=3, n=1 << 14)
    centers = 2500.0 * np.arange(1 << 13) / ((1 << 13) - 1)
    cs = D.ChannelShard(c3.times, centers, 2500.0, c3.f_w, 9, 1e-5, precision="f32")
    pl = torch.zeros((3, centers.size), dtype=torch.float32, device="cuda")
    cs.estimate_local(torch.as_tensor(c3.values, dtype=torch.float32, device="cuda"), pl)
    allp = cs.gather(pl).cpu().numpy()
    wc = cs.est.tapers()
    for ch in range(3):
        ref = C.mtnufft_power(c3.times[ch], wc[ch], c3.values[ch], centers, 1e-9)
        assert rel_l2(allp[ch], ref) <= 1e-4


@pytest.mark.parametrize("kern", ["gaussian", "es"])
@pytest.mark.parametrize("ranks", [2, 4])
def test_sample_split_emulated_ranks_on_one_gpu(kern, ranks):
    """The sample split's device path with G ranks emulated on one GPU (no collective: the
    reduce-scatter is a sum of the G partial grids): each chunk's estimator occupies different
    pass-A rows (C2-like Poisson times span half the grid period), so the row intervals are
    widened to their union first (nus_mtnufft_set_grid_rows); P equals the single-GPU P."""
    import torch
    wl = W.c2(n=1 << 18)
    eng = D.DeviceEngine()
    full = eng.create(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), 7, 1e-9, "f64", None)
    w = full.tapers()[0]
    p_full = full.power(wl.values)[0]
    kpad = -(-7 // ranks) * ranks
    per = kpad // ranks
    parts, rows = [], []
    for r in range(ranks):
        s0, s1 = D.split_range(wl.n, ranks, r)
        e = eng.create(wl.times[s0:s1], wl.centers, wl.f_max, float(wl.f_w[0]), 7, 1e-9, "f64", w[:, s0:s1])
        parts.append((e, s0, s1))
        rows.append(eng.grid_rows(e))
    nr = rows[0][2]
    assert nr > 0 and len({(lo, cnt) for lo, cnt, _ in rows}) > 1  # the chunks occupy different rows
    occ = np.zeros(nr, dtype=bool)
    for lo, cnt, _ in rows:
        occ[(lo + np.arange(cnt)) % nr] = True
    lo, cnt = D.covering_interval(occ)
    mr = eng.mr(full)
    total = torch.zeros((kpad, 2 * mr), dtype=torch.float64, device="cuda")
    for e, s0, s1 in parts:
        eng.set_grid_rows(e, lo, cnt)
        g = torch.zeros((kpad, 2 * mr), dtype=torch.float64, device="cuda")
        x = torch.as_tensor(wl.values[s0:s1], device="cuda")
        eng.spread(e, x, 0, s1 - s0, g, kpad)
        total += g
    power = torch.zeros(wl.centers.size, dtype=torch.float64, device="cuda")
    for r, (e, _, _) in enumerate(parts):
        k0, k1 = r * per, min(7, (r + 1) * per)
        if k1 > k0:
            owned = total[k0:k0 + per].contiguous()
            pr = torch.zeros_like(power)
            eng.transform(e, owned, k0, k1, 1.0, pr)
            power += pr
    torch.cuda.synchronize()
    p = power.cpu().numpy() / 7.0
    assert rel_l2(p, p_full) < 1e-12


@pytest.mark.parametrize("kern", ["gaussian", "es"])
@pytest.mark.parametrize("ranks,cfg", [(2, "c2"), (3, "c2"), (2, "c4"), (3, "c4")])
def test_fused_slot_exchange_emulated_ranks_on_one_gpu(kern, ranks, cfg):
    """The fused sample-split exchange with G ranks emulated on one GPU: rank r's spread stores
    taper k straight into owner k // per's receive slot r (device pointer table; peer NVLink
    addresses on a multi-GPU box), each owner sums its G slots in rank order and transforms its
    tapers.  P equals the single-GPU P; K = 7 / 15 pads to a multiple of G (empty padding tapers);
    C4's structure (K = 15, dense windows) takes the two-taper-group spread into the slots."""
    import torch
    wl = W.c2(n=1 << 18) if cfg == "c2" else W.c4(n=1 << 18, n_centers=1 << 16, windows=40)
    K = wl.k
    eng = D.DeviceEngine()
    full = eng.create(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), K, 1e-9, "f64", None)
    w = full.tapers()[0]
    p_full = full.power(wl.values)[0]
    kpad = -(-K // ranks) * ranks
    per = kpad // ranks
    mr = eng.mr(full)
    parts, rows = [], []
    for r in range(ranks):
        s0, s1 = D.split_range(wl.n, ranks, r)
        e = eng.create(wl.times[s0:s1], wl.centers, wl.f_max, float(wl.f_w[0]), K, 1e-9, "f64", w[:, s0:s1])
        parts.append((e, s0, s1))
        rows.append(eng.grid_rows(e))
    occ = np.zeros(rows[0][2], dtype=bool)
    for lo, cnt, nr in rows:
        occ[(lo + np.arange(cnt)) % nr] = True
    lo, cnt = D.covering_interval(occ)
    recv = [torch.zeros((ranks, per, 2 * mr), dtype=torch.float64, device="cuda") for _ in range(ranks)]
    for r, (e, s0, s1) in enumerate(parts):
        eng.set_grid_rows(e, lo, cnt)
        ptrs = torch.tensor([recv[o].data_ptr() + r * per * mr * 16 for o in range(ranks)], dtype=torch.int64,
                            device="cuda")
        eng.spread_slots(e, torch.as_tensor(wl.values[s0:s1], device="cuda"), 0, s1 - s0, ptrs, per)
    power = torch.zeros(wl.centers.size, dtype=torch.float64, device="cuda")
    for o, (e, _, _) in enumerate(parts):
        owned = torch.zeros((per, 2 * mr), dtype=torch.float64, device="cuda")
        eng.sum_slots(recv[o], ranks, per * mr, per * mr, owned)
        k0, k1 = o * per, min(K, (o + 1) * per)
        if k1 > k0:
            pr = torch.zeros_like(power)
            eng.transform(e, owned, k0, k1, 1.0, pr)
            power += pr
    torch.cuda.synchronize()
    assert rel_l2(power.cpu().numpy() / K, p_full) < 1e-12


def _ipc_worker(rank, world, port, q, tapers, kern):
    import torch
    import torch.distributed as dist

    import paper_2407_01943_b200 as nus
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        nus.set_spread_kernel(kern)  # the parent's window (the comparison is bit-level)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        wl = W.c2(n=1 << 18)
        ss = D.SampleSplit(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), 7, 1e-9, tapers=tapers, fused=True)
        assert ss.fused and len(ss.peers) == world - 1
        x = torch.as_tensor(wl.values[ss.s0:ss.s1], device="cuda")
        p = torch.zeros(wl.centers.size, dtype=torch.float64, device="cuda")
        ss.estimate(x, p)
        p2 = torch.zeros_like(p)
        ss.estimate(x, p2)  # a second spectrum through the same slots
        if rank == 0:
            q.put((p.cpu().numpy(), p2.cpu().numpy()))
        ss.close()  # barrier + unmap the peer slots
        assert ss.peers == {}
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures instead of waiting for the timeout
        q.put(e)
        raise


@pytest.mark.parametrize("kern", ["gaussian", "es"])
def test_fused_exchange_real_cuda_ipc_two_processes_one_gpu(kern):
    """The fused exchange with real CUDA IPC: two processes on one GPU (gloo for the host-side
    barrier and the small collectives; no kernel waits on another process), each spreading its
    half of the samples straight into both owners' receive slots through the peer mappings
    (handle + allocation offset exchanged with all_gather_object).  P equals the single-GPU P."""
    import multiprocessing as mp

    from paper_2407_01943_b200.api import _Estimator
    wl = W.c2(n=1 << 18)
    full = _Estimator(wl.times, wl.centers, wl.f_max, float(wl.f_w[0]), 7, 1e-9, 1, "f64", 0)
    tapers = full.tapers()[0]
    p_full = full.power(wl.values)[0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q, tapers, kern)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    if isinstance(res, Exception):
        raise res
    assert all(p.exitcode == 0 for p in procs)
    p1, p2 = res
    assert rel_l2(p1, p_full) < 1e-12
    assert np.array_equal(p1, p2)
