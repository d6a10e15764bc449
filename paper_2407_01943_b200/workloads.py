"""Seeded synthetic inputs for the BASELINE.json configurations (C1..C5).

No public dataset is involved (the paper's impedance data is proprietary);
these generators follow the shapes, sizes and value distributions that
BASELINE.json states for each config.  Every draw comes from
the reference's own generator (``Rng`` of src/simkit.cpp:19-57: SplitMix64,
uniform = (u64 >> 11) 2^-53 rejecting 0, polar Box-Muller with a cached spare),
consumed in bulk by :class:`RefRng` -- bit-identical to calling the reference's
next_uniform / next_gauss in the same order -- with one substream per config
and channel, ``Rng::substream(Rng::substream(20240702, config), channel)``
(SURVEY §8(d)); the reference's own tooling regenerates the same inputs.

Conventions shared by all configs:
  * f_w = NW / (h N) with h = span / (N - 1), so the reference's
    tw = f_w * h * N equals NW exactly in exact arithmetic (tapers.cpp:156-157);
  * centres are the uniform grid the config names, built as (F * i) / (I - 1)
    (or i / 32 for C4, which must be dyadic to pass nufft.cpp:23-32 at I = 2^24);
  * the band plan uses half-width f_w and boundary margin 2 f_w (grid.cpp:53-72).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
from scipy.signal import lfilter

BASE_SEED = 20240702
_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def substream(seed: int, key: int) -> int:
    """Rng::substream (simkit.cpp:50-56): one SplitMix64 scramble of (seed, key)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + _GAMMA * np.uint64(key + 1)
    return int(_mix64(np.array([z], dtype=np.uint64))[0])


def stream_seed(config: int, channel: int = 0) -> int:
    return substream(substream(BASE_SEED, config), channel)


class RefRng:
    """The reference Rng (simkit.cpp:19-48) with a numpy-Generator-like surface, vectorised.

    ``random`` / ``uniform`` consume next_uniform() calls and ``standard_normal`` next_gauss()
    calls in order, exactly as a loop over the reference's methods would (tests/test_workloads.py
    checks this against the scalar restatement simkit.Rng); the other draws are defined on top:
    exponential = -scale ln(U), lognormal = exp(mu + sigma Z), integers = lo + floor(U (hi - lo)),
    permutation = stable argsort of m uniforms."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.spare = None

    def _u64(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            z = self.state + _GAMMA * np.arange(1, n + 1, dtype=np.uint64)
            self.state = self.state + _GAMMA * np.uint64(n)
        return _mix64(z)

    def random(self, n=None):
        m = 1 if n is None else int(n)
        out = (self._u64(m) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        while True:  # next_uniform rejects 0 (probability 2^-53 per draw): refill in order
            bad = np.flatnonzero(out == 0.0)
            if bad.size == 0:
                break
            i = int(bad[0])
            out[i:] = np.concatenate([out[i + 1:], (self._u64(1) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53])
        return float(out[0]) if n is None else out

    def uniform(self, lo=0.0, hi=1.0, n=None):
        return lo + (hi - lo) * self.random(n)

    def standard_normal(self, n=None):
        m = 1 if n is None else int(n)
        out = np.empty(m)
        k = 0
        if self.spare is not None and m > 0:
            out[0] = self.spare
            self.spare = None
            k = 1
        while k < m:
            need = m - k
            pairs = max(16, int((need + 1) // 2 * 1.3) + 8)
            r = self.random(2 * pairs)
            u, v = 2.0 * r[0::2] - 1.0, 2.0 * r[1::2] - 1.0
            s = u * u + v * v
            ok = np.flatnonzero((s < 1.0) & (s != 0.0))
            if ok.size == 0:
                continue
            # a pair is consumed only up to the one that completes the request: rewind the rest
            used_pairs = int(ok[min(ok.size, (need + 1) // 2) - 1]) + 1
            acc = ok[ok < used_pairs]
            f = np.sqrt(-2.0 * np.log(s[acc]) / s[acc])
            z = np.empty(2 * acc.size)
            z[0::2] = u[acc] * f
            z[1::2] = v[acc] * f
            with np.errstate(over="ignore"):
                self.state = self.state - _GAMMA * np.uint64(2 * (pairs - used_pairs))
            take = min(need, z.size)
            out[k:k + take] = z[:take]
            k += take
            if take < z.size:
                self.spare = float(z[take])
        return float(out[0]) if n is None else out

    def exponential(self, scale=1.0, n=None):
        return -scale * np.log(self.random(n))

    def lognormal(self, mu=0.0, sigma=1.0, n=None):
        return np.exp(mu + sigma * self.standard_normal(n))

    def integers(self, lo, hi, n=None):
        v = lo + np.floor(self.random(n) * (hi - lo)).astype(np.int64)
        return int(v) if n is None else v

    def permutation(self, m: int) -> np.ndarray:
        return np.argsort(self.random(m), kind="stable")


@dataclass
class Workload:
    name: str
    times: np.ndarray          # [C][N] or [N]
    values: np.ndarray         # [C][N] or [N]
    centers: np.ndarray        # [I]
    f_max: float
    nw: float
    k: int
    eps: float
    precision: str
    f_w: np.ndarray = field(default=None)  # per channel
    note: str = ""

    @property
    def channels(self) -> int:
        return 1 if self.times.ndim == 1 else self.times.shape[0]

    @property
    def n(self) -> int:
        return self.times.shape[-1]


def half_width_for(times: np.ndarray, nw: float) -> float:
    n = times.size
    h = (times[-1] - times[0]) / (n - 1)
    return nw / (h * n)


def _uniform_centers(f_max: float, count: int) -> np.ndarray:
    return (f_max * np.arange(count, dtype=np.float64)) / (count - 1)


def _strict(t: np.ndarray) -> np.ndarray:
    assert np.all(np.diff(t) > 0), "generated grid is not strictly increasing"
    return t


def c1(scale: int = 1) -> Workload:
    """N=4096 from a 256 Hz grid, +-0.3/fs jitter, 20% dropped; 3 lines + AR(2)."""
    rng = RefRng(stream_seed(1))
    fs = 256.0
    n = 4096 // scale
    m = (n * 5) // 4
    j = np.arange(m)
    base = j / fs + rng.uniform(-0.3, 0.3, m) / fs
    keep = np.sort(rng.permutation(m)[:n])
    t = _strict(base[keep])
    # AR(2) a1=0.75, a2=-0.5, innovation sigma 0.75 (unit stationary variance), burn-in 1000
    e = 0.75 * rng.standard_normal(m + 1000)
    ar = lfilter([1.0], [1.0, -0.75, 0.5], e)[1000:]
    x = (np.sin(2 * np.pi * 10 * t) + 0.5 * np.sin(2 * np.pi * 40 * t)
         + 0.1 * np.sin(2 * np.pi * 97 * t) + ar[keep])
    centers = _uniform_centers(128.0, n)
    wl = Workload("c1", t, x, centers, 128.0, 4.0, 7, 1e-9, "f64")
    wl.f_w = np.array([half_width_for(t, 4.0)])
    return wl


def c2(n: int = 1 << 20, precision: str = "f64", seed_offset: int = 0) -> Workload:
    """Poisson times (mean 1 ms), AR(4) poles 0.95 e^{+-i0.1pi}, e^{+-i0.3pi} + 60 Hz line."""
    rng = RefRng(stream_seed(2, seed_offset))
    while True:
        t = np.cumsum(rng.exponential(1e-3, n))
        t -= t[0]
        if np.all(np.diff(t) > 0):
            break
    poles = 0.95 * np.exp(1j * np.pi * np.array([0.1, -0.1, 0.3, -0.3]))
    a = np.real(np.poly(poles))
    e = rng.standard_normal(n + 4096)
    x = lfilter([1.0], a, e)[4096:] + 0.2 * np.cos(2 * np.pi * 60 * t)
    centers = _uniform_centers(500.0, n)
    eps = 1e-9 if precision == "f64" else 1e-5
    wl = Workload("c2", t, x, centers, 500.0, 4.0, 7, eps, precision)
    wl.f_w = np.array([half_width_for(t, 4.0)])
    return wl


def c3(channels: int = 256, n: int = 1 << 18, first_channel: int = 0) -> Workload:
    """Jittered 5 kHz grids with 1-5 gaps each; 1/f^alpha noise + 80-250 Hz bursts; fp32."""
    fs = 5000.0
    times = np.empty((channels, n))
    vals = np.empty((channels, n))
    for c in range(channels):
        rng = RefRng(stream_seed(3, first_channel + c))
        t = np.arange(n) / fs + rng.uniform(-0.1, 0.1, n) / fs
        for _ in range(int(rng.integers(1, 6))):
            at = int(rng.integers(1, n))
            t[at:] += rng.uniform(0.05, 0.5)
        times[c] = _strict(t)
        alpha = rng.uniform(1.0, 2.0)
        spec = np.fft.rfft(rng.standard_normal(n))
        f = np.fft.rfftfreq(n)
        shape = np.zeros_like(f)
        shape[1:] = f[1:] ** (-alpha / 2.0)
        noise = np.fft.irfft(spec * shape, n)
        noise /= noise.std()
        x = noise
        for _ in range(int(rng.integers(1, 4))):
            f0 = rng.uniform(80.0, 250.0)
            dur = rng.uniform(0.1, 0.5)
            amp = rng.uniform(0.5, 2.0)
            t0 = rng.uniform(t[0], max(t[0], t[-1] - dur))
            inside = (t >= t0) & (t < t0 + dur)
            ph = (t[inside] - t0) / dur
            x[inside] += amp * np.sin(np.pi * ph) ** 2 * np.sin(2 * np.pi * f0 * t[inside])
        vals[c] = x
    centers = _uniform_centers(2500.0, n // 2)
    wl = Workload("c3", times, vals, centers, 2500.0, 5.0, 9, 1e-5, "f32")
    wl.f_w = np.array([half_width_for(times[c], 5.0) for c in range(channels)])
    return wl


def c4(n: int = 1 << 26, n_centers: int = 1 << 24, windows: int = 400) -> Workload:
    """Clustered: 400 nightly windows (lognormal length), Poisson inside; 5 lines + noise."""
    rng = RefRng(stream_seed(4))
    start = np.arange(windows) + rng.uniform(0.0, 0.25, windows)
    length = np.minimum(rng.lognormal(np.log(0.2), 0.5, windows), 0.7)
    share = length / length.sum() * n
    counts = np.floor(share).astype(np.int64)
    rem = n - counts.sum()
    counts[np.argsort(-(share - counts))[:rem]] += 1
    parts = []
    for w in range(windows):
        parts.append(np.sort(start[w] + length[w] * rng.random(counts[w])))
    t = np.concatenate(parts)
    dup = np.flatnonzero(np.diff(t) <= 0)
    while dup.size:
        t[dup + 1] = np.nextafter(t[dup + 1], np.inf)
        dup = np.flatnonzero(np.diff(t) <= 0)
    periods = np.exp(rng.uniform(np.log(0.1), np.log(50.0), 5))
    phases = rng.uniform(0.0, 2 * np.pi, 5)
    sig = np.zeros(n)
    for p, ph in zip(periods, phases):
        sig += np.sin(2 * np.pi * t / p + ph)
    power = np.mean(sig ** 2)
    x = sig + np.sqrt(10.0 * power) * rng.standard_normal(n)
    centers = np.arange(n_centers, dtype=np.float64) / 32.0
    f_max = (n_centers - 1) / 32.0
    wl = Workload("c4", t, x, centers, f_max, 8.0, 15, 1e-9, "f64")
    wl.f_w = np.array([half_width_for(t, 8.0)])
    return wl


def c5(n: int = 1 << 22, k: int = 7, eps: float = 1e-9, precision: str = "f64") -> Workload:
    """Jittered unit grid (+-0.4), 10% dropped; unit white noise."""
    rng = RefRng(stream_seed(5))
    m = int(np.ceil(n / 0.9))
    base = np.arange(m) + rng.uniform(-0.4, 0.4, m)
    keep = np.sort(rng.permutation(m)[:n])
    t = _strict(base[keep])
    x = rng.standard_normal(n)
    centers = _uniform_centers(0.5, n // 2)
    nw = (k + 1) / 2.0
    wl = Workload("c5", t, x, centers, 0.5, nw, k, eps, precision)
    wl.f_w = np.array([half_width_for(t, nw)])
    return wl


def small(n: int = 2048, n_centers: Optional[int] = None, k: int = 5, nw: float = 3.0,
          eps: float = 1e-9, seed: int = 0, precision: str = "f64", f_max: float = 0.5) -> Workload:
    """Small jittered/dropout grid for quick parity cases."""
    rng = RefRng(stream_seed(100, seed))
    m = int(n * 1.25)
    base = np.arange(m) + rng.uniform(-0.35, 0.35, m)
    keep = np.sort(rng.permutation(m)[:n])
    t = _strict(base[keep])
    x = rng.standard_normal(n) + np.cos(2 * np.pi * 0.1234 * t)
    nc = n_centers or n // 2
    centers = _uniform_centers(f_max, nc)
    wl = Workload("small", t, x, centers, f_max, nw, k, eps, precision)
    wl.f_w = np.array([half_width_for(t, nw)])
    return wl


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
