"""Input generators of the paper's benchmark protocols (reference src/simkit.cpp), restated.

Only what the speed / error harness (:mod:`.harness`) consumes: the
SplitMix64 + polar Box-Muller ``Rng`` with ``substream`` (simkit.cpp:19-57), the paper's four
sampling schemes (simkit.cpp:77-141), white noise (:143-153) and Cholesky-coloured band-limited
noise with covariance density * R(B) (:155-186; R(B) is filled on the device).  Same seeds give
the same grids and series as the reference.  This is input generation, not the estimator path.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _capi as C
from .api import InvalidArgument, NumericError, SamplingGrid, SignalBand, SignalSeries

__all__ = ["Rng", "SamplingScheme", "SimConfig", "scheme_name", "generate_grid", "generate_white_noise",
           "BandlimitedNoiseGenerator", "generate_bandlimited_noise"]

_M64 = 0xFFFFFFFFFFFFFFFF


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class Rng:
    """SplitMix64 with polar Box-Muller Gaussians (simkit.cpp:19-48)."""

    def __init__(self, seed: int):
        self._state = seed & _M64
        self._spare = None

    def next_u64(self) -> int:
        self._state = (self._state + 0x9E3779B97F4A7C15) & _M64
        return _mix(self._state)

    def next_uniform(self) -> float:
        while True:
            u = (self.next_u64() >> 11) * 2.0 ** -53
            if u > 0.0:
                return u

    def next_gauss(self) -> float:
        if self._spare is not None:
            v, self._spare = self._spare, None
            return v
        while True:
            u = 2.0 * self.next_uniform() - 1.0
            v = 2.0 * self.next_uniform() - 1.0
            s = u * u + v * v
            if s >= 1.0 or s == 0.0:
                continue
            f = math.sqrt(-2.0 * math.log(s) / s)
            self._spare = v * f
            return u * f

    @staticmethod
    def substream(seed: int, key: int) -> int:
        """One SplitMix64 scramble of the pair (simkit.cpp:50-56)."""
        return _mix((seed + 0x9E3779B97F4A7C15 * (key + 1)) & _M64)


class SamplingScheme(enum.IntEnum):
    uniform = 0
    jitter = 1
    missing = 2
    arithmetic = 3


def scheme_name(s: SamplingScheme) -> str:
    return SamplingScheme(s).name


@dataclass
class SimConfig:
    """simkit.hpp:44-55."""
    scheme: SamplingScheme = SamplingScheme.uniform
    n: int = 50
    jitter_sigma: float = 0.1
    intensity: float = 1.0
    missing_indices: Sequence[int] = field(default_factory=lambda: [1, 5, 17, 18, 19, 23, 27, 32, 53, 56])
    missing_base_dt: float = 5.0 / 6.0
    arith_a: float = 2.0 / 3.0
    arith_b: float = (2.0 / 3.0) / 48.0
    seed: int = 0
    retry_budget: int = 100


def generate_grid(config: SimConfig) -> SamplingGrid:
    if config.n < 2:
        raise InvalidArgument("generate_grid: n must be >= 2")
    s = SamplingScheme(config.scheme)
    if s == SamplingScheme.uniform:
        t = [float(i) for i in range(1, config.n + 1)]
    elif s == SamplingScheme.jitter:
        if not config.jitter_sigma >= 0.0:
            raise InvalidArgument("generate_grid: jitter_sigma must be >= 0")
        if not config.intensity > 0.0:
            raise InvalidArgument("generate_grid: intensity must be > 0")
        rng = Rng(Rng.substream(config.seed, 0x6A69747465720000))
        for _ in range(config.retry_budget):
            t = [i / config.intensity + config.jitter_sigma * rng.next_gauss() for i in range(1, config.n + 1)]
            if all(t[i] > t[i - 1] for i in range(1, len(t))):
                break
        else:
            raise NumericError("generate_grid: jitter draws never produced an increasing grid")
    elif s == SamplingScheme.missing:
        omit = set(config.missing_indices)
        if len(omit) != len(config.missing_indices):
            raise InvalidArgument("generate_grid: duplicate missing indices")
        base = config.n + len(config.missing_indices)
        if any(i < 1 or i > base for i in omit):
            raise InvalidArgument("generate_grid: missing index out of range")
        t = [config.missing_base_dt * i for i in range(1, base + 1) if i not in omit]
    else:
        t = [1.0 + config.arith_a * k + config.arith_b * k * (k - 1.0) / 2.0 for k in range(config.n)]
    return SamplingGrid(t)


def generate_white_noise(grid: SamplingGrid, variance: float, seed: int) -> SignalSeries:
    if not variance > 0.0:
        raise InvalidArgument("generate_white_noise: variance must be > 0")
    rng = Rng(Rng.substream(seed, 0x676175737300))
    sd = math.sqrt(variance)
    return SignalSeries(grid, [sd * rng.next_gauss() for _ in range(grid.n_samples())])


class BandlimitedNoiseGenerator:
    """Samples with covariance density * R(B) by Cholesky colouring (simkit.cpp:155-186): the
    factor of density * (R(B) + ridge * trace/n * I), ridge 1e-12 then 1e-9, computed once."""

    def __init__(self, grid: SamplingGrid, band: SignalBand, density: float, device: int = 0):
        if not density > 0.0:
            raise InvalidArgument("BandlimitedNoiseGenerator: density must be > 0")
        self._grid = grid
        t = C.f64(grid.times())
        n = t.size
        rb = np.empty((n, n))
        C.check(C.lib().nus_signal_band_matrix(C.dptr(t), n, band.f_max, device, C.dptr(rb)))
        unit = np.trace(rb) / n
        for f in (1e-12, 1e-9):
            try:
                self._chol = np.linalg.cholesky(density * rb + (f * unit * density) * np.eye(n))
                return
            except np.linalg.LinAlgError:
                continue
        from ._capi import ConditioningError
        raise ConditioningError("BandlimitedNoiseGenerator: kernel not factorizable")

    def generate(self, seed: int) -> SignalSeries:
        rng = Rng(Rng.substream(seed, 0x636F6C6F72656400))
        z = np.array([rng.next_gauss() for _ in range(self._grid.n_samples())])
        return SignalSeries(self._grid, self._chol @ z)


def generate_bandlimited_noise(grid: SamplingGrid, band: SignalBand, density: float, seed: int) -> SignalSeries:
    return BandlimitedNoiseGenerator(grid, band, density).generate(seed)
