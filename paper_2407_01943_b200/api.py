"""Python mirror of the reference's public interface for the MTNUFFT path.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/nuspectral/{grid,tapers,nufft,estimators}.hpp),
so the parity tests read like the reference's own doctest files.  All compute
goes through the C-ABI (include/nus_c.h) into libnus_b200.so on the GPU;
the small host-side pieces here are the reference's input validation
(grid.cpp) and plain data containers.
"""
from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as C
from ._capi import (BandRangeError, ConditioningError, DegenerateTapers, ExtrapolationError, InvalidArgument,
                    NoDeviceError, NusError, NumericError, PlanMismatch, SpectralRangeError)

__all__ = [
    "SamplingGrid", "SignalSeries", "SignalBand", "AnalysisBand", "BandPlan", "make_band_plan",
    "band_near_boundary", "NufftPath", "NufftPathPolicy", "NufftPlan", "ndft_direct", "nufft_fast",
    "DpssSet", "dpss_uniform", "tridiagonal_eigen", "TaperSet", "gpss_interpolated",
    "signal_band_quadform", "signal_band_quadform_fast", "EigenCoefficients", "eigencoefficients", "SpectrumEstimate",
    "MtnufftEstimator", "estimate_mtnufft", "default_taper_count", "kBandBoundary", "kBandFailed",
    "NusError", "InvalidArgument", "PlanMismatch", "BandRangeError", "ExtrapolationError",
    "NumericError", "NoDeviceError", "Precision", "DegenerateTapers", "FTestResult", "FTestOptions",
    "f_test", "f_quantile", "kFtestConditionViolated", "kFtestSaturated",
    "GeneralizedEigenOptions", "generalized_hermitian_eigen", "gpss_exact", "EigenPairs",
    "ConditioningError", "SpectralRangeError", "SpreadKernel", "set_spread_kernel",
    "get_spread_kernel", "spread_kernel", "Radix2Fft", "MultiDeviceEstimator",
]

kBandBoundary = 1  # grid.hpp:10
kBandFailed = 2    # grid.hpp:11


class Precision(enum.IntEnum):
    f64 = C.F64
    f32 = C.F32


def _prec(p) -> int:
    if isinstance(p, str):
        return {"f64": C.F64, "fp64": C.F64, "float64": C.F64, "f32": C.F32, "fp32": C.F32,
                "float32": C.F32}[p]
    return int(p)


# ---------------------------------------------------------------- grid.hpp

class SamplingGrid:
    """Strictly increasing sample instants (grid.cpp:9-22)."""

    def __init__(self, times):
        t = np.array(times, dtype=np.float64).reshape(-1)
        if t.size < 2:
            raise InvalidArgument("SamplingGrid: need at least 2 samples")
        if not np.all(np.isfinite(t)):
            raise InvalidArgument("SamplingGrid: non-finite sample time")
        if not np.all(t[1:] > t[:-1]):
            raise InvalidArgument("SamplingGrid: times must be strictly increasing")
        self._t = t
        self._t.setflags(write=False)
        self.mean_dt = (t[-1] - t[0]) / t.size

    def times(self) -> np.ndarray:
        return self._t

    def n_samples(self) -> int:
        return self._t.size

    def span(self) -> float:
        return float(self._t[-1] - self._t[0])

    def __eq__(self, other):
        return isinstance(other, SamplingGrid) and np.array_equal(self._t, other._t)


class SignalSeries:
    def __init__(self, grid: SamplingGrid, values):
        v = np.array(values, dtype=np.float64).reshape(-1)
        if v.size != grid.n_samples():
            raise InvalidArgument("SignalSeries: values length must match grid")
        self.grid = grid
        self.values = v


class SignalBand:
    def __init__(self, f_max: float):
        if not (f_max > 0.0) or not math.isfinite(f_max):
            raise InvalidArgument("SignalBand: f_max must be positive")
        self.f_max = float(f_max)


class AnalysisBand:
    def __init__(self, f_center: float, half_width: float):
        if not (f_center >= 0.0) or not math.isfinite(f_center):
            raise InvalidArgument("AnalysisBand: f_center must be >= 0")
        if not (half_width > 0.0) or not math.isfinite(half_width):
            raise InvalidArgument("AnalysisBand: half_width must be positive")
        self.f_center = float(f_center)
        self.half_width = float(half_width)


def band_near_boundary(f_center, f_max, margin) -> bool:  # grid.cpp:46-51
    tol = 1e-9 * margin
    return f_center < margin - tol or (f_max - f_center) < margin - tol


class BandPlan:
    """Equal-width bands with strictly increasing centres (grid.cpp:53-78)."""

    def __init__(self, bands: Sequence[AnalysisBand], f_max: float, boundary_margin: float):
        bands = list(bands)
        if not bands:
            raise InvalidArgument("BandPlan: empty band set")
        fw = bands[0].half_width
        for i, b in enumerate(bands):
            if b.half_width != fw:
                raise InvalidArgument("BandPlan: bands must share one half_width")
            if i > 0 and not (b.f_center > bands[i - 1].f_center):
                raise InvalidArgument("BandPlan: centers must be strictly increasing")
        self._centers = np.array([b.f_center for b in bands])
        self._fw = fw
        self.f_max = float(f_max)
        self.boundary_margin = float(boundary_margin)
        c = self._centers
        tol = 1e-9 * boundary_margin
        self._flags = ((c < boundary_margin - tol) | ((f_max - c) < boundary_margin - tol)).astype(np.uint8)

    @classmethod
    def from_centers(cls, centers, half_width, f_max, boundary_margin=None):
        """Vectorised constructor (same validation) for large I."""
        obj = cls.__new__(cls)
        c = np.array(centers, dtype=np.float64).reshape(-1)
        if c.size == 0:
            raise InvalidArgument("BandPlan: empty band set")
        if not (half_width > 0.0):
            raise InvalidArgument("AnalysisBand: half_width must be positive")
        if c.size > 1 and not np.all(c[1:] > c[:-1]):
            raise InvalidArgument("BandPlan: centers must be strictly increasing")
        if not np.all(c >= 0.0):
            raise InvalidArgument("AnalysisBand: f_center must be >= 0")
        obj._centers = c
        obj._fw = float(half_width)
        obj.f_max = float(f_max)
        obj.boundary_margin = 2.0 * half_width if boundary_margin is None else float(boundary_margin)
        tol = 1e-9 * obj.boundary_margin
        m = obj.boundary_margin
        obj._flags = ((c < m - tol) | ((f_max - c) < m - tol)).astype(np.uint8)
        return obj

    def size(self) -> int:
        return self._centers.size

    def half_width(self) -> float:
        return self._fw

    def center(self, i: int) -> float:
        return float(self._centers[i])

    def centers(self) -> np.ndarray:
        return self._centers.copy()

    def flags(self) -> np.ndarray:
        return self._flags.copy()

    def flagged(self, i: int) -> bool:
        return bool(self._flags[i])


def make_band_plan(f_max: float, f_w: float, spacing: float, boundary_margin: Optional[float] = None):
    """grid.cpp:80-103."""
    if not (f_max > 0.0):
        raise InvalidArgument("make_band_plan: f_max must be positive")
    if not (f_w > 0.0):
        raise InvalidArgument("make_band_plan: f_w must be positive")
    if not (spacing > 0.0):
        raise InvalidArgument("make_band_plan: spacing must be positive")
    if not (f_w <= f_max / 2.0):
        raise InvalidArgument("make_band_plan: f_w must be <= f_max/2")
    if not (spacing <= 2.0 * f_w):
        raise InvalidArgument("make_band_plan: spacing must be <= 2*f_w")
    count = int(math.floor(f_max / spacing + 1e-9)) + 1
    margin = 2.0 * f_w if boundary_margin is None else boundary_margin
    return BandPlan([AnalysisBand(i * spacing, f_w) for i in range(count)], f_max, margin)


# ---------------------------------------------------------------- nufft.hpp

class NufftPath(enum.IntEnum):
    direct = C.PATH_DIRECT
    fast = C.PATH_FAST


class NufftPathPolicy(enum.IntEnum):
    auto_select = C.AUTO_SELECT
    force_fast = C.FORCE_FAST
    force_direct = C.FORCE_DIRECT


class SpreadKernel(enum.IntEnum):
    """Fast-path window: ``gaussian`` is the reference's (nufft.cpp:90-142, replicated to
    ~1e-12); ``es`` (exponential of semicircle, the default) meets the same error contract
    max|fast - direct| <= eps ||y||_1 with ~2.4x narrower support (es.cu)."""
    gaussian = 0
    es = 1


def set_spread_kernel(kind) -> None:
    """Process-wide window for plans / estimators created afterwards (nus_set_spread_kernel)."""
    k = SpreadKernel[kind] if isinstance(kind, str) else SpreadKernel(int(kind))
    C.check(C.lib().nus_set_spread_kernel(int(k)))


def get_spread_kernel() -> SpreadKernel:
    v = ctypes.c_int32()
    C.check(C.lib().nus_get_spread_kernel(ctypes.byref(v)))
    return SpreadKernel(v.value)


class spread_kernel:
    """Context manager: ``with spread_kernel("gaussian"): ...`` restores the previous window."""

    def __init__(self, kind):
        self.kind = kind

    def __enter__(self):
        self.prev = get_spread_kernel()
        set_spread_kernel(self.kind)
        return self

    def __exit__(self, *a):
        set_spread_kernel(self.prev)


class NufftPlan:
    """Device-resident NufftPlan (nufft.hpp:31-76).  execute() runs on the GPU."""

    kFastThreshold = 1 << 14

    def __init__(self, grid: SamplingGrid, centers, epsilon: float,
                 policy: NufftPathPolicy = NufftPathPolicy.auto_select, oversampling: int = 2,
                 precision="f64", device: int = 0):
        self._grid = grid
        self._centers = C.f64(centers).reshape(-1)
        h = ctypes.c_void_p()
        t = C.f64(grid.times())
        C.check(C.lib().nus_plan_create(C.dptr(t), t.size, C.dptr(self._centers), self._centers.size,
                                        float(epsilon), int(policy), int(oversampling),
                                        _prec(precision), int(device), ctypes.byref(h)))
        self._h = h
        info = C.PlanInfo()
        C.check(C.lib().nus_plan_info(self._h, ctypes.byref(info)))
        self._info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            try:
                C.lib().nus_plan_destroy(h)
            except Exception:  # interpreter shutdown: the module globals may already be gone
                pass

    # accessors (nufft.hpp:41-48)
    def n_samples(self):
        return int(self._info.n_samples)

    def n_centers(self):
        return int(self._info.n_centers)

    def centers(self):
        return self._centers.copy()

    def epsilon(self):
        return float(self._info.epsilon)

    def oversampling(self):
        return int(self._info.oversampling)

    def spread_width(self):
        return int(self._info.spread_width)

    def path(self) -> NufftPath:
        return NufftPath(self._info.path)

    def centers_uniform(self) -> bool:
        return bool(self._info.centers_uniform)

    def grid_size(self) -> int:
        return int(self._info.mr)

    def tau(self) -> float:
        return float(self._info.tau)

    def spread_kernel(self) -> SpreadKernel:
        return SpreadKernel(self._info.kernel)

    def support(self) -> int:
        """Cells per sample actually spread: 2w (Gaussian) or ns (ES)."""
        return int(self._info.support)

    def grid(self) -> SamplingGrid:
        return self._grid

    def first_cells(self) -> np.ndarray:
        out = np.empty(self.n_samples(), np.int64)
        C.check(C.lib().nus_plan_first_cells(self._h, out.ctypes.data_as(C._i64p)))
        return out

    def sort_order(self) -> np.ndarray:
        out = np.empty(self.n_samples(), np.int32)
        C.check(C.lib().nus_plan_sort_order(self._h, out.ctypes.data_as(C._i32p)))
        return out

    def execute(self, weighted_values) -> np.ndarray:
        y = C.c128_as_f64(np.asarray(weighted_values, dtype=np.complex128).reshape(-1))
        out = np.empty(2 * self.n_centers())
        C.check(C.lib().nus_plan_execute(self._h, C.dptr(y), y.size // 2, C.dptr(out)))
        return out.view(np.complex128)


def nufft_fast(plan: NufftPlan, weighted_values) -> np.ndarray:
    return plan.execute(weighted_values)


def ndft_direct(grid: SamplingGrid, weighted_values, centers, device: int = 0) -> np.ndarray:
    """Exact NUDFT on the device in fp64 (nufft.cpp:36-54)."""
    t = C.f64(grid.times())
    y = C.c128_as_f64(np.asarray(weighted_values, dtype=np.complex128).reshape(-1))
    if y.size // 2 != t.size:
        raise InvalidArgument("ndft_direct: length mismatch")
    c = C.f64(centers).reshape(-1)
    out = np.empty(2 * c.size)
    C.check(C.lib().nus_ndft_direct(C.dptr(t), t.size, C.dptr(y), C.dptr(c), c.size, device,
                                    C.dptr(out)))
    return out.view(np.complex128)


# ---------------------------------------------------------------- fft.hpp

class Radix2Fft:
    """fft.hpp:12-29: forward X_k = sum_j x_j e^{-2 pi i jk/n}; inverse the conjugate transform
    without the 1/n scale.  Runs on the device (fft.cu's radix-2 Stockham kernels)."""

    def __init__(self, n: int, device: int = 0):
        n = int(n)
        if n <= 0 or (n & (n - 1)) != 0:
            raise InvalidArgument("Radix2Fft: size must be a power of two")
        self._n, self._device = n, int(device)

    def size(self) -> int:
        return self._n

    @staticmethod
    def is_power_of_two(n: int) -> bool:
        return n != 0 and (n & (n - 1)) == 0

    @staticmethod
    def next_power_of_two(n: int) -> int:
        p = 1
        while p < n:
            p <<= 1
        return p

    def _run(self, data, inverse):
        z = np.ascontiguousarray(np.asarray(data, np.complex128).reshape(-1)).copy()
        if z.size != self._n:
            raise InvalidArgument("Radix2Fft: data length differs from the transform size")
        C.check(C.lib().nus_fft_inplace(z.view(np.float64).ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        self._n, int(inverse), self._device))
        return z

    def forward(self, data) -> np.ndarray:
        return self._run(data, False)

    def inverse(self, data) -> np.ndarray:
        return self._run(data, True)


# ---------------------------------------------------------------- tapers.hpp

@dataclass
class DpssSet:
    tapers: np.ndarray          # K x n, unit norm
    concentrations: np.ndarray  # K, in [0, 1]
    eigenvalues: np.ndarray = field(default=None)  # of the commuting tridiagonal


def dpss_uniform(n: int, time_half_bandwidth: float, k_tapers: int, device: int = 0,
                 concentrations: bool = True) -> DpssSet:
    if n < 2:
        raise InvalidArgument("dpss_uniform: n must be >= 2")
    if k_tapers < 1 or k_tapers > n:
        raise InvalidArgument("dpss_uniform: k_tapers out of range")
    tap = np.empty((k_tapers, n))
    ev = np.empty(k_tapers)
    conc = np.empty(k_tapers) if concentrations else None
    C.check(C.lib().nus_dpss(n, float(time_half_bandwidth), k_tapers, device, C.dptr(tap), C.dptr(ev),
                             C.dptr(conc) if conc is not None else None))
    return DpssSet(tap, conc, ev)


@dataclass
class EigenPairs:
    values: np.ndarray
    vectors: np.ndarray
    residuals: np.ndarray


def tridiagonal_eigen(diag, offdiag, k_top: int, device: int = 0) -> EigenPairs:
    d, e = C.f64(diag).reshape(-1), C.f64(offdiag).reshape(-1)
    n = d.size
    if n == 0:
        raise InvalidArgument("tridiagonal_eigenvalues: empty matrix")
    if k_top == 0 or k_top > n:
        raise InvalidArgument("tridiagonal_eigen: k_top out of range")
    if e.size + 1 != n:
        raise InvalidArgument("tridiagonal_eigenvalues: offdiag length must be n-1")
    vals, res = np.empty(k_top), np.empty(k_top)
    vecs = np.empty((k_top, n))
    e_arg = e if e.size else np.zeros(1)
    C.check(C.lib().nus_tridiagonal_eigen(C.dptr(d), C.dptr(e_arg), n, k_top, device, C.dptr(vals),
                                          C.dptr(vecs), C.dptr(res)))
    return EigenPairs(vals, vecs, res)


class TaperSet:
    """K real weight sequences on a grid (tapers.hpp:29-63)."""

    def __init__(self, grid: SamplingGrid, band: AnalysisBand, f_max: float, weights,
                 eigenvalues=None, is_real: bool = True):
        w = np.array(weights, dtype=np.float64 if is_real else np.complex128)
        if w.ndim != 2 or w.shape[0] == 0:
            raise InvalidArgument("TaperSet: no tapers")
        if w.shape[1] != grid.n_samples():
            raise InvalidArgument("TaperSet: taper length mismatch")
        if eigenvalues is not None and len(eigenvalues) and len(eigenvalues) != w.shape[0]:
            raise InvalidArgument("TaperSet: eigenvalue count mismatch")
        self._grid, self._band, self._f_max = grid, band, float(f_max)
        self._real = bool(is_real)
        self._w = w
        self._ev = np.array(eigenvalues if eigenvalues is not None else [], dtype=np.float64)

    def k_tapers(self):
        return self._w.shape[0]

    def n_samples(self):
        return self._w.shape[1]

    def grid(self):
        return self._grid

    def band(self):
        return self._band

    def f_max(self):
        return self._f_max

    def is_real(self):
        return self._real

    def has_eigenvalues(self):
        return self._ev.size > 0

    def eigenvalues(self):
        return self._ev

    def weights(self, k):
        return self._w[k].astype(np.complex128)

    def weights_real(self, k):
        if not self._real:
            raise InvalidArgument("TaperSet: weights_real on complex tapers")
        return self._w[k]

    def weights_matrix(self):
        return self._w

    def zero_frequency_responses(self):
        return self._w.sum(axis=1).astype(np.complex128)


def signal_band_quadform(grid: SamplingGrid, band: SignalBand, w, rows=None, device: int = 0):
    """w^T R(B) w per row of w, on the device (kernels.cpp:28-37,100-115, no dense matrix)."""
    t = C.f64(grid.times())
    w = C.f64(np.atleast_2d(w))
    r0, r1 = (0, t.size) if rows is None else rows
    q = np.empty(w.shape[0])
    C.check(C.lib().nus_signal_band_quadform(C.dptr(t), t.size, band.f_max, C.dptr(w), w.shape[0],
                                             r0, r1, device, C.dptr(q)))
    return q


def signal_band_quadform_fast(grid: SamplingGrid, band: SignalBand, w, device: int = 0):
    """The same w^T R(B) w in O(N log N): windowed lattice sum of |W(f)|^2 over [-F, F] from the
    path's own type-1 NUFFT (normalise.cu)."""
    t = C.f64(grid.times())
    w = C.f64(np.atleast_2d(w))
    q = np.empty(w.shape[0])
    C.check(C.lib().nus_signal_band_quadform_fast(C.dptr(t), t.size, band.f_max, C.dptr(w), w.shape[0],
                                                  device, C.dptr(q)))
    return q


def taper_spline(grid: SamplingGrid, band: SignalBand, f_w: float, k_tapers: int, device: int = 0):
    """Un-normalised interpolated DPSS (tapers.cpp:156-174)."""
    t = C.f64(grid.times())
    w = np.empty((k_tapers, t.size))
    C.check(C.lib().nus_taper_spline(C.dptr(t), t.size, band.f_max, float(f_w), k_tapers, device,
                                     C.dptr(w)))
    return w


def gpss_interpolated(grid: SamplingGrid, signal_band: SignalBand, f_w: float, k_tapers: int,
                      device: int = 0) -> TaperSet:
    """tapers.cpp:146-182 on the device."""
    t = C.f64(grid.times())
    w = np.empty((max(k_tapers, 1), t.size))
    C.check(C.lib().nus_gpss_interpolated(C.dptr(t), t.size, signal_band.f_max, float(f_w), k_tapers,
                                          device, C.dptr(w)))
    return TaperSet(grid, AnalysisBand(0.0, f_w), signal_band.f_max, w, None, True)


@dataclass
class GeneralizedEigenOptions:
    """eig.hpp:38-44."""
    want_vectors: bool = True
    ridge_first: float = 1e-12
    ridge_retry: float = 1e-9


def generalized_hermitian_eigen(a, m, k_top: int, opts: Optional[GeneralizedEigenOptions] = None,
                                device: int = 0) -> EigenPairs:
    """A w = lambda M w on the device (eig.cpp:612-659): Cholesky with ridge, dense Hermitian
    eigensolve (cuSOLVER), the k largest pairs with values clamped into [0, 1], M-normalised
    vectors with the canonical phase, residuals ||A w - lambda M w|| / (||A||_F ||w||)."""
    opts = opts or GeneralizedEigenOptions()
    a = np.asarray(a)
    m = C.f64(m)
    if a.ndim != 2 or a.shape[0] != a.shape[1] or m.shape != a.shape:
        raise InvalidArgument("generalized_hermitian_eigen: size mismatch")
    if np.iscomplexobj(m) or np.iscomplexobj(np.asarray(m)):
        raise InvalidArgument("generalized_hermitian_eigen: metric must be the real signal-band kernel")
    if k_top < 1:
        raise InvalidArgument("generalized_hermitian_eigen: k_top must be >= 1")
    n = a.shape[0]
    k = min(int(k_top), n)
    are = C.f64(np.real(a))
    aim = C.f64(np.imag(a)) if np.iscomplexobj(a) else None
    vals, res = np.empty(k), np.empty(k)
    vecs = np.empty((k, n, 2))
    C.check(C.lib().nus_generalized_eigen(C.dptr(are), C.dptr(aim) if aim is not None else None, C.dptr(m), n, k,
                                          opts.ridge_first, opts.ridge_retry, 1 if opts.want_vectors else 0, device,
                                          C.dptr(vals), C.dptr(vecs), C.dptr(res)))
    if not opts.want_vectors:
        return EigenPairs(vals, np.empty((0, n), np.complex128), np.empty(0))
    return EigenPairs(vals, vecs[..., 0] + 1j * vecs[..., 1], res)


def gpss_exact(grid: SamplingGrid, signal_band: SignalBand, band: AnalysisBand, k_tapers: int,
               opts: Optional[GeneralizedEigenOptions] = None, device: int = 0) -> TaperSet:
    """Exact nominal-band GPSS tapers (tapers.cpp:118-144): R(A) w = lambda R(B) w on the device,
    each taper scaled to w^H R(B) w = 2 f_w.  Real for a band centred at 0."""
    opts = opts or GeneralizedEigenOptions()
    t = C.f64(grid.times())
    k = int(k_tapers)
    w = np.empty((max(k, 1), t.size, 2))
    conc = np.empty(max(k, 1))
    C.check(C.lib().nus_gpss_exact(C.dptr(t), t.size, signal_band.f_max, band.f_center, band.half_width, k,
                                   opts.ridge_first, opts.ridge_retry, device, C.dptr(w), C.dptr(conc)))
    real_band = band.f_center == 0.0
    wc = w[..., 0] + 1j * w[..., 1]
    return TaperSet(grid, band, signal_band.f_max, wc.real.copy() if real_band else wc, conc, real_band)


def default_taper_count(time_half_bandwidth: float) -> int:  # tapers.cpp:219-222
    k = int(math.floor(2.0 * time_half_bandwidth + 0.5)) - 1 if time_half_bandwidth >= 0 else -1
    return max(k, 1)


# ---------------------------------------------------------------- estimators.hpp

@dataclass
class EigenCoefficients:
    n_tapers: int
    n_bands: int
    data: np.ndarray  # K x I complex

    def at(self, k, i):
        return self.data[k, i]

    def row(self, k):
        return self.data[k]


@dataclass
class SpectrumEstimate:
    plan: BandPlan
    power: np.ndarray
    method: str
    k_used: np.ndarray
    f_w_used: np.ndarray
    flags: np.ndarray


class _Estimator:
    """Owns one nus_mtnufft handle (channels share n, centres, K, epsilon)."""

    def __init__(self, times, centers, f_max, f_w, k, epsilon, policy, precision, device,
                 tapers=None):
        t = C.f64(times)
        if t.ndim == 1:
            t = t[None, :]
        self.channels, self.n = t.shape
        c = C.f64(centers).reshape(-1)
        # f_w: one half-bandwidth for every channel, or one per channel (each channel's tapers are
        # built on its own grid with its own f_w, as one reference estimator per channel would)
        fw = np.atleast_1d(C.f64(f_w)).reshape(-1)
        if fw.size not in (1, self.channels):
            raise InvalidArgument("MtnufftEstimator: f_w must be a scalar or one value per channel")
        fw = np.ascontiguousarray(np.broadcast_to(fw, (self.channels,)), dtype=np.float64)
        self.f_w = fw
        cfg = C.MtnufftConfig(self.channels, self.n, c.size, int(k), float(f_max), float(fw[0]),
                              float(epsilon), int(policy), _prec(precision), int(device), 0)
        tp = None
        if tapers is not None:
            tp = C.f64(tapers).reshape(self.channels, int(k), self.n)
        h = ctypes.c_void_p()
        C.check(C.lib().nus_mtnufft_create_channels(ctypes.byref(cfg), C.dptr(t), C.dptr(c), C.dptr(fw),
                                                    C.dptr(tp) if tp is not None else None, ctypes.byref(h)))
        self.h = h
        self.k = int(k)
        self.nc = c.size
        info = C.PlanInfo()
        C.check(C.lib().nus_mtnufft_plan_info(self.h, ctypes.byref(info)))
        self.info = info

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.h = None
            try:
                C.lib().nus_mtnufft_destroy(h)
            except Exception:  # interpreter shutdown: the module globals may already be gone
                pass

    def stage_kernels(self):
        """Names of the kernels of the three per-spectrum stages (spread; FFT pass A; pass B + crop)."""
        buf = ctypes.create_string_buffer(256)
        C.check(C.lib().nus_mtnufft_stage_kernels(self.h, buf, 256))
        return buf.value.decode().split(";")

    def tapers(self):
        out = np.empty((self.channels, self.k, self.n))
        C.check(C.lib().nus_mtnufft_tapers(self.h, C.dptr(out)))
        return out

    def setup_ms(self):
        out = np.empty(5)
        C.check(C.lib().nus_mtnufft_setup_ms(self.h, C.dptr(out)))
        return dict(zip(["dpss", "spline", "normalise", "plan", "total"], out.tolist()))

    def power(self, x):
        x = C.f64(x).reshape(self.channels, self.n)
        out = np.empty((self.channels, self.nc))
        C.check(C.lib().nus_mtnufft_estimate(self.h, C.dptr(x), C.dptr(out)))
        return out

    def power_batch(self, xs):
        """[steps][channels][n] -> [steps][channels][I]; copies overlapped across steps."""
        xs = C.f64(xs).reshape(-1, self.channels, self.n)
        out = np.empty((xs.shape[0], self.channels, self.nc))
        C.check(C.lib().nus_mtnufft_estimate_batch(self.h, C.dptr(xs), xs.shape[0], C.dptr(out)))
        return out

    def f_test(self, x, cap=1e12):
        x = C.f64(x).reshape(self.channels, self.n)
        f = np.empty((self.channels, self.nc))
        amp = np.empty(2 * self.channels * self.nc)
        flags = np.empty((self.channels, self.nc), np.uint8)
        C.check(C.lib().nus_mtnufft_f_test(self.h, C.dptr(x), cap, C.dptr(f), C.dptr(amp),
                                           flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return f, amp.view(np.complex128).reshape(self.channels, self.nc), flags

    def eigencoefficients(self, x):
        x = C.f64(x).reshape(self.channels, self.n)
        out = np.empty(2 * self.channels * self.k * self.nc)
        C.check(C.lib().nus_mtnufft_eigencoefficients(self.h, C.dptr(x), C.dptr(out)))
        return out.view(np.complex128).reshape(self.channels, self.k, self.nc)

    def bytes_model(self, x_dtype=0):
        vals = [ctypes.c_double() for _ in range(4)]
        C.check(C.lib().nus_mtnufft_bytes_model(self.h, x_dtype, *[ctypes.byref(v) for v in vals]))
        return dict(zip(["total", "spread", "fft", "crop"], [v.value for v in vals]))


class MultiDeviceEstimator:
    """MtnufftEstimator over several GPUs of this process (include/nus_c.h nus_mtnufft_multi_*):
    ``sharding`` "channels" (independent channels, no exchange), "tapers" (one series, tapers
    split, partial spectra summed on devices[0]) or "samples" (one series, contiguous sample chunks,
    the spread storing each taper's grid straight into its owner device's slot over peer memory).
    A device may be listed more than once (emulated parts on one GPU)."""

    SHARDINGS = {"channels": 0, "tapers": 1, "samples": 2}

    def __init__(self, times, centers, f_max, f_w, k, epsilon, devices, sharding="samples", precision="f64",
                 tapers=None, policy=NufftPathPolicy.auto_select):
        t = C.f64(times)
        if t.ndim == 1:
            t = t[None, :]
        self.channels, self.n = t.shape
        c = C.f64(centers).reshape(-1)
        fw = np.ascontiguousarray(np.broadcast_to(np.atleast_1d(C.f64(f_w)).reshape(-1), (self.channels,)),
                                  dtype=np.float64)
        devs = np.ascontiguousarray(devices, dtype=np.int32).reshape(-1)
        if sharding not in self.SHARDINGS:
            raise InvalidArgument(f"MultiDeviceEstimator: unknown sharding {sharding!r}")
        # an empty device list reaches the C-ABI, which rejects it (NUS_ERR_INVALID_ARGUMENT)
        cfg = C.MtnufftConfig(self.channels, self.n, c.size, int(k), float(f_max), float(fw[0]), float(epsilon),
                              int(policy), _prec(precision), int(devs[0]) if devs.size else 0, 0)
        tp = None if tapers is None else C.f64(tapers).reshape(self.channels, int(k), self.n)
        h = ctypes.c_void_p()
        C.check(C.lib().nus_mtnufft_multi_create(ctypes.byref(cfg), devs.ctypes.data_as(C._i32p), devs.size,
                                                 self.SHARDINGS[sharding], C.dptr(t), C.dptr(c), C.dptr(fw),
                                                 C.dptr(tp) if tp is not None else None, ctypes.byref(h)))
        self.h, self.k, self.nc = h, int(k), c.size

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.h = None
            try:
                C.lib().nus_mtnufft_multi_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    def estimate(self, x) -> np.ndarray:
        x = C.f64(x).reshape(self.channels, self.n)
        out = np.empty((self.channels, self.nc))
        C.check(C.lib().nus_mtnufft_multi_estimate(self.h, C.dptr(x), C.dptr(out)))
        return out

    def tapers(self) -> np.ndarray:
        out = np.empty((self.channels, self.k, self.n))
        C.check(C.lib().nus_mtnufft_multi_tapers(self.h, C.dptr(out)))
        return out

    def peer_bytes(self) -> int:
        v = ctypes.c_int64()
        C.check(C.lib().nus_mtnufft_multi_peer_bytes(self.h, ctypes.byref(v)))
        return int(v.value)


def eigencoefficients(tapers: TaperSet, series: SignalSeries, plan: NufftPlan,
                      precision=None) -> EigenCoefficients:
    """nufft.cpp:194-227: row k = transform of w_k * x onto the plan's centres."""
    n = series.grid.n_samples()
    if tapers.n_samples() != n or plan.n_samples() != n:
        raise PlanMismatch("eigencoefficients: tapers, series and plan must share one grid")
    if not (tapers.grid() == series.grid):
        raise PlanMismatch("eigencoefficients: taper grid differs from series grid")
    est = _Estimator(series.grid.times(), plan.centers(), tapers.f_max(), tapers.band().half_width,
                     tapers.k_tapers(), plan.epsilon(), int(plan.path() == NufftPath.fast and 1 or 2),
                     precision if precision is not None else plan._info.precision, 0,
                     tapers=tapers.weights_matrix())
    j = est.eigencoefficients(series.values)[0]
    return EigenCoefficients(tapers.k_tapers(), plan.n_centers(), j)


class MtnufftEstimator:
    """estimators.hpp:39-62.  Setup (tapers, bins, sort, tables) and estimate() on the GPU."""

    @dataclass
    class Options:
        k_tapers: int = 4
        epsilon: float = 1e-8
        taper_mode: str = "interpolated"
        path_policy: NufftPathPolicy = NufftPathPolicy.auto_select
        precision: str = "f64"
        device: int = 0

    def __init__(self, grid: SamplingGrid, signal_band: SignalBand, plan: BandPlan,
                 opts: Optional["MtnufftEstimator.Options"] = None, tapers=None):
        opts = opts or MtnufftEstimator.Options()
        if opts.taper_mode not in ("interpolated", "exact_nominal"):
            raise InvalidArgument(f"MtnufftEstimator: unknown taper mode {opts.taper_mode!r}")
        self._grid, self._plan, self._opts = grid, plan, opts
        self._method = "mtnufft"
        self._conc = None
        if opts.taper_mode == "exact_nominal" and tapers is None:
            # MTNUFFT0 (estimators.cpp:91-104): exact nominal-band tapers from the dense GEP
            ts = gpss_exact(grid, signal_band, AnalysisBand(0.0, plan.half_width()), opts.k_tapers,
                            device=opts.device)
            tapers, self._conc = ts.weights_matrix(), ts.eigenvalues()
            self._method = "mtnufft0"
        self._est = _Estimator(grid.times(), plan.centers(), signal_band.f_max, plan.half_width(),
                               opts.k_tapers, opts.epsilon, int(opts.path_policy), opts.precision,
                               opts.device, tapers=tapers)

    def estimate(self, values) -> SpectrumEstimate:
        v = np.asarray(values, dtype=np.float64).reshape(-1)
        if v.size != self._grid.n_samples():
            raise InvalidArgument("estimate: series length does not match grid")
        p = self._est.power(v)[0]
        bands = self._plan.size()
        if np.any(~(p >= 0.0)):
            raise InvalidArgument("SpectrumEstimate: negative power")
        return SpectrumEstimate(self._plan, p, self._method, np.full(bands, self._opts.k_tapers),
                                np.full(bands, self._plan.half_width()), self._plan.flags())

    def estimate_many(self, series) -> List[SpectrumEstimate]:
        """estimate() of many series on this grid in one pipelined call (the H2D / D2H copies of
        one series overlap the compute of its neighbours).  Same results as estimate() each."""
        v = np.asarray(series, dtype=np.float64)
        if v.ndim != 2 or v.shape[1] != self._grid.n_samples():
            raise InvalidArgument("estimate_many: expected [series][n_samples] values")
        p = self._est.power_batch(v)
        bands = self._plan.size()
        return [SpectrumEstimate(self._plan, p[i, 0], self._method, np.full(bands, self._opts.k_tapers),
                                 np.full(bands, self._plan.half_width()), self._plan.flags()) for i in range(len(v))]

    def eigencoefficients(self, values) -> EigenCoefficients:
        j = self._est.eigencoefficients(values)[0]
        return EigenCoefficients(self._opts.k_tapers, self._plan.size(), j)

    def f_test(self, values, opts: Optional["FTestOptions"] = None) -> "FTestResult":
        """Harmonic F-test with the eigencoefficients kept on the device (inference.cpp:132-186)."""
        opts = opts or FTestOptions()
        v = np.asarray(values, dtype=np.float64).reshape(-1)
        if v.size != self._grid.n_samples():
            raise InvalidArgument("estimate: series length does not match grid")
        if self._opts.k_tapers < 2:
            raise InvalidArgument("f_test: need at least 2 tapers")
        f, amp, flags = self._est.f_test(v, opts.saturation_cap)
        return _ftest_result(self._plan, f[0], amp[0], flags[0], self._opts.k_tapers,
                             self._grid.n_samples(), opts)

    def tapers(self) -> TaperSet:
        w = self._est.tapers()[0]
        return TaperSet(self._grid, AnalysisBand(0.0, self._plan.half_width()), self._plan.f_max, w, self._conc)

    def transform_info(self):
        return self._est.info

    def stage_kernels(self):
        """Kernels launched per spectrum: [spread, FFT pass A, pass B + crop/power]."""
        return self._est.stage_kernels()

    def method(self) -> str:
        return self._method

    def setup_ms(self):
        return self._est.setup_ms()


def estimate_mtnufft(series: SignalSeries, signal_band: SignalBand, plan: BandPlan, k_tapers: int,
                     epsilon: float, precision="f64") -> SpectrumEstimate:
    """Cold one-shot (estimators.cpp:261-270)."""
    opts = MtnufftEstimator.Options(k_tapers=k_tapers, epsilon=epsilon, precision=precision)
    return MtnufftEstimator(series.grid, signal_band, plan, opts).estimate(series.values)


# ---------------------------------------------------------------- inference.hpp

kFtestConditionViolated = 1  # inference.hpp:16
kFtestSaturated = 2          # inference.hpp:17


@dataclass
class FTestOptions:
    p_levels: Sequence[float] = ()
    saturation_cap: float = 1e12


@dataclass
class FTestResult:
    plan: BandPlan
    f_stat: np.ndarray
    amplitude: np.ndarray
    dof: tuple
    critical_values: List[tuple]
    flags: np.ndarray
    saturation_cap: float


def f_quantile(p: float, d1: int, d2: int) -> float:
    """Upper-tail F(d1, d2) critical value (inference.cpp:94-130); host scalar math in the library."""
    out = ctypes.c_double()
    C.check(C.lib().nus_f_quantile(float(p), int(d1), int(d2), ctypes.byref(out)))
    return out.value


def _ftest_result(plan, f, amp, flags, k, n, opts):
    levels = list(opts.p_levels) or [0.05, 0.01, 1.0 / n]
    crit = [(p, f_quantile(p, 2, 2 * k - 2)) for p in levels]
    return FTestResult(plan, f, amp, (2, 2 * k - 2), crit, flags, opts.saturation_cap)


def f_test(eigencoeffs: EigenCoefficients, tapers: TaperSet, plan: BandPlan,
           opts: Optional[FTestOptions] = None, device: int = 0) -> FTestResult:
    """inference.cpp:132-186 on the device (host eigencoefficients in, as the reference API)."""
    opts = opts or FTestOptions()
    k = tapers.k_tapers()
    if k < 2:
        raise InvalidArgument("f_test: need at least 2 tapers")
    if eigencoeffs.n_tapers != k or eigencoeffs.n_bands != plan.size():
        raise InvalidArgument("f_test: eigencoefficient shape mismatch")
    j = C.c128_as_f64(np.asarray(eigencoeffs.data, np.complex128).reshape(k, plan.size()))
    w0 = C.c128_as_f64(tapers.zero_frequency_responses())
    c = C.f64(plan.centers())
    nb = plan.size()
    f = np.empty(nb)
    amp = np.empty(2 * nb)
    flags = np.empty(nb, np.uint8)
    C.check(C.lib().nus_f_test(C.dptr(j), k, nb, C.dptr(w0), tapers.n_samples(), C.dptr(c), plan.half_width(),
                               opts.saturation_cap, device, C.dptr(f), C.dptr(amp),
                               flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
    return _ftest_result(plan, f, amp.view(np.complex128), flags, k, tapers.n_samples(), opts)
