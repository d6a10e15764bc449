"""The paper's speed and error protocols for the MTNUFFT estimators.

Mirrors the reference's bench.hpp / src/bench.cpp:130-275 for the methods on this path,
``mtnufft`` (interpolated DPSS tapers) and ``mtnufft0`` (exact nominal-band GPSS), run on the
B200 through :class:`~.api.MtnufftEstimator`.  The Bronez estimators (bg_fixed, bg_adaptive)
and the baseline are out of scope and rejected.

* :func:`run_error_analysis` — per (method, scheme) mean and standard error over ``trials`` of
  the squared dB error against the flat unit spectrum, P / (2 f_w) -> 0 dB, on band-limited
  noise coloured with R(B) (bench.cpp:130-204).
* :func:`run_speed_analysis` — wall-clock spectra/s of COLD estimation (tapers and plan rebuilt
  per call) in batches of at least ``min_batch_seconds`` after a warm-up call (bench.cpp:206-275).
* :func:`write_error_reports_json` / :func:`write_speed_reports_json` — the reference's report
  files (io.cpp:191-262): 2-space indent, keys in byte order, NaN as null.
"""
from __future__ import annotations

import math
import platform
import time
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import api
from .api import InvalidArgument, MtnufftEstimator, SignalBand, make_band_plan
from .simkit import BandlimitedNoiseGenerator, Rng, SamplingScheme, SimConfig, generate_grid, generate_white_noise

__all__ = ["BenchConfig", "ErrorReport", "SpeedConfig", "SpeedReport", "run_error_analysis", "run_speed_analysis",
           "write_error_reports_json", "write_speed_reports_json", "METHODS"]

METHODS = ("mtnufft", "mtnufft0")
_ALL_METHODS = ("mtnufft", "mtnufft0", "bg_fixed", "bg_adaptive", "baseline")  # EstimatorMethod order


def _method_name(m) -> str:
    name = _ALL_METHODS[int(m)] if isinstance(m, (int, np.integer)) else str(m)
    if name not in METHODS:
        raise InvalidArgument(f"harness: method {name!r} is outside the MTNUFFT path (mtnufft, mtnufft0 only)")
    return name


@dataclass
class BenchConfig:
    """bench.hpp:15-24 (the error-analysis defaults)."""
    f_max: float = 0.5
    f_w: float = 0.05
    k_tapers: int = 4
    spacing: float = 0.01
    n_samples: int = 50
    epsilon: float = 1e-8
    device: int = 0


@dataclass
class ErrorReport:
    method: str
    scheme: SamplingScheme
    centers: np.ndarray
    mse_db_mean: np.ndarray
    mse_db_sem: np.ndarray
    flags: np.ndarray
    trials: int = 0
    base_seed: int = 0
    f_w: float = 0.0
    k_tapers: int = 0
    failed_bands: int = 0


@dataclass
class SpeedConfig:
    bench: BenchConfig = field(default_factory=BenchConfig)
    min_batch_seconds: float = 0.05
    max_cell_seconds: float = 120.0


@dataclass
class SpeedReport:
    method: str
    scheme: SamplingScheme
    spectra_per_second_mean: float = 0.0
    spectra_per_second_std: float = 0.0
    calls: int = 0
    batches: int = 0
    environment: str = ""
    timestamp: str = ""


def _estimator(method: str, grid, band, plan, cfg: BenchConfig) -> MtnufftEstimator:
    mode = "interpolated" if method == "mtnufft" else "exact_nominal"
    opts = MtnufftEstimator.Options(k_tapers=cfg.k_tapers, epsilon=cfg.epsilon, taper_mode=mode, device=cfg.device)
    return MtnufftEstimator(grid, band, plan, opts)


def _scheme_config(scheme, n, seed) -> SimConfig:
    return SimConfig(scheme=SamplingScheme(scheme), n=n, seed=seed)


def run_error_analysis(methods: Sequence, schemes: Sequence, trials: int, base_seed: int,
                       config: BenchConfig = BenchConfig()) -> List[ErrorReport]:
    if trials < 2:
        raise InvalidArgument("run_error_analysis: trials must be >= 2")
    names = [_method_name(m) for m in methods]
    band = SignalBand(config.f_max)
    plan = make_band_plan(config.f_max, config.f_w, config.spacing)
    bands = plan.size()
    reports = []
    for s, scheme in enumerate(schemes):
        grid = generate_grid(_scheme_config(scheme, config.n_samples, Rng.substream(base_seed, s)))
        noise = BandlimitedNoiseGenerator(grid, band, 1.0, device=config.device)
        est = [_estimator(m, grid, band, plan, config) for m in names]
        sq = np.zeros((len(names), trials, bands))
        flags = [plan.flags() for _ in names]
        for m in range(trials):
            series = noise.generate(Rng.substream(base_seed, (s + 1) * 1000003 + m))
            for q, e in enumerate(est):
                r = e.estimate(series.values)
                if m == 0:
                    flags[q] = np.asarray(r.flags)
                failed = (np.asarray(r.flags) & api.kBandFailed) != 0
                db = 10.0 * np.log10(np.asarray(r.power) / (2.0 * np.asarray(r.f_w_used)))
                sq[q, m] = np.where(failed, np.nan, db * db)
        for q, name in enumerate(names):
            failed = (flags[q] & api.kBandFailed) != 0
            mean = sq[q].mean(axis=0)
            sem = np.sqrt(sq[q].var(axis=0, ddof=1) / trials)
            reports.append(ErrorReport(name, SamplingScheme(scheme), np.asarray(plan.centers()),
                                       np.where(failed, np.nan, mean), np.where(failed, np.nan, sem),
                                       np.asarray(flags[q], np.uint8), trials, base_seed, config.f_w,
                                       config.k_tapers, int(failed.sum())))
    return reports


def _environment() -> str:
    from . import _capi
    return f"device={_capi.device_name() if hasattr(_capi, 'device_name') else 'cuda'} host={platform.machine()}"


def run_speed_analysis(methods: Sequence, schemes: Sequence, reps: int,
                       config: SpeedConfig = SpeedConfig()) -> List[SpeedReport]:
    if reps < 10:
        raise InvalidArgument("run_speed_analysis: reps must be >= 10")
    cfg = config.bench
    names = [_method_name(m) for m in methods]
    band = SignalBand(cfg.f_max)
    plan = make_band_plan(cfg.f_max, cfg.f_w, cfg.spacing)
    env = _environment()
    reports = []
    for s, scheme in enumerate(schemes):
        grid = generate_grid(_scheme_config(scheme, cfg.n_samples, Rng.substream(17, s)))
        series = generate_white_noise(grid, 1.0, 99 + s)

        for name in names:
            def cold():  # tapers and plan rebuilt per call (bench.cpp:101-126)
                return _estimator(name, grid, band, plan, cfg).estimate(series.values)

            t0 = time.perf_counter()
            cold()
            per_call = max(time.perf_counter() - t0, 1e-9)
            batch = max(1, math.ceil(config.min_batch_seconds / per_call))
            rates, calls = [], 0
            cell0 = time.perf_counter()
            while calls < reps and time.perf_counter() - cell0 < config.max_cell_seconds:
                b0 = time.perf_counter()
                for _ in range(batch):
                    cold()
                rates.append(batch / (time.perf_counter() - b0))
                calls += batch
                if len(rates) >= 2 and calls >= reps:
                    break
            while len(rates) < 2:
                b0 = time.perf_counter()
                for _ in range(batch):
                    cold()
                rates.append(batch / (time.perf_counter() - b0))
                calls += batch
            mean = float(np.mean(rates))
            std = float(np.std(rates, ddof=1)) if len(rates) > 1 else 0.0
            reports.append(SpeedReport(name, SamplingScheme(scheme), mean, std, calls, len(rates), env,
                                       time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())))
    return reports


# ---- report files (io.cpp:191-262) ---------------------------------------------------------

def _json(v, indent: int = 0) -> str:
    pad, inner = "  " * indent, "  " * (indent + 1)
    if isinstance(v, dict):
        if not v:
            return "{}"
        keys = sorted(v, key=lambda k: k.encode())
        return "{\n" + ",\n".join(f"{inner}{_json(k)}: {_json(v[k], indent + 1)}" for k in keys) + f"\n{pad}}}"
    if isinstance(v, (list, tuple, np.ndarray)):
        v = list(v)
        if not v:
            return "[]"
        return "[\n" + ",\n".join(f"{inner}{_json(x, indent + 1)}" for x in v) + f"\n{pad}]"
    if isinstance(v, str):
        from .io import _json_str
        return _json_str(v)
    if v is None:
        return "null"
    if isinstance(v, (bool, np.bool_)):
        return "true" if v else "false"
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    f = float(v)
    if math.isnan(f):
        return "null"
    return repr(f)  # shortest round-trip form, as nlohmann's dump


def write_error_reports_json(reports: Sequence[ErrorReport], hash_: str) -> str:
    rows = [{"method": r.method, "scheme": SamplingScheme(r.scheme).name, "trials": int(r.trials),
             "base_seed": int(r.base_seed), "f_w": r.f_w, "k_tapers": int(r.k_tapers),
             "failed_bands": int(r.failed_bands), "centers": list(map(float, r.centers)),
             "mse_db_mean": [None if math.isnan(x) else float(x) for x in r.mse_db_mean],
             "mse_db_sem": [None if math.isnan(x) else float(x) for x in r.mse_db_sem],
             "flags": [int(x) for x in r.flags]} for r in reports]
    return _json({"config_hash": hash_, "kind": "error_analysis", "reports": rows}) + "\n"


def write_speed_reports_json(reports: Sequence[SpeedReport], hash_: str) -> str:
    rows = [{"method": r.method, "scheme": SamplingScheme(r.scheme).name,
             "spectra_per_second_mean": r.spectra_per_second_mean,
             "spectra_per_second_std": r.spectra_per_second_std, "calls": int(r.calls), "batches": int(r.batches),
             "environment": r.environment, "timestamp": r.timestamp} for r in reports]
    return _json({"config_hash": hash_, "kind": "speed_analysis", "reports": rows}) + "\n"
