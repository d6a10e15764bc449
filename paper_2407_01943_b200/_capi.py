"""ctypes binding of include/nus_c.h (libnus_b200.so).

The product path is the CUDA library: if the shared object is missing this
module raises immediately, and every compute call fails with NoDeviceError
when no sm_100 GPU is visible.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libnus_b200.so")

NUS_OK = 0
AUTO_SELECT, FORCE_FAST, FORCE_DIRECT = 0, 1, 2
PATH_DIRECT, PATH_FAST = 0, 1
F64, F32 = 0, 1


class NusError(RuntimeError):
    """Base class; mirrors nuspectral::Error (errors.hpp:9-15)."""


class InvalidArgument(NusError, ValueError):
    """std::invalid_argument in the reference."""


class PlanMismatch(NusError):
    """nuspectral::PlanMismatch (errors.hpp:30-34)."""


class BandRangeError(NusError):
    """nuspectral::BandRangeError (errors.hpp:42-46)."""


class ExtrapolationError(NusError):
    """nuspectral::ExtrapolationError (errors.hpp:24-28)."""


class NumericError(NusError):
    """nuspectral::Error raised for numeric failure."""


class DegenerateTapers(NusError):
    """nuspectral::DegenerateTapers (errors.hpp:36-40)."""


class ConditioningError(NumericError):
    """errors.hpp ConditioningError: metric not positive definite after the ridge retries."""


class SpectralRangeError(NumericError):
    """errors.hpp SpectralRangeError: generalized eigenvalue outside [0, 1] beyond 1e-6."""


class CudaError(NusError):
    pass


class OutOfMemory(CudaError, MemoryError):
    pass


class NoDeviceError(CudaError):
    pass


_ERRORS = {1: InvalidArgument, 2: PlanMismatch, 3: BandRangeError, 4: ExtrapolationError,
           5: NumericError, 6: CudaError, 7: OutOfMemory, 8: NoDeviceError, 9: DegenerateTapers, 10: ConditioningError, 11: SpectralRangeError}

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_d = ctypes.c_double
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)


class PlanInfo(ctypes.Structure):
    _fields_ = [("n_samples", _i64), ("n_centers", _i64), ("epsilon", _d), ("oversampling", _i32),
                ("path", _i32), ("centers_uniform", _i32), ("precision", _i32),
                ("spread_width", _i64), ("mr", _i64), ("tau", _d), ("df", _d), ("fshift", _d),
                ("kernel", _i32), ("support", _i32)]


class MtnufftConfig(ctypes.Structure):
    _fields_ = [("channels", _i64), ("n", _i64), ("n_centers", _i64), ("k_tapers", _i64),
                ("f_max", _d), ("f_w", _d), ("epsilon", _d), ("policy", _i32), ("precision", _i32),
                ("device", _i32), ("reserved", _i32)]


# name -> argtypes (restype int unless listed in _RESTYPE)
_SIGS = {
    "nus_last_error": [],
    "nus_device_info": [ctypes.c_int, _i32p, _i32p, _i32p, _i64p],
    "nus_kernel_launch_count": [],
    "nus_set_spread_kernel": [_i32],
    "nus_mtnufft_grid_rows": [_vp, _i32p, _i32p, _i32p],
    "nus_mtnufft_spread_slots_device": [_vp, _vp, _i32, _i64, _i64, _vp, _i64, _vp],
    "nus_sum_slots_device": [_vp, _i64, _i64, _i64, _vp, _i32, _vp],
    "nus_ipc_get_handle": [_vp, _vp],
    "nus_ipc_get_handle_offset": [_vp, _vp, _i64p],
    "nus_ipc_open": [_vp, _i32, ctypes.POINTER(_vp)],
    "nus_ipc_close": [_vp],
    "nus_mtnufft_set_grid_rows": [_vp, _i32, _i32],
    "nus_get_spread_kernel": [_i32p],
    "nus_plan_create": [_dp, _i64, _dp, _i64, _d, _i32, _i32, _i32, _i32, ctypes.POINTER(_vp)],
    "nus_plan_destroy": [_vp],
    "nus_plan_info": [_vp, ctypes.POINTER(PlanInfo)],
    "nus_plan_first_cells": [_vp, _i64p],
    "nus_plan_sort_order": [_vp, _i32p],
    "nus_plan_execute": [_vp, _dp, _i64, _dp],
    "nus_plan_execute_device": [_vp, _vp, _i64, _vp, _vp],
    "nus_ndft_direct": [_dp, _i64, _dp, _dp, _i64, _i32, _dp],
    "nus_fft_inplace": [_dp, _i64, _i32, _i32],
    "nus_signal_band_matrix": [_dp, _i64, _d, _i32, _dp],
    "nus_dpss": [_i64, _d, _i64, _i32, _dp, _dp, _dp],
    "nus_tridiagonal_eigen": [_dp, _dp, _i64, _i64, _i32, _dp, _dp, _dp],
    "nus_signal_band_quadform": [_dp, _i64, _d, _dp, _i64, _i64, _i64, _i32, _dp],
    "nus_signal_band_quadform_fast": [_dp, _i64, _d, _dp, _i64, _i32, _dp],
    "nus_taper_spline": [_dp, _i64, _d, _d, _i64, _i32, _dp],
    "nus_gpss_interpolated": [_dp, _i64, _d, _d, _i64, _i32, _dp],
    "nus_mtnufft_create": [ctypes.POINTER(MtnufftConfig), _dp, _dp, _dp, ctypes.POINTER(_vp)],
    "nus_mtnufft_create_channels": [ctypes.POINTER(MtnufftConfig), _dp, _dp, _dp, _dp, ctypes.POINTER(_vp)],
    "nus_mtnufft_multi_create": [ctypes.POINTER(MtnufftConfig), _i32p, _i32, _i32, _dp, _dp, _dp, _dp,
                                 ctypes.POINTER(_vp)],
    "nus_mtnufft_multi_destroy": [_vp],
    "nus_mtnufft_multi_estimate": [_vp, _dp, _dp],
    "nus_mtnufft_multi_tapers": [_vp, _dp],
    "nus_mtnufft_multi_peer_bytes": [_vp, _i64p],
    "nus_mtnufft_destroy": [_vp],
    "nus_mtnufft_plan_info": [_vp, ctypes.POINTER(PlanInfo)],
    "nus_mtnufft_tapers": [_vp, _dp],
    "nus_mtnufft_setup_ms": [_vp, _dp],
    "nus_mtnufft_estimate": [_vp, _dp, _dp],
    "nus_mtnufft_eigencoefficients": [_vp, _dp, _dp],
    "nus_mtnufft_estimate_device": [_vp, _vp, _i32, _vp, _vp, _vp],
    "nus_mtnufft_spread_device": [_vp, _vp, _i32, _i64, _i64, _vp, _i64, _vp],
    "nus_mtnufft_stage_kernels": [_vp, ctypes.c_char_p, _i64],
    "nus_mtnufft_estimate_batch": [_vp, _dp, _i64, _dp],
    "nus_generalized_eigen": [_dp, _dp, _dp, _i64, _i64, _d, _d, _i32, _i32, _dp, _dp, _dp],
    "nus_gpss_exact": [_dp, _i64, _d, _d, _d, _i64, _d, _d, _i32, _dp, _dp],
    "nus_band_matrix": [_dp, _i64, _d, _d, _i32, _dp, _dp],
    "nus_mtnufft_transform_device": [_vp, _vp, _i64, _i64, _d, _i32, _vp, _vp],
    "nus_mtnufft_bytes_model": [_vp, _i32, _dp, _dp, _dp, _dp],
    "nus_f_test": [_dp, _i64, _i64, _dp, _i64, _dp, _d, _d, _i32, _dp, _dp, ctypes.POINTER(ctypes.c_uint8)],
    "nus_mtnufft_f_test": [_vp, _dp, _d, _dp, _dp, ctypes.POINTER(ctypes.c_uint8)],
    "nus_f_quantile": [_d, _i64, _i64, _dp],
    "nus_mtnufft_timing": [_vp, _i64],
    "nus_mtnufft_timing_read": [_vp, _dp, _i64p],
}
_RESTYPE = {"nus_last_error": ctypes.c_char_p, "nus_kernel_launch_count": _i64}

_lib = None


def lib():
    """Load libnus_b200.so (fails loudly when the CUDA extension is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or `make lib`)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != NUS_OK:
        msg = lib().nus_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, NusError)(msg)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def c128_as_f64(a) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64)


def launch_count() -> int:
    return int(lib().nus_kernel_launch_count())


def device_info(device: int = 0) -> dict:
    ma, mi, sm = _i32(), _i32(), _i32()
    mem = _i64()
    check(lib().nus_device_info(device, ctypes.byref(ma), ctypes.byref(mi), ctypes.byref(sm),
                                ctypes.byref(mem)))
    return {"cc": (ma.value, mi.value), "sm_count": sm.value, "total_mem": mem.value}
