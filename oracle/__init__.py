"""TEST INFRASTRUCTURE ONLY — ctypes bindings to the two CPU oracles.

* ``C`` — ``liboracle.so``: the plain-C restatement of the reference MTNUFFT
  path (``oracle/nus_oracle.c``; each function cites the reference file:line).
* ``REF`` — ``_ref/libnusref.so``: the unmodified reference library compiled
  from /root/reference/proj/src plus the ``ref_shim.cpp`` adapter.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The product (``paper_2407_01943_b200``) never
does: it runs on the GPU or fails loudly.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_TREE = "/root/reference/proj"

_c = None
_ref = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64
_d = ctypes.c_double
_i = ctypes.c_int


def build(ref: bool = True) -> None:
    """Compile the restatement (and, where the reference tree exists, the reference)."""
    targets = ["oracle"]
    if ref and os.path.isdir(REF_TREE):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _p(a):
    return a.ctypes.data_as(_dp)


def _arr(x, dtype=np.float64):
    return np.ascontiguousarray(x, dtype=dtype)


def lib_c():
    global _c
    if _c is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build(ref=False)
        _c = ctypes.CDLL(path)
        L = _c
        L.or_spread_width.restype = _i64
        L.or_next_pow2.restype = _i64
        L.or_centers_uniform.restype = _i
        L.or_select_path.restype = _i
        for name in ("or_eigencoefficients", "or_mtnufft_power", "or_dpss", "or_tridiag_top",
                     "or_spline", "or_gpss_interpolated"):
            getattr(L, name).restype = _i
    return _c


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libnusref.so"))


def lib_ref():
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libnusref.so")
        if not os.path.exists(path):
            if os.path.isdir(REF_TREE):
                build(ref=True)
            else:
                raise FileNotFoundError("oracle/_ref/libnusref.so not built and no reference tree")
        _ref = ctypes.CDLL(path)
        _ref.ref_last_error.restype = ctypes.c_char_p
        _ref.ref_injected_create.restype = ctypes.c_void_p
        _ref.ref_injected_create.argtypes = [_dp, _i64, _dp, _i64, _dp, _i64, _d, _i, _d, _d]
        _ref.ref_injected_destroy.argtypes = [ctypes.c_void_p]
        _ref.ref_injected_power.argtypes = [ctypes.c_void_p, _dp, _dp]
        _ref.ref_injected_power_many.argtypes = [ctypes.c_void_p, _dp, _i64, _i, _dp]
        _ref.ref_injected_power_tapers.argtypes = [ctypes.c_void_p, _dp, _i, _dp]
        _ref.ref_injected_taper_powers.argtypes = [ctypes.c_void_p, _dp, _i, _dp]
        _ref.ref_default_taper_count.restype = _i64
        _ref.ref_default_taper_count.argtypes = [_d]
    return _ref


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_REF_KIND = {1: "invalid_argument", 2: "PlanMismatch", 3: "BandRangeError",
             4: "ExtrapolationError", 5: "Error", 9: "other"}


def _chk(rc):
    if rc != 0:
        raise RefError(_REF_KIND.get(rc, rc), lib_ref().ref_last_error().decode())


# ---------------------------------------------------------------- restatement

class C:
    """Plain-C restatement (oracle/nus_oracle.c)."""

    @staticmethod
    def spread_width(eps):
        return lib_c().or_spread_width(_d(eps))

    @staticmethod
    def centers_uniform(c):
        c = _arr(c)
        return bool(lib_c().or_centers_uniform(_p(c), _i64(c.size)))

    @staticmethod
    def select_path(n, c, policy=0):
        c = _arr(c)
        return lib_c().or_select_path(_i64(n), _p(c), _i64(c.size), _i(policy))

    @staticmethod
    def plan_params(c, eps, oversampling=2):
        class P(ctypes.Structure):
            _fields_ = [("n_centers", _i64), ("spread_width", _i64), ("mr", _i64),
                        ("mode_offset", _i64), ("f0", _d), ("df", _d), ("tau", _d), ("fshift", _d)]
        c = _arr(c)
        p = P()
        lib_c().or_plan_params(_p(c), _i64(c.size), _d(eps), _i(oversampling), ctypes.byref(p))
        return {k: getattr(p, k) for k, _ in P._fields_}, p

    @staticmethod
    def first_cells(t, c, eps, oversampling=2):
        t = _arr(t)
        _, p = C.plan_params(c, eps, oversampling)
        out = np.empty(t.size, np.int64)
        lib_c().or_first_cells(_p(t), _i64(t.size), ctypes.byref(p), out.ctypes.data_as(_i64p))
        return out

    @staticmethod
    def nufft_fast(t, c, eps, y, oversampling=2):
        t, c = _arr(t), _arr(c)
        y = _arr(np.asarray(y, np.complex128).view(np.float64))
        out = np.empty(2 * c.size)
        lib_c().or_nufft_fast(_p(t), _i64(t.size), _p(c), _i64(c.size), _d(eps), _i(oversampling),
                              _p(y), _p(out))
        return out.view(np.complex128)

    @staticmethod
    def ndft_direct(t, y, c):
        t, c = _arr(t), _arr(c)
        y = _arr(np.asarray(y, np.complex128).view(np.float64))
        out = np.empty(2 * c.size)
        lib_c().or_ndft_direct(_p(t), _i64(t.size), _p(y), _p(c), _i64(c.size), _p(out))
        return out.view(np.complex128)

    @staticmethod
    def fft(z, inverse=False):
        z = _arr(np.asarray(z, np.complex128).view(np.float64)).copy()
        lib_c().or_fft(_p(z), _i64(z.size // 2), _i(int(inverse)))
        return z.view(np.complex128)

    @staticmethod
    def eigencoefficients(t, w, x, c, eps, policy=0):
        t, w, x, c = _arr(t), _arr(w), _arr(x), _arr(c)
        k = w.shape[0]
        out = np.empty(2 * k * c.size)
        rc = lib_c().or_eigencoefficients(_p(t), _i64(t.size), _p(w), _i64(k), _p(x), _p(c),
                                          _i64(c.size), _d(eps), _i(policy), _p(out))
        if rc:
            raise ValueError("fast path requires uniformly spaced centers")
        return out.view(np.complex128).reshape(k, c.size)

    @staticmethod
    def mtnufft_power(t, w, x, c, eps, policy=0):
        t, w, x, c = _arr(t), _arr(w), _arr(x), _arr(c)
        out = np.empty(c.size)
        rc = lib_c().or_mtnufft_power(_p(t), _i64(t.size), _p(w), _i64(w.shape[0]), _p(x), _p(c),
                                      _i64(c.size), _d(eps), _i(policy), _p(out))
        if rc:
            raise ValueError("fast path requires uniformly spaced centers")
        return out

    @staticmethod
    def dpss(n, tw, k, threads=8):
        tap = np.empty((k, n))
        ev = np.empty(k)
        rc = lib_c().or_dpss(_i64(n), _d(tw), _i64(k), _p(tap), _p(ev), _i(threads))
        if rc:
            raise ValueError("dpss: invalid arguments")
        return tap, ev

    @staticmethod
    def tridiag_top(d, e, k, threads=8):
        d, e = _arr(d), _arr(e)
        vals = np.empty(k)
        vecs = np.empty((k, d.size))
        rc = lib_c().or_tridiag_top(_p(d), _p(e), _i64(d.size), _i64(k), _p(vals), _p(vecs),
                                    _i(threads))
        if rc:
            raise ValueError("tridiag_top: invalid arguments")
        return vals, vecs

    @staticmethod
    def spline(xk, yk, xq):
        xk, yk, xq = _arr(xk), _arr(yk), _arr(xq)
        out = np.empty(xq.size)
        rc = lib_c().or_spline(_p(xk), _p(yk), _i64(xk.size), _p(xq), _i64(xq.size), _p(out))
        if rc == 2:
            raise ValueError("extrapolation")
        if rc:
            raise ValueError("spline: invalid arguments")
        return out

    @staticmethod
    def quadform(t, f_max, w, threads=8):
        t, w = _arr(t), _arr(np.atleast_2d(w))
        q = np.empty(w.shape[0])
        lib_c().or_signal_band_quadform(_p(t), _i64(t.size), _d(f_max), _p(w), _i64(w.shape[0]),
                                        _p(q), _i(threads))
        return q

    @staticmethod
    def gpss_interpolated(t, f_max, f_w, k, threads=8):
        t = _arr(t)
        w = np.empty((k, t.size))
        q = np.empty(k)
        rc = lib_c().or_gpss_interpolated(_p(t), _i64(t.size), _d(f_max), _d(f_w), _i64(k),
                                          _p(w), _p(q), _i(threads))
        if rc:
            raise ValueError(f"gpss_interpolated failed ({rc})")
        return w, q


# ------------------------------------------------------------------ reference

class REF:
    """The reference library itself (oracle/_ref/libnusref.so)."""

    @staticmethod
    def plan_info(t, c, eps, policy=0, oversampling=2):
        t, c = _arr(t), _arr(c)
        info = np.zeros(4, np.int64)
        tau = _d(0)
        _chk(lib_ref().ref_plan_info(_p(t), _i64(t.size), _p(c), _i64(c.size), _d(eps), _i(policy),
                                     _i(oversampling), info.ctypes.data_as(_i64p), ctypes.byref(tau)))
        return {"path": "fast" if info[0] else "direct", "spread_width": int(info[1]),
                "centers_uniform": bool(info[2]), "mr": int(info[3]), "tau": tau.value}

    @staticmethod
    def first_cells(t, c, eps, oversampling=2):
        t, c = _arr(t), _arr(c)
        out = np.empty(t.size, np.int64)
        _chk(lib_ref().ref_plan_first_cells(_p(t), _i64(t.size), _p(c), _i64(c.size), _d(eps),
                                            _i(oversampling), out.ctypes.data_as(_i64p)))
        return out

    @staticmethod
    def plan_execute(t, c, eps, y, policy=0, oversampling=2):
        t, c = _arr(t), _arr(c)
        y = _arr(np.asarray(y, np.complex128).view(np.float64))
        out = np.empty(2 * c.size)
        _chk(lib_ref().ref_plan_execute(_p(t), _i64(t.size), _p(c), _i64(c.size), _d(eps),
                                        _i(policy), _i(oversampling), _p(y), _i64(y.size // 2),
                                        _p(out)))
        return out.view(np.complex128)

    @staticmethod
    def ndft_direct(t, y, c):
        t, c = _arr(t), _arr(c)
        y = _arr(np.asarray(y, np.complex128).view(np.float64))
        out = np.empty(2 * c.size)
        _chk(lib_ref().ref_ndft_direct(_p(t), _i64(t.size), _p(y), _i64(y.size // 2), _p(c),
                                       _i64(c.size), _p(out)))
        return out.view(np.complex128)

    @staticmethod
    def fft(z, inverse=False):
        z = _arr(np.asarray(z, np.complex128).view(np.float64)).copy()
        _chk(lib_ref().ref_fft_forward(_p(z), _i64(z.size // 2), _i(int(inverse))))
        return z.view(np.complex128)

    @staticmethod
    def dpss(n, tw, k):
        tap = np.empty((k, n))
        conc = np.empty(k)
        _chk(lib_ref().ref_dpss(_i64(n), _d(tw), _i64(k), _p(tap), _p(conc)))
        return tap, conc

    @staticmethod
    def tridiagonal_eigen(d, e, k):
        d, e = _arr(d), _arr(e)
        vals, res = np.empty(k), np.empty(k)
        vecs = np.empty((k, d.size))
        _chk(lib_ref().ref_tridiagonal_eigen(_p(d), _p(e), _i64(d.size), _i64(e.size), _i64(k),
                                             _p(vals), _p(vecs), _p(res)))
        return vals, vecs, res

    @staticmethod
    def spline(xk, yk, xq):
        xk, yk, xq = _arr(xk), _arr(yk), _arr(np.atleast_1d(xq))
        out = np.empty(xq.size)
        _chk(lib_ref().ref_spline(_p(xk), _p(yk), _i64(xk.size), _p(xq), _i64(xq.size), _p(out)))
        return out

    @staticmethod
    def quadform(t, f_max, w):
        t, w = _arr(t), _arr(np.atleast_2d(w))
        q = np.empty(w.shape[0])
        _chk(lib_ref().ref_signal_band_quadform(_p(t), _i64(t.size), _d(f_max), _p(w),
                                                _i64(w.shape[0]), _p(q)))
        return q

    @staticmethod
    def gpss_interpolated(t, f_max, f_w, k):
        t = _arr(t)
        w = np.empty((k, t.size))
        _chk(lib_ref().ref_gpss_interpolated(_p(t), _i64(t.size), _d(f_max), _d(f_w), _i64(k),
                                             _p(w)))
        return w

    @staticmethod
    def eigencoefficients(t, w, x, c, eps, f_max, f_w, policy=0):
        t, w, x, c = _arr(t), _arr(np.atleast_2d(w)), _arr(x), _arr(c)
        k = w.shape[0]
        out = np.empty(2 * k * c.size)
        _chk(lib_ref().ref_eigencoefficients(_p(t), _i64(t.size), _p(w), _i64(k), _p(x), _p(c),
                                             _i64(c.size), _d(eps), _i(policy), _d(f_max), _d(f_w),
                                             _p(out)))
        return out.view(np.complex128).reshape(k, c.size)

    @staticmethod
    def mtnufft(t, x, f_max, c, f_w, k, eps, margin=None, policy=0):
        """Oracle-A: the full reference MtnufftEstimator (setup + estimate)."""
        t, x, c = _arr(t), _arr(x), _arr(c)
        p = np.empty(c.size)
        w = np.empty((k, t.size))
        flags = np.empty(c.size, np.uint8)
        margin = 2.0 * f_w if margin is None else margin
        _chk(lib_ref().ref_mtnufft(_p(t), _i64(t.size), _p(x), _d(f_max), _p(c), _i64(c.size),
                                   _d(f_w), _d(margin), _i64(k), _d(eps), _i(policy), _p(p), _p(w),
                                   flags.ctypes.data_as(_u8p)))
        return p, w, flags

    @staticmethod
    def f_test(t, w, x, c, eps, f_max, f_w, margin=None, cap=1e12, policy=0):
        """Reference eigencoefficients + f_test (inference.cpp:132-186)."""
        t, w, x, c = _arr(t), _arr(np.atleast_2d(w)), _arr(x), _arr(c)
        f = np.empty(c.size)
        amp = np.empty(2 * c.size)
        flags = np.empty(c.size, np.uint8)
        crit = np.zeros(3)
        margin = 2.0 * f_w if margin is None else margin
        _chk(lib_ref().ref_f_test(_p(t), _i64(t.size), _p(w), _i64(w.shape[0]), _p(x), _p(c),
                                  _i64(c.size), _d(eps), _i(policy), _d(f_max), _d(f_w), _d(margin),
                                  _d(cap), _p(f), _p(amp), flags.ctypes.data_as(_u8p), _p(crit)))
        return f, amp.view(np.complex128), flags, crit

    @staticmethod
    def f_quantile(p, d1, d2):
        out = _d(0)
        _chk(lib_ref().ref_f_quantile(_d(p), _i64(d1), _i64(d2), ctypes.byref(out)))
        return out.value

    # ---- MTNUFFT0 -------------------------------------------------------

    @staticmethod
    def generalized_eigen(a, m, k, ridge_first=1e-12, ridge_retry=1e-9, vectors=True):
        a = np.asarray(a)
        n = a.shape[0]
        are = _arr(np.real(a))
        aim = _arr(np.imag(a)) if np.iscomplexobj(a) else None
        mm = _arr(m)
        vals = np.empty(k)
        vec = np.empty((k, n, 2)) if vectors else None
        res = np.empty(k)
        _chk(lib_ref().ref_generalized_eigen(_p(are), _p(aim) if aim is not None else None, _p(mm), _i64(n),
                                             _i64(k), _d(ridge_first), _d(ridge_retry), _p(vals),
                                             _p(vec) if vectors else None, _p(res)))
        return vals, (vec[..., 0] + 1j * vec[..., 1]) if vectors else None, res

    @staticmethod
    def gpss_exact(t, f_max, f_c, f_w, k):
        t = _arr(t)
        w = np.empty((k, t.size, 2))
        conc = np.empty(k)
        _chk(lib_ref().ref_gpss_exact(_p(t), _i64(t.size), _d(f_max), _d(f_c), _d(f_w), _i64(k), _p(w),
                                      _p(conc)))
        return w[..., 0] + 1j * w[..., 1], conc

    @staticmethod
    def mtnufft0(t, x, f_max, c, f_w, k, eps, margin=None):
        t, x, c = _arr(t), _arr(x), _arr(c)
        p = np.empty(c.size)
        w = np.empty((k, t.size))
        method = ctypes.c_int32(-1)
        _chk(lib_ref().ref_mtnufft0(_p(t), _i64(t.size), _p(x), _d(f_max), _p(c), _i64(c.size), _d(f_w),
                                    _d(2.0 * f_w if margin is None else margin), _i64(k), _d(eps), _p(p), _p(w),
                                    ctypes.byref(method)))
        return p, w, method.value

    @staticmethod
    def run_error_analysis(methods, schemes, trials, base_seed, f_max=0.5, f_w=0.05, k=4, spacing=0.01,
                           n_samples=50, eps=1e-8):
        """bench.cpp:130-204 -> list of dicts (scheme-major, method-minor)."""
        ms = np.ascontiguousarray(methods, np.int32)
        ss = np.ascontiguousarray(schemes, np.int32)
        cap = int(round(f_max / spacing)) + 8
        nrep = ms.size * ss.size
        cen, mean, sem = np.empty((nrep, cap)), np.empty((nrep, cap)), np.empty((nrep, cap))
        fl = np.empty((nrep, cap), np.uint8)
        bands, failed = _i64(0), np.empty(nrep, np.int64)
        _chk(lib_ref().ref_run_error_analysis(
            ms.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _i64(ms.size),
            ss.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _i64(ss.size), _i64(trials),
            ctypes.c_uint64(base_seed), _d(f_max), _d(f_w), _i64(k), _d(spacing), _i64(n_samples), _d(eps),
            _i64(cap), _p(cen), _p(mean), _p(sem), fl.ctypes.data_as(_u8p), ctypes.byref(bands),
            failed.ctypes.data_as(_i64p)))
        b = bands.value
        return [{"centers": cen[r, :b].copy(), "mean": mean[r, :b].copy(), "sem": sem[r, :b].copy(),
                 "flags": fl[r, :b].copy(), "failed": int(failed[r])} for r in range(nrep)]

    @staticmethod
    def default_taper_count(tw):
        return int(lib_ref().ref_default_taper_count(tw))

    @staticmethod
    def rng_gauss(seed, count):
        out = np.empty(count)
        _chk(lib_ref().ref_rng_gauss(ctypes.c_uint64(seed), _i64(count), _p(out)))
        return out

    @staticmethod
    def rng_uniform(seed, count):
        out = np.empty(count)
        _chk(lib_ref().ref_rng_uniform(ctypes.c_uint64(seed), _i64(count), _p(out)))
        return out

    @staticmethod
    def generate_grid(scheme, n, seed=0, jitter_sigma=-1.0):
        """scheme: 0 uniform, 1 jitter, 2 missing, 3 arithmetic (simkit.cpp:77-141)."""
        out = np.empty(n + 64)
        cnt = _i64(0)
        _chk(lib_ref().ref_generate_grid(_i(scheme), _i64(n), ctypes.c_uint64(seed),
                                         _d(jitter_sigma), _p(out), ctypes.byref(cnt)))
        return out[: cnt.value].copy()

    @staticmethod
    def line_plus_noise(t, freq, amp, phase, noise_var, seed):
        t = _arr(t)
        out = np.empty(t.size)
        _chk(lib_ref().ref_line_plus_noise(_p(t), _i64(t.size), _d(freq), _d(amp), _d(phase),
                                           _d(noise_var), ctypes.c_uint64(seed), _p(out)))
        return out


class Injected:
    """Oracle-B handle: the reference NufftPlan + eigencoefficients + power loop
    with injected taper weights (one taper at a time)."""

    def __init__(self, t, w, c, eps, f_max, f_w, policy=1):
        t, w, c = _arr(t), _arr(np.atleast_2d(w)), _arr(c)
        self.n, self.nc, self.k = t.size, c.size, w.shape[0]
        self.h = lib_ref().ref_injected_create(_p(t), _i64(t.size), _p(w), _i64(w.shape[0]), _p(c),
                                               _i64(c.size), _d(eps), _i(policy), _d(f_max), _d(f_w))
        if not self.h:
            raise RefError("create", lib_ref().ref_last_error().decode())

    def power(self, x):
        x = _arr(x)
        out = np.empty(self.nc)
        _chk(lib_ref().ref_injected_power(self.h, _p(x), _p(out)))
        return out

    def power_tapers(self, x, threads):
        """One series, the K tapers on `threads` host threads; bit-identical to power()."""
        x = _arr(x)
        out = np.empty(self.nc)
        _chk(lib_ref().ref_injected_power_tapers(self.h, _p(x), _i(threads), _p(out)))
        return out

    def taper_powers(self, x, threads):
        """|J_k(i)|^2 of every injected taper [K][I] (tapers on `threads` host threads)."""
        x = _arr(x)
        out = np.empty((self.k, self.nc))
        _chk(lib_ref().ref_injected_taper_powers(self.h, _p(x), _i(threads), _p(out)))
        return out

    def power_many(self, xs, threads):
        xs = _arr(xs)
        out = np.empty((xs.shape[0], self.nc))
        _chk(lib_ref().ref_injected_power_many(self.h, _p(xs), _i64(xs.shape[0]), _i(threads),
                                               _p(out)))
        return out

    def close(self):
        if self.h:
            lib_ref().ref_injected_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
