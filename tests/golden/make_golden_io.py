"""Golden fixtures for the I/O around the MTNUFFT path, from the REFERENCE.

Runs the reference's own src/io.cpp (compiled unmodified into oracle/_ref/libnusref.so,
adapter oracle/ref_io_shim.cpp) on crafted inputs and records its exact outputs in
tests/golden/io_golden.json:
  read_time_series_csv  io.cpp:37-101   header / comment / whitespace rules, strtod parsing with
                                        full consumption, finiteness, stable sort, duplicates
  config_hash           io.cpp:109-118  FNV-1a 64, 16 hex digits
  write_time_series_csv io.cpp:120-130  %.17g, nan
  write_spectrum_csv    io.cpp:132-156  power_db = 10 log10 P (-inf at 0, nan), k_used, flags
  write_ftest_csv       io.cpp:158-188  dof / critical-value header, exceeds_p columns
  write_manifest_json   io.cpp:265-274  nlohmann dump(2): sorted keys, JSON escaping

Deliberately standalone (ctypes + json, NO numpy): the reference's iostream code crashes in a
process that has imported numpy (a runtime-library interaction of the numpy wheel), so this
generator must not share a process with the oracle package.

Run in the build container: python tests/golden/make_golden_io.py
"""
import ctypes
import json
import math
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(ROOT, "oracle", "_ref", "libnusref.so")

_i64 = ctypes.c_int64
_d = ctypes.c_double


def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    L = ctypes.CDLL(LIB)
    return L


L = lib()


def dbuf(vals):
    return (ctypes.c_double * max(1, len(vals)))(*vals)


def read_csv(text):
    raw = text.encode()
    cap = raw.count(b"\n") + 2
    t, x = (ctypes.c_double * cap)(), (ctypes.c_double * cap)()
    n, srt, line = _i64(0), ctypes.c_int32(0), _i64(-1)
    err = ctypes.create_string_buffer(1024)
    rc = L.ref_io_read_csv(ctypes.c_char_p(raw), t, x, _i64(cap), ctypes.byref(n), ctypes.byref(srt), err,
                           _i64(1024), ctypes.byref(line))
    if rc == 0:
        return {"status": "ok", "t": [t[i].hex() for i in range(n.value)], "x": [x[i].hex() for i in range(n.value)],
                "was_sorted": bool(srt.value)}
    if rc == 3:
        return {"status": "parse", "message": err.value.decode(), "line": int(line.value)}
    return {"status": "error", "message": err.value.decode()}


def text_call(fn, *args):
    cap = 1 << 20
    out = ctypes.create_string_buffer(cap)
    ln = _i64(0)
    rc = fn(*args, out, _i64(cap), ctypes.byref(ln))
    assert rc == 0, rc
    return out.raw[:ln.value].decode()


def config_hash(s):
    out = ctypes.create_string_buffer(64)
    assert L.ref_io_config_hash(ctypes.c_char_p(s.encode()), out, _i64(64)) == 0
    return out.value.decode()


def main():
    csv_cases = {
        "sorted": "t,x\n0,1\n1,2\n2.5,-3\n",
        "unsorted": "t,x\n2,1\n0.5,2\n1,0.25\n-1,7\n",
        "comments_blank_ws": "# leading comment\n\n  t , x  \n# mid\n 1 , 2 \n\t2\t,\t3\t\n\n3,4\n",
        "crlf": "t,x\r\n0,1\r\n1,2\r\n",
        "tab_header": "t\t,\tx\n0,1\n1,2\n",
        "bad_header": "time,x\n0,1\n",
        "no_header": "# only a comment\n\n",
        "empty": "",
        "no_comma": "t,x\n0 1\n",
        "extra_field": "t,x\n0,1,2\n",
        "inf_value": "t,x\n0,inf\n1,2\n",
        "nan_time": "t,x\nnan,1\n1,2\n",
        "hex_float": "t,x\n0x1p-2,3\n0x1.8p1,-0x1p0\n",
        "exp_forms": "t,x\n1e3,2E-2\n+1.5,-.5\n5.,1\n",
        "underflow": "t,x\n1,1e-400\n2,3\n",
        "denormal": "t,x\n1,4e-320\n2,3\n",
        "overflow": "t,x\n1,1e400\n2,3\n",
        "duplicates": "t,x\n1,2\n0,1\n1,3\n",
        "one_sample": "t,x\n1,2\n",
        "underscore": "t,x\n1_0,2\n3,4\n",
        "inner_space": "t,x\n1 2,3\n4,5\n",
        "empty_field": "t,x\n,3\n4,5\n",
        "negative_times": "t,x\n-3,1\n-1,2\n-2,3\n",
        "many_decimals": "t,x\n0.1000000000000000055511151231257827,1\n0.2,2\n",
        "leading_zeros_plus": "t,x\n007,+08\n9,-0\n",
        "exact_subnormal_hex": "t,x\n1,0x1p-1074\n2,3\n",
        "zero_big_exponent": "t,x\n1,0e999\n2,0x0p99\n",
        "below_dbl_min": "t,x\n1,2.2250738585072011e-308\n2,3\n",
        "dbl_min": "t,x\n1,2.2250738585072014e-308\n2,3\n",
        "hex_no_exponent": "t,x\n0x10,1\n0x1.8,2\n",
        "infinity_word": "t,x\n1,Infinity\n2,3\n",
        "no_trailing_newline": "t,x\n1,2\n3,4",
        "cr_only_row": "t,x\n1,2\r\n\r\n3,4\r\n",
    }
    reads = {k: {"input": v, "expect": read_csv(v)} for k, v in csv_cases.items()}

    hashes = {s: config_hash(s) for s in ["", "a", "abc", "method=mtnufft;k=7;eps=1e-9", "é ü 中", "x" * 1000]}

    version = ctypes.create_string_buffer(64)
    assert L.ref_io_library_version(version, _i64(64)) == 0

    t = [-2.5, 1e-300, 0.1, 0.2, 3.0, 12345678.9]  # a valid SignalSeries: increasing, finite
    x = [1.0, -0.0, 1e300, 5e-324, 2.0 / 3.0, -7.25]
    series_csv = text_call(L.ref_io_write_series_csv, dbuf(t), dbuf(x), _i64(len(t)), ctypes.c_char_p(b"0123abcd"))

    centers = [1.0, 2.0, 3.0, 4.5, 6.0]
    power = [1.5, 0.0, math.nan, 1e-300, 123456.789]
    k_used = (ctypes.c_int64 * 5)(7, 7, 0, 7, 3)
    fw_used = [0.25, 0.25, math.nan, 0.25, 0.125]
    flags = (ctypes.c_uint8 * 5)(1, 0, 2, 0, 1)
    spectra = {}
    for method in (0, 1):
        spectra[str(method)] = text_call(L.ref_io_write_spectrum_csv, dbuf(centers), _i64(5), _d(0.25), _d(10.0),
                                         _d(0.5), dbuf(power), k_used, dbuf(fw_used), flags,
                                         ctypes.c_int32(method), ctypes.c_char_p(b"feedbeef"))

    f_stat = [3.0, 0.5, 1e12, 7.25]
    amp = [1.0, 2.0, 0.0, -1.0, 1e-5, 3.0, -2.0, 0.5]
    fflags = (ctypes.c_uint8 * 4)(0, 2, 2, 1)
    p_levels = [0.05, 0.01, 0.000244140625]
    crits = [3.8852938346523933, 6.9266081401913, 20.5]
    ftest = text_call(L.ref_io_write_ftest_csv, dbuf(centers[:4]), _i64(4), _d(0.25), _d(10.0), _d(0.5),
                      dbuf(f_stat), dbuf(amp), fflags, _i64(2), _i64(12), dbuf(p_levels), dbuf(crits),
                      _i64(3), _d(1e12), ctypes.c_char_p(b"h"))

    fields = [("k_tapers", "7"), ("epsilon", "1e-09"), ("note", 'quote " backslash \\ tab \t nl \n end'),
              ("unicode", "é中"), ("ctrl", "\x01\x1f"), ("k_tapers", "8"), ("Zeta", "upper")]
    keys = (ctypes.c_char_p * len(fields))(*[k.encode() for k, _ in fields])
    vals = (ctypes.c_char_p * len(fields))(*[v.encode() for _, v in fields])
    manifest = text_call(L.ref_io_write_manifest, ctypes.c_char_p(b"estimate"), keys, vals, _i64(len(fields)),
                         ctypes.c_char_p(b"abcdef0123456789"))
    manifest_empty = text_call(L.ref_io_write_manifest, ctypes.c_char_p(b"bench"), keys, vals, _i64(0),
                               ctypes.c_char_p(b"0"))

    out = {
        "read": reads,
        "config_hash": hashes,
        "library_version": version.value.decode(),
        "series": {"t": [v.hex() for v in t], "x": [v.hex() for v in x], "hash": "0123abcd", "csv": series_csv},
        "spectrum": {"centers": centers, "f_w": 0.25, "f_max": 10.0, "margin": 0.5,
                     "power": [v.hex() for v in power], "k_used": list(k_used), "f_w_used": [v.hex() for v in fw_used],
                     "flags": list(flags), "hash": "feedbeef", "csv": spectra},
        "ftest": {"centers": centers[:4], "f_stat": f_stat, "amp": amp, "flags": list(fflags), "dof": [2, 12],
                  "p_levels": p_levels, "crits": crits, "cap": 1e12, "hash": "h", "csv": ftest},
        "manifest": {"command": "estimate", "fields": fields, "hash": "abcdef0123456789", "json": manifest,
                     "empty": {"command": "bench", "hash": "0", "json": manifest_empty}},
    }
    path = os.path.join(HERE, "io_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, ensure_ascii=False)
    print(f"wrote {path}")


if __name__ == "__main__":
    sys.exit(main())
