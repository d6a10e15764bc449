"""TEST INFRASTRUCTURE: drive OUR C++ drop-in I/O (tests/io/libiocheck.so) on every case of
tests/golden/io_golden.json and print the results as JSON.  Runs in its own process without
numpy: in a process where numpy's extension modules were loaded first, the C++ stream code of a
library dlopen()ed afterwards crashes in this image (the reference's own io.cpp as well)."""
import ctypes
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "..", "golden", "io_golden.json")))
L = ctypes.CDLL(os.path.join(HERE, "libiocheck.so"))
_i64, _d = ctypes.c_int64, ctypes.c_double


def dbuf(vals):
    return (ctypes.c_double * max(1, len(vals)))(*vals)


def text(fn, *args):
    out = ctypes.create_string_buffer(1 << 20)
    ln = _i64(0)
    rc = fn(*args, out, _i64(1 << 20), ctypes.byref(ln))
    return out.raw[:ln.value].decode() if rc == 0 else f"<rc={rc}>"


def read(t_in):
    raw = t_in.encode()
    cap = raw.count(b"\n") + 2
    t, x = (ctypes.c_double * cap)(), (ctypes.c_double * cap)()
    n, srt, line = _i64(0), ctypes.c_int32(0), _i64(-1)
    err = ctypes.create_string_buffer(1024)
    rc = L.io_read_csv(ctypes.c_char_p(raw), t, x, _i64(cap), ctypes.byref(n), ctypes.byref(srt), err, _i64(1024),
                       ctypes.byref(line))
    if rc == 0:
        return {"status": "ok", "t": [t[i].hex() for i in range(n.value)], "x": [x[i].hex() for i in range(n.value)],
                "was_sorted": bool(srt.value)}
    if rc == 3:
        return {"status": "parse", "message": err.value.decode(), "line": int(line.value)}
    return {"status": "error", "message": err.value.decode()}


def main():
    res = {"read": {k: read(v["input"]) for k, v in GOLD["read"].items()}, "config_hash": {}}
    for s in GOLD["config_hash"]:
        out = ctypes.create_string_buffer(64)
        L.io_config_hash(ctypes.c_char_p(s.encode()), out, _i64(64))
        res["config_hash"][s] = out.value.decode()
    out = ctypes.create_string_buffer(64)
    L.io_library_version(out, _i64(64))
    res["library_version"] = out.value.decode()
    g = GOLD["series"]
    t, x = [float.fromhex(v) for v in g["t"]], [float.fromhex(v) for v in g["x"]]
    res["series"] = text(L.io_write_series_csv, dbuf(t), dbuf(x), _i64(len(t)), ctypes.c_char_p(g["hash"].encode()))
    g = GOLD["spectrum"]
    power, fw = [float.fromhex(v) for v in g["power"]], [float.fromhex(v) for v in g["f_w_used"]]
    n = len(power)
    res["spectrum"] = {str(m): text(L.io_write_spectrum_csv, dbuf(g["centers"]), _i64(n), _d(g["f_w"]),
                                    _d(g["f_max"]), _d(g["margin"]), dbuf(power), (ctypes.c_int64 * n)(*g["k_used"]),
                                    dbuf(fw), (ctypes.c_uint8 * n)(*g["flags"]), ctypes.c_int32(m),
                                    ctypes.c_char_p(g["hash"].encode())) for m in (0, 1)}
    g = GOLD["ftest"]
    n = len(g["f_stat"])
    res["ftest"] = text(L.io_write_ftest_csv, dbuf(g["centers"]), _i64(n), _d(0.25), _d(10.0), _d(0.5),
                        dbuf(g["f_stat"]), dbuf(g["amp"]), (ctypes.c_uint8 * n)(*g["flags"]), _i64(g["dof"][0]),
                        _i64(g["dof"][1]), dbuf(g["p_levels"]), dbuf(g["crits"]), _i64(len(g["crits"])),
                        _d(g["cap"]), ctypes.c_char_p(g["hash"].encode()))
    g = GOLD["manifest"]
    fields = [tuple(f) for f in g["fields"]]
    keys = (ctypes.c_char_p * len(fields))(*[k.encode() for k, _ in fields])
    vals = (ctypes.c_char_p * len(fields))(*[v.encode() for _, v in fields])
    res["manifest"] = text(L.io_write_manifest, ctypes.c_char_p(g["command"].encode()), keys, vals,
                           _i64(len(fields)), ctypes.c_char_p(g["hash"].encode()))
    res["manifest_empty"] = text(L.io_write_manifest, ctypes.c_char_p(g["empty"]["command"].encode()), keys, vals,
                                 _i64(0), ctypes.c_char_p(g["empty"]["hash"].encode()))
    json.dump(res, sys.stdout)


if __name__ == "__main__":
    main()
