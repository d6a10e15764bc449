"""I/O around the MTNUFFT path against the reference's own outputs.

tests/golden/io_golden.json was produced by the reference's src/io.cpp
(tests/golden/make_golden_io.py); both our C++ drop-in (include/nuspectral/io.hpp, driven
through the test adapter tests/io/libiocheck.so) and the Python mirror
(paper_2407_01943_b200.io) must reproduce it byte for byte: the t,x reader's sorting,
duplicate and parse-error contract (incl. line numbers), the FNV-1a config hash, and the
series / spectrum / F-test / manifest writers.  Host code only: runs on CPU.
"""
import json
import math
import os
import subprocess
import sys

import pytest

from paper_2407_01943_b200 import io as pio

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = json.load(open(os.path.join(HERE, "golden", "io_golden.json")))


def _cpp_results():
    lib = os.path.join(HERE, "io", "libiocheck.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", ROOT, "iocheck"], check=True)
    r = subprocess.run([sys.executable, os.path.join(HERE, "io", "run_cpp_io.py")], capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout)


@pytest.fixture(scope="module")
def cpp():
    """Our C++ drop-in's outputs on every golden case (separate process, see run_cpp_io.py)."""
    return _cpp_results()


def _hex(vals):
    return [float.fromhex(v) for v in vals]


def _py_read(text):
    try:
        r = pio.read_time_series_csv(text)
    except pio.ParseError as e:
        return {"status": "parse", "message": str(e), "line": e.line}
    return {"status": "ok", "t": [v.hex() for v in r.times], "x": [v.hex() for v in r.values],
            "was_sorted": r.was_sorted}


@pytest.mark.parametrize("case", sorted(GOLD["read"]))
def test_read_csv_matches_reference(cpp, case):
    g = GOLD["read"][case]
    assert cpp["read"][case] == g["expect"], "C++ drop-in"
    assert _py_read(g["input"]) == g["expect"], "Python mirror"


def test_read_csv_file_and_series(tmp_path):
    p = tmp_path / "s.csv"
    p.write_text(GOLD["read"]["unsorted"]["input"])
    r = pio.read_time_series_csv_file(str(p))
    assert r.was_sorted is False and r.times == sorted(r.times)
    with pytest.raises(pio.NusError, match="cannot open input file"):
        pio.read_time_series_csv_file(str(tmp_path / "missing.csv"))


def test_config_hash(cpp):
    for s, h in GOLD["config_hash"].items():
        assert pio.config_hash(s) == h
        assert cpp["config_hash"][s] == h
    assert pio.library_version() == GOLD["library_version"] == cpp["library_version"]


def test_write_series(cpp):
    g = GOLD["series"]
    t, x = _hex(g["t"]), _hex(g["x"])
    assert pio.write_time_series_csv(t, x, g["hash"]) == g["csv"]
    assert cpp["series"] == g["csv"]


@pytest.mark.parametrize("method", [0, 1])
def test_write_spectrum(cpp, method):
    g = GOLD["spectrum"]
    power, fw = _hex(g["power"]), _hex(g["f_w_used"])
    expect = g["csv"][str(method)]
    assert pio.write_spectrum_csv(g["centers"], power, g["k_used"], fw, g["flags"], pio.METHOD_NAMES[method],
                                  g["hash"]) == expect
    assert cpp["spectrum"][str(method)] == expect


def test_write_ftest(cpp):
    g = GOLD["ftest"]
    amp = [complex(g["amp"][2 * i], g["amp"][2 * i + 1]) for i in range(len(g["f_stat"]))]
    crit = list(zip(g["p_levels"], g["crits"]))
    assert pio.write_ftest_csv(g["centers"], g["f_stat"], amp, g["flags"], tuple(g["dof"]), crit, g["hash"]) \
        == g["csv"]
    assert cpp["ftest"] == g["csv"]


def test_write_manifest(cpp):
    g = GOLD["manifest"]
    fields = [tuple(f) for f in g["fields"]]
    assert pio.write_manifest_json(g["command"], fields, g["hash"]) == g["json"]
    assert pio.write_manifest_json(g["empty"]["command"], [], g["empty"]["hash"]) == g["empty"]["json"]
    assert cpp["manifest"] == g["json"] and cpp["manifest_empty"] == g["empty"]["json"]
    json.loads(g["json"])  # and it is valid JSON


def test_roundtrip_read_write_read():
    """write_time_series_csv -> read_time_series_csv is the identity at 17 significant digits."""
    t = [0.0, 1e-3, 0.1, 1.0 / 3.0, 2.5, 1e6 + 0.125]
    x = [math.pi, -math.e, 1e-300, 0.0, -7.0, 1e300]
    text = pio.write_time_series_csv(t, x, pio.config_hash("roundtrip"))
    r = pio.read_time_series_csv(text)
    assert r.times == t and r.values == x and r.was_sorted
