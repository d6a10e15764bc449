"""I/O around the MTNUFFT path — Python mirror of include/nuspectral/io.hpp.

Same behaviour as the reference's src/io.cpp (and our C++ drop-in, csrc/host/io.cpp),
byte-exact on tests/golden/io_golden.json:

* ``read_time_series_csv`` (io.cpp:37-101): header ``t,x`` (blanks/tabs ignored), ``#``
  comments and blank lines skipped, every field parsed like ``std::stod`` with full
  consumption (decimal or hex floats; overflow, underflow and non-finite values rejected),
  stable sort by t when unsorted (``was_sorted`` False), duplicate times rejected.
  Errors raise :class:`ParseError` carrying the line number (0 for duplicates).
* ``config_hash`` (io.cpp:109-118): FNV-1a 64-bit, 16 lower-case hex digits.
* ``write_time_series_csv`` / ``write_spectrum_csv`` / ``write_ftest_csv``
  (io.cpp:120-188) and ``write_manifest_json`` (io.cpp:265-274) return the text.
"""
from __future__ import annotations

import math
import re
import sys
from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, List, Sequence, Tuple

from ._capi import NusError

__all__ = ["ParseError", "ReadResult", "read_time_series_csv", "read_time_series_csv_file", "config_hash",
           "write_time_series_csv", "write_spectrum_csv", "write_ftest_csv", "write_manifest_json",
           "library_version", "METHOD_NAMES"]

METHOD_NAMES = ("mtnufft", "mtnufft0", "bg_fixed", "bg_adaptive", "baseline")  # estimators.cpp:46-55
_DBL_MIN = sys.float_info.min

_DEC = re.compile(r"[+-]?(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?\Z")
_HEX = re.compile(r"[+-]?0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?\d+)?\Z")
_NONZERO_MANTISSA = re.compile(r"[1-9a-fA-F]")


class ParseError(NusError):
    """Malformed input with the offending line number (io.hpp:14-24)."""

    def __init__(self, what: str, line: int):
        super().__init__(f"{what} (line {line})")
        self.line = line


@dataclass
class ReadResult:
    times: List[float]
    values: List[float]
    was_sorted: bool

    def series(self):
        """As the product's SignalSeries (validated like the reference's SamplingGrid)."""
        from .api import SamplingGrid, SignalSeries
        return SignalSeries(SamplingGrid(self.times), self.values)


def _stod(s: str) -> float:
    """std::stod + full consumption: None when the reference would throw."""
    if _HEX.match(s):
        body = s.lstrip("+-")
        mant = body[2:].split("p")[0].split("P")[0]
        v = float.fromhex(s)
    elif _DEC.match(s):
        mant = s.lstrip("+-").split("e")[0].split("E")[0]
        v = float(s)
    else:
        return None
    # strtod reports ERANGE on overflow and on inexact underflow (a zero or subnormal result
    # that is not the exact value): std::stod throws out_of_range for both
    if math.isinf(v):
        return None
    if (v == 0.0 and _NONZERO_MANTISSA.search(mant)) or (v != 0.0 and abs(v) < _DBL_MIN):
        if v == 0.0 or Fraction(v) != _exact(s):
            return None
    return v


def _exact(s: str) -> Fraction:
    """The exact rational value of a decimal or hex float literal."""
    sign = -1 if s.startswith("-") else 1
    body = s.lstrip("+-")
    if body[:2].lower() == "0x":
        digits, _, exp = body[2:].lower().partition("p")
        whole, _, frac = digits.partition(".")
        m = int((whole + frac) or "0", 16)
        return sign * Fraction(m) * Fraction(2) ** (int(exp or "0") - 4 * len(frac))
    return sign * Fraction(body)


def read_time_series_csv(text: str) -> ReadResult:
    t: List[float] = []
    x: List[float] = []
    header = False
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # getline: no extra empty line after a trailing newline
    line = 0
    for raw in lines:
        line += 1
        s = raw.strip(" \t\r\n")
        if not s or s[0] == "#":
            continue
        if not header:
            if s.replace(" ", "").replace("\t", "") != "t,x":
                raise ParseError(f"expected header 't,x', got '{s}'", line)
            header = True
            continue
        comma = s.find(",")
        if comma < 0:
            raise ParseError("expected 't,x' row", line)
        tv = _stod(s[:comma].strip(" \t\r\n"))
        xv = _stod(s[comma + 1:].strip(" \t\r\n"))
        if tv is None or xv is None or not math.isfinite(tv) or not math.isfinite(xv):
            raise ParseError(f"could not parse row '{s}'", line)
        t.append(tv)
        x.append(xv)
    if not header:
        raise ParseError("empty input: missing 't,x' header", line)
    if len(t) < 2:
        raise ParseError("need at least 2 samples", line)
    was_sorted = all(t[i - 1] <= t[i] for i in range(1, len(t)))
    if not was_sorted:
        order = sorted(range(len(t)), key=lambda i: t[i])  # stable
        t = [t[i] for i in order]
        x = [x[i] for i in order]
    for i in range(1, len(t)):
        if t[i] == t[i - 1]:
            raise ParseError("duplicate sample time %f" % t[i], 0)
    return ReadResult(t, x, was_sorted)


def read_time_series_csv_file(path: str) -> ReadResult:
    try:
        with open(path, "r", newline="") as f:
            text = f.read()
    except OSError:
        raise NusError(f"cannot open input file: {path}") from None
    return read_time_series_csv(text)


def config_hash(canonical: str) -> str:
    h = 0xCBF29CE484222325
    for c in canonical.encode():
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


class _Stream:
    """ostream with the reference's sticky precision (6 until the first full print, then 17)."""

    def __init__(self):
        self.parts: List[str] = []
        self.prec = 6

    def s(self, v: str):
        self.parts.append(v)

    def num(self, v: float):  # out << double
        self.parts.append(_g(v, self.prec))

    def full(self, v: float):  # print_full (io.cpp:25-31)
        if math.isnan(v):
            self.parts.append("nan")
            return
        self.prec = 17
        self.parts.append(_g(v, 17))

    def text(self) -> str:
        return "".join(self.parts)


def _g(v: float, prec: int) -> str:
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.*g" % (prec, v)


def write_time_series_csv(times: Sequence[float], values: Sequence[float], hash_: str) -> str:
    o = _Stream()
    o.s(f"# config_hash={hash_}\nt,x\n")
    for tv, xv in zip(times, values):
        o.full(tv)
        o.s(",")
        o.full(xv)
        o.s("\n")
    return o.text()


def write_spectrum_csv(centers: Sequence[float], power: Sequence[float], k_used: Sequence[int],
                       f_w_used: Sequence[float], flags: Sequence[int], method: str, hash_: str) -> str:
    o = _Stream()
    o.s(f"# config_hash={hash_}\n# method={method}\nf_center,power,power_db,k_used,f_w_used,flag\n")
    for c, p, k, fw, fl in zip(centers, power, k_used, f_w_used, flags):
        o.full(c)
        o.s(",")
        o.full(p)
        o.s(",")
        db = 10.0 * math.log10(p) if p > 0.0 else -math.inf
        if math.isnan(p):
            o.s("nan")
        elif math.isinf(db):
            o.s("-inf")
        else:
            o.full(db)
        o.s(f",{int(k)},")
        o.full(fw)
        o.s(f",{int(fl)}\n")
    return o.text()


def write_ftest_csv(centers: Sequence[float], f_stat: Sequence[float], amplitude: Sequence[complex],
                    flags: Sequence[int], dof: Tuple[int, int], critical_values: Sequence[Tuple[float, float]],
                    hash_: str) -> str:
    o = _Stream()
    o.s(f"# config_hash={hash_}\n# dof={int(dof[0])},{int(dof[1])}\n")
    for p, crit in critical_values:
        o.s("# critical p=")
        o.num(p)
        o.s(" value=")
        o.full(crit)
        o.s("\n")
    o.s("f_center,f_stat,amp_re,amp_im")
    for p, _ in critical_values:
        o.s(",exceeds_p")
        o.num(p)
    o.s(",flag\n")
    for c, f, a, fl in zip(centers, f_stat, amplitude, flags):
        o.full(c)
        o.s(",")
        o.full(f)
        o.s(",")
        o.full(complex(a).real)
        o.s(",")
        o.full(complex(a).imag)
        for _, crit in critical_values:
            o.s(",1" if f > crit else ",0")
        o.s(f",{int(fl)}\n")
    return o.text()


_JSON_ESC = {'"': '\\"', "\\": "\\\\", "\b": "\\b", "\f": "\\f", "\n": "\\n", "\r": "\\r", "\t": "\\t"}


def _json_str(s: str) -> str:
    out = ['"']
    for ch in s:
        if ch in _JSON_ESC:
            out.append(_JSON_ESC[ch])
        elif ord(ch) < 0x20:
            out.append("\\u%04x" % ord(ch))
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def write_manifest_json(command: str, fields: Iterable[Tuple[str, str]], hash_: str) -> str:
    config = {}
    for k, v in fields:
        config[k] = v  # the last duplicate wins
    lines = ["{", f'  "command": {_json_str(command)},']
    if config:
        lines.append('  "config": {')
        keys = sorted(config, key=lambda k: k.encode())  # std::map byte order
        for i, k in enumerate(keys):
            lines.append(f"    {_json_str(k)}: {_json_str(config[k])}" + ("," if i + 1 < len(keys) else ""))
        lines.append("  },")
    lines.append(f'  "config_hash": {_json_str(hash_)},')
    lines.append(f'  "version": {_json_str(library_version())}')
    lines.append("}")
    return "\n".join(lines) + "\n"


def library_version() -> str:
    return "0.1.0"  # the reference's manifest version string (io.cpp:276), kept for interchangeability
