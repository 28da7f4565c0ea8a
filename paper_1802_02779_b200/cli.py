"""Command-line front end over the device engine: the reference CLI's
Store-zechin and boson-sampling subcommands with the same arguments, output
formats and exit codes (reference ``proj/tools/permlab_cli.cpp``).

    python -m paper_1802_02779_b200.cli perm --matrix FILE --algorithm store-zechin|ryser [--ring int|complex] [--format text|json]
    python -m paper_1802_02779_b200.cli bs-dist --unitary FILE --input 1,2,3 [--format text|csv|json]
    python -m paper_1802_02779_b200.cli bs-sample --unitary FILE --input 1,2 --count N --seed S [--format text|json]
    python -m paper_1802_02779_b200.cli randu --modes M --seed S --out FILE

Every permanent and probability is computed on the GPU (``api`` / ``boson``);
this module parses the reference's matrix files (JSON schema of
``matrix.cpp:200-250``, CSV of ``matrix.cpp:100-160``) and renders the
reference's outputs: ``%.17g`` values (``ring.cpp:95-120``), and JSON as the
reference's nlohmann::json ``dump`` writes it (keys sorted, 2-space indent,
shortest round-trip doubles with exponents outside [1e-4, 1e15)). Exit codes:
0 ok, 1 usage error, 2 ``error: <message>`` on stderr (``permlab_cli.cpp:360-377``).
The naive and Ryser engines, the cost-model subcommands (count, attribute,
table, verdict) and the Rational ring are not offered by the device engine.
"""
from __future__ import annotations

import argparse
import json
import math
import re
import sys
from typing import List

import numpy as np

from . import api
from . import boson as B
from .api import DomainError, Limits

# ---------------------------------------------------------------- rendering


def g17(x: float) -> str:
    """printf("%.17g") (reference ring.cpp double_to_string)."""
    return "%.17g" % x


def value_text(v) -> str:
    """permlab::to_string of a ring element (reference ring.cpp:102-120)."""
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    z = complex(v)
    if z.imag == 0.0:
        return g17(z.real)
    s = g17(z.real)
    if not z.imag < 0:
        s += "+"
    return s + g17(z.imag) + "i"


# nlohmann::json writes doubles with Grisu2 (Loitsch 2010: a 64-bit "diy fp"
# approximation scaled by a cached power of ten, digits generated until they
# fall inside the rounding interval, then nudged towards the exact value). It
# is not always the shortest representation, so Python's repr would differ in
# the last digit for ~0.1 % of values; this restates the published algorithm.
_M64 = (1 << 64) - 1


def _cached_power(k: int):
    """(f, e): the 64-bit significand of 10^k rounded to nearest, 10^k ~ f * 2^e."""
    from fractions import Fraction

    v = Fraction(10) ** k
    e = (v.numerator.bit_length() - v.denominator.bit_length()) - 64
    while v / Fraction(2) ** e >= (1 << 64):
        e += 1
    while v / Fraction(2) ** e < (1 << 63):
        e -= 1
    f = v / Fraction(2) ** e
    return int(f + Fraction(1, 2)), e


_CACHED = {}


def _diy_mul(xf: int, xe: int, yf: int, ye: int):
    return ((xf * yf + (1 << 63)) >> 64) & _M64, xe + ye + 64


def _normalize(f: int, e: int):
    sh = 64 - f.bit_length()
    return f << sh, e - sh


def _grisu2(x: float):
    """(digit string, decimal exponent) of x > 0 as nlohmann's dtoa_impl::grisu2."""
    import struct

    bits = struct.unpack("<Q", struct.pack("<d", x))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    if E == 0:
        vf, ve = F, 1 - 1075
    else:
        vf, ve = F + (1 << 52), E - 1075
    lower_closer = F == 0 and E > 1
    mpf, mpe = 2 * vf + 1, ve - 1
    if lower_closer:
        mmf, mme = 4 * vf - 1, ve - 2
    else:
        mmf, mme = 2 * vf - 1, ve - 1
    wpf, wpe = _normalize(mpf, mpe)
    wmf, wme = mmf << (mme - wpe), wpe
    wf, we = _normalize(vf, ve)
    # cached power c = 10^-k with the product exponent in [-60, -32]
    fk = -60 - wpe - 1
    k = (fk * 78913) // (1 << 18) + (1 if fk > 0 else 0)
    if fk * 78913 < 0 and (fk * 78913) % (1 << 18):
        k = -((-fk * 78913) // (1 << 18)) + (1 if fk > 0 else 0)  # C++ division truncates toward zero
    index = (300 + k + 7) // 8
    dk = -300 + 8 * index
    if dk not in _CACHED:
        _CACHED[dk] = _cached_power(dk)
    cf, ce = _CACHED[dk]
    w = _diy_mul(wf, we, cf, ce)
    w_minus = _diy_mul(wmf, wme, cf, ce)
    w_plus = _diy_mul(wpf, wpe, cf, ce)
    Mm, Mp = w_minus[0] + 1, w_plus[0] - 1
    e = w_plus[1]
    dec_exp = -dk
    # digit generation
    delta = Mp - Mm
    p1_dist = Mp - w[0]
    one = 1 << -e
    p1 = Mp >> -e
    p2 = Mp & (one - 1)
    buf = []
    kk = len(str(p1)) if p1 > 0 else 1
    pow10 = 10 ** (kk - 1)
    n = kk
    while n > 0:
        d, r = divmod(p1, pow10)
        buf.append(d)
        p1 = r
        n -= 1
        rest = (p1 << -e) + p2
        if rest <= delta:
            dec_exp += n
            _grisu2_round(buf, p1_dist, delta, rest, pow10 << -e)
            return "".join(map(str, buf)), dec_exp
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        d, r = p2 >> -e, p2 & (one - 1)
        buf.append(d)
        p2 = r
        m += 1
        delta *= 10
        p1_dist *= 10
        if p2 <= delta:
            break
    dec_exp -= m
    _grisu2_round(buf, p1_dist, delta, p2, one)
    return "".join(map(str, buf)), dec_exp


def _grisu2_round(buf, dist, delta, rest, ten_k):
    while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
        buf[-1] -= 1
        rest += ten_k


def _json_double(x: float) -> str:
    """A double as nlohmann::json dumps it: Grisu2 digits, decimal notation
    for decimal-point positions in (-4, 15], exponent otherwise (explicit
    sign, at least two digits), integral values with a trailing .0."""
    if math.isnan(x) or math.isinf(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign = "-" if x < 0 else ""
    digits, dec_exp = _grisu2(abs(x))
    k = len(digits)
    n = k + dec_exp
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    ee = n - 1
    m = digits[0] + ("." + digits[1:] if k > 1 else "")
    return sign + m + "e" + ("-" if ee < 0 else "+") + ("%02d" % abs(ee))


def json_dump(obj, indent: int = -1, _level: int = 0) -> str:
    """nlohmann::json::dump(indent) for the value types the CLI emits."""
    if isinstance(obj, bool):
        return "true" if obj else "false"
    if isinstance(obj, (int, np.integer)):
        return str(int(obj))
    if isinstance(obj, (float, np.floating)):
        return _json_double(float(obj))
    if isinstance(obj, str):
        return json.dumps(obj)
    pad = " " * (indent * (_level + 1)) if indent >= 0 else ""
    end = " " * (indent * _level) if indent >= 0 else ""
    nl = "\n" if indent >= 0 else ""
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        sep = ": " if indent >= 0 else ":"
        items = [pad + json.dumps(k) + sep + json_dump(obj[k], indent, _level + 1) for k in sorted(obj)]
        return "{" + nl + ("," + nl).join(items) + nl + end + "}"
    if isinstance(obj, (list, tuple)):
        if not obj:
            return "[]"
        items = [pad + json_dump(v, indent, _level + 1) for v in obj]
        return "[" + nl + ("," + nl).join(items) + nl + end + "]"
    raise TypeError(type(obj))


def pattern_text(occ) -> str:
    return "[" + ",".join(str(int(c)) for c in occ) + "]"


# ---------------------------------------------------------------- parsing


def _read(path: str) -> str:
    try:
        with open(path, "rb") as f:
            return f.read().decode("utf-8", errors="surrogateescape")
    except OSError:
        raise DomainError("cannot read file: " + path)


def _ring_from_name(name: str) -> str:
    if name not in ("int", "rational", "complex"):
        raise DomainError("unknown ring name: " + name)
    return name


def _parse_int_literal(tok: str) -> int:
    if not re.fullmatch(r"[+-]?\d+", tok):
        raise DomainError("malformed integer literal: " + tok)
    return int(tok)


def parse_csv(text: str, ring: str) -> np.ndarray:
    """Reference matrix.cpp parse_csv: one row per nonblank line, comma cells."""
    if ring == "rational":
        raise DomainError("csv holds integers/decimals only; use json for rational matrices")
    lines = []
    for line in text.split("\n"):
        if line.endswith("\r"):
            line = line[:-1]
        if line.strip():
            lines.append(line)
    n = len(lines)
    if n < 1:
        raise DomainError("csv matrix is empty")
    vals: List = []
    for line in lines:
        cells = line.split(",")
        if len(cells) != n:
            raise DomainError("csv matrix is not square")
        for cell in cells:
            tok = cell.strip()
            if not tok:
                raise DomainError("empty csv cell")
            if ring == "int":
                vals.append(_parse_int_literal(tok))
            else:
                try:
                    vals.append(complex(float(tok), 0.0))
                except ValueError:
                    raise DomainError("malformed decimal literal: " + tok)
    if ring == "int":
        return _int_matrix(n, vals)
    return np.array(vals, dtype=np.complex128).reshape(n, n)


def _int_matrix(n: int, vals) -> np.ndarray:
    if any(v < -(1 << 63) or v >= (1 << 63) for v in vals):
        # entries beyond int64: Python integers, computed by the residue passes (api.store_zechin_permanent)
        return np.array(vals, dtype=object).reshape(n, n)
    return np.array(vals, dtype=np.int64).reshape(n, n)


def matrix_from_json(j) -> np.ndarray:
    """Reference matrix.cpp matrix_from_json."""
    if not isinstance(j, dict):
        raise DomainError("matrix json must be an object")
    order = j.get("order")
    if not isinstance(order, int) or isinstance(order, bool):
        raise DomainError('matrix json needs an integer "order"')
    if order < 1:
        raise DomainError("matrix order must be >= 1")
    ring = j.get("ring")
    if not isinstance(ring, str):
        raise DomainError('matrix json needs a "ring" of int|rational|complex')
    ring = _ring_from_name(ring)
    entries = j.get("entries")
    if not isinstance(entries, list) or len(entries) != order:
        raise DomainError("entries must form a square row-major array")
    for row in entries:
        if not isinstance(row, list) or len(row) != order:
            raise DomainError("entries must form a square row-major array")
    if ring == "rational":
        raise DomainError("the rational ring is not offered by the device engine")
    if ring == "int":
        vals = []
        for row in entries:
            for cell in row:
                if isinstance(cell, bool) or not isinstance(cell, (int, str)):
                    raise DomainError("int ring entries must be integers or decimal strings")
                if isinstance(cell, str):
                    try:
                        cell = int(cell.strip())
                    except ValueError:
                        raise DomainError("malformed integer literal: " + cell)
                vals.append(cell)
        return _int_matrix(order, vals)
    out = np.empty((order, order), dtype=np.complex128)
    for i, row in enumerate(entries):
        for k, cell in enumerate(row):
            if (not isinstance(cell, list) or len(cell) != 2 or
                    not all(isinstance(x, (int, float)) and not isinstance(x, bool) for x in cell)):
                raise DomainError("complex ring entries must be [re, im] number pairs")
            out[i, k] = complex(float(cell[0]), float(cell[1]))
    return out


def load_matrix(path: str, csv_ring: str) -> np.ndarray:
    text = _read(path)
    if path.endswith(".csv"):
        return parse_csv(text, _ring_from_name(csv_ring))
    try:
        j = json.loads(text)
    except ValueError as e:
        raise DomainError("malformed json: " + str(e))
    return matrix_from_json(j)


def interferometer_from_json(text: str) -> B.Interferometer:
    """Reference boson.cpp Interferometer::from_json."""
    try:
        j = json.loads(text)
    except ValueError as e:
        raise DomainError("malformed json: " + str(e))
    if not isinstance(j, dict) or not isinstance(j.get("modes"), int) or isinstance(j.get("modes"), bool):
        raise DomainError('interferometer json needs an integer "modes"')
    m = matrix_from_json(j)
    if m.dtype != np.complex128:
        raise DomainError("interferometer unitary must use the complex ring")
    return B.Interferometer(j["modes"], m)


def interferometer_to_json(itf: B.Interferometer) -> str:
    u = itf.unitary()
    entries = [[[float(z.real), float(z.imag)] for z in row] for row in u]
    return json_dump({"order": u.shape[0], "ring": "complex", "entries": entries, "modes": itf.modes()}, 2) + "\n"


def parse_modes(text: str) -> List[int]:
    """1-based mode list (reference permlab_cli.cpp parse_modes; std::stoi
    accepts a leading integer)."""
    out = []
    items = text.split(",")
    if items and items[-1] == "":  # std::getline yields no trailing empty field
        items.pop()
    for item in items:
        mt = re.match(r"\s*([+-]?\d+)", item)
        if not mt or not (-(1 << 31) <= int(mt.group(1)) < (1 << 31)):
            raise DomainError("malformed mode list: " + text)
        v = int(mt.group(1))
        if v < 1:
            raise DomainError("mode indices are 1-based")
        out.append(v - 1)
    if not out:
        raise DomainError("mode list is empty")
    return out


# ---------------------------------------------------------------- subcommands


def run_perm(opt) -> str:
    m = load_matrix(opt.matrix, opt.ring)
    if opt.algorithm not in ("naive", "ryser", "store-zechin"):
        raise DomainError("unknown algorithm: " + opt.algorithm)
    if opt.algorithm == "naive":
        raise DomainError("the naive engine is not offered by the device engine (store-zechin and ryser only)")
    run = api.ryser_permanent if opt.algorithm == "ryser" else api.store_zechin_permanent
    r = run(m, opt.limits)
    n = m.shape[0]
    if opt.format == "json":
        v = r.value
        if isinstance(v, (int, np.integer)):
            # reference tools/permlab_cli.cpp:91-99: a number inside long long, else the decimal string
            vj = int(v) if -(1 << 63) <= int(v) < (1 << 63) else str(int(v))
        else:
            vj = [complex(v).real, complex(v).imag]
        return json_dump({"algorithm": opt.algorithm, "order": n, "value": vj,
                          "counts": {"multiplications": r.counts.multiplications,
                                     "additions": r.counts.additions}}, 2) + "\n"
    return ("algorithm: " + opt.algorithm + "\n" + "value: " + value_text(r.value) + "\n" +
            "multiplications: %d\n" % r.counts.multiplications + "additions: %d\n" % r.counts.additions)


def run_bs_dist(opt) -> str:
    itf = interferometer_from_json(_read(opt.unitary))
    modes = parse_modes(opt.input)
    dist = B.full_distribution(itf, modes, opt.limits)
    occ = B.pattern_occupancies(itf.modes(), len(modes))
    probs = dist.probabilities
    if opt.format == "json":
        entries = [{"pattern": [int(c) for c in o], "probability": float(p)} for o, p in zip(occ, probs)]
        return json_dump({"modes": itf.modes(), "photons": len(modes), "entries": entries}, 2) + "\n"
    out = []
    if opt.format == "csv":
        out.append("pattern,probability\n")
        for o, p in zip(occ, probs):
            out.append(pattern_text(o).replace(",", " ") + "," + g17(float(p)) + "\n")
        return "".join(out)
    for o, p in zip(occ, probs):
        out.append(pattern_text(o) + " " + ("%.12g" % float(p)) + "\n")
    return "".join(out)


def run_bs_sample(opt) -> str:
    itf = interferometer_from_json(_read(opt.unitary))
    modes = parse_modes(opt.input)
    dist = B.full_distribution(itf, modes, opt.limits)
    idx = B.sample_indices(dist, opt.count, opt.seed) if opt.count else np.zeros(0, dtype=np.int64)
    occ = B.pattern_occupancies(itf.modes(), len(modes))
    draws = occ[idx]
    if opt.format == "json":
        return json_dump([[int(c) for c in o] for o in draws]) + "\n"
    return "".join(pattern_text(o) + "\n" for o in draws)


def run_randu(opt) -> str:
    itf = B.haar_unitary(opt.modes, opt.seed)
    try:
        with open(opt.out, "w") as f:
            f.write(interferometer_to_json(itf))
    except OSError:
        raise DomainError("cannot write file: " + opt.out)
    return "wrote %s (modes=%d, seed=%d)\n" % (opt.out, opt.modes, opt.seed)


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (reference: CLI11 ParseError -> 1)
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        sys.exit(1)


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="permlab", description="permlab on the B200 engine: Store-zechin permanents and "
                                             "boson-sampling probabilities")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    p = sub.add_parser("perm", help="Compute a permanent and its operation counts")
    p.add_argument("--matrix", required=True)
    p.add_argument("--algorithm", required=True)
    p.add_argument("--ring", default="int")
    p.add_argument("--format", default="text", choices=["text", "json"])
    d = sub.add_parser("bs-dist", help="Full boson-sampling output distribution")
    d.add_argument("--unitary", required=True)
    d.add_argument("--input", required=True)
    d.add_argument("--format", default="text", choices=["text", "csv", "json"])
    s = sub.add_parser("bs-sample", help="Seeded draws from the output distribution")
    s.add_argument("--unitary", required=True)
    s.add_argument("--input", required=True)
    s.add_argument("--count", required=True, type=int)
    s.add_argument("--seed", required=True, type=int)
    s.add_argument("--format", default="text", choices=["text", "json"])
    r = sub.add_parser("randu", help="Write a seeded Haar-random interferometer")
    r.add_argument("--modes", required=True, type=int)
    r.add_argument("--seed", required=True, type=int)
    r.add_argument("--out", required=True)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        limits = Limits.from_env()
        opt = ap.parse_args(argv)
        opt.limits = limits
        out = {"perm": run_perm, "bs-dist": run_bs_dist, "bs-sample": run_bs_sample, "randu": run_randu}[opt.cmd](opt)
    except SystemExit as e:
        return int(e.code or 0)
    except Exception as e:  # DomainError and device errors: the reference's "error: ..." and exit 2
        sys.stderr.write("error: " + str(e) + "\n")
        return 2
    sys.stdout.write(out)
    sys.stdout.flush()
    return 0


if __name__ == "__main__":
    sys.exit(main())
