"""CLI front end (paper_1802_02779_b200/cli.py) — host side, no GPU: matrix
file parsing against the reference's own parse_matrix (oracle/_ref), the
value text against the reference's permlab::to_string, JSON layout and number
round trips against nlohmann::json as the reference CLI dumps it, argument
errors and exit codes (reference tools/permlab_cli.cpp)."""
import json
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1802_02779_b200 import boson as B
from paper_1802_02779_b200 import cli
from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]
FIX = ROOT / "tests" / "cli_fixtures"
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@need_ref
@pytest.mark.parametrize("name,ring", [("dev4.json", "int"), ("a2.csv", "int"), ("r2.csv", "complex"),
                                       ("c3.json", "complex")])
def test_matrix_files_parse_like_the_reference(name, ring):
    text = (FIX / name).read_text()
    n, rring, want = O.ref_parse_matrix(text, name.endswith(".csv"), ring == "complex")
    got = cli.load_matrix(str(FIX / name), ring)
    assert got.shape == (n, n)
    assert (got.dtype == np.int64) == (rring == "int")
    assert np.array_equal(got, want)


@need_ref
@pytest.mark.parametrize("text,csv,msg", [
    ("1,2\n3\n", True, "csv matrix is not square"),
    ("1,,\n1,2,3\n4,5,6\n", True, "empty csv cell"),
    ("1,x\n3,4\n", True, "malformed integer literal: x"),
    ("", True, "csv matrix is empty"),
    ('{"order": 2, "ring": "int", "entries": [[1, 2]]}', False, "entries must form a square row-major array"),
    ('{"order": 1, "ring": "quaternion", "entries": [[1]]}', False, "unknown ring name: quaternion"),
    ('{"ring": "int", "entries": [[1]]}', False, 'matrix json needs an integer "order"'),
    ('{"order": 1, "ring": "complex", "entries": [[1]]}', False, "complex ring entries must be [re, im] number pairs"),
    ('[1]', False, "matrix json must be an object"),
])
def test_parse_errors_match_reference_messages(tmp_path, text, csv, msg):
    with pytest.raises(O.OracleError, match=re.escape(msg)):
        O.ref_parse_matrix(text, csv)
    f = tmp_path / ("m.csv" if csv else "m.json")
    f.write_text(text)
    with pytest.raises(cli.DomainError, match=re.escape(msg)):
        cli.load_matrix(str(f), "int")


@need_ref
def test_value_text_matches_reference_to_string():
    vals = [0, -5, 2 ** 62, 12345, 1 + 2j, 1 - 2j, 3 + 0j, complex(-0.0, 0.0), complex(1e-30, -1e30),
            complex(0.1, 0.0), complex(2.0, -0.0), complex(-1.5e300, 7e-300)]
    rng = np.random.default_rng(3)
    vals += [complex(x, y) for x, y in rng.standard_normal((200, 2)) * 10.0 ** rng.integers(-40, 40, (200, 2))]
    for v in vals:
        assert cli.value_text(v) == O.ref_fmt_value_text(v), v


def _skeleton(text):
    # JSON layout with every number replaced: indentation, keys, separators
    return re.sub(r"-?\d+(\.\d+)?(e[+-]\d+)?", "#", text)


@need_ref
def test_json_layout_and_numbers_match_nlohmann():
    z = 1.2345e-7 - 3.3e2j
    a = O.ref_fmt_perm_json(z, 5, 75, 49)
    b = cli.json_dump({"algorithm": "store-zechin", "order": 5, "value": [z.real, z.imag],
                       "counts": {"multiplications": 75, "additions": 49}}, 2) + "\n"
    assert a == b
    assert O.ref_fmt_perm_json(-42, 3, 9, 5) == cli.json_dump(
        {"algorithm": "store-zechin", "order": 3, "value": -42, "counts": {"multiplications": 9, "additions": 5}},
        2) + "\n"
    occ = np.array([[1, 0, 2], [0, 3, 0]], dtype=np.int32)
    assert O.ref_fmt_sample_json(occ) == cli.json_dump(occ.tolist()) + "\n"
    # interferometer files: byte-identical (arrays of doubles)
    for m, seed in ((6, 7), (25, 2)):
        u = O.ref_haar(m, seed)
        assert O.ref_fmt_itf_json(u) == cli.interferometer_to_json(B.Interferometer(m, u))
    # doubles exactly as nlohmann's Grisu2 writes them (subnormals, extremes, random bits)
    rng = np.random.default_rng(0)
    vals = [1e15, 1e16, 9.99e14, 123456789012345.0, 1e-4, 1e-5, 0.00012, 0.1, 1.0, 123.0, 2.5e-300,
            1.7976931348623157e308, 5e-324, 2.2250738585072014e-308, 1e22, 0.0, -0.0, -1.5e-7]
    vals += list(rng.random(3000)) + list(10 ** rng.uniform(-300, 300, 3000))
    raw = np.frombuffer(rng.integers(0, 2 ** 63, 3000, dtype=np.int64).tobytes(), dtype=np.float64)
    vals += [float(v) for v in raw if np.isfinite(v)]
    occ = np.zeros((len(vals), 1), dtype=np.int32)
    ref = O.ref_fmt_dist_json(1, 0, occ, np.array(vals, dtype=np.float64))
    rp = [l.split(": ")[1].rstrip(",") for l in ref.splitlines() if "probability" in l]
    assert rp == [cli.json_dump(float(v)) for v in vals]


@need_ref
def test_distribution_json_matches_reference_layout():
    # the image's nlohmann copy (cudnn_frontend) prints integer arrays on one line, a local
    # modification; the reference's stock nlohmann 3.11.3 breaks every array across lines,
    # which is what the CLI writes. Everything else is compared byte for byte.
    u = O.ref_haar(5, 3)
    occ, probs = O.ref_full_distribution(u, [0, 2])
    ref = O.ref_fmt_dist_json(5, 2, occ, probs)
    mine = cli.json_dump({"modes": 5, "photons": 2, "entries": [
        {"pattern": o.tolist(), "probability": float(p)} for o, p in zip(occ, probs)]}, 2) + "\n"
    compact = re.sub(r"\[\s*((?:-?\d+,\s*)*-?\d+)\s*\]", lambda mt: "[" + re.sub(r"\s+", "", mt.group(1)) + "]", mine)
    assert compact == ref
    assert json.loads(mine) == json.loads(ref)


def test_parse_modes():
    assert cli.parse_modes("1,2,3") == [0, 1, 2]
    assert cli.parse_modes(" 2,3,") == [1, 2]
    for bad, msg in [("0,1", "mode indices are 1-based"), ("a,1", "malformed mode list"), ("", "mode list is empty"),
                     ("1,,2", "malformed mode list")]:
        with pytest.raises(cli.DomainError, match=msg):
            cli.parse_modes(bad)


def test_usage_errors_exit_1_and_domain_errors_exit_2(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_1802_02779_b200.cli", "perm", "--matrix", "x.json"],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 1 and r.stdout == ""
    r = subprocess.run([sys.executable, "-m", "paper_1802_02779_b200.cli", "perm", "--matrix",
                        str(tmp_path / "missing.json"), "--algorithm", "store-zechin"],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 2 and r.stderr.startswith("error: cannot read file:") and r.stdout == ""
    r = subprocess.run([sys.executable, "-m", "paper_1802_02779_b200.cli", "perm", "--matrix",
                        str(FIX / "dev4.json"), "--algorithm", "naive"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 2 and "store-zechin and ryser only" in r.stderr
