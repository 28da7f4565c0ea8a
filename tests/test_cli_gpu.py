"""CLI front end end to end on the device: every output byte-compared with
fixtures assembled from the reference's own values and formatting primitives
(tests/golden/make_cli_goldens.py, oracle/_ref: the reference engine,
permlab::to_string, Interferometer::to_json, nlohmann dumps). The fixtures are
committed, so this runs where oracle/_ref is not built."""
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
FIX = ROOT / "tests" / "cli_fixtures"
GOLD = ROOT / "tests" / "golden" / "cli"


def run(*args):
    r = subprocess.run([sys.executable, "-m", "paper_1802_02779_b200.cli", *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    return r.stdout


def gold(name):
    return (GOLD / name).read_text()


def compact_int_arrays(text):
    # the reference's stock nlohmann breaks integer arrays across lines; the fixture was
    # dumped by the image's nlohmann copy, which prints them on one line (tests/test_cli.py)
    return re.sub(r"\[\s*((?:-?\d+,\s*)*-?\d+)\s*\]", lambda mt: "[" + re.sub(r"\s+", "", mt.group(1)) + "]", text)


def test_perm_int_json_and_text():
    out = run("perm", "--matrix", str(FIX / "dev4.json"), "--algorithm", "store-zechin")
    assert out == "algorithm: store-zechin\nvalue: 9722\nmultiplications: 28\nadditions: 17\n"
    out = run("perm", "--matrix", str(FIX / "dev4.json"), "--algorithm", "store-zechin", "--format", "json")
    assert out == gold("perm_dev4.json")
    out = run("perm", "--matrix", str(FIX / "a2.csv"), "--algorithm", "store-zechin")
    assert "value: 10\n" in out


def test_perm_int_beyond_int64(tmp_path):
    # the reference's Int ring is arbitrary precision: text prints the decimal value, JSON carries
    # a string once the value leaves long long (reference tools/permlab_cli.cpp:91-99, 160-169)
    import json
    import math

    ones = tmp_path / "ones21.csv"
    ones.write_text("\n".join(",".join("1" for _ in range(21)) for _ in range(21)) + "\n")
    out = run("perm", "--matrix", str(ones), "--algorithm", "store-zechin")
    assert out.splitlines()[1] == "value: %d" % math.factorial(21)
    js = json.loads(run("perm", "--matrix", str(ones), "--algorithm", "store-zechin", "--format", "json"))
    assert js["value"] == str(math.factorial(21)) and js["order"] == 21
    # entries beyond int64 as well: per([[10^30, 1], [2, -10^25]]) = -10^55 + 2
    big = tmp_path / "big2.csv"
    big.write_text("1" + "0" * 30 + ",1\n2,-1" + "0" * 25 + "\n")
    out = run("perm", "--matrix", str(big), "--algorithm", "store-zechin")
    assert out.splitlines()[1] == "value: %d" % (2 - 10 ** 55)


def test_perm_complex_matches_reference_bytes():
    assert run("perm", "--matrix", str(FIX / "c3.json"), "--algorithm", "store-zechin") == gold("perm_c3.txt")
    assert run("perm", "--matrix", str(FIX / "c3.json"), "--algorithm", "store-zechin", "--format",
               "json") == gold("perm_c3.json")
    out = run("perm", "--matrix", str(FIX / "r2.csv"), "--ring", "complex", "--algorithm", "store-zechin")
    r = 0.5 * 1e-3 + (-1.25) * 2.0
    assert out.splitlines()[1] == "value: " + "%.17g" % r


def test_boson_workflow_matches_reference(tmp_path):
    f = tmp_path / "u.json"
    assert run("randu", "--modes", "6", "--seed", "7", "--out", str(f)) == f"wrote {f} (modes=6, seed=7)\n"
    assert f.read_text() == gold("u6_seed7.json")
    assert run("bs-dist", "--unitary", str(f), "--input", "1,3,4") == gold("dist_u6_134.txt")
    assert run("bs-dist", "--unitary", str(f), "--input", "1,3,4", "--format", "csv") == gold("dist_u6_134.csv")
    js = run("bs-dist", "--unitary", str(f), "--input", "1,3,4", "--format", "json")
    assert compact_int_arrays(js) == gold("dist_u6_134.compact.json")
    assert run("bs-sample", "--unitary", str(f), "--input", "1,3,4", "--count", "50", "--seed",
               "9") == gold("sample_u6_134_50_9.txt")
    assert run("bs-sample", "--unitary", str(f), "--input", "1,3,4", "--count", "50", "--seed", "9", "--format",
               "json") == gold("sample_u6_134_50_9.json")
    assert run("bs-sample", "--unitary", str(f), "--input", "1,2", "--count", "0", "--seed", "1") == ""


def test_perm_ryser(tmp_path):
    # reference tests/test_cli.cpp:114-121: `perm --algorithm ryser --format json` on I3
    id3 = tmp_path / "id3.csv"
    id3.write_text("1,0,0\n0,1,0\n0,0,1\n")
    import json

    js = json.loads(run("perm", "--matrix", str(id3), "--algorithm", "ryser", "--format", "json"))
    assert js["value"] == 1 and js["algorithm"] == "ryser"
    assert js["counts"] == {"multiplications": 14, "additions": 18}
    out = run("perm", "--matrix", str(FIX / "dev4.json"), "--algorithm", "ryser")
    assert out == "algorithm: ryser\nvalue: 9722\nmultiplications: 45\nadditions: 58\n"
