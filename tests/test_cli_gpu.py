"""CLI front end end to end on the device: every output byte-compared with the
reference's own values and formatting primitives (oracle/_ref)."""
import json
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1802_02779_b200 as pl
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]
ROOT = Path(__file__).resolve().parents[1]
FIX = ROOT / "tests" / "cli_fixtures"


def run(*args):
    r = subprocess.run([sys.executable, "-m", "paper_1802_02779_b200.cli", *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_perm_int_json_and_text():
    out = run("perm", "--matrix", str(FIX / "dev4.json"), "--algorithm", "store-zechin")
    assert out == "algorithm: store-zechin\nvalue: 9722\nmultiplications: 28\nadditions: 17\n"
    out = run("perm", "--matrix", str(FIX / "dev4.json"), "--algorithm", "store-zechin", "--format", "json")
    assert out == O.ref_fmt_perm_json(9722, 4, 28, 17)
    out = run("perm", "--matrix", str(FIX / "a2.csv"), "--algorithm", "store-zechin")
    assert "value: 10\n" in out


def test_perm_complex_matches_reference_bytes():
    from paper_1802_02779_b200 import cli

    m = cli.load_matrix(str(FIX / "c3.json"), "int")
    want, (mults, adds) = O.ref_sz_c128(m)
    out = run("perm", "--matrix", str(FIX / "c3.json"), "--algorithm", "store-zechin")
    assert out == f"algorithm: store-zechin\nvalue: {O.ref_fmt_value_text(want)}\nmultiplications: {mults}\nadditions: {adds}\n"
    out = run("perm", "--matrix", str(FIX / "c3.json"), "--algorithm", "store-zechin", "--format", "json")
    assert out == O.ref_fmt_perm_json(want, 3, mults, adds)
    out = run("perm", "--matrix", str(FIX / "r2.csv"), "--ring", "complex", "--algorithm", "store-zechin")
    r = 0.5 * 1e-3 + (-1.25) * 2.0
    assert out.splitlines()[1] == "value: " + O.ref_fmt_value_text(complex(r, 0.0))


def test_boson_workflow_matches_reference(tmp_path):
    f = tmp_path / "u.json"
    assert run("randu", "--modes", "6", "--seed", "7", "--out", str(f)) == f"wrote {f} (modes=6, seed=7)\n"
    u = O.ref_haar(6, 7)
    assert f.read_text() == O.ref_fmt_itf_json(u)
    occ, probs = O.ref_full_distribution(u, [0, 2, 3])
    txt = run("bs-dist", "--unitary", str(f), "--input", "1,3,4")
    assert txt == "".join("[" + ",".join(map(str, o)) + "] " + ("%.12g" % p) + "\n" for o, p in zip(occ, probs))
    csv = run("bs-dist", "--unitary", str(f), "--input", "1,3,4", "--format", "csv")
    assert csv == "pattern,probability\n" + "".join(
        "[" + " ".join(map(str, o)) + "]," + ("%.17g" % p) + "\n" for o, p in zip(occ, probs))
    js = run("bs-dist", "--unitary", str(f), "--input", "1,3,4", "--format", "json")
    ref = O.ref_fmt_dist_json(6, 3, occ, probs)
    compact = re.sub(r"\[\s*((?:-?\d+,\s*)*-?\d+)\s*\]", lambda mt: "[" + re.sub(r"\s+", "", mt.group(1)) + "]", js)
    assert compact == ref  # stock-nlohmann integer arrays span lines (see tests/test_cli.py)
    draws = O.ref_sample(u, [0, 2, 3], 50, 9)
    smp = run("bs-sample", "--unitary", str(f), "--input", "1,3,4", "--count", "50", "--seed", "9")
    assert smp == "".join("[" + ",".join(map(str, o)) + "]\n" for o in draws)
    smj = run("bs-sample", "--unitary", str(f), "--input", "1,3,4", "--count", "50", "--seed", "9", "--format",
              "json")
    assert smj == O.ref_fmt_sample_json(draws)
    assert run("bs-sample", "--unitary", str(f), "--input", "1,2", "--count", "0", "--seed", "1") == ""
