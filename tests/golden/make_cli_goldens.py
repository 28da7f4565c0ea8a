"""Writes tests/golden/cli/*: expected CLI outputs assembled from the reference's own values
and formatting primitives (oracle/_ref: the reference engine, permlab::to_string,
Interferometer::to_json, nlohmann dumps), so tests/test_cli_gpu.py can compare the device
CLI byte for byte where oracle/_ref is not built. Run in the build container:
    python tests/golden/make_cli_goldens.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_1802_02779_b200 import cli  # noqa: E402  (parsing only: no device work)

out = ROOT / "tests" / "golden" / "cli"
out.mkdir(parents=True, exist_ok=True)
FIX = ROOT / "tests" / "cli_fixtures"
m = cli.load_matrix(str(FIX / "c3.json"), "int")
v, (mults, adds) = O.ref_sz_c128(m)
(out / "perm_c3.txt").write_text(f"algorithm: store-zechin\nvalue: {O.ref_fmt_value_text(v)}\n"
                                 f"multiplications: {mults}\nadditions: {adds}\n")
(out / "perm_c3.json").write_text(O.ref_fmt_perm_json(v, 3, mults, adds))
(out / "perm_dev4.json").write_text(O.ref_fmt_perm_json(9722, 4, 28, 17))
u = O.ref_haar(6, 7)
(out / "u6_seed7.json").write_text(O.ref_fmt_itf_json(u))
occ, probs = O.ref_full_distribution(u, [0, 2, 3])
(out / "dist_u6_134.txt").write_text("".join("[" + ",".join(map(str, o)) + "] " + ("%.12g" % p) + "\n"
                                             for o, p in zip(occ, probs)))
(out / "dist_u6_134.csv").write_text("pattern,probability\n" + "".join(
    "[" + " ".join(map(str, o)) + "]," + ("%.17g" % p) + "\n" for o, p in zip(occ, probs)))
(out / "dist_u6_134.compact.json").write_text(O.ref_fmt_dist_json(6, 3, occ, probs))
draws = O.ref_sample(u, [0, 2, 3], 50, 9)
(out / "sample_u6_134_50_9.txt").write_text("".join("[" + ",".join(map(str, o)) + "]\n" for o in draws))
(out / "sample_u6_134_50_9.json").write_text(O.ref_fmt_sample_json(draws))
print("wrote", sorted(p.name for p in out.iterdir()))
