"""Writes tests/golden/boson.json from the reference engine (oracle/_ref,
compiled from /root/reference sources). Run in the build container:
    python tests/golden/make_boson_goldens.py
Fixtures: enumeration order of (m=25, n=5); a full distribution and 1000
inverse-CDF draws of Haar(6, seed 3) with input modes [0, 1, 4]; the
distribution of Haar(25, seed 2) with input modes 0..4 (the collision-aware
version of config C2's matrices) as SHA-256 of its probabilities."""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402

out = {}
occ = O.ref_enumerate_patterns(25, 5)
out["enumerate_25_5"] = {"count": int(occ.shape[0]), "occupancy_sha256": hashlib.sha256(occ.astype(np.int32).tobytes()).hexdigest()}
u = O.ref_haar(6, 3)
occ, probs = O.ref_full_distribution(u, [0, 1, 4])
draws = O.ref_sample(u, [0, 1, 4], 1000, 3)
index = {tuple(o): i for i, o in enumerate(occ.tolist())}
out["sample_haar6_seed3"] = {
    "modes": 6, "input_modes": [0, 1, 4], "seed": 3, "count": 1000,
    "probabilities_hex": [float(p).hex() for p in probs],
    "indices": [index[tuple(d)] for d in draws.tolist()],
}
u = O.ref_haar(25, 2)
occ, probs = O.ref_full_distribution(u, [0, 1, 2, 3, 4], enumeration_cap=200000)
acc = 0.0
for p in probs.tolist():  # left fold, as OutcomeDistribution::total_probability (boson.cpp:242-248)
    acc += p
out["haar25_seed2_modes0to4"] = {"count": int(probs.shape[0]), "probabilities_sha256": hashlib.sha256(probs.tobytes()).hexdigest(),
                                 "total_probability_hex": acc.hex()}
(ROOT / "tests" / "golden" / "boson.json").write_text(json.dumps(out, indent=1) + "\n")
print("wrote", {k: (v.get("count")) for k, v in out.items()})
