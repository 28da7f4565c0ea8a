"""The NCCL form of the multi-GPU plans (paper_1802_02779_b200/sharded.py) on the one GPU of the
box: a one-rank NCCL group runs every collective the plans issue (tests/helpers/nccl_one_rank.py).
The multi-rank logic is covered on CPU with gloo (tests/test_sharding.py) and on the device with
virtual ranks (tests/test_parity_gpu.py)."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_nccl_collectives_on_one_rank():
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "helpers" / "nccl_one_rank.py"), "29633"],
                       capture_output=True, text=True, cwd=ROOT, timeout=240)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    for tag in ("ok allgather_inplace", "ok gather_last_layer", "ok status all_reduce", "ok sharded_permanent",
                "ok int64 overflow", "done"):
        assert tag in out, out
