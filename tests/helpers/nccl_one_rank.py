"""The NCCL branches of paper_1802_02779_b200/sharded.py on one B200: a one-rank NCCL process
group (the box has one GPU), every collective the multi-GPU plans issue executed for real on the
device -- the in-place all_gather_into_tensor of a complex layer viewed as float64, the last-layer
gather, the status all-reduce, the barrier that precedes batched P2P -- and the sharded driver end
to end against the oracle. Run by tests/test_sharding_gpu.py in a subprocess (a hung collective
must not hang pytest). Prints "ok" lines; exits non-zero on a mismatch."""
import os
import struct
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1802_02779_b200 import configs  # noqa: E402
from paper_1802_02779_b200 import sharded as S  # noqa: E402


def hexf(x):
    return struct.pack(">d", x).hex()


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", sys.argv[1] if len(sys.argv) > 1 else "29631")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    assert dist.get_backend() == "nccl"
    dist.barrier()
    # equal-slice plan: in-place all-gather of every dtype the layers have (complex as float64 pairs)
    for dtype in (torch.complex128, torch.float64, torch.int64):
        buf = (torch.arange(1000, device="cuda") * 3 + 1).to(dtype)
        if dtype == torch.complex128:
            buf = buf + 1j * torch.arange(1000, device="cuda").to(torch.float64)
        want = buf.clone()
        S.allgather_inplace(buf, 1000, 0, 1)
        torch.cuda.synchronize()
        assert torch.equal(buf, want), dtype
    print("ok allgather_inplace (nccl, in place, c128/f64/i64)")
    # block plan: replicate the last layer (NCCL all_gather_into_tensor into a flat buffer)
    n = 20
    for cplx in (False, True):
        a_np = configs.complex_uniform((n, n), seed=77) if cplx else configs.uniform((n, n), seed=78)
        last = torch.from_numpy(a_np[0].copy()).cuda()
        buf = torch.zeros(64, dtype=last.dtype, device="cuda")
        buf[:n] = last
        S.gather_last_layer(buf, n, 0, 1)
        torch.cuda.synchronize()
        assert torch.equal(buf[:n], last)
    print("ok gather_last_layer (nccl)")
    status = torch.tensor([1], dtype=torch.int32, device="cuda")
    dist.all_reduce(status, op=dist.ReduceOp.MAX)
    assert int(status.item()) == 1
    print("ok status all_reduce MAX (nccl)")
    # the driver end to end on the process group, device layer kernels, bitwise
    for cplx in (False, True):
        a_np = configs.complex_uniform((n, n), seed=79) if cplx else configs.uniform((n, n), seed=80)
        want = complex(O.sz_c128(a_np) if cplx else O.sz_f64(a_np))
        a = torch.from_numpy(a_np).cuda()
        got = complex(S.sharded_permanent(a))
        assert (hexf(got.real), hexf(got.imag)) == (hexf(want.real), hexf(want.imag)), (got, want)
        layer_fn, top_fn = S.device_hooks(a)
        # (the block plan needs world = 2^t >= 2; its exchange is covered by gloo and virtual ranks)
        got = complex(S.sharded_layer_dp(a, 0, 1, layer_fn, top_fn, plan="allgather", status=layer_fn.status))
        assert (hexf(got.real), hexf(got.imag)) == (hexf(want.real), hexf(want.imag)), (got, want)
    print("ok sharded_permanent / sharded_layer_dp on the nccl group (bitwise the oracle)")
    ones = torch.ones((21, 21), dtype=torch.int64, device="cuda")
    try:
        S.sharded_permanent(ones)
    except Exception as e:  # noqa: BLE001
        assert "overflow" in str(e), e
        print("ok int64 overflow raised through the sharded path")
    else:
        raise AssertionError("21! must not fit int64")
    dist.destroy_process_group()
    print("done")


if __name__ == "__main__":
    main()
