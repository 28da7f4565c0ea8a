"""Multi-rank layer sharding (paper_1802_02779_b200/sharded.py) on CPU.

The schedule that runs over NCCL on GPUs (slice every layer into equal padded
colex-rank ranges, compute the own slice, all-gather in place) is executed
here on world_size 2 and 3 gloo process groups, with the CPU oracle's
single-layer step standing in for the device layer kernel, and must reproduce
the unsharded oracle bit for bit. A virtual-rank test covers p = 2, 4, 8 in
one process (memcpy as the all-gather)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1802_02779_b200 import configs
from math import comb

from paper_1802_02779_b200.sharded import (block_plan_applies, layer_slices, max_padded_layer, sharded_layer_dp,
                                           top_block)

_dp = C.POINTER(C.c_double)


def _bind():
    L = O.lib()
    for name in ("orc_sz_layer_step_f64", "orc_sz_layer_step_c128"):
        f = getattr(L, name)
        f.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, C.c_uint64, C.c_uint64]
        f.restype = C.c_int
    for name in ("orc_sz_top_f64", "orc_sz_top_c128"):
        f = getattr(L, name)
        f.argtypes = [C.c_int, _dp, _dp, _dp]
        f.restype = C.c_int
    return L


def _dptr(t: torch.Tensor):
    return C.cast(C.c_void_p(t.data_ptr()), _dp)


def cpu_hooks(a: torch.Tensor):
    L = _bind()
    n = a.shape[0]
    cplx = a.is_complex()
    step = L.orc_sz_layer_step_c128 if cplx else L.orc_sz_layer_step_f64
    top = L.orc_sz_top_c128 if cplx else L.orc_sz_top_f64

    def layer_fn(k, prev, cur, r0, r1):
        assert step(n, _dptr(a), k, _dptr(prev), _dptr(cur), r0, r1) == 0

    def top_fn(a_, last):
        out = torch.zeros(2, dtype=torch.float64)
        assert top(n, _dptr(a_), _dptr(last), _dptr(out)) == 0
        return complex(out[0], out[1]) if cplx else float(out[0])

    return layer_fn, top_fn


def cpu_overlap_hooks(a: torch.Tensor, rank: int, world: int):
    """CPU stand-ins of pl_shard_block_partial / pl_shard_block_top_terms (oracle C code)."""
    L = _bind()
    n = a.shape[0]
    cplx = a.is_complex()
    _i32p, _u64p = C.POINTER(C.c_int), C.POINTER(C.c_uint64)
    part = L.orc_sz_layer_partial_c128 if cplx else L.orc_sz_layer_partial_f64
    part.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, C.c_uint64, C.c_uint64, C.c_int]
    tt = L.orc_sz_top_terms_c128 if cplx else L.orc_sz_top_terms_f64
    tt.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp, C.c_uint64, C.c_uint64, C.c_int, _i32p, _u64p, C.c_int]
    t = world.bit_length() - 1

    def partial_fn(k, prev, cur):
        r0, r1 = top_block(n, k, world, rank)
        assert part(n, _dptr(a), k, _dptr(prev), _dptr(cur), r0, r1, n - t) == 0

    def top_terms_fn(k, prev, cur):
        r0, r1 = top_block(n, k, world, rank)
        bits = [i for i in range(t) if rank >> i & 1]
        cols = (C.c_int * 8)(*[n - t + i for i in bits])
        bases = (C.c_uint64 * 8)(*[top_block(n, k - 1, world, rank & ~(1 << i))[0] for i in bits])
        assert tt(n, _dptr(a), k, _dptr(prev), _dptr(cur), r0, r1 - r0, len(bits), cols, bases,
                  int(k == len(bits))) == 0

    return partial_fn, top_terms_fn


def test_layer_slices_cover_exactly():
    for n in (5, 9, 26, 32):
        for world in (1, 2, 3, 4, 8):
            for k in range(2, n):
                per, sl = layer_slices(n, k, world)
                covered = [r for r0, r1 in sl for r in range(r0, r1)] if n <= 9 else None
                if covered is not None:
                    assert covered == list(range(len(covered)))
                assert sl[0][0] == 0 and sl[-1][1] == __import__("math").comb(n, k)
                assert all(sl[g][1] == sl[g + 1][0] for g in range(world - 1))
                assert per * world >= sl[-1][1]
            assert max_padded_layer(n, world) >= max(__import__("math").comb(n, k) for k in range(2, n))


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("cplx", [False, True])
def test_virtual_ranks_bitwise(world, cplx):
    n = 11
    a_np = configs.complex_uniform((n, n), seed=7) if cplx else configs.uniform((n, n), seed=7)
    a = torch.from_numpy(a_np)
    layer_fn, top_fn = cpu_hooks(a)
    size = max_padded_layer(n, world)
    replicas = [[torch.zeros(size, dtype=a.dtype) for _ in range(2)] for _ in range(world)]
    for k in range(2, n):
        per, sl = layer_slices(n, k, world)
        for g in range(world):
            prev, cur = replicas[g]
            layer_fn(k, prev, cur, *sl[g])
        for g in range(world):  # all-gather by memcpy
            for h in range(world):
                replicas[g][1][h * per:(h + 1) * per] = replicas[h][1][h * per:(h + 1) * per]
        for g in range(world):
            replicas[g].reverse()
    values = {top_fn(a, replicas[g][0]) for g in range(world)}
    want = O.sz_c128(a_np) if cplx else O.sz_f64(a_np)
    assert values == {want}


def test_top_blocks_tile_every_layer():
    for n in (5, 9, 12, 26, 32, 34):
        for world in (2, 4, 8, 16):
            if not block_plan_applies(n, world):
                continue
            for k in range(2, n):
                blocks = sorted(b for b in (top_block(n, k, world, g) for g in range(world)) if b[1] > b[0])
                assert blocks[0][0] == 0 and blocks[-1][1] == comb(n, k)
                assert all(blocks[i][1] == blocks[i + 1][0] for i in range(len(blocks) - 1))


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("cplx", [False, True])
def test_virtual_ranks_top_blocks_bitwise(world, cplx):
    # each rank computes only its block and only receives the blocks with one
    # top column less: a rank must never read a predecessor it was not sent
    n = 11
    t = world.bit_length() - 1
    a_np = configs.complex_uniform((n, n), seed=17) if cplx else configs.uniform((n, n), seed=17)
    a = torch.from_numpy(a_np)
    layer_fn, top_fn = cpu_hooks(a)
    size = max(comb(n, k) for k in range(2, n)) + 4
    nan = complex("nan") if cplx else float("nan")
    replicas = [[torch.full((size,), nan, dtype=a.dtype) for _ in range(2)] for _ in range(world)]
    for k in range(2, n):
        for g in range(world):
            prev, cur = replicas[g]
            cur.fill_(nan)  # whatever this rank does not own or receive stays NaN
            r0, r1 = top_block(n, k, world, g)
            if r1 > r0:
                layer_fn(k, prev, cur, r0, r1)
        if k < n - 1:
            for g in range(world):  # point-to-point: g receives from g & ~2^i
                for i in range(t):
                    if g >> i & 1:
                        h = g ^ (1 << i)
                        h0, h1 = top_block(n, k, world, h)
                        replicas[g][1][h0:h1] = replicas[h][1][h0:h1]
        for g in range(world):
            replicas[g].reverse()
    want = O.sz_c128(a_np) if cplx else O.sz_f64(a_np)
    for g in range(world):
        last = replicas[g][0].clone()
        for h in range(world):  # the final gather of layer n-1
            h0, h1 = top_block(n, n - 1, world, h)
            last[h0:h1] = replicas[h][0][h0:h1]
        assert top_fn(a, last) == want


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, cplx, q, overlap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a_np = configs.complex_uniform((n, n), seed=31) if cplx else configs.uniform((n, n), seed=31)
        a = torch.from_numpy(a_np)
        layer_fn, top_fn = cpu_hooks(a)
        pf = tf = None
        if overlap:
            pf, tf = cpu_overlap_hooks(a, rank, world)
        v = sharded_layer_dp(a, rank, world, layer_fn, top_fn, partial_fn=pf, top_terms_fn=tf)
        q.put((rank, v))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])  # 2, 4: top-column blocks; 3: all-gather
@pytest.mark.parametrize("cplx", [False, True])
def test_gloo_sharded_dp_bitwise(world, cplx):
    n = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, cplx, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a_np = configs.complex_uniform((n, n), seed=31) if cplx else configs.uniform((n, n), seed=31)
    want = O.sz_c128(a_np) if cplx else O.sz_f64(a_np)
    assert set(results.values()) == {want}


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("cplx", [False, True])
def test_gloo_overlapped_block_plan_bitwise(world, cplx):
    # the exchange of layer k-1 in flight while layer k is computed without its
    # top-column terms, which are added once the blocks have landed
    n = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, cplx, q, True)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a_np = configs.complex_uniform((n, n), seed=31) if cplx else configs.uniform((n, n), seed=31)
    want = O.sz_c128(a_np) if cplx else O.sz_f64(a_np)
    assert set(results.values()) == {want}


def _overflow_worker(rank, world, port, n, bad_rank, plan, q):
    """Rank `bad_rank`'s layer step flags an int64 overflow in its own status
    word; every rank must raise (the status is combined over the group
    before the top level), none may return a value."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = torch.from_numpy(configs.uniform((n, n), seed=5))
        layer_fn, _ = cpu_hooks(a)
        status = torch.zeros(1, dtype=torch.int32)

        def flagged_layer(k, prev, cur, r0, r1):
            layer_fn(k, prev, cur, r0, r1)
            if rank == bad_rank and k == n // 2:
                status[0] |= 1  # what the device layer kernel does on an actual overflow

        def top_fn(a_, last):
            if int(status[0]) & 1:
                return "overflow"
            return "value"

        q.put((rank, sharded_layer_dp(a, rank, world, flagged_layer, top_fn, plan=plan, status=status)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,plan", [(2, "blocks"), (3, "allgather"), (4, "blocks")])
def test_gloo_overflow_status_combined_over_ranks(world, plan):
    n = 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overflow_worker, args=(r, world, port, n, world - 1, plan, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert set(results.values()) == {"overflow"}


# ---------------------------------------------------------------- the C ABI's single-process plans

def _c_plan(n, world, rank, k):
    import ctypes as C
    from paper_1802_02779_b200 import _native as N

    r0, r1 = C.c_uint64(), C.c_uint64()
    assert N.lib.pl_shard_range(n, world, rank, k, C.byref(r0), C.byref(r1)) == 0
    cnt = N.lib.pl_shard_exchange(n, world, rank, k, None, 0)
    buf = (C.c_uint64 * (4 * max(cnt, 1)))()
    assert N.lib.pl_shard_exchange(n, world, rank, k, buf, cnt) == cnt
    ops = [("recv" if buf[4 * i] else "send", int(buf[4 * i + 1]), int(buf[4 * i + 2]), int(buf[4 * i + 3]))
           for i in range(cnt)]
    return (int(r0.value), int(r1.value)), ops


def _py_exchange(n, k, rank, world):
    """The schedule sharded.exchange_blocks / gather_last_layer run, as a list."""
    from paper_1802_02779_b200.sharded import top_columns

    t = top_columns(world)
    ops = []
    if k < n - 1:
        for i in range(t):
            partner = rank ^ (1 << i)
            if rank >> i & 1:
                r0, r1 = top_block(n, k, world, partner)
                if r1 > r0:
                    ops.append(("recv", partner, r0, r1))
            else:
                r0, r1 = top_block(n, k, world, rank)
                if r1 > r0:
                    ops.append(("send", partner, r0, r1))
    else:  # layer n-1 to rank 0 (the C path's top level runs on device 0)
        for h in range(1, world):
            r0, r1 = top_block(n, k, world, h)
            if r1 > r0:
                if rank == 0:
                    ops.append(("recv", h, r0, r1))
                if rank == h:
                    ops.append(("send", 0, r0, r1))
    return ops


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 8, 16])
def test_c_abi_shard_plan_matches_sharded_py(world):
    """pl_shard_* (the single-process NCCL path of pl_sz_permanent_multi) use
    the same ranges and point-to-point schedule as sharded.py; every output
    is owned by exactly one rank and every received block is sent by its
    owner."""
    from paper_1802_02779_b200 import _native as N

    for n in (5, 9, 12, 20, 26, 32):
        blocks = block_plan_applies(n, world)
        assert N.lib.pl_shard_plan(n, world) == (N.PL_SHARD_BLOCKS if blocks else N.PL_SHARD_ALLGATHER)
        for k in range(2, n):
            owned = []
            sends, recvs = set(), set()
            for rank in range(world):
                rng, ops = _c_plan(n, world, rank, k)
                want = top_block(n, k, world, rank) if blocks else layer_slices(n, k, world)[1][rank]
                assert rng == tuple(want)
                if rng[1] > rng[0]:
                    owned.append(rng)
                if blocks:
                    assert ops == _py_exchange(n, k, rank, world)
                    for kind, peer, r0, r1 in ops:
                        (sends if kind == "send" else recvs).add((rank, peer, r0, r1) if kind == "send" else
                                                                 (peer, rank, r0, r1))
                else:
                    assert ops == []
            owned.sort()
            assert owned[0][0] == 0 and owned[-1][1] == comb(n, k)
            assert all(owned[i][1] == owned[i + 1][0] for i in range(len(owned) - 1))
            assert sends == recvs
