"""Device parity: the CUDA path (through the C ABI) against the oracle on the
same seeded inputs, at the BASELINE.json config sizes and at edge cases.

Bars (BASELINE.json north_star): int64 bit-exact; float64 / complex128 within
relative 1e-9 — and, in the default (non-FMA) mode, bitwise equal to the
oracle, which is bitwise the reference engine (tests/test_oracle.py)."""
import ctypes as C
import math
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import _native as N
from paper_1802_02779_b200 import configs

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REL_TOL = 1e-9  # north_star: relative error <= 1e-9 in fp64 / complex128 (no absolute floor)


def hexf(x):
    return struct.pack(">d", x).hex()


def rel_err(got, want):
    got, want = np.asarray(got), np.asarray(want)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)))


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if pl.device_count() == 0:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


# ---------------------------------------------------------------- configs

def test_c1_bit_exact(goldens):
    a = configs.c1()
    out = pl.store_zechin_permanent_batch(a)
    assert out.dtype == np.int64
    assert configs.sha256(out) == goldens["c1"]["output_sha256"]
    assert np.array_equal(out, O.sz_batch(a))


@pytest.mark.parametrize("fma", [False, True])
def test_c2_complex(goldens, fma):
    a = configs.c2()
    out = pl.store_zechin_permanent_batch(a, fma=fma)
    want = O.sz_batch(a)
    assert rel_err(out, want) <= REL_TOL
    if not fma:
        assert configs.sha256(out) == goldens["c2"]["output_sha256"]


@pytest.mark.parametrize("dtype,count", [("c128", 200_003), ("i64", 350_017)])
def test_pipelined_batch_kernel(dtype, count):
    # inputs of >= 64 MiB take the pipelined n = 5 kernel (one CTA per SM, producer
    # warp + ring); odd counts exercise the remainder path of the last CTA
    if dtype == "c128":
        a = configs.complex_uniform((count, 5, 5), seed=9)
    else:
        a = configs.int_matrices(5, count, seed=9)
    assert a.nbytes >= 64 << 20
    out = pl.store_zechin_permanent_batch(a)
    assert np.array_equal(out, O.sz_batch(a))


def test_c3_bit_exact(goldens):
    a = configs.c3()
    out = pl.store_zechin_permanent_batch(a)
    assert configs.sha256(out) == goldens["c3"]["output_sha256"]


@pytest.mark.parametrize("fma", [False, True])
def test_c4_float64(goldens, fma):
    a = configs.c4()
    v = pl.store_zechin_permanent(a, fma=fma).value
    assert rel_err(v, goldens["c4"]["value"]) <= REL_TOL
    if not fma:
        assert hexf(v) == goldens["c4"]["value_hex"] == goldens["c4"]["reference_value_hex"]


@pytest.mark.parametrize("fma", [False, True])
def test_c5_complex128(goldens, fma):
    a = configs.c5()
    assert configs.sha256(a) == goldens["c5"]["input_sha256"]
    v = pl.store_zechin_permanent(a, fma=fma).value
    want = complex(*goldens["c5"]["value"])
    assert abs(v - want) <= REL_TOL * abs(want)  # pure relative: |per| ~ 3e-32
    if not fma:
        assert [hexf(v.real), hexf(v.imag)] == goldens["c5"]["value_hex"]


# ---------------------------------------------------------------- orders / rings

@pytest.mark.parametrize("n", list(range(1, 21)))
def test_int_orders_vs_oracle(n):
    count = 64 if n <= 12 else (4 if n <= 16 else 1)
    lo, hi = (-9, 9) if n <= 10 else (-1, 2)
    a = configs.int_matrices(n, count, seed=1000 + n, lo=lo, hi=hi)
    out = pl.store_zechin_permanent_batch(a)
    assert np.array_equal(out, O.sz_batch(a))


@pytest.mark.parametrize("n,h", [(6, 300), (8, 100), (9, 40), (11, 12)])
def test_int_orders_checked_paths(n, h):
    # entries up to +-h: the guard bound exceeds 2^53, so the batch kernels take
    # the int64 / checked-int64 paths instead of exact doubles (every true value
    # fits int64 for these seeds)
    a = configs.int_matrices(n, 96, seed=4000 + n, lo=-h, hi=h)
    out = pl.store_zechin_permanent_batch(a)
    assert np.array_equal(out, O.sz_batch(a))


@pytest.mark.parametrize("n", list(range(1, 21)) + [23, 24])
def test_complex_orders_bitwise(n):
    count = 33 if n <= 12 else (3 if n <= 16 else 1)
    a = configs.complex_uniform((count, n, n), seed=2000 + n)
    out = pl.store_zechin_permanent_batch(a)
    want = O.sz_batch(a)
    assert np.array_equal(out.view(np.uint64), want.view(np.uint64))
    out_f = pl.store_zechin_permanent_batch(a, fma=True)
    assert rel_err(out_f, want) <= REL_TOL


@pytest.mark.parametrize("n", [1, 2, 3, 6, 7, 9, 13, 15, 16, 17, 22])
def test_float_orders_bitwise(n):
    count = 17 if n <= 13 else 2
    a = configs.uniform((count, n, n), seed=3000 + n)
    out = pl.store_zechin_permanent_batch(a)
    assert np.array_equal(out.view(np.uint64), O.sz_batch(a).view(np.uint64))


# ---------------------------------------------------------------- edge cases

def test_empty_and_ragged_batches():
    for dt in (np.int64, np.float64, np.complex128):
        assert pl.store_zechin_permanent_batch(np.zeros((0, 5, 5), dtype=dt)).shape == (0,)
    for count in (1, 31, 127, 129, 1000):  # CTA tails of the batched kernels
        for n in (5, 8):
            a = configs.int_matrices(n, count, seed=count + n)
            assert np.array_equal(pl.store_zechin_permanent_batch(a), O.sz_batch(a))


@pytest.mark.parametrize("dt", [np.int64, np.float64, np.complex128])
def test_small_orders_batches_tails_and_alignment(dt):
    # n <= 5 stage whole 32-matrix batches through shared memory by TMA; tails and
    # inputs that are not 16-byte aligned take the direct path
    import torch

    for n in (1, 2, 3, 4, 5):
        for count in (1, 32, 33, 95, 4097):
            if dt is np.int64:
                a = configs.int_matrices(n, count + 1, seed=n * 131 + count)
            else:
                a = configs.uniform((count + 1, n, n), seed=n * 131 + count).astype(dt)
                if dt is np.complex128:
                    a = a + 1j * configs.uniform((count + 1, n, n), seed=n * 7 + count)
            want = O.sz_batch(a)
            got = pl.store_zechin_permanent_batch(a[1:])
            assert np.array_equal(np.asarray(got).view(np.uint64), want[1:].view(np.uint64)), (n, count)
            # device tensor viewed one matrix in: 16-byte aligned only when n^2 * size is
            t = torch.from_numpy(a).cuda()
            out = torch.empty(count, dtype=t.dtype, device="cuda")
            pl.store_zechin_permanent_batch(t[1:], out=out)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), want[1:].view(np.uint64)), (n, count, "dev")


def test_reference_goldens_on_device():
    dev4 = np.array([7, 0, 1, 2, 5, 3, 4, 5, 3, 5, 6, 7, 1, 7, 8, 9]).reshape(4, 4)
    assert pl.store_zechin_permanent(dev4).value == 9722
    assert pl.store_zechin_permanent(np.array([[42]])).value == 42
    r = pl.store_zechin_permanent(np.array([[2, 3], [5, 7]]))
    assert (r.value, r.counts) == (29, pl.OpCount(2, 1))
    run = pl.store_zechin_run(np.ones((8, 8), dtype=np.int64))
    assert run.result.value == math.factorial(8)
    assert run.cache_misses == run.distinct_subsets == 2 ** 8 - 8 - 2


def test_int64_overflow_guard():
    # every intermediate fits: the checked path computes it exactly (20! < 2^63)
    assert pl.store_zechin_permanent(np.ones((20, 20), dtype=np.int64)).value == math.factorial(20)
    # 21! > 2^63 (layer path), 5! 10^20 (register kernel), 9! 10^27 (shared-memory kernel): never wrap.
    # The C ABI's int64 entry point reports it; the single-matrix Python call then returns the exact
    # integer through the residue passes (tests/test_bigint_gpu.py), int64 batches raise.
    ones21 = np.ones((21, 21), dtype=np.int64)
    out = np.zeros(1, dtype=np.int64)
    lim = pl.Limits().to_c()
    assert N.lib.pl_sz_permanent(N.PL_I64, 21, ones21.ctypes.data, out.ctypes.data, 0, C.byref(lim),
                                 None) == N.PL_ERR_OVERFLOW
    assert pl.store_zechin_permanent(ones21).value == math.factorial(21)
    with pytest.raises(pl.DomainError, match="overflow"):
        pl.store_zechin_permanent_batch(np.full((3, 5, 5), 10 ** 4, dtype=np.int64))
    with pytest.raises(pl.DomainError, match="overflow"):
        pl.store_zechin_permanent_batch(np.full((3, 9, 9), 10 ** 3, dtype=np.int64))
    # batches of large orders (one lean launch per layer for the whole batch): the
    # overflowing member is reported, the others' checked / exact paths stay exact
    with pytest.raises(pl.DomainError, match="overflow"):
        pl.store_zechin_permanent_batch(np.stack([np.eye(21, dtype=np.int64), np.ones((21, 21), dtype=np.int64)]))
    b = np.stack([np.ones((20, 20), dtype=np.int64), np.eye(20, dtype=np.int64) * 2])
    assert pl.store_zechin_permanent_batch(b).tolist() == [math.factorial(20), 2 ** 20]
    # INT64_MIN entry can never be exact-negated: guard -> checked path
    a = np.zeros((3, 3), dtype=np.int64)
    a[0, 0] = np.iinfo(np.int64).min
    a[1, 1] = a[2, 2] = 1
    assert pl.store_zechin_permanent(a).value == int(np.iinfo(np.int64).min)


def test_zero_rows_and_signed_zero():
    a = configs.uniform((7, 7), seed=9)
    a[3] = 0.0
    assert pl.store_zechin_permanent(a).value == O.sz_f64(a)
    z = -np.zeros((6, 6))
    assert hexf(pl.store_zechin_permanent(z).value) == hexf(O.sz_f64(z))


# ---------------------------------------------------------------- size-independent properties at full size

def test_c4_permutation_and_transpose_invariance():
    a = configs.c4()
    base = pl.store_zechin_permanent(a).value
    rng = np.random.default_rng(4)
    p = a[rng.permutation(26)][:, rng.permutation(26)]
    assert rel_err(pl.store_zechin_permanent(p).value, base) <= REL_TOL
    assert rel_err(pl.store_zechin_permanent(a.T.copy()).value, base) <= REL_TOL


def test_c5_repeatable(goldens):
    # every run of the layer DP is bitwise the same (regression: a missing
    # generic -> async proxy fence after the PDL wait let ~1 in 8 runs read
    # stale layer entries, sz_ws.cuh)
    a = configs.c5()
    want = complex(*goldens["c5"]["value"])
    vals = {complex(pl.store_zechin_permanent(a).value) for _ in range(8)}
    assert len(vals) == 1
    assert abs(vals.pop() - want) <= REL_TOL * abs(want)


def test_c5_row_linearity():
    a = configs.c5()
    x = configs.complex_uniform((32,), seed=77) * 1e-2
    b, c = a.copy(), a.copy()
    b[31] = x
    c[31] = a[31] - x
    pa, pb, pc = (pl.store_zechin_permanent(m, fma=True).value for m in (a, b, c))
    assert abs(pb + pc - pa) <= 1e-9 * max(abs(pa), abs(pb), abs(pc))


@pytest.mark.parametrize("n,cplx", [(33, False), (34, True)])
def test_max_orders_power_of_two_scaling_bitwise(n, cplx):
    # the order cap (n = 34, C(34,17) < 2^32 colex ranks): scaling one row by 2 scales
    # every partial sum touching it by 2 exactly, so the permanent doubles bit for bit;
    # a row swap leaves the result unchanged up to summation order (<= 1e-9)
    a = configs.uniform((n, n), seed=n) * 0.3
    if cplx:
        a = a + 1j * configs.uniform((n, n), seed=n + 1) * 0.3
    b = a.copy()
    b[n // 2] *= 2.0
    pa = complex(pl.store_zechin_permanent(a).value)
    pb = complex(pl.store_zechin_permanent(b).value)
    assert (hexf(pb.real), hexf(pb.imag)) == (hexf(2 * pa.real), hexf(2 * pa.imag))
    c = a[:, ::-1].copy()  # column reversal: a different summation order, same value
    pc = complex(pl.store_zechin_permanent(c).value)
    assert abs(pc - pa) <= 1e-9 * abs(pa)


# ---------------------------------------------------------------- device pointers / layer primitives

def test_torch_device_batch_and_async_status():
    import torch

    a = configs.c3(2000)
    want = O.sz_batch(a)
    ad = torch.from_numpy(a).cuda()
    out = pl.store_zechin_permanent_batch(ad)
    assert np.array_equal(out.cpu().numpy(), want)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out2 = pl.store_zechin_permanent_batch(ad, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0 and np.array_equal(out2.cpu().numpy(), want)
    bad = torch.full((4, 9, 9), 10 ** 17, dtype=torch.int64, device="cuda")
    pl.store_zechin_permanent_batch(bad, status=status)
    torch.cuda.synchronize()
    assert int(status.item()) & 1
    pin = torch.from_numpy(configs.c2(500)).pin_memory()
    out3 = pl.store_zechin_permanent_batch(pin)
    assert np.array_equal(out3.numpy().view(np.uint64), O.sz_batch(pin.numpy()).view(np.uint64))


def test_layer_primitive_ranges_match_oracle():
    import torch

    from paper_1802_02779_b200.sharded import device_hooks, layer_slices, sharded_layer_dp

    n = 14
    a_np = configs.uniform((n, n), seed=123)
    a = torch.from_numpy(a_np).cuda()
    layer_fn, top_fn = device_hooks(a)
    prev = torch.zeros(4000, dtype=a.dtype, device="cuda")
    cur = torch.zeros_like(prev)
    for k in range(2, n):
        full = torch.from_numpy(O.sz_layer_f64(a_np, k)).cuda()
        if k > 2:
            src = torch.from_numpy(O.sz_layer_f64(a_np, k - 1)).cuda()
            prev[: src.numel()] = src
        for world in (1, 3):
            _, sl = layer_slices(n, k, world)
            for r0, r1 in sl:  # every rank's slice, one at a time
                cur.zero_()
                layer_fn(k, prev, cur, r0, r1)
                assert torch.equal(cur[r0:r1], full[r0:r1])
    v = sharded_layer_dp(a, 0, 1, layer_fn, top_fn)
    assert hexf(v) == hexf(O.sz_f64(a_np))


def test_layer_slices_large_order_bitwise():
    # rank slices that cut tiles anywhere (world 2, 5, 8) through the tiled layer kernel
    import torch

    from paper_1802_02779_b200.sharded import device_hooks, layer_slices

    n = 22
    a_np = configs.uniform((n, n), seed=2222)
    a = torch.from_numpy(a_np).cuda()
    layer_fn, _ = device_hooks(a)
    size = O.binom(n, n // 2) + 64
    prev = torch.zeros(size, dtype=a.dtype, device="cuda")
    cur = torch.zeros_like(prev)
    for k in (3, 8, 11, 15, 20):
        full = torch.from_numpy(O.sz_layer_f64(a_np, k)).cuda()
        src = torch.from_numpy(O.sz_layer_f64(a_np, k - 1)).cuda()
        prev[: src.numel()] = src
        for world in (2, 5, 8):
            _, sl = layer_slices(n, k, world)
            cur.zero_()
            for r0, r1 in sl:
                layer_fn(k, prev, cur, r0, r1)
            assert torch.equal(cur[: full.numel()], full), (k, world)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("cplx", [False, True])
def test_top_block_plan_on_device_virtual_ranks(world, cplx):
    # the multi-GPU top-column plan with the device layer kernel: each virtual
    # rank holds only its block and the blocks it receives (everything else NaN)
    import torch
    from math import comb

    from paper_1802_02779_b200.sharded import device_hooks, top_block

    n = 20
    t = world.bit_length() - 1
    a_np = configs.complex_uniform((n, n), seed=20 + world) if cplx else configs.uniform((n, n), seed=20 + world)
    a = torch.from_numpy(a_np).cuda()
    layer_fn, top_fn = device_hooks(a)
    size = max(comb(n, k) for k in range(2, n)) + 64
    nan = complex("nan") if cplx else float("nan")
    reps = [[torch.full((size,), nan, dtype=a.dtype, device="cuda") for _ in range(2)] for _ in range(world)]
    for k in range(2, n):
        for g in range(world):
            prev, cur = reps[g]
            cur.fill_(nan)
            r0, r1 = top_block(n, k, world, g)
            if r1 > r0:
                layer_fn(k, prev, cur, r0, r1)
        if k < n - 1:
            for g in range(world):
                for i in range(t):
                    if g >> i & 1:
                        h = g ^ (1 << i)
                        h0, h1 = top_block(n, k, world, h)
                        reps[g][1][h0:h1] = reps[h][1][h0:h1]
        for g in range(world):
            reps[g].reverse()
    want = O.sz_c128(a_np) if cplx else O.sz_f64(a_np)
    last = reps[0][0].clone()
    for h in range(world):
        h0, h1 = top_block(n, n - 1, world, h)
        last[h0:h1] = reps[h][0][h0:h1]
    got = complex(top_fn(a, last))
    want = complex(want)
    assert (hexf(got.real), hexf(got.imag)) == (hexf(want.real), hexf(want.imag))


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("cplx", [False, True])
def test_overlapped_block_plan_on_device_virtual_ranks(world, cplx):
    # the overlapped form (pl_shard_block_partial, then pl_shard_block_top_terms
    # once the blocks P \ {c} of layer k-1 have "arrived"): the partial step
    # runs BEFORE the exchange copies (the received regions are NaN when it
    # runs, so reading them would show), the top terms after; bitwise the
    # oracle. Both the lean (small layers) and ws (large layers) kernels cut.
    import torch
    from math import comb

    from paper_1802_02779_b200.sharded import device_hooks, device_overlap_hooks, top_block

    n = 24
    t = world.bit_length() - 1
    a_np = configs.complex_uniform((n, n), seed=40 + world) if cplx else configs.uniform((n, n), seed=40 + world)
    a = torch.from_numpy(a_np).cuda()
    layer_fn, top_fn = device_hooks(a)
    hooks = [device_overlap_hooks(a, layer_fn, g, world) for g in range(world)]
    size = max(comb(n, k) for k in range(2, n)) + 64
    nan = complex("nan") if cplx else float("nan")
    reps = [[torch.full((size,), nan, dtype=a.dtype, device="cuda") for _ in range(2)] for _ in range(world)]
    for k in range(2, n):
        for g in range(world):
            prev, cur = reps[g]
            cur.fill_(nan)
            r0, r1 = top_block(n, k, world, g)
            if k == 2:
                if r1 > r0:
                    layer_fn(k, prev, cur, r0, r1)
            elif r1 > r0:
                hooks[g][0](k, prev, cur)  # partial: own block of layer k-1 only
        if k >= 3:
            # the exchange of layer k-1 lands now, then the top-column terms
            for g in range(world):
                for i in range(t):
                    if g >> i & 1:
                        h = g ^ (1 << i)
                        h0, h1 = top_block(n, k - 1, world, h)
                        reps[g][0][h0:h1] = reps[h][0][h0:h1]
            for g in range(world):
                r0, r1 = top_block(n, k, world, g)
                if r1 > r0:
                    hooks[g][1](k, reps[g][0], reps[g][1])
        for g in range(world):
            reps[g].reverse()
    want = O.sz_c128(a_np) if cplx else O.sz_f64(a_np)
    last = reps[0][0].clone()
    for h in range(world):
        h0, h1 = top_block(n, n - 1, world, h)
        last[h0:h1] = reps[h][0][h0:h1]
    got = complex(top_fn(a, last))
    want = complex(want)
    assert (hexf(got.real), hexf(got.imag)) == (hexf(want.real), hexf(want.imag))


def test_cpp_device_suite():
    exe = ROOT / "tests" / "cpp" / "test_permanent_device"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr


def test_concurrent_host_threads():
    # the entry points are reentrant (reference SPEC: pure, no global state): host
    # threads calling at once get the same results as serial calls
    import threading

    jobs = [configs.c1(3000, seed=s) for s in (11, 12)] + [configs.complex_uniform((64, 9, 9), seed=13),
                                                           configs.complex_uniform((1, 21, 21), seed=14)]
    want = [O.sz_batch(a) for a in jobs]
    got = [None] * len(jobs)
    errs = []

    def work(i):
        try:
            for _ in range(3):
                got[i] = pl.store_zechin_permanent_batch(jobs[i])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs
    for g, w in zip(got, want):
        assert np.array_equal(g.view(np.uint64) if g.dtype == np.complex128 else g,
                              w.view(np.uint64) if w.dtype == np.complex128 else w)


@pytest.mark.parametrize("n", [10, 12, 14])
def test_pair_kernel_mixed_modes_and_odd_counts(n):
    # the pair kernel runs two matrices in lockstep when their int64 guards agree and
    # one at a time otherwise; alternate small (exact-in-double) and larger entries
    # (int64 / checked paths) and leave an odd matrix at the end
    small = configs.int_matrices(n, 9, seed=5000 + n, lo=0, hi=1)
    h = {10: 20, 12: 15, 14: 8}[n]  # guard bounds above 2^53: the int64 / checked-int64 paths
    big = configs.int_matrices(n, 8, seed=6000 + n, lo=-h, hi=h)
    a = np.empty((17, n, n), dtype=np.int64)
    a[0::2], a[1::2] = small, big
    try:
        want = O.sz_batch(a)
    except Exception:  # pragma: no cover
        pytest.skip("oracle overflow")
    if np.any(np.abs(want.astype(object)) >= 2 ** 63):  # pragma: no cover
        pytest.skip("values beyond int64")
    assert np.array_equal(pl.store_zechin_permanent_batch(a), want)
    f = configs.uniform((17, n, n), seed=7000 + n)
    assert np.array_equal(pl.store_zechin_permanent_batch(f).view(np.uint64), O.sz_batch(f).view(np.uint64))


@pytest.mark.parametrize("n", [10, 11, 12, 13, 14])
def test_f32_pack_kernel_paths(n):
    # int64 10 <= n <= 14: packs of four run on the FP32 pipe when every member's
    # bound (row sums, or Bregman's for 0/1 matrices) is below 2^24; mix in
    # all-ones (Bregman 12! > 2^24 at n >= 11: the double path), 0/1 matrices with
    # one entry 2 (not 0/1, row-sum bound over 2^24) and a count that leaves a
    # partial pack
    count = 4 * 9 + 3
    a = configs.int_matrices(n, count, seed=8100 + n, lo=0, hi=1)
    a[5] = 1
    a[9, 3, 4] = 2
    a[22] = np.eye(n, dtype=np.int64) * 3
    want = O.sz_batch(a)
    assert np.array_equal(pl.store_zechin_permanent_batch(a), want)


@pytest.mark.parametrize("n", [10, 12, 14])
def test_f32_pack_byte_coefficients(n):
    # FP32-exact packs whose entries all fit a signed byte read their coefficient packs as
    # one word of four biased bytes (smem_dp_f32c); a pack with an entry outside
    # [-128, 127] keeps the 16-byte coefficient packs. Sparse matrices keep the row-sum
    # bound below 2^24 with entries at the byte limits; a ragged tail runs member by member.
    rng = np.random.default_rng(8300 + n)
    count = 4 * 8 + 2
    a = np.zeros((count, n, n), dtype=np.int64)
    for b in range(count):
        p = rng.permutation(n)
        a[b, np.arange(n), p] = rng.integers(1, 3, n)  # a permutation pattern: one term, product <= 2^n
        a[b, rng.integers(0, n), rng.integers(0, n)] += 1
    a[4, 0, np.argmax(a[4, 0])] = 127
    a[5, 1, np.argmax(a[5, 1])] = -128
    a[8, 2, np.argmax(a[8, 2])] = 128   # outside a byte: this pack takes the float4 coefficient path
    a[13, 3, np.argmax(a[13, 3])] = -129
    a[16:20] = configs.int_matrices(n, 4, seed=8400 + n, lo=-1, hi=2)  # small mixed signs
    want = O.sz_batch(a)
    assert np.array_equal(pl.store_zechin_permanent_batch(a), want)


@pytest.mark.parametrize("n", [15, 17, 20, 22])
def test_large_order_batches_one_launch_per_layer(n):
    # batches of 15 <= n <= ~22 run every layer of a group of matrices in one lean
    # launch (tiles of all the group's matrices); compare with the oracle per
    # ring, with an int64 member that needs the checked path and a tail group
    rng = np.random.default_rng(9100 + n)
    count = 5
    c = rng.standard_normal((count, n, n)) + 1j * rng.standard_normal((count, n, n))
    assert np.array_equal(pl.store_zechin_permanent_batch(c).view(np.uint64), O.sz_batch(c).view(np.uint64))
    f = rng.uniform(-1, 1, (count, n, n))
    assert np.array_equal(pl.store_zechin_permanent_batch(f).view(np.uint64), O.sz_batch(f).view(np.uint64))
    i = rng.integers(0, 2, (count, n, n)).astype(np.int64)
    i[2] = rng.integers(-3, 4, (n, n))  # guard bound above 2^63: checked int64
    want = O.sz_batch(i)
    assert np.array_equal(pl.store_zechin_permanent_batch(i), want)


def test_large_order_batch_groups():
    # several groups (PL_BATCH_SCRATCH_MB=1 forces tiny groups) and the per-matrix path agree
    n = 16
    a = np.random.default_rng(9200).standard_normal((7, n, n)) + 0j
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); import paper_1802_02779_b200 as pl; "
        "a = np.load(sys.argv[1]); np.save(sys.argv[2], pl.store_zechin_permanent_batch(a))" % str(ROOT))
    import os
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        np.save(os.path.join(d, "a.npy"), a)
        outs = []
        for env in ({"PL_BATCH_SCRATCH_MB": "1"}, {"PL_BATCH_LAYERS": "0"}):
            p = os.path.join(d, "o%d.npy" % len(outs))
            subprocess.run(["python", "-c", code, os.path.join(d, "a.npy"), p], check=True,
                           env={**os.environ, **env}, timeout=300)
            outs.append(np.load(p))
    want = O.sz_batch(a)
    for o in outs:
        assert np.array_equal(o.view(np.uint64), want.view(np.uint64))


def test_round2_kernels_repeatable():
    # races show as run-to-run differences (round 1f's stage-ring race did): the lean
    # kernel (batched large orders and a single matrix's outer layers), the FP32 packs
    # and the overlapped-plan kernels, each run several times bitwise identical and
    # equal to the oracle
    rng = np.random.default_rng(9900)
    b = rng.standard_normal((48, 18, 18)) + 1j * rng.standard_normal((48, 18, 18))
    runs = [pl.store_zechin_permanent_batch(b).view(np.uint64) for _ in range(4)]
    assert all(np.array_equal(r, runs[0]) for r in runs)
    assert np.array_equal(runs[0][:6], O.sz_batch(b[:3]).view(np.uint64))  # 3 complex = 6 words
    c3 = configs.c3(4000)
    r3 = [pl.store_zechin_permanent_batch(c3) for _ in range(4)]
    assert all(np.array_equal(r, r3[0]) for r in r3)
    f = rng.uniform(-1, 1, (23, 23))
    v = {struct.pack(">d", pl.store_zechin_permanent(f).value) for _ in range(4)}
    assert v == {struct.pack(">d", O.sz_f64(f))}


_BLK_SCRIPT = r"""
import sys, json
import numpy as np
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
out = {}
for n in (15, 16, 19, 21):
    a = configs.uniform((n, n), seed=3000 + n)
    out["f%d" % n] = float(pl.store_zechin_permanent(a).value).hex()
    out["F%d" % n] = float(pl.store_zechin_permanent(a, fma=True).value)
    c = configs.complex_uniform((n, n), seed=2000 + n)
    v = complex(pl.store_zechin_permanent(c).value)
    out["c%d" % n] = [v.real.hex(), v.imag.hex()]
z = configs.uniform((16, 16), seed=5)
z[3] = 0.0
z[:, 7] = -0.0
out["zero"] = float(pl.store_zechin_permanent(z).value).hex()
a = configs.c4()
out["c4"] = [float(pl.store_zechin_permanent(a).value).hex() for _ in range(3)]
print(json.dumps(out))
"""


def test_register_blocked_engine_bitwise():
    # the opt-in register-blocked engine (sz_blk.cuh, PL_BLK=1): super-layers of
    # 32- (f64) or 16-value (c128) blocks; bitwise the oracle's fold for single
    # matrices of every order it takes, repeatable, and C4 equal to the golden value
    import json
    import os
    import sys

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PL_BLK="1", PYTHONPATH=str(root))
    r = subprocess.run([sys.executable, "-c", _BLK_SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    for n in (15, 16, 19, 21):
        a = configs.uniform((n, n), seed=3000 + n)
        want = O.sz_f64(a)
        assert got["f%d" % n] == float(want).hex()
        assert rel_err(got["F%d" % n], want) <= REL_TOL
        c = configs.complex_uniform((n, n), seed=2000 + n)
        w = complex(O.sz_batch(c[None])[0])
        assert got["c%d" % n] == [w.real.hex(), w.imag.hex()]
    z = configs.uniform((16, 16), seed=5)
    z[3] = 0.0
    z[:, 7] = -0.0
    assert got["zero"] == float(O.sz_f64(z)).hex()
    g = json.loads((root / "tests/golden/goldens.json").read_text())
    assert len(set(got["c4"])) == 1
    assert struct.pack(">d", float.fromhex(got["c4"][0])).hex() == g["c4"]["value_hex"]


def test_blocked_f32_pack_kernel_opt_in():
    # the opt-in register-blocked FP32-exact pack kernel (sz_batch_blk.cuh,
    # PL_BATCH_F32_BLK=1) for int64 batches 10 <= n <= 12: exact integers equal to the
    # oracle's, including packs that fall back member by member and a ragged tail
    import os
    import sys

    root = Path(__file__).resolve().parents[1]
    script = (
        "import numpy as np, paper_1802_02779_b200 as pl\n"
        "from paper_1802_02779_b200 import configs\n"
        "for n in (10, 11, 12):\n"
        "    a = configs.int_matrices(n, 203, seed=77 + n, lo=-1, hi=2)\n"
        "    a[5] *= 3\n"
        "    np.save('/tmp/_blk_f32_%d.npy' % n, pl.store_zechin_permanent_batch(a))\n"
    )
    env = dict(os.environ, PL_BATCH_F32_BLK="1", PYTHONPATH=str(root))
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    for n in (10, 11, 12):
        a = configs.int_matrices(n, 203, seed=77 + n, lo=-1, hi=2)
        a[5] *= 3  # its pack leaves the FP32 bound: member-by-member fallback
        assert np.array_equal(np.load("/tmp/_blk_f32_%d.npy" % n), O.sz_batch(a))


@pytest.mark.parametrize("dtype,n", [("int64", 5), ("complex128", 5), ("float64", 4), ("complex128", 3), ("int64", 1),
                                     ("int64", 7), ("float64", 8), ("complex128", 9), ("complex128", 12)])
def test_input_ready_flag_overlapped_launches_equal_to_oracle(dtype, n):
    # PL_FLAG_INPUT_READY: the n <= 5 batch kernel loads before griddepcontrol.wait, so back-to-back
    # launches (plain stream and CUDA graph) overlap; every launch's results are those of the oracle,
    # also with a ragged tail (count % 32 != 0), a misaligned input and an output the previous launch wrote
    import torch

    count = 32 * 257 + 19 if n <= 5 else 32 * 20 + 19  # n >= 6: the warp / CTA shared-memory kernels
    if dtype == "int64":
        a_np = configs.int_matrices(n, count, seed=8100 + n, lo=-9, hi=9)
    elif dtype == "float64":
        a_np = configs.uniform((count, n, n), seed=8200 + n)
    else:
        a_np = configs.complex_uniform((count, n, n), seed=8300 + n)
    want = O.sz_batch(a_np)
    bufs = [torch.from_numpy(a_np).cuda() for _ in range(3)]
    outs = [torch.zeros(count, dtype=bufs[0].dtype, device="cuda") for _ in range(3)]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    for rep in range(4):
        for b, o in zip(bufs, outs):
            o.zero_()
            pl.store_zechin_permanent_batch(b, out=o, status=status, input_ready=True)
        pl.store_zechin_permanent_batch(bufs[0], out=outs[1], status=status, input_ready=True)  # rewrite an output
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint64), want.view(np.uint64))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    for o in outs:
        o.zero_()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(12):
            pl.store_zechin_permanent_batch(bufs[i % 3], out=outs[i % 3], status=status, stream=s, input_ready=True)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert int(status.item()) == 0
    if n >= 2:  # a misaligned device view (8-byte entries, odd element offset): the direct-load path
        flat = torch.zeros(a_np.size + 1, dtype=bufs[0].dtype, device="cuda")
        flat[1:] = bufs[0].reshape(-1)
        view = flat[1:].reshape(count, n, n)
        o = pl.store_zechin_permanent_batch(view, status=status, input_ready=True)
        torch.cuda.synchronize()
        assert np.array_equal(o.cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("n", [10, 12, 14])
def test_input_ready_flag_f32_packs_equal_to_oracle(n):
    # the FP32-exact int64 pack kernel (10 <= n <= 14) under programmatic dependent launch, with and
    # without PL_FLAG_INPUT_READY: back-to-back and graph-replayed launches, ragged last pack, a
    # member outside the byte range of the packed coefficients
    import torch

    count = 4 * 301 + 3
    a_np = configs.int_matrices(n, count, seed=8400 + n, lo=0, hi=1)
    a_np[5, 0, 0] = 300
    a_np[9, 0, 0] = 10 ** 9  # leaves the FP32-exact range: its pack runs member by member (int64 paths)
    want = O.sz_batch(a_np)
    bufs = [torch.from_numpy(a_np).cuda() for _ in range(2)]
    outs = [torch.zeros(count, dtype=torch.int64, device="cuda") for _ in range(2)]
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    for ready in (False, True):
        for o in outs:
            o.zero_()
        for rep in range(6):
            pl.store_zechin_permanent_batch(bufs[rep % 2], out=outs[rep % 2], status=status, input_ready=ready)
        torch.cuda.synchronize()
        for o in outs:
            assert np.array_equal(o.cpu().numpy(), want)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    for o in outs:
        o.zero_()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(8):
            pl.store_zechin_permanent_batch(bufs[i % 2], out=outs[i % 2], status=status, stream=s, input_ready=True)
    g.replay()
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), want)
    assert int(status.item()) == 0
