"""Host-side logic of the engine that needs no GPU: the C ABI library loads and
exports every symbol its header declares, closed forms, colex ranking, limit
and error mapping, the reference-shaped Python/C++ API surface."""
import math
import re
import subprocess
from itertools import combinations
from pathlib import Path

import numpy as np
import pytest

import paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def header_symbols():
    text = (ROOT / "include" / "permlab_b200.h").read_text()
    return sorted(set(re.findall(r"\b(pl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert set(syms) == set(N.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True, text=True, check=True)
    exported = set(line.split()[-1] for line in out.stdout.splitlines())
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert "sm_100a" in pl.version()


def test_kernels_are_sm100a_cubins():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_counts_and_diagnostics():
    assert pl.store_zechin_counts(1) == pl.OpCount(0, 0)
    assert pl.store_zechin_counts(2) == pl.OpCount(2, 1)
    for n, (m, a) in {3: (9, 5), 4: (28, 17), 5: (75, 49)}.items():  # reference PAPER.md table / acceptance.cpp:73
        assert pl.store_zechin_counts(n) == pl.OpCount(m, a)
    for n in range(3, 40):
        c = pl.store_zechin_counts(n)
        assert (c.multiplications, c.additions) == (n * 2 ** (n - 1) - n, n * 2 ** (n - 1) - 2 ** n + 1)


def test_ryser_counts_match_reference_tables():
    # reference tests/test_cost_model.cpp:28 and tests/acceptance.cpp:72
    # (count_formula == the instrumented engine's counts, acceptance.cpp:236)
    assert pl.ryser_counts(3) == pl.OpCount(14, 18)
    assert pl.ryser_counts(4) == pl.OpCount(45, 58)
    assert pl.ryser_counts(5) == pl.OpCount(124, 160)
    assert pl.ryser_counts(1) == pl.OpCount(0, 0)
    for n in range(2, 30):
        assert pl.ryser_counts(n) == pl.OpCount((2**n - 1) * (n - 1), (2**n - n) * (n + 1) - 2)


def test_binomials_and_colex():
    for s in range(0, 40):
        for k in range(0, s + 1):
            assert pl.binom(s, k) == math.comb(s, k)
    for n in range(1, 13):
        for k in range(1, n + 1):
            masks = sorted(sum(1 << e for e in c) for c in combinations(range(n), k))
            assert [pl.colex_rank(m) for m in masks] == list(range(len(masks)))
            assert [pl.colex_unrank(k, r) for r in range(len(masks))] == masks
    rng = np.random.default_rng(5)
    for _ in range(2000):
        n = int(rng.integers(13, 35))
        k = int(rng.integers(1, n))
        mask = sum(1 << int(e) for e in rng.choice(n, size=k, replace=False))
        r = pl.colex_rank(mask)
        assert r == O.colex_rank(mask) and r < math.comb(n, k)
        assert pl.colex_unrank(k, r) == mask


def test_scratch_bytes():
    assert pl.scratch_bytes(np.complex128, 32) == 2 * math.comb(32, 16) * 16
    assert pl.scratch_bytes(np.float64, 26) == 2 * math.comb(26, 13) * 8


@need_ref
def test_attribution_closed_form_matches_reference():
    for n in range(3, 11):
        ones = np.ones((n, n), dtype=np.int64)
        rep = pl.store_zechin_attributed(ones)
        ref = O.ref_sz_run_int(ones)
        assert [(t.multiplications, t.additions) for t in rep.per_term] == ref["per_term"]
        assert rep.final_combination_adds == ref["final_combination_adds"]
        c = pl.store_zechin_counts(n)
        assert rep.totals == c


def test_attribution_tables():
    # reference tests/test_permanent.cpp:149-168
    rep = pl.store_zechin_attributed(np.ones((5, 5), dtype=np.int64))
    assert [(t.multiplications, t.additions) for t in rep.per_term] == [(29, 17), (20, 12), (13, 8), (8, 5), (5, 3)]
    with pytest.raises(pl.DomainError):
        pl.store_zechin_attributed(np.eye(2, dtype=np.int64))


def test_limits_from_env(monkeypatch):
    monkeypatch.setenv("PERMLAB_LIMITS", "naive_order_limit=10,subset_order_limit=24,enumeration_cap=10000")
    lim = pl.Limits.from_env()
    assert (lim.naive_order_limit, lim.subset_order_limit, lim.enumeration_cap) == (10, 24, 10000)
    for bad in ("bogus=1", "subset_order_limit", "subset_order_limit=x", "subset_order_limit="):
        monkeypatch.setenv("PERMLAB_LIMITS", bad)
        with pytest.raises(pl.DomainError):
            pl.Limits.from_env()


def test_domain_errors_before_device_work():
    # reference tests/test_permanent.cpp:280-294: limits reject before any arithmetic
    a5 = np.ones((5, 5), dtype=np.int64)
    with pytest.raises(pl.DomainError, match="subset_order_limit"):
        pl.store_zechin_permanent(a5, pl.Limits(subset_order_limit=4))
    with pytest.raises(pl.DomainError, match="memory budget"):
        pl.store_zechin_permanent(a5, pl.Limits(memo_budget_bytes=16))
    with pytest.raises(pl.DomainError):
        pl.store_zechin_permanent(np.ones((35, 35), dtype=np.int64))
    with pytest.raises(pl.DomainError):
        pl.store_zechin_permanent(np.ones((3, 4)))
    with pytest.raises(pl.DomainError):
        pl.store_zechin_permanent(np.array([["a", "b"], ["c", "d"]], dtype=object))
    # Python integers beyond int64 (the residue path): limits still reject before any device work
    big = np.array([[10 ** 30, 1], [2, 3]], dtype=object)
    with pytest.raises(pl.DomainError, match="subset_order_limit"):
        pl.store_zechin_permanent(big, pl.Limits(subset_order_limit=1))
    with pytest.raises(pl.DomainError, match="subset_order_limit"):
        pl.ryser_permanent(big, pl.Limits(subset_order_limit=1))
    with pytest.raises(pl.DomainError):
        pl.store_zechin_permanent_batch(np.ones((3, 4, 4), dtype=np.float32))
    with pytest.raises(pl.DomainError, match="subset_order_limit"):
        pl.ryser_permanent(a5, pl.Limits(subset_order_limit=4))
    with pytest.raises(pl.DomainError):
        pl.ryser_permanent(np.ones((35, 35), dtype=np.int64))


def test_no_cpu_fallback_without_device():
    if pl.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(pl.DeviceError, match="NODEVICE"):
        pl.store_zechin_permanent(np.eye(3))
    with pytest.raises(pl.DeviceError, match="NODEVICE"):
        pl.store_zechin_permanent_batch(np.ones((4, 5, 5), dtype=np.int64))
    with pytest.raises(pl.DeviceError, match="NODEVICE"):
        pl.ryser_permanent(np.eye(3))
    with pytest.raises(pl.DeviceError, match="NODEVICE"):
        pl.store_zechin_permanent(np.array([[10 ** 30, 1], [2, 3]], dtype=object))


def test_bigint_primes_are_the_largest_31_bit_primes():
    # host-only part of the exact big-integer path (csrc/bigint.cu): deterministic Miller-Rabin
    import ctypes as C

    from paper_1802_02779_b200 import _native as N

    k = 80  # a 34 x 34 matrix of full-range int64 entries needs 80 passes
    primes = np.zeros(k, dtype=np.uint32)
    assert N.lib.pl_bigint_primes(k, primes.ctypes.data) == k

    def is_prime(v):
        return v > 1 and all(v % q for q in range(2, int(v ** 0.5) + 1))

    want, v = [], 2 ** 31 - 1
    while len(want) < 6:
        if is_prime(v):
            want.append(v)
        v -= 2
    assert primes[:6].tolist() == want
    assert all(2 ** 30 < int(p) < 2 ** 31 for p in primes) and len(set(primes.tolist())) == k
    assert all(int(a) > int(b) for a, b in zip(primes, primes[1:]))
    # Fermat check of the rest (base 2 and 3; Miller-Rabin inside is deterministic below 3.2e9)
    assert all(pow(2, int(p) - 1, int(p)) == 1 and pow(3, int(p) - 1, int(p)) == 1 for p in primes)
    assert N.lib.pl_bigint_primes(0, primes.ctypes.data) == 0
    # argument errors come before the device check
    lim = pl.Limits().to_c()
    nl, neg = C.c_size_t(0), C.c_int32(0)
    assert N.lib.pl_sz_permanent_bigint(0, primes.ctypes.data, None, 0, C.byref(nl), C.byref(neg), C.byref(lim),
                                        None) == N.PL_ERR_ARG
    a35 = np.ones((35, 35), dtype=np.int64)
    assert N.lib.pl_sz_permanent_bigint(35, a35.ctypes.data, None, 0, C.byref(nl), C.byref(neg), C.byref(lim),
                                        None) == N.PL_ERR_LIMIT


def test_cpp_host_suite():
    exe = ROOT / "tests" / "cpp" / "test_permanent_device"
    assert exe.exists(), "run `make` first"
    out = subprocess.run([str(exe), "--host-only"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout
