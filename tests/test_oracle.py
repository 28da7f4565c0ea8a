"""Pins the CPU oracle (oracle/sz_oracle.c) before anything is checked
against it: the reference's own golden values (reference
proj/tests/test_permanent.cpp), the reference engine itself compiled from
/root/reference (oracle/_ref, when present), and the committed config
fixtures (tests/golden/goldens.json)."""
import struct

import numpy as np
import pytest

from oracle import oracle as O
from paper_1802_02779_b200 import configs

need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")

DEV4 = np.array([7, 0, 1, 2, 5, 3, 4, 5, 3, 5, 6, 7, 1, 7, 8, 9]).reshape(4, 4)
A5 = np.array([1, 1, 0, 2, 3, 2, 0, 1, 1, 4, 3, 1, 2, 0, 1, 0, 2, 1, 3, 2, 1, 0, 4, 1, 2]).reshape(5, 5)


def hexf(x):
    return struct.pack(">d", x).hex()


def test_reference_goldens():
    # reference tests/test_permanent.cpp:48-92, 246-255
    assert O.sz_int(np.array([[1, 2], [3, 4]])) == 10
    assert O.sz_int(np.arange(1, 10).reshape(3, 3)) == 450
    assert O.sz_int(DEV4) == 9722
    assert O.sz_int(A5) == 988
    assert O.sz_int(np.array([[42]])) == 42
    assert O.sz_int(np.array([[2, 3], [5, 7]])) == 29
    assert O.sz_int(np.ones((3, 3), dtype=np.int64)) == 6
    minors = [1116, 258, 166, 122]
    for i in range(4):
        m = np.delete(np.delete(DEV4, i, 0), 0, 1)
        assert O.sz_int(m) == minors[i]


def test_exact_beyond_int64():
    # all-ones n=21: 21! > 2^63; the int128 oracle stays exact
    import math

    assert O.sz_int(np.ones((21, 21), dtype=np.int64)) == math.factorial(21)


def test_colex_roundtrip():
    from itertools import combinations

    for n in range(1, 11):
        for k in range(1, n + 1):
            masks = sorted(sum(1 << e for e in c) for c in combinations(range(n), k))
            for r, m in enumerate(masks):
                assert O.colex_rank(m) == r
                assert O.colex_unrank(k, r) == m


def test_layer_matches_full_dp():
    a = configs.uniform((9, 9), seed=11)
    last = O.sz_layer_f64(a, 8)
    top = sum(a[8, j] * last[8 - j] for j in range(9))  # order differs from the oracle's left fold only by rounding
    assert abs(top - O.sz_f64(a)) <= 1e-12 * abs(top)


@need_ref
def test_oracle_equals_reference_int():
    # reference tests/test_permanent.cpp:94-106 sweep (n = 1..6, 20 each), extended to n = 8
    for n in range(1, 9):
        mats = configs.int_matrices(n, 20, seed=41 + n)
        for m in mats:
            v, counts = O.ref_sz_int(m)
            assert O.sz_int(m) == v
            assert O.ref_naive_int(m) == v
            assert O.ref_ryser_int(m) == v


@need_ref
def test_oracle_equals_reference_counts_and_tables():
    for n in range(2, 13):
        _, counts = O.ref_sz_int(np.ones((n, n), dtype=np.int64))
        half = 1 << (n - 1)
        assert counts == (n * half - n, n * half - 2 * half + 1)
    run = O.ref_sz_run_int(np.ones((5, 5), dtype=np.int64))
    assert run["per_term"] == [(29, 17), (20, 12), (13, 8), (8, 5), (5, 3)]
    assert run["cache_misses"] == run["distinct_subsets"] == 2 ** 5 - 5 - 2


@need_ref
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11, 14, 17])
def test_oracle_bitwise_equals_reference_float(n):
    a = configs.complex_uniform((n, n), seed=100 + n)
    got = O.sz_c128(a)
    ref, _ = O.ref_sz_c128(a)
    assert hexf(got.real) == hexf(ref.real) and hexf(got.imag) == hexf(ref.imag)
    b = configs.uniform((n, n), seed=200 + n)
    assert hexf(O.sz_f64(b)) == hexf(O.ref_sz_f64(b))


def test_oracle_against_committed_fixtures(goldens):
    for name in ("c1", "c3"):
        g = goldens[name]
        a = configs.generate(name)
        assert configs.sha256(a) == g["input_sha256"]
        out = O.sz_batch(a)
        assert configs.sha256(out) == g["output_sha256"]
        assert [int(v) for v in out[:32]] == g["first32"]
    g = goldens["c2"]
    a = configs.c2()
    assert configs.sha256(a) == g["input_sha256"]
    assert configs.sha256(O.sz_batch(a)) == g["output_sha256"]
    g = goldens["c4"]
    a = configs.c4()
    assert configs.sha256(a) == g["input_sha256"]
    assert hexf(O.sz_f64(a)) == g["value_hex"] == g["reference_value_hex"]


# ---------------------------------------------------------------- Ryser

def test_ryser_restatement_goldens():
    # reference tests/test_permanent.cpp: the Ryser engine agrees with the
    # others on the golden matrices
    assert O.ryser(np.array([[1, 2], [3, 4]], dtype=np.int64)) == 10
    assert O.ryser(np.arange(1, 10, dtype=np.int64).reshape(3, 3)) == 450
    assert O.ryser(DEV4.astype(np.int64)) == 9722
    assert O.ryser(A5.astype(np.int64)) == 988
    assert O.ryser(np.array([[42]], dtype=np.int64)) == 42


@need_ref
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 11, 14])
def test_ryser_restatement_bitwise_equals_reference(n):
    rng = np.random.default_rng(100 + n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    assert O.ryser(a) == O.ref_ryser_c128(a)
    r = rng.uniform(-1, 1, (n, n))
    assert hexf(O.ryser(r)) == hexf(O.ref_ryser_c128(r.astype(np.complex128)).real)
    i = rng.integers(-9, 10, (n, n)).astype(np.int64)
    assert O.ryser(i) == O.ref_ryser_int(i) == O.sz_int(i)
