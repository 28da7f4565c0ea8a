"""Ryser device engine (reference permanent.hpp:84,
permanent.cpp:85-136) against the oracle restatement of the reference's
RyserEval (bitwise, pinned to the reference in tests/test_oracle.py) and the
Store-zechin engine (exact integers)."""
import struct

import numpy as np
import pytest

import paper_1802_02779_b200 as pl
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def hexf(x):
    return struct.pack(">d", x).hex()


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if pl.device_count() == 0:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


@pytest.mark.parametrize("n", list(range(1, 16)) + [18, 20])
def test_ryser_complex_bitwise(n):
    rng = np.random.default_rng(7000 + n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    r = pl.ryser_permanent(a)
    assert r.algorithm == "ryser"
    assert r.value == O.ryser(a)
    assert r.counts == pl.ryser_counts(n)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 10, 13, 17, 21])
def test_ryser_real_bitwise(n):
    rng = np.random.default_rng(7100 + n)
    a = rng.uniform(-1, 1, (n, n))
    assert hexf(pl.ryser_permanent(a).value) == hexf(O.ryser(a))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 9, 12, 16, 20])
def test_ryser_int_exact(n):
    rng = np.random.default_rng(7200 + n)
    hi = 10 if n <= 16 else 3  # keep prod_i (row |sums|) under the 2^126 guard
    a = rng.integers(-hi + 1, hi, (n, n)).astype(np.int64)
    v = pl.ryser_permanent(a).value
    assert v == O.sz_int(a)
    if n <= 14:
        assert v == O.ryser(a)


def test_ryser_reference_goldens():
    # reference tests/test_permanent.cpp golden matrices
    assert pl.ryser_permanent(np.array([[1, 2], [3, 4]])).value == 10
    assert pl.ryser_permanent(np.arange(1, 10).reshape(3, 3)).value == 450
    dev4 = np.array([7, 0, 1, 2, 5, 3, 4, 5, 3, 5, 6, 7, 1, 7, 8, 9]).reshape(4, 4)
    assert pl.ryser_permanent(dev4).value == 9722
    assert pl.ryser_permanent(np.array([[42]])).value == 42


def test_ryser_agrees_with_store_zechin_complex():
    # reference tests/acceptance.cpp:212-214: the two engines agree (approx_equal)
    rng = np.random.default_rng(7300)
    for n in (6, 12, 16):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        r, s = pl.ryser_permanent(a).value, pl.store_zechin_permanent(a).value
        assert abs(r - s) <= 1e-9 * max(abs(s), 1e-300) * 1e3  # both are reference-order roundings


def test_ryser_int_overflow_guard():
    import ctypes as C
    import math

    from paper_1802_02779_b200 import _native as N

    # all-ones 21 x 21: per = 21! > 2^63 -- the int64 entry point of the C ABI refuses (never wraps) ...
    ones21 = np.ones((21, 21), dtype=np.int64)
    out = np.zeros(1, dtype=np.int64)
    lim = pl.Limits().to_c()
    assert N.lib.pl_ryser_permanent(N.PL_I64, 21, ones21.ctypes.data, out.ctypes.data, 0, C.byref(lim),
                                    None) == N.PL_ERR_OVERFLOW
    # ... and the Python call returns the reference's unbounded Int through the residue sums
    assert pl.ryser_permanent(ones21).value == math.factorial(21)
    # 26 x 26 with row sums 260: the 128-bit guard (260^26 > 2^126) refuses, the residue path is exact
    tens = np.full((26, 26), 10, dtype=np.int64)
    assert N.lib.pl_ryser_permanent(N.PL_I64, 26, tens.ctypes.data, out.ctypes.data, 0, C.byref(lim),
                                    None) == N.PL_ERR_OVERFLOW
    r = pl.ryser_permanent(tens)
    assert r.value == 10 ** 26 * math.factorial(26) and r.algorithm == "ryser" and r.counts == pl.ryser_counts(26)
    assert pl.ryser_permanent(np.ones((12, 12), dtype=np.int64)).value == 479001600
    assert pl.ryser_permanent(np.ones((20, 20), dtype=np.int64)).value == 2432902008176640000


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_ryser_bitwise_equals_reference_engine():
    rng = np.random.default_rng(7400)
    for n in (5, 9, 13):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        assert pl.ryser_permanent(a).value == O.ref_ryser_c128(a)


def test_ryser_multi_chunk_fold():
    # n = 25: 2^25 - 1 subsets, two chunks of 2^24 terms folded in sequence
    rng = np.random.default_rng(7500)
    a = rng.uniform(-1, 1, (25, 25))
    assert hexf(pl.ryser_permanent(a).value) == hexf(O.ryser(a))
