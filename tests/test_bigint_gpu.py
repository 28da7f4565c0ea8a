"""Exact integer permanents beyond int64 (csrc/bigint.cu): the reference's Int ring is
arbitrary precision (reference ring.hpp:29-31), so store_zechin_permanent
(permanent.cpp:314-316) returns the exact integer for any entries. The device runs the layer
DP on residues modulo 31-bit primes and recombines them; checked here against the oracle
(128-bit Int), against closed forms, and against a Python-integer restatement of the
recurrence (small orders only)."""
import ctypes as C
import math

import numpy as np
import pytest

import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import _native as N
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if pl.device_count() == 0:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


def py_permanent(rows):
    """The subset recurrence of reference permanent.cpp:151-177 on Python integers."""
    n = len(rows)
    x = {0: 1}
    for k in range(1, n + 1):
        nxt = {}
        for s, v in x.items():
            for j in range(n):
                if not (s >> j) & 1:
                    t = s | (1 << j)
                    nxt[t] = nxt.get(t, 0) + rows[k - 1][j] * v
        x = nxt
    return x[(1 << n) - 1]


def derangements(n):
    d = [1, 0]
    for i in range(2, n + 1):
        d.append((i - 1) * (d[i - 1] + d[i - 2]))
    return d[n]


@pytest.mark.parametrize("n", [21, 22, 26, 32])
def test_all_ones_factorial_beyond_int64(n):
    # n! > 2^63 for n >= 21: the int64 guard trips and the residue path takes over
    assert pl.store_zechin_permanent(np.ones((n, n), dtype=np.int64)).value == math.factorial(n)


@pytest.mark.parametrize("n", [5, 9, 14, 15, 20])
def test_scaled_ones_and_signs(n):
    c = -(10 ** 6 + 3)
    assert pl.store_zechin_permanent(np.full((n, n), c, dtype=np.int64)).value == c ** n * math.factorial(n)
    # J - I: the derangement numbers, with a large common factor
    a = (np.ones((n, n), dtype=np.int64) - np.eye(n, dtype=np.int64)) * (2 ** 40)
    assert pl.store_zechin_permanent(a).value == derangements(n) * 2 ** (40 * n)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 6, 8, 10])
def test_random_int64_entries_vs_python_integers(n):
    rng = np.random.default_rng(9100 + n)
    a = rng.integers(-(2 ** 62), 2 ** 62, (n, n), dtype=np.int64)
    if n >= 2:
        a[0, 0] = np.iinfo(np.int64).min
        a[1, 1] = np.iinfo(np.int64).max
    want = py_permanent([[int(v) for v in r] for r in a])
    got = pl.store_zechin_permanent(a).value
    assert got == want
    assert n < 2 or abs(got) >= 2 ** 63  # these do leave int64


@pytest.mark.parametrize("n", [12, 15, 17])
def test_vs_oracle_128_bit(n):
    rng = np.random.default_rng(9200 + n)
    a = rng.integers(-50, 51, (n, n), dtype=np.int64)  # |per| <= (50 n)^n < 2^127 for n <= 17... checked below
    want = O.sz_int(a)
    assert abs(want) < 2 ** 126
    lim = pl.Limits().to_c()
    limbs = np.zeros(40, dtype=np.uint64)
    nl, neg = C.c_size_t(0), C.c_int32(0)
    assert N.lib.pl_sz_permanent_bigint(n, a.ctypes.data, limbs.ctypes.data, 40, C.byref(nl), C.byref(neg),
                                        C.byref(lim), None) == N.PL_OK
    v = sum(int(limbs[i]) << (64 * i) for i in range(nl.value))
    assert (-v if neg.value else v) == want


def test_python_integers_beyond_int64_entries():
    rng = np.random.default_rng(9300)
    for n in (1, 3, 7, 11):
        rows = [[int(rng.integers(-(2 ** 62), 2 ** 62)) * (3 ** 50) + int(rng.integers(0, 100)) for _ in range(n)]
                for _ in range(n)]
        assert pl.store_zechin_permanent(np.array(rows, dtype=object)).value == py_permanent(rows)
    n = 16
    rows = [[(10 ** 30 if i == j else 0) + (i + 2 * j) % 3 for j in range(n)] for i in range(n)]
    small = np.array([[(i + 2 * j) % 3 for j in range(n)] for i in range(n)], dtype=np.int64)
    got = pl.store_zechin_permanent(np.array(rows, dtype=object)).value
    # per(D + S) mod 10^30 = per(S) for D = 10^30 I: every term with a diagonal factor is a multiple
    assert got % 10 ** 30 == O.sz_int(small) % 10 ** 30
    assert got > 10 ** (30 * n)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 10, 13, 18])
def test_ryser_residue_sums_equal_store_zechin(n):
    # Ryser's formula on the same residues (pl_ryser_permanent_bigint): the same integer
    rng = np.random.default_rng(9400 + n)
    a = rng.integers(-(2 ** 62), 2 ** 62, (n, n), dtype=np.int64)
    want = pl.store_zechin_permanent(a).value
    if n <= 10:
        assert want == py_permanent([[int(v) for v in r] for r in a])
    assert pl.ryser_permanent(a).value == want
    rows = [[int(v) * 7 ** 30 + 1 for v in r] for r in a]  # entries beyond int64: Python integers
    if n <= 10:
        assert pl.ryser_permanent(np.array(rows, dtype=object)).value == py_permanent(rows)
    else:
        assert (pl.ryser_permanent(np.array(rows, dtype=object)).value
                == pl.store_zechin_permanent(np.array(rows, dtype=object)).value)


def test_zero_small_and_values_that_fit():
    a = np.zeros((21, 21), dtype=np.int64)
    lim = pl.Limits().to_c()
    limbs = np.zeros(4, dtype=np.uint64)
    nl, neg = C.c_size_t(7), C.c_int32(7)
    assert N.lib.pl_sz_permanent_bigint(21, a.ctypes.data, limbs.ctypes.data, 4, C.byref(nl), C.byref(neg),
                                        C.byref(lim), None) == N.PL_OK
    assert (nl.value, neg.value) == (0, 0)
    # a value that fits int64 comes back the same through the residue path
    dev4 = np.array([7, 0, 1, 2, 5, 3, 4, 5, 3, 5, 6, 7, 1, 7, 8, 9], dtype=np.int64).reshape(4, 4)
    assert N.lib.pl_sz_permanent_bigint(4, dev4.ctypes.data, limbs.ctypes.data, 4, C.byref(nl), C.byref(neg),
                                        C.byref(lim), None) == N.PL_OK
    assert (nl.value, neg.value, int(limbs[0])) == (1, 0, 9722)
    neg4 = -dev4
    neg4[1:] = dev4[1:]
    assert N.lib.pl_sz_permanent_bigint(4, neg4.ctypes.data, limbs.ctypes.data, 4, C.byref(nl), C.byref(neg),
                                        C.byref(lim), None) == N.PL_OK
    assert (nl.value, neg.value, int(limbs[0])) == (1, 1, 9722)
    # too small a limb buffer: PL_ERR_ARG and the size needed
    big = np.full((10, 10), 2 ** 62, dtype=np.int64)
    assert N.lib.pl_sz_permanent_bigint(10, big.ctypes.data, limbs.ctypes.data, 4, C.byref(nl), C.byref(neg),
                                        C.byref(lim), None) == N.PL_ERR_ARG
    assert nl.value == (((2 ** 62) ** 10 * math.factorial(10)).bit_length() + 63) // 64


def test_residue_passes_argument_checks_and_limits():
    primes = np.zeros(3, dtype=np.uint32)
    assert N.lib.pl_bigint_primes(3, primes.ctypes.data) == 3
    assert int(primes[0]) == 2 ** 31 - 1 and all(2 ** 30 < int(p) < 2 ** 31 for p in primes)
    assert len(set(primes.tolist())) == 3
    lim = pl.Limits().to_c()
    out = np.zeros(3, dtype=np.uint32)
    res = np.zeros((3, 4, 4), dtype=np.int64)
    res[1, 0, 0] = int(primes[1])  # not reduced
    assert N.lib.pl_sz_permanent_modp(4, 3, primes.ctypes.data, res.ctypes.data, out.ctypes.data, C.byref(lim),
                                      None) == N.PL_ERR_ARG
    # moduli need not be prime for the passes themselves: per(J_5) mod 1000 = 120
    mods = np.array([1000, 7, 2], dtype=np.uint32)
    ones = np.ones((3, 5, 5), dtype=np.int64)
    assert N.lib.pl_sz_permanent_modp(5, 3, mods.ctypes.data, ones.ctypes.data, out.ctypes.data, C.byref(lim),
                                      None) == N.PL_OK
    assert out.tolist() == [120, 120 % 7, 0]
    # the order limit applies as for the int64 path
    with pytest.raises(pl.DomainError, match="subset_order_limit"):
        pl.store_zechin_permanent(np.full((21, 21), 2 ** 40, dtype=np.int64), pl.Limits(subset_order_limit=20))
