"""Boson-sampling driver, host side (no GPU): the pattern enumerator and
unranker against the reference's enumerate_patterns, the inverse-CDF sampler
against the reference's sample(), the argument checks and messages of the
reference (boson.cpp:63-92, 250-260), and no CPU fallback for probabilities.

The reference engine (oracle/_ref, compiled from the reference sources) is the
checker; golden fixtures in tests/golden/boson.json pin the same facts where
oracle/_ref is absent."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import _native as N
from paper_1802_02779_b200 import boson as B
from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def bgold():
    return json.loads((ROOT / "tests" / "golden" / "boson.json").read_text())


@need_ref
@pytest.mark.parametrize("m,n", [(1, 1), (1, 4), (3, 1), (4, 3), (8, 4), (25, 5), (7, 6), (2, 6)])
def test_enumeration_order_matches_reference(m, n):
    ref = O.ref_enumerate_patterns(m, n)
    assert B.pattern_count(m, n) == ref.shape[0]
    assert np.array_equal(B.pattern_occupancies(m, n), ref)
    assert [p.occupancy for p in B.enumerate_patterns(m, n)] == [tuple(r) for r in ref]


@pytest.mark.parametrize("m,n", [(1, 1), (4, 3), (9, 4), (25, 5), (13, 6), (1024, 3)])
def test_c_abi_unrank_matches_enumeration(m, n):
    total = B.pattern_count(m, n)
    rng = np.random.default_rng(m * 10 + n)
    idx = sorted(set([0, min(1, total - 1), total - 1] + [int(x) for x in rng.integers(0, total, 200)]))
    rows = np.zeros(n, dtype=np.int32)
    for i in idx:
        assert N.lib.pl_boson_unrank_pattern(m, n, i, rows.ctypes.data) == N.PL_OK
        assert rows.tolist() == _unrank_linear(m, n, i), (m, n, i)
        if i < 5000:
            assert np.array_equal(rows, B.pattern_rows(m, n, i, 1)[0])
    assert N.lib.pl_boson_unrank_pattern(m, n, total, rows.ctypes.data) == N.PL_ERR_ARG


def _unrank_linear(m, n, idx):
    # independent restatement: at each position count the completions per value
    import math

    rows, prev = [], 0
    for i in range(n):
        rest = n - 1 - i
        v = prev
        while True:
            c = math.comb(m - v + rest - 1, rest)  # sequences of length rest over [v, m)
            if idx < c:
                break
            idx -= c
            v += 1
        rows.append(v)
        prev = v
    return rows


def test_pattern_count_closed_form():
    import math

    for m in (1, 2, 25, 1000):
        for n in (0, 1, 5, 6):
            assert B.pattern_count(m, n) == math.comb(m + n - 1, n)
    assert B.pattern_count(0, 3) == 0
    assert B.pattern_count(1 << 30, 6) == 0  # beyond 64 bits


def test_enumeration_golden(bgold):
    g = bgold["enumerate_25_5"]
    rows = B.pattern_rows(25, 5)
    assert rows.shape[0] == g["count"]
    import hashlib

    assert hashlib.sha256(B.pattern_occupancies(25, 5).tobytes()).hexdigest() == g["occupancy_sha256"]


@need_ref
@pytest.mark.parametrize("seed,m,modes", [(3, 6, [0, 1, 4]), (7, 8, [2, 3, 5, 7]), (11, 5, [4, 0])])
def test_sampler_matches_reference(seed, m, modes):
    u = O.ref_haar(m, seed)
    occ, probs = O.ref_full_distribution(u, modes)
    d = B.OutcomeDistribution(input_modes=modes, modes=m, probabilities=probs)
    idx = B.sample_indices(d, 2000, seed + 100)
    assert np.array_equal(occ[idx], O.ref_sample(u, modes, 2000, seed + 100))
    acc = 0.0
    for p in probs.tolist():
        acc += p
    assert d.total_probability() == acc


def test_sampler_golden(bgold):
    g = bgold["sample_haar6_seed3"]
    probs = np.array([float.fromhex(x) for x in g["probabilities_hex"]])
    d = B.OutcomeDistribution(input_modes=g["input_modes"], modes=g["modes"], probabilities=probs)
    assert B.sample_indices(d, g["count"], g["seed"]).tolist() == g["indices"]


def test_haar_unitary_matches_reference_bitwise():
    u = B.haar_unitary(7, 9).unitary()
    if O.ref_available():
        assert np.array_equal(u, O.ref_haar(7, 9))
    assert np.max(np.abs(u.conj().T @ u - np.eye(7))) < 1e-12


def test_interferometer_checks():
    with pytest.raises(pl.DomainError, match="mode count must be >= 1"):
        B.Interferometer(0, np.zeros((0, 0)))
    with pytest.raises(pl.DomainError, match="unitary order must equal the mode count"):
        B.Interferometer(3, np.eye(2))
    with pytest.raises(pl.DomainError, match="not unitary within 1e-10"):
        B.Interferometer(2, np.array([[1, 0], [0, 1.001]]))


def test_input_mode_and_pattern_checks():
    itf = B.Interferometer(4, np.eye(4))
    with pytest.raises(pl.DomainError, match="at least one input mode is required"):
        B.extract_submatrix(itf, [], B.OutputPattern([0, 0, 0, 0]))
    with pytest.raises(pl.DomainError, match="input mode index out of range"):
        B.extract_submatrix(itf, [4], B.OutputPattern([1, 0, 0, 0]))
    with pytest.raises(pl.DomainError, match="input modes must be distinct"):
        B.extract_submatrix(itf, [1, 1], B.OutputPattern([2, 0, 0, 0]))
    with pytest.raises(pl.DomainError, match="occupancy vector length"):
        B.extract_submatrix(itf, [1], B.OutputPattern([1, 0, 0]))
    with pytest.raises(pl.DomainError, match="nonnegative"):
        B.extract_submatrix(itf, [1], B.OutputPattern([2, -1, 0, 0]))
    with pytest.raises(pl.DomainError, match="does not match"):
        B.extract_submatrix(itf, [1, 2], B.OutputPattern([1, 0, 0, 0]))
    sub = B.extract_submatrix(itf, [2, 0], B.OutputPattern([0, 0, 2, 0]))
    assert np.array_equal(sub, np.array([[1, 0], [1, 0]], dtype=np.complex128))


def test_distribution_limits():
    itf = B.haar_unitary(8, 1)
    with pytest.raises(pl.DomainError, match="at most 6 photons"):
        B.full_distribution(itf, list(range(7)))
    with pytest.raises(pl.DomainError, match="enumeration_cap"):
        B.full_distribution(itf, [0, 1, 2], pl.Limits(enumeration_cap=100))
    # the C ABI checks the same before touching a device
    u = itf.unitary()
    modes = np.arange(7, dtype=np.int32)
    probs = np.zeros(1)
    assert N.lib.pl_boson_distribution(8, u.ctypes.data, 7, modes.ctypes.data, 0, 1, probs.ctypes.data, 0, None) \
        == N.PL_ERR_LIMIT
    assert "at most 6 photons" in N.last_error()
    bad = np.array([0, 0], dtype=np.int32)
    assert N.lib.pl_boson_distribution(8, u.ctypes.data, 2, bad.ctypes.data, 0, 1, probs.ctypes.data, 0, None) \
        == N.PL_ERR_ARG
    assert "distinct" in N.last_error()


@pytest.mark.skipif(pl.device_count() > 0, reason="checks the no-device behaviour")
def test_no_cpu_fallback():
    itf = B.haar_unitary(5, 2)
    with pytest.raises(pl.DeviceError, match="PL_ERR_NODEVICE"):
        B.full_distribution(itf, [0, 1])
    with pytest.raises(pl.DeviceError, match="PL_ERR_NODEVICE"):
        B.outcome_probability(itf, [0, 1], B.OutputPattern([1, 1, 0, 0, 0]))
