"""Device parity of the boson-sampling driver (pl_boson_distribution /
pl_boson_probabilities) against the reference engine (oracle/_ref: the
reference's own full_distribution / outcome_probability / sample compiled
from its sources) and the committed fixtures.

Bar: in the default (non-FMA) mode every probability is bitwise the
reference's (same DP order, same rounding, |z|^2 = x*x + y*y then / prod occ!);
with FMA within relative 1e-9 (north_star's fp64 / complex128 tolerance)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import _native as N
from paper_1802_02779_b200 import boson as B
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REL_TOL = 1e-9
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module", autouse=True)
def _need_device():
    if pl.device_count() == 0:
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")


@pytest.fixture(scope="module")
def bgold():
    return json.loads((ROOT / "tests" / "golden" / "boson.json").read_text())


def _oracle_probs(u, modes, rows):
    """|per|^2 / prod occ! with the restated DP (bitwise the reference engine)."""
    subs = u[rows[:, :, None], np.asarray(modes)[None, None, :]]
    per = O.sz_batch(np.ascontiguousarray(subs))
    div = np.ones(rows.shape[0])
    for t in range(rows.shape[0]):
        run = 1
        for i in range(1, rows.shape[1]):
            run = run + 1 if rows[t, i] == rows[t, i - 1] else 1
            if run >= 2:
                div[t] *= run
    return (per.real * per.real + per.imag * per.imag) / div


def test_haar25_distribution_golden(bgold):
    g = bgold["haar25_seed2_modes0to4"]
    itf = B.haar_unitary(25, 2)
    d = B.full_distribution(itf, [0, 1, 2, 3, 4], pl.Limits(enumeration_cap=200000))
    assert d.probabilities.shape[0] == g["count"] == 118755
    assert hashlib.sha256(d.probabilities.tobytes()).hexdigest() == g["probabilities_sha256"]
    assert d.total_probability().hex() == g["total_probability_hex"]
    assert abs(d.total_probability() - 1.0) < 1e-12


@need_ref
@pytest.mark.parametrize("m,modes,seed", [(1, [0], 1), (2, [1, 0], 2), (5, [0, 1, 2, 3, 4], 3), (6, [5, 0, 2], 4),
                                         (8, [1, 2, 3, 4, 5, 6], 5), (10, [9, 3, 0, 7], 6), (3, [2, 1, 0], 7),
                                         (25, [0, 1, 2, 3, 4], 8)])
def test_distribution_bitwise_vs_reference(m, modes, seed):
    itf = B.haar_unitary(m, seed)
    occ, want = O.ref_full_distribution(itf.unitary(), modes, enumeration_cap=10 ** 6)
    d = B.full_distribution(itf, modes, pl.Limits(enumeration_cap=10 ** 6))
    assert np.array_equal(d.probabilities, want)  # bitwise
    assert [p.occupancy for p, _ in d.entries[:50]] == [tuple(o) for o in occ[:50].tolist()]
    f = B.full_distribution(itf, modes, pl.Limits(enumeration_cap=10 ** 6), fma=True).probabilities
    nz = want > 1e-300
    assert np.all(np.abs(f[nz] - want[nz]) <= REL_TOL * want[nz])


def test_distribution_ranges_concatenate():
    itf = B.haar_unitary(12, 11)
    modes = [0, 3, 5, 7, 9, 11]
    full = B.distribution_probabilities(itf, modes)
    total = B.pattern_count(12, 6)
    assert full.shape[0] == total
    cuts = [0, 1, 127, 128, 4097, total - 1, total]
    parts = [B.distribution_probabilities(itf, modes, a, b - a) for a, b in zip(cuts[:-1], cuts[1:])]
    assert np.array_equal(np.concatenate(parts), full)
    assert B.distribution_probabilities(itf, modes, total, 0).shape[0] == 0


def test_distribution_device_buffers_async():
    import torch

    itf = B.haar_unitary(25, 2)
    modes = [0, 1, 2, 3, 4]
    host = B.distribution_probabilities(itf, modes)
    out = torch.empty(host.shape[0], dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    B.distribution_probabilities(itf, modes, out=out, status=st)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), host)
    assert int(st.item()) == 0


def test_distribution_input_ready_overlapped_launches():
    # PL_FLAG_INPUT_READY: the fused kernel computes before griddepcontrol.wait and stores after it;
    # back-to-back and graph-replayed launches into alternating (and rewritten) outputs are bitwise
    # the plain results
    import torch

    itf = B.haar_unitary(25, 2)
    for modes in ([0, 1, 2, 3, 4], [3, 9, 20]):
        host = B.distribution_probabilities(itf, modes)
        outs = [torch.zeros(host.shape[0], dtype=torch.float64, device="cuda") for _ in range(2)]
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        for i in range(7):
            B.distribution_probabilities(itf, modes, out=outs[i % 2], status=st, input_ready=True)
        torch.cuda.synchronize()
        for o in outs:
            assert np.array_equal(o.cpu().numpy(), host)
            o.zero_()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(9):
                B.distribution_probabilities(itf, modes, out=outs[i % 2], status=st, stream=s, input_ready=True)
        g.replay()
        g.replay()
        torch.cuda.synchronize()
        for o in outs:
            assert np.array_equal(o.cpu().numpy(), host)
        assert int(st.item()) == 0


@need_ref
@pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 8])
def test_outcome_probabilities_vs_reference(n):
    m = 10
    itf = B.haar_unitary(m, 20 + n)
    rng = np.random.default_rng(n)
    modes = sorted(rng.choice(m, n, replace=False).tolist(), key=lambda x: rng.random())
    occ = np.zeros((24, m), dtype=np.int32)
    for t in range(24):  # collisions included: photons land independently
        for r in rng.integers(0, m, n):
            occ[t, r] += 1
    occ[0] = 0
    occ[0, m - 1] = n  # every photon in the last mode
    got = B.outcome_probabilities(itf, modes, occ)
    want = np.array([O.ref_outcome_probability(itf.unitary(), modes, o) for o in occ])
    assert np.array_equal(got, want)
    assert B.outcome_probability(itf, modes, B.OutputPattern(occ[3])) == want[3]


def test_large_mode_count_global_path():
    # m = 2000, n = 6: V = U[:, modes] (192 KB) + the table exceed shared memory,
    # so entries are read from U in global memory. The C ABI takes any matrix.
    m, n = 2000, 6
    rng = np.random.default_rng(5)
    u = (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(m)
    u = np.ascontiguousarray(u)
    modes = np.array([1999, 0, 17, 512, 1024, 3], dtype=np.int32)
    first, count = 123_456_789_012, 3000
    probs = np.empty(count)
    assert N.lib.pl_boson_distribution(m, u.ctypes.data, n, modes.ctypes.data, first, count, probs.ctypes.data, 0,
                                       None) == N.PL_OK, N.last_error()
    rows = np.array([_unrank(m, n, first + t) for t in (0, 1, 2)] + [_unrank(m, n, first + count - 1)], dtype=np.int32)
    want = _oracle_probs(u, modes, rows)
    assert np.array_equal(probs[[0, 1, 2, count - 1]], want)
    # the same patterns through the row-list entry point
    got = np.empty(rows.shape[0])
    lim = pl.Limits().to_c()
    import ctypes as C

    assert N.lib.pl_boson_probabilities(m, u.ctypes.data, n, modes.ctypes.data, rows.shape[0], rows.ctypes.data,
                                        got.ctypes.data, 0, C.byref(lim), None, None) == N.PL_OK
    assert np.array_equal(got, want)


def _unrank(m, n, idx):
    rows = np.zeros(n, dtype=np.int32)
    assert N.lib.pl_boson_unrank_pattern(m, n, idx, rows.ctypes.data) == N.PL_OK
    return rows


def test_malformed_rows():
    import ctypes as C

    import torch

    itf = B.haar_unitary(6, 1)
    u = itf.unitary()
    modes = np.array([0, 1, 2], dtype=np.int32)
    rows = np.array([[0, 1, 2], [2, 1, 0], [0, 0, 6]], dtype=np.int32)  # descending; out of range
    probs = np.empty(3)
    lim = pl.Limits().to_c()
    assert N.lib.pl_boson_probabilities(6, u.ctypes.data, 3, modes.ctypes.data, 3, rows.ctypes.data,
                                        probs.ctypes.data, 0, C.byref(lim), None, None) == N.PL_ERR_ARG
    assert "nondecreasing" in N.last_error()
    # asynchronous device call: NaN for the malformed lists, status bit set
    ud = itf.device_unitary("cuda")
    rd = torch.from_numpy(rows).cuda()
    pd = torch.empty(3, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    flags = N.PL_FLAG_DEVICE_PTRS | N.PL_FLAG_ASYNC
    assert N.lib.pl_boson_probabilities(6, ud.data_ptr(), 3, modes.ctypes.data, 3, rd.data_ptr(), pd.data_ptr(),
                                        flags, C.byref(lim), torch.cuda.current_stream().cuda_stream,
                                        st.data_ptr()) == N.PL_OK
    torch.cuda.synchronize()
    p = pd.cpu().numpy()
    assert np.isfinite(p[0]) and np.isnan(p[1]) and np.isnan(p[2])
    assert int(st.item()) & N.PL_STATUS_BIT_ROWS


@need_ref
def test_sample_matches_reference():
    itf = B.haar_unitary(7, 13)
    modes = [6, 2, 4]
    got = B.sample(itf, modes, 5000, 99)
    want = O.ref_sample(itf.unitary(), modes, 5000, 99)
    assert [p.occupancy for p in got] == [tuple(o) for o in want.tolist()]


def test_sample_golden(bgold):
    g = bgold["sample_haar6_seed3"]
    itf = B.haar_unitary(6, 3)
    d = B.full_distribution(itf, g["input_modes"])
    assert [p.hex() for p in d.probabilities.tolist()] == g["probabilities_hex"]
    assert B.sample_indices(d, g["count"], g["seed"]).tolist() == g["indices"]
