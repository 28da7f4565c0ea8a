"""Python mirror of the reference's boson-sampling API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference's
``permlab::Interferometer`` / ``haar_unitary`` / ``enumerate_patterns`` /
``extract_submatrix`` / ``outcome_probability`` / ``full_distribution`` /
``sample`` (reference ``proj/include/permlab/boson.hpp:30-99``,
``proj/src/boson.cpp``). Every probability is computed on the GPU
(``pl_boson_probabilities`` / ``pl_boson_distribution``: the submatrix
gather, the Store-zechin permanent and |per|^2 / prod occ! fused in one
kernel); host code here validates, enumerates patterns for the returned
objects, and draws samples with the reference's generator
(``std::mt19937_64``, 53-bit uniforms, inverse CDF in enumeration order).
"""
from __future__ import annotations

import ctypes as C
import itertools
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence

import numpy as np

from . import _native as N
from .api import DomainError, Limits, _check

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

UNITARITY_TOL = 1e-10  # reference boson.hpp:31 (kUnitarityTol)
MAX_DISTRIBUTION_PHOTONS = 6  # reference boson.cpp:254-256


@dataclass(frozen=True)
class OutputPattern:
    """Photon occupancy per output mode (reference ``boson.hpp:34-39``)."""

    occupancy: tuple

    def __init__(self, occupancy: Iterable[int]):
        object.__setattr__(self, "occupancy", tuple(int(c) for c in occupancy))

    def total(self) -> int:
        return sum(self.occupancy)

    def rows(self) -> List[int]:
        """The submatrix rows: mode i repeated occupancy[i] times (boson.cpp:213-219)."""
        return [mode for mode, c in enumerate(self.occupancy) for _ in range(c)]


def _check_unitary(u: np.ndarray):
    # reference boson.cpp:47-61: every |(U^+ U)_ij - delta_ij| <= 1e-10
    g = u.conj().T @ u
    if np.max(np.abs(g - np.eye(u.shape[0]))) > UNITARITY_TOL:
        raise DomainError("matrix is not unitary within 1e-10")


class Interferometer:
    """An m-mode linear interferometer given by its unitary (reference
    ``boson.hpp:40-56``; the constructor rejects non-unitary matrices)."""

    def __init__(self, modes: int, unitary):
        if modes < 1:
            raise DomainError("mode count must be >= 1")
        u = np.ascontiguousarray(np.asarray(unitary, dtype=np.complex128))
        if u.ndim != 2 or u.shape[0] != u.shape[1] or u.shape[0] != modes:
            raise DomainError("unitary order must equal the mode count")
        _check_unitary(u)
        self._modes = int(modes)
        self._u = u
        self._u_dev = {}

    def modes(self) -> int:
        return self._modes

    def unitary(self) -> np.ndarray:
        return self._u

    def device_unitary(self, device):
        """The unitary as a device tensor (cached per device)."""
        key = str(device)
        if key not in self._u_dev:
            self._u_dev[key] = torch.from_numpy(self._u).to(device)
        return self._u_dev[key]


def haar_unitary(modes: int, seed: int) -> Interferometer:
    """Haar-random unitary, bitwise the reference's ``haar_unitary``
    (``boson.cpp:149-181``: mt19937_64, Box-Muller, modified Gram-Schmidt)."""
    from . import configs

    if modes < 1:
        raise DomainError("mode count must be >= 1")
    return Interferometer(modes, configs.haar(modes, seed))


def pattern_count(modes: int, photons: int) -> int:
    """C(m + n - 1, n) (0 on 64-bit overflow)."""
    return int(N.lib.pl_boson_pattern_count(modes, photons))


def enumerate_patterns(modes: int, photons: int) -> List[OutputPattern]:
    """All C(m+n-1, n) patterns, ascending mode multisets (reference
    ``boson.cpp:185-205``: mode 0 takes the most photons first)."""
    if modes < 1 or photons < 0:
        raise DomainError("need modes >= 1 and photons >= 0")
    return [OutputPattern(o) for o in pattern_occupancies(modes, photons)]


def pattern_occupancies(modes: int, photons: int) -> np.ndarray:
    """(count, modes) int32 occupancies in enumerate_patterns order."""
    if modes < 1 or photons < 0:
        raise DomainError("need modes >= 1 and photons >= 0")
    if photons == 0:
        return np.zeros((1, modes), dtype=np.int32)
    rows = pattern_rows(modes, photons)
    occ = np.zeros((rows.shape[0], modes), dtype=np.int32)
    idx = np.repeat(np.arange(rows.shape[0]), photons)
    np.add.at(occ, (idx, rows.ravel()), 1)
    return occ


def pattern_rows(modes: int, photons: int, first: int = 0, count: Optional[int] = None) -> np.ndarray:
    """(count, photons) int32 row lists of patterns [first, first + count) in
    enumerate_patterns order: the nondecreasing row sequences in lexicographic
    order, which is itertools.combinations_with_replacement's order (the
    device enumerator unranks the same order, pl_boson_unrank_pattern)."""
    total = pattern_count(modes, photons)
    if count is None:
        count = total - first
    if first < 0 or count < 0 or first + count > total:
        raise DomainError("pattern range outside the distribution")
    it = itertools.islice(itertools.combinations_with_replacement(range(modes), photons), first, first + count)
    flat = np.fromiter(itertools.chain.from_iterable(it), dtype=np.int32, count=count * photons)
    return flat.reshape(count, photons)


def _check_input_modes(input_modes: Sequence[int], modes: int) -> List[int]:
    # reference boson.cpp:63-77
    im = [int(x) for x in input_modes]
    if not im:
        raise DomainError("at least one input mode is required")
    seen = set()
    for x in im:
        if x < 0 or x >= modes:
            raise DomainError("input mode index out of range")
        if x in seen:
            raise DomainError("input modes must be distinct")
        seen.add(x)
    return im


def _check_pattern(out: OutputPattern, modes: int, photons: int):
    # reference boson.cpp:79-92
    if len(out.occupancy) != modes:
        raise DomainError("occupancy vector length must equal the mode count")
    if any(c < 0 for c in out.occupancy):
        raise DomainError("occupancy counts must be nonnegative")
    if out.total() != photons:
        raise DomainError("output photon count does not match the input photon count")


def extract_submatrix(itf: Interferometer, input_modes: Sequence[int], out: OutputPattern) -> np.ndarray:
    """Rows = occupied output modes (repeated by occupancy), columns = input
    modes (reference ``boson.cpp:207-227``)."""
    im = _check_input_modes(input_modes, itf.modes())
    _check_pattern(out, itf.modes(), len(im))
    return np.ascontiguousarray(itf.unitary()[np.ix_(out.rows(), im)])


def _to_rows(itf: Interferometer, im: List[int], patterns) -> np.ndarray:
    if isinstance(patterns, np.ndarray) and patterns.ndim == 2 and patterns.shape[1] == itf.modes():
        occ = patterns.astype(np.int64, copy=False)
        if (occ < 0).any():
            raise DomainError("occupancy counts must be nonnegative")
        if (occ.sum(axis=1) != len(im)).any():
            raise DomainError("output photon count does not match the input photon count")
        rows = np.repeat(np.tile(np.arange(itf.modes(), dtype=np.int32), occ.shape[0]), occ.ravel())
        return rows.reshape(occ.shape[0], len(im))
    pats = list(patterns)
    for p in pats:
        _check_pattern(p, itf.modes(), len(im))
    return np.asarray([p.rows() for p in pats], dtype=np.int32).reshape(len(pats), len(im))


def outcome_probabilities(itf: Interferometer, input_modes: Sequence[int], patterns, limits: Optional[Limits] = None,
                          fma: bool = False) -> np.ndarray:
    """|per(submatrix)|^2 / prod occ! for many patterns in one device call
    (``patterns``: OutputPattern objects or a (count, m) occupancy array)."""
    im = _check_input_modes(input_modes, itf.modes())
    rows = np.ascontiguousarray(_to_rows(itf, im, patterns), dtype=np.int32)
    probs = np.empty(rows.shape[0], dtype=np.float64)
    modes = np.asarray(im, dtype=np.int32)
    lim = (limits or Limits()).to_c()
    flags = N.PL_FLAG_FMA if fma else 0
    _check(N.lib.pl_boson_probabilities(itf.modes(), itf.unitary().ctypes.data, len(im), modes.ctypes.data,
                                        rows.shape[0], rows.ctypes.data, probs.ctypes.data, flags, C.byref(lim),
                                        None, None))
    return probs


def outcome_probability(itf: Interferometer, input_modes: Sequence[int], out: OutputPattern,
                        limits: Optional[Limits] = None) -> float:
    """Reference ``boson.cpp:229-240``."""
    return float(outcome_probabilities(itf, input_modes, [out], limits)[0])


@dataclass
class OutcomeDistribution:
    """Reference ``boson.hpp:78-83``; ``entries`` (pattern, p) pairs in
    enumerate_patterns order are built on first access."""

    input_modes: List[int]
    modes: int
    probabilities: np.ndarray
    _entries: Optional[list] = field(default=None, repr=False)

    @property
    def entries(self):
        if self._entries is None:
            occ = pattern_occupancies(self.modes, len(self.input_modes))
            self._entries = [(OutputPattern(o), float(p)) for o, p in zip(occ, self.probabilities)]
        return self._entries

    def total_probability(self) -> float:
        # left-to-right sum (reference boson.cpp:242-248)
        s = 0.0
        for p in self.probabilities.tolist():
            s += p
        return s


def _distribution_checks(itf: Interferometer, input_modes, limits: Optional[Limits]):
    im = _check_input_modes(input_modes, itf.modes())
    n = len(im)
    if n > MAX_DISTRIBUTION_PHOTONS:
        raise DomainError("full distributions are enumerated for at most 6 photons")
    cap = (limits or Limits()).enumeration_cap
    cnt = pattern_count(itf.modes(), n)
    if cnt == 0 or cnt > cap:
        raise DomainError("outcome count exceeds enumeration_cap")
    return im, cnt


def distribution_probabilities(itf: Interferometer, input_modes: Sequence[int], first: int = 0,
                               count: Optional[int] = None, fma: bool = False, out=None, stream=None, status=None,
                               input_ready: bool = False):
    """Probabilities of patterns [first, first + count) of the full
    distribution, enumerated on the device (no enumeration_cap check: the
    pattern range is the caller's). With a CUDA ``out`` tensor the call runs
    on device buffers (``itf``'s cached device unitary) and, given ``status``,
    is asynchronous on ``stream``. ``input_ready=True`` (``PL_FLAG_INPUT_READY``, device path): the
    unitary is not written by work still running on the stream, so back-to-back calls overlap
    (the kernel computes before ``griddepcontrol.wait`` and stores after it)."""
    im = _check_input_modes(input_modes, itf.modes())
    total = pattern_count(itf.modes(), len(im))
    if count is None:
        count = total - first
    modes = np.asarray(im, dtype=np.int32)
    flags = N.PL_FLAG_FMA if fma else 0
    if torch is not None and isinstance(out, torch.Tensor) and out.is_cuda:
        flags |= N.PL_FLAG_DEVICE_PTRS
        if status is not None:
            flags |= N.PL_FLAG_ASYNC
        if input_ready:
            flags |= N.PL_FLAG_INPUT_READY
        st = (stream or torch.cuda.current_stream(out.device)).cuda_stream
        u = itf.device_unitary(out.device)
        _check(N.lib.pl_boson_distribution(itf.modes(), u.data_ptr(), len(im), modes.ctypes.data, first, count,
                                           out.data_ptr(), flags, st))
        return out
    probs = np.empty(count, dtype=np.float64) if out is None else out
    st = stream.cuda_stream if stream is not None else None
    _check(N.lib.pl_boson_distribution(itf.modes(), itf.unitary().ctypes.data, len(im), modes.ctypes.data, first,
                                       count, probs.ctypes.data, flags, st))
    return probs


def full_distribution(itf: Interferometer, input_modes: Sequence[int], limits: Optional[Limits] = None,
                      fma: bool = False) -> OutcomeDistribution:
    """Exhaustive outcome distribution (reference ``boson.cpp:250-269``)."""
    im, cnt = _distribution_checks(itf, input_modes, limits)
    probs = distribution_probabilities(itf, im, 0, cnt, fma=fma)
    return OutcomeDistribution(input_modes=im, modes=itf.modes(), probabilities=probs)


def _uniform53(seed: int, count: int) -> np.ndarray:
    from . import configs

    raw = configs.mt64_stream(seed, count)
    return (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def sample_indices(dist: OutcomeDistribution, count: int, seed: int) -> np.ndarray:
    """Indices (enumeration order) of `count` inverse-CDF draws (reference
    ``boson.cpp:271-290``): cdf by a left-to-right running sum, draws u from
    mt19937_64(seed) 53-bit uniforms, index = min(upper_bound(cdf, u), size-1)."""
    cdf = np.cumsum(dist.probabilities)  # sequential left fold, as the reference's acc += p
    u = _uniform53(seed, count)
    idx = np.searchsorted(cdf, u, side="right")
    return np.minimum(idx, cdf.shape[0] - 1)


def sample(itf: Interferometer, input_modes: Sequence[int], count: int, seed: int,
           limits: Optional[Limits] = None) -> List[OutputPattern]:
    dist = full_distribution(itf, input_modes, limits)
    idx = sample_indices(dist, count, seed)
    occ = pattern_occupancies(itf.modes(), len(dist.input_modes))
    return [OutputPattern(occ[i]) for i in idx]
