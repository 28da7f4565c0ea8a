"""Python mirror of the reference's Store-zechin API over the B200 C ABI.

Same names, argument meaning and error behaviour as the reference's
``permlab::store_zechin_permanent`` / ``store_zechin_run`` /
``store_zechin_attributed`` (reference ``proj/include/permlab/permanent.hpp:34-96``),
plus the batch entry point the reference's callers write by hand
(``proj/src/boson.cpp:262-265``). Every value is computed on the GPU; host
code here only validates, moves buffers and maps status codes to
:class:`DomainError` (reference ``errors.hpp:24-27``).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N

try:  # torch is plumbing only (device buffers, streams); optional for host arrays
    import torch
except Exception:  # pragma: no cover
    torch = None


class DomainError(ValueError):
    """Contract violation or exceeded limit (reference ``permlab::DomainError``)."""


class DeviceError(RuntimeError):
    """CUDA / device failure (no device, out of memory, launch error)."""


@dataclass
class Limits:
    """Resource guards (reference ``limits.hpp:23-33``). ``subset_order_limit``
    defaults to the device cap 34 (reference: 30, mask cap 31);
    ``memo_budget_bytes`` caps device layer scratch (0 = uncapped)."""

    naive_order_limit: int = 12
    subset_order_limit: int = N.PL_MAX_ORDER
    enumeration_cap: int = 100000
    memo_budget_bytes: int = 0
    num_gpus: int = 0  # 0: current device; g >= 1: devices 0..g-1 (sharded layer DP / split batch)

    @staticmethod
    def from_env() -> "Limits":
        """``PERMLAB_LIMITS=key=value,...`` (reference ``limits.cpp:43-76``)."""
        lim = Limits()
        raw = os.environ.get("PERMLAB_LIMITS")
        if raw is None:
            return lim
        for item in raw.split(","):
            if not item:
                continue
            if "=" not in item:
                raise DomainError(f"PERMLAB_LIMITS: expected key=value, got '{item}'")
            key, value = item.split("=", 1)
            if not value:
                raise DomainError(f"PERMLAB_LIMITS: empty value for {key}")
            if not value.isdigit():
                raise DomainError(f"PERMLAB_LIMITS: non-numeric value for {key}")
            if key not in ("naive_order_limit", "subset_order_limit", "enumeration_cap", "memo_budget_bytes",
                           "num_gpus"):
                raise DomainError(f"PERMLAB_LIMITS: unknown key '{key}'")
            setattr(lim, key, int(value))
        return lim

    def to_c(self) -> N.pl_limits:
        return N.pl_limits(int(self.subset_order_limit), int(self.memo_budget_bytes), int(self.num_gpus))


@dataclass(frozen=True)
class OpCount:
    multiplications: int = 0
    additions: int = 0

    def __add__(self, o: "OpCount") -> "OpCount":
        return OpCount(self.multiplications + o.multiplications, self.additions + o.additions)


@dataclass
class PermanentResult:
    value: object
    counts: OpCount
    algorithm: str = "store-zechin"


@dataclass
class AttributionReport:
    per_term: list = field(default_factory=list)
    final_combination_adds: int = 0
    totals: OpCount = OpCount()


@dataclass
class StoreZechinRun:
    result: PermanentResult
    attribution: AttributionReport
    cache_misses: int
    distinct_subsets: int


_DTYPES = {np.dtype(np.int64): N.PL_I64, np.dtype(np.float64): N.PL_F64, np.dtype(np.complex128): N.PL_C128}


def _raise(status: int):
    msg = N.last_error()
    if status in (N.PL_ERR_ARG, N.PL_ERR_LIMIT, N.PL_ERR_OVERFLOW):
        raise DomainError(msg)
    raise DeviceError(f"{N.STATUS_NAMES.get(status, status)}: {msg}")


def _check(status: int):
    if status != N.PL_OK:
        _raise(status)


def store_zechin_counts(n: int) -> OpCount:
    m, a = C.c_uint64(), C.c_uint64()
    _check(N.lib.pl_sz_counts(int(n), C.byref(m), C.byref(a)))
    return OpCount(m.value, a.value)


def _as_matrix(a) -> np.ndarray:
    arr = np.asarray(a)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise DomainError("entry count does not match order^2")
    if arr.shape[0] < 1:
        raise DomainError("matrix order must be >= 1")
    if arr.dtype.kind in "ib" or (arr.dtype.kind == "u" and arr.dtype.itemsize < 8):
        arr = arr.astype(np.int64)
    elif arr.dtype.kind == "u" or (arr.dtype == object and all(isinstance(v, (int, np.integer)) for v in arr.flat)):
        # Python integers / uint64: int64 when they fit, else an object matrix for the residue path
        vals = [int(v) for v in arr.flat]
        if all(-(1 << 63) <= v < (1 << 63) for v in vals):
            arr = np.array(vals, dtype=np.int64).reshape(arr.shape)
        else:
            arr = np.array(vals, dtype=object).reshape(arr.shape)
            return arr
    elif arr.dtype.kind == "f":
        arr = arr.astype(np.float64)
    elif arr.dtype.kind == "c":
        arr = arr.astype(np.complex128)
    else:
        raise DomainError(f"unsupported entry type {arr.dtype}")
    return np.ascontiguousarray(arr)


def _bigint_from_int64(m: np.ndarray, lim, ryser: bool = False) -> int:
    """Exact permanent of an int64 matrix whose intermediates leave int64
    (``pl_sz_permanent_bigint``: residue passes on the device, CRT in the library)."""
    n = m.shape[0]
    cap = 40
    limbs = np.zeros(cap, dtype=np.uint64)
    nl, neg = C.c_size_t(0), C.c_int32(0)
    fn = N.lib.pl_ryser_permanent_bigint if ryser else N.lib.pl_sz_permanent_bigint
    _check(fn(n, m.ctypes.data, limbs.ctypes.data, cap, C.byref(nl), C.byref(neg), C.byref(lim), None))
    v = 0
    for i in reversed(range(nl.value)):
        v = (v << 64) | int(limbs[i])
    return -v if neg.value else v


def _bigint_from_objects(m: np.ndarray, lim, ryser: bool = False) -> int:
    """Exact permanent of a matrix of Python integers of any size: residues modulo the
    engine's primes go through ``pl_sz_permanent_modp``; the CRT runs on Python integers."""
    n = m.shape[0]
    rows = [[int(v) for v in r] for r in m]
    bound = 1
    for r in rows:
        bound *= sum(abs(v) for v in r)
    k = max(1, (bound.bit_length() + 2 + 29) // 30)
    primes = np.zeros(k, dtype=np.uint32)
    if N.lib.pl_bigint_primes(k, primes.ctypes.data) != k:
        raise DeviceError("pl_bigint_primes failed")
    res = np.array([[[v % int(p) for v in r] for r in rows] for p in primes], dtype=np.int64)
    out = np.zeros(k, dtype=np.uint32)
    fn = N.lib.pl_ryser_permanent_modp if ryser else N.lib.pl_sz_permanent_modp
    _check(fn(n, k, primes.ctypes.data, res.ctypes.data, out.ctypes.data, C.byref(lim), None))
    x, mod = 0, 1
    for p, r in zip((int(p) for p in primes), (int(r) for r in out)):
        x += mod * (((r - x) * pow(mod, -1, p)) % p)
        mod *= p
    return x - mod if 2 * x > mod else x


def _py_value(arr: np.ndarray, i: int = 0):
    v = arr.reshape(-1)[i]
    if arr.dtype == np.int64:
        return int(v)
    if arr.dtype == np.float64:
        return float(v)
    return complex(v)


def store_zechin_permanent(a, limits: Optional[Limits] = None, fma: bool = False) -> PermanentResult:
    """Permanent of one square matrix (reference ``permanent.hpp:90``).

    Integer matrices are exact at any magnitude, like the reference's
    arbitrary-precision Int ring (``ring.hpp:29-31``): when the int64 guard
    reports an overflow (or the entries themselves exceed int64) the layer DP
    runs on residues modulo enough 31-bit primes and the result is recombined
    (``csrc/bigint.cu``)."""
    m = _as_matrix(a)
    n = m.shape[0]
    lim = (limits or Limits()).to_c()
    if m.dtype == object:
        return PermanentResult(_bigint_from_objects(m, lim), store_zechin_counts(n))
    out = np.zeros(1, dtype=m.dtype)
    flags = N.PL_FLAG_FMA if fma else 0
    status = N.lib.pl_sz_permanent(_DTYPES[m.dtype], n, m.ctypes.data, out.ctypes.data, flags, C.byref(lim), None)
    if status == N.PL_ERR_OVERFLOW and m.dtype == np.int64:
        return PermanentResult(_bigint_from_int64(m, lim), store_zechin_counts(n))
    _check(status)
    return PermanentResult(_py_value(out), store_zechin_counts(n))


def ryser_counts(n: int) -> OpCount:
    """Ryser operation counts (reference ``cost_model.cpp:168-174``)."""
    m, a = C.c_uint64(), C.c_uint64()
    _check(N.lib.pl_ryser_counts(int(n), C.byref(m), C.byref(a)))
    return OpCount(m.value, a.value)


def ryser_permanent(a, limits: Optional[Limits] = None) -> PermanentResult:
    """Permanent by Ryser's formula on the device (reference ``permanent.hpp:84``,
    ``permanent.cpp:85-136``): float rings bitwise the reference's visit-order
    fold; integers exact at any magnitude (128-bit wrapping sums where the
    guard bound allows, else inclusion-exclusion on residues, ``csrc/bigint.cu``)."""
    m = _as_matrix(a)
    n = m.shape[0]
    lim = (limits or Limits()).to_c()
    if m.dtype == object:
        return PermanentResult(_bigint_from_objects(m, lim, ryser=True), ryser_counts(n), "ryser")
    out = np.zeros(1, dtype=m.dtype)
    status = N.lib.pl_ryser_permanent(_DTYPES[m.dtype], n, m.ctypes.data, out.ctypes.data, 0, C.byref(lim), None)
    if status == N.PL_ERR_OVERFLOW and m.dtype == np.int64:
        return PermanentResult(_bigint_from_int64(m, lim, ryser=True), ryser_counts(n), "ryser")
    _check(status)
    return PermanentResult(_py_value(out), ryser_counts(n), "ryser")


def store_zechin_attributed(a, limits: Optional[Limits] = None) -> AttributionReport:
    """Per-term cost split of the reference's DFS order (``permanent.cpp:179-199``),
    in closed form: term j first demands the subsets T of full\\{j} that
    contain {0..j-1}, 2 <= |T| <= n-1."""
    m = _as_matrix(a)
    n = m.shape[0]
    lim = limits or Limits()
    if n < 3:
        raise DomainError("attribution needs order >= 3; orders 1 and 2 are base cases")
    if n > lim.subset_order_limit:
        raise DomainError(f"matrix order exceeds subset_order_limit ({lim.subset_order_limit})")
    from math import comb

    per_term = []
    for j in range(n):
        mults, adds = 1, 0
        free = n - 1 - j
        for u in range(free + 1):
            t = j + u
            if t < 2 or t > n - 1:
                continue
            cm, ca = (2, 1) if t == 2 else (t, t - 1)
            mults += comb(free, u) * cm
            adds += comb(free, u) * ca
        per_term.append(OpCount(mults, adds))
    totals = OpCount()
    for t in per_term:
        totals = totals + t
    totals = totals + OpCount(0, n - 1)
    return AttributionReport(per_term, n - 1, totals)


def store_zechin_run(a, limits: Optional[Limits] = None) -> StoreZechinRun:
    """Full-detail entry point (reference ``permanent.hpp:96``)."""
    res = store_zechin_permanent(a, limits)
    n = np.asarray(a).shape[0]
    misses, distinct = C.c_uint64(), C.c_uint64()
    _check(N.lib.pl_sz_diagnostics(n, C.byref(misses), C.byref(distinct)))
    attribution = store_zechin_attributed(a, limits) if n >= 3 else AttributionReport([], 0, res.counts)
    return StoreZechinRun(res, attribution, misses.value, distinct.value)


def _torch_dtype_code(t) -> int:
    if t.dtype == torch.int64:
        return N.PL_I64
    if t.dtype == torch.float64:
        return N.PL_F64
    if t.dtype == torch.complex128:
        return N.PL_C128
    raise DomainError(f"unsupported entry type {t.dtype}")


def store_zechin_permanent_batch(a, limits: Optional[Limits] = None, out=None, fma: bool = False,
                                 stream=None, status=None, input_ready: bool = False):
    """Permanents of a batch ``(count, n, n)``.

    * numpy array (host): returns a numpy array of ``count`` values; the copy
      to and from the device happens inside the call.
    * torch tensor on CUDA: computed in place on the device; ``out`` (a CUDA
      tensor of ``count`` values) may be given; ``stream`` is a
      ``torch.cuda.Stream`` (default: the current stream). With ``status`` (a
      CUDA int32 tensor of one element, zeroed by the caller) the call is
      asynchronous and int64 overflow is reported there.
      ``input_ready=True`` (``PL_FLAG_INPUT_READY``) states that ``a`` is not written by work
      still running on the stream: consecutive batch kernels of orders <= 5 then overlap their
      load ramp with the previous kernel's tail (same results).
    * torch tensor on CPU (pinned or not): host path like numpy.
    """
    lim = (limits or Limits()).to_c()
    flags = N.PL_FLAG_FMA if fma else 0
    if torch is not None and isinstance(a, torch.Tensor):
        if a.dim() != 3 or a.shape[1] != a.shape[2]:
            raise DomainError("batch must have shape (count, n, n)")
        count, n = int(a.shape[0]), int(a.shape[1])
        code = _torch_dtype_code(a)
        a = a.contiguous()
        if out is None:
            out = torch.empty(count, dtype=a.dtype, device=a.device, pin_memory=False)
        if a.is_cuda:
            if not out.is_cuda:
                raise DomainError("device input needs a device output")
            flags |= N.PL_FLAG_DEVICE_PTRS
            if input_ready:
                flags |= N.PL_FLAG_INPUT_READY
            st = (stream or torch.cuda.current_stream(a.device)).cuda_stream
            status_ptr = None
            if status is not None:
                flags |= N.PL_FLAG_ASYNC
                status_ptr = status.data_ptr()
            _check(N.lib.pl_sz_permanent_batch(code, n, count, a.data_ptr(), out.data_ptr(), flags, C.byref(lim),
                                               st, status_ptr))
            return out
        st = stream.cuda_stream if stream is not None else None
        _check(N.lib.pl_sz_permanent_batch(code, n, count, a.data_ptr(), out.data_ptr(), flags, C.byref(lim), st,
                                           None))
        return out
    arr = np.asarray(a)
    if arr.ndim != 3 or arr.shape[1] != arr.shape[2]:
        raise DomainError("batch must have shape (count, n, n)")
    arr = np.ascontiguousarray(arr)
    if arr.dtype not in _DTYPES:
        raise DomainError(f"unsupported entry type {arr.dtype}")
    count, n = arr.shape[0], arr.shape[1]
    res = np.empty(count, dtype=arr.dtype) if out is None else out
    _check(N.lib.pl_sz_permanent_batch(_DTYPES[arr.dtype], n, count, arr.ctypes.data, res.ctypes.data, flags,
                                       C.byref(lim), None, None))
    return res


def binom(s: int, k: int) -> int:
    return int(N.lib.pl_binom(s, k))


def colex_rank(mask: int) -> int:
    return int(N.lib.pl_colex_rank(mask))


def colex_unrank(k: int, rank: int) -> int:
    return int(N.lib.pl_colex_unrank(k, rank))


def scratch_bytes(dtype, n: int) -> int:
    return int(N.lib.pl_sz_scratch_bytes(_DTYPES[np.dtype(dtype)], n))


def release_scratch() -> None:
    """Free the idle layer scratch the large-order path keeps cached between
    calls (``pl_release_scratch``)."""
    N.lib.pl_release_scratch()


def version() -> str:
    return N.lib.pl_version().decode()


def device_count() -> int:
    return int(N.lib.pl_device_count())
