"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

* ``liboracle.so``: the C restatement of the reference Store-zechin DP
  (``oracle/sz_oracle.c``, citing reference ``proj/src/permanent.cpp``).
* ``_ref/libpermlab_ref.so``: the reference engine itself, compiled from
  ``/root/reference/proj/src`` against the Boost shim (``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module, and only as the checker / timed CPU baseline. The product
(``paper_1802_02779_b200``) never imports it and has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_ORACLE_SO = HERE / "liboracle.so"
_REF_SO = HERE / "_ref" / "libpermlab_ref.so"

_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_dp = C.POINTER(C.c_double)


def _ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(ctype)


class OracleError(RuntimeError):
    pass


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not _ORACLE_SO.exists():
            raise OracleError(f"{_ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(_ORACLE_SO))
        L.orc_sz_i64.argtypes = [C.c_int, _i64p, _i64p, _i64p, C.c_int]
        L.orc_sz_f64.argtypes = [C.c_int, _dp, _dp, C.c_int]
        L.orc_sz_c128.argtypes = [C.c_int, _dp, _dp, C.c_int]
        L.orc_sz_batch_i64.argtypes = [C.c_int, C.c_int64, _i64p, _i64p, C.c_int]
        L.orc_sz_batch_f64.argtypes = [C.c_int, C.c_int64, _dp, _dp, C.c_int]
        L.orc_sz_batch_c128.argtypes = [C.c_int, C.c_int64, _dp, _dp, C.c_int]
        L.orc_sz_layer_f64.argtypes = [C.c_int, _dp, C.c_int, _dp]
        L.orc_ryser_f64.argtypes = [C.c_int, _dp, _dp]
        L.orc_ryser_c128.argtypes = [C.c_int, _dp, _dp]
        L.orc_ryser_i64.argtypes = [C.c_int, _i64p, _i64p, _i64p]
        L.orc_binom.argtypes = [C.c_int, C.c_int]
        L.orc_binom.restype = C.c_uint64
        L.orc_colex_rank.argtypes = [C.c_uint64]
        L.orc_colex_rank.restype = C.c_uint64
        L.orc_colex_unrank.argtypes = [C.c_int, C.c_uint64]
        L.orc_colex_unrank.restype = C.c_uint64
        _lib = L
    return _lib


def ref_available() -> bool:
    return _REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        if not _REF_SO.exists():
            raise OracleError(f"{_REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        R = C.CDLL(str(_REF_SO))
        R.ref_last_error.restype = C.c_char_p
        R.ref_sz_i64.argtypes = [C.c_int, _i64p, _i64p, _i64p, _u64p, _u64p, C.c_int, C.c_uint64]
        R.ref_sz_c128.argtypes = [C.c_int, _dp, _dp, _u64p, _u64p, C.c_int, C.c_uint64]
        R.ref_sz_f64.argtypes = [C.c_int, _dp, _dp, C.c_int, C.c_uint64]
        R.ref_sz_run_i64.argtypes = [C.c_int, _i64p, _i64p, _i64p, _u64p, _u64p, _u64p, _u64p]
        R.ref_naive_i64.argtypes = [C.c_int, _i64p, _i64p, _i64p]
        R.ref_ryser_i64.argtypes = [C.c_int, _i64p, _i64p, _i64p]
        R.ref_ryser_c128.argtypes = [C.c_int, _dp, _dp]
        R.ref_sz_batch_i64.argtypes = [C.c_int, C.c_int64, _i64p, _i64p, C.c_int]
        R.ref_sz_batch_c128.argtypes = [C.c_int, C.c_int64, _dp, _dp, C.c_int]
        R.ref_sz_batch_f64.argtypes = [C.c_int, C.c_int64, _dp, _dp, C.c_int, C.c_uint64]
        R.ref_haar.argtypes = [C.c_int, C.c_uint64, _dp]
        _ip = C.POINTER(C.c_int)
        R.ref_outcome_probability.argtypes = [C.c_int, _dp, C.c_int, _ip, _ip, _dp]
        R.ref_full_distribution.argtypes = [C.c_int, _dp, C.c_int, _ip, C.c_uint64, _i64p, _ip, _dp]
        R.ref_sample.argtypes = [C.c_int, _dp, C.c_int, _ip, C.c_uint64, C.c_uint64, C.c_uint64, _ip]
        R.ref_enumerate_patterns.argtypes = [C.c_int, C.c_int, _i64p, _ip]
        cp, sz = C.c_char_p, C.c_size_t
        R.ref_fmt_value_text.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, cp, sz]
        R.ref_fmt_perm_json.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_uint64,
                                        cp, sz]
        R.ref_fmt_dist_json.argtypes = [C.c_int, C.c_int, C.c_int64, _ip, _dp, cp, sz]
        R.ref_fmt_sample_json.argtypes = [C.c_int, C.c_int64, _ip, cp, sz]
        R.ref_fmt_itf_json.argtypes = [C.c_int, _dp, cp, sz]
        R.ref_parse_matrix.argtypes = [cp, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), _i64p, _dp,
                                       C.c_int]
        _ref = R
    return _ref


def _threads(nthreads):
    return int(nthreads) if nthreads else (os.cpu_count() or 1)


def _lohi_to_int(lo: int, hi: int) -> int:
    return (int(hi) << 64) | (int(lo) & ((1 << 64) - 1))


# ----------------------------------------------------------------- restatement

def sz_int(a: np.ndarray, nthreads: int | None = None) -> int:
    """Exact Store-zechin permanent of an integer matrix (Python int)."""
    a = np.ascontiguousarray(a, dtype=np.int64)
    n = a.shape[0]
    lo, hi = C.c_int64(), C.c_int64()
    rc = lib().orc_sz_i64(n, _ptr(a, _i64p), C.byref(lo), C.byref(hi), _threads(nthreads))
    if rc != 0:
        raise OracleError(f"orc_sz_i64 status {rc}")
    return _lohi_to_int(lo.value, hi.value)


def sz_f64(a: np.ndarray, nthreads: int | None = None) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = C.c_double()
    rc = lib().orc_sz_f64(a.shape[0], _ptr(a, _dp), C.byref(out), _threads(nthreads))
    if rc != 0:
        raise OracleError(f"orc_sz_f64 status {rc}")
    return out.value


def sz_c128(a: np.ndarray, nthreads: int | None = None) -> complex:
    a = np.ascontiguousarray(a, dtype=np.complex128)
    out = np.zeros(2, dtype=np.float64)
    rc = lib().orc_sz_c128(a.shape[0], _ptr(a.view(np.float64), _dp), _ptr(out, _dp), _threads(nthreads))
    if rc != 0:
        raise OracleError(f"orc_sz_c128 status {rc}")
    return complex(out[0], out[1])


def sz_batch(a: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    """Batch (count, n, n) -> (count,) in the input's ring. Integer batches
    return int64 and raise if any exact value leaves int64."""
    count, n = a.shape[0], a.shape[1]
    L = lib()
    if a.dtype == np.int64:
        a = np.ascontiguousarray(a)
        lohi = np.zeros((count, 2), dtype=np.int64)
        rc = L.orc_sz_batch_i64(n, count, _ptr(a, _i64p), _ptr(lohi, _i64p), _threads(nthreads))
        if rc != 0:
            raise OracleError(f"orc_sz_batch_i64 status {rc}")
        lo, hi = lohi[:, 0], lohi[:, 1]
        if not np.all(hi == (lo >> 63)):
            raise OracleError("exact permanent outside int64")
        return lo.copy()
    if a.dtype == np.float64:
        a = np.ascontiguousarray(a)
        out = np.zeros(count, dtype=np.float64)
        rc = L.orc_sz_batch_f64(n, count, _ptr(a, _dp), _ptr(out, _dp), _threads(nthreads))
    elif a.dtype == np.complex128:
        a = np.ascontiguousarray(a)
        out = np.zeros(count, dtype=np.complex128)
        rc = L.orc_sz_batch_c128(n, count, _ptr(a.view(np.float64), _dp), _ptr(out.view(np.float64), _dp),
                                 _threads(nthreads))
    else:
        raise TypeError(a.dtype)
    if rc != 0:
        raise OracleError(f"oracle batch status {rc}")
    return out


def ryser(a: np.ndarray):
    """Restated reference Ryser (visit-order fold, sz_oracle.c): int / float / complex."""
    a = np.ascontiguousarray(a)
    n = a.shape[0]
    if a.dtype == np.int64:
        lo, hi = C.c_int64(), C.c_int64()
        if lib().orc_ryser_i64(n, _ptr(a, _i64p), C.byref(lo), C.byref(hi)):
            raise OracleError("128-bit overflow")
        return _lohi_to_int(lo.value, hi.value)
    if a.dtype == np.float64:
        out = np.zeros(1)
        lib().orc_ryser_f64(n, _ptr(a, _dp), _ptr(out, _dp))
        return float(out[0])
    out = np.zeros(2)
    lib().orc_ryser_c128(n, _ptr(a.view(np.float64), _dp), _ptr(out, _dp))
    return complex(out[0], out[1])


def ref_ryser_c128(a: np.ndarray) -> complex:
    """The reference engine's ryser_permanent on a complex (or real) matrix."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    out = np.zeros(2)
    rc = ref().ref_ryser_c128(a.shape[0], _ptr(a.view(np.float64), _dp), _ptr(out, _dp))
    if rc:
        raise _ref_err(rc)
    return complex(out[0], out[1])


def sz_layer_f64(a: np.ndarray, k: int) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = a.shape[0]
    out = np.zeros(int(lib().orc_binom(n, k)), dtype=np.float64)
    rc = lib().orc_sz_layer_f64(n, _ptr(a, _dp), k, _ptr(out, _dp))
    if rc != 0:
        raise OracleError(f"orc_sz_layer_f64 status {rc}")
    return out


def binom(s: int, l: int) -> int:
    return int(lib().orc_binom(s, l))


def colex_rank(mask: int) -> int:
    return int(lib().orc_colex_rank(mask))


def colex_unrank(k: int, rank: int) -> int:
    return int(lib().orc_colex_unrank(k, rank))


# ----------------------------------------------------------------- reference

def _ref_err(rc: int) -> OracleError:
    return OracleError(f"reference status {rc}: {ref().ref_last_error().decode()}")


def ref_sz_int(a: np.ndarray, subset_order_limit: int = 0, memo_budget_bytes: int = 0):
    """(value, (mults, adds)) from the reference's store_zechin_permanent."""
    a = np.ascontiguousarray(a, dtype=np.int64)
    lo, hi = C.c_int64(), C.c_int64()
    m, d = C.c_uint64(), C.c_uint64()
    rc = ref().ref_sz_i64(a.shape[0], _ptr(a, _i64p), C.byref(lo), C.byref(hi), C.byref(m), C.byref(d),
                          subset_order_limit, memo_budget_bytes)
    if rc != 0:
        raise _ref_err(rc)
    return _lohi_to_int(lo.value, hi.value), (m.value, d.value)


def ref_sz_c128(a: np.ndarray, subset_order_limit: int = 0, memo_budget_bytes: int = 0):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    out = np.zeros(2, dtype=np.float64)
    m, d = C.c_uint64(), C.c_uint64()
    rc = ref().ref_sz_c128(a.shape[0], _ptr(a.view(np.float64), _dp), _ptr(out, _dp), C.byref(m), C.byref(d),
                           subset_order_limit, memo_budget_bytes)
    if rc != 0:
        raise _ref_err(rc)
    return complex(out[0], out[1]), (m.value, d.value)


def ref_sz_f64(a: np.ndarray, memo_budget_bytes: int = 0) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = C.c_double()
    rc = ref().ref_sz_f64(a.shape[0], _ptr(a, _dp), C.byref(out), 0, memo_budget_bytes)
    if rc != 0:
        raise _ref_err(rc)
    return out.value


def ref_sz_run_int(a: np.ndarray):
    a = np.ascontiguousarray(a, dtype=np.int64)
    n = a.shape[0]
    lo, hi = C.c_int64(), C.c_int64()
    misses, distinct, fin = C.c_uint64(), C.c_uint64(), C.c_uint64()
    per_term = np.zeros(2 * max(n, 1), dtype=np.uint64)
    rc = ref().ref_sz_run_i64(n, _ptr(a, _i64p), C.byref(lo), C.byref(hi), C.byref(misses), C.byref(distinct),
                              _ptr(per_term, _u64p), C.byref(fin))
    if rc != 0:
        raise _ref_err(rc)
    terms = [(int(per_term[2 * t]), int(per_term[2 * t + 1])) for t in range(n)] if n >= 3 else []
    return {
        "value": _lohi_to_int(lo.value, hi.value),
        "cache_misses": misses.value,
        "distinct_subsets": distinct.value,
        "per_term": terms,
        "final_combination_adds": fin.value,
    }


def ref_naive_int(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a, dtype=np.int64)
    lo, hi = C.c_int64(), C.c_int64()
    rc = ref().ref_naive_i64(a.shape[0], _ptr(a, _i64p), C.byref(lo), C.byref(hi))
    if rc != 0:
        raise _ref_err(rc)
    return _lohi_to_int(lo.value, hi.value)


def ref_ryser_int(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a, dtype=np.int64)
    lo, hi = C.c_int64(), C.c_int64()
    rc = ref().ref_ryser_i64(a.shape[0], _ptr(a, _i64p), C.byref(lo), C.byref(hi))
    if rc != 0:
        raise _ref_err(rc)
    return _lohi_to_int(lo.value, hi.value)


def ref_sz_batch(a: np.ndarray, nthreads: int | None = None, memo_budget_bytes: int = 0) -> np.ndarray:
    """The reference's own store_zechin_permanent over a batch (threads over
    contiguous chunks). Integer results must fit int64."""
    count, n = a.shape[0], a.shape[1]
    R = ref()
    if a.dtype == np.int64:
        a = np.ascontiguousarray(a)
        lohi = np.zeros((count, 2), dtype=np.int64)
        rc = R.ref_sz_batch_i64(n, count, _ptr(a, _i64p), _ptr(lohi, _i64p), _threads(nthreads))
        if rc != 0:
            raise _ref_err(rc)
        return lohi[:, 0].copy()
    if a.dtype == np.complex128:
        a = np.ascontiguousarray(a)
        out = np.zeros(count, dtype=np.complex128)
        rc = R.ref_sz_batch_c128(n, count, _ptr(a.view(np.float64), _dp), _ptr(out.view(np.float64), _dp),
                                 _threads(nthreads))
    elif a.dtype == np.float64:
        a = np.ascontiguousarray(a)
        out = np.zeros(count, dtype=np.float64)
        rc = R.ref_sz_batch_f64(n, count, _ptr(a, _dp), _ptr(out, _dp), _threads(nthreads), memo_budget_bytes)
    else:
        raise TypeError(a.dtype)
    if rc != 0:
        raise _ref_err(rc)
    return out


def ref_haar(m: int, seed: int) -> np.ndarray:
    u = np.zeros((m, m), dtype=np.complex128)
    rc = ref().ref_haar(m, seed, _ptr(u.view(np.float64), _dp))
    if rc != 0:
        raise _ref_err(rc)
    return u


# ----------------------------------------------------------------- boson sampling (reference)
# Reference include/permlab/boson.hpp:67-99, src/boson.cpp:185-290. `u` is the
# m x m unitary (complex128); occupancies are (count, m) int32 arrays.

def _u_arg(u):
    u = np.ascontiguousarray(u, dtype=np.complex128)
    return u, _ptr(u.view(np.float64), _dp)


def _modes_arg(modes):
    a = np.ascontiguousarray(modes, dtype=np.int32)
    return a, _ptr(a, C.POINTER(C.c_int))


def ref_outcome_probability(u, input_modes, occupancy) -> float:
    u, up = _u_arg(u)
    im, imp = _modes_arg(input_modes)
    oc, ocp = _modes_arg(occupancy)
    p = C.c_double()
    rc = ref().ref_outcome_probability(u.shape[0], up, len(im), imp, ocp, C.byref(p))
    if rc != 0:
        raise _ref_err(rc)
    return p.value


def ref_full_distribution(u, input_modes, enumeration_cap: int = 0):
    """(occupancies (count, m) int32, probabilities (count,) float64)."""
    u, up = _u_arg(u)
    im, imp = _modes_arg(input_modes)
    m = u.shape[0]
    cnt = C.c_int64()
    R = ref()
    rc = R.ref_full_distribution(m, up, len(im), imp, enumeration_cap, C.byref(cnt), None, None)
    if rc != 0:
        raise _ref_err(rc)
    occ = np.zeros((cnt.value, m), dtype=np.int32)
    probs = np.zeros(cnt.value, dtype=np.float64)
    rc = R.ref_full_distribution(m, up, len(im), imp, enumeration_cap, C.byref(cnt), _ptr(occ, C.POINTER(C.c_int)),
                                 _ptr(probs, _dp))
    if rc != 0:
        raise _ref_err(rc)
    return occ, probs


def ref_sample(u, input_modes, count: int, seed: int, enumeration_cap: int = 0) -> np.ndarray:
    u, up = _u_arg(u)
    im, imp = _modes_arg(input_modes)
    occ = np.zeros((count, u.shape[0]), dtype=np.int32)
    rc = ref().ref_sample(u.shape[0], up, len(im), imp, count, seed, enumeration_cap, _ptr(occ, C.POINTER(C.c_int)))
    if rc != 0:
        raise _ref_err(rc)
    return occ


def ref_enumerate_patterns(m: int, n: int) -> np.ndarray:
    cnt = C.c_int64()
    R = ref()
    rc = R.ref_enumerate_patterns(m, n, C.byref(cnt), None)
    if rc != 0:
        raise _ref_err(rc)
    occ = np.zeros((cnt.value, m), dtype=np.int32)
    rc = R.ref_enumerate_patterns(m, n, C.byref(cnt), _ptr(occ, C.POINTER(C.c_int)))
    if rc != 0:
        raise _ref_err(rc)
    return occ


# ----------------------------------------------------------------- CLI formats (reference primitives)

def _fmt_call(fn, *args) -> str:
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        rc = fn(*args, buf, cap)
        if rc == 0:
            return buf.value.decode()
        if rc < 0:
            raise _ref_err(-rc)
        cap = max(cap * 2, rc)


def ref_fmt_value_text(v) -> str:
    if isinstance(v, (int, np.integer)):
        return _fmt_call(ref().ref_fmt_value_text, 0, int(v), 0.0, 0.0)
    z = complex(v)
    return _fmt_call(ref().ref_fmt_value_text, 1, 0, z.real, z.imag)


def ref_fmt_perm_json(v, order: int, mults: int, adds: int) -> str:
    if isinstance(v, (int, np.integer)):
        return _fmt_call(ref().ref_fmt_perm_json, 0, int(v), 0.0, 0.0, order, mults, adds)
    z = complex(v)
    return _fmt_call(ref().ref_fmt_perm_json, 1, 0, z.real, z.imag, order, mults, adds)


def ref_fmt_dist_json(m: int, photons: int, occupancy: np.ndarray, probs: np.ndarray) -> str:
    occ = np.ascontiguousarray(occupancy, dtype=np.int32)
    pr = np.ascontiguousarray(probs, dtype=np.float64)
    return _fmt_call(ref().ref_fmt_dist_json, m, photons, occ.shape[0], _ptr(occ, C.POINTER(C.c_int)), _ptr(pr, _dp))


def ref_fmt_sample_json(occupancy: np.ndarray) -> str:
    occ = np.ascontiguousarray(occupancy, dtype=np.int32)
    return _fmt_call(ref().ref_fmt_sample_json, occ.shape[1], occ.shape[0], _ptr(occ, C.POINTER(C.c_int)))


def ref_fmt_itf_json(u: np.ndarray) -> str:
    u, up = _u_arg(u)
    return _fmt_call(ref().ref_fmt_itf_json, u.shape[0], up)


def ref_parse_matrix(text: str, csv: bool, csv_complex: bool = False):
    """(order, ring 'int'|'complex'|'rational', entries) parsed by the reference."""
    cap = 4096
    ints = np.zeros(cap, dtype=np.int64)
    cplx = np.zeros(2 * cap, dtype=np.float64)
    order, ring = C.c_int(), C.c_int()
    rc = ref().ref_parse_matrix(text.encode(), int(csv), int(csv_complex), C.byref(order), C.byref(ring),
                                _ptr(ints, _i64p), _ptr(cplx, _dp), cap)
    if rc != 0:
        raise _ref_err(rc)
    n = order.value
    if ring.value == 0:
        return n, "int", ints[:n * n].reshape(n, n).copy()
    if ring.value == 1:
        return n, "complex", cplx[:2 * n * n].view(np.complex128).reshape(n, n).copy()
    return n, "rational", None
