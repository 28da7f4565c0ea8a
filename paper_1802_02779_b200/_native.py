"""ctypes binding of the C ABI in ``include/permlab_b200.h``.

The shared object is built in-tree (``make``, or ``__graft_entry__.build()``)
and loaded from this package directory. There is no fallback: importing the
package without the built library raises immediately, and every compute entry
point fails with ``PL_ERR_NODEVICE`` when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("PL_NATIVE_LIB", PKG_DIR / "libpermlab_b200.so"))  # override: tuning variants
GEN_PATH = PKG_DIR / "libpermlab_gen.so"

PL_OK, PL_ERR_ARG, PL_ERR_LIMIT, PL_ERR_OVERFLOW, PL_ERR_NOMEM, PL_ERR_CUDA, PL_ERR_NODEVICE, PL_ERR_NCCL = range(8)
PL_SHARD_ALLGATHER, PL_SHARD_BLOCKS = 0, 1
PL_I64, PL_F64, PL_C128 = 0, 1, 2
PL_FLAG_DEVICE_PTRS = 0x1
PL_FLAG_FMA = 0x2
PL_FLAG_ASYNC = 0x4
PL_FLAG_INPUT_READY = 0x8
PL_STATUS_BIT_OVERFLOW = 0x1
PL_STATUS_BIT_ROWS = 0x2
PL_MAX_ORDER = 34

STATUS_NAMES = {
    PL_OK: "PL_OK",
    PL_ERR_ARG: "PL_ERR_ARG",
    PL_ERR_LIMIT: "PL_ERR_LIMIT",
    PL_ERR_OVERFLOW: "PL_ERR_OVERFLOW",
    PL_ERR_NOMEM: "PL_ERR_NOMEM",
    PL_ERR_CUDA: "PL_ERR_CUDA",
    PL_ERR_NODEVICE: "PL_ERR_NODEVICE",
    PL_ERR_NCCL: "PL_ERR_NCCL",
}

# Every symbol include/permlab_b200.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "pl_version",
    "pl_last_error",
    "pl_limits_default",
    "pl_device_count",
    "pl_sz_permanent",
    "pl_sz_permanent_batch",
    "pl_sz_counts",
    "pl_sz_diagnostics",
    "pl_binom",
    "pl_colex_rank",
    "pl_colex_unrank",
    "pl_sz_layer",
    "pl_sz_top",
    "pl_sz_guard_i64",
    "pl_sz_scratch_bytes",
    "pl_release_scratch",
    "pl_sz_permanent_multi",
    "pl_shard_plan",
    "pl_shard_range",
    "pl_shard_exchange",
    "pl_boson_pattern_count",
    "pl_boson_unrank_pattern",
    "pl_boson_probabilities",
    "pl_boson_distribution",
    "pl_ryser_permanent",
    "pl_ryser_counts",
    "pl_shard_block_partial",
    "pl_shard_block_top_terms",
    "pl_sz_permanent_bigint",
    "pl_sz_permanent_modp",
    "pl_bigint_primes",
    "pl_ryser_permanent_bigint",
    "pl_ryser_permanent_modp",
)


class pl_limits(C.Structure):
    _fields_ = [("subset_order_limit", C.c_int32), ("memo_budget_bytes", C.c_uint64), ("num_gpus", C.c_int32)]


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 engine has no CPU fallback. Build it with "
            "`make` at the repo root (or __graft_entry__.build())."
        )
    L = C.CDLL(str(LIB_PATH))
    vp, i32, i64, u32, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64
    L.pl_version.restype = C.c_char_p
    L.pl_last_error.restype = C.c_char_p
    L.pl_limits_default.argtypes = [C.POINTER(pl_limits)]
    L.pl_limits_default.restype = None
    L.pl_device_count.restype = i32
    L.pl_sz_permanent.argtypes = [C.c_int, i32, vp, vp, u32, C.POINTER(pl_limits), vp]
    L.pl_sz_permanent.restype = C.c_int
    L.pl_sz_permanent_batch.argtypes = [C.c_int, i32, i64, vp, vp, u32, C.POINTER(pl_limits), vp, vp]
    L.pl_sz_permanent_batch.restype = C.c_int
    L.pl_sz_counts.argtypes = [i32, C.POINTER(u64), C.POINTER(u64)]
    L.pl_sz_counts.restype = C.c_int
    L.pl_sz_diagnostics.argtypes = [i32, C.POINTER(u64), C.POINTER(u64)]
    L.pl_sz_diagnostics.restype = C.c_int
    L.pl_binom.argtypes = [i32, i32]
    L.pl_binom.restype = u64
    L.pl_colex_rank.argtypes = [u64]
    L.pl_colex_rank.restype = u64
    L.pl_colex_unrank.argtypes = [i32, u64]
    L.pl_colex_unrank.restype = u64
    L.pl_sz_layer.argtypes = [C.c_int, i32, vp, i32, vp, vp, u64, u64, u32, vp, vp, vp]
    L.pl_sz_layer.restype = C.c_int
    L.pl_sz_top.argtypes = [C.c_int, i32, vp, vp, vp, u32, vp, vp, vp]
    L.pl_sz_top.restype = C.c_int
    L.pl_sz_guard_i64.argtypes = [i32, vp, vp, vp]
    L.pl_sz_guard_i64.restype = C.c_int
    L.pl_sz_scratch_bytes.argtypes = [C.c_int, i32]
    L.pl_sz_scratch_bytes.restype = u64
    L.pl_release_scratch.argtypes = []
    L.pl_release_scratch.restype = None
    L.pl_sz_permanent_multi.argtypes = [C.c_int, i32, i64, vp, vp, u32, C.POINTER(pl_limits), i32, vp]
    L.pl_sz_permanent_multi.restype = C.c_int
    L.pl_shard_plan.argtypes = [i32, i32]
    L.pl_shard_plan.restype = i32
    L.pl_shard_range.argtypes = [i32, i32, i32, i32, C.POINTER(u64), C.POINTER(u64)]
    L.pl_shard_range.restype = C.c_int
    L.pl_shard_exchange.argtypes = [i32, i32, i32, i32, C.POINTER(u64), i32]
    L.pl_shard_exchange.restype = i32
    L.pl_boson_pattern_count.argtypes = [i32, i32]
    L.pl_boson_pattern_count.restype = u64
    L.pl_boson_unrank_pattern.argtypes = [i32, i32, u64, vp]
    L.pl_boson_unrank_pattern.restype = C.c_int
    L.pl_boson_probabilities.argtypes = [i32, vp, i32, vp, i64, vp, vp, u32, C.POINTER(pl_limits), vp, vp]
    L.pl_boson_probabilities.restype = C.c_int
    L.pl_boson_distribution.argtypes = [i32, vp, i32, vp, u64, i64, vp, u32, vp]
    L.pl_boson_distribution.restype = C.c_int
    L.pl_ryser_permanent.argtypes = [C.c_int, i32, vp, vp, u32, C.POINTER(pl_limits), vp]
    L.pl_ryser_permanent.restype = C.c_int
    L.pl_ryser_counts.argtypes = [i32, C.POINTER(u64), C.POINTER(u64)]
    L.pl_ryser_counts.restype = C.c_int
    L.pl_shard_block_partial.argtypes = [C.c_int, i32, vp, i32, vp, vp, i32, i32, u32, vp, vp, vp]
    L.pl_shard_block_partial.restype = C.c_int
    L.pl_shard_block_top_terms.argtypes = [C.c_int, i32, vp, i32, vp, vp, i32, i32, u32, vp, vp]
    L.pl_shard_block_top_terms.restype = C.c_int
    L.pl_sz_permanent_bigint.argtypes = [i32, vp, vp, C.c_size_t, C.POINTER(C.c_size_t), C.POINTER(i32),
                                         C.POINTER(pl_limits), vp]
    L.pl_sz_permanent_bigint.restype = C.c_int
    L.pl_sz_permanent_modp.argtypes = [i32, i32, vp, vp, vp, C.POINTER(pl_limits), vp]
    L.pl_sz_permanent_modp.restype = C.c_int
    L.pl_ryser_permanent_bigint.argtypes = L.pl_sz_permanent_bigint.argtypes
    L.pl_ryser_permanent_bigint.restype = C.c_int
    L.pl_ryser_permanent_modp.argtypes = L.pl_sz_permanent_modp.argtypes
    L.pl_ryser_permanent_modp.restype = C.c_int
    L.pl_bigint_primes.argtypes = [i32, vp]
    L.pl_bigint_primes.restype = i32
    return L


lib = _load()


def last_error() -> str:
    return lib.pl_last_error().decode()


def gen():
    """Seeded config generators (``csrc/gen/configs.c``), loaded by configs.py."""
    from .configs import N as _G

    return _G.gen()
