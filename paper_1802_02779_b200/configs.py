"""Seeded synthetic inputs for BASELINE.json's five configs.

Thin numpy wrappers around ``csrc/gen/configs.c`` (recipes in its header,
following the reference's RNG conventions: ``std::mt19937_64``, 53-bit
uniforms, Box-Muller, Gram-Schmidt Haar unitaries; reference
``proj/src/boson.cpp:29-45, 149-181, 207-227``).
"""
from __future__ import annotations

import ctypes as C
import hashlib
from pathlib import Path

import numpy as np

# Self-contained on purpose (no package-relative imports): bench.py's reference
# arm loads this file by path, so generating the workload never maps the
# engine's libpermlab_b200.so into the reference arm's process.
GEN_PATH = Path(__file__).resolve().parent / "libpermlab_gen.so"


class _Gen:
    _lib = None

    def gen(self):
        """Seeded config generators (``csrc/gen/configs.c``)."""
        if self._lib is None:
            if not GEN_PATH.exists():
                raise ImportError(f"{GEN_PATH} is missing: run `make` at the repo root")
            G = C.CDLL(str(GEN_PATH))
            vp, i32, i64, u64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
            for name, args, res in (("pl_gen_haar", [i32, u64, i32, vp], C.c_int),
                                    ("pl_gen_c1", [i64, u64, vp], None), ("pl_gen_c2", [i64, u64, vp], C.c_int),
                                    ("pl_gen_c3", [i64, u64, vp], None), ("pl_gen_c4", [i32, u64, vp], None),
                                    ("pl_gen_c5", [i32, i32, u64, vp], C.c_int),
                                    ("pl_gen_int_matrices", [i32, i64, u64, i64, i64, vp], None),
                                    ("pl_gen_uniform", [i64, u64, C.c_double, C.c_double, vp], None),
                                    ("pl_gen_mt64_stream", [u64, i64, vp], None)):
                f = getattr(G, name)
                f.argtypes = args
                f.restype = res
            self._lib = G
        return self._lib


N = _Gen()

CONFIGS = {
    "c1": dict(n=5, count=100_000, dtype="int64", seed=1,
               desc="100,000 x 5x5 int64, entries uniform {0..9}, seed 1"),
    "c2": dict(n=5, count=100_000, dtype="complex128", seed=2,
               desc="100,000 x 5x5 complex128 boson-sampling submatrices of Haar(25), seed 2"),
    "c3": dict(n=12, count=10_000, dtype="int64", seed=3,
               desc="10,000 x 12x12 int64 Bernoulli(0.5), seed 3"),
    "c4": dict(n=26, count=1, dtype="float64", seed=4, desc="1 x 26x26 float64 uniform [-1,1), seed 4"),
    "c5": dict(n=32, count=1, dtype="complex128", seed=5,
               desc="1 x 32x32 complex128 = U[0:32,0:32] of Haar(1024), seed 5"),
}


def _p(arr: np.ndarray):
    return arr.ctypes.data


def c1(count: int = 100_000, seed: int = 1) -> np.ndarray:
    out = np.empty((count, 5, 5), dtype=np.int64)
    N.gen().pl_gen_c1(count, seed, _p(out))
    return out


def c2(count: int = 100_000, seed: int = 2) -> np.ndarray:
    out = np.empty((count, 5, 5), dtype=np.complex128)
    if N.gen().pl_gen_c2(count, seed, _p(out)) != 0:
        raise RuntimeError("pl_gen_c2 failed")
    return out


def c3(count: int = 10_000, seed: int = 3) -> np.ndarray:
    out = np.empty((count, 12, 12), dtype=np.int64)
    N.gen().pl_gen_c3(count, seed, _p(out))
    return out


def c4(n: int = 26, seed: int = 4) -> np.ndarray:
    out = np.empty((n, n), dtype=np.float64)
    N.gen().pl_gen_c4(n, seed, _p(out))
    return out


def c5(n: int = 32, m: int = 1024, seed: int = 5) -> np.ndarray:
    out = np.empty((n, n), dtype=np.complex128)
    if N.gen().pl_gen_c5(m, n, seed, _p(out)) != 0:
        raise RuntimeError("pl_gen_c5 failed")
    return out


def haar(m: int, seed: int, ncols: int | None = None) -> np.ndarray:
    out = np.empty((m, m), dtype=np.complex128)
    if N.gen().pl_gen_haar(m, seed, m if ncols is None else ncols, _p(out)) != 0:
        raise RuntimeError("pl_gen_haar failed")
    return out


def int_matrices(n: int, count: int, seed: int, lo: int = -9, hi: int = 9) -> np.ndarray:
    out = np.empty((count, n, n), dtype=np.int64)
    N.gen().pl_gen_int_matrices(n, count, seed, lo, hi, _p(out))
    return out


def uniform(shape, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    out = np.empty(shape, dtype=np.float64)
    N.gen().pl_gen_uniform(out.size, seed, lo, hi, _p(out))
    return out


def complex_uniform(shape, seed: int) -> np.ndarray:
    flat = uniform(tuple(shape) + (2,), seed)
    return np.ascontiguousarray(flat[..., 0] + 1j * flat[..., 1])


def mt64_stream(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    N.gen().pl_gen_mt64_stream(seed, count, _p(out))
    return out


def generate(name: str) -> np.ndarray:
    name = name.lower()
    if name == "c1":
        return c1()
    if name == "c2":
        return c2()
    if name == "c3":
        return c3()
    if name == "c4":
        return c4()[None]
    if name == "c5":
        return c5()[None]
    raise KeyError(name)


def sha256(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()
