"""Multi-GPU Store-zechin for large orders: per-layer subset-range sharding.

One process per GPU (torchrun); ``torch.distributed`` over NCCL is the
plumbing. Every layer k of the DP (subset size k, colex order) is split into
``world`` equal padded slices of ``L_k = ceil(C(n,k) / world)`` ranks; rank g
computes ``[g L_k, min((g+1) L_k, C(n,k)))`` with the device layer kernel
(``pl_sz_layer``) and an in-place all-gather replicates the layer on every
GPU, because the next layer reads predecessors from the whole previous layer
(the last slice of layer k needs all of layer k-1). The final n-term
development runs on every rank from its replicated layer n-1 (``pl_sz_top``).

Batches are not handled here: they shard trivially by matrix with no
collective (``bench.py`` gives each rank its contiguous slice).

The orchestration is written against two hooks so that the identical
schedule runs on CPU ranks in the tests (gloo, with the CPU oracle's layer
step as the stand-in compute) and on GPUs (NCCL, with the CUDA kernels).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from math import comb
from typing import Callable, List, Tuple

import torch
import torch.distributed as dist

_ELEM_BYTES = {torch.int64: 8, torch.float64: 8, torch.complex128: 16}


def layer_slices(n: int, k: int, world: int) -> Tuple[int, List[Tuple[int, int]]]:
    """(L, [(r0, r1) per rank]) for layer k of order n over `world` ranks."""
    total = comb(n, k)
    per = -(-total // world)
    return per, [(min(g * per, total), min((g + 1) * per, total)) for g in range(world)]


def max_padded_layer(n: int, world: int) -> int:
    return max(layer_slices(n, k, world)[0] * world for k in range(2, n))


def _as_gather_view(t: torch.Tensor) -> torch.Tensor:
    # NCCL has no complex type; gather the float64 view.
    if t.is_complex():
        return torch.view_as_real(t).reshape(-1)
    return t


def allgather_inplace(buf: torch.Tensor, per: int, rank: int, world: int, group=None):
    """All-gather equal slices of `buf[:world*per]`, slice g owned by rank g."""
    full = _as_gather_view(buf[: world * per])
    mine = _as_gather_view(buf[rank * per:(rank + 1) * per])
    if full.is_cuda:
        dist.all_gather_into_tensor(full, mine, group=group)  # in place: NCCL allows send == recv + rank*count
    else:
        parts = list(full.chunk(world))
        dist.all_gather(parts, mine.clone(), group=group)


@dataclass
class ShardPlan:
    n: int
    world: int
    rank: int

    def slice(self, k: int) -> Tuple[int, int, int]:
        per, sl = layer_slices(self.n, k, self.world)
        r0, r1 = sl[self.rank]
        return per, r0, r1


def sharded_layer_dp(a: torch.Tensor, rank: int, world: int,
                     layer_fn: Callable[[int, torch.Tensor, torch.Tensor, int, int], None],
                     top_fn: Callable[[torch.Tensor, torch.Tensor], object],
                     group=None, on_layer: Callable[[int], None] | None = None):
    """Run the layer DP of matrix `a` (n x n, already on this rank's device)
    sharded over `world` ranks. `layer_fn(k, prev, cur, r0, r1)` fills
    cur[r0:r1] of layer k; `top_fn(a, last)` returns the permanent."""
    n = a.shape[0]
    if n < 3:
        raise ValueError("sharded DP needs n >= 3")
    size = max_padded_layer(n, world) + 4  # slack: 16-byte aligned ring copies may read one entry past a layer
    bufs = [torch.zeros(size, dtype=a.dtype, device=a.device) for _ in range(2)]
    plan = ShardPlan(n, world, rank)
    prev, cur = bufs
    for k in range(2, n):
        per, r0, r1 = plan.slice(k)
        layer_fn(k, prev, cur, r0, r1)
        if world > 1:
            allgather_inplace(cur, per, rank, world, group)
        if on_layer is not None:
            on_layer(k)
        prev, cur = cur, prev
    return top_fn(a, prev)


# ---------------------------------------------------------------- device hooks

def device_hooks(a: torch.Tensor, fma: bool = False, stream=None):
    """layer_fn / top_fn running the CUDA kernels through the C ABI."""
    from . import _native as N
    from .api import DomainError, _check, _torch_dtype_code

    code = _torch_dtype_code(a)
    n = a.shape[0]
    flags = N.PL_FLAG_FMA if fma else 0
    st = (stream or torch.cuda.current_stream(a.device)).cuda_stream
    status = torch.zeros(1, dtype=torch.int32, device=a.device)
    guard = torch.zeros(1, dtype=torch.int32, device=a.device)
    if code == N.PL_I64:
        _check(N.lib.pl_sz_guard_i64(n, a.data_ptr(), guard.data_ptr(), st))

    def layer_fn(k, prev, cur, r0, r1):
        _check(N.lib.pl_sz_layer(code, n, a.data_ptr(), k, prev.data_ptr(), cur.data_ptr(), r0, r1, flags,
                                 guard.data_ptr(), status.data_ptr(), st))

    def top_fn(a_, last):
        out = torch.zeros(1, dtype=a.dtype, device=a.device)
        _check(N.lib.pl_sz_top(code, n, a_.data_ptr(), last.data_ptr(), out.data_ptr(), flags, guard.data_ptr(),
                               status.data_ptr(), st))
        if int(status.item()) & N.PL_STATUS_BIT_OVERFLOW:
            raise DomainError("int64 overflow: an intermediate sub-permanent does not fit the exact int64 ring")
        return out.item()

    return layer_fn, top_fn


def sharded_permanent(a: torch.Tensor, group=None, fma: bool = False):
    """Permanent of one large matrix on this process's GPU, cooperating with
    every rank of the (NCCL) process group."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    layer_fn, top_fn = device_hooks(a, fma=fma)
    return sharded_layer_dp(a, rank, world, layer_fn, top_fn, group=group)
