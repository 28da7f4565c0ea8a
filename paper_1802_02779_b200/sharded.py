"""Multi-GPU Store-zechin for large orders: per-layer subset-range sharding.

One process per GPU (torchrun); ``torch.distributed`` over NCCL is the
plumbing. Two plans, both computing every output once with the device layer
kernel (``pl_sz_layer`` on a colex-rank range) and ending with the n-term
development (``pl_sz_top``) on every rank:

* **top-column blocks** (world = 2^t, the default when it applies): rank g
  owns the k-subsets whose intersection with the top t columns is the pattern
  P_g = {n - t + i : bit i of g}. In colex order those subsets are ONE
  contiguous range of C(n - t, k - |P_g|) ranks (the top elements are the most
  significant), and every predecessor of such a subset lies in block P_g or in
  a block P_g minus one top column. So after each layer a rank only sends its
  block to the t - |P_g| ranks g | 2^i and receives the |P_g| blocks of ranks
  g & ~2^i — point-to-point, about (t / 2) / 2^t of a layer per rank instead of
  the (2^t - 1) / 2^t an all-gather moves.
* **equal slices + all-gather** (any world): every layer is split into
  ``world`` equal padded slices of ``L_k = ceil(C(n,k) / world)`` ranks, rank g
  computes ``[g L_k, min((g+1) L_k, C(n,k)))`` and an in-place all-gather
  replicates the layer, because an arbitrary rank range of layer k reads
  predecessors from all of layer k-1.

Batches are not handled here: they shard trivially by matrix with no
collective (``bench.py`` gives each rank its contiguous slice).

The orchestration is written against two hooks so that the identical
schedule runs on CPU ranks in the tests (gloo, with the CPU oracle's layer
step as the stand-in compute) and on GPUs (NCCL, with the CUDA kernels).
"""
from __future__ import annotations

import ctypes as C
import os
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


def top_columns(world: int) -> int:
    """t with world = 2^t, or -1 when world is not a power of two."""
    return world.bit_length() - 1 if world >= 1 and world & (world - 1) == 0 else -1


def block_plan_applies(n: int, world: int) -> bool:
    t = top_columns(world)
    return t >= 1 and n - t >= 3


def top_block(n: int, k: int, world: int, g: int) -> Tuple[int, int]:
    """Colex-rank range of layer k owned by rank g under the top-column plan:
    the k-subsets S with S n {n-t..n-1} = P_g. Empty (0, 0) when no such subset."""
    t = top_columns(world)
    cols = [n - t + i for i in range(t) if (g >> i) & 1]  # ascending
    m = k - len(cols)
    if m < 0 or m > n - t:
        return 0, 0
    base = sum(comb(p, m + l + 1) for l, p in enumerate(cols))
    return base, base + comb(n - t, m)


def exchange_blocks(buf: torch.Tensor, n: int, k: int, rank: int, world: int, group=None, wait: bool = True):
    """After layer k: hand rank `rank`'s block of layer k to the ranks that add
    one top column to its pattern, and receive the blocks with one column less.
    wait=False returns the pending requests (the overlapped plan waits for them
    after the next layer's partial compute)."""
    t = top_columns(world)
    ops = []
    for i in range(t):
        partner = rank ^ (1 << i)
        if rank >> i & 1:  # receive block P \ {n-t+i}
            r0, r1 = top_block(n, k, world, partner)
            if r1 > r0:
                ops.append(("recv", partner, r0, r1))
        else:  # send own block to P u {n-t+i}
            r0, r1 = top_block(n, k, world, rank)
            if r1 > r0:
                ops.append(("send", partner, r0, r1))
    if not ops:
        return []
    if buf.is_cuda:
        p2p = [dist.P2POp(dist.isend if kind == "send" else dist.irecv, _as_gather_view(buf[r0:r1]), peer,
                          group=group) for kind, peer, r0, r1 in ops]
        reqs = dist.batch_isend_irecv(p2p)
    else:
        reqs = []
        for kind, peer, r0, r1 in ops:
            view = _as_gather_view(buf[r0:r1])
            reqs.append(dist.isend(view, peer, group=group) if kind == "send" else dist.irecv(view, peer, group=group))
    if wait:
        for req in reqs:
            req.wait()
        return []
    return reqs


def gather_last_layer(buf: torch.Tensor, n: int, rank: int, world: int, group=None):
    """Replicate layer n-1 (n entries) from its owners onto every rank, bit for bit."""
    k = n - 1
    mine = torch.zeros(n, dtype=buf.dtype, device=buf.device)
    r0, r1 = top_block(n, k, world, rank)
    mine[r0:r1] = buf[r0:r1]
    parts = [torch.zeros_like(mine) for _ in range(world)]
    if buf.is_cuda:
        flat = torch.zeros(world * n, dtype=buf.dtype, device=buf.device)
        dist.all_gather_into_tensor(_as_gather_view(flat), _as_gather_view(mine), group=group)
        parts = list(flat.chunk(world))
    else:
        rp = [_as_gather_view(p) for p in parts]
        dist.all_gather(rp, _as_gather_view(mine), group=group)
    for h in range(world):
        h0, h1 = top_block(n, k, world, h)
        buf[h0:h1] = parts[h][h0:h1]


def sharded_layer_dp(a: torch.Tensor, rank: int, world: int,
                     layer_fn: Callable[[int, torch.Tensor, torch.Tensor, int, int], None],
                     top_fn: Callable[[torch.Tensor, torch.Tensor], object],
                     group=None, on_layer: Callable[[int], None] | None = None, plan: str = "auto",
                     status: torch.Tensor | None = None, partial_fn=None, top_terms_fn=None):
    """Run the layer DP of matrix `a` (n x n, already on this rank's device)
    sharded over `world` ranks. `layer_fn(k, prev, cur, r0, r1)` fills
    cur[r0:r1] of layer k; `top_fn(a, last)` returns the permanent.
    plan: "blocks" (top-column blocks, world = 2^t), "allgather", or "auto".
    `status` (int32, on the device the collectives use) is the rank's overflow
    status word written by its layer kernels: before the top level it is
    combined over the group (MAX), so either every rank sees an int64
    overflow and raises, or none does (a wrapped value exchanged by one rank
    never reaches a result silently).

    Overlap (block plan, when `partial_fn(k, prev, cur)` and
    `top_terms_fn(k, prev, cur)` are given): the exchange of layer k-1 runs
    while the rank computes layer k without its top-column terms from its own
    block; the top-column terms follow once the blocks have landed. The top
    columns are the highest, so their terms come last in the reference's
    ascending order and the result is bit-for-bit the non-overlapped one."""
    n = a.shape[0]
    if n < 3:
        raise ValueError("sharded DP needs n >= 3")
    if plan == "auto":
        plan = "blocks" if world > 1 and block_plan_applies(n, world) else "allgather"
    if plan == "blocks":
        if not block_plan_applies(n, world):
            raise ValueError("top-column blocks need world = 2^t with n - t >= 3")
        size = max(comb(n, k) for k in range(2, n)) + 4
        bufs = [torch.zeros(size, dtype=a.dtype, device=a.device) for _ in range(2)]
        prev, cur = bufs
        if world > 1 and a.is_cuda:
            # NCCL: batched P2P among a subset of ranks is only defined once the
            # group has run a collective
            dist.barrier(group=group)
        overlap = partial_fn is not None and top_terms_fn is not None and world > 1
        pending = []
        for k in range(2, n):
            r0, r1 = top_block(n, k, world, rank)
            if not overlap or k == 2:
                if r1 > r0:
                    layer_fn(k, prev, cur, r0, r1)
            else:
                # layer k-1's exchange (started below in the previous iteration) is in flight
                if r1 > r0:
                    partial_fn(k, prev, cur)
                for req in pending:
                    req.wait()
                pending = []
                if r1 > r0:
                    top_terms_fn(k, prev, cur)
            if k < n - 1:
                pending = exchange_blocks(cur, n, k, rank, world, group, wait=not overlap)
            if on_layer is not None:
                on_layer(k)
            prev, cur = cur, prev
        gather_last_layer(prev, n, rank, world, group)
        _combine_status(status, world, group)
        return top_fn(a, prev)
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
    _combine_status(status, world, group)
    return top_fn(a, prev)


def _combine_status(status: torch.Tensor | None, world: int, group) -> None:
    if status is not None and world > 1:
        dist.all_reduce(status, op=dist.ReduceOp.MAX, group=group)


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

    layer_fn.guard = guard
    layer_fn.status = status  # the rank's overflow word (combined over ranks by sharded_layer_dp)
    return layer_fn, top_fn


def device_overlap_hooks(a: torch.Tensor, layer_fn, rank: int, world: int, fma: bool = False, stream=None):
    """partial_fn / top_terms_fn of the overlapped block plan (pl_shard_block_partial / _top_terms)."""
    from . import _native as N
    from .api import _check, _torch_dtype_code

    code = _torch_dtype_code(a)
    n = a.shape[0]
    flags = N.PL_FLAG_FMA if fma else 0
    st = (stream or torch.cuda.current_stream(a.device)).cuda_stream
    status = layer_fn.status
    guard = layer_fn.guard

    def partial_fn(k, prev, cur):
        _check(N.lib.pl_shard_block_partial(code, n, a.data_ptr(), k, prev.data_ptr(), cur.data_ptr(), world, rank,
                                            flags, guard.data_ptr(), status.data_ptr(), st))

    def top_terms_fn(k, prev, cur):
        _check(N.lib.pl_shard_block_top_terms(code, n, a.data_ptr(), k, prev.data_ptr(), cur.data_ptr(), world, rank,
                                              flags, status.data_ptr(), st))

    return partial_fn, top_terms_fn


def sharded_permanent(a: torch.Tensor, group=None, fma: bool = False):
    """Permanent of one large matrix on this process's GPU, cooperating with
    every rank of the (NCCL) process group."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    layer_fn, top_fn = device_hooks(a, fma=fma)
    partial_fn = top_terms_fn = None
    if world > 1 and block_plan_applies(a.shape[0], world) and os.environ.get("PL_SHARD_OVERLAP", "1") != "0":
        partial_fn, top_terms_fn = device_overlap_hooks(a, layer_fn, rank, world, fma=fma)
    return sharded_layer_dp(a, rank, world, layer_fn, top_fn, group=group, status=layer_fn.status,
                            partial_fn=partial_fn, top_terms_fn=top_terms_fn)
