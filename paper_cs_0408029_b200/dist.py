"""Multi-GPU plumbing for the NNLS hot path (one process per GPU,
torch.distributed over NCCL on NVLink; gloo for CPU tests).  Argument
marshalling and collectives only -- no arithmetic of the method.

Two ways the path uses several GPUs (BASELINE.json north_star; SURVEY.md §8(e);
DESIGN.md §8):

* Row-sharded Gram (A^T A is formed once, and it is a sum over the
  rows of A): rank k forms the packed partial G_k = A_k^T A_k, c_k = A_k^T b_k
  of its row block -- the root from the full A it keeps for the loop
  (ShardSolver), every other rank from ONLY its block (BlockSolver) -- and the
  partials are summed with ONE collective: a reduce to the root (default:
  only the root runs the pivot loop) or an all-reduce (every rank holds the
  sum).  The buffer is the packed lower triangle + c, n(n+1)/2 + n doubles.
  With quantized inputs every partial sum is exact, so the reduced Gram is
  bitwise independent of the number of ranks.
* Independent problems (batched config 4): disjoint slices of the batch, no
  communication.
"""
from __future__ import annotations

import numpy as np


def row_shards(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row blocks [r0, r1) of m rows over `world` ranks (sizes
    differ by at most one)."""
    if world < 1 or m < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(m, world)
    out, r0 = [], 0
    for r in range(world):
        r1 = r0 + base + (1 if r < extra else 0)
        out.append((r0, r1))
        r0 = r1
    return out


def batch_shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of rank's slice of `total` independent problems; the
    remainder is spread one problem each over the first ranks (nothing is
    dropped)."""
    r0, r1 = row_shards(total, world)[rank]
    return r0, r1 - r0


def row_block(rowptr, colind, vals, b, r0: int, r1: int):
    """Local CSR (rowptr rebased to 0) and b of rows [r0, r1): what a non-root
    rank uploads (numpy arrays)."""
    rowptr = np.asarray(rowptr)
    e0, e1 = int(rowptr[r0]), int(rowptr[r1])
    return ((rowptr[r0:r1 + 1] - e0).astype(np.int32), np.ascontiguousarray(colind[e0:e1], dtype=np.int32),
            np.ascontiguousarray(vals[e0:e1], dtype=np.float64), np.ascontiguousarray(b[r0:r1], dtype=np.float64))


def packed_count(n: int) -> int:
    """Doubles in the reduction buffer: packed lower triangle + c."""
    return n * (n + 1) // 2 + n


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


def gram_tensor(solver, device=None):
    """torch tensor aliasing the handle's device [G packed | c] buffer."""
    import torch
    ptr, count = solver.gram_buffer()
    return torch.as_tensor(_CudaArray(ptr, count), device=device or "cuda")


def reduce_gram_buffer(buf, mode: str = "reduce", root: int = 0, group=None):
    """SUM the ranks' packed partial-Gram buffers in place: mode "reduce" ->
    the sum lands on `root` only, "allreduce" -> on every rank.  Device
    agnostic (NCCL for CUDA tensors, gloo for CPU tensors)."""
    import torch.distributed as dist
    if mode == "reduce":
        dist.reduce(buf, dst=root, op=dist.ReduceOp.SUM, group=group)
    elif mode == "allreduce":
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    else:
        raise ValueError(f"unknown reduction mode {mode!r}")
    return buf


def reduce_gram(solver, mode: str = "reduce", root: int = 0, group=None, stream=None):
    """The sharded-Gram exchange for a ShardSolver (root) or BlockSolver:
    reduce the packed partials, then (root) finalize the handle.  `stream`:
    the torch stream the handle was created on -- the collective is issued
    on it, so it orders after the partial-Gram kernels and the finalize after
    the collective without a host synchronisation."""
    import contextlib

    import torch
    import torch.distributed as dist
    t = gram_tensor(solver)
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:
        if stream is None:
            torch.cuda.synchronize()  # (handle on another stream: order by a host sync)
        reduce_gram_buffer(t, mode, root, group)
    rank = dist.get_rank(group)
    if hasattr(solver, "finalize") and (mode == "allreduce" or rank == root):
        if stream is None:
            torch.cuda.synchronize()
        solver.finalize()
    return t


# backwards-compatible name (round 1): all-reduce + finalize
def allreduce_gram(solver, group=None, stream=None):
    return reduce_gram(solver, "allreduce", 0, group, stream)
