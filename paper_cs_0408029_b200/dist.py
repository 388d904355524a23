"""Multi-GPU plumbing for the NNLS hot path (one process per GPU,
torch.distributed over NCCL on NVLink; gloo for CPU tests).

Two ways the path uses several GPUs (BASELINE.json north_star):

* Row-sharded Gram: rank r forms G_r = A_r^T A_r, c_r = A_r^T b_r over its
  row block (nnls_setup_shard), the [G | c] buffers are summed with ONE
  all-reduce (the only GPU<->GPU exchange of the method), nnls_gram_finalize,
  then the pivot loop runs on the full Gram.  With quantized inputs every
  partial sum is exact, so the reduced Gram is bitwise independent of the
  number of ranks.
* Independent problems (batched config 4, or one problem per rank): disjoint
  slices, no communication.
"""
from __future__ import annotations


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
    """(start, count) of rank's slice of `total` independent problems."""
    r0, r1 = row_shards(total, world)[rank]
    return r0, r1 - r0


class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


def gram_tensor(shard_solver):
    """torch tensor aliasing the solver's device [G | c] buffer."""
    import torch
    ptr, count, _ = shard_solver.gram_buffer()
    return torch.as_tensor(_CudaArray(ptr, count), device="cuda")


def allreduce_gram(shard_solver, group=None):
    """Sum the row-shard partial Grams of all ranks in place (one
    all_reduce(SUM, float64)), then finalize the handle."""
    import torch
    import torch.distributed as dist
    t = gram_tensor(shard_solver)
    torch.cuda.synchronize()  # the partial Gram kernels ran on the handle's stream
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    torch.cuda.synchronize()
    shard_solver.finalize()
    return t
