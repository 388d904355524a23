"""Multi-process host logic of the multi-GPU paths (-m "not gpu"; gloo,
world_size 2 on CPU): row sharding of the Gram and its all-reduce, batch
sharding.  The exchange is the one the NCCL path does (one all_reduce SUM of
the float64 [G | c] buffer); quantized inputs make the reduced Gram bitwise
equal to the single-process Gram."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nnls_gen as g
import oracle as O
from paper_cs_0408029_b200.dist import batch_shard, row_shards


def test_row_shards_partition():
    for m in (1, 7, 2000, 40000):
        for w in (1, 2, 3, 8):
            sh = row_shards(m, w)
            assert sh[0][0] == 0 and sh[-1][1] == m and len(sh) == w
            assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
            sizes = [r1 - r0 for r0, r1 in sh]
            assert max(sizes) - min(sizes) <= 1


def test_batch_shard_covers():
    total = 65536
    for w in (1, 2, 4, 8):
        got = [batch_shard(total, w, r) for r in range(w)]
        assert sum(c for _, c in got) == total
        assert got[0][0] == 0 and all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(w - 1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _row_block(prob, r0, r1):
    rp = prob.rowptr
    e0, e1 = rp[r0], rp[r1]
    return g.Problem(r1 - r0, prob.n, (rp[r0:r1 + 1] - e0).astype(np.int32), prob.colind[e0:e1],
                     prob.vals[e0:e1], prob.b[r0:r1], prob.x_gen, prob.kind, prob.seed)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = g.make_problem(dict(m=600, n=120, density=0.05), seed=3)
    r0, r1 = row_shards(prob.m, world)[rank]
    G, c = O.gram(_row_block(prob, r0, r1))          # partial A_r^T A_r, A_r^T b_r
    buf = torch.from_numpy(np.concatenate([G.ravel(), c]))
    dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    if rank == 0:
        q.put(buf.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_gram_allreduce_bitwise():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prob = g.make_problem(dict(m=600, n=120, density=0.05), seed=3)
    G, c = O.gram(prob)
    n = prob.n
    assert np.array_equal(got[:n * n].reshape(n, n), G)
    assert np.array_equal(got[n * n:], c)
