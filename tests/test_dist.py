"""Multi-process host logic of the multi-GPU paths (-m "not gpu"; gloo,
world_size 2 on CPU): row sharding of the Gram and its reduction, batch
sharding.  The exchange runs through the PRODUCT's helpers
(paper_cs_0408029_b200.dist.row_block / reduce_gram_buffer, the same calls
the NCCL path makes on device tensors), on packed lower-triangle partial Grams
the oracle forms for each rank's row block; quantized inputs make the reduced
Gram bitwise equal to the single-process Gram."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nnls_gen as g
import oracle as O
from paper_cs_0408029_b200.dist import batch_shard, packed_count, reduce_gram_buffer, row_block, row_shards


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


def _pack_lower(G):
    """Packed lower triangle, row i = G[i, :i+1] at offset i(i+1)/2 (the layout
    include/nnls.h documents for nnls_gram_buffer), written out by index."""
    n = G.shape[0]
    out = np.empty(n * (n + 1) // 2)
    for i in range(n):
        out[i * (i + 1) // 2: i * (i + 1) // 2 + i + 1] = G[i, :i + 1]
    return out


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prob = g.make_problem(dict(m=600, n=120, density=0.05), seed=3)
    r0, r1 = row_shards(prob.m, world)[rank]
    rp, ci, v, b = row_block(prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1)
    blk = g.Problem(r1 - r0, prob.n, rp, ci, v, b, prob.x_gen, prob.kind, prob.seed)
    G, c = O.gram(blk)                                  # partial A_r^T A_r, A_r^T b_r
    buf = torch.from_numpy(np.concatenate([_pack_lower(G), c]))
    assert buf.numel() == packed_count(prob.n)
    reduce_gram_buffer(buf, mode=mode, root=0)          # the product's collective helper
    q.put((rank, buf.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["reduce", "allreduce"])
def test_gloo_sharded_gram_reduce_bitwise(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prob = g.make_problem(dict(m=600, n=120, density=0.05), seed=3)
    G, c = O.gram(prob)
    want = np.concatenate([_pack_lower(G), c])
    assert np.array_equal(got[0], want)                 # root holds the exact full Gram
    if mode == "allreduce":
        assert np.array_equal(got[1], want)


def test_row_block_rebases():
    prob = g.make_problem(dict(m=50, n=20, density=0.2), seed=1)
    for r0, r1 in [(0, 50), (0, 17), (17, 50), (20, 20)]:
        rp, ci, v, b = row_block(prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1)
        assert rp[0] == 0 and rp.size == r1 - r0 + 1 and rp[-1] == ci.size == v.size
        A = prob.dense()[r0:r1]
        B = np.zeros_like(A)
        rows = np.repeat(np.arange(r1 - r0), np.diff(rp))
        B[rows, ci] = v
        assert np.array_equal(A, B) and np.array_equal(b, prob.b[r0:r1])
