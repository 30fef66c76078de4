"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host
logic: window sharding, lock-step counts, the flat-bucket gradient average
and the max/sum-over-ranks timing reductions used by bench.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _flat(grads):
    return np.concatenate([np.concatenate([w.ravel(), b.ravel()]) for w, b in grads]).astype(np.float32)


def _batch_grads(rank):
    g, x, labels = oracle.two_cluster_task(200, 16, 0)
    params = oracle.init_params((16, 8, 2), 0)
    seeds = np.arange(rank * 40, rank * 40 + 40, dtype=np.uint64)
    b = oracle.sample_khop(g, seeds, [3, 2], oracle.derive_seed(0, 13, rank))
    _, grads = oracle.train_step(b, x, labels, [[w.copy(), bb.copy()] for w, bb in params], 0.0)
    return _flat(grads)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2409_14939_b200 import dist as fdist
    r, w = fdist.init("gloo")
    assert (r, w) == (rank, world)
    windows = list(range(13))
    mine = fdist.shard(windows, rank, world)
    steps = fdist.lockstep_count(len(mine), world)
    flat = torch.from_numpy(_batch_grads(rank))
    fdist.GradAllReduce(world).allreduce_mean(flat)
    mx = fdist.max_over_ranks(float(rank + 1), world)
    sm = fdist.sum_over_ranks(float(rank + 1), world)
    q.put((rank, mine, steps, flat.numpy(), mx, sm))
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, m0, s0, f0, x0, y0), (_, m1, s1, f1, x1, y1) = res
    assert m0 == list(range(0, 13, 2)) and m1 == list(range(1, 13, 2))
    assert s0 == s1 == 6  # min over ranks of 7 and 6 windows
    want = (_batch_grads(0) + _batch_grads(1)) * np.float32(0.5)
    np.testing.assert_allclose(f0, want, rtol=1e-6, atol=1e-7)
    assert np.array_equal(f0, f1)  # every rank applies the identical averaged bucket
    assert x0 == x1 == 2.0 and y0 == y1 == 3.0
