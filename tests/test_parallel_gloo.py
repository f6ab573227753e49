"""N>1 host paths on CPU: world_size-2 gloo process groups (no GPU needed).

Covers the collectives of parallel.py (head-output and score all-gathers, the
max-over-ranks timing reduction), the partitions, and that every rank reaches
the identical greedy assignment (C solver) from gathered scores -- equal to
the single-process assignment of the full table.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2601_20499_b200 as df
from paper_2601_20499_b200 import parallel as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, H, HW, d = 3, 8, 5, 4
        g = torch.Generator().manual_seed(0)
        full_out = torch.randn(H, HW, d, generator=g)
        heads = P.head_partition(H, world, rank)
        got = P.gather_head_outputs(full_out[heads.start:heads.stop].clone())
        ok_out = torch.equal(got, full_out)

        rng = np.random.default_rng(1)
        F = rng.random((L, H, 3))
        F /= F.sum(axis=2, keepdims=True)
        local = torch.from_numpy(F[:, heads.start:heads.stop].copy())
        table = P.gather_head_scores(local).reshape(-1, 3).numpy()
        ok_scores = np.array_equal(table, F.reshape(-1, 3))
        assignment, obj = df.greedy_classify(table, 7)

        t = P.max_over_ranks(float(rank + 1))
        streams = P.stream_partition(7, world, rank)
        out_q.put((rank, ok_out, ok_scores, [c.value for c in assignment.classes], obj, t, streams))
    finally:
        dist.destroy_process_group()


def test_head_parallel_collectives_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(1)
    F = rng.random((3, 8, 3))
    F /= F.sum(axis=2, keepdims=True)
    ref, ref_obj = df.greedy_classify(F.reshape(-1, 3), 7)
    for rank, ok_out, ok_scores, classes, obj, t, streams in res:
        assert ok_out and ok_scores
        assert classes == [c.value for c in ref.classes]  # identical on every rank
        assert obj == ref_obj
        assert t == 2.0  # max over ranks
    assert sorted(res[0][6] + res[1][6]) == list(range(7))  # streams: disjoint cover, no collective


def test_partitions_validate():
    assert P.head_partition(12, 4, 3) == range(9, 12)
    assert P.stream_partition(10, 4, 1) == [1, 5, 9]
    with pytest.raises(df.ConfigError):
        P.head_partition(12, 5, 0)
    with pytest.raises(df.ConfigError):
        P.stream_partition(3, 2, 2)
