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


def _costs(L=4, H=8, seed=3):
    """Post-classification ring sizes of a planted-style assignment: packed dummy
    2 slots, sink 2, neighbour W=6 (kv_cache.py policies)."""
    rng = np.random.default_rng(seed)
    return rng.choice([2, 2, 6], size=(L, H))


def _rebalance_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L, H, HW, d = 4, 8, 3, 4
        costs = _costs(L, H)
        old = P.contiguous_owners(L, H, world)
        new = P.lpt_owners(costs, world)
        keep, send, recv = P.rebalance_plan(old, new, rank)
        # every (layer, head) ring holds costs[l, h] frames of distinct data
        frame = lambda l, h, f: torch.full((HW, d), float(1000 * l + 10 * h + f))
        sends = [(dst, frame(l, h, f).clone()) for l, h, dst in send for f in range(int(costs[l, h]))]
        bufs = [(src, torch.zeros(HW, d)) for l, h, src in recv for f in range(int(costs[l, h]))]
        P.exchange_frames(sends, bufs, None)
        expect = [frame(l, h, f) for l, h, _ in recv for f in range(int(costs[l, h]))]
        ok_move = all(torch.equal(b, e) for (_, b), e in zip(bufs, expect))
        # uneven per-layer output gather in global head order
        full = torch.randn(H, HW, d, generator=torch.Generator().manual_seed(5))
        ok_gather = True
        for layer in range(L):
            mine = [h for h in range(H) if new[layer, h] == rank]
            got = P.gather_head_outputs_owned(full[mine].clone(), new[layer])
            ok_gather &= torch.equal(got, full)
        out_q.put((rank, new.tolist(), keep, send, recv, ok_move, ok_gather))
    finally:
        dist.destroy_process_group()


def test_lpt_rebalance_world2():
    """Post-classification rebalancing over 2 gloo ranks: both ranks derive the
    same LPT owner table, every head is kept, or sent by its old owner and
    received by its new one, the moved frames arrive intact, and the uneven
    per-layer output gather restores global head order."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rebalance_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] == res[1][1]
    for rank, _, keep, send, recv, ok_move, ok_gather in res:
        assert ok_move and ok_gather
    L, H = 4, 8
    seen = sorted([(l, h) for r in res for l, h in r[2]] + [(l, h) for r in res for l, h, _ in r[3]])
    assert seen == [(l, h) for l in range(L) for h in range(H)]
    sent = sorted((l, h, res_rank, dst) for res_rank, _, _, send, _, _, _ in res for l, h, dst in send)
    got = sorted((l, h, src, res_rank) for res_rank, _, _, _, recv, _, _ in res for l, h, src in recv)
    assert sent == got


def test_lpt_owners_balance():
    costs = _costs(30, 12, seed=7)
    for world in (1, 2, 4):
        owners = P.lpt_owners(costs, world)
        for layer in range(costs.shape[0]):
            loads = [int(costs[layer][owners[layer] == r].sum()) for r in range(world)]
            # LPT bound: the heaviest rank exceeds the lightest by at most the largest job
            assert max(loads) - min(loads) <= costs[layer].max()
            contiguous = [int(costs[layer][r * (12 // world):(r + 1) * (12 // world)].sum()) for r in range(world)]
            assert max(loads) <= max(contiguous)
    assert np.array_equal(P.lpt_owners(costs, 2), P.lpt_owners(costs.copy(), 2))  # deterministic
    assert (P.lpt_owners(costs, 1) == 0).all()
    with pytest.raises(df.ConfigError):
        P.lpt_owners(costs[0], 2)


def test_bench_gpus_n_starts_n_ranks():
    """``bench.py --gpus 2`` without a launcher re-executes itself under torchrun, one rank per GPU
    (the --rank-check hook reports each rank's RANK / WORLD_SIZE and exits before touching a GPU)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--rank-check"],
                         capture_output=True, text=True, timeout=300, check=True).stdout
    lines = sorted((json.loads(l) for l in out.splitlines() if l.startswith("{")), key=lambda d: d["rank"])
    assert lines == [{"rank": 0, "world": 2}, {"rank": 1, "world": 2}]
    # a launcher whose world size disagrees with --gpus is refused
    bad = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--rank-check"],
                         capture_output=True, text=True, timeout=120, env=dict(os.environ, WORLD_SIZE="2"))
    assert bad.returncode != 0 and "WORLD_SIZE=2" in bad.stderr


def test_fused_gather_buffers_alternate_per_gather_with_odd_layer_count():
    """The fused all-gather's two symmetric buffers alternate once per gather, not by layer index:
    with an odd layer count, layer L-1 of one denoise iteration and layer 0 of the next write
    different buffers, so a fast rank never stores into the buffer a slow rank still reads."""
    calls = []

    class _H:
        def __init__(self, i):
            self.i = i

        def barrier(self, channel=0):
            calls.append(self.i)

    fg = object.__new__(P.FusedHeadGather)
    fg.bufs = [torch.zeros(2, 2), torch.zeros(2, 2)]
    fg.handles = [_H(0), _H(1)]
    fg.peers = [[11], [22]]
    fg.turn = 0
    L, iters = 3, 3
    used = []
    for _ in range(iters):
        for layer in range(L):
            tgt = fg.target(layer, [0])
            assert tgt.out is fg.current()
            used.append(fg.bufs.index(tgt.out) if tgt.out is fg.bufs[0] else 1)
            assert tgt.peers == fg.peers[used[-1]]
            fg.barrier()
    assert used == [i % 2 for i in range(L * iters)]
    assert calls == used
    assert all(a != b for a, b in zip(used, used[1:]))
