"""HeadParallelSession at world size 2 (SURVEY.md 8(e) strategy 2).

Two processes share this one GPU (the round's boxes have a single B200) and a
gloo process group; gloo stages the head-output / score all-gathers and the
post-classification ring moves through the host, so no kernel of one rank
ever waits on the other's.  Each rank projects, attends and caches only its
heads; the assignment, the LPT owner table and ring moves, and the output
digest of the closed-loop session must equal the single-process Session
(reference permission: SPEC.md:152,227; engine.py:111-137).  An odd layer
count covers the per-gather turn of the fused gather's buffers as well.
"""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

import paper_2601_20499_b200 as df
from oracle import df_oracle as O

pytestmark = pytest.mark.gpu

OCFG = dict(num_layers=3, num_heads=4, head_dim=64, HW=192, window_len=4, ar_steps=7, denoise_steps=2,
            dummy_count=5, probe_ar_step=2, subsample_ratio=0.25)


def _model():
    toy = O.ToyModel(OCFG["num_layers"], OCFG["num_heads"], OCFG["head_dim"], OCFG["HW"], O.derive(9, "toy-model"))
    return df.ProjectedModel(toy.weights, toy.frame_input, OCFG["num_heads"], OCFG["head_dim"], OCFG["HW"])


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    from paper_2601_20499_b200.parallel import HeadParallelSession

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = HeadParallelSession(_model(), df.SessionConfig(**OCFG), "packed")
        frames, rep = s.run()
        torch.cuda.synchronize()
        out_q.put((rank, [c.value for c in s.assignment.classes], rep.output_digest, s.owners.tolist(),
                   s.rebalance_stats, s.layer_heads, [[c.frame_ids for c in layer] for layer in s.caches],
                   rep.kernel_calls_steady, [st["key_token_macs"] for st in rep.steps], None))
    except BaseException as e:  # reported to the parent
        out_q.put((rank, None, None, None, None, None, None, None, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_head_parallel_session_world2_equals_single_process():
    from paper_2601_20499_b200.parallel import contiguous_owners, lpt_owners

    cfg = df.SessionConfig(**OCFG)
    ref = df.Session(_model(), cfg, "packed")
    ref_frames, ref_rep = ref.run()
    torch.cuda.synchronize()
    ref_classes = [c.value for c in ref.assignment.classes]

    world = 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[-1] is None, r[-1]
    owners = res[0][3]
    for rank, classes, digest, own, stats, heads, frame_ids, calls, macs, _ in res:
        assert classes == ref_classes
        assert digest == ref_rep.output_digest
        assert own == owners
        # this rank's rings hold exactly the single-process rings of the heads it owns
        for layer in range(cfg.num_layers):
            assert heads[layer] == [h for h in range(cfg.num_heads) if owners[layer][h] == rank]
            assert frame_ids[layer] == [ref.caches[layer][h].frame_ids for h in heads[layer]]
    # every rank counts the key-token MACs of its own heads: together they are the session's
    assert [a + b for a, b in zip(res[0][8], res[1][8])] == [st["key_token_macs"] for st in ref_rep.steps]
    # the owner table is the LPT deal of the reference assignment's ring sizes, and rings moved
    pol = [[df.derive_policy(ref.assignment.classes[l * cfg.num_heads + h], cfg).ring_slots
            for h in range(cfg.num_heads)] for l in range(cfg.num_layers)]
    assert owners == lpt_owners(pol, world).tolist()
    moved = int((contiguous_owners(cfg.num_layers, cfg.num_heads, world) != lpt_owners(pol, world)).sum())
    assert moved > 0  # the test exercises real ring moves
    s0, s1 = res[0][4], res[1][4]
    assert s0["sent"] + s1["sent"] == s0["received"] + s1["received"] == moved
    assert s0["kept"] + s1["kept"] + moved == cfg.num_layers * cfg.num_heads
