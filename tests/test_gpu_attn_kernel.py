"""Raw df_attn_fwd numerics against a plain PyTorch fp32 reference."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(q, k, v, scale):
    s = (q.float() @ k.float().T) * scale
    return torch.softmax(s, dim=-1) @ v.float()


@pytest.mark.parametrize("width,hw,ctxs", [
    (128, 256, [256]),
    (128, 300, [300, 600, 1000]),
    (64, 192, [192, 384, 1344, 576]),
    (128, 4680, [9360, 4680 * 7]),
    (128, 600, [131072]),            # one long head: planner splits kv, in-kernel combine
    (64, 300, [40000, 300, 900]),    # split + unsplit heads in one launch, ragged tails
    (128, 200, [2000] * 40),         # many heads; last pair has a single valid tile
])
@pytest.mark.parametrize("pair", [False, True])
def test_attention_matches_torch(width, hw, ctxs, pair):
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(0)
    dev = torch.device("cuda:0")
    H = len(ctxs)
    total = sum(K.KVArena.region_rows(c) for c in ctxs)
    arena = K.KVArena(total, width, dev)
    q = torch.randn(H * hw, width, device=dev).to(torch.bfloat16)
    out = torch.zeros(H * hw, width, device=dev, dtype=torch.bfloat16)
    work = []
    for h, c in enumerate(ctxs):
        base = arena.allocate(c)
        arena.k[base:base + c] = torch.randn(c, width, device=dev).to(torch.bfloat16)
        arena.v[base:base + c] = torch.randn(c, width, device=dev).to(torch.bfloat16)
        work.append(K.HeadWork(arena, base, c, h, h))
    scale = 1.0 / math.sqrt(width)
    K.attention(q, out, work, hw, scale, pair=pair)
    torch.cuda.synchronize()
    for h, w in enumerate(work):
        ref = _ref(q[h * hw:(h + 1) * hw], arena.k[w.base_row:w.base_row + w.n_tok],
                   arena.v[w.base_row:w.base_row + w.n_tok], scale)
        got = out[h * hw:(h + 1) * hw].float()
        err = (got - ref).abs().max().item() / ref.abs().max().item()
        assert err <= 2e-2, (h, err)


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("scale_q", [1.0, 6.0])
def test_stale_rows_and_masked_tails(scale_q, pair):
    """Arena rows past each head's context hold stale finite data (as after an
    eviction): masked tail columns must contribute nothing, with both the MUFU
    and the polynomial exp2 paths; large logits exercise the lazy rescale."""
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(1)
    dev = torch.device("cuda:0")
    hw, width, ctxs = 300, 128, [300, 600, 1000, 4680 * 2 + 77]
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev)
    arena.k.normal_()
    arena.v.normal_()
    q = (torch.randn(len(ctxs) * hw, width, device=dev) * scale_q).to(torch.bfloat16)
    out = torch.full((len(ctxs) * hw, width), float("nan"), device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    scale = 1.0 / math.sqrt(width)
    K.attention(q, out, work, hw, scale, pair=pair)
    torch.cuda.synchronize()
    assert not torch.isnan(out.float()).any()
    for h, w in enumerate(work):
        ref = _ref(q[h * hw:(h + 1) * hw], arena.k[w.base_row:w.base_row + w.n_tok],
                   arena.v[w.base_row:w.base_row + w.n_tok], scale)
        err = (out[h * hw:(h + 1) * hw].float() - ref).abs().max().item() / ref.abs().max().item()
        assert err <= 2e-2, (h, err)


@pytest.mark.parametrize("pair", [False, True])
def test_running_max_jumps_inside_later_tiles(pair):
    """Logit spikes placed in a later kv tile's first half, its second half, and tiles after a jump:
    the CTA pair's single-pass softmax must fall back (first half: two-pass redo; second half: O and
    the row sum rescaled after the first-half PV) and the next warpgroups must pick up the moved m."""
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(7)
    dev = torch.device("cuda:0")
    hw, width = 256, 128
    ctx = 128 * 16
    spikes = [  # per head: (key index, logit in nats along the shared direction)
        [(128 * 4 + 10, 30.0), (128 * 7 + 100, 60.0), (128 * 9 + 3, 90.0)],
        [(128 * 5 + 70, 25.0), (128 * 6 + 127, 50.0), (128 * 13 + 64, 75.0)],
        [(128 * 3 + 64, 40.0), (128 * 3 + 65, 41.0), (128 * 11 + 1, 80.0)],
    ]
    H = len(spikes)
    arena = K.KVArena(H * K.KVArena.region_rows(ctx), width, dev)
    u = torch.randn(width, device=dev)
    u = u / u.norm()
    # q rows: the shared direction plus per-row noise (rows differ in where their own max lands)
    qf = u[None, :] * 4.0 + 0.3 * torch.randn(H * hw, width, device=dev)
    q = qf.to(torch.bfloat16)
    scale = 1.0 / math.sqrt(width)
    work = []
    for h, sp in enumerate(spikes):
        base = arena.allocate(ctx)
        k = torch.randn(ctx, width, device=dev)
        for key, logit in sp:
            k[key] += u * (logit / (4.0 * scale))
        arena.k[base:base + ctx] = k.to(torch.bfloat16)
        arena.v[base:base + ctx] = torch.randn(ctx, width, device=dev).to(torch.bfloat16)
        work.append(K.HeadWork(arena, base, ctx, h, h))
    out = torch.zeros(H * hw, width, device=dev, dtype=torch.bfloat16)
    K.attention(q, out, work, hw, scale, pair=pair)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    for h, w in enumerate(work):
        kk = arena.k[w.base_row:w.base_row + ctx].double()
        vv = arena.v[w.base_row:w.base_row + ctx].double()
        ref = torch.softmax((q[h * hw:(h + 1) * hw].double() @ kk.T) * scale, dim=-1) @ vv
        got = out[h * hw:(h + 1) * hw].double()
        err = (got - ref).abs().max().item() / ref.abs().max().item()
        assert err <= 2e-2, (h, err)


def test_probe_region_masses_with_split_kv():
    """DF_ATTN_PROBE on a launch the planner splits (2 heads, 94 kv tiles, 4 items on 148 SMs):
    the combine merges O, l and the three region masses of every piece (profiler.py:118-129)."""
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(3)
    dev = torch.device("cuda:0")
    hw, width, slots = 300, 128, 40
    ctxs = [hw * slots, hw * 17]
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev)
    arena.k.normal_()
    arena.v.normal_()
    H = len(ctxs)
    q = (torch.randn(H * hw, width, device=dev) * 2.0).to(torch.bfloat16)
    out = torch.empty(H * hw, width, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    codes = torch.randint(0, 3, (H, slots), dtype=torch.uint8)
    sampled = torch.zeros(hw, dtype=torch.uint8)
    sampled[::3] = 1
    probe = K.ProbeBuffers(codes.to(dev), sampled.to(dev), torch.zeros(H, hw, 3, device=dev))
    scale = 1.0 / math.sqrt(width)
    K.attention(q, out, work, hw, scale, probe=probe)
    torch.cuda.synchronize()
    for h, w in enumerate(work):
        s = (q[h * hw:(h + 1) * hw].float() @ arena.k[w.base_row:w.base_row + w.n_tok].float().T) * scale
        pmat = torch.softmax(s, dim=-1)
        region = codes[h].to(dev).long().repeat_interleave(hw)[: w.n_tok]
        want = torch.stack([pmat[:, region == r].sum(-1) for r in range(3)], dim=-1)
        rows = sampled.bool().to(dev)
        err = (probe.probe_rows[h][rows] - want[rows]).abs().max().item()
        assert err <= 2e-3, (h, err)
        assert bool((probe.probe_rows[h][~rows] == 0).all())
        ref = pmat @ arena.v[w.base_row:w.base_row + w.n_tok].float()
        oerr = (out[h * hw:(h + 1) * hw].float() - ref).abs().max().item() / ref.abs().max().item()
        assert oerr <= 2e-2, (h, oerr)


def test_hires_c4_full_size_sampled_rows():
    """C4 at full size (HW 18720, d 128): a packed-dummy head (2 frames), a sink head (2 frames) and
    a neighbor head (6 frames = 112,320 keys, split-KV with the in-kernel combine) in one launch,
    checked against fp32 torch on 256 sampled query rows per head (the full score matrix is 8 GB),
    plus run-to-run bitwise determinism of the whole output."""
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(7)
    dev = torch.device("cuda:0")
    hw, width = 18720, 128
    ctxs = [2 * hw, 2 * hw, 6 * hw]
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev)
    arena.k.normal_()
    arena.v.normal_()
    q = torch.randn(len(ctxs) * hw, width, device=dev).to(torch.bfloat16)
    out = torch.full((len(ctxs) * hw, width), float("nan"), device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    scale = 1.0 / math.sqrt(width)
    K.attention(q, out, work, hw, scale)
    again = torch.full_like(out, float("nan"))
    K.attention(q, again, work, hw, scale)
    torch.cuda.synchronize()
    for o in (out, again):
        bad = torch.isnan(o.float()).any(dim=1).nonzero().flatten()
        assert bad.numel() == 0, (bad.numel(), bad[:8].tolist(), (bad // hw).unique().tolist())
    assert torch.equal(out, again)
    rows = torch.randperm(hw, device=dev)[:256]
    for h, w in enumerate(work):
        qh = q[h * hw:(h + 1) * hw][rows]
        ref = _ref(qh, arena.k[w.base_row:w.base_row + w.n_tok], arena.v[w.base_row:w.base_row + w.n_tok], scale)
        got = out[h * hw:(h + 1) * hw][rows].float()
        err = (got - ref).abs().max().item() / ref.abs().max().item()
        assert err <= 2e-2, (h, err)


def test_split_workspace_reuse_across_plans():
    """Regression: one split workspace serves launches with different split plans.  A launch with few
    split groups writes partials where a later launch with more groups used to keep its combine
    counters; with the counters in a fixed region at the end of the workspace every row of the later
    launch is still combined and written."""
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(3)
    dev = torch.device("cuda:0")

    def launch(hw, width, ctxs):
        arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev)
        arena.k.normal_()
        arena.v.normal_()
        q = torch.randn(len(ctxs) * hw, width, device=dev).to(torch.bfloat16)
        out = torch.full((len(ctxs) * hw, width), float("nan"), device=dev, dtype=torch.bfloat16)
        work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
        K.attention(q, out, work, hw, 1 / math.sqrt(width))
        torch.cuda.synchronize()
        return int(torch.isnan(out.float()).any(dim=1).sum().item())

    assert launch(2048, 64, [16 * 2048] * 8) == 0          # 64 split groups, partials right after
    assert launch(18720, 128, [2 * 18720, 2 * 18720, 6 * 18720]) == 0  # more groups, same workspace
    assert launch(2048, 64, [16 * 2048] * 8) == 0


def test_randomized_ragged_launches_shared_workspace():
    """30 seeded random launches back to back on one stream (shared split workspace and plan cache):
    head counts 1-64 over 1-4 arenas, d 64/128, HW 1-5000, ragged contexts from one token to 20 frames,
    logit scales 0.5-6; every row written, rows sampled against fp32 torch."""
    import random

    from paper_2601_20499_b200 import kernels as K

    rng = random.Random(11)
    torch.manual_seed(11)
    dev = torch.device("cuda:0")
    for it in range(30):
        width = rng.choice([64, 128])
        hw = rng.choice([1, 7, 128, 300, 1000, 2048, 4680, rng.randint(1, 5000)])
        heads = rng.randint(1, 64 if hw <= 1000 else 12)
        n_arenas = rng.randint(1, min(4, heads))
        ctxs = [rng.randint(1, 20) * hw + rng.choice([0, 0, -rng.randint(0, max(0, hw - 1))]) for _ in range(heads)]
        ctxs = [max(1, c) for c in ctxs]
        arenas = [K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev) for _ in range(n_arenas)]
        for a in arenas:
            a.k.normal_()
            a.v.normal_()
        scale_q = rng.choice([0.5, 1.0, 3.0, 6.0])
        q = (torch.randn(heads * hw, width, device=dev) * scale_q).to(torch.bfloat16)
        out = torch.full((heads * hw, width), float("nan"), device=dev, dtype=torch.bfloat16)
        work = []
        for h, c in enumerate(ctxs):
            a = arenas[h % n_arenas]
            work.append(K.HeadWork(a, a.allocate(c), c, h, h))
        scale = 1.0 / math.sqrt(width)
        K.attention(q, out, work, hw, scale)
        torch.cuda.synchronize()
        assert not torch.isnan(out.float()).any(), (it, width, hw, heads, ctxs[:4])
        rows = torch.randint(0, hw, (min(hw, 64),), device=dev)
        for h in rng.sample(range(heads), min(heads, 4)):
            w = work[h]
            ref = _ref(q[h * hw:(h + 1) * hw][rows], w.arena.k[w.base_row:w.base_row + w.n_tok],
                       w.arena.v[w.base_row:w.base_row + w.n_tok], scale)
            got = out[h * hw:(h + 1) * hw][rows].float()
            err = (got - ref).abs().max().item() / ref.abs().max().item()
            assert err <= 2e-2, (it, h, err, width, hw, ctxs[h])
        del arenas, q, out


@pytest.mark.parametrize("pair", [False, True])
def test_attention_writes_only_its_rows(pair):
    """Bounds check of df_attn_fwd (compute-sanitizer is not available on the GPU pool): the
    output is a strided view with guard rows around it and gaps between the heads it names (o_head
    permuted, every other slot skipped); Q and both K/V planes must come back bit-identical, every
    guard byte untouched, the split-KV combine counters back at zero, and the written rows right."""
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(5)
    dev = torch.device("cuda:0")
    width, hw, G = 128, 700, 37
    ctxs = [60000, 130, 4000, 1, 9360]  # long head: split-KV partials + in-kernel combine
    H = len(ctxs)
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs) + 256, width, dev)
    arena.k.normal_()
    arena.v.normal_()
    q = (torch.randn(H * hw, width, device=dev) * 2).to(torch.bfloat16)
    o_heads = [8, 0, 4, 2, 6]  # out has 2H-1 head slots; odd slots are gaps
    q_heads = [3, 1, 4, 0, 2]
    big = torch.full((G + (2 * H - 1) * hw + G, width + 40), 7.0, device=dev, dtype=torch.bfloat16)
    out = big[G:G + (2 * H - 1) * hw, :width]
    work = [K.HeadWork(arena, arena.allocate(c), c, q_heads[h], o_heads[h]) for h, c in enumerate(ctxs)]
    k0, v0, q0 = arena.k.clone(), arena.v.clone(), q.clone()
    stream = torch.cuda.current_stream()
    launches = K.prepare_attention(q, out, work, hw, 1 / math.sqrt(width), pair=pair, stream=stream)
    for launch in launches:
        launch.launch(stream)
    torch.cuda.synchronize()
    assert torch.equal(arena.k, k0) and torch.equal(arena.v, v0) and torch.equal(q, q0)
    written = torch.zeros(big.shape[0], dtype=torch.bool, device=dev)
    for o in o_heads:
        written[G + o * hw:G + (o + 1) * hw] = True
    assert bool((big[~written] == 7.0).all())
    assert bool((big[:, width:] == 7.0).all())
    ws = launches[0].keep[3]
    if ws is not None:  # the combine returns its counters to zero for the next launch
        cnt = (ws.numel() - 64 * 1024) & ~255
        assert int(ws[cnt:cnt + 64 * 1024].count_nonzero()) == 0
    rows = torch.randint(0, hw, (48,), device=dev)
    for h, w in enumerate(work):
        ref = _ref(q[w.q_head * hw:(w.q_head + 1) * hw][rows], arena.k[w.base_row:w.base_row + w.n_tok],
                   arena.v[w.base_row:w.base_row + w.n_tok], 1 / math.sqrt(width))
        got = out[w.o_head * hw:(w.o_head + 1) * hw][rows].float()
        assert float((got - ref).abs().max() / ref.abs().max()) <= 2e-2, h


def test_attention_over_launch_limits_splits_and_c_abi_rejects():
    """More heads than DF_MAX_HEADS and more arenas than DF_MAX_ARENAS: prepare_attention splits the
    list into contiguous launches (results as one launch); the C ABI itself rejects an over-long
    descriptor table with DF_E_SHAPE instead of reading past its arrays."""
    import ctypes

    from paper_2601_20499_b200 import _lib, errors
    from paper_2601_20499_b200 import kernels as K

    torch.manual_seed(11)
    dev = torch.device("cuda:0")
    width, hw, H, n_arenas = 64, 130, 70, 6
    ctxs = [int(c) for c in torch.randint(1, 700, (H,))]
    arenas = [K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev) for _ in range(n_arenas)]
    for a in arenas:
        a.k.normal_()
        a.v.normal_()
    q = torch.randn(H * hw, width, device=dev).to(torch.bfloat16)
    out = torch.full((H * hw, width), float("nan"), device=dev, dtype=torch.bfloat16)
    work = []
    for h, c in enumerate(ctxs):
        a = arenas[(h // 3) % n_arenas]  # runs of 3 heads per arena: a launch may not exceed 4 arenas
        work.append(K.HeadWork(a, a.allocate(c), c, h, h))
    launches = K.prepare_attention(q, out, work, hw, 1 / math.sqrt(width))
    assert len(launches) >= 3  # 70 heads > 64, and 4-arena runs of 12 heads
    for launch in launches:
        launch.launch()
    torch.cuda.synchronize()
    assert not torch.isnan(out.float()).any()
    for h in (0, 13, 40, 64, 69):
        w = work[h]
        ref = _ref(q[h * hw:(h + 1) * hw], w.arena.k[w.base_row:w.base_row + w.n_tok],
                   w.arena.v[w.base_row:w.base_row + w.n_tok], 1 / math.sqrt(width))
        assert float((out[h * hw:(h + 1) * hw].float() - ref).abs().max() / ref.abs().max()) <= 2e-2, h
    # the C ABI: num_heads beyond DF_MAX_HEADS is a shape error, not an out-of-bounds read
    args = launches[0].keep[0]
    saved = args.num_heads
    args.num_heads = _lib.DF_MAX_HEADS + 1
    try:
        with pytest.raises(errors.ShapeError):
            _lib.call("df_attn_fwd", ctypes.byref(args), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    finally:
        args.num_heads = saved
