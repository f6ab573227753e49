"""Fused projection GEMMs on the device.

* df_qkv_project vs an fp32 torch GEMM on the same bf16 operands; Q lands in
  the FMHA layout, K/V in strided ring-slot views, nothing outside them moves.
* df_out_project: x += merge(o) @ W_o in place, bf16 copy == bf16(fp32 result).
* ProjectedModel drives the reference's C1 toy session (closed loop: QKV ->
  attention -> out-projection + residual) and reproduces the reference's
  classes / MACs / calls / cache ratio (tests/golden/toy_c1_reports.json);
  its frames match the bit-exact oracle ToyModel normwise.
"""
import json
import os

import numpy as np
import pytest
import torch

import paper_2601_20499_b200 as df
from paper_2601_20499_b200 import kernels as K
from oracle import df_oracle as O

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")
GEMM_TOL = 1e-2  # normwise, bf16 outputs of fp32-accumulated GEMMs
FRAME_TOL = 2e-2  # north-star attention tolerance, applied to the layer output x


def _rel(got: torch.Tensor, want: torch.Tensor) -> float:
    got, want = got.float().cpu(), want.float().cpu()
    return float((got - want).abs().max() / want.abs().max().clamp_min(1e-30))


@pytest.fixture(params=[None, "128", "192", "256"], ids=["auto", "bn128", "bn192", "bn256"])
def tile_n(request, monkeypatch):
    if request.param is not None:
        monkeypatch.setenv("DF_PROJ_BN", request.param)
    return request.param


@pytest.mark.parametrize("hw,heads,d,in_dim", [(192, 4, 64, 256), (4680, 12, 128, 1536), (300, 3, 128, 200),
                                               (1, 1, 64, 64), (129, 5, 64, 320)])
def test_qkv_projection_matches_torch(hw, heads, d, in_dim, tile_n):
    g = torch.Generator(device="cuda").manual_seed(hw + heads + d)
    dev = torch.device("cuda")
    x = torch.randn(hw, in_dim, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(3 * heads * d, in_dim, device=dev, generator=g) / in_dim**0.5).to(torch.bfloat16)
    width = d + 64  # arena-like plane wider than the head: columns d.. must stay untouched
    slots = 3
    kplane = torch.full((heads * slots * hw + 7, width), 7.0, dtype=torch.bfloat16, device=dev)
    vplane = torch.full_like(kplane, -7.0)
    k_dst = [kplane[(h * slots + 1) * hw : (h * slots + 2) * hw, :d] for h in range(heads)]
    v_dst = [vplane[(h * slots + 1) * hw : (h * slots + 2) * hw, :d] for h in range(heads)]
    q = torch.empty(heads, hw, d, dtype=torch.bfloat16, device=dev)
    K.prepare_qkv_projection(x, w, q, k_dst, v_dst, d).launch()
    ref = (x.float() @ w.float().T).view(hw, 3, heads, d).permute(1, 2, 0, 3)  # (3, heads, hw, d)
    assert _rel(q, ref[0]) <= GEMM_TOL
    for h in range(heads):
        assert _rel(k_dst[h], ref[1, h]) <= GEMM_TOL
        assert _rel(v_dst[h], ref[2, h]) <= GEMM_TOL
    written = torch.zeros(kplane.shape[0], dtype=torch.bool, device=dev)
    for h in range(heads):
        written[(h * slots + 1) * hw : (h * slots + 2) * hw] = True
    assert bool((kplane[~written] == 7.0).all()) and bool((vplane[~written] == -7.0).all())
    assert bool((kplane[:, d:] == 7.0).all()) and bool((vplane[:, d:] == -7.0).all())


@pytest.mark.parametrize("hw,heads,d,out_dim", [(192, 4, 64, 256), (4680, 12, 128, 1536), (300, 3, 128, 96),
                                                (1, 2, 64, 128)])
def test_out_projection_residual(hw, heads, d, out_dim, tile_n):
    g = torch.Generator(device="cuda").manual_seed(hw * 7 + heads)
    dev = torch.device("cuda")
    o = torch.randn(heads, hw, d, device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn(out_dim, heads * d, device=dev, generator=g) / (heads * d) ** 0.5).to(torch.bfloat16)
    x = torch.randn(hw, out_dim, device=dev, generator=g)
    x0 = x.clone()
    xb = torch.empty(hw, out_dim, dtype=torch.bfloat16, device=dev)
    K.prepare_out_projection(o, w, x, xb, d).launch()
    merged = o.float().permute(1, 0, 2).reshape(hw, heads * d)  # scenario.py:118 head merge
    want = x0 + merged @ w.float().T
    assert _rel(x - x0, want - x0) <= 1e-4  # fp32 epilogue: only accumulation-order error
    assert torch.equal(xb, x.to(torch.bfloat16))


def test_projection_argument_errors():
    dev = torch.device("cuda")
    x = torch.zeros(64, 128, dtype=torch.bfloat16, device=dev)
    w = torch.zeros(3 * 2 * 64, 128, dtype=torch.bfloat16, device=dev)
    q = torch.empty(2, 64, 64, dtype=torch.bfloat16, device=dev)
    kv = [torch.empty(64, 64, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    with pytest.raises(df.ShapeError):
        K.prepare_qkv_projection(x, w[:-1], q, kv, kv, 64)
    with pytest.raises(df.ShapeError):
        K.prepare_qkv_projection(x.float(), w, q, kv, kv, 64)
    with pytest.raises(df.ShapeError):
        K.prepare_out_projection(q, torch.zeros(96, 100, dtype=torch.bfloat16, device=dev),
                                 torch.zeros(64, 96, device=dev), None, 64)
    with pytest.raises(df.ShapeError):  # out_dim not a multiple of 32 (C-ABI check)
        K.prepare_out_projection(q, torch.zeros(40, 128, dtype=torch.bfloat16, device=dev),
                                 torch.zeros(64, 40, device=dev), None, 64).launch()


def _toy_c1():
    ocfg = O.Config(num_layers=2, num_heads=4, head_dim=64, HW=192, window_len=6, ar_steps=10, denoise_steps=2,
                    dummy_count=2, probe_ar_step=2, subsample_ratio=0.25)
    toy = O.ToyModel(2, 4, 64, 192, O.derive(42, "toy-model"))
    return ocfg, toy


@pytest.mark.parametrize("mode", ["baseline", "hma", "packed"])
def test_projected_model_reproduces_reference_toy_session(mode):
    g = json.load(open(os.path.join(G, "toy_c1_reports.json")))[mode]
    ocfg, toy = _toy_c1()
    cfg = df.SessionConfig(**ocfg.__dict__)
    model = df.ProjectedModel(toy.weights, toy.frame_input, 4, 64, 192)
    frames, rep = df.generate_session(model, cfg, mode)
    assert [s["key_token_macs"] for s in rep.steps] == [s["key_token_macs"] for s in g["steps"]]
    assert rep.kernel_calls_steady == g["kernel_calls_steady"]
    assert rep.cache_reduction_ratio == g["cache_reduction_ratio"]
    assert rep.physical_launches_steady == [1, 1]  # K/V produced in the ring: no staging / append copy
    if g["assignment"]:
        assert [h["class"] for h in rep.to_dict()["assignment"]["heads"]] == [h["class"] for h in g["assignment"]["heads"]]
        assert rep.to_dict()["assignment"]["objective"] == pytest.approx(g["assignment"]["objective"], abs=2e-3)
    run = O.run_session(toy, ocfg, mode)
    assert len(frames) == len(run.frames)
    worst = max(_rel(f, torch.from_numpy(r)) for f, r in zip(frames, run.frames))
    assert worst <= FRAME_TOL, worst


def test_projected_model_fused_equals_unfused_protocol():
    """qkv_into/mix_into (in-place ring + residual) == plain qkv/mix (copies), bitwise."""
    ocfg, toy = _toy_c1()
    cfg = df.SessionConfig(**{**ocfg.__dict__, "ar_steps": 5})
    fused = df.ProjectedModel(toy.weights, toy.frame_input, 4, 64, 192)

    class Plain:
        def __init__(self, m):
            self.m = m

        def frame_input(self, i, t):
            return self.m.frame_input(i, t)

        def qkv(self, layer, x, i, t):
            return self.m.qkv(layer, x, i, t)

        def mix(self, layer, outputs):
            return self.m.mix(layer, outputs)

    a, ra = df.generate_session(fused, cfg, "packed")
    b, rb = df.generate_session(Plain(fused), cfg, "packed")
    assert all(torch.equal(x.to(torch.bfloat16), getattr(y, "f32", y).to(torch.bfloat16)) for x, y in zip(a, b))
    assert ra.to_dict()["assignment"] == rb.to_dict()["assignment"]
    assert rb.physical_launches_steady == [2, 2]


def test_projected_model_head_range_slices_weights():
    """Head-parallel ranks project only their heads (ProjectedModel._w_heads): bitwise equal to the
    corresponding heads of the full projection."""
    _, toy = _toy_c1()
    m = df.ProjectedModel(toy.weights, toy.frame_input, 4, 64, 192)
    x = m.frame_input(0, 0)
    q_full, k_full, v_full = m.qkv(1, x, 0, 0)
    heads = range(1, 3)
    q = torch.empty(2, 192, 64, dtype=torch.bfloat16, device="cuda")
    k = torch.empty_like(q)
    v = torch.empty_like(q)
    m.qkv_into(1, x, 0, 0, q, list(k), list(v), heads=heads)
    torch.cuda.synchronize()
    assert torch.equal(q, q_full[1:3]) and torch.equal(k, k_full[1:3]) and torch.equal(v, v_full[1:3])


def test_session_cuda_graphs_equal_eager():
    """Session(graphs=True): whole denoise iterations captured per cache
    signature and replayed -- frames, assignment and counters bitwise equal to the eager session,
    graphs reused across denoise iterations and AR steps with the same slot tables."""
    ocfg, toy = _toy_c1()
    cfg = df.SessionConfig(**{**ocfg.__dict__, "ar_steps": 14, "denoise_steps": 3})
    model = df.ProjectedModel(toy.weights, toy.frame_input, 4, 64, 192)
    a, ra = df.Session(model, cfg, "packed").run()
    s = df.Session(model, cfg, "packed", graphs=True)
    b, rb = s.run()
    assert all(torch.equal(x, y) for x, y in zip(a, b))
    assert ra.to_dict()["assignment"] == rb.to_dict()["assignment"]
    assert ra.kernel_calls_steady == rb.kernel_calls_steady
    assert [st["key_token_macs"] for st in ra.steps] == [st["key_token_macs"] for st in rb.steps]
    # the probe iteration runs eagerly; every other iteration replays a captured graph
    assert s.graph_stats["replayed"] + s.graph_stats["captured"] == cfg.ar_steps * cfg.denoise_steps - 1
    assert s.graph_stats["captured"] < cfg.ar_steps  # the warm ring cycles through its slots
    # frames are distinct tensors (the graph's residual buffers are reused)
    assert len({f.data_ptr() for f in b}) == len(b)


_PAIR_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2601_20499_b200 import kernels as K
torch.manual_seed(0)
dev = torch.device("cuda")
for (hw, H, d) in ((4680, 12, 128), (300, 4, 64), (1000, 3, 128)):
    D = H * d
    x = torch.randn(hw, D, device=dev).to(torch.bfloat16)
    w = (torch.randn(3 * D, D, device=dev) / D ** 0.5).to(torch.bfloat16)
    q = torch.empty(H, hw, d, dtype=torch.bfloat16, device=dev)
    k = torch.empty_like(q)
    v = torch.empty_like(q)
    K.prepare_qkv_projection(x, w, q, list(k), list(v), d).launch()
    o = torch.randn(H, hw, d, device=dev).to(torch.bfloat16)
    wo = (torch.randn(D, D, device=dev) / D ** 0.5).to(torch.bfloat16)
    xf = torch.randn(hw, D, device=dev)
    xb = torch.empty(hw, D, dtype=torch.bfloat16, device=dev)
    K.prepare_out_projection(o, wo, xf, xb, d).launch()
    torch.cuda.synchronize()
    ref_q = (x.float() @ w.float().T)[:, :D].reshape(hw, H, d).transpose(0, 1)
    err = ((q.float() - ref_q).abs().max() / ref_q.abs().max()).item()
    assert err < 1e-2, err
    torch.save({"q": q.cpu(), "k": k.cpu(), "v": v.cpu(), "xf": xf.cpu(), "xb": xb.cpu()}, f"{sys.argv[2]}_{hw}.pt")
"""


@pytest.mark.parametrize("bn", ["", "128", "256"])
def test_pair_and_single_cta_gemms_bitwise_equal(tmp_path, bn):
    """The CTA-pair projection GEMM (cta_group::2) and the 1-CTA GEMM produce bitwise identical Q/K/V and
    residual updates (same K order per output element), on the Wan shape and ragged ones, with the
    tiling picker free or forced to N = 128 / 256 (subprocesses: DF_PROJ_PAIR / DF_PROJ_BN are read once)."""
    import subprocess
    import sys as _sys

    script = tmp_path / "pair.py"
    script.write_text(_PAIR_SCRIPT)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for pair in ("0", "1"):
        env = dict(os.environ, DF_PROJ_PAIR=pair)
        if bn:
            env["DF_PROJ_BN"] = bn
        subprocess.run([_sys.executable, str(script), root, str(tmp_path / f"p{pair}")], check=True, env=env)
    for hw in (4680, 300, 1000):
        a = torch.load(tmp_path / f"p0_{hw}.pt")
        b = torch.load(tmp_path / f"p1_{hw}.pt")
        for key in a:
            assert torch.equal(a[key], b[key]), (hw, key)


def test_session_nvtx_ranges(monkeypatch):
    """DF_NVTX tracing: one range per AR step, per (denoise iteration, layer), around the
    classify + pack and the append copies (ring compaction), balanced push / pop."""
    from paper_2601_20499_b200 import engine

    pushed, depth = [], [0]

    def push(name):
        pushed.append(name)
        depth[0] += 1

    def pop():
        depth[0] -= 1

    monkeypatch.setattr(engine, "NVTX", True)
    monkeypatch.setattr(torch.cuda.nvtx, "range_push", push)
    monkeypatch.setattr(torch.cuda.nvtx, "range_pop", pop)
    ocfg, toy = _toy_c1()
    cfg = df.SessionConfig(**{**ocfg.__dict__, "ar_steps": 4})
    df.Session(df.ProjectedModel(toy.weights, toy.frame_input, 4, 64, 192), cfg, "packed").run()
    assert depth[0] == 0
    assert [n for n in pushed if "/" not in n] == [f"ar{i}" for i in range(4)]
    assert "ar0/denoise1/layer1" in pushed and "ar2/classify+pack" in pushed
    assert sum(n.endswith("/layer0") for n in pushed) == cfg.ar_steps * cfg.denoise_steps
