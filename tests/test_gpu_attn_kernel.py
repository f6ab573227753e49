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
def test_attention_matches_torch(width, hw, ctxs):
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
    K.attention(q, out, work, hw, scale)
    torch.cuda.synchronize()
    for h, w in enumerate(work):
        ref = _ref(q[h * hw:(h + 1) * hw], arena.k[w.base_row:w.base_row + w.n_tok],
                   arena.v[w.base_row:w.base_row + w.n_tok], scale)
        got = out[h * hw:(h + 1) * hw].float()
        err = (got - ref).abs().max().item() / ref.abs().max().item()
        assert err <= 2e-2, (h, err)
