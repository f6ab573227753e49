"""Small launches of every kernel for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize.py

Covers: df_attn_fwd (CTA pair and single CTA, split-KV with the in-kernel combine, ragged
heads, the DHP probe epilogue inside a Session), df_kv_append (+ overlapped), df_kv_pack,
df_proj (QKV into ring slots, out-projection + residual).
"""

import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_20499_b200 as df  # noqa: E402
from paper_2601_20499_b200 import kernels as K  # noqa: E402
from paper_2601_20499_b200.sweep import RandomStream  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)


def rnd(*s, scale=1.0):
    return (torch.randn(*s, device=dev, generator=g) * scale).to(torch.bfloat16)


# 1. a packed Session: probe epilogue, classification, pack, staging copies, packed attention
cfg = df.SessionConfig(num_layers=2, num_heads=6, head_dim=128, HW=1560, window_len=4, ar_steps=6, denoise_steps=1,
                       dummy_count=4, probe_ar_step=2, subsample_ratio=0.25)
_, rep = df.Session(RandomStream(cfg, 5), cfg, "packed").run()
print("session ok", rep.kernel_calls_steady)

# 2. ragged heads in one launch, both MMA shapes; long contexts force split-KV plans
arena = K.KVArena(4 * 9000, 128, dev)
arena.k.copy_(rnd(*arena.k.shape))
arena.v.copy_(rnd(*arena.v.shape))
hw = 700
lens = [8800, 130, 4000, 1]
work = [K.HeadWork(arena, h * 9000, n, h, h) for h, n in enumerate(lens)]
q = rnd(len(lens) * hw, 128, scale=2.0)
for pair in (True, False):
    out = torch.empty(len(lens) * hw, 128, dtype=torch.bfloat16, device=dev)
    for launch in K.prepare_attention(q, out, work, hw, 1 / math.sqrt(128), pair=pair):
        launch.launch()
    torch.cuda.synchronize()
    print("attention ok pair" if pair else "attention ok single", bool(torch.isfinite(out.float()).all()))

# 3. projections
x = rnd(1000, 512)
w = rnd(3 * 4 * 128, 512, scale=512**-0.5)
qp = torch.empty(4, 1000, 128, dtype=torch.bfloat16, device=dev)
kd = [arena.k[h * 9000 : h * 9000 + 1000] for h in range(4)]
vd = [arena.v[h * 9000 : h * 9000 + 1000] for h in range(4)]
K.prepare_qkv_projection(x, w, qp, kd, vd, 128).launch()
xr = torch.randn(1000, 256, device=dev, generator=g)
xb = torch.empty(1000, 256, dtype=torch.bfloat16, device=dev)
K.prepare_out_projection(qp, rnd(256, 4 * 128, scale=(4 * 128) ** -0.5), xr, xb, 128).launch()
torch.cuda.synchronize()
print("projections ok")
