"""Dev: one wave of equal work items (74 query tiles of 220 kv tiles; no tail, no split) -- the steady-state
per-tile rate of the CTA-pair FMHA, free of scheduling effects."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K  # noqa: E402
dev = torch.device("cuda:0"); D = 128
for name, (ctxs, hw) in {"onewave_2x37x220": ([28160] * 2, 256 * 37), "onewave_1x74x64": ([8192], 256 * 74)}.items():
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    ls = K.prepare_attention(q, out, work, hw, 1 / math.sqrt(D), pair=True)
    for _ in range(5):
        for l in ls: l.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        for l in ls: l.launch()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    tiles = sum((c + 127) // 128 for c in ctxs) * (hw // 256)
    print(f"{name}: {us:.1f} us, {us / (tiles / 74):.4f} us per tile per cluster, {4 * D * hw * sum(ctxs) / us / 1e6:.0f} TFLOP/s", flush=True)
