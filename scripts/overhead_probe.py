"""Dev: per-launch fixed cost of the FMHA (64 CTAs x n kv tiles, one 256-row pair per head)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device("cuda:0"); D = 128
for n in (16, 64, 128, 256):
    ctxs = [n * 128] * 64
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(64 * 256, D, device=dev).to(torch.bfloat16)
    out = torch.empty(64 * 256, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    launches = K.prepare_attention(q, out, work, 256, 1 / math.sqrt(D))
    for _ in range(3):
        for l in launches: l.launch()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(10):
        e[0].record()
        for l in launches: l.launch()
        e[1].record(); torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]) * 1e3)
    print(f"n={n}: min {min(ts):.1f} us, median {sorted(ts)[5]:.1f} us")
