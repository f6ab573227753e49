"""Dev: packed Wan FMHA at logit std 1 and 3 (lazy-rescale sensitivity)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device('cuda:0')
D, HW = 128, 4680
ctxs = [2 * HW] * 9 + [6 * HW] * 3
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_(); arena.v.normal_()
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
for std in (1.0, 3.0, 6.0):
    q = (torch.randn(len(ctxs) * HW, D, device=dev) * std).to(torch.bfloat16)
    ls = K.prepare_attention(q, out, work, HW, 1 / math.sqrt(D))
    for _ in range(3):
        for l in ls: l.launch(None)
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for l in ls: l.launch(None)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"logit std {std}: {sorted(ts)[7] * 1e3:.1f} us", flush=True)
