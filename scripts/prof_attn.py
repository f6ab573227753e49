"""Small driver for ncu: a few launches of the packed Wan layer (dev tool)."""
import math, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device('cuda:0'); D = 128; HW = 4680
mode = sys.argv[1] if len(sys.argv) > 1 else 'packed'
if mode == 'hires':
    HW = 18720
ctxs = {'packed': [28080] * 3 + [9360] * 9, 'baseline': [32760] * 12, 'hires': [131040] * 4}[mode]
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_(); arena.v.normal_()
q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
for _ in range(4):
    K.attention(q, out, work, HW, 1 / math.sqrt(D))
torch.cuda.synchronize()
print("ok", out.float().abs().mean().item())
