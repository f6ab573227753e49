import math, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device("cuda:0"); D = 128
ctxs, hw = [28080] * 3 + [9360] * 9, 4680
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_(); arena.v.normal_()
q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
for _ in range(3):
    K.attention(q, out, work, hw, 1 / math.sqrt(D))
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
for _ in range(5):
    K.attention(q, out, work, hw, 1 / math.sqrt(D))
e[1].record(); torch.cuda.synchronize()
print("us per launch", e[0].elapsed_time(e[1]) / 5 * 1e3)
