"""Dev: packed Wan FMHA under sustained load (30 layers round robin, 16 passes), median launch time."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K

dev = torch.device('cuda:0')
D, HW = 128, 4680
ctxs = [28080] * 3 + [9360] * 9
if len(sys.argv) > 1 and sys.argv[1] == "baseline":
    ctxs = [32760] * 12
flops = 4 * D * HW * sum(ctxs)
launches = []
for _ in range(30):
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    launches.append((K.prepare_attention(q, out, work, HW, 1 / math.sqrt(D)), q, out, arena))
for p in range(20):
    for l, *_ in launches:
        for x in l: x.launch(None)
torch.cuda.synchronize()
ev = []
for p in range(16):
    for l, *_ in launches:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for x in l: x.launch(None)
        b.record()
        ev.append((a, b))
torch.cuda.synchronize()
ts = sorted(a.elapsed_time(b) for a, b in ev)
us = ts[len(ts) // 2] * 1e3
print(f"sustained {sys.argv[1] if len(sys.argv) > 1 else 'packed'}: median {us:.1f} us  {flops / us / 1e6:.0f} TFLOP/s")
