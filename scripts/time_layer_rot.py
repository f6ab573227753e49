"""Dev: packed Wan FMHA launch timed on one resident layer vs rotating over 30 layers' K/V (cold L2 per launch)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K

dev = torch.device('cuda:0')
D, HW = 128, 4680
ctxs = [28080] * 3 + [9360] * 9
flops = 4 * D * HW * sum(ctxs)
layers = []
for _ in range(30):
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    layers.append((q, out, work))
launches = [K.prepare_attention(q, out, work, HW, 1 / math.sqrt(D)) for q, out, work in layers]
def run(idx, reps):
    for i in idx[:3]:
        for l in launches[i]: l.launch(None)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps * len(idx))]
    k = 0
    for _ in range(reps):
        for i in idx:
            ev[k].record()
            for l in launches[i]: l.launch(None)
            ev[k + 1].record()
            k += 2
    torch.cuda.synchronize()
    ts = sorted(ev[j].elapsed_time(ev[j + 1]) for j in range(0, k, 2))
    return ts[len(ts) // 2] * 1e3
for name, idx in (("same layer", [0]), ("30 layers round robin", list(range(30)))):
    us = run(idx, 30 if len(idx) == 1 else 2)
    print(f"{name}: median {us:.1f} us  {flops / us / 1e6:.0f} TFLOP/s")
us = run([0], 30)
print(f"same layer again: median {us:.1f} us")
for reps in (2, 8, 16):
    us = run(list(range(30)), reps)
    print(f"30 layers x {reps} reps: median {us:.1f} us  {flops / us / 1e6:.0f} TFLOP/s")
