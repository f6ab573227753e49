"""Quick per-layer timing of df_attn_fwd at the Wan-1.3B shape (dev tool)."""
import math, sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K

dev = torch.device('cuda:0')
HW, D = 4680, 128
def run(ctxs, reps=20, probe=False):
    H = len(ctxs)
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(H * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(H * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    pb = None
    if probe:
        pb = K.ProbeBuffers(torch.zeros(H, 16, dtype=torch.uint8, device=dev), torch.ones(HW, dtype=torch.uint8, device=dev), torch.zeros(H, HW, 3, device=dev))
    for _ in range(3): K.attention(q, out, work, HW, 1/math.sqrt(D), pb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); K.attention(q, out, work, HW, 1/math.sqrt(D), pb); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort(); t = ts[len(ts)//2]
    flops = 4 * D * HW * sum(ctxs)
    return t * 1e3, flops / (t * 1e-3) / 1e12
res = {}
res['baseline_12x32760'] = run([32760] * 12)
res['packed_6d3s3n'] = run([28080] * 3 + [9360] * 9)
res['packed_3d4s5n'] = run([28080] * 5 + [9360] * 7)
res['probe_baseline'] = run([32760] * 12, probe=True)
for k, (us, tf) in res.items():
    print(f"{k}: {us:.1f} us/layer  {tf:.1f} TFLOP/s  ({tf/1672.3*100:.1f}% of measured bf16 peak)")
