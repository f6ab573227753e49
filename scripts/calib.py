"""Calibrate per-tile and per-CTA costs of df_attn_kernel (dev tool)."""
import math, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device('cuda:0'); D = 128
def run(ctxs, HW, reps=10, split=True):
    H = len(ctxs)
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(H * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(H * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    for _ in range(2): K.attention(q, out, work, HW, 1/math.sqrt(D))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    import time
    h0 = time.perf_counter()
    for _ in range(reps): K.attention(q, out, work, HW, 1/math.sqrt(D))
    host_us = (time.perf_counter() - h0) / reps * 1e6
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps): K.attention(q, out, work, HW, 1/math.sqrt(D))
    e1.record(); torch.cuda.synchronize()
    global HOST_US; HOST_US = host_us
    return e0.elapsed_time(e1) / reps * 1e3
# 148 CTAs (148 heads x 1 qpair of 256 rows), n tiles each
for n in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    us = run([n * 128] * 64, 256, split=False)   # 64 heads -> 64 CTAs (< 148 SMs, one wave)
    print(f"64 CTAs x {n} tiles: {us:.1f} us  -> {us/n:.2f} us/tile (host {HOST_US:.0f} us/call)", flush=True)
for name, ctxs, hw in [('base', [32760]*12, 4680), ('6d3s3n', [28080]*3 + [9360]*9, 4680), ('3d4s5n', [28080]*5+[9360]*7, 4680)]:
    a = run(ctxs, hw, split=True); b = run(ctxs, hw, split=False)
    f = 4*D*hw*sum(ctxs)
    print(f"{name}: split {a:.1f} us ({f/a/1e6:.0f} TF/s)  nosplit {b:.1f} us ({f/b/1e6:.0f} TF/s)", flush=True)
