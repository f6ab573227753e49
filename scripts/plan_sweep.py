"""Dev: packed Wan layer time under different planner overhead constants (env DF_PLAN_*)."""
import os
import subprocess
import sys

code = r'''
import math, sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2601_20499_b200 import kernels as K
dev = torch.device("cuda:0"); D = 128; HW = 4680
res = []
for name, ctxs in [("6d3s3n", [28080] * 3 + [9360] * 9), ("3d4s5n", [28080] * 5 + [9360] * 7), ("base", [32760] * 12)]:
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    for _ in range(3): K.attention(q, out, work, HW, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): K.attention(q, out, work, HW, 1 / math.sqrt(D))
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    res.append(f"{name} {us:.1f}us {4 * D * HW * sum(ctxs) / us / 1e6:.0f}TF")
print(" | ".join(res))
'''
grid = [(3, 1, 1.0), (2, 1, 1.0), (4, 1, 1.0), (3, 0.5, 1.0), (3, 2, 1.0), (3, 1, 0.5), (3, 1, 1.5), (1, 1, 1.0), (6, 1, 1.0)]
for piece, split, comb in grid:
    env = dict(os.environ, DF_PLAN_PIECE=str(piece), DF_PLAN_SPLIT=str(split), DF_PLAN_COMBINE=str(comb))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"piece {piece} split {split} combine {comb}: {r.stdout.strip() or r.stderr[-300:]}", flush=True)
