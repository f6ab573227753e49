"""Dev: per-iteration timeline of CTA 0 (the leader) of the CTA-pair FMHA (DF_TRACE build, clock64 cycles)."""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import _lib, kernels as K  # noqa: E402

dev = torch.device("cuda:0")
D, HW = 128, 18720
ctxs = [131040] * 4
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_()
arena.v.normal_()
q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
for _ in range(3):
    K.attention(q, out, work, HW, 1 / math.sqrt(D), pair=True)
torch.cuda.synchronize()
buf = np.zeros((3, 128, 10), dtype=np.uint64)
lib = _lib.load()
lib.df_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert lib.df_trace_fetch(buf.ctypes.data, buf.nbytes) == 0
t0 = int(buf[2, 0, 0])
b = buf.astype(np.int64) - t0
print("it | MMA: kwait qk0 | pv1(wait P1) | qk1 | pv0(wait P0) || SM0: wait S  ldtm  max  half  full || SM1: wait S ldtm max half full")
for it in range(20, 30):
    m = b[2, it]
    s0, s1 = b[0, it], b[1, it]
    print(f"{it:3d} | {m[1]-m[0]:5d} {m[2]-m[1]:5d} | {m[3]-m[2]:5d} | {m[4]-m[3]:5d} | {m[5]-m[4]:5d} || "
          f"{s0[1]-s0[0]:5d} {s0[2]-s0[1]:5d} {s0[3]-s0[2]:5d} {s0[4]-s0[3]:5d} {s0[5]-s0[4]:5d} || "
          f"{s1[1]-s1[0]:5d} {s1[2]-s1[1]:5d} {s1[3]-s1[2]:5d} {s1[4]-s1[3]:5d} {s1[5]-s1[4]:5d}")
per_it = (b[2, 100, 0] - b[2, 20, 0]) / 80
print("pair softmax first half: max->exps(q0,q1) | wait_st | wg_bar | remote arrive")
for it in range(20, 30):
    s0 = b[0, it]
    print(it, s0[6] - s0[3], s0[7] - s0[6], s0[8] - s0[7], s0[4] - s0[8])
print("MMA loop period (cycles/iteration):", per_it, " ideal MMA at 8192 flop/clk:", 4 * 2 * 128 * 128 * 128 / 8192)
print("absolute stamps it 30 (rel. MMA k-wait start):")
for name, row in (("MMA", b[2, 30, :6]), ("SM0", b[0, 30, :6]), ("SM1", b[1, 30, :6])):
    print(name, (row - b[2, 30, 0]).tolist())
