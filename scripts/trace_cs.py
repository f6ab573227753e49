"""Dev: per-iteration timeline of CTA 0 of the column-split FMHA (DF_TRACE build, clock64 cycles)."""
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
    K.attention(q, out, work, HW, 1 / math.sqrt(D))
torch.cuda.synchronize()
buf = np.zeros((3, 128, 10), dtype=np.uint64)
lib = _lib.load()
lib.df_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert lib.df_trace_fetch(buf.ctypes.data, buf.nbytes) == 0
b = buf.astype(np.int64) - int(buf[2, 0, 0])
print("it | MMA: kwait qk0 | pv1 | qk1 | pv0 || SMt: waitS ldtm xchg exp+st arrive (t=0) || (t=1)")
for it in range(20, 40):
    m, s0, s1 = b[2, it], b[0, it], b[1, it]
    print(f"{it:3d} | {m[1]-m[0]:5d} {m[2]-m[1]:5d} | {m[3]-m[2]:5d} | {m[4]-m[3]:5d} | {m[5]-m[4]:5d} || "
          + " ".join(f"{s0[k+1]-s0[k]:5d}" for k in range(5)) + " || "
          + " ".join(f"{s1[k+1]-s1[k]:5d}" for k in range(5)))
print("MMA loop period (cycles/iteration):", (b[2, 100, 0] - b[2, 20, 0]) / 80, " ideal:", 2048)
for name, row in (("MMA", b[2, 30, :6]), ("SM0", b[0, 30, :6]), ("SM1", b[1, 30, :6])):
    print(name, (row - b[2, 30, 0]).tolist())
