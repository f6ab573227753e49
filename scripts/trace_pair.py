"""Dev: per-tile timeline of CTA 0 of the CTA-pair FMHA (DF_TRACE build, clock64 cycles).

MMA (who 3) per kv tile j: [0] QK_j issue (K_j landed), [1] PV_j issue (P first half + V landed),
[2] PV_j issued.  Softmax WG g (who g) per use u (tile j = 3u + g): [0] wait S, [1] S ready,
[2] row max done, [5] m handed on, [3] rescale done, [4] P released.
"""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import _lib, kernels as K  # noqa: E402

dev = torch.device("cuda:0")
D = 128
HW = int(os.environ.get("HW", 18720))
ctxs = [int(os.environ.get("CTX", 131040))] * int(os.environ.get("HEADS", 4))
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_()
arena.v.normal_()
q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
for _ in range(3):
    K.attention(q, out, work, HW, 1 / math.sqrt(D), pair=True)
torch.cuda.synchronize()
buf = np.zeros((4, 128, 10), dtype=np.uint64)
lib = _lib.load()
lib.df_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int64]
assert lib.df_trace_fetch(buf.ctypes.data, buf.nbytes) == 0
t0 = int(buf[3, 0, 0])
b = buf.astype(np.int64) - t0
print(" j |  QK_j  PV_j-start PV_j-issued || WG: waitS  Sready  max  handed  resc  Prel | Swait ld+max hand resc exp")
for j in range(18, 54):
    m = b[3, j]
    w, u = j % 3, j // 3
    s = b[w, u]
    print(f"{j:3d} | {m[0]:7d} {m[1]:7d} {m[2]:7d} || {s[0]:7d} {s[1]:7d} {s[2]:7d} {s[5]:7d} {s[3]:7d} {s[4]:7d} | "
          f"{s[1]-s[0]:5d} {s[2]-s[1]:5d} {s[5]-s[2]:5d} {s[3]-s[5]:5d} {s[4]-s[3]:5d}")
per = (b[3, 100, 0] - b[3, 20, 0]) / 80
print("MMA period (cycles per kv tile):", per, " ideal (QK + PV, M=256 over 2 SMs):", 1024)
