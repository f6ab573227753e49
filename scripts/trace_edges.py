"""Dev: prologue / epilogue timeline of CTA 0 (DF_TRACE build): where the per-launch fixed cost goes."""
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
lib = _lib.load()
lib.df_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int64]
for name, ctxs, hw in [("64x64tiles", [64 * 128] * 64, 256), ("wan_packed", [28080] * 3 + [9360] * 9, 4680)]:
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_()
    arena.v.normal_()
    q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    for _ in range(3):
        K.attention(q, out, work, hw, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    buf = np.zeros((3, 128, 10), dtype=np.uint64)
    assert lib.df_trace_fetch(buf.ctypes.data, buf.nbytes) == 0
    b = buf.astype(np.int64)
    t0 = b[2, 127, 6]
    n = int((b[2, :127, 0] > 0).sum())
    last = n - 1
    print(f"== {name}: CTA0 {n} kv tiles traced")
    print("  setup (barrier init + TMEM alloc + sync):", b[2, 127, 7] - t0)
    print("  first MMA k-wait start / k ready:", b[2, 0, 0] - t0, b[2, 0, 1] - t0)
    print("  first S0 seen by softmax0:", b[0, 0, 1] - t0, " first S1:", b[1, 0, 1] - t0)
    print("  last tile: S0 seen", b[0, last, 1] - t0, " P0 full", b[0, last, 5] - t0, " P1 full", b[1, last, 5] - t0)
    print("  epilogue start t0/t1:", b[0, 127, 6] - t0, b[1, 127, 6] - t0, " epilogue end:", b[0, 127, 7] - t0,
          b[1, 127, 7] - t0, " kernel end:", b[2, 127, 8] - t0)
    per = (b[2, last, 0] - b[2, 1, 0]) / max(1, last - 1)
    print(f"  steady period {per:.0f} cycles/kv tile")
