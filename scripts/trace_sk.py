"""Dev: stream-K timeline of CTA 0 (DF_TRACE build)."""
import ctypes, math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import _lib, kernels as K  # noqa: E402
dev = torch.device("cuda:0"); D = 128
lib = _lib.load()
lib.df_trace_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int64]
ctxs, hw = [28080] * 3 + [9360] * 9, 4680
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_(); arena.v.normal_()
q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
for _ in range(3):
    K.attention(q, out, work, hw, 1 / math.sqrt(D))
torch.cuda.synchronize()
buf = np.zeros((3, 128, 10), dtype=np.uint64)
assert lib.df_trace_fetch(buf.ctypes.data, buf.nbytes) == 0
b = buf.astype(np.int64); t0 = b[2, 127, 6]
for it in list(range(0, 8)) + list(range(160, 175)):
    if it >= 127: break
    m = b[2, it] - t0; s0 = b[0, it] - t0; s1 = b[1, it] - t0
    print(it, "MMA", m[:6].tolist(), "| SM0", s0[:6].tolist(), "| SM1", s1[:6].tolist())
for it in range(100, 127):
    m = b[2, it] - t0
    print(it, "MMA", m[:6].tolist())
