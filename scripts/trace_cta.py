"""Dev: per-CTA durations (clock64) vs the stream-K model loads (DF_SK_DUMP), packed Wan layer."""
import ctypes, math, os, re, sys, subprocess
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import _lib, kernels as K  # noqa: E402
dev = torch.device("cuda:0"); D = 128
lib = _lib.load()
ctxs, hw = [28080] * 3 + [9360] * 9, 4680
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_(); arena.v.normal_()
q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
for _ in range(3):
    K.attention(q, out, work, hw, 1 / math.sqrt(D))
torch.cuda.synchronize()
buf = np.zeros((1024, 2), dtype=np.uint64)
assert lib.df_trace_cta(buf.ctypes.data) == 0
dur = (buf[:, 1].astype(np.int64) - buf[:, 0].astype(np.int64))
plan = [l for l in open(os.environ.get("DUMP", "/dev/null")).read().splitlines() if l.startswith("cta ")][:148]
rows = []
for c, l in enumerate(plan):
    load = float(re.search(r"load ([\d.]+)", l).group(1))
    nseg = l.count("[h")
    rows.append((dur[c], load, nseg, l[:150]))
rows.sort(key=lambda r: -r[0])
for r in rows[:12]:
    print(f"{r[0]:9d} cyc  model {r[1]:6.1f}  segs {r[2]}  cyc/unit {r[0]/r[1]:.0f}  {r[3]}")
print("...")
for r in rows[-5:]:
    print(f"{r[0]:9d} cyc  model {r[1]:6.1f}  segs {r[2]}  cyc/unit {r[0]/r[1]:.0f}  {r[3]}")
