"""Dev: per-CTA globaltimer timeline of one packed Wan launch (DF_TRACE build): SM occupancy and idle."""
import math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import _lib, kernels as K  # noqa: E402
dev = torch.device("cuda:0"); D = 128
lib = _lib.load()
cases = {"packed": ([28080] * 3 + [9360] * 9, 4680), "hires_packed": ([112320] * 3 + [37440] * 9, 18720)}
for name, (ctxs, hw) in cases.items():
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    for _ in range(3):
        K.attention(q, out, work, hw, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    buf = np.zeros((1024, 4), dtype=np.uint64)
    assert lib.df_trace_cta(buf.ctypes.data) == 0
    n = int((buf[:, 0] > 0).sum())
    b = buf[:n].astype(np.int64)
    t0 = b[:, 0].min()
    start, loop_end, end, sm = b[:, 0] - t0, b[:, 1] - t0, b[:, 2] - t0, b[:, 3]
    span = end.max()
    busy = np.zeros(148)
    for i in range(n):
        busy[sm[i]] += end[i] - start[i]
    last_end = np.zeros(148)
    for i in range(n):
        last_end[sm[i]] = max(last_end[sm[i]], end[i])
    epi = (end - loop_end).mean()
    print(f"{name}: {n} CTAs, span {span / 1e3:.1f} us, SM busy {busy.sum() / (148 * span) * 100:.1f}% of span, "
          f"mean CTA {np.mean(end - start) / 1e3:.1f} us, epilogue (loop end -> CTA end) {epi / 1e3:.2f} us, "
          f"launch ramp (last CTA start of wave 1) {np.sort(start)[147] / 1e3:.2f} us, "
          f"SM finish spread {(last_end.max() - last_end.min()) / 1e3:.1f} us (min {last_end.min() / 1e3:.1f})")
    gaps = []
    order = np.argsort(start)
    for s_id in range(148):
        idx = [i for i in order if sm[i] == s_id]
        for a, c in zip(idx, idx[1:]):
            gaps.append(start[c] - end[a])
    if gaps:
        print(f"   between-CTA gaps on an SM: mean {np.mean(gaps) / 1e3:.2f} us, max {np.max(gaps) / 1e3:.2f} us, n {len(gaps)}")

# per-CTA detail of the packed launch (blockIdx order = launch order)
ctxs, hw = cases["packed"]
arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
arena.k.normal_(); arena.v.normal_()
q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
for _ in range(3):
    K.attention(q, out, work, hw, 1 / math.sqrt(D))
torch.cuda.synchronize()
buf = np.zeros((1024, 4), dtype=np.uint64)
assert lib.df_trace_cta(buf.ctypes.data) == 0
b = buf[:285].astype(np.int64)
t0 = b[:, 0].min()
print("blockIdx: start end dur(us) loop(us) sm")
for i in list(range(0, 285, 12)) + list(range(270, 285)):
    print(i, round((b[i, 0] - t0) / 1e3, 1), round((b[i, 2] - t0) / 1e3, 1), round((b[i, 2] - b[i, 0]) / 1e3, 1),
          round((b[i, 1] - b[i, 0]) / 1e3, 1), b[i, 3])
