"""Dev: per-CTA globaltimer timeline of the CTA-pair FMHA (DF_TRACE build): SM occupancy, finish spread,
item durations per head class.  DF_LIB_PATH=build_variants/trace/libdfb200.so python scripts/trace_timeline_pair.py"""
import math, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import _lib, kernels as K  # noqa: E402
dev = torch.device("cuda:0"); D = 128
lib = _lib.load()
cases = {"packed": ([28080] * 3 + [9360] * 9, 4680), "all_context": ([32760] * 12, 4680),
         "ext_c5": ([102960] * 3 + [9360] * 9, 4680), "hires_packed": ([112320] * 3 + [37440] * 9, 18720)}
only = sys.argv[1:] or list(cases)
for name in only:
    ctxs, hw = cases[name]
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * hw, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    for _ in range(3):
        K.attention(q, out, work, hw, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        e0.record(); K.attention(q, out, work, hw, 1 / math.sqrt(D)); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    buf = np.zeros((1024, 4), dtype=np.uint64)
    assert lib.df_trace_cta(buf.ctypes.data) == 0
    n = int((buf[:, 0] > 0).sum())
    b = buf[:n].astype(np.int64)
    t0 = b[:, 0].min()
    start, loop_end, end, sm = b[:, 0] - t0, b[:, 1] - t0, b[:, 2] - t0, b[:, 3]
    span = end.max()
    busy = np.zeros(148)
    last_end = np.zeros(148)
    for i in range(n):
        busy[sm[i]] += end[i] - start[i]
        last_end[sm[i]] = max(last_end[sm[i]], end[i])
    dur = (end - start) / 1e3
    print(f"{name}: event {np.median(ts):.1f} us; {n} CTAs ({n // 2} items), span {span / 1e3:.1f} us, "
          f"SM busy {busy.sum() / (148 * span) * 100:.1f}% of span, "
          f"SM finish min {last_end.min() / 1e3:.1f} median {np.median(last_end) / 1e3:.1f} max {last_end.max() / 1e3:.1f} us, "
          f"epilogue (loop end -> CTA end) {(end - loop_end).mean() / 1e3:.2f} us")
    # item durations grouped (even CTA of each pair)
    d_items = dur[0::2]
    hist = np.round(d_items).astype(int)
    vals, cnt = np.unique((hist // 5) * 5, return_counts=True)
    print("   item duration histogram (us bucket: count):", dict(zip(vals.tolist(), cnt.tolist())))
    gaps = []
    order = np.argsort(start)
    for s_id in range(148):
        idx = [i for i in order if sm[i] == s_id]
        for a, c in zip(idx, idx[1:]):
            gaps.append(start[c] - end[a])
    if gaps:
        print(f"   between-CTA gaps on an SM: mean {np.mean(gaps) / 1e3:.2f} us, max {np.max(gaps) / 1e3:.2f} us, n {len(gaps)}")
    print("   last 12 SM finishes (us):", np.round(np.sort(last_end)[-12:] / 1e3, 1).tolist(),
          "first 12:", np.round(np.sort(last_end)[:12] / 1e3, 1).tolist())
