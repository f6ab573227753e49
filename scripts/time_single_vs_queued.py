import math, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2601_20499_b200 import kernels as K
dev = torch.device("cuda:0"); D = 128; HW = 4680
for name, ctxs in {"ext": [2 * HW] * 9 + [22 * HW] * 3, "packed": [2 * HW] * 9 + [6 * HW] * 3}.items():
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    ls = K.prepare_attention(q, out, work, HW, 1 / math.sqrt(D))
    print(name, "launches", len(ls))
    for _ in range(3):
        for l in ls: l.launch(None)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for l in ls: l.launch(None)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, "single+sync", [round(t) for t in sorted(ts)])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        for l in ls: l.launch(None)
    e1.record(); torch.cuda.synchronize()
    print(name, "back-to-back mean", round(e0.elapsed_time(e1) * 100))
    # with a sleep kernel before to isolate launch latency
    ts = []
    for _ in range(10):
        torch.cuda._sleep(20000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for l in ls: l.launch(None)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    print(name, "queued behind sleep", [round(t) for t in sorted(ts)])
