"""Dev: B independent streams' packed Wan layers in ONE FMHA launch (48 heads, 4 arenas) vs B launches."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K

dev = torch.device('cuda:0')
D, HW = 128, 4680
ctxs = [2 * HW] * 9 + [6 * HW] * 3
flops1 = 4 * D * HW * sum(ctxs)
for B in (1, 2, 4):
    arenas = []
    for _ in range(B):
        a = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
        a.k.normal_(); a.v.normal_()
        arenas.append(a)
    H = len(ctxs)
    q = torch.randn(B * H * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(B * H * HW, D, device=dev, dtype=torch.bfloat16)
    work = []
    for b, a in enumerate(arenas):
        work += [K.HeadWork(a, a.allocate(c), c, b * H + h, b * H + h) for h, c in enumerate(ctxs)]
    batched = K.prepare_attention(q, out, work, HW, 1 / math.sqrt(D))
    single = [K.prepare_attention(q, out, work[b * H:(b + 1) * H], HW, 1 / math.sqrt(D)) for b in range(B)]
    def t(launch_lists, reps=20):
        for _ in range(3):
            for ll in launch_lists:
                for l in ll: l.launch(None)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for ll in launch_lists:
                for l in ll: l.launch(None)
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        return sorted(ts)[len(ts) // 2] * 1e3
    ub, us = t([batched]), t(single)
    print(f"B={B}: one launch {ub:.1f} us ({B * flops1 / ub / 1e6:.0f} TFLOP/s, {len(batched)} launch)  |  "
          f"{B} launches {us:.1f} us ({B * flops1 / us / 1e6:.0f} TFLOP/s)", flush=True)
    del arenas, q, out
    torch.cuda.empty_cache()
