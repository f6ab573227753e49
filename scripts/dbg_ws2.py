import math, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device('cuda:0')
def counters():
    return {k: int((v[:1024].view(torch.int32) != 0).sum().item()) for k, v in K._WORKSPACES.items()}
def run(hw, width, ctxs):
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * hw, width, device=dev).to(torch.bfloat16)
    out = torch.full((len(ctxs) * hw, width), float('nan'), device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    K.attention(q, out, work, hw, 1 / math.sqrt(width))
    torch.cuda.synchronize()
    return bool(torch.isnan(out.float()).any())
for w in (5, 9, 15):
    for n in range(1, w + 2):
        nan = run(2048, 64, [n * 2048] * 8)
        c = counters()
        if nan or any(c.values()):
            print("d64 window", w, "frames", n, "unwritten rows:", nan, "nonzero counter words:", c)
print("hires unwritten rows:", run(18720, 128, [2 * 18720, 2 * 18720, 6 * 18720]), counters())
