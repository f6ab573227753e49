import math, sys, torch
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device('cuda:0')
def ws_nonzero():
    bad = {k: int((v[:256].view(torch.int32) != 0).sum().item()) for k, v in K._WORKSPACES.items()}
    return bad
def run(hw, width, ctxs, pair, scale_q=1.0):
    pass
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), width, dev)
    arena.k.normal_(); arena.v.normal_()
    q = (torch.randn(len(ctxs) * hw, width, device=dev) * scale_q).to(torch.bfloat16)
    out = torch.empty(len(ctxs) * hw, width, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    K.attention(q, out, work, hw, 1/math.sqrt(width), pair=pair)
    torch.cuda.synchronize()
    return out
for pair in (False, True):
    for hw, width, ctxs in [(256,128,[256]), (300,128,[300,600,1000]), (64*3,64,[192,384,1344,576]), (300,128,[300,600,1000,4680*2+77])]:
        if width == 64 and pair: continue
        run(hw, width, ctxs, pair)
        print("pair", pair, hw, ctxs, "nonzero counters:", ws_nonzero())

# the failing sequence: small splits, then the hi-res launch twice
a = run(18720, 128, [2 * 18720, 2 * 18720, 6 * 18720], False)
print("hires nonzero counters:", ws_nonzero(), "nan/huge:", bool((a.float().abs() > 1e4).any()))
b = run(18720, 128, [2 * 18720, 2 * 18720, 6 * 18720], False)
print("hires again:", ws_nonzero(), "huge:", bool((b.float().abs() > 1e4).any()))
