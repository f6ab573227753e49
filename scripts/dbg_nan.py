import math, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K
dev = torch.device('cuda:0')
def case(D, HW, ctxs, fill='randn'):
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    if fill == 'randn': arena.k.normal_(); arena.v.normal_()
    q = torch.randn(len(ctxs) * HW, D, device=dev).to(torch.bfloat16)
    out = torch.full((len(ctxs) * HW, D), float('nan'), device=dev, dtype=torch.bfloat16)
    work = []
    for h, c in enumerate(ctxs):
        b = arena.allocate(c)
        if fill != 'randn':
            arena.k[b:b+c] = torch.randn(c, D, device=dev).to(torch.bfloat16); arena.v[b:b+c] = torch.randn(c, D, device=dev).to(torch.bfloat16)
        work.append(K.HeadWork(arena, b, c, h, h))
    K.attention(q, out, work, HW, 1 / math.sqrt(D)); torch.cuda.synchronize()
    res = []
    for h, w in enumerate(work):
        ref = torch.softmax(q[h*HW:(h+1)*HW].float() @ arena.k[w.base_row:w.base_row+w.n_tok].float().T / math.sqrt(D), -1) @ arena.v[w.base_row:w.base_row+w.n_tok].float()
        got = out[h*HW:(h+1)*HW].float()
        nanrows = torch.isnan(got).any(1).nonzero().flatten().tolist()
        err = ((got-ref).abs().nan_to_num(1e9).max()/ref.abs().max()).item()
        res.append((round(err, 4), len(nanrows), nanrows[:4]))
    return res
print(os.environ.get('DF_LIB_PATH'))
print('300', case(128, 300, [300, 600, 1000], 'slices'))
print('256', case(128, 256, [256], 'slices'))
print('packed', case(128, 4680, [28080]*3 + [9360]*9)[:4])
