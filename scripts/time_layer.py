"""Per-layer timing of df_attn_fwd at the Wan-1.3B shape (dev tool; not the bench)."""
import math, sys, os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K

dev = torch.device('cuda:0')
D = 128
PAIR = os.environ.get("DF_PAIR") == "1"
def run(ctxs, HW=4680, reps=20, probe=False):
    H = len(ctxs)
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_(); arena.v.normal_()
    q = torch.randn(H * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(H * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    pb = None
    if probe:
        pb = K.ProbeBuffers(torch.zeros(H, 64, dtype=torch.uint8, device=dev), torch.ones(HW, dtype=torch.uint8, device=dev), torch.zeros(H, HW, 3, device=dev))
    for _ in range(3): K.attention(q, out, work, HW, 1/math.sqrt(D), pb, pair=PAIR)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    e0.record()
    for _ in range(reps): K.attention(q, out, work, HW, 1/math.sqrt(D), pb, pair=PAIR)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    return t * 1e3, 4 * D * HW * sum(ctxs) / (t * 1e-3) / 1e12
cases = {
 'small_12x9360': ([9360] * 12, 4680),
 'small_2x32760': ([32760] * 2, 4680),
 'baseline_12x32760': ([32760] * 12, 4680),
 'packed_6d3s3n': ([28080] * 3 + [9360] * 9, 4680),
 'packed_3d4s5n': ([28080] * 5 + [9360] * 7, 4680),
 'ext_3nb_102960': ([102960] * 3 + [9360] * 9, 4680),
 'hires_baseline_12x131040': ([131040] * 12, 18720),
 'hires_packed_6d3s3n': ([112320] * 3 + [37440] * 9, 18720),
}
for k, (c, hw) in cases.items():
    us, tf = run(c, hw, reps=10 if hw > 5000 else 20)
    print(f"{k}: {us:.1f} us/layer  {tf:.1f} TFLOP/s  ({tf/1672.3*100:.1f}% of measured bf16 peak)", flush=True)
us, tf = run([32760] * 12, probe=True)
print(f"probe_baseline: {us:.1f} us/layer  {tf:.1f} TFLOP/s", flush=True)
