"""Dev: 30-layer packed step through packed_step(timed=False) -- no event records between launches,
so the staging copy can pair with the previous FMHA by programmatic dependent launch (DF_APPEND_PDL)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2601_20499_b200 as df

dev = torch.device("cuda:0")
L, H, D, HW, W = bench.L, bench.H, bench.D, bench.HW, bench.W
cfg = df.SessionConfig(num_layers=L, num_heads=H, head_dim=D, HW=HW, window_len=W, ar_steps=W + 1,
                       denoise_steps=bench.DENOISE, dummy_count=6 * L)
gen = torch.Generator(device=dev).manual_seed(1)
caches, _ = bench.build_caches(df, cfg, dev, gen)
classes = [df.HeadClass.DUMMY] * 6 + [df.HeadClass.SINK] * 3 + [df.HeadClass.NEIGHBOR] * 3
pols = [df.derive_policy(c, cfg) for _ in range(L) for c in classes]
new = df.rebuild_caches([c for layer in caches for c in layer], pols)
packed = [new[l * H:(l + 1) * H] for l in range(L)]
inputs = [tuple(torch.randn(H, HW, D, device=dev, generator=gen).to(torch.bfloat16) for _ in range(3)) for _ in range(L)]
def step():
    for layer in range(L):
        q, k, v = inputs[layer]
        df.packed_step(q, packed[layer], [df.FrameBlock(W, k[h], v[h]) for h in range(H)], classes, cfg, timed=False)
for timed_name in ("timed=False",):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        step()
    e1.record(); torch.cuda.synchronize()
    print(f"PDL={os.environ.get('DF_APPEND_PDL', '1')} {timed_name}: {e0.elapsed_time(e1) / 20:.3f} ms per step")
