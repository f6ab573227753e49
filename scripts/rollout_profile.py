"""Dev: per-AR-step device time of the C3 rollout (Wan shape, ProjectedModel, DHP + packing)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_20499_b200 as df
from paper_2601_20499_b200 import engine

L, H, D, HW, W = 30, 12, 128, 4680, 6
dev = torch.device("cuda:0")
Dm = H * D
g = torch.Generator(device=dev).manual_seed(11)
weights = [{n: torch.randn(Dm, Dm, device=dev, generator=g) * (0.5 / Dm ** 0.5) for n in ("q", "k", "v", "o")} for _ in range(L)]
fg = torch.Generator(device=dev)
def frames(ar, t):
    fg.manual_seed(1000 * ar + t)
    return torch.randn(HW, Dm, device=dev, generator=fg)
model = df.ProjectedModel(weights, frames, H, D, HW, device=dev)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
cfg = df.SessionConfig(num_layers=L, num_heads=H, head_dim=D, HW=HW, window_len=W, ar_steps=steps, denoise_steps=4,
                       dummy_count=L * H // 2, probe_ar_step=2, subsample_ratio=0.25)
for graphs in [False, True][: 2 if len(sys.argv) < 3 else 1]:
    s = df.Session(model, cfg, "packed", device=dev, graphs=graphs)
    orig = s._run_step
    def timed(ar, orig=orig):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); orig(ar); e1.record(); torch.cuda.synchronize()
        if ar < 12 or ar % 5 == 0:
            print(f"graphs={graphs} step {ar}: device {e0.elapsed_time(e1):7.1f} ms  host {1e3*(time.perf_counter()-t0):7.1f} ms", flush=True)
    s._run_step = timed
    t0 = time.perf_counter()
    s.run()
    print(f"total {time.perf_counter() - t0:.2f} s", flush=True)
    if s.assignment is not None:
        import collections
        per_layer = collections.Counter()
        for l in range(L):
            cl = s.assignment.classes[l * H:(l + 1) * H]
            per_layer[(sum(c is df.HeadClass.DUMMY for c in cl), sum(c is df.HeadClass.SINK for c in cl))] += 1
        print("per-layer (dummy, sink) counts:", dict(per_layer))
