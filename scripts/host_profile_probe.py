"""Dev: cProfile of the probe/classification AR step of a Wan-shape Session."""
import cProfile, os, pstats, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_20499_b200 as df

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
cfg = df.SessionConfig(num_layers=L, num_heads=H, head_dim=D, HW=HW, window_len=W, ar_steps=6, denoise_steps=4,
                       dummy_count=L * H // 2, probe_ar_step=2, subsample_ratio=0.25)
s = df.Session(model, cfg, "packed", device=dev)
for ar in range(2):
    s._run_step(ar)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
s._run_step(2)
torch.cuda.synchronize()
pr.disable()
print(f"probe step: {(time.perf_counter() - t0) * 1e3:.1f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
