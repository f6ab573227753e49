"""Dev: pinned H2D / D2H bandwidth with 1, 2, 4 copy streams, and H2D concurrent with D2H."""
import torch, time
dev = torch.device("cuda:0")
n = 43 * 2**20 // 2  # one Wan layer's Q+K+V in bf16 elements (~43 MB)
hs = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(8)]
ds = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(8)]
def run(nstreams, reps=8, d2h=False):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    back = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(reps):
        for i in range(8):
            s = streams[i % nstreams]
            with torch.cuda.stream(s):
                ds[i].copy_(hs[i], non_blocking=True)
            if d2h:
                with torch.cuda.stream(back):
                    hs[(i + 4) % 8][: n // 3].copy_(ds[(i + 4) % 8][: n // 3], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return reps * 8 * n * 2 / dt / 1e9
for k in (1, 2, 4):
    print(f"H2D {k} stream(s): {run(k):.1f} GB/s;  with concurrent D2H: {run(k, d2h=True):.1f} GB/s H2D")
