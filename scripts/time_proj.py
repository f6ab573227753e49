"""Dev timing: fused projection GEMMs vs cuBLAS (torch.matmul) at the Wan shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
hw, H, d = 4680, 12, 128
D = H * d


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


x = torch.randn(hw, D, device=dev).to(torch.bfloat16)
w = (torch.randn(3 * D, D, device=dev) / D**0.5).to(torch.bfloat16)
q = torch.empty(H, hw, d, dtype=torch.bfloat16, device=dev)
plane_k = torch.empty(H * 7 * hw, d, dtype=torch.bfloat16, device=dev)
plane_v = torch.empty_like(plane_k)
kd = [plane_k[h * 7 * hw + 3 * hw : h * 7 * hw + 4 * hw] for h in range(H)]
vd = [plane_v[h * 7 * hw + 3 * hw : h * 7 * hw + 4 * hw] for h in range(H)]
o = torch.randn(H, hw, d, device=dev).to(torch.bfloat16)
wo = (torch.randn(D, D, device=dev) / D**0.5).to(torch.bfloat16)
xf = torch.randn(hw, D, device=dev)
xb = torch.empty(hw, D, dtype=torch.bfloat16, device=dev)

for bn in ("128", "192", "256", None):
    if bn:
        os.environ["DF_PROJ_BN"] = bn
    else:
        os.environ.pop("DF_PROJ_BN", None)
    lq = K.prepare_qkv_projection(x, w, q, kd, vd, d)
    lo = K.prepare_out_projection(o, wo, xf, xb, d)
    tq = timeit(lambda: lq.launch())
    to = timeit(lambda: lo.launch())
    fq, fo = 2 * hw * 3 * D * D, 2 * hw * D * D
    print(f"BN={bn or 'auto'}: qkv {tq:.1f} us {fq / tq / 1e6:.0f} TFLOP/s | out-proj {to:.1f} us {fo / to / 1e6:.0f} TFLOP/s")

out = torch.empty(hw, 3 * D, dtype=torch.bfloat16, device=dev)
tc = timeit(lambda: torch.matmul(x, w.T, out=out))
tc2 = timeit(lambda: torch.matmul(o.permute(1, 0, 2).reshape(hw, D), wo.T))
print(f"cuBLAS qkv GEMM only {tc:.1f} us {2 * hw * 3 * D * D / tc / 1e6:.0f} TFLOP/s; "
      f"out-proj (+merge copy, no residual) {tc2:.1f} us")
ref = torch.empty(H, hw, d, dtype=torch.bfloat16, device=dev)
def unfused():
    y = torch.matmul(x, w.T, out=out).view(hw, 3, H, d)
    ref.copy_(y[:, 0].transpose(0, 1))
    for h in range(H):
        kd[h].copy_(y[:, 1, h])
        vd[h].copy_(y[:, 2, h])
print(f"cuBLAS + scatter copies (unfused qkv) {timeit(unfused):.1f} us")

# out-projection with cold operands: 8 rotating (o, x, x_bf16) sets (8 x 58 MB > L2), as in the 30-layer step
sets = [(torch.randn(H, hw, d, device=dev).to(torch.bfloat16), torch.randn(hw, D, device=dev),
         torch.empty(hw, D, dtype=torch.bfloat16, device=dev)) for _ in range(8)]
for bn in ("192", "256", None):
    if bn:
        os.environ["DF_PROJ_BN"] = bn
    else:
        os.environ.pop("DF_PROJ_BN", None)
    ls = [K.prepare_out_projection(o_, wo, x_, xb_, d) for o_, x_, xb_ in sets]
    i = [0]
    def step():
        ls[i[0] % 8].launch()
        i[0] += 1
    t = timeit(step, reps=80)
    print(f"cold out-proj BN={bn or 'auto'}: {t:.1f} us {2 * hw * D * D / t / 1e6:.0f} TFLOP/s")
