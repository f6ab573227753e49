"""Small driver for ncu: the two projection GEMMs at the Wan shape (dev tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
hw, H, d = 4680, 12, 128
D = H * d
x = torch.randn(hw, D, device=dev).to(torch.bfloat16)
w = (torch.randn(3 * D, D, device=dev) / D**0.5).to(torch.bfloat16)
q = torch.empty(H, hw, d, dtype=torch.bfloat16, device=dev)
plane_k = torch.empty(H * 7 * hw, d, dtype=torch.bfloat16, device=dev)
plane_v = torch.empty_like(plane_k)
kd = [plane_k[h * 7 * hw + 3 * hw: h * 7 * hw + 4 * hw] for h in range(H)]
vd = [plane_v[h * 7 * hw + 3 * hw: h * 7 * hw + 4 * hw] for h in range(H)]
o = torch.randn(H, hw, d, device=dev).to(torch.bfloat16)
wo = (torch.randn(D, D, device=dev) / D**0.5).to(torch.bfloat16)
xf = torch.randn(hw, D, device=dev)
xb = torch.empty(hw, D, dtype=torch.bfloat16, device=dev)
lq = K.prepare_qkv_projection(x, w, q, kd, vd, d)
lo = K.prepare_out_projection(o, wo, xf, xb, d)
for _ in range(3):
    lq.launch()
    lo.launch()
torch.cuda.synchronize()
print("ok")
