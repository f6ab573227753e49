"""ncu driver: the out-projection alone at the Wan shape, cold operands (8 rotating sets); DF_PROJ_BN / DF_PROJ_PAIR pick the tiling."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
hw, H, d = 4680, 12, 128
D = H * d
wo = (torch.randn(D, D, device=dev) / D**0.5).to(torch.bfloat16)
sets = [(torch.randn(H, hw, d, device=dev).to(torch.bfloat16), torch.randn(hw, D, device=dev),
         torch.empty(hw, D, dtype=torch.bfloat16, device=dev)) for _ in range(8)]
ls = [K.prepare_out_projection(o_, wo, x_, xb_, d) for o_, x_, xb_ in sets]
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    ls[i % 8].launch()
torch.cuda.synchronize()
print("ok")
