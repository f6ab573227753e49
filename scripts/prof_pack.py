"""Small driver for ncu: the classification-time context pack of a whole Wan-shape session (dev tool).

30 layers x 12 heads of warm baseline rings (7 slots x 4680 tokens, d 128) re-laid under the
6d/3s/3n policies by ONE df_kv_pack launch (rebuild_caches), twice."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_20499_b200 as df  # noqa: E402
from paper_2601_20499_b200 import kernels as K  # noqa: E402
from paper_2601_20499_b200.kv_cache import RingStorage  # noqa: E402

dev = torch.device("cuda:0")
L, H, D, HW, W = 30, 12, 128, 4680, 6
cfg = df.SessionConfig(num_layers=L, num_heads=H, head_dim=D, HW=HW, window_len=W, ar_steps=W + 1,
                       denoise_steps=4, dummy_count=6 * L)
pol = df.baseline_policy(cfg)
per = K.KVArena.region_rows(pol.ring_slots * HW)
arena = K.KVArena(per * L * H, D, dev)
arena.k.normal_()
arena.v.normal_()
caches = []
for _ in range(L * H):
    c = df.HeadKVCache(pol, storage=RingStorage(arena, arena.allocate(pol.ring_slots * HW), pol.ring_slots, HW, D))
    for f in range(W):  # slot table only: the rows already hold data
        c._slot_frame[f] = f
    caches.append(c)
assign = ["dummy"] * 6 + ["sink"] * 3 + ["neighbor"] * 3
pols = [df.derive_policy(df.HeadClass(assign[i % H]), cfg) for i in range(L * H)]
for _ in range(2):
    stats = {}
    new = df.rebuild_caches(caches, pols, stats=stats)
    torch.cuda.synchronize()
    ms = stats["events"][0].elapsed_time(stats["events"][1])
    print(f"pack {stats['bytes'] / 1e9:.3f} GB in {ms * 1e3:.1f} us = {stats['bytes'] / ms / 1e6:.0f} GB/s")
    del new
