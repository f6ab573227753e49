"""Dev: SM clock and power while one FMHA launch shape runs back to back for ~1.5 s (NVML samples).

Tells a power-capped kernel (clock drops under load) from a cycle-bound one.  DF_PAIR=1 picks the
CTA-pair kernel; DF_LIB_PATH a build variant."""
import math
import os
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_20499_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
D = 128
PAIR = os.environ.get("DF_PAIR") == "1"
pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)


def run(name, ctxs, HW):
    H = len(ctxs)
    arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
    arena.k.normal_()
    arena.v.normal_()
    q = torch.randn(H * HW, D, device=dev).to(torch.bfloat16)
    out = torch.empty(H * HW, D, device=dev, dtype=torch.bfloat16)
    work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
    launches = K.prepare_attention(q, out, work, HW, 1 / math.sqrt(D), pair=PAIR)
    for _ in range(3):
        for l in launches:
            l.launch()
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(hnd) / 1000.0))
            time.sleep(0.005)

    th = threading.Thread(target=poll)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    th.start()
    e0.record()
    t0 = time.time()
    while time.time() - t0 < 1.5:
        for _ in range(5):
            for l in launches:
                l.launch()
        n += 5
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    us = e0.elapsed_time(e1) * 1e3 / n
    tf = 4 * D * HW * sum(ctxs) / (us * 1e-6) / 1e12
    late = samples[len(samples) // 3:]
    mhz = sorted(s[0] for s in late)[len(late) // 2]
    w = sorted(s[1] for s in late)[len(late) // 2]
    reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd)
    print(f"{name}: {us:.1f} us  {tf:.0f} TFLOP/s  sm {mhz} MHz  {w:.0f} W  reasons 0x{reasons:x}", flush=True)


run("packed_6d3s3n", [28080] * 3 + [9360] * 9, 4680)
run("hires_baseline", [131040] * 12, 18720)
