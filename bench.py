#!/usr/bin/env python
"""Benchmark of the Dummy Forcing attention hot path on B200 (BASELINE.json).

Workload (BASELINE.json configs[1]): Wan-2.1-1.3B attention shape -- 30
layers x 12 heads x d128, HW = 3 x 1560 = 4680 tokens per AR chunk, window
W=6 (sink + 5 recent), warm cache, bf16, synthetic random Q/K/V resident in
HBM.  Fixed paper-default assignment per layer: 6 dummy / 3 sink / 3
neighbor heads (50% dummy), packed mode.

One *step* = one denoise iteration of a warm AR step across all 30 layers,
each layer = one public-API ``packed_step`` call (current-frame staging
kernel + ONE ragged tcgen05 FMHA launch).  An AR step is 4 denoise iterations
and yields 3 latent frames, so

    value (attention-only AR FPS, latent frames/s) = N * 3 / (4 * t_step)

The same kernel with every head a baseline-window head (all-context) is timed
beside it (the >=1.8x comparator), as is the classification-time context
packing (df_kv_pack, HBM-bound).  ``e2e`` repeats the packed step through the
same public API with the Q/K/V of every layer coming from pinned HOST memory
and the outputs copied back to the host inside the timed region.

``--impl reference`` times the reference algorithm on the host cores: the
numpy oracle port of engine.py:87-137 (the reference is pure Python/numpy and
cannot travel to the GPU box), one whole warm layer (all 12 heads) per step,
the FPS extrapolated to 30 layers x 4 denoise iterations and marked so.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dummy-head attention µs/layer & TFLOP/s; AR video FPS (Wan-1.3B shape), 1–8 GPU"
UNIT = "latent frames/s (attention-only AR FPS)"
L, H, D, HW, W = 30, 12, 128, 4680, 6
DENOISE, FRAMES_PER_STEP = 4, 3
ASSIGN = ["dummy"] * 6 + ["sink"] * 3 + ["neighbor"] * 3


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j["bf16_tflops"], j["hbm_gbs"], "measured (MEASURED_PEAKS.json: bf16_tflops burst, hbm_gbs)"
    return 1590.0, 6650.0, "fallback (B200_PROFILING.md)"


def sustained_peak(burst: float) -> float:
    """bf16_tflops_sustained of MEASURED_PEAKS.json (cuBLAS back to back for 4 s), else the burst figure."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p)).get("bf16_tflops_sustained", burst))
    return burst


def layer_flops(ctxs):
    return 4 * D * HW * sum(ctxs)


PACKED_CTX = [2 * HW] * 6 + [2 * HW] * 3 + [6 * HW] * 3  # dummy [i-1,i], sink [0,i], neighbor [i-5..i]
BASE_CTX = [7 * HW] * 12


NCU_ATTN = os.path.join("profiles", "r2_attn_packed_ncu.json")


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of one packed launch from the committed ncu capture."""
    return ncu_bytes(NCU_ATTN)


NCU_PACK = os.path.join("profiles", "r2_pack_ncu.json")


def ncu_bytes(rel):
    """dram__bytes_read.sum + dram__bytes_write.sum of a committed ncu summary (bytes), or None."""
    p = os.path.join(ROOT, rel)
    if not os.path.exists(p):
        return None
    j = json.load(open(p))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return int(sum(float(j[k]["value"]) * scale.get(j[k]["unit"], 1) for k in ("dram__bytes_read.sum",
                                                                               "dram__bytes_write.sum")))


def attn_alg_bytes():
    """Q + K/V of every head once + O (packed layer)."""
    return (H * HW * D * 2) * 2 + sum(PACKED_CTX) * D * 2 * 2


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) from a background thread every 2 ms -- the handle is
    opened before the region, so the first sample lands at its start; falls
    back to ``nvidia-smi -lms 20`` when NVML is unavailable.
    """

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    PERIOD_S = 0.002

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.samples: list[tuple[float, int]] = []  # (sm MHz, reason bitmask)
        self.max_mhz = None
        self.lines: list[str] = []
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
        except Exception:  # no NVML: nvidia-smi fallback
            self.nvml = None

    def _poll(self):
        nv, h = self.nvml, self.handle
        while not self._stop.is_set():
            try:
                self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                     int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:
                pass
            self._stop.wait(self.PERIOD_S)

    def __enter__(self):
        if self.nvml is not None:
            import threading

            self._stop = threading.Event()
            self._thread = threading.Thread(target=self._poll, daemon=True)
            self._thread.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self._stop.set()
            self._thread.join()
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self) -> dict:
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], self.max_mhz or 0, set()
        if self.nvml is not None:
            nv = self.nvml
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            for mhz, mask in self.samples:
                sm.append(mhz)
                reasons.update(n for n in names if mask & bits[n])
            source = f"nvml every {self.PERIOD_S * 1e3:.0f} ms"
        else:
            for l in self.lines:
                parts = [x.strip() for x in l.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            source = "nvidia-smi -lms 20"
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "sm_min_mhz": min(sm) if sm else None, "reasons": sorted(reasons), "samples": len(sm),
                "source": source}


# ------------------------------------------------------------------ helpers
def dist_setup():
    import torch

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier_max(value: float, ws: int) -> float:
    if ws == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def build_caches(df, cfg, dev, gen):
    """Warm baseline rings for every layer: frames 0..W-1 appended (sink 0 + W-1 recent)."""
    import torch

    from paper_2601_20499_b200 import kernels as K
    from paper_2601_20499_b200.kv_cache import RingStorage, launch_segments

    pol = df.baseline_policy(cfg)
    per = K.KVArena.region_rows(pol.ring_slots * HW)
    arena = K.KVArena(per * L * H, K.padded_width(D), dev)
    caches = [[df.HeadKVCache(pol, storage=RingStorage(arena, arena.allocate(pol.ring_slots * HW), pol.ring_slots,
                                                         HW, D)) for _ in range(H)] for _ in range(L)]
    for f in range(W):
        for layer in range(L):
            k = torch.randn(H, HW, D, device=dev, generator=gen).to(torch.bfloat16)
            v = torch.randn(H, HW, D, device=dev, generator=gen).to(torch.bfloat16)
            segs = []
            for h in range(H):
                segs += caches[layer][h].append_segments(df.FrameBlock(f, k[h], v[h]), dev)
            launch_segments(segs)
    torch.cuda.synchronize()
    return caches, arena


def run_layers(df, cfg, caches, inputs, classes, mode, timed=True, chain=None):
    """One step (30 layers) through the public step functions.  ``timed``: True = CUDA events around
    every launch, False = none, an int = only that layer (per-launch events between a layer's FMHA and
    the next layer's staging copy break their programmatic-dependent-launch pairing).  ``chain``: a
    kernels.LaunchChain -- this loop issues nothing but library launches on the stream, so each
    layer's staging copy may overlap the previous layer's FMHA."""
    lcs = []
    for layer in range(L):
        q, k, v = inputs[layer]
        blocks = [df.FrameBlock(W, k[h], v[h]) for h in range(H)]
        t = timed if isinstance(timed, bool) else (layer == timed)
        if mode == "baseline":
            out, lc = df.baseline_step(q, caches[layer], blocks, cfg, timed=t, chain=chain)
        else:
            out, lc = df.packed_step(q, caches[layer], blocks, classes, cfg, timed=t, chain=chain)
        lcs.append(lc)
    return lcs


def time_steps(fn, steps, warmup):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    all_lcs = []
    e0.record()
    for _ in range(steps):
        all_lcs.append(fn())
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps, all_lcs


def full_layer(df, cfg, packed, classes, dev, gen, args, ws, bf16_peak):
    """the whole attention block of a layer on the device.

    x (fp32 residual + bf16 copy) -> df_qkv_project (Q + K/V written into the
    pending ring slots) -> packed_step (ONE FMHA, no staging copy) ->
    df_out_project (head merge @ W_o + residual).  Random W (x @ W scale
    1/sqrt(D)); reported beside the attention-only metric, not in `value`.
    """
    import torch

    from paper_2601_20499_b200 import kernels as K

    Dm = H * D
    wqkv = [(torch.randn(3 * Dm, Dm, device=dev, generator=gen) / Dm**0.5).to(torch.bfloat16) for _ in range(L)]
    wo = [(torch.randn(Dm, Dm, device=dev, generator=gen) / Dm**0.5).to(torch.bfloat16) for _ in range(L)]
    xs = df.ResidualStream(torch.randn(HW, Dm, device=dev, generator=gen))
    views = [[c.pending_view(HW, D, dev) for c in packed[layer]] for layer in range(L)]
    qbuf = [torch.empty(H, HW, D, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    proj = [K.prepare_qkv_projection(xs.bf16, wqkv[layer], qbuf[layer], [kv[0] for kv in views[layer]],
                                     [kv[1] for kv in views[layer]], D) for layer in range(L)]
    blocks = [[df.FrameBlock(W, k, v) for k, v in views[layer]] for layer in range(L)]
    split = {"qkv": 0.0, "attn": 0.0, "oproj": 0.0}

    def step(ev=None):
        for layer in range(L):
            if ev is not None:
                ev[layer][0].record()
            proj[layer].launch()
            if ev is not None:
                ev[layer][1].record()
            out, _ = df.packed_step(qbuf[layer], packed[layer], blocks[layer], classes, cfg)
            if ev is not None:
                ev[layer][2].record()
            K.prepare_out_projection(out, wo[layer], xs.f32, xs.bf16, D).launch()
            if ev is not None:
                ev[layer][3].record()
        return []

    barrier(ws)
    t, _ = time_steps(step, args.steps, args.warmup)
    t = barrier_max(t, ws)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(L)]
    step(ev)
    torch.cuda.synchronize()
    for e in ev:
        split["qkv"] += e[0].elapsed_time(e[1]) / L
        split["attn"] += e[1].elapsed_time(e[2]) / L
        split["oproj"] += e[2].elapsed_time(e[3]) / L
    # end to end with host buffers: the layer-0 input x comes from pinned host memory each step
    # (the only per-step input once projections run on the device) and the output x goes back
    x_host = torch.randn(HW, Dm, generator=torch.Generator().manual_seed(5)).pin_memory()
    y_host = torch.empty(HW, Dm).pin_memory()
    # Pipelined like a serving loop: the next frame's x is uploaded (copy stream) and the previous
    # step's result downloaded (a second stream) while this step's 30 layers run; device-side
    # staging buffers decouple them from the residual the kernels update in place.
    ms = torch.cuda.current_stream(dev)
    cs_in, cs_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    x_in, y_dev = torch.empty_like(xs.f32), torch.empty_like(xs.f32)
    ev = {k: torch.cuda.Event() for k in ("in_ready", "in_free", "y_ready", "y_free")}
    with torch.cuda.stream(cs_in):
        x_in.copy_(x_host, non_blocking=True)
        ev["in_ready"].record(cs_in)
    ev["y_free"].record(ms)

    def e2e_step():
        ms.wait_event(ev["in_ready"])           # this step's x has arrived
        xs.f32.copy_(x_in)
        xs.bf16.copy_(xs.f32)
        ev["in_free"].record(ms)
        with torch.cuda.stream(cs_in):          # upload the next step's x during this step
            cs_in.wait_event(ev["in_free"])
            x_in.copy_(x_host, non_blocking=True)
            ev["in_ready"].record(cs_in)
        step()
        ms.wait_event(ev["y_free"])             # the previous download is done with y_dev
        y_dev.copy_(xs.f32)
        ev["y_ready"].record(ms)
        with torch.cuda.stream(cs_out):         # download this step's result during the next step
            cs_out.wait_event(ev["y_ready"])
            y_host.copy_(y_dev, non_blocking=True)
            ev["y_free"].record(cs_out)

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ms)
    for _ in range(args.steps):
        e2e_step()
    ms.wait_event(ev["y_free"])                 # the last step's result is on the host
    e1.record(ms)
    torch.cuda.synchronize()
    t_e2e = barrier_max(e0.elapsed_time(e1) / args.steps, ws)
    fq, fo = 2 * HW * 3 * Dm * Dm, 2 * HW * Dm * Dm
    tq, to = split["qkv"] * 1e-3, split["oproj"] * 1e-3
    return {
        "ms_per_step": t, "us_per_layer": t * 1e3 / L,
        "fps": ws * FRAMES_PER_STEP / (DENOISE * t * 1e-3),
        "split_us_per_layer": {k: v * 1e3 for k, v in split.items()},
        "qkv_project": {"kernel": "df_proj_kernel<N,qkv>", "flops": fq, "tflops": fq / tq / 1e12,
                        "frac": fq / tq / 1e12 / bf16_peak,
                        "epilogue": "Q -> FMHA layout, K/V -> pending ring slots (no staging/append copy)"},
        "out_project": {"kernel": "df_proj_kernel<N,out>", "flops": fo, "tflops": fo / to / 1e12,
                        "frac": fo / to / 1e12 / bf16_peak,
                        "epilogue": "x += merge(o) @ W_o (fp32 residual + bf16 copy)"},
        "gpu_launches_per_layer": 3,
        "e2e": {"value": ws * FRAMES_PER_STEP / (DENOISE * t_e2e * 1e-3), "unit": "latent frames/s (full attention "
                "block: QKV + attention + out-projection)", "ms_per_step": t_e2e,
                "h2d_bytes_per_step": HW * Dm * 4, "d2h_bytes_per_step": HW * Dm * 4,
                "path": "pinned host x -> device (next step's x on a copy stream during this step), 30 fused "
                        "layers, x -> pinned host (on a second stream during the next step; the last one inside "
                        "the timed region)"},
        "path": "x -> df_qkv_project -> packed_step (1 FMHA) -> df_out_project, 30 layers per step",
    }


# ------------------------------------------------------------------ CPU leg
def kernel_configs(df, dev, bf16_peak):
    """Single-launch FMHA timings of the other configs SURVEY 8(d) names (CUDA events, median of 10 after
    3 warm-ups, fresh K/V per config): 3d/4s/5n, N(0,3) logits (lazy rescaling is data dependent),
    and the C4 high-resolution frame (HW 18720) packed and all-context."""
    import math

    import torch

    from paper_2601_20499_b200 import kernels as K

    def one(ctxs, hw, q_std=1.0):
        arena = K.KVArena(sum(K.KVArena.region_rows(c) for c in ctxs), D, dev)
        arena.k.normal_()
        arena.v.normal_()
        q = (torch.randn(len(ctxs) * hw, D, device=dev) * q_std).to(torch.bfloat16)
        out = torch.empty(len(ctxs) * hw, D, device=dev, dtype=torch.bfloat16)
        work = [K.HeadWork(arena, arena.allocate(c), c, h, h) for h, c in enumerate(ctxs)]
        launches = K.prepare_attention(q, out, work, hw, 1 / math.sqrt(D))
        for _ in range(3):
            for l in launches:
                l.launch(None)
        # burst conditions for every config: let the clocks recover from the previous (possibly
        # power-capped) measurement, e.g. the 13 hi-res all-context launches before the C5 one
        torch.cuda.synchronize()
        time.sleep(0.5)
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for l in launches:
                l.launch(None)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        us = sorted(ts)[len(ts) // 2] * 1e3
        tf = 4 * D * hw * sum(ctxs) / (us * 1e-6) / 1e12
        del arena, q, out
        torch.cuda.empty_cache()
        return {"us_per_layer": us, "tflops": tf, "frac": tf / bf16_peak}

    hr = 4 * HW
    res = {
        "packed_3d4s5n": one([2 * HW] * 7 + [6 * HW] * 5, HW),
        "packed_6d3s3n_logit_std3": one(PACKED_CTX, HW, 3.0),
        "hires_c4_packed_6d3s3n": one([2 * hr] * 9 + [6 * hr] * 3, hr),
        "hires_c4_all_context": one([7 * hr] * 12, hr),
        # C5 context extension: the budget freed by sink/dummy heads goes to the neighbor heads
        # (kv_cache.py:143-158, 6d/3s/3n: 21 frames per neighbor head), FLOPs equal to all-context
        "context_extension_c5": one([2 * HW] * 9 + [22 * HW] * 3, HW),
    }
    # C5: B independent streams' packed layers in ONE launch (batched_step; 4 arenas, 48 heads)
    B = 4
    arenas = []
    for _ in range(B):
        a = K.KVArena(sum(K.KVArena.region_rows(c) for c in PACKED_CTX), D, dev)
        a.k.normal_()
        a.v.normal_()
        arenas.append(a)
    qb = torch.randn(B * H * HW, D, device=dev).to(torch.bfloat16)
    ob = torch.empty(B * H * HW, D, device=dev, dtype=torch.bfloat16)
    wb = [K.HeadWork(a, a.allocate(c), c, b * H + h, b * H + h) for b, a in enumerate(arenas)
          for h, c in enumerate(PACKED_CTX)]
    lb = K.prepare_attention(qb, ob, wb, HW, 1 / math.sqrt(D))
    for _ in range(3):
        for l in lb:
            l.launch(None)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for l in lb:
            l.launch(None)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    us = sorted(ts)[len(ts) // 2] * 1e3
    tf = B * 4 * D * HW * sum(PACKED_CTX) / (us * 1e-6) / 1e12
    res["streams4_batched_c5"] = {"us_per_layer_all_streams": us, "us_per_layer_per_stream": us / B, "tflops": tf,
                                  "frac": tf / bf16_peak, "launches": len(lb),
                                  "note": "4 independent packed Wan layers (4 arenas, 48 heads) in one FMHA launch"}
    del arenas, qb, ob
    torch.cuda.empty_cache()
    res["hires_c4_speedup_packed_vs_all_context"] = (res["hires_c4_all_context"]["us_per_layer"]
                                                     / res["hires_c4_packed_6d3s3n"]["us_per_layer"])
    res["timing"] = "single launch, CUDA events, median of 10 (burst clocks)"
    return res


def batched_streams(df, cfg, dev, gen, packed, inputs, classes, args, B=4):
    """BASELINE configs[4] at the step level: B independent streams per GPU, each with its own warm packed
    rings and inputs, every layer's B requests in ONE FMHA launch through the public batched_step."""
    import torch

    from paper_2601_20499_b200 import kernels as K

    caches_b, inputs_b = [packed], [inputs]
    pols = [df.derive_policy(df.HeadClass(ASSIGN[i % H]), cfg) for i in range(L * H)]
    for b in range(1, B):
        base, _ = build_caches(df, cfg, dev, gen)
        new = df.rebuild_caches([c for layer in base for c in layer], pols)
        caches_b.append([new[l * H:(l + 1) * H] for l in range(L)])
        inputs_b.append([tuple(torch.randn(H, HW, D, device=dev, generator=gen).to(torch.bfloat16) for _ in range(3))
                         for _ in range(L)])
        del base
        torch.cuda.empty_cache()
    # the streams' Q of a layer back to back in one allocation (as a batched projection would write it):
    # batched_step then launches on it without a gather copy
    q_all = [torch.stack([inputs_b[b][layer][0] for b in range(B)]) for layer in range(L)]

    chain = K.LaunchChain()

    def step():
        for layer in range(L):
            reqs = []
            for b in range(B):
                _, k, v = inputs_b[b][layer]
                q = q_all[layer][b]
                reqs.append(df.StepRequest("packed", q, caches_b[b][layer],
                                           [df.FrameBlock(W, k[h], v[h]) for h in range(H)], classes))
            df.batched_step(reqs, cfg, timed=False, chain=chain)
        return []

    t, _ = time_steps(step, max(3, args.steps // 2), args.warmup)
    res = {"streams": B, "ms_per_step": t, "fps_all_streams": B * FRAMES_PER_STEP / (DENOISE * t * 1e-3),
           "us_per_layer_per_stream": t * 1e3 / L / B,
           "path": "per layer ONE batched_step over the B streams' requests (4 arenas, 48 heads per FMHA launch)"}
    del caches_b, inputs_b, q_all
    torch.cuda.empty_cache()
    return res


def rollout_c3(df, dev, ar_steps=40):
    """BASELINE configs[2]: a whole Wan-shape rollout through the public Session -- fused QKV projection ->
    FMHA -> out-projection per layer, probe with the DHP epilogue at AR step 2 (ratio 0.25), greedy
    classification of 180 of the 360 heads as dummies, one df_kv_pack, then packed attention to the end
    (40 AR steps = 120 latent frames).  Random-init weights of the Wan attention shape, synthetic frames."""
    import torch

    Dm = H * D
    g = torch.Generator(device=dev).manual_seed(11)
    weights = [{n: torch.randn(Dm, Dm, device=dev, generator=g) * (0.5 / Dm ** 0.5) for n in ("q", "k", "v", "o")}
               for _ in range(L)]
    frames = lambda ar, t: torch.randn(HW, Dm, device=dev, generator=g)
    model = df.ProjectedModel(weights, frames, H, D, HW, device=dev)
    cfg = df.SessionConfig(num_layers=L, num_heads=H, head_dim=D, HW=HW, window_len=W, ar_steps=ar_steps,
                           denoise_steps=DENOISE, dummy_count=L * H // 2, probe_ar_step=2, subsample_ratio=0.25)
    def run(graphs):
        sess = df.Session(model, cfg, "packed", device=dev, graphs=graphs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        frames_out, report = sess.run()
        e1.record()
        torch.cuda.synchronize()
        del frames_out
        return sess, report, e0.elapsed_time(e1)

    sess, report, ms = run(False)
    n_dummy = sum(c is df.HeadClass.DUMMY for c in sess.assignment.classes)
    steady = [st["wall_time_ns"] for st in report.steps[W + 1:]]
    res = {"latent_frames": ar_steps * FRAMES_PER_STEP, "ms": ms,
           "fps": ar_steps * FRAMES_PER_STEP / (ms * 1e-3),
           "dummy_heads": n_dummy, "pack_gb": (sess.pack_stats or {}).get("bytes", 0) / 1e9,
           "cache_reduction_ratio": report.cache_reduction_ratio,
           "attn_ms_per_step_steady": sum(steady) / len(steady) / 1e6 if steady else None,
           "path": "Session.run(): per layer df_qkv_project -> df_attn_fwd -> df_out_project; probe (DHP epilogue) + "
                   "classify + df_kv_pack inside the timed region; device-timed (CUDA events)"}
    del sess
    del model, weights
    torch.cuda.empty_cache()
    return res


class CpuLayer:
    """One warm Wan layer for the reference algorithm on the host cores: the oracle
    port of engine.py:87-137 (fp64 numpy / OpenBLAS), all 12 heads, each logical group split into calls
    of <= 4 heads so the softmax matrices stay ~5 GB (the 12-head all-context batch would need ~44 GB).
    Packed: [dummy + sink heads] ctx 2 frames, [neighbor heads] ctx 6 frames (engine.py:192-195);
    baseline: every head ctx 7 frames (engine.py:140-152).  Operands are generated once, outside timing."""

    def __init__(self, mode: str, seed: int = 0):
        import numpy as np

        rng = np.random.default_rng(seed)
        self.ctxs = PACKED_CTX if mode == "packed" else BASE_CTX
        self.q = rng.standard_normal((H, HW, D))
        self.k = [rng.standard_normal((c, D)) for c in self.ctxs]
        self.v = [rng.standard_normal((c, D)) for c in self.ctxs]
        if mode == "packed":
            logical = [[h for h in range(H) if ASSIGN[h] != "neighbor"], [h for h in range(H) if ASSIGN[h] == "neighbor"]]
        else:
            logical = [list(range(H))]
        self.calls = [g[i:i + 4] for g in logical for i in range(0, len(g), 4)]
        self.mode = mode

    def run(self) -> float:
        from oracle import df_oracle as O

        t0 = time.perf_counter()
        O.run_groups(self.q, self.k, self.v, self.calls, D)
        return time.perf_counter() - t0


def cpu_c1_session() -> dict:
    """C1 (BASELINE configs[0]) end to end through the oracle Session restatement (engine.py:268-476):
    the reference's toy model, 2 layers x 4 heads x d64, HW 192, 10 AR steps x 2 denoise, packed."""
    from oracle import df_oracle as O

    cfg = O.Config(num_layers=2, num_heads=4, head_dim=64, HW=192, window_len=6, ar_steps=10, denoise_steps=2,
                   dummy_count=2, probe_ar_step=2, subsample_ratio=0.25)
    toy = O.ToyModel(2, 4, 64, 192, O.derive(42, "toy-model"))
    t0 = time.perf_counter()
    O.run_session(toy, cfg, "packed")
    t = time.perf_counter() - t0
    return {"seconds": t, "latent_frames": 10 * FRAMES_PER_STEP, "fps": 10 * FRAMES_PER_STEP / t,
            "config": "configs[0]: 2 layers x 4 heads x d64, HW 192, W 6, 10 AR steps x 2 denoise, packed, toy model"}


def fps_of_layer(t_layer_s: float) -> float:
    return FRAMES_PER_STEP / (DENOISE * L * t_layer_s)


def cpu_sample(reps: int = 1):
    """cpu_baseline of the GPU arm: one warm packed Wan layer, all 12 heads (the reference algorithm on the
    host cores), extrapolated to 30 layers x 4 denoise iterations."""
    layer = CpuLayer("packed")
    t = min(layer.run() for _ in range(reps))
    return {"value": fps_of_layer(t), "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "extrapolated": True,
            "sample": f"oracle packed attention, all 12 heads of one warm Wan layer in {len(layer.calls)} calls of "
                      f"<= 4 heads (ctx {2 * HW} / {6 * HW}), fp64 numpy/OpenBLAS, {t:.2f} s per layer, "
                      f"extrapolated to 30 layers x 4 denoise",
            "us_per_layer": t * 1e6}


def reference_arm(args, ws, rank):
    """The reference algorithm on the host cores, on the GPU arm's metric: each step times ONE warm packed
    Wan layer (all 12 heads) and the FPS is extrapolated to 30 layers x 4 denoise iterations (marked
    "extrapolated"); ms_per_step is the measured layer.  Beside it, once: the all-context layer (the
    1.8x comparator on CPU) and C1 end to end through the oracle Session.  numpy has no JIT, so at most
    one warm-up layer runs; the timed steps are capped so the run stays within a few minutes."""
    if rank != 0:
        return
    layer = CpuLayer("packed")
    for _ in range(min(args.warmup, 1)):
        layer.run()
    budget_s, t_first = 150.0, layer.run()
    n = max(1, min(args.steps, int(budget_s / max(t_first, 1e-3))))
    times = [t_first] + [layer.run() for _ in range(n - 1)]
    t_layer = statistics.median(times)
    v = fps_of_layer(t_layer)
    base = CpuLayer("baseline", seed=1)
    t_base = base.run()
    del base
    c1 = cpu_c1_session()
    cb = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "extrapolated": True,
          "sample": f"{n} timed warm packed Wan layers (12 heads, 6d/3s/3n, {len(layer.calls)} calls of <= 4 heads), "
                    f"fp64 numpy/OpenBLAS; FPS extrapolated to 30 layers x 4 denoise"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "steps_timed": n,
            "ms_per_step": t_layer * 1e3,
            "step_unit": "one warm Wan layer, all 12 heads, packed (the measured sample; value extrapolates it)",
            "extrapolated": True, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "Wan-2.1-1.3B attention, warm packed 6d/3s/3n, one whole layer per step on host "
                                   "cores", "layers": L, "heads": H, "head_dim": D, "HW": HW, "window": W},
            "baseline_all_context_layer_ms": t_base * 1e3,
            "cpu_speedup_packed_vs_all_context": t_base / t_layer,
            "c1_session_e2e": c1,
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ head-parallel leg (--mode headpar)
def headpar_arm(args, ws, rank, local):
    """BASELINE configs[3]: the high-resolution frame (HW 18720, ~720p-class) with its heads sharded over
    the N GPUs of one box (parallel.HeadParallelSession: H/N heads per rank before classification, LPT
    rebalance after it, the head-output all-gather fused into the FMHA epilogue over NVLink).  One
    rollout of --steps AR steps (probe at step 2, 50% dummies) through the fused projections; device
    time, max over ranks; value = latent frames/s of the one video all ranks produce together."""
    import torch
    import torch.distributed as dist

    import paper_2601_20499_b200 as df
    from paper_2601_20499_b200 import _lib
    from paper_2601_20499_b200.parallel import HeadParallelSession

    dev = torch.device("cuda", local)
    _lib.require_device(local)
    hw = 4 * HW
    ar_steps = max(args.steps, W + 3)
    Dm = H * D
    g = torch.Generator(device=dev).manual_seed(21)  # identical weights and frames on every rank
    weights = [{n: torch.randn(Dm, Dm, device=dev, generator=g) * (0.5 / Dm ** 0.5) for n in ("q", "k", "v", "o")}
               for _ in range(L)]
    fg = torch.Generator(device=dev)

    def frames(ar, t):
        fg.manual_seed(1000 * ar + t)
        return torch.randn(hw, Dm, device=dev, generator=fg)

    model = df.ProjectedModel(weights, frames, H, D, hw, device=dev)
    cfg = df.SessionConfig(num_layers=L, num_heads=H, head_dim=D, HW=hw, window_len=W, ar_steps=ar_steps,
                           denoise_steps=DENOISE, dummy_count=L * H // 2, probe_ar_step=2, subsample_ratio=0.25)
    if ws == 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    sess = HeadParallelSession(model, cfg, "packed", fused_gather=True, device=dev)
    barrier(ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sess.run()
    e1.record()
    torch.cuda.synchronize()
    ms = barrier_max(e0.elapsed_time(e1), ws)
    fps = ar_steps * FRAMES_PER_STEP / (ms * 1e-3)
    line = {"metric": METRIC, "value": fps, "unit": "latent frames/s (one high-resolution video, heads sharded)",
            "n_gpus": ws, "steps": ar_steps, "warmup": 0, "ms_per_step": ms / ar_steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init Wan attention "
            "weights, random frames)",
            "config": {"workload": "configs[3]: Wan-2.1-1.3B attention at HW 18720 (4x tokens/frame), 30 layers x 12 "
                                   "heads x d128, W 6, 50% dummies via DHP, head-parallel with the fused all-gather",
                       "HW": hw, "heads_per_rank_before_rebalance": H // ws, "parallelism": f"head-parallel x{ws}"},
            "rebalance": getattr(sess, "rebalance_stats", None), "gpu_launches": None}
    if rank == 0:
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def gpu_arm(args, ws, rank, local):
    import torch

    import paper_2601_20499_b200 as df
    from paper_2601_20499_b200 import _lib
    from paper_2601_20499_b200 import kernels as K

    dev = torch.device("cuda", local)
    _lib.require_device(local)
    bf16_peak, hbm_peak, peak_kind = peaks()
    cfg = df.SessionConfig(num_layers=L, num_heads=H, head_dim=D, HW=HW, window_len=W, ar_steps=W + 1,
                           denoise_steps=DENOISE, dummy_count=6 * L)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    caches, arena0 = build_caches(df, cfg, dev, gen)
    inputs = [tuple(torch.randn(H, HW, D, device=dev, generator=gen).to(torch.bfloat16) for _ in range(3))
              for _ in range(L)]
    classes = [df.HeadClass(c) for c in ASSIGN]

    # all-context comparator (same kernel, every head baseline-window)
    barrier(ws)
    chain = K.LaunchChain()
    t_base, _ = time_steps(lambda: run_layers(df, cfg, caches, inputs, None, "baseline", timed=False, chain=chain),
                           args.steps, args.warmup)

    # classification-time context packing: one df_kv_pack launch for all 360 heads
    flat = [c for layer in caches for c in layer]
    pols = [df.derive_policy(df.HeadClass(ASSIGN[i % H]), cfg) for i in range(L * H)]
    pack_ms = []
    new = None
    for _ in range(3):
        stats: dict = {}
        new = df.rebuild_caches(flat, pols, stats=stats)
        torch.cuda.synchronize()
        pack_ms.append(stats["events"][0].elapsed_time(stats["events"][1]))
        del stats
    retained = sum(len(c) for c in new)
    pack_bytes = retained * HW * D * 2 * 2 * 2  # frames x (K,V) x (read+write)
    packed = [new[l * H:(l + 1) * H] for l in range(L)]
    del caches, flat
    torch.cuda.empty_cache()

    # the packed hot path (timed region, with clocks sampled during it)
    barrier(ws)
    with ClockSampler(local) as clk:
        # one timed region for the value and the roofline: CUDA events bracket the region, and the
        # FMHA launch of one layer per step (the middle one) is bracketed by its own events for the
        # roofline's launch duration; the other layers carry no per-launch events, which would sit
        # between a layer's FMHA and the next layer's staging copy and break their programmatic-
        # dependent-launch pairing (the copy fills the FMHA's last wave)
        chain = K.LaunchChain()
        sampled = []  # the FMHA of one layer per step carries its own events, a different layer each step

        def packed_step_fn():
            layer = (7 * len(sampled) + L // 2) % L
            sampled.append(layer)
            return run_layers(df, cfg, packed, inputs, classes, "packed", timed=layer, chain=chain)

        t_step, lcs = time_steps(packed_step_fn, args.steps, args.warmup)
    t_step = barrier_max(t_step, ws)
    attn_ns = [step[layer].attn_time_ns for step, layer in zip(lcs, sampled[args.warmup:])]

    # the same step replayed as one CUDA graph (no host work per layer)
    sg = df.StepGraph(packed, cfg, frame_id=W, mode="packed", classes=[classes] * L)
    for layer in range(L):
        for dst, src in zip((sg.q[layer], sg.k[layer], sg.v[layer]), inputs[layer]):
            dst.copy_(src)
    t_graph, _ = time_steps(sg.replay, args.steps, args.warmup)
    t_graph = barrier_max(t_graph, ws)
    del sg
    launches = sum(lc.physical_launches for step in lcs for lc in step)

    fused = full_layer(df, cfg, packed, classes, dev, gen, args, ws, bf16_peak)
    extra = {}
    if ws > 1:
        extra = {"note": "per-GPU config timings are measured in the N=1 run"}
    elif not args.no_configs:
        extra = kernel_configs(df, dev, bf16_peak)
        extra["rollout_c3"] = rollout_c3(df, dev)
        extra["streams4_batched_step_c5"] = batched_streams(df, cfg, dev, gen, packed, inputs, classes, args)

    # e2e through the public API with host buffers
    pinned = [tuple(x.cpu().pin_memory() for x in layer) for layer in inputs]
    outs_host = [torch.empty(H, HW, D, dtype=torch.bfloat16).pin_memory() for _ in range(L)]

    # User-level pipelining around the public API: H2D of layer l+1 on a copy
    # stream and D2H of layer l-1 on another overlap layer l's kernels.
    ms = torch.cuda.current_stream(dev)
    cs, ds = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    stage = [tuple(torch.empty(H, HW, D, dtype=torch.bfloat16, device=dev) for _ in range(3)) for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    for e in freed:
        e.record(ms)

    def e2e_step():
        cs.wait_stream(ms)  # copies of this step start after the timing event
        for layer in range(L):
            buf = stage[layer % 2]
            ready = torch.cuda.Event()
            with torch.cuda.stream(cs):
                cs.wait_event(freed[layer % 2])
                for dst, src in zip(buf, pinned[layer]):
                    dst.copy_(src, non_blocking=True)
                ready.record(cs)
            ms.wait_event(ready)
            q, k, v = buf
            blocks = [df.FrameBlock(W, k[h], v[h]) for h in range(H)]
            out, lc = df.packed_step(q, packed[layer], blocks, classes, cfg)
            done = torch.cuda.Event()
            done.record(ms)
            freed[layer % 2] = done
            with torch.cuda.stream(ds):
                ds.wait_event(done)
                out.record_stream(ds)
                outs_host[layer].copy_(out, non_blocking=True)
        ms.wait_stream(ds)
        return []

    barrier(ws)
    t_e2e, _ = time_steps(e2e_step, max(2, args.steps // 2), 1)
    t_e2e = barrier_max(t_e2e, ws)
    h2d = L * 3 * H * HW * D * 2
    d2h = L * H * HW * D * 2

    flops_packed = layer_flops(PACKED_CTX)
    flops_base = layer_flops(BASE_CTX)
    attn_avg_s = statistics.mean(attn_ns) * 1e-9
    achieved = flops_packed / attn_avg_s / 1e12
    sustained = sustained_peak(bf16_peak)
    fps = ws * FRAMES_PER_STEP / (DENOISE * t_step * 1e-3)
    fps_e2e = ws * FRAMES_PER_STEP / (DENOISE * t_e2e * 1e-3)
    pack_gbs = pack_bytes / (min(pack_ms) * 1e-3) / 1e9

    line = {
        "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random normal Q/K/V, resident in HBM; per-layer K/V 86 MB, 2.6 GB per step > L2)",
        "config": {"workload": "Wan-2.1-1.3B attention (configs[1]): 30 layers x 12 heads x d128, HW 4680 "
                               "(3 x 1560), W 6 warm, packed 6 dummy / 3 sink / 3 neighbor per layer; step = one "
                               "denoise iteration over 30 layers; FPS = 3 latent frames / 4 denoise steps",
                   "layers": L, "heads": H, "head_dim": D, "HW": HW, "window": W, "denoise_steps": DENOISE,
                   "assignment_per_layer": "6d/3s/3n", "l2": "inputs larger than L2 (no flush needed)",
                   "parallelism": f"independent streams x{ws} (no collective)"},
        "us_per_layer": t_step * 1e3 / L,
        "graph_ms_per_step": t_graph,
        "attn_us_per_layer": attn_avg_s * 1e6,
        "tflops": achieved,
        "baseline_all_context": {"ms_per_step": t_base, "us_per_layer": t_base * 1e3 / L,
                                 "tflops_step": flops_base * L / (t_base * 1e-3) / 1e12,
                                 "speedup_packed_vs_all_context": t_base / t_step},
        # the FMHA is timed inside the long 30-layer step (sw_power_cap): the denominator is the
        # SUSTAINED measured bf16 peak (B200_PROFILING.md); the burst-peak fraction is kept beside it
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
                     "frac": achieved / sustained, "traffic": ncu_traffic(),
                     "traffic_unit": f"bytes per launch (dram read+write, {NCU_ATTN})",
                     "algorithmic_bytes": attn_alg_bytes(), "kernel": "df_attn_pair_kernel<false> (cta_group::2)",
                     "flops_per_launch": flops_packed,
                     "peak_source": "measured bf16_tflops_sustained (MEASURED_PEAKS.json; kernel timed inside the "
                                    "30-layer step under sw_power_cap)",
                     "frac_vs_burst": achieved / bf16_peak, "burst_peak": bf16_peak,
                     "sampled_launches": len(attn_ns),
                     "achieved_step": flops_packed * L / (t_step * 1e-3) / 1e12,
                     "achieved_step_note": "30 FMHA launches' FLOPs / the whole step (incl. the 30 staging copies)"},
        "pack_roofline": {"bound": "hbm", "achieved": pack_gbs, "peak": hbm_peak, "unit": "GB/s",
                          "frac": pack_gbs / hbm_peak, "frac_vs_nominal_8tbs": pack_gbs / 8000.0,
                          "bytes": pack_bytes, "ms": min(pack_ms), "kernel": "df_pack_kernel",
                          "traffic": ncu_bytes(NCU_PACK), "traffic_unit": f"dram read+write bytes ({NCU_PACK})"},
        "e2e": {"value": fps_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": t_e2e,
                "path": "public packed_step per layer; pinned host Q/K/V H2D on a copy stream (double-buffered), "
                        "outputs D2H on a second stream, all inside the timed region"},
        "layer_fused": fused,
        "configs": extra,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if ws > 1:  # every rank's clocks during its timed region; the line's clocks are the slowest rank's
        import torch.distributed as dist

        per_rank = [None] * ws
        dist.all_gather_object(per_rank, line["clocks"])
        line["clocks_per_rank"] = per_rank
        line["clocks"] = dict(min(per_rank, key=lambda c: c["sm_mhz"] or 0),
                              reasons=sorted({r for c in per_rank for r in c["reasons"]}))
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_sample(1)
    if rank == 0:
        print(json.dumps(line), flush=True)


def spawn_command(args_argv: list[str], gpus: int, port: int) -> list[str]:
    """torchrun command that re-launches this script with one rank per GPU (``--gpus N`` without a
    launcher around it)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *args_argv]


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs[2..3] / SURVEY 8(d) extra timings")
    ap.add_argument("--mode", default="streams", choices=["streams", "headpar"],
                    help="streams: independent streams per GPU (default, weak scaling); headpar: configs[3], one "
                         "high-resolution video with its heads sharded over the GPUs (strong scaling)")
    ap.add_argument("--rank-check", action="store_true", help=argparse.SUPPRESS)  # test hook: report ranks, exit
    args = ap.parse_args()
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1 and args.impl == "ours":
        # one process per GPU: re-launch under torchrun (NCCL INIT lines on stderr let a reader count ranks)
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        sys.exit(subprocess.call(spawn_command(sys.argv[1:], args.gpus, _free_port()), env=env))
    if ws_env is not None and int(ws_env) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}; launch one rank per GPU")
    if args.rank_check:
        print(json.dumps({"rank": int(os.environ.get("RANK", "0")), "world": int(ws_env or 1)}), flush=True)
        return
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        reference_arm(args, int(ws_env or "1"), rank)
        return
    ws, rank, local = dist_setup()
    if args.mode == "headpar":
        headpar_arm(args, ws, rank, local)
    else:
        gpu_arm(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
