"""Per-layer heterogeneous attention and the AR session driver.

Drop-in for the reference's engine.py (baseline_step / hma_step /
packed_step / expected_step_macs / Session / generate_session).  Every layer
is ONE ragged ``df_attn_fwd`` launch over all heads, whatever the mode: the
mode only decides (a) which cache policies are legal and (b) the *logical*
``kernel_calls`` the reference would have issued (baseline 1, hma up to 3,
packed up to 2; engine.py:134), kept for report parity.  Physical launches are
reported separately.
"""

from __future__ import annotations

import contextlib
import hashlib
import math
import os
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import torch

from . import kernels as K
from .config import SessionConfig
from .errors import AssignmentError, ConfigError, PackingError, ShapeError
from .head_programming import HeadAssignment, HeadClass, greedy_classify
from .kv_cache import (
    CachePolicy,
    FrameBlock,
    HeadKVCache,
    RingStorage,
    as_device_bf16,
    baseline_policy,
    cache_stats,
    derive_policy,
    extension_window,
    launch_segments,
    rebuild_caches,
)
from .layout import FrameLayout
from .profiler import Probe, subsample_rows

MODES = ("baseline", "hma", "packed")
# NVTX ranges per (AR step, denoise iteration, layer) and around classify / pack / append (SURVEY.md 5,
# tracing) for nsys / ncu --nvtx; off unless DF_NVTX=1 (a range push/pop pair costs ~2 us of host time)
NVTX = os.environ.get("DF_NVTX", "0") == "1"


@contextlib.contextmanager
def _nvtx(name: str):
    if not NVTX:
        yield
        return
    torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        torch.cuda.nvtx.range_pop()
_HMA_GROUP_ORDER = (HeadClass.DUMMY, HeadClass.SINK, HeadClass.NEIGHBOR)


class LayerCounters:
    """Counters of one layer call; wall time is device time (CUDA events), resolved lazily."""

    __slots__ = ("kernel_calls", "key_token_macs", "physical_launches", "_events", "_wall", "_attn")

    def __init__(self, kernel_calls: int = 0, key_token_macs: int = 0, physical_launches: int = 0):
        self.kernel_calls = kernel_calls
        self.key_token_macs = key_token_macs
        self.physical_launches = physical_launches
        self._events = None
        self._wall: int | None = 0
        self._attn: int | None = 0

    def _resolve(self) -> None:
        if self._events is not None:
            e0, em, e1 = self._events
            e1.synchronize()
            self._wall = int(round(e0.elapsed_time(e1) * 1e6))
            self._attn = int(round(em.elapsed_time(e1) * 1e6))
            self._events = None

    @property
    def wall_time_ns(self) -> int:
        """Device time of the layer call (current-frame staging + attention)."""
        self._resolve()
        return int(self._wall or 0)

    @property
    def attn_time_ns(self) -> int:
        """Device time of the df_attn_fwd launch alone."""
        self._resolve()
        return int(self._attn or 0)

    @wall_time_ns.setter
    def wall_time_ns(self, v: int) -> None:
        self._events = None
        self._wall = int(v)

    def __repr__(self) -> str:
        return (f"LayerCounters(kernel_calls={self.kernel_calls}, key_token_macs={self.key_token_macs}, "
                f"physical_launches={self.physical_launches})")


@dataclass
class StepCounters:
    """Aggregated counters of one (AR step, denoise iteration)."""

    kernel_calls: list[int] = field(default_factory=list)
    key_token_macs: int = 0
    physical_launches: int = 0
    layers: list[LayerCounters] = field(default_factory=list, repr=False)

    def add_layer(self, lc: LayerCounters) -> None:
        self.kernel_calls.append(lc.kernel_calls)
        self.key_token_macs += lc.key_token_macs
        self.physical_launches += lc.physical_launches
        self.layers.append(lc)

    @property
    def wall_time_ns(self) -> int:
        return sum(lc.wall_time_ns for lc in self.layers)


@dataclass
class StepTrace:
    """Per-layer observation handed to a session observer (engine.py:73-84)."""

    ar_step: int
    denoise_step: int
    layer: int
    q: torch.Tensor
    outputs: torch.Tensor
    classes: list[HeadClass] | None
    contexts: list
    shadow_contexts: list | None


@dataclass
class ProbeRequest:
    """Fused DHP epilogue for one layer launch."""

    row_sampled: torch.Tensor  # uint8 [HW]
    probe_rows: torch.Tensor  # float32 [H, HW, 3]


# ----------------------------------------------------------------- one layer
def _q_rows(q_heads: torch.Tensor, H: int, hw: int, d: int, width: int, device) -> torch.Tensor:
    q = as_device_bf16(q_heads, device)
    if tuple(q.shape) != (H, hw, d):
        raise ShapeError(f"q_heads shape {tuple(q.shape)} != ({H}, {hw}, {d})")
    if d != width:
        q = torch.nn.functional.pad(q, (0, width - d))
    return q.reshape(H * hw, width).contiguous()


@dataclass(frozen=True)
class OutputTarget:
    """Where a layer's outputs land in a head-parallel session with the fused
    all-gather: ``out`` is this rank's bf16 [total_heads * HW, d8] gathered
    buffer, ``heads`` the global index of each local head, ``peers`` device
    pointers of the other ranks' buffers of the same layout; the FMHA epilogue
    stores every output row into all of them (df_attn_args.peer_out)."""

    out: torch.Tensor
    heads: Sequence[int]
    peers: Sequence[int] = ()


def _dispatch(q_heads, caches: list[HeadKVCache], current_blocks: list[FrameBlock], head_dim: int,
              groups: list[list[int]], probe: ProbeRequest | None = None, stream=None, timed: bool = True,
              target: OutputTarget | None = None, chain: K.LaunchChain | None = None,
              workspace: K.Workspace | None = None):
    """Stage current frames, check the logical groups, launch one ragged FMHA."""
    if stream is not None:
        with torch.cuda.stream(stream):
            return _dispatch_on(q_heads, caches, current_blocks, head_dim, groups, probe, stream, timed, target,
                                chain, workspace)
    return _dispatch_on(q_heads, caches, current_blocks, head_dim, groups, probe, None, timed, target, chain,
                        workspace)


def _dispatch_on(q_heads, caches, current_blocks, head_dim, groups, probe, stream, timed, target=None, chain=None,
                 workspace=None):
    H = len(caches)
    if len(current_blocks) != H:
        raise ShapeError(f"{len(current_blocks)} current blocks for {H} caches")
    if H == 0:
        raise ShapeError("no heads")
    hw = current_blocks[0].tokens
    for b in current_blocks:
        if b.tokens != hw:
            raise ShapeError("current blocks of one layer must share HW")
    for c, b in zip(caches, current_blocks):
        c.check_current(b.frame_id)
    n_tok = [c.context_tokens(hw) for c in caches]
    calls = macs = 0
    for g in groups:
        if not g:
            continue
        lens = {n_tok[h] for h in g}
        if len(lens) != 1:
            raise PackingError(f"context lengths {sorted(lens)} differ within one batch")
        calls += 1
        macs += len(g) * hw * n_tok[g[0]] * head_dim
    device = q_heads.device if isinstance(q_heads, torch.Tensor) and q_heads.is_cuda else None
    if device is None:
        st = next((c.storage for c in caches if c.storage is not None), None)
        device = st.arena.device if st is not None else torch.device("cuda", torch.cuda.current_device())
    segs = []
    for c, b in zip(caches, current_blocks):
        segs += c.stage_segments(b, device)
    width = caches[0].storage.arena.width
    q2 = _q_rows(q_heads, H, hw, head_dim, width, device)
    d8 = ((head_dim + 7) // 8) * 8
    if target is None:
        out, o_heads, peers = torch.empty(H * hw, d8, dtype=torch.bfloat16, device=device), list(range(H)), None
    else:
        out, o_heads, peers = target.out, list(target.heads), list(target.peers)
        if len(o_heads) != H or out.dim() != 2 or out.shape[1] != d8 or out.shape[0] % hw:
            raise ShapeError(f"output target {tuple(out.shape)} / {len(o_heads)} heads do not fit {H} x {hw} x {d8}")
    work = [K.HeadWork(c.storage.arena, c.storage.base_row, n_tok[h], h, o_heads[h]) for h, c in enumerate(caches)]
    pb = None
    if probe is not None:
        max_slots = max(c.storage.slots for c in caches)
        tab = np.ones((H, max_slots), dtype=np.uint8)
        for h, c in enumerate(caches):
            tab[h, : c.storage.slots] = c.region_codes()
        # pinned + non_blocking: a pageable upload would wait for every queued launch (one host/device
        # serialisation per probe layer)
        pb = K.ProbeBuffers(torch.from_numpy(tab).pin_memory().to(device, non_blocking=True), probe.row_sampled,
                            probe.probe_rows)
    lc = LayerCounters(kernel_calls=calls, key_token_macs=macs, physical_launches=0)
    s = stream if stream is not None else torch.cuda.current_stream(device)
    # build every launch first so the timed region holds no host work.  Inside a caller's
    # LaunchChain the staging copy may overlap the previous FMHA of the chain (programmatic
    # dependent launch) when the two touch disjoint bytes -- checked when the copy launches
    copies = K.prepare_copies([sg[:6] for sg in segs], overlapped=chain is not None)
    attn = K.prepare_attention(q2, out, work, hw, 1.0 / math.sqrt(head_dim), pb, None, s, peers, workspace)
    if timed:
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(s)
    for launch in copies:
        launch.launch(s, chain)
    if timed:
        ev[1].record(s)
    for launch in attn:
        launch.launch(s, chain)
    if timed:
        ev[2].record(s)
        lc._events = tuple(ev)
    lc.physical_launches = len(copies) + len(attn)
    del segs
    o = out.view(-1, hw, d8)
    if d8 != head_dim:
        o = o[..., :head_dim]
    return o, lc


def baseline_step(q_heads, caches: list[HeadKVCache], current_blocks: list[FrameBlock], config: SessionConfig,
                  *, stream=None, probe: ProbeRequest | None = None, timed: bool = True,
                  target: OutputTarget | None = None, chain: K.LaunchChain | None = None,
                  workspace: K.Workspace | None = None):
    """Full-window attention for every head of one layer (engine.py:140-152).

    Keyword extensions of the reference signature: ``stream``; ``probe`` (fused DHP epilogue);
    ``timed`` (CUDA events -> LayerCounters.wall_time_ns); ``target`` (head-parallel output
    buffer); ``chain`` (kernels.LaunchChain: the caller issues its steps back to back on one
    stream, so the staging copy may overlap the previous FMHA); ``workspace`` (split-KV
    workspace, default the caches' arena's).
    """
    for c in caches:
        if c.policy.kind != "baseline_window":
            raise ConfigError(f"baseline_step got a {c.policy.kind} cache")
    return _dispatch(q_heads, caches, current_blocks, config.head_dim, [list(range(len(caches)))], probe, stream,
                     timed, target, chain, workspace)


def _class_groups(classes: list[HeadClass]) -> list[list[int]]:
    return [[h for h, c in enumerate(classes) if c is want] for want in _HMA_GROUP_ORDER]


def hma_step(q_heads, caches, current_blocks, classes: list[HeadClass], config: SessionConfig, *, stream=None,
             probe: ProbeRequest | None = None, timed: bool = True, target: OutputTarget | None = None,
             chain: K.LaunchChain | None = None, workspace: K.Workspace | None = None):
    """Class-specific contexts; logically one call per class present (engine.py:161-174)."""
    if len(classes) != len(caches):
        raise AssignmentError(f"{len(classes)} classes for {len(caches)} heads in this layer")
    return _dispatch(q_heads, caches, current_blocks, config.head_dim, _class_groups(list(classes)), probe, stream,
                     timed, target, chain, workspace)


def packed_step(q_heads, caches, current_blocks, classes: list[HeadClass], config: SessionConfig, *, stream=None,
                probe: ProbeRequest | None = None, timed: bool = True, target: OutputTarget | None = None,
                chain: K.LaunchChain | None = None, workspace: K.Workspace | None = None):
    """Dummy+sink share one logical call, neighbors the other (engine.py:177-195)."""
    if not config.packing_enabled:
        raise ConfigError("packed_step requires packing_enabled")
    if len(classes) != len(caches):
        raise AssignmentError(f"{len(classes)} classes for {len(caches)} heads in this layer")
    ds = [h for h, c in enumerate(classes) if c is not HeadClass.NEIGHBOR]
    nb = [h for h, c in enumerate(classes) if c is HeadClass.NEIGHBOR]
    return _dispatch(q_heads, caches, current_blocks, config.head_dim, [ds, nb], probe, stream, timed, target, chain,
                     workspace)


@dataclass
class StepRequest:
    """One session's layer for ``batched_step``: the arguments of baseline_step / hma_step / packed_step."""

    mode: str
    q_heads: object
    caches: list
    current_blocks: list
    classes: list | None = None


def _request_groups(r: StepRequest, config: SessionConfig) -> list[list[int]]:
    """The logical calls of one request, with the checks of the matching step function."""
    if r.mode == "baseline":
        for c in r.caches:
            if c.policy.kind != "baseline_window":
                raise ConfigError(f"baseline_step got a {c.policy.kind} cache")
        return [list(range(len(r.caches)))]
    if r.mode not in ("hma", "packed"):
        raise ConfigError(f"unknown mode {r.mode!r}, expected one of {MODES}")
    classes = list(r.classes or [])
    if len(classes) != len(r.caches):
        raise AssignmentError(f"{len(classes)} classes for {len(r.caches)} heads in this layer")
    if r.mode == "hma":
        return _class_groups(classes)
    if not config.packing_enabled:
        raise ConfigError("packed_step requires packing_enabled")
    return [[h for h, c in enumerate(classes) if c is not HeadClass.NEIGHBOR],
            [h for h, c in enumerate(classes) if c is HeadClass.NEIGHBOR]]


def _adjacent_rows(qs: list[torch.Tensor]) -> torch.Tensor | None:
    """One [sum rows, width] view over row blocks that sit back to back in memory (e.g. the streams'
    Q as slices of one batched tensor), else None."""
    q0 = qs[0]
    nxt = q0.data_ptr()
    for q in qs:
        if not q.is_contiguous() or q.data_ptr() != nxt or q.dtype != q0.dtype or q.shape[1] != q0.shape[1]:
            return None
        nxt += q.numel() * q.element_size()
    rows = sum(q.shape[0] for q in qs)
    end = q0.storage_offset() + rows * q0.shape[1]
    if end > q0.untyped_storage().nbytes() // q0.element_size():
        return None
    return q0.as_strided((rows, q0.shape[1]), (q0.shape[1], 1))


def batched_step(requests: Sequence[StepRequest], config: SessionConfig, *, stream=None, timed: bool = True,
                 chain: K.LaunchChain | None = None, workspace: K.Workspace | None = None):
    """Several independent sessions' layers (SURVEY 8(e) / BASELINE configs[4]: a batch of video streams
    on one GPU) in ONE ragged FMHA launch (more launches only past DF_MAX_HEADS heads or DF_MAX_ARENAS
    arenas).  Each request keeps its own logical calls, MAC counters and errors; the batch fills the
    SMs' last wave that a single stream's layer leaves partly idle.  Returns [(outputs, LayerCounters)]
    in request order; the outputs are views of one batched buffer.
    """
    if not requests:
        raise ShapeError("no requests")
    groups = [_request_groups(r, config) for r in requests]
    d = config.head_dim
    hw = requests[0].current_blocks[0].tokens if requests[0].current_blocks else config.HW
    device = None
    for r in requests:
        if len(r.current_blocks) != len(r.caches) or not r.caches:
            raise ShapeError(f"{len(r.current_blocks)} current blocks for {len(r.caches)} caches")
        for c, b in zip(r.caches, r.current_blocks):
            if b.tokens != hw:
                raise ShapeError("current blocks of one batch must share HW")
            c.check_current(b.frame_id)
        if device is None and isinstance(r.q_heads, torch.Tensor) and r.q_heads.is_cuda:
            device = r.q_heads.device
    if device is None:
        device = requests[0].caches[0].storage.arena.device
    width = requests[0].caches[0].storage.arena.width
    d8 = ((d + 7) // 8) * 8
    s = stream if stream is not None else torch.cuda.current_stream(device)
    ctx = torch.cuda.stream(stream) if stream is not None else None
    if ctx is not None:
        ctx.__enter__()
    try:
        counters, segs, work, qs = [], [], [], []
        base = 0
        for r, g in zip(requests, groups):
            n_tok = [c.context_tokens(hw) for c in r.caches]
            calls = macs = 0
            for grp in g:
                if not grp:
                    continue
                lens = {n_tok[h] for h in grp}
                if len(lens) != 1:
                    raise PackingError(f"context lengths {sorted(lens)} differ within one batch")
                calls += 1
                macs += len(grp) * hw * n_tok[grp[0]] * d
            counters.append(LayerCounters(kernel_calls=calls, key_token_macs=macs, physical_launches=0))
            for c, b in zip(r.caches, r.current_blocks):
                segs += c.stage_segments(b, device)
            qs.append(_q_rows(r.q_heads, len(r.caches), hw, d, width, device))
            work += [K.HeadWork(c.storage.arena, c.storage.base_row, n_tok[h], base + h, base + h)
                     for h, c in enumerate(r.caches)]
            base += len(r.caches)
        q2 = _adjacent_rows(qs) if len(qs) > 1 else qs[0]
        if q2 is None:  # requests' Q not laid out back to back in one allocation: gather them
            q2 = torch.cat(qs, 0)
        out = torch.empty(base * hw, d8, dtype=torch.bfloat16, device=device)
        copies = K.prepare_copies([sg[:6] for sg in segs], overlapped=chain is not None)
        attn = K.prepare_attention(q2, out, work, hw, 1.0 / math.sqrt(d), None, None, s, workspace=workspace)
        if timed:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(s)
        for launch in copies:
            launch.launch(s, chain)
        if timed:
            ev[1].record(s)
        for launch in attn:
            launch.launch(s, chain)
        if timed:
            ev[2].record(s)
        del segs
    finally:
        if ctx is not None:
            ctx.__exit__(None, None, None)
    o = out.view(base, hw, d8)
    if d8 != d:
        o = o[..., :d]
    res, h0 = [], 0
    for r, lc in zip(requests, counters):
        lc.physical_launches = len(copies) + len(attn)
        if timed:
            lc._events = tuple(ev)
        res.append((o[h0:h0 + len(r.caches)], lc))
        h0 += len(r.caches)
    return res


def expected_step_macs(config: SessionConfig, mode: str, history_frames: int,
                       assignment: HeadAssignment | None = None) -> int:
    """Closed-form key-token MACs of one denoise iteration (engine.py:198-237)."""
    if mode not in MODES:
        raise ConfigError(f"unknown mode {mode!r}")
    ext = extension_window(assignment, config) if (assignment is not None and config.context_extension) else None

    def past(p: CachePolicy) -> int:
        h = history_frames
        if h == 0:
            return 0
        sink_seen = p.sink_frame < h
        if p.kind == "baseline_window":
            return min(h - 1 if sink_seen else h, p.window_len - 1) + (1 if sink_seen else 0)
        if p.kind == "sink_only":
            return 1 if sink_seen else 0
        return min(h, p.recent_capacity)

    if mode == "baseline" or assignment is None:
        ctxs = [(past(baseline_policy(config)) + 1) * config.HW] * config.total_heads
    else:
        ctxs = [(past(derive_policy(c, config, extended_window=ext)) + 1) * config.HW for c in assignment.classes]
    return sum(config.HW * c * config.head_dim for c in ctxs)


# ------------------------------------------------------------------- session
@dataclass
class RunReport:
    mode: str
    config: dict
    cache_reduction_ratio: float
    assignment: dict | None
    steps: list[dict]
    kernel_calls_steady: list[int]
    total_key_token_macs: int
    total_wall_time_ns: int
    physical_launches_steady: list[int] = field(default_factory=list)
    frames: list = field(default_factory=list, repr=False, compare=False)
    _digest: str | None = field(default=None, repr=False, compare=False)

    @property
    def output_digest(self) -> str:
        """sha256 over the step outputs (engine.py report digest), computed on first access: it
        reads every frame back to the host, which a rollout's timing should not include."""
        if self._digest is None:
            self._digest = _digest(self.frames)
        return self._digest

    def to_dict(self) -> dict:
        return {
            "mode": self.mode,
            "config": self.config,
            "cache_reduction_ratio": self.cache_reduction_ratio,
            "assignment": self.assignment,
            "steps": self.steps,
            "kernel_calls_steady": self.kernel_calls_steady,
            "total_key_token_macs": self.total_key_token_macs,
            "total_wall_time_ns": self.total_wall_time_ns,
            "output_digest": self.output_digest,
            "physical_launches_steady": self.physical_launches_steady,
        }


def _digest(frames) -> str:
    h = hashlib.sha256()
    for x in frames:
        if x is None:
            continue
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
        t = t.detach().contiguous().cpu()
        h.update(str(tuple(t.shape)).encode())
        h.update(t.view(torch.uint8).numpy().tobytes() if t.dtype != torch.bool else t.numpy().tobytes())
    return h.hexdigest()


class Session:
    """One generation run on the device (engine.py:268-576).

    The model protocol is the reference's: ``frame_input(ar, t)``,
    ``qkv(layer, x, ar, t) -> (q, k, v)`` each (heads, HW, head_dim) (torch
    CUDA tensors preferred; host arrays are uploaded), and ``mix(layer,
    outputs)`` whose result is added to ``x`` (None = open loop).
    """

    def __init__(self, model, config: SessionConfig, mode: str = "baseline",
                 observer: Callable[[StepTrace], None] | None = None, shadow: bool = False,
                 device: torch.device | str | None = None, stream: torch.cuda.Stream | None = None,
                 graphs: bool = False):
        if mode not in MODES:
            raise ConfigError(f"unknown mode {mode!r}, expected one of {MODES}")
        if mode == "packed" and not config.packing_enabled:
            raise ConfigError("packed mode requires packing_enabled")
        if mode == "packed" and config.merged_window is not None:
            raise ConfigError("merged_window gives sink heads a context longer than packed "
                              "dummy heads; packing requires the plain sink policy")
        self.model = model
        self.config = config
        self.mode = mode
        # heads this process owns ([h0, h1) of every layer); head-parallel
        # subclasses narrow it and override the three collective hooks below.
        self.head_range = self._owned_heads()
        # heads of every layer this process runs, ascending (head_range until a
        # head-parallel rebalance gives each layer its own set)
        self.layer_heads: list[list[int]] = [list(self.head_range) for _ in range(config.num_layers)]
        self.observer = observer
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream
        self.assignment: HeadAssignment | None = None
        self.objective: float | None = None
        self.pack_stats: dict | None = None
        self._next_step = 0
        self._frames: list = []
        self._step_counters: list[tuple[int, list[StepCounters]]] = []
        self._kernel_calls_last: list[int] = []
        self._phys_last: list[int] = []
        self._probe_requests: dict[tuple[int, int], set[float]] = {}
        self._probe_tables: dict[tuple[int, int, float], np.ndarray] = {}
        self._row_flags: dict[float, torch.Tensor] = {}
        self._classify_at: tuple[int, int] | None = None
        if mode != "baseline" and config.dummy_count > 0 and config.probe_ar_step < config.ar_steps:
            self._classify_at = self._probe_key(None)
            self._probe_requests.setdefault(self._classify_at, set()).add(config.subsample_ratio)
        self.caches = self._fresh_caches()
        self._shadow = shadow and mode != "baseline"
        self.shadow_caches = self._fresh_caches() if self._shadow else None
        # CUDA-graph replay of whole denoise iterations: one graph per cache
        # signature (pending slots + context lengths), captured on first use, all sharing one pool
        self.graphs = graphs
        self._graph_cache: dict[tuple, tuple] = {}
        self._graph_pool = None
        self._capture_stream: torch.cuda.Stream | None = None
        self.graph_stats = {"captured": 0, "replayed": 0}

    def _owned_heads(self) -> range:
        return range(self.config.num_heads)

    # collective hooks (identity on one process; see parallel.HeadParallelSession)
    def _gather_outputs(self, layer: int, outputs: torch.Tensor) -> torch.Tensor:
        """Local heads' outputs (h_local, HW, d) -> all heads, for ``mix``."""
        return outputs

    def _gather_scores(self, local: torch.Tensor) -> torch.Tensor:
        """(layers, h_local, 3) probe scores -> (layers, heads, 3) on every process."""
        return local

    def _after_step(self, ar_step: int) -> None:
        """Hook after a step's cache appends (head-parallel rebalancing)."""

    def _fresh_caches(self) -> list[list[HeadKVCache]]:
        cfg = self.config
        pol = baseline_policy(cfg)
        per = K.KVArena.region_rows(pol.ring_slots * cfg.HW)
        nh = len(self.head_range)
        arena = K.KVArena(per * cfg.num_layers * nh, K.padded_width(cfg.head_dim), self.device)
        return [[HeadKVCache(pol, storage=RingStorage(arena, arena.allocate(pol.ring_slots * cfg.HW), pol.ring_slots,
                                                      cfg.HW, cfg.head_dim))
                 for _ in range(nh)] for _ in range(cfg.num_layers)]

    # ------------------------------------------------------------ probe
    def _probe_key(self, probe: Probe | None) -> tuple[int, int]:
        if probe is None:
            probe = Probe(self.config.probe_ar_step, self.config.probe_denoise_step)
        dn = probe.denoise_step if probe.denoise_step is not None else self.config.denoise_steps - 1
        if not 0 <= dn < self.config.denoise_steps:
            raise ConfigError(f"probe denoise step {dn} out of range")
        if not 0 <= probe.ar_step < self.config.ar_steps:
            raise ConfigError(f"probe AR step {probe.ar_step} out of range")
        return probe.ar_step, dn

    def probe_scores(self, probe: Probe | None = None, subsample_ratio: float | None = None) -> np.ndarray:
        """(total_heads, 3) region scores at the probe (runs forward if needed)."""
        ratio = self.config.subsample_ratio if subsample_ratio is None else subsample_ratio
        subsample_rows(self.config.HW, ratio)  # validates (ConfigError)
        key = self._probe_key(probe)
        if (key[0], key[1], ratio) not in self._probe_tables:
            if self._next_step > key[0]:
                raise ConfigError(f"session already advanced past AR step {key[0]}")
            if self._classify_at is not None and key[0] > self._classify_at[0]:
                raise ConfigError("probe lies beyond the classification step of this session")
            self._probe_requests.setdefault(key, set()).add(ratio)
            while self._next_step <= key[0]:
                self._run_step(self._next_step)
        return self._probe_tables[(key[0], key[1], ratio)]

    # ------------------------------------------------------------ stepping
    def _effective_mode(self) -> str:
        return "baseline" if (self.mode == "baseline" or self.assignment is None) else self.mode

    def _classes_for_layer(self, layer: int) -> list[HeadClass]:
        h = self.config.num_heads
        return [self.assignment.classes[layer * h + i] for i in self.layer_heads[layer]]

    def _output_target(self, layer: int) -> OutputTarget | None:
        """Hook: where the layer's outputs land (head-parallel fused gather); None = a fresh tensor."""
        return None

    def _layer_attention(self, layer, q, caches, current_blocks, probe=None, timed: bool = True):
        mode = self._effective_mode()
        tgt = self._output_target(layer) if probe is None else None
        kw = dict(stream=self.stream, probe=probe, target=tgt, timed=timed)
        if mode == "baseline":
            return baseline_step(q, caches, current_blocks, self.config, **kw)
        classes = self._classes_for_layer(layer)
        if mode == "hma":
            return hma_step(q, caches, current_blocks, classes, self.config, **kw)
        return packed_step(q, caches, current_blocks, classes, self.config, **kw)

    # ------------------------------------------------------------ CUDA graphs
    def _graphable(self, ratios) -> bool:
        """A denoise iteration can be captured: projected model (device-only, in-place residual),
        no probe epilogue, no per-layer observer or shadow caches."""
        return (self.graphs and not ratios and self.observer is None and self.shadow_caches is None
                and hasattr(self.model, "qkv_into") and hasattr(self.model, "mix_into"))

    def _layers(self, x, ar_step: int, t: int, timed: bool):
        """One denoise iteration over every layer; returns (x, blocks per layer, counters)."""
        counters = StepCounters()
        blocks_all = []
        for layer in range(self.config.num_layers):
            q, blocks = self._project(layer, x, ar_step, t)
            outputs, lc = self._layer_attention(layer, q, self.caches[layer], blocks, None, timed)
            counters.add_layer(lc)
            blocks_all.append(blocks)
            x = self._mix(layer, outputs, x)
        return x, blocks_all, counters

    def _graph_iteration(self, x_in, ar_step: int, t: int):
        """Replay (capturing on first use) the iteration graph of the current cache signature.

        The graph is a function of the slot tables only: every denoise iteration of an AR step, and
        every AR step whose pending slots repeat (the ring cycles), replays the same one.  ``x_in``
        is copied into the graph's static residual buffers; the result lands there in place.
        """
        HW = self.config.HW
        key = (self._effective_mode(), id(self.caches),
               tuple((c.pending_slot, c.context_tokens(HW)) for row in self.caches for c in row))
        entry = self._graph_cache.get(key)
        s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        if entry is None:
            if self._capture_stream is None:
                self._capture_stream = torch.cuda.Stream(self.device)
                self._graph_pool = torch.cuda.graph_pool_handle()
            cs = self._capture_stream
            x_static = type(x_in)(x_in.f32.clone(), x_in.bf16.clone())
            cs.wait_stream(s)
            saved, self.stream = self.stream, cs
            try:
                with torch.cuda.stream(cs):  # eager warm-up on the capture stream: its split workspace, error paths
                    x_out, blocks_all, counters = self._layers(x_static, ar_step, t, timed=False)
                s.wait_stream(cs)
                g = torch.cuda.CUDAGraph()
                x_cap = type(x_in)(x_in.f32.clone(), x_in.bf16.clone())
                with torch.cuda.graph(g, stream=cs, pool=self._graph_pool, capture_error_mode="thread_local"):
                    self._layers(x_cap, ar_step, t, timed=False)
            finally:
                self.stream = saved
            self._graph_cache[key] = (g, x_cap, blocks_all, counters)
            self.graph_stats["captured"] += 1
            return x_out, blocks_all, counters
        g, x_cap, blocks_all, counters = entry
        with torch.cuda.stream(s):
            x_cap.f32.copy_(x_in.f32)
            x_cap.bf16.copy_(x_in.bf16)
            g.replay()
        self.graph_stats["replayed"] += 1
        return x_cap, blocks_all, counters

    def _classify(self) -> None:
        cfg = self.config
        key = self._classify_at
        table = self._probe_tables[(key[0], key[1], cfg.subsample_ratio)]
        self.assignment, self.objective = greedy_classify(table, cfg.dummy_count)
        ext = extension_window(self.assignment, cfg) if cfg.context_extension else None
        flat_caches = [c for layer in self.caches for c in layer]
        policies = [derive_policy(c, cfg, extended_window=ext)
                    for layer in range(cfg.num_layers) for c in self._classes_for_layer(layer)]
        rows = sum(K.KVArena.region_rows(p.ring_slots * cfg.HW) for p in policies)
        arena = K.KVArena(rows, K.padded_width(cfg.head_dim), self.device)
        s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        stats: dict = {}
        new = rebuild_caches(flat_caches, policies, arena, stream=s, stats=stats)
        self.pack_stats = stats
        H = len(self.head_range)
        self.caches = [new[l * H : (l + 1) * H] for l in range(cfg.num_layers)]

    def _probe_buffers(self, ratio: float) -> ProbeRequest:
        cfg = self.config
        flags = self._row_flags.get(ratio)
        if flags is None:  # once per ratio (a pageable upload per layer would serialise host and device)
            rows = subsample_rows(cfg.HW, ratio)
            host = torch.zeros(cfg.HW, dtype=torch.uint8)
            host[torch.from_numpy(rows)] = 1
            flags = self._row_flags[ratio] = host.to(self.device)
        return ProbeRequest(flags, torch.zeros(len(self.head_range), cfg.HW, 3, dtype=torch.float32, device=self.device))

    def _finalize_probe(self, key, ratio, per_layer: list[ProbeRequest]) -> None:
        tables = []
        for pr in per_layer:
            F = K.scores_finalize(K.ProbeBuffers(None, pr.row_sampled, pr.probe_rows), self.stream)
            tables.append(F)
        full = self._gather_scores(torch.stack(tables))  # (layers, heads, 3), layer-major flat order
        self._probe_tables[(key[0], key[1], ratio)] = full.reshape(-1, 3).cpu().numpy()

    def _model_qkv(self, layer, x, ar, t):
        q, k, v = self.model.qkv(layer, x, ar, t)
        heads = self.layer_heads[layer]
        if len(heads) != self.config.num_heads:
            if heads == list(range(heads[0], heads[-1] + 1)):
                q, k, v = q[heads[0] : heads[-1] + 1], k[heads[0] : heads[-1] + 1], v[heads[0] : heads[-1] + 1]
            else:
                q, k, v = q[heads], k[heads], v[heads]
        return as_device_bf16(q, self.device), as_device_bf16(k, self.device), as_device_bf16(v, self.device)

    def _project(self, layer, x, ar, t):
        """(q, current blocks) of one layer.

        A model with ``qkv_into`` (projection.ProjectedModel) writes K/V of the
        current frame straight into the pending ring slots (df_qkv_project), so
        the blocks are views of the ring and staging/append move nothing.
        """
        into = getattr(self.model, "qkv_into", None)
        if into is None:
            q, k, v = self._model_qkv(layer, x, ar, t)
            return q, [FrameBlock(ar, k[h], v[h]) for h in range(k.shape[0])]
        cfg = self.config
        caches = self.caches[layer]
        views = [c.pending_view(cfg.HW, cfg.head_dim, self.device) for c in caches]
        q = torch.empty(len(caches), cfg.HW, cfg.head_dim, dtype=torch.bfloat16, device=self.device)
        into(layer, x, ar, t, q, [kv[0] for kv in views], [kv[1] for kv in views], heads=self.layer_heads[layer],
             stream=self.stream)
        return q, [FrameBlock(ar, k, v) for k, v in views]

    def _mix(self, layer, outputs, x):
        """engine.py:443: x = x + mix(outputs); fused in-place for models with ``mix_into``."""
        gathered = self._gather_outputs(layer, outputs)
        into = getattr(self.model, "mix_into", None)
        if into is not None:
            return into(layer, gathered, x, stream=self.stream)
        m = self.model.mix(layer, gathered)
        if m is None:
            return x
        return m if x is None else x + m

    def _run_step(self, ar_step: int) -> None:
        with _nvtx(f"ar{ar_step}"):
            self._run_step_ranged(ar_step)

    def _run_step_ranged(self, ar_step: int) -> None:
        cfg = self.config
        final_kv = []
        step_counters: list[StepCounters] = []
        x = None
        graphed = False
        for t in range(cfg.denoise_steps):
            x = self.model.frame_input(ar_step, t)
            final = t == cfg.denoise_steps - 1
            ratios = sorted(self._probe_requests.get((ar_step, t), ()))
            if self._graphable(ratios):
                with _nvtx(f"ar{ar_step}/denoise{t}/graph"):
                    x, blocks_all, counters = self._graph_iteration(x, ar_step, t)
                graphed = True
                if final:  # the views are the pending ring slots; the frame id is this step's
                    final_kv = [[FrameBlock(ar_step, b.keys, b.values) for b in row] for row in blocks_all]
                step_counters.append(counters)
                continue
            graphed = False
            probes: dict[float, list[ProbeRequest]] = {r: [] for r in ratios}
            counters = StepCounters()
            for layer in range(cfg.num_layers):
                with _nvtx(f"ar{ar_step}/denoise{t}/layer{layer}"):
                    q, blocks = self._project(layer, x, ar_step, t)
                    pr = None
                    if ratios:
                        pr = self._probe_buffers(ratios[0])
                        probes[ratios[0]].append(pr)
                    outputs, lc = self._layer_attention(layer, q, self.caches[layer], blocks, pr)
                    for extra in ratios[1:]:  # another ratio at the same key: re-run the probe epilogue
                        pe = self._probe_buffers(extra)
                        probes[extra].append(pe)
                        self._layer_attention(layer, q, self.caches[layer], blocks, pe)
                    counters.add_layer(lc)
                    if self.observer is not None:
                        self._notify(ar_step, t, layer, q, outputs, blocks)
                    if final:
                        final_kv.append(blocks)
                    x = self._mix(layer, outputs, x)
            for r in ratios:
                self._finalize_probe((ar_step, t), r, probes[r])
            step_counters.append(counters)
        if self._classify_at is not None and self.assignment is None and ar_step == self._classify_at[0]:
            with _nvtx(f"ar{ar_step}/classify+pack"):
                self._classify()
        s = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        segs = []
        for layer in range(cfg.num_layers):
            for h, block in enumerate(final_kv[layer]):
                segs += self.caches[layer][h].append_segments(block, self.device)
                if self.shadow_caches is not None:
                    segs += self.shadow_caches[layer][h].append_segments(block, self.device)
        if segs:
            with _nvtx(f"ar{ar_step}/append"):
                launch_segments(segs, s)
        self._after_step(ar_step)
        frame = getattr(x, "f32", x)
        self._frames.append(frame.clone() if graphed else frame)  # graph buffers are reused by the next replay
        self._step_counters.append((ar_step, step_counters))
        self._kernel_calls_last = list(step_counters[-1].kernel_calls)
        self._phys_last = [lc.physical_launches for lc in step_counters[-1].layers]
        self._next_step = ar_step + 1

    def _notify(self, ar_step, t, layer, q, outputs, blocks) -> None:
        contexts = []
        for c, b in zip(self.caches[layer], blocks):
            keys, values, lay = c.gather_context(b)
            contexts.append((keys, values, lay, c.frame_ids + [b.frame_id]))
        shadow = None
        if self.shadow_caches is not None:
            shadow = []
            for c, b in zip(self.shadow_caches[layer], blocks):
                keys, values, _ = c.gather_context(b)
                shadow.append((keys, values, c.frame_ids + [ar_step]))
        classes = self._classes_for_layer(layer) if self._effective_mode() != "baseline" else None
        self.observer(StepTrace(ar_step, t, layer, q, outputs, classes, contexts, shadow))

    def run(self):
        while self._next_step < self.config.ar_steps:
            self._run_step(self._next_step)
        return self._frames, self._report()

    def time_step(self, reps: int = 5) -> dict:
        """Re-dispatch the next step's final denoise iteration ``reps`` times (engine.py:511-550).

        Device-timed (CUDA events); the session does not advance.
        """
        if reps < 1:
            raise ConfigError("reps must be >= 1")
        cfg = self.config
        ar_step = self._next_step
        t = cfg.denoise_steps - 1
        walls = []
        counters = StepCounters()
        for _ in range(reps):
            counters = StepCounters()
            x = self.model.frame_input(ar_step, t)
            for layer in range(cfg.num_layers):
                q, blocks = self._project(layer, x, ar_step, t)
                outputs, lc = self._layer_attention(layer, q, self.caches[layer], blocks)
                counters.add_layer(lc)
                x = self._mix(layer, outputs, x)
            walls.append(counters.wall_time_ns)
        walls.sort()
        mid = len(walls) // 2
        median = walls[mid] if len(walls) % 2 else (walls[mid - 1] + walls[mid]) // 2
        return {"wall_time_ns_median": int(median), "key_token_macs": counters.key_token_macs,
                "kernel_calls_per_layer": counters.kernel_calls,
                "physical_launches_per_layer": [lc.physical_launches for lc in counters.layers]}

    def _report(self) -> RunReport:
        cfg = self.config
        if self.assignment is not None:
            ratio = cache_stats(self.assignment, cfg).reduction_ratio
            assignment = {
                "n_dummy": self.assignment.dummy_count,
                "objective": self.objective,
                "counts": self.assignment.counts(),
                "per_layer": self.assignment.per_layer_histogram(cfg.num_heads),
                "heads": self.assignment.to_records(cfg.num_heads),
            }
        else:
            ratio, assignment = 1.0, None
        steps = []
        for ar, scs in self._step_counters:
            steps.append({
                "ar_step": ar,
                "key_token_macs": sum(sc.key_token_macs for sc in scs),
                "kernel_calls_per_layer": list(scs[-1].kernel_calls),
                "wall_time_ns": sum(sc.wall_time_ns for sc in scs),
                "layer_wall_time_ns": [lc.wall_time_ns for sc in scs for lc in sc.layers],
            })
        return RunReport(
            mode=self.mode,
            config=cfg.to_dict(),
            cache_reduction_ratio=ratio,
            assignment=assignment,
            steps=steps,
            kernel_calls_steady=self._kernel_calls_last,
            total_key_token_macs=sum(s["key_token_macs"] for s in steps),
            total_wall_time_ns=sum(s["wall_time_ns"] for s in steps),
            frames=list(self._frames),
            physical_launches_steady=self._phys_last,
        )


class StepGraph:
    """One denoise iteration over every layer, captured once as a CUDA graph.

    SURVEY.md 8(f) row 3 (Session._run_step / time_step, engine.py:407-550):
    the per-layer Python dispatch (staging copy + ragged FMHA launch) is
    recorded for a fixed cache state and replayed with no host work.  Inputs
    are the static device buffers ``q[l]``, ``k[l]``, ``v[l]`` (heads, HW, d)
    -- copy the iteration's projections into them (or have the producer
    write there) and call :meth:`replay`; ``outputs[l]`` hold the results.
    A graph stays valid while the caches' slot tables do not change, i.e.
    for every denoise iteration of one AR step (the cache is appended only
    after the final iteration, engine.py:457-463).
    """

    def __init__(self, caches: list[list[HeadKVCache]], config: SessionConfig, frame_id: int, mode: str = "baseline",
                 classes: list[list[HeadClass]] | None = None, device=None):
        if mode not in MODES:
            raise ConfigError(f"unknown mode {mode!r}")
        self.config = config
        self.caches = caches
        self.mode = mode
        self.classes = classes
        self.frame_id = frame_id
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        cfg = config
        H = len(caches[0])
        shape = (H, cfg.HW, cfg.head_dim)
        self.q = [torch.zeros(shape, dtype=torch.bfloat16, device=dev) for _ in caches]
        self.k = [torch.zeros(shape, dtype=torch.bfloat16, device=dev) for _ in caches]
        self.v = [torch.zeros(shape, dtype=torch.bfloat16, device=dev) for _ in caches]
        self.outputs: list[torch.Tensor] = []
        # the graph's own split workspace (eager launches on the caches' arena never share its counters)
        self.workspace = K.Workspace(dev)
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            self._launch_all()  # eager warm-up: allocates the stream's workspace, checks every error path
        torch.cuda.current_stream(dev).wait_stream(side)
        with torch.cuda.graph(self.graph, stream=side, capture_error_mode="thread_local"):
            self.outputs = self._launch_all()
        self.kernel_launches = 2 * len(caches)

    def _launch_all(self) -> list[torch.Tensor]:
        outs = []
        chain = K.LaunchChain()  # every launch of the iteration is the library's own, back to back
        kw = dict(timed=False, chain=chain, workspace=self.workspace)
        for layer, caches in enumerate(self.caches):
            blocks = [FrameBlock(self.frame_id, self.k[layer][h], self.v[layer][h]) for h in range(len(caches))]
            if self.mode == "baseline" or self.classes is None:
                o, _ = baseline_step(self.q[layer], caches, blocks, self.config, **kw)
            elif self.mode == "hma":
                o, _ = hma_step(self.q[layer], caches, blocks, self.classes[layer], self.config, **kw)
            else:
                o, _ = packed_step(self.q[layer], caches, blocks, self.classes[layer], self.config, **kw)
            outs.append(o)
        return outs

    def replay(self) -> list[torch.Tensor]:
        self.graph.replay()
        return self.outputs


def generate_session(model, config: SessionConfig, mode: str = "baseline",
                     observer: Callable[[StepTrace], None] | None = None, shadow: bool = False, **kw):
    """Run a full session; returns (per-step frame outputs, report)."""
    return Session(model, config, mode, observer=observer, shadow=shadow, **kw).run()
