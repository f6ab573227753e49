"""Torch-facing wrappers of the C ABI: KV arenas and the three device ops.

Only device tensors cross into the library (as raw pointers).  Nothing here
computes on the CPU: a missing extension or device raises.
"""

from __future__ import annotations

import bisect
import ctypes
import math
import os
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib
from .errors import ShapeError

TOKEN_ALIGN = 128  # head regions start on a kv-tile boundary
# d = 128 launches use the CTA-pair kernel (cta_group::2) unless DF_CTA_PAIR=0 or per call (pair=False).
USE_CTA_PAIR = os.environ.get("DF_CTA_PAIR", "1") == "1"
SUPPORTED_WIDTHS = (64, 128)


def padded_width(head_dim: int) -> int:
    """Arena / Q row width the kernel runs at for a given head_dim."""
    if head_dim < 1 or head_dim > 128:
        raise ShapeError(f"head_dim {head_dim} outside [1, 128] on the B200 path")
    return 64 if head_dim <= 64 else 128


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(stream: torch.cuda.Stream | None) -> ctypes.c_void_p:
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    if _RAW_STREAM is not None:  # the current stream's handle without torch.cuda.current_stream()'s Python layers
        return ctypes.c_void_p(_RAW_STREAM(torch.cuda.current_device()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Workspace:
    """Split-KV workspace of df_attn_fwd (piece partials + combine counters), owned by its user.

    Zero-filled at allocation; the kernel returns every combine counter to
    zero, so the next launch reuses it without a memset.  Launches that share
    one workspace must be stream-ordered: each KVArena (one per session) and
    each captured graph owns its own, so independent sessions on different
    streams never share counters.  Growing keeps the old buffer alive, since a
    captured CUDA graph may still launch into it.
    """

    def __init__(self, device: torch.device | str):
        self.device = torch.device(device)
        self.buf: torch.Tensor | None = None
        self._retired: list[torch.Tensor] = []

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes:
            if torch.cuda.is_current_stream_capturing():
                raise ShapeError(f"split workspace must grow to {nbytes} B during CUDA-graph capture; "
                                 "run the captured launches once eagerly first")
            if self.buf is not None:
                self._retired.append(self.buf)
            self.buf = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self.buf


class KVArena:
    """One device allocation holding the K and V rings of many heads.

    Layout: two bf16 planes ``k``/``v`` of shape [rows, width]; each head owns
    a region of whole frames starting on a 128-token boundary (so a head's
    last kv tile never straddles into another head's region except through
    zero/stale rows that the kernel masks).  The TMA descriptors of both
    planes are encoded once here and passed by value to every launch.
    """

    def __init__(self, total_rows: int, width: int, device: torch.device | str):
        if width not in SUPPORTED_WIDTHS:
            raise ShapeError(f"arena width {width} not in {SUPPORTED_WIDTHS}")
        total_rows = max(int(total_rows), TOKEN_ALIGN)
        self.device = torch.device(device)
        self.width = width
        self.rows = total_rows
        # zero-init: rows past a head's context are read (then masked) by the
        # last partial kv tile; zeros keep them finite.
        self.k = torch.zeros(total_rows, width, dtype=torch.bfloat16, device=self.device)
        self.v = torch.zeros(total_rows, width, dtype=torch.bfloat16, device=self.device)
        _lib.require_device(self.device.index if self.device.index is not None else torch.cuda.current_device())
        buf = (ctypes.c_uint8 * (_lib.DF_MAPS_PER_ARENA * _lib.DF_TMAP_BYTES))()
        _lib.call(
            "df_kv_arena_maps",
            ctypes.c_void_p(self.k.data_ptr()),
            ctypes.c_void_p(self.v.data_ptr()),
            ctypes.c_int64(total_rows),
            ctypes.c_int32(width),
            buf,
        )
        self.maps = bytes(buf)
        self._next = 0
        self.workspace = Workspace(self.device)

    def allocate(self, tokens: int) -> int:
        """Reserve a region of ``tokens`` rows; returns its first row."""
        start = self._next
        need = int(math.ceil(max(tokens, 1) / TOKEN_ALIGN) * TOKEN_ALIGN)
        if start + need > self.rows:
            raise ShapeError(f"arena full: {start}+{need} > {self.rows} rows")
        self._next = start + need
        return start

    @staticmethod
    def region_rows(tokens: int) -> int:
        return int(math.ceil(max(tokens, 1) / TOKEN_ALIGN) * TOKEN_ALIGN)

    @property
    def nbytes(self) -> int:
        return 2 * self.rows * self.width * 2


@dataclass
class HeadWork:
    """One head of one attention launch (df_head_desc)."""

    arena: KVArena
    base_row: int
    n_tok: int
    q_head: int
    o_head: int


@dataclass
class ProbeBuffers:
    """Device buffers of the fused DHP epilogue for one launch."""

    region_of_slot: torch.Tensor  # uint8 [heads, max_slots]
    row_sampled: torch.Tensor  # uint8 [hw]
    probe_rows: torch.Tensor  # float32 [heads, hw, 3]


def _merge(ranges: list[tuple[int, int]]) -> tuple[list[int], list[int]]:
    """Sorted, merged [lo, hi) byte ranges as two parallel lists."""
    los: list[int] = []
    his: list[int] = []
    for lo, hi in sorted(r for r in ranges if r[1] > r[0]):
        if his and lo <= his[-1]:
            his[-1] = max(his[-1], hi)
        else:
            los.append(lo)
            his.append(hi)
    return los, his


def _hits(merged: tuple[list[int], list[int]], ranges: list[tuple[int, int]]) -> bool:
    los, his = merged
    for lo, hi in ranges:
        i = bisect.bisect_right(los, lo) - 1
        if (i >= 0 and his[i] > lo) or (i + 1 < len(los) and los[i + 1] < hi):
            return True
    return False


class LaunchChain:
    """Library launches that one caller issues back to back on one stream.

    The staging copy of a layer may run as ``df_kv_append_overlapped``
    (programmatic dependent launch: it starts on the SMs the previous FMHA's
    last wave leaves idle) only inside a chain: the caller that owns the chain
    promises that no kernel outside the library runs on the stream between its
    chained launches (a foreign producer that triggers its dependents early
    could otherwise let the copy read unfinished data).  StepGraph, the
    benchmark's step loops and batched streams hold chains; the public step
    functions without ``chain=`` always emit the plain, fully serialised copy.

    State is per chain object: the footprint of the last FMHA launched through
    it, on which stream.  A copy overlaps only when that FMHA touches none of
    the bytes the copy writes and writes none it reads.
    """

    __slots__ = ("_stream", "_touched", "_written")

    def __init__(self):
        self.reset()

    def reset(self) -> None:
        self._stream = None
        self._touched = self._written = None

    def _may_overlap(self, stream: int, reads, writes) -> bool:
        return (self._touched is not None and self._stream == stream and not _hits(self._touched, writes)
                and not _hits(self._written, reads))


class PreparedLaunch:
    """A fully built df_attn_fwd / df_kv_append call: launching is one C call.

    ``touched`` / ``written`` (df_attn_fwd): the byte ranges the launch reads or writes / writes.
    ``reads`` / ``writes`` (a df_kv_append_overlapped candidate): the copy's source and
    destination ranges.  The overlapped variant is used only through a :class:`LaunchChain`
    whose last FMHA is disjoint from the copy; otherwise the plain df_kv_append runs.
    ``last_fn``: the entry point the most recent ``launch`` called.
    """

    def __init__(self, fn: str, args: tuple, keep: tuple, touched=None, written=None, reads=None, writes=None):
        self.fn, self.args, self.keep = fn, args, keep
        self.touched = _merge(touched) if touched is not None else None
        self.written = _merge(written) if written is not None else None
        self.reads, self.writes = reads, writes
        self.last_fn = None

    def launch(self, stream: torch.cuda.Stream | None = None, chain: LaunchChain | None = None) -> None:
        h = _stream_handle(stream)
        fn = self.fn
        if self.writes is not None:
            if chain is None or not chain._may_overlap(h.value or 0, self.reads, self.writes):
                fn = "df_kv_append"
        elif chain is not None:
            if self.touched is not None:
                chain._stream, chain._touched, chain._written = h.value or 0, self.touched, self.written
            elif fn != "df_kv_append":
                chain.reset()
        self.last_fn = fn
        _lib.call(fn, *self.args, h)


def prepare_attention(
    q: torch.Tensor,
    out: torch.Tensor,
    work: list[HeadWork],
    hw: int,
    scale: float,
    probe: ProbeBuffers | None = None,
    pair: bool | None = None,
    stream: torch.cuda.Stream | None = None,
    peer_out: Sequence[int] | None = None,
    workspace: "Workspace | None" = None,
) -> list[PreparedLaunch]:
    """Build the launch(es) of one ragged attention over every head in ``work``.

    ``q``: bf16 [q_heads*hw, width] (width = arena width); ``out``: bf16
    [o_heads*hw, d_out] with row stride ``out.stride(0)``.  One launch carries
    <= DF_MAX_HEADS heads from <= DF_MAX_ARENAS arenas; longer lists split into
    contiguous runs (a session uses one arena: one launch).  ``peer_out``:
    device pointers of buffers laid out like ``out`` (other ranks' gathered
    outputs) that receive the same rows -- the fused head-output all-gather.
    ``workspace``: split-KV partials + combine counters; default: the first
    head's arena's (one session = one arena = one writer, so launches sharing it
    are stream-ordered).
    """
    if not work:
        return []
    chunks, cur, seen = [], [], set()
    for i, w in enumerate(work):
        new_arena = id(w.arena) not in seen
        if cur and (len(cur) == _lib.DF_MAX_HEADS or (new_arena and len(seen) == _lib.DF_MAX_ARENAS)):
            chunks.append(cur)
            cur, seen = [], set()
        cur.append(i)
        seen.add(id(w.arena))
    chunks.append(cur)
    if len(chunks) > 1:
        out_launches = []
        for c in chunks:
            sl = slice(c[0], c[-1] + 1)
            sub_probe = None
            if probe is not None:
                sub_probe = ProbeBuffers(probe.region_of_slot[sl], probe.row_sampled, probe.probe_rows[sl])
            out_launches += prepare_attention(q, out, work[sl], hw, scale, sub_probe, pair, stream, peer_out,
                                              workspace)
        return out_launches
    if q.dtype != torch.bfloat16 or out.dtype != torch.bfloat16:
        raise ShapeError("q and out must be bfloat16")
    if not q.is_cuda or not out.is_cuda:
        raise ShapeError("q and out must be CUDA tensors")
    width = work[0].arena.width
    if q.dim() != 2 or q.shape[1] != width or not q.is_contiguous():
        raise ShapeError(f"q must be contiguous [rows, {width}], got {tuple(q.shape)}")
    if out.dim() != 2 or out.stride(1) != 1:
        raise ShapeError("out must be a row-major 2-D view")
    arenas: list[KVArena] = []
    idx: dict[int, int] = {}
    descs = (_lib.HeadDesc * len(work))()
    for i, w in enumerate(work):
        if w.arena.width != width:
            raise ShapeError("all heads of one launch must share the arena width")
        a = idx.get(id(w.arena))
        if a is None:
            a = len(arenas)
            idx[id(w.arena)] = a
            arenas.append(w.arena)
        descs[i].base_row = w.base_row
        descs[i].n_tok = w.n_tok
        descs[i].q_head = w.q_head
        descs[i].o_head = w.o_head
        descs[i].arena = a
    maps = b"".join(a.maps for a in arenas)
    maps_buf = ctypes.create_string_buffer(maps, len(maps))
    args = _lib.AttnArgs()
    args.q = q.data_ptr()
    args.q_rows = q.shape[0]
    args.out = out.data_ptr()
    args.out_ld = out.stride(0)
    args.hw = hw
    args.head_dim = width
    args.d_out = out.shape[1]
    args.scale = scale
    args.num_heads = len(work)
    args.num_arenas = len(arenas)
    args.heads = descs
    args.kv_maps = ctypes.cast(maps_buf, ctypes.c_void_p)
    use_pair = USE_CTA_PAIR if pair is None else pair
    args.flags = _lib.DF_ATTN_PAIR if use_pair else _lib.DF_ATTN_SINGLE_CTA
    if probe is not None:
        args.flags |= _lib.DF_ATTN_PROBE
        args.max_slots = probe.region_of_slot.shape[1]
        args.region_of_slot = probe.region_of_slot.data_ptr()
        args.row_sampled = probe.row_sampled.data_ptr()
        args.probe_rows = probe.probe_rows.data_ptr()
    peers = None
    if peer_out:
        if len(peer_out) > _lib.DF_MAX_PEERS:
            raise ShapeError(f"{len(peer_out)} peer outputs > {_lib.DF_MAX_PEERS}")
        peers = (ctypes.c_void_p * len(peer_out))(*peer_out)
        args.peer_out = ctypes.cast(peers, ctypes.POINTER(ctypes.c_void_p))
        args.n_peers = len(peer_out)
    need = ctypes.c_int64(0)
    _lib.call("df_attn_workspace_bytes", ctypes.byref(args), ctypes.byref(need))
    ws = None
    if need.value > 0:
        if workspace is None:
            workspace = work[0].arena.workspace
        ws = workspace.get(need.value)
        args.workspace = ws.data_ptr()
        args.workspace_bytes = ws.numel()
    written = [_span(out)]
    touched = [_span(q)]
    for w in work:
        # the last kv tile of a head is read whole (TMA box of 128 rows), masked in-kernel
        rows = min(-(-max(w.n_tok, 1) // 128) * 128, w.arena.rows - w.base_row)
        lo = w.base_row * w.arena.width * 2
        for plane in (w.arena.k, w.arena.v):
            touched.append((plane.data_ptr() + lo, plane.data_ptr() + lo + rows * w.arena.width * 2))
    if probe is not None:
        touched += [_span(probe.region_of_slot), _span(probe.row_sampled)]
        written.append(_span(probe.probe_rows))
    if ws is not None:
        written.append(_span(ws))
    return [PreparedLaunch("df_attn_fwd", (ctypes.byref(args),), (args, descs, maps_buf, ws, q, out, probe, peers),
                           touched=touched + written, written=written)]


def _span(t: torch.Tensor) -> tuple[int, int]:
    """[lo, hi) bytes a strided tensor view can touch."""
    if t.numel() == 0:
        return (t.data_ptr(), t.data_ptr())
    last = sum((n - 1) * st for n, st in zip(t.shape, t.stride()))
    return (t.data_ptr(), t.data_ptr() + (last + 1) * t.element_size())


def attention(
    q: torch.Tensor,
    out: torch.Tensor,
    work: list[HeadWork],
    hw: int,
    scale: float,
    probe: ProbeBuffers | None = None,
    stream: torch.cuda.Stream | None = None,
    pair: bool | None = None,
    workspace: "Workspace | None" = None,
    chain: LaunchChain | None = None,
) -> None:
    """Ragged attention over every head in ``work`` (see prepare_attention)."""
    for launch in prepare_attention(q, out, work, hw, scale, probe, pair, stream, workspace=workspace):
        launch.launch(stream, chain)


def prepare_copies(segs: list[tuple[int, int, int, int, int, int]], overlapped: bool = False) -> list[PreparedLaunch]:
    """df_kv_append launches (<= DF_MAX_APPEND_SEGS segments each), built ahead of time.

    ``overlapped``: the first launch is a df_kv_append_overlapped candidate; launched through a
    LaunchChain whose last FMHA touches none of its bytes it may start during that FMHA, otherwise
    (no chain, or a possible overlap) it runs as the serialised df_kv_append.
    """
    out = []
    for i in range(0, len(segs), _lib.DF_MAX_APPEND_SEGS):
        chunk = segs[i : i + _lib.DF_MAX_APPEND_SEGS]
        arr = (_lib.CopySeg * len(chunk))()
        for j, s in enumerate(chunk):
            arr[j].src, arr[j].dst, arr[j].rows, arr[j].src_ld, arr[j].dst_ld, arr[j].row_bytes = s
        if overlapped and i == 0:
            reads = [(s[0], s[0] + (s[2] - 1) * s[3] + s[5]) for s in chunk if s[2] > 0]
            writes = [(s[1], s[1] + (s[2] - 1) * s[4] + s[5]) for s in chunk if s[2] > 0]
            out.append(PreparedLaunch("df_kv_append_overlapped", (arr, ctypes.c_int32(len(chunk))), (arr,),
                                      reads=reads, writes=writes))
        else:
            out.append(PreparedLaunch("df_kv_append", (arr, ctypes.c_int32(len(chunk))), (arr,)))
    return out


def copy_segments(segs: list[tuple[int, int, int, int, int, int]], stream: torch.cuda.Stream | None = None) -> None:
    """Batched 16-byte-vectorised device copies, (src, dst, rows, src_ld, dst_ld, row_bytes) each."""
    for launch in prepare_copies(segs):
        launch.launch(stream)


class PackPlan:
    """A device-resident segment list for df_kv_pack (built once, launched once)."""

    def __init__(self, segs: list[tuple[int, int, int, int, int, int]], device: torch.device):
        n = len(segs)
        arr = (_lib.CopySeg * max(n, 1))()
        for j, s in enumerate(segs):
            arr[j].src, arr[j].dst, arr[j].rows, arr[j].src_ld, arr[j].dst_ld, arr[j].row_bytes = s
        prefix = (ctypes.c_int64 * (n + 1))()
        total = ctypes.c_int64(0)
        _lib.call("df_kv_pack_plan", arr, ctypes.c_int32(n), prefix, ctypes.byref(total))
        self.n = n
        self.total_blocks = int(total.value)
        self.bytes_moved = sum(2 * s[2] * s[5] for s in segs)  # read + write
        raw = bytes(memoryview(arr).cast("B"))[: n * ctypes.sizeof(_lib.CopySeg)]
        self.segs_dev = torch.frombuffer(bytearray(raw) or bytearray(8), dtype=torch.uint8).to(device)
        self.prefix_dev = torch.tensor(list(prefix), dtype=torch.int64, device=device)

    def launch(self, stream: torch.cuda.Stream | None = None) -> None:
        _lib.call(
            "df_kv_pack",
            ctypes.c_void_p(self.segs_dev.data_ptr()),
            ctypes.c_void_p(self.prefix_dev.data_ptr()),
            ctypes.c_int32(self.n),
            ctypes.c_int64(self.total_blocks),
            _stream_handle(stream),
        )


def scores_finalize(probe: ProbeBuffers, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Per-head mean region masses over the sampled rows -> float64 [heads, 3]."""
    heads, hw = probe.probe_rows.shape[0], probe.probe_rows.shape[1]
    F = torch.empty(heads, 3, dtype=torch.float64, device=probe.probe_rows.device)
    _lib.call(
        "df_scores_finalize",
        ctypes.c_void_p(probe.probe_rows.data_ptr()),
        ctypes.c_void_p(probe.row_sampled.data_ptr()),
        ctypes.c_int32(heads),
        ctypes.c_int32(hw),
        ctypes.c_void_p(F.data_ptr()),
        _stream_handle(stream),
    )
    return F


# ------------------------------------------------------------ fused projections
def _bf16_rows(t: torch.Tensor, name: str, cols: int | None = None) -> None:
    if t.dtype != torch.bfloat16 or not t.is_cuda:
        raise ShapeError(f"{name} must be a bf16 CUDA tensor, got {t.dtype} on {t.device}")
    if t.dim() != 2 or t.stride(1) != 1 or (cols is not None and t.shape[1] != cols):
        raise ShapeError(f"{name} must be a row-major 2-D matrix{'' if cols is None else f' with {cols} columns'}, "
                         f"got shape {tuple(t.shape)} strides {t.stride()}")


def prepare_qkv_projection(x: torch.Tensor, w_qkv: torch.Tensor, q_out: torch.Tensor, k_dst: list[torch.Tensor],
                           v_dst: list[torch.Tensor], head_dim: int) -> PreparedLaunch:
    """df_qkv_project: ``[q|k|v] = x @ [W_q|W_k|W_v]`` (scenario.py:102-114), fused scatter.

    ``x`` bf16 [hw, in_dim]; ``w_qkv`` bf16 [3*heads*head_dim, in_dim] (the
    transposed, concatenated projection weights of the heads); ``q_out`` bf16
    [heads, hw, head_dim] contiguous; ``k_dst[h]`` / ``v_dst[h]`` bf16 [hw,
    head_dim] row-strided views (the heads' pending ring slots) sharing one row
    stride.
    """
    heads = len(k_dst)
    if heads != len(v_dst) or not 1 <= heads <= _lib.DF_MAX_HEADS:
        raise ShapeError(f"{heads} K / {len(v_dst)} V destinations (1..{_lib.DF_MAX_HEADS} heads per launch)")
    _bf16_rows(x, "x")
    hw, in_dim = x.shape
    _bf16_rows(w_qkv, "w_qkv", in_dim)
    if w_qkv.shape[0] != 3 * heads * head_dim:
        raise ShapeError(f"w_qkv has {w_qkv.shape[0]} rows, expected 3*{heads}*{head_dim}")
    if q_out.dtype != torch.bfloat16 or tuple(q_out.shape) != (heads, hw, head_dim) or not q_out.is_contiguous():
        raise ShapeError(f"q_out must be contiguous bf16 {(heads, hw, head_dim)}, got {tuple(q_out.shape)}")
    ld = None
    for t in list(k_dst) + list(v_dst):
        if t.dtype != torch.bfloat16 or tuple(t.shape) != (hw, head_dim) or t.stride(1) != 1:
            raise ShapeError(f"K/V destination must be a bf16 ({hw}, {head_dim}) row view, got {tuple(t.shape)}")
        ld = t.stride(0) if ld is None else ld
        if t.stride(0) != ld:
            raise ShapeError("K/V destinations must share one row stride")
    args = _lib.QkvArgs()
    args.x, args.w_qkv = x.data_ptr(), w_qkv.data_ptr()
    args.hw, args.num_heads, args.head_dim, args.in_dim = hw, heads, head_dim, in_dim
    args.q_out = q_out.data_ptr()
    for h in range(heads):
        args.k_dst[h] = k_dst[h].data_ptr()
        args.v_dst[h] = v_dst[h].data_ptr()
    args.kv_ld = ld
    return PreparedLaunch("df_qkv_project", (ctypes.byref(args),), (args, x, w_qkv, q_out, k_dst, v_dst))


def prepare_out_projection(o: torch.Tensor, w_o: torch.Tensor, x: torch.Tensor, x_bf16: torch.Tensor | None,
                           head_dim: int) -> PreparedLaunch:
    """df_out_project: ``x += merge(o) @ W_o`` (scenario.py:116-120 + engine.py:443 residual).

    ``o`` bf16 [heads, hw, head_dim] contiguous (the FMHA output); ``w_o`` bf16
    [out_dim, heads*head_dim]; ``x`` fp32 [hw, out_dim] updated in place;
    ``x_bf16`` (optional) bf16 [hw, out_dim] receives the updated x.
    """
    if o.dtype != torch.bfloat16 or o.dim() != 3 or o.shape[2] != head_dim or not o.is_contiguous():
        raise ShapeError(f"o must be contiguous bf16 (heads, hw, {head_dim}), got {tuple(o.shape)}")
    heads, hw, _ = o.shape
    _bf16_rows(w_o, "w_o", heads * head_dim)
    out_dim = w_o.shape[0]
    if x.dtype != torch.float32 or tuple(x.shape) != (hw, out_dim) or not x.is_contiguous():
        raise ShapeError(f"x must be contiguous fp32 ({hw}, {out_dim}), got {x.dtype} {tuple(x.shape)}")
    if x_bf16 is not None and (x_bf16.dtype != torch.bfloat16 or tuple(x_bf16.shape) != (hw, out_dim)
                               or not x_bf16.is_contiguous()):
        raise ShapeError(f"x_bf16 must be contiguous bf16 ({hw}, {out_dim})")
    args = _lib.OprojArgs()
    args.o, args.w_o = o.data_ptr(), w_o.data_ptr()
    args.hw, args.num_heads, args.head_dim, args.out_dim = hw, heads, head_dim, out_dim
    args.x = x.data_ptr()
    args.x_bf16 = x_bf16.data_ptr() if x_bf16 is not None else None
    return PreparedLaunch("df_out_project", (ctypes.byref(args),), (args, o, w_o, x, x_bf16))
