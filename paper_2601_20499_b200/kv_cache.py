"""Per-head KV ring buffers in HBM with the reference's retention policies.

Semantics follow the reference's kv_cache.py:1-285 (policies, eviction,
rebuild, gather order, accounting); storage is B200-native:

* Every head owns a ring of ``warm_past_frames() + 1`` frame slots (the +1 is
  the current frame) inside a shared :class:`~.kernels.KVArena`.  Slot ``s``
  is arena rows ``[base_row + s*HW, base_row + (s+1)*HW)``.
* Invariant: the occupied slots plus the *pending* slot (where the current
  frame is staged before attention) are exactly slots ``[0, len+1)``.  The
  attention kernel therefore reads each head's context as ONE contiguous row
  range; key order inside it is irrelevant (softmax is permutation
  invariant).  Eviction is a slot-table update -- the next frame simply
  lands in the freed slot -- so steady state moves no data except the
  appended frame itself (kv_cache.py:187-197 without list copies).
* ``rebuild`` (classification time) compacts the retained frames of many
  heads into a fresh arena with one ``df_kv_pack`` launch.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import kernels as K
from .config import SessionConfig
from .errors import ConfigError, OrderingError, ShapeError
from .head_programming import HeadAssignment, HeadClass
from .layout import REGION_CODE, FrameLayout

POLICY_KINDS = ("baseline_window", "sink_only", "neighbor_window", "dummy_empty", "dummy_packed")


def _device_of(x) -> torch.device:
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.device
    return torch.device("cuda", torch.cuda.current_device())


def as_device_bf16(x, device: torch.device | None = None) -> torch.Tensor:
    """Host/numpy/float operands -> bf16 on the device (data movement only)."""
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    dev = device if device is not None else _device_of(x)
    if x.device != dev or x.dtype != torch.bfloat16:
        x = x.to(device=dev, dtype=torch.bfloat16, non_blocking=True)
    return x


@dataclass(frozen=True, eq=False)
class FrameBlock:
    """K/V rows of one frame for one head: keys/values are (HW, head_dim)."""

    frame_id: int
    keys: object
    values: object

    def __post_init__(self):
        k, v = self.keys, self.values
        if getattr(k, "ndim", None) != 2 or getattr(v, "ndim", None) != 2:
            raise ShapeError("frame keys/values must be 2-D")
        if k.shape[0] != v.shape[0]:
            raise ShapeError(f"keys rows {k.shape[0]} != values rows {v.shape[0]}")

    @property
    def tokens(self) -> int:
        return int(self.keys.shape[0])


@dataclass(frozen=True)
class CachePolicy:
    """Retention policy (kv_cache.py:58-101)."""

    kind: str
    window_len: int
    sink_frame: int = 0
    extended_window: int | None = None

    def __post_init__(self):
        if self.kind not in POLICY_KINDS:
            raise ConfigError(f"unknown policy kind {self.kind!r}")
        if self.kind in ("baseline_window", "neighbor_window") and self.window_len < 2:
            raise ConfigError(f"{self.kind} needs window_len >= 2")
        if self.extended_window is not None:
            if self.kind != "neighbor_window":
                raise ConfigError("extended_window only applies to neighbor_window")
            if self.extended_window < self.window_len - 1:
                raise ConfigError("extended_window must be at least the plain window size")

    @property
    def recent_capacity(self) -> int:
        if self.kind == "baseline_window":
            return self.window_len - 1
        if self.kind == "neighbor_window":
            return self.window_len - 1 if self.extended_window is None else self.extended_window
        if self.kind == "dummy_packed":
            return 1
        return 0  # sink_only, dummy_empty

    @property
    def keeps_sink(self) -> bool:
        return self.kind in ("baseline_window", "sink_only")

    def warm_past_frames(self) -> int:
        return self.recent_capacity + (1 if self.keeps_sink else 0)

    @property
    def ring_slots(self) -> int:
        """Device slots: every retained past frame plus the current frame."""
        return self.warm_past_frames() + 1

    def retain(self, frame_ids: list[int]) -> list[int]:
        """Frames kept after an append (kv_cache.py:187-197)."""
        pinned = [f for f in frame_ids if self.keeps_sink and f == self.sink_frame]
        others = [f for f in frame_ids if not (self.keeps_sink and f == self.sink_frame)]
        n = min(self.recent_capacity, len(others))
        return sorted(pinned + (others[len(others) - n :] if n else []))


def derive_policy(head_class: HeadClass, config: SessionConfig, extended_window: int | None = None) -> CachePolicy:
    """Class -> policy (kv_cache.py:104-132)."""
    common = dict(window_len=config.window_len, sink_frame=config.sink_frame)
    if head_class is HeadClass.DUMMY:
        return CachePolicy("dummy_packed" if config.packing_enabled else "dummy_empty", **common)
    if config.merged_window is not None:
        return CachePolicy("baseline_window", window_len=config.merged_window, sink_frame=config.sink_frame)
    if head_class is HeadClass.SINK:
        return CachePolicy("sink_only", **common)
    if config.context_extension and extended_window is not None:
        return CachePolicy("neighbor_window", extended_window=extended_window, **common)
    return CachePolicy("neighbor_window", **common)


def baseline_policy(config: SessionConfig) -> CachePolicy:
    return CachePolicy("baseline_window", window_len=config.window_len, sink_frame=config.sink_frame)


def extension_window(assignment: HeadAssignment, config: SessionConfig) -> int | None:
    """Neighbor window grown by the budget sink/dummy heads free (kv_cache.py:143-158)."""
    counts = assignment.counts()
    n_nb = counts[HeadClass.NEIGHBOR.value]
    if n_nb == 0:
        return None
    budget = assignment.total_heads * config.baseline_past_frames
    spent = counts[HeadClass.SINK.value] + counts[HeadClass.DUMMY.value] * (1 if config.packing_enabled else 0)
    return max((budget - spent) // n_nb, config.window_len - 1)


@dataclass
class RingStorage:
    """Where a head's ring lives."""

    arena: K.KVArena
    base_row: int
    slots: int
    hw: int
    head_dim: int

    def rows(self, slot: int) -> slice:
        a = self.base_row + slot * self.hw
        return slice(a, a + self.hw)


def _row_bytes(d: int) -> int:
    return ((d + 7) // 8) * 8 * 2


def _in_place(block: FrameBlock, st: RingStorage, slot: int) -> bool:
    """``block`` IS ring slot ``slot`` (df_qkv_project wrote it there): checked on raw pointers, no views."""
    k, v = block.keys, block.values
    if not (isinstance(k, torch.Tensor) and isinstance(v, torch.Tensor)) or k.dtype != torch.bfloat16:
        return False
    row0 = st.base_row + slot * st.hw
    step = st.arena.width * 2
    return (k.data_ptr() == st.arena.k.data_ptr() + row0 * step and v.data_ptr() == st.arena.v.data_ptr() + row0 * step
            and k.stride(0) == st.arena.width and v.stride(0) == st.arena.width and k.shape[0] == st.hw)


def _block_segments(block: FrameBlock, st: RingStorage, slot: int, device) -> list[tuple]:
    """Copy segments (K and V) writing `block` into ring slot `slot`."""
    if _in_place(block, st, slot):
        return []  # produced in place: nothing to move
    segs = []
    d = st.head_dim
    width = st.arena.width
    for src, plane in ((block.keys, st.arena.k), (block.values, st.arena.v)):
        t = as_device_bf16(src, device)
        if t.shape != (st.hw, d):
            raise ShapeError(f"frame block {tuple(t.shape)} != ({st.hw}, {d})")
        if d % 8 or t.stride(1) != 1 or (t.stride(0) * 2) % 16 or t.data_ptr() % 16:
            t = torch.nn.functional.pad(t, (0, (-d) % 8)).contiguous()
        dst = plane[st.rows(slot)]
        if t.data_ptr() == dst.data_ptr() and t.stride(0) == dst.stride(0):
            continue  # produced in place (df_qkv_project wrote the pending slot): nothing to move
        segs.append((t.data_ptr(), dst.data_ptr(), st.hw, t.stride(0) * 2, width * 2, _row_bytes(d)))
        # keep the temporary alive until the copy is enqueued
        segs[-1] = segs[-1] + (t,)
    return segs


def launch_segments(segs: list[tuple], stream=None) -> None:
    K.copy_segments([s[:6] for s in segs], stream)


class HeadKVCache:
    """Frame ring of one head (API of kv_cache.py:161-222)."""

    def __init__(self, policy: CachePolicy, blocks: list[FrameBlock] | None = None, *, storage: RingStorage | None = None):
        self.policy = policy
        self.storage = storage
        self._slot_frame: list[int | None] = [None] * (storage.slots if storage else policy.ring_slots)
        self._staged: tuple | None = None
        self._views: dict[int, tuple] = {}  # pending-slot views (pending_view), per storage
        self._views_of: RingStorage | None = None
        for b in blocks or []:
            self.append_and_evict(b)

    # ------------------------------------------------------------ storage
    def ensure_storage(self, hw: int, head_dim: int, device=None) -> RingStorage:
        if self.storage is None:
            width = K.padded_width(head_dim)
            slots = self.policy.ring_slots
            arena = K.KVArena(K.KVArena.region_rows(slots * hw), width, device or torch.device("cuda", torch.cuda.current_device()))
            self.storage = RingStorage(arena, arena.allocate(slots * hw), slots, hw, head_dim)
            self._slot_frame = [None] * slots
        elif self.storage.hw != hw or self.storage.head_dim != head_dim:
            raise ShapeError(f"block ({hw}, {head_dim}) does not match cache ({self.storage.hw}, {self.storage.head_dim})")
        return self.storage

    # ------------------------------------------------------------ views
    def __len__(self) -> int:
        return sum(f is not None for f in self._slot_frame)

    @property
    def frame_ids(self) -> list[int]:
        return sorted(f for f in self._slot_frame if f is not None)

    def slot_of(self, frame_id: int) -> int:
        return self._slot_frame.index(frame_id)

    @property
    def pending_slot(self) -> int:
        """Slot the current frame occupies during attention (lowest free)."""
        for s, f in enumerate(self._slot_frame):
            if f is None:
                return s
        raise ShapeError("ring has no free slot")  # unreachable by construction

    @property
    def blocks(self) -> list[FrameBlock]:
        st = self.storage
        if st is None:
            return []
        out = []
        for f in self.frame_ids:
            r = st.rows(self.slot_of(f))
            out.append(FrameBlock(f, st.arena.k[r, : st.head_dim], st.arena.v[r, : st.head_dim]))
        return out

    def pending_view(self, hw: int, head_dim: int, device=None) -> tuple[torch.Tensor, torch.Tensor]:
        """(K, V) bf16 [hw, head_dim] views of the pending slot.

        A producer (``df_qkv_project``) may write the current frame here in
        place; a FrameBlock over these views then stages and appends with no
        copy at all.
        """
        st = self.ensure_storage(hw, head_dim, device)
        slot = self.pending_slot
        views = self._views.get(slot) if self._views_of is st else None
        if views is None:  # views of a slot are reused across layers' denoise iterations
            if self._views_of is not st:
                self._views, self._views_of = {}, st
            r = st.rows(slot)
            views = self._views[slot] = (st.arena.k[r, :head_dim], st.arena.v[r, :head_dim])
        return views

    def past_tokens(self) -> int:
        return len(self) * (self.storage.hw if self.storage else 0)

    def context_tokens(self, hw: int) -> int:
        return (len(self) + 1) * hw

    def region_codes(self) -> list[int]:
        """Per ring slot: 0 sink, 1 neighbor, 2 current (kv_cache.py:214-217 labels)."""
        pend = self.pending_slot
        codes = []
        for s, f in enumerate(self._slot_frame):
            if s == pend:
                codes.append(REGION_CODE["current"])
            elif f is not None and f == self.policy.sink_frame:
                codes.append(REGION_CODE["sink"])
            else:
                codes.append(REGION_CODE["neighbor"])
        return codes

    # ------------------------------------------------------------ updates
    def _newest(self) -> int | None:
        return max((f for f in self._slot_frame if f is not None), default=None)

    def check_current(self, frame_id: int) -> None:
        newest = self._newest()
        if newest is not None and frame_id <= newest:
            raise OrderingError(f"current frame {frame_id} not newer than cache")

    def stage_segments(self, block: FrameBlock, device=None) -> list[tuple]:
        """Copy plan putting the current frame into the pending slot."""
        self.check_current(block.frame_id)
        dev = device or _device_of(block.keys)
        st = self.ensure_storage(block.tokens, int(block.keys.shape[1]), dev)
        slot = self.pending_slot
        segs = _block_segments(block, st, slot, dev)
        self._staged = (block.frame_id, slot, st.arena, block.keys, block.values) + _versions(block)
        return segs

    def append_and_evict(self, block: FrameBlock, stream=None) -> "HeadKVCache":
        """Append one frame, then drop what the policy does not keep."""
        segs = self.append_segments(block)
        if segs:
            launch_segments(segs, stream)
        return self

    def append_segments(self, block: FrameBlock, device=None) -> list[tuple]:
        """Slot-table append + eviction; returns the copies still needed."""
        ids = self.frame_ids
        if ids and block.frame_id <= ids[-1]:
            raise OrderingError(f"frame {block.frame_id} not newer than cached {ids[-1]}")
        dev = device or _device_of(block.keys)
        st = self.ensure_storage(block.tokens, int(block.keys.shape[1]), dev)
        slot = self.pending_slot
        segs: list[tuple] = []
        if not _same_staging(self._staged, block, slot, st.arena):
            segs = _block_segments(block, st, slot, dev)
        self._staged = None
        for src, dst in self._append_slots(block.frame_id):
            for plane in (st.arena.k, st.arena.v):
                a, b = plane[st.rows(src)], plane[st.rows(dst)]
                segs.append((a.data_ptr(), b.data_ptr(), st.hw, st.arena.width * 2, st.arena.width * 2,
                             st.arena.width * 2))
        return segs

    def _append_slots(self, frame_id: int) -> list[tuple[int, int]]:
        """Slot-table half of an append: ``frame_id`` takes the pending slot, the policy evicts
        (kv_cache.py:187-197), then the prefix invariant (occupied + pending == [0, len+1)) is
        restored by moving the highest occupied slots down.  Returns the (src, dst) slot moves.
        A pure function of the table, so another process can replay a ring's layout."""
        self._slot_frame[self.pending_slot] = frame_id
        keep = set(self.policy.retain(self.frame_ids))
        self._slot_frame = [f if (f is not None and f in keep) else None for f in self._slot_frame]
        moves = []
        while True:
            n = len(self)
            high = [s for s, f in enumerate(self._slot_frame) if f is not None and s > n]
            if not high:
                return moves
            src = max(high)
            dst = self.pending_slot
            moves.append((src, dst))
            self._slot_frame[dst], self._slot_frame[src] = self._slot_frame[src], None

    def rebuild(self, policy: CachePolicy) -> "HeadKVCache":
        """A new cache holding what ``policy`` keeps of this history (kv_cache.py:199-201)."""
        return rebuild_caches([self], [policy])[0]

    def gather_context(self, current: FrameBlock):
        """(keys, values, FrameLayout): cached frames in frame order, then current."""
        self.check_current(current.frame_id)
        blocks = self.blocks
        dev = _device_of(current.keys) if self.storage is None else self.storage.arena.device
        keys = torch.cat([b.keys for b in blocks] + [as_device_bf16(current.keys, dev)], dim=0)
        values = torch.cat([b.values for b in blocks] + [as_device_bf16(current.values, dev)], dim=0)
        kinds = ["sink" if b.frame_id == self.policy.sink_frame else "neighbor" for b in blocks] + ["current"]
        return keys, values, FrameLayout.from_frame_kinds(current.tokens, kinds)


def _versions(block: FrameBlock) -> tuple:
    k, v = block.keys, block.values
    return (getattr(k, "_version", None), getattr(v, "_version", None))


def _same_staging(staged, block: FrameBlock, slot: int, arena) -> bool:
    """True when ``block`` is exactly what the last step staged into ``slot``.

    The staged record holds the tensors themselves (not addresses), so an
    allocator reusing an address can never alias; in-place edits bump
    ``_version``.  Then the append is a pure slot-table update.
    """
    if staged is None:
        return False
    fid, s, a, k, v, kv, vv = staged
    return (fid == block.frame_id and s == slot and a is arena and k is block.keys and v is block.values
            and (kv, vv) == _versions(block))


def replay_slot_table(policy: CachePolicy, history: list[int], appended: list[int]) -> list[int | None]:
    """The slot table of a ring rebuilt under ``policy`` from the frame ids ``history`` (rebuild_caches
    lays the retained frames in frame order) and then appended ``appended`` -- what that ring holds in
    which slot, computed without storage (a head-parallel rank receiving the ring lays the rows out
    identically, so key order and hence the attention's summation order match the sender's)."""
    n = HeadKVCache(policy)
    kept: list[int] = []
    for f in history:
        kept = policy.retain(kept + [f])
    for s, f in enumerate(kept):
        n._slot_frame[s] = f
    for f in appended:
        n._append_slots(f)
    return list(n._slot_frame)


def rebuild_caches(caches: list[HeadKVCache], policies: list[CachePolicy], arena: K.KVArena | None = None,
                   stream=None, stats: dict | None = None) -> list[HeadKVCache]:
    """Re-lay many heads' retained frames under new policies: ONE df_kv_pack launch.

    The new rings live in ``arena`` (allocated here if None).  Retention is
    the reference's re-append of the history under the new policy.
    """
    if len(caches) != len(policies):
        raise ShapeError("one policy per cache")
    stores = [c.storage for c in caches]
    template = next((s for s in stores if s is not None), None)
    if template is None:  # nothing stored yet: just replay ids
        out = []
        for c, p in zip(caches, policies):
            n = HeadKVCache(p)
            for f in c.frame_ids:
                n._slot_frame[n.pending_slot] = f
                keep = set(p.retain(n.frame_ids))
                n._slot_frame = [x if (x is not None and x in keep) else None for x in n._slot_frame]
            out.append(n)
        return out
    hw, d = template.hw, template.head_dim
    if arena is None:
        rows = sum(K.KVArena.region_rows(p.ring_slots * hw) for p in policies)
        arena = K.KVArena(rows, template.arena.width, template.arena.device)
    segs = []
    out = []
    for c, p in zip(caches, policies):
        kept: list[int] = []
        for f in c.frame_ids:
            kept = p.retain(kept + [f])
        st = RingStorage(arena, arena.allocate(p.ring_slots * hw), p.ring_slots, hw, d)
        n = HeadKVCache(p, storage=st)
        for s, f in enumerate(kept):
            n._slot_frame[s] = f
            src = c.storage.rows(c.slot_of(f))
            dst = st.rows(s)
            for sp, dp in ((c.storage.arena.k, arena.k), (c.storage.arena.v, arena.v)):
                segs.append((sp[src].data_ptr(), dp[dst].data_ptr(), hw, sp.shape[1] * 2, dp.shape[1] * 2,
                             min(sp.shape[1], dp.shape[1]) * 2))
        out.append(n)
    if segs:
        plan = K.PackPlan(segs, arena.device)
        if stats is not None:  # device time of the df_kv_pack launch alone
            s = stream if stream is not None else torch.cuda.current_stream(arena.device)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(s)
            plan.launch(s)
            ev[1].record(s)
            stats.update(bytes=plan.bytes_moved, events=tuple(ev), blocks=plan.total_blocks)
        else:
            plan.launch(stream)
    return out


@dataclass(frozen=True)
class CacheStats:
    """Warm-state accounting of an assignment (kv_cache.py:225-236)."""

    per_head_past_frames: tuple[int, ...]
    baseline_past_frames: int
    tokens_per_frame: int
    reduction_ratio: float

    @property
    def total_cached_tokens(self) -> int:
        return sum(self.per_head_past_frames) * self.tokens_per_frame


def cache_stats(assignment: HeadAssignment, config: SessionConfig) -> CacheStats:
    """Cached past frames per head and the reduction ratio (kv_cache.py:239-260)."""
    ext = extension_window(assignment, config) if config.context_extension else None
    per = tuple(derive_policy(c, config, extended_window=ext).warm_past_frames() for c in assignment.classes)
    base = config.baseline_past_frames
    return CacheStats(per, base, config.HW, sum(per) / (assignment.total_heads * base))


def uniform_budget_ratio(budget_frames: float, baseline_past_frames: int) -> float:
    if baseline_past_frames < 1:
        raise ConfigError("baseline_past_frames must be >= 1")
    if budget_frames < 0:
        raise ConfigError("budget_frames must be >= 0")
    return budget_frames / baseline_past_frames


def cache_snapshot(caches: list[list[HeadKVCache]]) -> dict[str, torch.Tensor]:
    """Named device tensors ``layer{l}/head{h}/frame{id}/{keys,values}`` (kv_cache.py:272-285)."""
    out: dict[str, torch.Tensor] = {}
    for li, layer in enumerate(caches):
        for hi, cache in enumerate(layer):
            for b in cache.blocks:
                out[f"layer{li}/head{hi}/frame{b.frame_id}/keys"] = b.keys
                out[f"layer{li}/head{hi}/frame{b.frame_id}/values"] = b.values
    return out
