"""Multi-GPU execution of the hot path, one process per GPU.

* Independent video streams (``stream_partition``): sessions share nothing
  (the reference allows concurrent independent sessions), so
  streams are dealt round-robin to ranks and the data path has NO collective.
  Only the benchmark's timing uses a max-reduction over ranks.
* Head-parallel sessions (``HeadParallelSession``, 2/4 GPUs for the 4x
  tokens-per-frame config): heads are independent inside attention
  (engine.py:111-137).  Each rank owns a contiguous block of
  H/P heads of every layer -- their Q/K/V, KV rings and attention launches.
  After each layer the head outputs are all-gathered (NCCL over NVLink) so
  every rank can run ``mix``; at the probe the per-head frame scores are
  all-gathered and every rank runs the same deterministic greedy
  (df_greedy_classify), so all ranks agree on the assignment bit for bit.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .config import SessionConfig
from .engine import Session
from .errors import ConfigError


def head_partition(num_heads: int, world: int, rank: int) -> range:
    """Contiguous, equal head block of ``rank`` (heads must divide evenly)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of {world}")
    if num_heads % world:
        raise ConfigError(f"{num_heads} heads do not split evenly over {world} ranks")
    per = num_heads // world
    return range(rank * per, (rank + 1) * per)


def stream_partition(num_streams: int, world: int, rank: int) -> list[int]:
    """Round-robin stream ids owned by ``rank`` (no collective needed)."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} of {world}")
    return list(range(rank, num_streams, world))


def _all_gather(t: torch.Tensor, group) -> torch.Tensor:
    """Stack every rank's equally shaped tensor along a new leading dim."""
    world = dist.get_world_size(group)
    t = t.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world, *t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return out
    # gloo (CPU tests; several ranks sharing one GPU in the 2-process session test): through the host
    host = t.cpu()
    out = torch.empty((world, *t.shape), dtype=t.dtype)
    dist.all_gather(list(out.unbind(0)), host, group=group)
    return out.to(t.device)


def gather_head_outputs(local: torch.Tensor, group=None) -> torch.Tensor:
    """(H/P, HW, d) per rank -> (H, HW, d) in global head order on every rank."""
    g = _all_gather(local, group)
    return g.reshape(g.shape[0] * g.shape[1], *g.shape[2:])


def gather_head_scores(local: torch.Tensor, group=None) -> torch.Tensor:
    """(layers, H/P, 3) per rank -> (layers, H, 3), flat index layer*H + head."""
    g = _all_gather(local, group)  # (P, layers, H/P, 3)
    return g.permute(1, 0, 2, 3).reshape(local.shape[0], -1, local.shape[2])


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max over ranks)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class HeadParallelSession(Session):
    """A Session whose heads are sharded over the ranks of ``group``.

    Until classification every rank owns a contiguous block of H/P heads of
    every layer.  With ``rebalance`` (default) the step that classifies ends by
    re-dealing each layer's heads to ranks by LPT over their post-
    classification context lengths (``lpt_owners``) and moving the rings of
    the heads that change owner once, rank to rank (``exchange_frames``).
    """

    def __init__(self, model, config: SessionConfig, mode: str = "baseline", group=None, rebalance: bool = True,
                 fused_gather: bool = False, **kw):
        if not dist.is_initialized():
            raise ConfigError("HeadParallelSession needs torch.distributed to be initialised")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        head_partition(config.num_heads, self.world, self.rank)  # validates divisibility
        super().__init__(model, config, mode, **kw)
        self.rebalance = rebalance and self.shadow_caches is None
        self.owners = None  # (layers, heads) owner table once rebalanced
        self._history: list[int] | None = None
        self.fused = None
        if fused_gather:
            d8 = ((config.head_dim + 7) // 8) * 8
            self.fused = FusedHeadGather(config.num_heads * config.HW, d8, group, self.device)

    def _graphable(self, ratios) -> bool:
        return False  # per-layer collectives (NCCL or the symmetric-memory barrier) stay eager

    def _output_target(self, layer: int):
        if self.fused is None:
            return None
        return self.fused.target(layer, self.layer_heads[layer])

    def _owned_heads(self) -> range:
        return head_partition(self.config.num_heads, self.world, self.rank)

    def _gather_outputs(self, layer: int, outputs: torch.Tensor) -> torch.Tensor:
        if self.fused is not None and outputs.data_ptr() == self.fused.current().data_ptr():
            # every rank's FMHA epilogue stored its heads' rows into all buffers
            if self.stream is not None:
                with torch.cuda.stream(self.stream):
                    self.fused.barrier()
            else:
                self.fused.barrier()
            return outputs[:, :, : self.config.head_dim]
        if self.owners is not None:
            return gather_head_outputs_owned(outputs, self.owners[layer], self.group)
        return gather_head_outputs(outputs, self.group)

    def _gather_scores(self, local: torch.Tensor) -> torch.Tensor:
        return gather_head_scores(local, self.group)

    def _classify(self) -> None:
        self._history = list(self.caches[0][0].frame_ids)  # identical for every head under the baseline policy
        super()._classify()

    def _after_step(self, ar_step: int) -> None:
        if self.rebalance and self.owners is None and self.assignment is not None:
            self._rebalance(ar_step)

    def _rebalance(self, frame_id: int) -> None:
        """Move heads to their LPT owners after the classifying step's append."""
        import numpy as np

        from . import kernels as K
        from .kv_cache import HeadKVCache, RingStorage, derive_policy, extension_window, replay_slot_table

        cfg = self.config
        L, H = cfg.num_layers, cfg.num_heads
        ext = extension_window(self.assignment, cfg) if cfg.context_extension else None
        pol = [[derive_policy(self.assignment.classes[l * H + h], cfg, extended_window=ext) for h in range(H)]
               for l in range(L)]
        old = contiguous_owners(L, H, self.world)
        new = lpt_owners(np.array([[p.ring_slots for p in row] for row in pol]), self.world)
        keep, send, recv = rebalance_plan(old, new, self.rank)

        def layout(p) -> list[int | None]:  # rebuild under p, then the classifying step's append
            return replay_slot_table(p, self._history, [frame_id])

        h0 = self.head_range.start
        sends = []
        for l, h, dst in send:
            c = self.caches[l][h - h0]
            if c._slot_frame != layout(pol[l][h]):
                raise ConfigError(f"layer {l} head {h}: ring slots {c._slot_frame} != {layout(pol[l][h])}")
            for f in c.frame_ids:
                rows = c.storage.rows(c.slot_of(f))
                sends += [(dst, c.storage.arena.k[rows]), (dst, c.storage.arena.v[rows])]
        incoming: dict[tuple[int, int], HeadKVCache] = {}
        recvs = []
        if recv:
            rows_needed = sum(K.KVArena.region_rows(pol[l][h].ring_slots * cfg.HW) for l, h, _ in recv)
            arena = K.KVArena(rows_needed, K.padded_width(cfg.head_dim), self.device)
            for l, h, src in recv:
                p = pol[l][h]
                st = RingStorage(arena, arena.allocate(p.ring_slots * cfg.HW), p.ring_slots, cfg.HW, cfg.head_dim)
                n = HeadKVCache(p, storage=st)
                n._slot_frame = layout(p)  # the sender's slots: same key order in the ring
                for f in n.frame_ids:  # frame order, as the sender sends
                    rows = st.rows(n.slot_of(f))
                    recvs += [(src, arena.k[rows]), (src, arena.v[rows])]
                incoming[(l, h)] = n
        torch.cuda.synchronize(self.device)  # the rings' last append is on the session stream
        exchange_frames(sends, recvs, self.group)
        torch.cuda.synchronize(self.device)
        heads = [[h for h in range(H) if new[l, h] == self.rank] for l in range(L)]
        self.caches = [[incoming[(l, h)] if (l, h) in incoming else self.caches[l][h - h0] for h in heads[l]]
                       for l in range(L)]
        self.layer_heads = heads
        self.owners = new
        self.rebalance_stats = {"kept": len(keep), "sent": len(send), "received": len(recv),
                                "bytes_sent": sum(t.numel() * t.element_size() for _, t in sends)}


# ---------------------------------------------------------------------------
# Post-classification LPT rebalancing: after the one-shot
# classification the heads of a layer cost very different amounts (a packed
# dummy head attends to 2 frames, a neighbour head to W), so the contiguous
# equal blocks of ``head_partition`` leave ranks idle at every per-layer
# all-gather.  Every rank computes the same longest-processing-time owner
# table from the policies, and the retained frames of the heads that change
# owner move ONCE, rank to rank (NCCL P2P over NVLink on the GPU box).


def lpt_owners(costs, world: int):
    """Owner rank of every (layer, head): per layer, heads by decreasing cost
    (lower index first on ties) go to the least-loaded rank (lowest rank on
    ties).  Deterministic, so all ranks agree without a collective."""
    import numpy as np

    costs = np.asarray(costs)
    if costs.ndim != 2:
        raise ConfigError("costs must be (layers, heads)")
    if world < 1:
        raise ConfigError("world must be >= 1")
    owners = np.zeros(costs.shape, dtype=np.int64)
    for layer in range(costs.shape[0]):
        load = [0] * world
        for h in sorted(range(costs.shape[1]), key=lambda h: (-int(costs[layer, h]), h)):
            r = min(range(world), key=lambda r: (load[r], r))
            owners[layer, h] = r
            load[r] += int(costs[layer, h])
    return owners


def contiguous_owners(layers: int, heads: int, world: int):
    """The owner table of ``head_partition`` (before classification)."""
    import numpy as np

    per = heads // world
    return np.tile(np.arange(heads, dtype=np.int64) // per, (layers, 1))


def rebalance_plan(old_owners, new_owners, rank: int):
    """(keep, send, recv) lists of this rank, each in global (layer, head) order:
    keep = [(l, h)], send = [(l, h, dst)], recv = [(l, h, src)]."""
    keep, send, recv = [], [], []
    L, H = old_owners.shape
    for layer in range(L):
        for h in range(H):
            o, n = int(old_owners[layer, h]), int(new_owners[layer, h])
            if o == rank and n == rank:
                keep.append((layer, h))
            elif o == rank:
                send.append((layer, h, n))
            elif n == rank:
                recv.append((layer, h, o))
    return keep, send, recv


def exchange_frames(sends, recvs, group=None) -> None:
    """Point-to-point moves of frame rows: ``sends`` / ``recvs`` are lists of
    (peer, tensor) in the same global order on both sides of every pair.
    NCCL moves device rows directly (NVLink); gloo stages them through the host."""
    if not sends and not recvs:
        return
    if dist.get_backend(group) != "nccl":
        host_recv = [(peer, torch.empty(t.shape, dtype=t.dtype)) for peer, t in recvs]
        ops = [dist.P2POp(dist.isend, t.contiguous().cpu(), peer, group) for peer, t in sends]
        ops += [dist.P2POp(dist.irecv, h, peer, group) for peer, h in host_recv]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for (_, dst), (_, h) in zip(recvs, host_recv):
            dst.copy_(h)
        return
    ops = [dist.P2POp(dist.isend, t, peer, group) for peer, t in sends]
    ops += [dist.P2POp(dist.irecv, t, peer, group) for peer, t in recvs]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def gather_head_outputs_owned(local: torch.Tensor, owners_layer, group=None) -> torch.Tensor:
    """(n_local, HW, d) of this rank's heads (ascending head index) -> (H, HW, d)
    in global head order, for an arbitrary owner vector (uneven counts are
    padded to the largest block for the all-gather)."""
    world = dist.get_world_size(group)
    owners = [int(o) for o in owners_layer]
    counts = [owners.count(r) for r in range(world)]
    width = max(counts)
    pad = local
    if local.shape[0] < width:
        pad = torch.cat([local, local.new_zeros((width - local.shape[0], *local.shape[1:]))])
    g = _all_gather(pad, group)  # (P, width, HW, d)
    slot = [0] * world
    index = []
    for o in owners:
        index.append(o * width + slot[o])
        slot[o] += 1
    flat = g.reshape(world * width, *g.shape[2:])
    return flat[torch.tensor(index, device=flat.device)]


class FusedHeadGather:
    """Gathered head-output buffers for the fused all-gather.

    Two bf16 [total_heads * HW, d8] buffers per rank in symmetric memory
    (torch.distributed._symmetric_memory: the allocation and the mapping of
    every rank's buffer into every process), used in turns.  The FMHA
    epilogue of each rank stores its heads' rows into its own buffer and, over
    NVLink, into the peers' (df_attn_args.peer_out), so the gather overlaps the
    attention tile by tile and no NCCL all-gather runs.  ``barrier()`` (a
    device-side signal/wait on the stream) orders the peers' stores before
    this rank reads the buffer, then passes the turn to the other buffer: the
    next fused gather's stores go to the buffer a slower rank is not reading.
    The turn advances once per fused gather (not by layer index), so it
    alternates across the end of a denoise iteration whatever the layer count
    (with an odd count, layer L-1 and the next iteration's layer 0 would
    otherwise share a buffer).  Every rank runs the same sequence of fused
    gathers, so the turns agree.
    """

    def __init__(self, rows: int, width: int, group, device):
        import torch.distributed._symmetric_memory as symm

        name = group.group_name if group is not None else dist.group.WORLD.group_name
        self.bufs, self.handles, self.peers = [], [], []
        for _ in range(2):
            t = symm.empty((rows, width), dtype=torch.bfloat16, device=device)
            h = symm.rendezvous(t, name)
            # the tensor may sit at an offset inside the symmetric allocation: map the same offset on every rank
            off = (t.data_ptr() - int(h.buffer_ptrs[h.rank])) // t.element_size()
            view = lambda r: h.get_buffer(r, tuple(t.shape), t.dtype, off).data_ptr()
            if view(h.rank) != t.data_ptr():
                raise ConfigError("symmetric-memory mapping of the gathered output buffer is inconsistent")
            self.bufs.append(t)
            self.handles.append(h)
            self.peers.append([view(r) for r in range(h.world_size) if r != h.rank])
        self.turn = 0

    def current(self) -> torch.Tensor:
        """The buffer the next (or pending) fused gather writes."""
        return self.bufs[self.turn % 2]

    def target(self, layer: int, heads):
        from .engine import OutputTarget

        i = self.turn % 2
        return OutputTarget(self.bufs[i], list(heads), self.peers[i])

    def barrier(self) -> None:
        self.handles[self.turn % 2].barrier(channel=0)
        self.turn += 1
