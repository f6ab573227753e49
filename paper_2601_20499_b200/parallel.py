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
    out = torch.empty((world, *t.shape), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t, group=group)
    else:  # gloo (CPU tests)
        dist.all_gather(list(out.unbind(0)), t, group=group)
    return out


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
    """A Session whose heads are sharded over the ranks of ``group``."""

    def __init__(self, model, config: SessionConfig, mode: str = "baseline", group=None, **kw):
        if not dist.is_initialized():
            raise ConfigError("HeadParallelSession needs torch.distributed to be initialised")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        head_partition(config.num_heads, self.world, self.rank)  # validates divisibility
        super().__init__(model, config, mode, **kw)

    def _owned_heads(self) -> range:
        return head_partition(self.config.num_heads, self.world, self.rank)

    def _gather_outputs(self, layer: int, outputs: torch.Tensor) -> torch.Tensor:
        return gather_head_outputs(outputs, self.group)

    def _gather_scores(self, local: torch.Tensor) -> torch.Tensor:
        return gather_head_scores(local, self.group)
