"""Projection GEMMs around the attention launch.

The reference's model protocol (scenario.py:70-120, driven by
engine.py:418-443) projects the layer input to per-head Q/K/V, wraps K/V of
every head into a FrameBlock that the cache later copies into its ring, and
adds ``mix(outputs)`` back into the residual stream.  ``ProjectedModel`` keeps
that protocol and runs both projections on the tensor cores:

* ``qkv_into`` -> ``df_qkv_project``: one persistent tcgen05 GEMM whose
  epilogue writes Q in the FMHA's layout and K/V straight into each head's
  pending ring slot, so neither the staging copy nor the append copy exists.
* ``mix_into`` -> ``df_out_project``: reads the FMHA output per head (the head
  merge of scenario.py:118 is just its addressing), multiplies by W_o and adds
  into the fp32 residual in the epilogue, also writing the bf16 copy the next
  layer's QKV GEMM reads.

The unfused ``qkv`` / ``mix`` methods use the same kernels, so the model also
drives code written against the plain protocol.
"""

from __future__ import annotations

from typing import Callable, Mapping, Sequence

import numpy as np
import torch

from . import kernels as K
from .errors import ConfigError, ShapeError


class ResidualStream:
    """The layer input ``x`` of one denoise iteration, resident on the device.

    ``f32`` is the master copy the residual adds accumulate into
    (engine.py:443); ``bf16`` is the operand the next QKV projection reads,
    rewritten by the same out-projection epilogue.
    """

    def __init__(self, f32: torch.Tensor, bf16: torch.Tensor | None = None):
        self.f32 = f32
        self.bf16 = f32.to(torch.bfloat16) if bf16 is None else bf16

    def __add__(self, delta) -> "ResidualStream":
        d = delta.f32 if isinstance(delta, ResidualStream) else torch.as_tensor(delta, device=self.f32.device)
        return ResidualStream(self.f32 + d.to(torch.float32))

    def numpy(self) -> np.ndarray:
        return self.f32.double().cpu().numpy()


class ProjectedModel:
    """Reference model protocol with tcgen05 projections (scenario.py:70-120).

    ``weights``: per layer a mapping ``{"q", "k", "v", "o"} -> (D, D)`` in the
    reference's ``x @ W`` convention (``ToyModel.weights``).  ``frames``:
    ``(ar_step, denoise_step) -> (HW, D)`` layer-0 input (``frame_input``).
    Weights are stored transposed and concatenated once, in bf16.
    """

    def __init__(self, weights: Sequence[Mapping[str, object]], frames: Callable[[int, int], object], num_heads: int,
                 head_dim: int, HW: int, device: torch.device | str | None = None):
        if head_dim not in K.SUPPORTED_WIDTHS:
            raise ConfigError(f"fused projections need head_dim 64 or 128, got {head_dim}")
        self.num_heads, self.head_dim, self.HW = num_heads, head_dim, HW
        self.model_dim = num_heads * head_dim
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._frames = frames
        D = self.model_dim
        self.w_qkv: list[torch.Tensor] = []
        self.w_o: list[torch.Tensor] = []
        for w in weights:
            mats = {n: torch.as_tensor(np.asarray(w[n]) if not isinstance(w[n], torch.Tensor) else w[n])
                    for n in ("q", "k", "v", "o")}
            for n, m in mats.items():
                if tuple(m.shape) != (D, D):
                    raise ShapeError(f"weight {n} has shape {tuple(m.shape)}, expected ({D}, {D})")
            wqkv = torch.cat([mats[n].T for n in ("q", "k", "v")], dim=0)
            self.w_qkv.append(wqkv.to(self.device, torch.bfloat16).contiguous())
            self.w_o.append(mats["o"].T.to(self.device, torch.bfloat16).contiguous())
        self._head_slices: dict[tuple[int, int, int], torch.Tensor] = {}

    @property
    def num_layers(self) -> int:
        return len(self.w_qkv)

    # ------------------------------------------------------------ protocol
    def frame_input(self, ar_step: int, denoise_step: int) -> ResidualStream:
        x = self._frames(ar_step, denoise_step)
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        t = t.to(self.device, torch.float32).contiguous()
        if tuple(t.shape) != (self.HW, self.model_dim):
            raise ShapeError(f"frame input {tuple(t.shape)} != ({self.HW}, {self.model_dim})")
        return ResidualStream(t)

    def _w_heads(self, layer: int, heads: Sequence[int]) -> torch.Tensor:
        """W_qkv rows of ``heads`` (any ascending head list: a head-parallel rank's share)."""
        heads = tuple(heads)
        if heads == tuple(range(self.num_heads)):
            return self.w_qkv[layer]
        key = (layer, heads)
        w = self._head_slices.get(key)
        if w is None:
            D, d = self.model_dim, self.head_dim
            rows = [self.w_qkv[layer][j * D + h * d : j * D + (h + 1) * d] for j in range(3) for h in heads]
            w = torch.cat(rows, dim=0).contiguous()
            self._head_slices[key] = w
        return w

    def qkv_into(self, layer: int, x: ResidualStream, ar_step: int, denoise_step: int, q_out: torch.Tensor,
                 k_dst: list[torch.Tensor], v_dst: list[torch.Tensor], heads: Sequence[int] | None = None,
                 stream: torch.cuda.Stream | None = None) -> None:
        """Q of ``heads`` into ``q_out`` (heads, HW, d); their K/V into ``k_dst`` / ``v_dst`` views."""
        heads = range(self.num_heads) if heads is None else heads
        K.prepare_qkv_projection(x.bf16, self._w_heads(layer, heads), q_out, k_dst, v_dst,
                                 self.head_dim).launch(stream)

    def qkv(self, layer: int, x: ResidualStream, ar_step: int, denoise_step: int):
        H, hw, d = self.num_heads, self.HW, self.head_dim
        q = torch.empty(H, hw, d, dtype=torch.bfloat16, device=self.device)
        k = torch.empty_like(q)
        v = torch.empty_like(q)
        self.qkv_into(layer, x, ar_step, denoise_step, q, list(k), list(v))
        return q, k, v

    def mix_into(self, layer: int, outputs: torch.Tensor, x: ResidualStream,
                 stream: torch.cuda.Stream | None = None) -> ResidualStream:
        """``x += merge(outputs) @ W_o`` in place (both copies); returns ``x``."""
        o = outputs if outputs.is_contiguous() else outputs.contiguous()
        K.prepare_out_projection(o, self.w_o[layer], x.f32, x.bf16, self.head_dim).launch(stream)
        return x

    def mix(self, layer: int, outputs: torch.Tensor) -> torch.Tensor:
        delta = torch.zeros(self.HW, self.model_dim, dtype=torch.float32, device=self.device)
        o = outputs if outputs.is_contiguous() else outputs.contiguous()
        K.prepare_out_projection(o, self.w_o[layer], delta, None, self.head_dim).launch(None)
        return delta
