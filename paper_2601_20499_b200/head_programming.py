"""Dynamic head programming: classify every head sink / neighbor / dummy.

Mirrors the reference's head_programming.py:26-164,213-229.  The solver is
``df_greedy_classify`` in libdfb200 (host C++): same lexsort tie rules and the
same numpy pairwise summation for the objective, so classes and objective are
bit-identical to the reference for identical scores.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import AssignmentError, ConfigError

COL_SINK, COL_NEIGHBOR, COL_CURRENT = 0, 1, 2


class HeadClass(str, enum.Enum):
    SINK = "sink"
    NEIGHBOR = "neighbor"
    DUMMY = "dummy"


# integer codes shared with the C ABI (df_greedy_classify) and the oracle
CLASS_CODES = (HeadClass.SINK, HeadClass.NEIGHBOR, HeadClass.DUMMY)
CODE_OF = {c: i for i, c in enumerate(CLASS_CODES)}


@dataclass(frozen=True)
class HeadAssignment:
    """One class per head in flat layer-major order, with exactly N dummies."""

    classes: tuple[HeadClass, ...]
    dummy_count: int

    def __post_init__(self):
        n = sum(c is HeadClass.DUMMY for c in self.classes)
        if n != self.dummy_count:
            raise AssignmentError(f"assignment has {n} dummy heads, expected {self.dummy_count}")

    @property
    def total_heads(self) -> int:
        return len(self.classes)

    def class_of(self, flat_index: int) -> HeadClass:
        return self.classes[flat_index]

    def indices_of(self, head_class: HeadClass) -> list[int]:
        return [i for i, c in enumerate(self.classes) if c is head_class]

    def counts(self) -> dict[str, int]:
        return {hc.value: sum(c is hc for c in self.classes) for hc in HeadClass}

    def per_layer_histogram(self, num_heads: int) -> list[dict[str, int]]:
        if self.total_heads % num_heads:
            raise AssignmentError("total heads not divisible by heads per layer")
        out = []
        for s in range(0, self.total_heads, num_heads):
            layer = self.classes[s : s + num_heads]
            out.append({hc.value: sum(c is hc for c in layer) for hc in HeadClass})
        return out

    def to_records(self, num_heads: int) -> list[dict]:
        return [{"layer": i // num_heads, "head": i % num_heads, "class": c.value} for i, c in enumerate(self.classes)]

    @classmethod
    def from_records(cls, records: list[dict], num_heads: int) -> "HeadAssignment":
        by_flat = {r["layer"] * num_heads + r["head"]: HeadClass(r["class"]) for r in records}
        if sorted(by_flat) != list(range(len(by_flat))):
            raise AssignmentError("records do not cover heads 0..H-1 exactly once")
        ordered = tuple(by_flat[i] for i in range(len(by_flat)))
        return cls(classes=ordered, dummy_count=sum(c is HeadClass.DUMMY for c in ordered))

    def codes(self) -> list[int]:
        return [CODE_OF[c] for c in self.classes]


def _score_array(scores) -> np.ndarray:
    from .profiler import GlobalFrameScore

    if isinstance(scores, GlobalFrameScore):
        a = scores.scores
    else:
        try:
            import torch

            if isinstance(scores, torch.Tensor):
                scores = scores.detach().to("cpu", torch.float64).numpy()
        except ImportError:  # pragma: no cover
            pass
        a = np.asarray(scores, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ConfigError(f"expected an (H, 3) score array, got {a.shape}")
    return np.ascontiguousarray(a, dtype=np.float64)


def value(score_row, head_class: HeadClass) -> float:
    """Mass a head keeps under a class (head_programming.py:112-119)."""
    r = np.asarray(score_row, dtype=np.float64)
    if head_class is HeadClass.SINK:
        return float(r[COL_SINK] + r[COL_CURRENT])
    if head_class is HeadClass.NEIGHBOR:
        return float(r[COL_NEIGHBOR] + r[COL_CURRENT])
    return float(r[COL_CURRENT])


def opportunity_cost(scores) -> np.ndarray:
    """Mass forfeited by making a head dummy: max(sink, neighbor)."""
    a = _score_array(scores)
    return np.maximum(a[:, COL_SINK], a[:, COL_NEIGHBOR])


def greedy_classify(scores, n_dummy: int) -> tuple[HeadAssignment, float]:
    """Optimal assignment with exactly ``n_dummy`` dummy heads (C solver)."""
    a = _score_array(scores)
    total = a.shape[0]
    if not 0 <= n_dummy <= total:
        raise ConfigError(f"n_dummy={n_dummy} outside [0, {total}]")
    codes = (ctypes.c_int8 * max(total, 1))()
    obj = ctypes.c_double(0.0)
    _lib.call(
        "df_greedy_classify",
        a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        ctypes.c_int64(total),
        ctypes.c_int64(n_dummy),
        codes,
        ctypes.byref(obj),
    )
    classes = tuple(CLASS_CODES[codes[i]] for i in range(total))
    return HeadAssignment(classes=classes, dummy_count=n_dummy), float(obj.value)


def classify_session(session, n_dummy: int | None = None, probe=None, subsample_ratio: float | None = None):
    """Profile a session once at the probe step and classify every head."""
    from . import profiler

    if n_dummy is None:
        n_dummy = session.config.dummy_count
    table = profiler.global_scores(session, probe=probe, subsample_ratio=subsample_ratio)
    return greedy_classify(table, n_dummy)
