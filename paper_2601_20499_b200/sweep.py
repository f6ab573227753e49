"""Context-length / dummy-ratio sweeps on the device.

Port of the reference's ``cmd_sweep`` (cli.py:301-343) with the same axis
rules (``_axis_configs``, cli.py:260-298), the same session-section parsing
(cli.py:128-145: ``dummy_count`` XOR ``dummy_fraction``, ``packing``) and the
same CSV columns.  Every point warms a device ``Session`` through all of its
AR steps, then times the next step's final denoise iteration with CUDA events
(``Session.time_step``).

The reference builds its toy / planted workloads from its own counter PRNG;
those stay on the oracle side (``oracle/``).  Here the model comes from the
caller (``model_factory(config) -> model``); the command line uses
``RandomStream`` -- seeded device Q/K/V, open loop -- which is all a timing
sweep needs.

    python -m paper_2601_20499_b200.sweep --config cfg.json --axis context_len --out sweep.csv
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys
from typing import Callable

import torch

from .config import SessionConfig
from .container import write_atomic
from .engine import MODES, Session, expected_step_macs
from .errors import ConfigError
from .kv_cache import cache_stats

CSV_HEADER = ["axis", "axis_value", "mode", "key_token_macs", "expected_key_token_macs", "kernel_calls",
              "wall_time_ns_median", "cache_reduction_ratio"]
AXES = ("context_len", "dummy_ratio")
_SESSION_KEYS = {"num_layers", "num_heads", "head_dim", "HW", "window_len", "ar_steps", "denoise_steps",
                 "sink_frame", "dummy_count", "dummy_fraction", "packing", "merged_window", "context_extension",
                 "probe_ar_step", "probe_denoise_step", "subsample_ratio"}
_SWEEP_KEYS = {"context_len", "dummy_ratio", "HW"}


def session_config(section: dict) -> SessionConfig:
    """cli.py:128-145: the session section of a run config -> SessionConfig."""
    unknown = set(section) - _SESSION_KEYS
    if unknown:
        raise ConfigError(f"unknown session fields: {sorted(unknown)}")
    missing = [k for k in ("num_layers", "num_heads", "head_dim", "HW", "window_len", "ar_steps") if k not in section]
    if missing:
        raise ConfigError(f"session is missing fields: {missing}")
    section = dict(section)
    fraction = section.pop("dummy_fraction", None)
    packing = section.pop("packing", True)
    if fraction is not None:
        if "dummy_count" in section:
            raise ConfigError("set either dummy_count or dummy_fraction, not both")
        section["dummy_count"] = int(section["num_layers"] * section["num_heads"] * float(fraction))
    try:
        return SessionConfig(packing_enabled=bool(packing), **section)
    except TypeError as e:
        raise ConfigError(f"bad session section: {e}") from e


def axis_configs(base: SessionConfig, axis: str, values, HW: int | None = None) -> list[tuple[float, SessionConfig]]:
    """cli.py:260-298: one SessionConfig per sweep point."""
    b = base.to_dict()
    if HW:
        b["HW"] = int(HW)
    out = []
    if axis == "context_len":
        if not values:
            raise ConfigError("sweep.context_len missing from config")
        for v in values:
            v = int(v)
            window = v - 1
            if window < 2:
                raise ConfigError(f"context_len {v} too small (needs >= 3 frames)")
            if window <= b["probe_ar_step"]:
                raise ConfigError(f"context_len {v} leaves no room for probe step {b['probe_ar_step']}")
            out.append((float(v), SessionConfig(**dict(b, window_len=window, ar_steps=window))))
        return out
    if axis == "dummy_ratio":
        if not values:
            raise ConfigError("sweep.dummy_ratio missing from config")
        if b["probe_ar_step"] >= b["window_len"]:
            raise ConfigError("dummy_ratio sweep needs probe_ar_step < window_len so heads are classified "
                              "before the timed warm step")
        total = b["num_layers"] * b["num_heads"]
        for r in values:
            r = float(r)
            if not 0.0 <= r <= 1.0:
                raise ConfigError(f"dummy_ratio {r} outside [0, 1]")
            out.append((r, SessionConfig(**dict(b, dummy_count=int(round(r * total)), ar_steps=b["window_len"]))))
        return out
    raise ConfigError(f"unknown sweep axis {axis!r}")


def sweep(model_factory: Callable[[SessionConfig], object], base: SessionConfig, axis: str, values,
          out_csv: str | None = None, reps: int = 5, HW: int | None = None) -> list[list]:
    """cli.py:301-343 on the device: rows of CSV_HEADER (written atomically to ``out_csv``)."""
    rows = []
    for value, cfg in axis_configs(base, axis, values, HW):
        history = cfg.ar_steps  # frames cached before the timed step
        for mode in MODES:
            session = Session(model_factory(cfg), cfg, mode)
            session.run()
            timing = session.time_step(reps=reps)
            expected = expected_step_macs(cfg, session._effective_mode(), history, session.assignment)
            ratio = cache_stats(session.assignment, cfg).reduction_ratio if session.assignment is not None else 1.0
            rows.append([axis, f"{value:g}", mode, timing["key_token_macs"], expected,
                         sum(timing["kernel_calls_per_layer"]), timing["wall_time_ns_median"], f"{ratio:.10g}"])
    if out_csv is not None:
        buf = io.StringIO()
        w = csv.writer(buf)
        w.writerow(CSV_HEADER)
        w.writerows(rows)
        write_atomic(out_csv, buf.getvalue().encode("utf-8"))
    return rows


class RandomStream:
    """Open-loop model protocol with seeded device Q/K/V (N(0, 1), bf16) per (layer, ar, denoise)."""

    def __init__(self, config: SessionConfig, seed: int = 0, device=None):
        self.config, self.seed = config, seed
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def frame_input(self, ar_step: int, denoise_step: int):
        return None

    def qkv(self, layer: int, x, ar_step: int, denoise_step: int):
        c = self.config
        g = torch.Generator(device=self.device)
        g.manual_seed((((self.seed * 1_000_003 + layer) * 1_000_003 + ar_step) * 1_000_003 + denoise_step) % (1 << 62))
        shape = (3, c.num_heads, c.HW, c.head_dim)
        qkv = torch.randn(shape, generator=g, device=self.device).to(torch.bfloat16)
        return qkv[0], qkv[1], qkv[2]

    def mix(self, layer: int, outputs):
        return None


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2601_20499_b200.sweep", description=__doc__.split("\n")[0])
    ap.add_argument("--config", required=True, help="reference-format run config (JSON, schema_version 1)")
    ap.add_argument("--axis", required=True, choices=AXES)
    ap.add_argument("--out", required=True, help="CSV path")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--reps", type=int, default=None)
    args = ap.parse_args(argv)
    try:
        raw = json.load(open(args.config))
    except (OSError, json.JSONDecodeError) as e:
        print(f"error: cannot read config: {e}", file=sys.stderr)
        return 2
    try:
        if raw.get("schema_version") != 1:
            raise ConfigError(f"schema_version must be 1, got {raw.get('schema_version')!r}")
        base = session_config(dict(raw.get("session") or {}))
        sw = dict(raw.get("sweep") or {})
        unknown = set(sw) - _SWEEP_KEYS
        if unknown:
            raise ConfigError(f"unknown sweep fields: {sorted(unknown)}")
        reps = args.reps or int((raw.get("timing") or {}).get("reps", 5))
        seed = args.seed if args.seed is not None else int(raw.get("seed", 0))
        sweep(lambda cfg: RandomStream(cfg, seed), base, args.axis, sw.get(args.axis), args.out, reps, sw.get("HW"))
    except ConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
