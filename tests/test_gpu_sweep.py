"""Device port of the reference's sweep command (cli.py:301-343; tests/test_cli.py TestSweep,
tests/test_acceptance.py criterion 7 through the sweep)."""
import csv
import json

import numpy as np
import pytest

from paper_2601_20499_b200 import sweep as S

pytestmark = pytest.mark.gpu
SEC = dict(num_layers=2, num_heads=4, head_dim=8, HW=6, window_len=3, ar_steps=6, denoise_steps=2,
           dummy_count=4, probe_ar_step=2)


def _rows(path):
    return list(csv.DictReader(open(path)))


def test_dummy_ratio_sweep_monotone_accounting(tmp_path):
    base = S.session_config({**SEC, "window_len": 4, "ar_steps": 4})
    out = str(tmp_path / "sweep.csv")
    S.sweep(lambda c: S.RandomStream(c, 42), base, "dummy_ratio", [0.0, 0.5, 1.0], out, reps=3)
    rows = _rows(out)
    assert list(rows[0]) == S.CSV_HEADER
    hma = [r for r in rows if r["mode"] == "hma"]
    ratios = [float(r["cache_reduction_ratio"]) for r in hma]
    assert ratios == sorted(ratios, reverse=True) and len(set(ratios)) == len(ratios)
    for r in rows:
        assert r["key_token_macs"] == r["expected_key_token_macs"]
    full = [r for r in rows if r["mode"] == "hma" and float(r["axis_value"]) == 1.0]
    hw, d, heads = 6, 8, 8
    assert int(full[0]["key_token_macs"]) == heads * hw * (2 * hw) * d


def test_context_len_sweep_macs_grow_linearly(tmp_path):
    out = str(tmp_path / "sweep.csv")
    S.sweep(lambda c: S.RandomStream(c, 42), S.session_config(SEC), "context_len", [4, 5, 6], out, reps=3)
    rows = _rows(out)
    base = {float(r["axis_value"]): int(r["key_token_macs"]) for r in rows if r["mode"] == "baseline"}
    hma = {float(r["axis_value"]): int(r["key_token_macs"]) for r in rows if r["mode"] == "hma"}
    gaps = [base[v] - hma[v] for v in sorted(base)]
    diffs = np.diff(gaps)
    assert gaps[0] > 0 and (diffs > 0).all() and len(set(diffs.tolist())) == 1


def test_criterion7_through_sweep_cli(tmp_path):
    """tests/test_acceptance.py:205-250: hma / packed wall <= baseline at every context length."""
    cfg = {"schema_version": 1, "seed": 11, "model": {"kind": "toy"},
           "session": {"num_layers": 1, "num_heads": 8, "head_dim": 64, "HW": 2048, "window_len": 5, "ar_steps": 6,
                       "denoise_steps": 1, "dummy_fraction": 0.5, "packing": True, "probe_ar_step": 2},
           "timing": {"reps": 5}, "sweep": {"context_len": [5, 9, 15]}}
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    out = tmp_path / "sweep.csv"
    assert S.main(["--config", str(path), "--axis", "context_len", "--out", str(out)]) == 0
    by = {}
    for r in _rows(out):
        by.setdefault(float(r["axis_value"]), {})[r["mode"]] = r
    for v, modes in by.items():
        base_wall = int(modes["baseline"]["wall_time_ns_median"])
        for mode in ("hma", "packed"):
            assert int(modes[mode]["wall_time_ns_median"]) <= base_wall, (v, mode)
            assert modes[mode]["key_token_macs"] == modes[mode]["expected_key_token_macs"]
