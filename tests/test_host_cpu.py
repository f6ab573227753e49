"""CPU-only checks of the host side: C-ABI library, C greedy, policies, accounting."""
import json
import os
import re

import numpy as np
import pytest
import torch

import paper_2601_20499_b200 as df
from paper_2601_20499_b200 import _lib
from paper_2601_20499_b200.kv_cache import RingStorage

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "df_b200.h")).read()
    declared = set(re.findall(r"DF_API\s+(?:const\s+char\s*\*|int)\s+(df_\w+)\s*\(", header))
    assert declared == set(_lib.exported_symbols())
    lib = _lib.load()
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.df_version() == 1


def test_c_greedy_bit_exact_with_reference_goldens():
    z = np.load(os.path.join(G, "greedy.npz"), allow_pickle=True)
    for F, n, codes, obj in zip(z["F"], z["n"], z["codes"], z["objective"]):
        a, got_obj = df.greedy_classify(np.asarray(F, dtype=np.float64), int(n))
        assert [df.head_programming.CODE_OF[c] for c in a.classes] == list(codes)
        assert got_obj == obj  # numpy pairwise summation reproduced bit for bit


def test_c_greedy_objective_matches_numpy_sum_all_sizes():
    rng = np.random.default_rng(5)
    for total in list(range(1, 300)) + [511, 512, 513, 1000, 4096]:
        F = rng.random((total, 3))
        F /= F.sum(axis=1, keepdims=True)
        n = int(rng.integers(0, total + 1))
        a, obj = df.greedy_classify(F, n)
        codes = np.array([df.head_programming.CODE_OF[c] for c in a.classes])
        table = np.stack([F[:, 0] + F[:, 2], F[:, 1] + F[:, 2], F[:, 2]], axis=1)
        assert obj == float(np.sum(table[np.arange(total), codes]))


def test_greedy_rules_and_errors():
    four = np.array([[0.5, 0.2, 0.3], [0.1, 0.15, 0.75], [0.05, 0.6, 0.35], [0.2, 0.1, 0.7]])
    a, obj = df.greedy_classify(four, 2)
    assert a.classes == (df.HeadClass.SINK, df.HeadClass.DUMMY, df.HeadClass.NEIGHBOR, df.HeadClass.DUMMY)
    assert obj == pytest.approx(3.2, abs=1e-12)
    a, _ = df.greedy_classify(np.array([[0.4, 0.4, 0.2]]), 0)
    assert a.classes == (df.HeadClass.SINK,)  # F0 >= F1 -> sink
    a, _ = df.greedy_classify(np.array([[0.4, 0.3, 0.3], [0.4, 0.3, 0.3], [0.5, 0.2, 0.3]]), 1)
    assert a.classes[0] is df.HeadClass.DUMMY and a.classes[1] is not df.HeadClass.DUMMY
    with pytest.raises(df.ConfigError):
        df.greedy_classify(four, 5)
    with pytest.raises(df.ConfigError):
        df.greedy_classify(np.zeros((3, 2)), 1)


def test_config_validation():
    ok = dict(num_layers=1, num_heads=2, head_dim=8, HW=4, window_len=3, ar_steps=2)
    df.SessionConfig(**ok)
    for bad in (dict(window_len=1), dict(ar_steps=0), dict(dummy_count=3), dict(subsample_ratio=0.0),
                dict(merged_window=1), dict(sink_frame=-1), dict(HW=0), dict(denoise_steps=0)):
        with pytest.raises(df.ConfigError):
            df.SessionConfig(**{**ok, **bad})


class _HostArena:
    """Stand-in arena (CPU planes) to drive the ring slot tables without a GPU."""

    def __init__(self, rows, width):
        self.k = torch.zeros(rows, width, dtype=torch.bfloat16)
        self.v = torch.zeros(rows, width, dtype=torch.bfloat16)
        self.width = width
        self.device = torch.device("cpu")


def _ring(policy, hw=4, d=8):
    arena = _HostArena(policy.ring_slots * hw + 128, 64)
    return df.HeadKVCache(policy, storage=RingStorage(arena, 0, policy.ring_slots, hw, d)), arena


def _block(fid, hw=4, d=8):
    return df.FrameBlock(fid, torch.full((hw, d), float(fid)), torch.full((hw, d), -float(fid)))


def test_ring_slot_tables_follow_reference_eviction():
    g = json.load(open(os.path.join(G, "eviction.json")))
    for c in g["policies"]:
        p = df.CachePolicy(c["kind"], c["window_len"], c["sink_frame"], c["extended_window"])
        cache, _ = _ring(p)
        for fid, want in enumerate(c["seq"]):
            cache.append_segments(_block(fid), device=torch.device("cpu"))
            assert cache.frame_ids == want
            occupied = {s for s, f in enumerate(cache._slot_frame) if f is not None}
            # prefix invariant: occupied + pending == [0, len+1)
            assert occupied | {cache.pending_slot} == set(range(len(cache) + 1))
            assert len(cache) <= p.warm_past_frames()


def test_ring_append_segments_and_staging_skip():
    p = df.CachePolicy("baseline_window", 3)
    cache, arena = _ring(p)
    b0 = _block(0)
    segs = cache.stage_segments(b0, torch.device("cpu"))
    assert len(segs) == 2  # K and V
    assert cache.append_segments(b0, device=torch.device("cpu")) == []  # staged: slot-table update only
    b1 = _block(1)
    segs = cache.append_segments(b1, device=torch.device("cpu"))
    assert len(segs) == 2 and segs[0][2] == 4 and segs[0][5] == 16  # 4 rows of 8 bf16
    with pytest.raises(df.OrderingError):
        cache.append_segments(_block(1), device=torch.device("cpu"))
    with pytest.raises(df.OrderingError):
        cache.stage_segments(_block(0), torch.device("cpu"))


def test_region_codes_label_sink_neighbor_current():
    p = df.CachePolicy("baseline_window", 4)
    cache, _ = _ring(p)
    for fid in range(6):
        cache.append_segments(_block(fid), device=torch.device("cpu"))
    codes = cache.region_codes()
    pend = cache.pending_slot
    for s, f in enumerate(cache._slot_frame):
        want = 2 if s == pend else (0 if f == 0 else 1)
        assert codes[s] == want


def test_policies_accounting_against_reference_goldens():
    g = json.load(open(os.path.join(G, "accounting.json")))
    C = [df.HeadClass.SINK, df.HeadClass.NEIGHBOR, df.HeadClass.DUMMY]
    for r in g["macs"]:
        cfg = df.SessionConfig(**r["cfg"])
        a = df.HeadAssignment(tuple(C[c] for c in r["codes"]), sum(c == 2 for c in r["codes"]))
        assert df.expected_step_macs(cfg, "baseline", r["history"]) == r["baseline"]
        assert df.expected_step_macs(cfg, "hma", r["history"], a) == r["hma"]
        assert df.expected_step_macs(cfg, "packed", r["history"], a) == r["packed"]
    for r in g["extension"]:
        a = df.HeadAssignment(tuple(C[c] for c in r["codes"]), sum(c == 2 for c in r["codes"]))
        assert df.extension_window(a, df.SessionConfig(**r["cfg"])) == r["ext"]
    for r in g["ratio"]:
        a = df.HeadAssignment(tuple(C[c] for c in r["codes"]), sum(c == 2 for c in r["codes"]))
        assert df.cache_stats(a, df.SessionConfig(**r["cfg"])).reduction_ratio == r["ratio"]
    for r in g["subsample"]:
        assert df.subsample_rows(r["n"], r["ratio"]).tolist() == r["rows"]


def test_paper_cache_identities():
    # 27.8% / 16.7% (tests/test_kv_cache.py:199-220 of the reference)
    cfg = df.SessionConfig(num_layers=1, num_heads=360, head_dim=3, HW=4, window_len=9, ar_steps=10,
                           dummy_count=180, packing_enabled=True, merged_window=4)
    classes = tuple([df.HeadClass.DUMMY] * 180 + [df.HeadClass.SINK] * 90 + [df.HeadClass.NEIGHBOR] * 90)
    assert df.cache_stats(df.HeadAssignment(classes, 180), cfg).reduction_ratio == pytest.approx(0.2778, abs=1e-4)
    assert df.uniform_budget_ratio(1.5, 9) == pytest.approx(0.1667, abs=1e-4)


def test_rebuild_without_storage_replays_ids():
    p = df.CachePolicy("baseline_window", 6)
    c = df.HeadKVCache(p)
    assert c.frame_ids == [] and len(c) == 0
    [n] = df.rebuild_caches([c], [df.CachePolicy("sink_only", 6)])
    assert n.frame_ids == []


def test_layout_and_scores_helpers():
    lay = df.FrameLayout.from_frame_kinds(4, ["sink", "neighbor", "neighbor", "current"])
    assert [r.kind for r in lay.regions] == ["sink", "neighbor", "current"]
    uniform = np.full((4, 16), 1 / 16)
    s = df.frame_attention_scores(uniform, lay)
    assert (s.alpha_sink, s.alpha_neighbor, s.alpha_current) == (0.25, 0.5, 0.25)
    with pytest.raises(df.ShapeError):
        df.frame_attention_scores(np.full((2, 8), 1 / 8), lay)


def test_container_byte_compatible_with_reference(tmp_path):
    from paper_2601_20499_b200 import container as C

    g = os.path.join(G, "ref_container.dfc")
    t = C.load_tensors(g)  # written by the reference's save_tensors
    assert set(t) == {"layer0/head0/frame0/keys", "layer0/head0/frame0/values", "scalar"}
    assert t["layer0/head0/frame0/keys"].dtype == np.float32 and t["scalar"].shape == (1,)  # as the reference writes 0-d
    want = json.load(open(os.path.join(G, "ref_container.json")))["digest"]
    assert C.array_digest(*t.values()) == want
    out = tmp_path / "re.dfc"
    C.save_tensors(str(out), t)
    assert open(out, "rb").read() == open(g, "rb").read()  # byte-identical rewrite
    # bf16 tensors widen exactly to f32
    x = torch.randn(3, 5).to(torch.bfloat16)
    C.save_tensors(str(out), {"x": x})
    np.testing.assert_array_equal(C.load_tensors(str(out))["x"], x.float().numpy())
    with pytest.raises(df.ConfigError):
        bad = tmp_path / "bad.dfc"
        bad.write_bytes(b"\x01")
        C.load_tensors(str(bad))


def test_sweep_axis_rules_follow_reference_cli():
    """cli.py:128-145 / 260-298 restated in paper_2601_20499_b200.sweep (no GPU needed)."""
    from paper_2601_20499_b200 import sweep as S

    sec = dict(num_layers=2, num_heads=4, head_dim=8, HW=6, window_len=3, ar_steps=6, denoise_steps=2,
               dummy_count=4, probe_ar_step=2)
    base = S.session_config(sec)
    pts = S.axis_configs(base, "context_len", [4, 5])
    assert [v for v, _ in pts] == [4.0, 5.0]
    assert [(c.window_len, c.ar_steps) for _, c in pts] == [(3, 3), (4, 4)]
    base4 = S.session_config({**sec, "window_len": 4, "ar_steps": 4})
    pts = S.axis_configs(base4, "dummy_ratio", [0.0, 0.5, 1.0])
    assert [c.dummy_count for _, c in pts] == [0, 4, 8] and all(c.ar_steps == 4 for _, c in pts)
    assert S.axis_configs(base, "context_len", [4], HW=10)[0][1].HW == 10
    frac = S.session_config({k: v for k, v in sec.items() if k != "dummy_count"} | {"dummy_fraction": 0.5})
    assert frac.dummy_count == 4 and frac.packing_enabled
    for bad in (lambda: S.axis_configs(base, "context_len", [3]),           # window < probe room
                lambda: S.axis_configs(base, "context_len", [2]),           # < 3 frames
                lambda: S.axis_configs(S.session_config({**sec, "window_len": 2}), "dummy_ratio", [0.5]),
                lambda: S.axis_configs(base4, "dummy_ratio", [1.5]),
                lambda: S.axis_configs(base, "context_len", []),
                lambda: S.axis_configs(base, "heads", [1]),
                lambda: S.session_config({**sec, "dummy_fraction": 0.5}),   # both count and fraction
                lambda: S.session_config({"num_layers": 1}),
                lambda: S.session_config({**sec, "bogus": 1})):
        with pytest.raises(df.ConfigError):
            bad()


def test_sweep_cli_config_errors(tmp_path):
    from paper_2601_20499_b200 import sweep as S

    assert S.main(["--config", str(tmp_path / "missing.json"), "--axis", "context_len", "--out", "x.csv"]) == 2
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"schema_version": 2, "session": {}}))
    assert S.main(["--config", str(p), "--axis", "context_len", "--out", str(tmp_path / "o.csv")]) == 1


def test_batched_step_request_checks_on_host():
    """batched_step's per-request checks are the single-request step functions' (engine.py:140-195):
    policy kind for baseline, class count, packing switch, unknown mode -- raised before any launch."""
    from paper_2601_20499_b200 import engine

    cfg = df.SessionConfig(num_layers=1, num_heads=2, head_dim=64, HW=8, window_len=4, ar_steps=5, dummy_count=1)
    base = [df.HeadKVCache(df.baseline_policy(cfg)) for _ in range(2)]
    classes = [df.HeadClass.DUMMY, df.HeadClass.NEIGHBOR]
    pruned = [df.HeadKVCache(df.derive_policy(c, cfg)) for c in classes]
    assert engine._request_groups(df.StepRequest("baseline", None, base, []), cfg) == [[0, 1]]
    assert engine._request_groups(df.StepRequest("packed", None, pruned, [], classes), cfg) == [[0], [1]]
    assert len(engine._request_groups(df.StepRequest("hma", None, pruned, [], classes), cfg)) == 3
    with pytest.raises(df.ConfigError):
        engine._request_groups(df.StepRequest("baseline", None, pruned, []), cfg)
    with pytest.raises(df.AssignmentError):
        engine._request_groups(df.StepRequest("packed", None, pruned, [], classes[:1]), cfg)
    with pytest.raises(df.ConfigError):
        engine._request_groups(df.StepRequest("bogus", None, pruned, [], classes), cfg)
    nopack = df.SessionConfig(**{**cfg.__dict__, "packing_enabled": False})
    with pytest.raises(df.ConfigError):
        engine._request_groups(df.StepRequest("packed", None, pruned, [], classes), nopack)
    with pytest.raises(df.ShapeError):
        df.batched_step([], cfg)


def test_overlapped_copy_only_inside_a_chain_and_when_disjoint(monkeypatch):
    """df_kv_append_overlapped (programmatic dependent launch) runs only through a LaunchChain whose
    last df_attn_fwd on the same stream touches none of the bytes the copy writes and writes none
    it reads; without a chain (the public default) the copy is always the serialised df_kv_append."""
    from paper_2601_20499_b200 import kernels as K

    calls = []
    monkeypatch.setattr(_lib, "call", lambda fn, *a: calls.append(fn))

    class _S:
        def __init__(self, h):
            self.cuda_stream = h

    s, s2 = _S(0x5EED), _S(0x5EEE)
    fmha = K.PreparedLaunch("df_attn_fwd", (), (), touched=[(1000, 2000), (5000, 6000)], written=[(5000, 6000)])
    other = K.PreparedLaunch("df_out_project", (), ())

    def copy(src, dst, rows=4, ld=64, nbytes=64):
        return K.prepare_copies([(src, dst, rows, ld, ld, nbytes)], overlapped=True)[0]

    chain = K.LaunchChain()
    copy(10_000, 20_000).launch(s, chain)  # no FMHA launched through the chain yet
    fmha.launch(s, chain)
    copy(10_000, 20_000).launch(s, chain)  # disjoint
    copy(10_000, 20_000).launch(s)  # disjoint, but no chain: plain
    copy(10_000, 20_000).launch(s2, chain)  # the chain's FMHA ran on another stream: plain
    copy(10_000, 1900).launch(s, chain)  # writes into bytes the FMHA reads
    copy(5900, 20_000).launch(s, chain)  # reads bytes the FMHA writes
    copy(1000, 20_000).launch(s, chain)  # reads what the FMHA reads: fine
    copy(10_000, 2000).launch(s, chain)  # [2000, 2256): adjacent, disjoint
    copy(10_000, 4800, rows=4, ld=64, nbytes=64).launch(s, chain)  # [4800, 5056) overlaps [5000, 6000)
    other.launch(s, chain)  # any other library launch ends the pairing
    copy(10_000, 20_000).launch(s, chain)
    p, o = "df_kv_append", "df_kv_append_overlapped"
    assert calls == [p, "df_attn_fwd", o, p, p, p, p, o, o, p, "df_out_project", p]
    assert K._merge([(5, 9), (0, 3), (3, 4), (8, 12)]) == ([0, 5], [4, 12])
