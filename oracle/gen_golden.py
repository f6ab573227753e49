"""Generate tests/golden/* from the REFERENCE implementation itself.

Run here (the container that has /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py
The reference is imported read-only from /root/reference/pkg/src; nothing is
copied.  Outputs are small JSON/NPZ fixtures the CPU suite pins the oracle
against (tests/test_oracle_golden.py) and the GPU suite checks the device
path against (tests/test_gpu_parity.py).  Operands are bf16-exact values
built with oracle.df_oracle.case_tensor so the device sees identical inputs.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import dummy_forcing as ref  # noqa: E402
from dummy_forcing import engine as ref_engine  # noqa: E402
from dummy_forcing import head_programming as ref_hp  # noqa: E402
from dummy_forcing import kv_cache as ref_kv  # noqa: E402
from dummy_forcing import profiler as ref_prof  # noqa: E402
from dummy_forcing import rng as ref_rng  # noqa: E402
from dummy_forcing.scenario import PlantedSpec, planted_stream  # noqa: E402

from oracle.df_oracle import case_tensor  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
CLS = {"sink": ref.HeadClass.SINK, "neighbor": ref.HeadClass.NEIGHBOR, "dummy": ref.HeadClass.DUMMY}
CODE = {ref.HeadClass.SINK: 0, ref.HeadClass.NEIGHBOR: 1, ref.HeadClass.DUMMY: 2}


def gen_rng():
    out = {
        "derive": [[7, "toy-model", [], ref_rng.derive(7, "toy-model")],
                   [42, "planted", [], ref_rng.derive(42, "planted")],
                   [3, "q", [1, 2, 3, 4], ref_rng.derive(3, "q", 1, 2, 3, 4)]],
        "uniform": ref_rng.uniform(ref_rng.derive(11, "u"), 16).tolist(),
        "matrix": ref_rng.matrix(ref_rng.derive(5, "m", 2), 3, 4, 0.5).tolist(),
    }
    json.dump(out, open(os.path.join(OUT, "rng.json"), "w"))


def gen_greedy():
    rng = np.random.default_rng(2601)
    Fs, ns, codes, objs = [], [], [], []
    sizes = list(range(1, 41)) + [64, 100, 127, 128, 129, 200, 255, 256, 257, 360, 361, 500]
    for total in sizes:
        for rep in range(3):
            F = rng.random((total, 3)) + 1e-9
            if rep == 1 and total > 2:  # exact ties in cost and in sink/neighbor
                F[1] = F[0]
                F[2, 1] = F[2, 0]
            F = F / F.sum(axis=1, keepdims=True)
            n = int(rng.integers(0, total + 1))
            a, obj = ref_hp.greedy_classify(F, n)
            Fs.append(F)
            ns.append(n)
            codes.append([CODE[c] for c in a.classes])
            objs.append(obj)
    np.savez_compressed(
        os.path.join(OUT, "greedy.npz"),
        F=np.array(Fs, dtype=object), n=np.array(ns), codes=np.array(codes, dtype=object),
        objective=np.array(objs), allow_pickle=True,
    )
    four = np.array([[0.5, 0.2, 0.3], [0.1, 0.15, 0.75], [0.05, 0.6, 0.35], [0.2, 0.1, 0.7]])
    known = []
    for n in range(5):
        a, obj = ref_hp.greedy_classify(four, n)
        known.append({"n": n, "codes": [CODE[c] for c in a.classes], "objective": obj})
    json.dump({"F": four.tolist(), "cases": known}, open(os.path.join(OUT, "greedy_known.json"), "w"))


def gen_eviction():
    pols = [
        ("baseline_window", 4, 0, None), ("baseline_window", 6, 0, None), ("baseline_window", 3, 5, None),
        ("sink_only", 4, 0, None), ("sink_only", 4, 2, None), ("neighbor_window", 3, 0, None),
        ("neighbor_window", 6, 0, None), ("neighbor_window", 4, 0, 6), ("neighbor_window", 6, 0, 21),
        ("dummy_empty", 4, 0, None), ("dummy_packed", 4, 0, None),
    ]
    cases = []
    for kind, w, sink, ext in pols:
        p = ref_kv.CachePolicy(kind, w, sink_frame=sink, extended_window=ext)
        c = ref_kv.HeadKVCache(p)
        seq = []
        for fid in range(15):
            c.append_and_evict(ref_kv.FrameBlock(fid, np.zeros((1, 1)), np.zeros((1, 1))))
            seq.append(list(c.frame_ids))
        cases.append({"kind": kind, "window_len": w, "sink_frame": sink, "extended_window": ext, "seq": seq})
    # classification-time rebuild from a baseline history (kv_cache.py:199-201)
    rebuilds = []
    for w, hist, sink in [(6, 3, 0), (6, 7, 0), (6, 12, 0), (4, 9, 0), (3, 8, 5)]:
        base = ref_kv.HeadKVCache(ref_kv.CachePolicy("baseline_window", w, sink_frame=sink))
        for fid in range(hist):
            base.append_and_evict(ref_kv.FrameBlock(fid, np.zeros((1, 1)), np.zeros((1, 1))))
        for kind, ext in [("sink_only", None), ("neighbor_window", None), ("neighbor_window", 2 * w),
                          ("dummy_packed", None), ("dummy_empty", None)]:
            nb = base.rebuild(ref_kv.CachePolicy(kind, w, sink_frame=sink, extended_window=ext))
            rebuilds.append({"window_len": w, "history": hist, "sink_frame": sink, "kind": kind,
                             "extended_window": ext, "before": base.frame_ids, "after": nb.frame_ids})
    # the SURVEY 8(c) P2 table: W=6, probe at step 2, classes sink/neighbor/dummy
    cfg = ref.SessionConfig(num_layers=1, num_heads=3, head_dim=1, HW=1, window_len=6, ar_steps=10,
                            dummy_count=1, probe_ar_step=2)
    caches = [ref_kv.HeadKVCache(ref_kv.baseline_policy(cfg)) for _ in range(3)]
    classes = [ref.HeadClass.SINK, ref.HeadClass.NEIGHBOR, ref.HeadClass.DUMMY]
    ctx = []
    for step in range(10):
        ctx.append([c.frame_ids + [step] for c in caches])
        if step == 2:
            caches = [c.rebuild(ref_kv.derive_policy(k, cfg)) for c, k in zip(caches, classes)]
        for c in caches:
            c.append_and_evict(ref_kv.FrameBlock(step, np.zeros((1, 1)), np.zeros((1, 1))))
    json.dump({"policies": cases, "rebuilds": rebuilds, "p2_table": ctx},
              open(os.path.join(OUT, "eviction.json"), "w"))


ATTN_CASES = [
    # name, H, HW, d, W, history, classes, packing, q_scale
    ("warm_hw128_d64", 4, 128, 64, 4, 5, ["sink", "neighbor", "dummy", "dummy"], True, 3.0),
    ("warm_hw192_d64", 4, 192, 64, 6, 7, ["neighbor", "dummy", "sink", "neighbor"], True, 3.0),
    ("cold_hw160_d128", 3, 160, 128, 3, 2, ["dummy", "neighbor", "sink"], True, 4.0),
    ("warm_hw200_d128_sharp", 6, 200, 128, 4, 6, ["sink", "sink", "neighbor", "dummy", "neighbor", "dummy"], True, 8.0),
    ("unpacked_hw64_d64", 4, 64, 64, 5, 6, ["dummy", "sink", "neighbor", "dummy"], False, 3.0),
    ("planted_like_hw8_d32", 8, 8, 32, 4, 5, ["sink", "neighbor", "dummy", "dummy", "neighbor", "sink", "dummy", "neighbor"], True, 3.0),
    ("first_step_hw96_d64", 2, 96, 64, 4, 0, ["sink", "neighbor"], True, 3.0),
]


def attn_operands(seed, H, HW, d, history, q_scale):
    q = np.stack([case_tensor(seed, "q", h, rows=HW, cols=d, scale=q_scale) for h in range(H)])
    k = {(h, f): case_tensor(seed, "k", h, f, rows=HW, cols=d) for h in range(H) for f in range(history + 1)}
    v = {(h, f): case_tensor(seed, "v", h, f, rows=HW, cols=d) for h in range(H) for f in range(history + 1)}
    return q, k, v


def gen_attention():
    meta, arrays = [], {}
    for ci, (name, H, HW, d, W, hist, classes, packing, qs) in enumerate(ATTN_CASES):
        seed = 1000 + ci
        cfg = ref.SessionConfig(num_layers=1, num_heads=H, head_dim=d, HW=HW, window_len=W,
                                ar_steps=hist + 1, packing_enabled=packing)
        q, k, v = attn_operands(seed, H, HW, d, hist, qs)
        base = []
        for h in range(H):
            c = ref_kv.HeadKVCache(ref_kv.baseline_policy(cfg))
            for f in range(hist):
                c.append_and_evict(ref_kv.FrameBlock(f, k[(h, f)], v[(h, f)]))
            base.append(c)
        cur = [ref_kv.FrameBlock(hist, k[(h, hist)], v[(h, hist)]) for h in range(H)]
        cls = [CLS[c] for c in classes]
        rec = {"name": name, "H": H, "HW": HW, "d": d, "W": W, "history": hist, "classes": classes,
               "packing": packing, "q_scale": qs, "seed": seed, "modes": {}}
        o, lc = ref_engine.baseline_step(q, base, cur, cfg)
        arrays[f"{name}/baseline"] = o.astype(np.float32)
        rec["modes"]["baseline"] = {"kernel_calls": lc.kernel_calls, "key_token_macs": lc.key_token_macs,
                                    "frames": [c.frame_ids + [hist] for c in base]}
        pruned = [c.rebuild(ref_kv.derive_policy(x, cfg)) for c, x in zip(base, cls)]
        o, lc = ref_engine.hma_step(q, pruned, cur, cls, cfg)
        arrays[f"{name}/hma"] = o.astype(np.float32)
        rec["modes"]["hma"] = {"kernel_calls": lc.kernel_calls, "key_token_macs": lc.key_token_macs,
                               "frames": [c.frame_ids + [hist] for c in pruned]}
        if packing:
            o, lc = ref_engine.packed_step(q, pruned, cur, cls, cfg)
            arrays[f"{name}/packed"] = o.astype(np.float32)
            rec["modes"]["packed"] = {"kernel_calls": lc.kernel_calls, "key_token_macs": lc.key_token_macs,
                                      "frames": [c.frame_ids + [hist] for c in pruned]}
        meta.append(rec)
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **arrays)
    json.dump(meta, open(os.path.join(OUT, "attention.json"), "w"), indent=1)


def gen_planted_sessions():
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import planted_setup  # reference fixture helper (read-only import)

    out = []
    for seed in range(6):
        for ratio in (1.0, 0.25):
            for mode in ("hma", "packed"):
                cfg, spec = planted_setup(seed, margin=2.0, subsample_ratio=ratio)
                cfg = ref.SessionConfig(**{**cfg.to_dict(), "ar_steps": 6})
                s = ref.Session(planted_stream(spec, cfg), cfg, mode)
                frames, rep = s.run()
                table = ref_prof.global_scores(
                    ref.Session(planted_stream(spec, cfg), cfg, "baseline"), subsample_ratio=ratio)
                out.append({
                    "seed": seed, "ratio": ratio, "mode": mode, "labels": list(spec.labels),
                    "noise_seed": spec.noise_seed, "config": cfg.to_dict(),
                    "F": table.scores.tolist(),
                    "classes": [CODE[c] for c in s.assignment.classes],
                    "objective": s.objective,
                    "cache_reduction_ratio": rep.cache_reduction_ratio,
                    "kernel_calls_steady": rep.kernel_calls_steady,
                    "step_macs": [st["key_token_macs"] for st in rep.steps],
                    "frame_ids": [[c.frame_ids for c in layer] for layer in s.caches],
                })
    json.dump(out, open(os.path.join(OUT, "planted_sessions.json"), "w"))


def gen_extension_sessions():
    """Planted sessions with the enlarged-context policies (BASELINE configs[4]; kv_cache.py:104-158,
    engine.py:390-405): context_extension (hma, packed), merged_window (hma) and both (hma).  Per AR
    step the final denoise iteration's context frame list of every (layer, head) is recorded through
    the reference's observer (engine.py:73-84), with the extension window, MACs, ratio, F, classes."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import planted_setup  # reference fixture helper (read-only import)

    variants = [("hma", {"context_extension": True}), ("packed", {"context_extension": True}),
                ("hma", {"merged_window": 5}), ("hma", {"merged_window": 3, "context_extension": True})]
    out = []
    for seed in range(3):
        for ratio in (1.0, 0.25):
            for mode, extra in variants:
                cfg, spec = planted_setup(seed, margin=2.0, subsample_ratio=ratio)
                cfg = ref.SessionConfig(**{**cfg.to_dict(), "ar_steps": 12, **extra})
                frames_seen = {}

                def observer(tr, frames_seen=frames_seen, cfg=cfg):
                    if tr.denoise_step == cfg.denoise_steps - 1:
                        frames_seen.setdefault(tr.ar_step, {})[tr.layer] = [list(c[3]) for c in tr.contexts]

                s = ref.Session(planted_stream(spec, cfg), cfg, mode, observer=observer)
                frames, rep = s.run()
                table = ref_prof.global_scores(
                    ref.Session(planted_stream(spec, cfg), cfg, "baseline"), subsample_ratio=ratio)
                ext = ref_kv.extension_window(s.assignment, cfg) if cfg.context_extension else None
                out.append({
                    "seed": seed, "ratio": ratio, "mode": mode, "labels": list(spec.labels),
                    "noise_seed": spec.noise_seed, "config": cfg.to_dict(),
                    "F": table.scores.tolist(),
                    "classes": [CODE[c] for c in s.assignment.classes],
                    "objective": s.objective,
                    "extension_window": ext,
                    "cache_reduction_ratio": rep.cache_reduction_ratio,
                    "kernel_calls_steady": rep.kernel_calls_steady,
                    "step_macs": [st["key_token_macs"] for st in rep.steps],
                    "context_frames": [[frames_seen[a][l] for l in range(cfg.num_layers)]
                                       for a in range(cfg.ar_steps)],
                    "frame_ids": [[c.frame_ids for c in layer] for layer in s.caches],
                    "output_digest": rep.to_dict()["output_digest"],
                })
    json.dump(out, open(os.path.join(OUT, "extension_sessions.json"), "w"))


def gen_accounting():
    out = {"macs": [], "subsample": [], "extension": [], "ratio": []}
    for (L, H, d, HW, W, sink), hist in [((2, 4, 64, 192, 6, 0), h) for h in range(0, 9)] + \
            [((30, 12, 128, 4680, 6, 0), h) for h in (0, 1, 3, 6, 7, 20)] + [((1, 5, 4, 3, 3, 2), h) for h in range(6)]:
        cfg = ref.SessionConfig(num_layers=L, num_heads=H, head_dim=d, HW=HW, window_len=W, ar_steps=40,
                                sink_frame=sink, dummy_count=H * L // 2, context_extension=(hist % 2 == 1))
        rng = np.random.default_rng(hist + 17 * L)
        codes = rng.permutation(([2] * (L * H // 2)) + [0] * (L * H // 4) + [1] * (L * H - L * H // 2 - L * H // 4))
        a = ref.HeadAssignment(tuple([ref.HeadClass.SINK, ref.HeadClass.NEIGHBOR, ref.HeadClass.DUMMY][c] for c in codes),
                               int((codes == 2).sum()))
        out["macs"].append({"cfg": cfg.to_dict(), "history": hist, "codes": codes.tolist(),
                            "baseline": ref_engine.expected_step_macs(cfg, "baseline", hist),
                            "hma": ref_engine.expected_step_macs(cfg, "hma", hist, a),
                            "packed": ref_engine.expected_step_macs(cfg, "packed", hist, a)})
        out["extension"].append({"cfg": cfg.to_dict(), "codes": codes.tolist(),
                                 "ext": ref_kv.extension_window(a, cfg)})
        out["ratio"].append({"cfg": cfg.to_dict(), "codes": codes.tolist(),
                             "ratio": ref_kv.cache_stats(a, cfg).reduction_ratio})
    for n, r in [(16, 0.25), (4680, 0.25), (192, 0.25), (7, 1.0), (1560, 0.1), (8, 0.5), (100, 0.33), (4680, 1.0)]:
        out["subsample"].append({"n": n, "ratio": r, "rows": ref_prof.subsample_rows(n, r).tolist()})
    json.dump(out, open(os.path.join(OUT, "accounting.json"), "w"))


def gen_toy_report():
    cfg = ref.SessionConfig(num_layers=2, num_heads=4, head_dim=64, HW=192, window_len=6, ar_steps=10,
                            denoise_steps=2, dummy_count=2, probe_ar_step=2, subsample_ratio=0.25)
    spec = ref.ToyModelSpec(num_layers=2, num_heads=4, head_dim=64, HW=192, denoise_steps=2, seed=ref_rng.derive(42, "toy-model"))
    out = {}
    for mode in ("baseline", "hma", "packed"):
        _, rep = ref.generate_session(ref.build_toy_model(spec), cfg, mode)
        d = rep.to_dict()
        d.pop("total_wall_time_ns")
        for st in d["steps"]:
            st.pop("wall_time_ns")
            st.pop("layer_wall_time_ns")
        out[mode] = d
    json.dump(out, open(os.path.join(OUT, "toy_c1_reports.json"), "w"))


def gen_container():
    """A small .dfc written by the reference's container.save_tensors."""
    from dummy_forcing import container as ref_container

    rng = np.random.default_rng(12)
    tensors = {"layer0/head0/frame0/keys": rng.standard_normal((4, 8)).astype(np.float32),
               "layer0/head0/frame0/values": rng.standard_normal((4, 8)),
               "scalar": np.array(3.5)}
    path = os.path.join(OUT, "ref_container.dfc")
    ref_container.save_tensors(path, tensors)
    json.dump({"digest": ref_container.array_digest(*tensors.values())},
              open(os.path.join(OUT, "ref_container.json"), "w"))



if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    gen_rng()
    gen_greedy()
    gen_eviction()
    gen_attention()
    gen_planted_sessions()
    gen_extension_sessions()
    gen_accounting()
    gen_toy_report()
    gen_container()
    print("golden fixtures written to", OUT)

