"""Independent sessions run concurrently (SURVEY.md 8(b) threading contract).

The reference allows several independent sessions at once (
verify.py:215-240; tests/test_verify.py:37-44).  Here every session owns its
rings, its split-KV workspace (one per KV arena) and its stream; the library
keeps no process-global mutable state on the launch path.  Four sessions on
four threads, each on its own CUDA stream, must give outputs and reports
bitwise equal to the same sessions run one after the other.
"""
import json
import os
import threading

import pytest
import torch

import paper_2601_20499_b200 as df
from oracle import df_oracle as O

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def _planted(i):
    rec = json.load(open(os.path.join(G, "planted_sessions.json")))[i]
    return rec, df.SessionConfig(**rec["config"]), O.PlantedStream(rec["labels"], 2.0, rec["noise_seed"],
                                                                    O.Config(**rec["config"]))


def _projected(seed):
    ocfg = O.Config(num_layers=2, num_heads=4, head_dim=64, HW=192, window_len=6, ar_steps=9, denoise_steps=2,
                    dummy_count=3, probe_ar_step=2, subsample_ratio=0.25)
    toy = O.ToyModel(2, 4, 64, 192, O.derive(seed, "toy-model"))
    return df.SessionConfig(**ocfg.__dict__), df.ProjectedModel(toy.weights, toy.frame_input, 4, 64, 192)


def _jobs():
    """(name, factory) pairs; each factory builds a fresh (model, config, mode, kwargs)."""
    jobs = []
    for i in (0, 3, 5):
        def mk(i=i):
            rec, cfg, stream = _planted(i)
            return stream, cfg, rec["mode"], {}
        jobs.append((f"planted{i}", mk))

    def mk_proj():
        cfg, model = _projected(7)
        return model, cfg, "packed", {"graphs": True}
    jobs.append(("projected_graphs", mk_proj))
    return jobs


def _summary(sess, frames, rep):
    d = rep.to_dict()
    d.pop("total_wall_time_ns")
    for st in d["steps"]:
        st.pop("wall_time_ns")
        st.pop("layer_wall_time_ns")
    return d, [c.frame_ids for layer in sess.caches for c in layer]


def test_four_sessions_on_four_threads_and_streams_equal_serial():
    serial = {}
    for name, mk in _jobs():
        model, cfg, mode, kw = mk()
        s = df.Session(model, cfg, mode, **kw)
        frames, rep = s.run()
        torch.cuda.synchronize()
        serial[name] = _summary(s, frames, rep)

    results, errors = {}, []
    barrier = threading.Barrier(len(serial))

    def worker(name, mk):
        try:
            model, cfg, mode, kw = mk()
            st = torch.cuda.Stream()
            s = df.Session(model, cfg, mode, stream=st, **kw)
            barrier.wait()
            with torch.cuda.stream(st):
                frames, rep = s.run()
            st.synchronize()
            results[name] = (s, frames, rep)
        except BaseException as e:  # surfaced in the main thread
            errors.append((name, e))
            barrier.abort()

    threads = [threading.Thread(target=worker, args=job) for job in _jobs()]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    torch.cuda.synchronize()
    for name, (s, frames, rep) in results.items():
        assert _summary(s, frames, rep) == serial[name], name
