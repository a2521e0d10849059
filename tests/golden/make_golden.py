"""Generate tests/golden/*.json from the reference itself (oracle/_ref, compiled from
/root/reference/proj/core/src).  Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The JSON files are committed; tests read them on any machine (the GPU box has no
/root/reference).  Floats are stored with repr(), which round-trips float64 exactly.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import ModelSpec, Oracle, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def run_dict(r):
    return {"tokens": r.tokens, "ledger": [list(x) for x in r.ledger],
            "outcomes": [list(o[:5]) + [list(o[5])] for o in r.outcomes],
            "trace": [[t[0], t[1], t[2], list(t[3])] for t in r.trace],
            "hotness": r.hotness.tolist(),
            "metrics": {k: v for k, v in r.metrics.items() if k != "wall_s"}}


def weights_digest(m, spec):
    """Cheap pins of the seeded weights (model.cpp:106-143): a few exact values + float64 sums."""
    out = {}
    for name, layer, expert in [("embedding", -1, -1), ("head", -1, -1), ("mix", 0, -1), ("gate", 0, -1),
                                ("up", 0, 0), ("down", spec.num_layers - 1, spec.experts - 1)]:
        t = m.tensor(name, layer, expert)
        out[f"{name}:{layer}:{expert}"] = {"n": int(t.size), "first": t[:4].tolist(), "last": t[-2:].tolist(),
                                           "sum": float(np.sum(t))}
    return out


def main():
    ref = Oracle("ref")
    gold = {}

    # SPEC.md:74-76 forward example spec (L=2, E=4, K=2, d=8, f=16, V=32), prefix [2, 7, 7]
    s = ModelSpec(num_layers=2, experts=4, top_k=2, hidden=8, ffn=16, vocab=32, seed=0)
    m = ref.build(s)
    lg, raw, fin = m.forward([2, 7, 7])
    gold["spec_forward"] = {"spec": s.__dict__, "prefix": [2, 7, 7], "logits": lg.tolist(), "raw": raw.tolist()}

    # SPEC acceptance toy (L4 E16 K2 d32 f64 V64, skewed), a few (seed, N, gamma) cells
    toy = []
    for seed, n_draft, gamma, B in [(0, 2, 5, 1), (1, 4, 5, 2), (2, 8, 10, 1), (3, 16, 10, 1), (4, 4, 5, 4)]:
        s = ModelSpec(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.5, seed=seed)
        m = ref.build(s)
        prompts = make_prompts(seed, B, 8, s.vocab)
        cfg = RunCfg(gamma=gamma, n_draft=n_draft, max_new_tokens=24, policy="hot_temporal", collect_trace=True,
                     run_seed=seed)
        sp = m.run_specmoe(cfg, prompts)
        od = m.run_ondemand(cfg, prompts)
        toy.append({"spec": s.__dict__, "cfg": cfg.__dict__, "prompts": prompts, "specmoe": run_dict(sp),
                    "ondemand": run_dict(od), "affinity": m.affinity().tolist(), "weights": weights_digest(m, s)})
    gold["toy"] = toy

    # C1 tiny (BASELINE configs[0]): L4 E8 K2 d512 f1024 V1024, gamma=4, B=1, N=4
    s = ModelSpec(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, seed=0)
    m = ref.build(s)
    prompts = make_prompts(0, 1, 8, s.vocab)
    cfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=16, policy="hot_temporal", collect_trace=True, run_seed=0)
    sp = m.run_specmoe(cfg, prompts)
    lg, raw, fin = m.forward(prompts[0])
    gold["c1"] = {"spec": s.__dict__, "cfg": cfg.__dict__, "prompts": prompts, "specmoe": run_dict(sp),
                  "forward_logits": lg.tolist(), "forward_raw": raw.tolist(),
                  "affinity": m.affinity().tolist(), "weights": weights_digest(m, s)}

    # the comparators (baselines.cpp:100-157): oracle overlap and caching, incl. an eviction-bound tier
    base = []
    for seed, B, frac, warm, cap in [(5, 3, 0.25, 6, 0), (6, 2, 0.10, 4, 0), (7, 2, 0.20, 16, 40 * 2 * 32 * 64 * 4)]:
        s = ModelSpec(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.5, seed=seed)
        m = ref.build(s)
        prompts = make_prompts(seed, B, 8, s.vocab)
        cfg = RunCfg(max_new_tokens=12, warmup_steps=warm, collect_trace=True, run_seed=seed,
                     device_capacity_bytes=cap)
        base.append({"spec": s.__dict__, "cfg": cfg.__dict__, "prompts": prompts, "cache_fraction": frac,
                     "overlap": run_dict(m.run_overlap(cfg, prompts)),
                     "caching": run_dict(m.run_caching(cfg, prompts, frac))})
    gold["baselines"] = base

    # the reference-API caller (tests/cpp/caller.cpp) compiled against the reference itself
    import subprocess
    exe = os.path.join(ROOT, "oracle", "_ref", "caller_ref")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I/root/reference/proj/core/include",
                    os.path.join(ROOT, "tests", "cpp", "caller.cpp")] +
                   sorted(__import__("glob").glob("/root/reference/proj/core/src/*.cpp")) + ["-o", exe], check=True)
    gold["cpp_caller"] = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)
    exe = os.path.join(ROOT, "oracle", "_ref", "caller_sampling_ref")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I/root/reference/proj/core/include",
                    os.path.join(ROOT, "tests", "cpp", "caller_sampling.cpp")] +
                   sorted(__import__("glob").glob("/root/reference/proj/core/src/*.cpp")) + ["-o", exe], check=True)
    gold["cpp_caller_sampling"] = json.loads(subprocess.run([exe], capture_output=True, text=True, check=True).stdout)

    for k, v in gold.items():
        with open(os.path.join(OUT, f"{k}.json"), "w") as f:
            json.dump(v, f)
    print("wrote", sorted(gold))


if __name__ == "__main__":
    main()
