"""Batch sweep of the speculative loop on the Mixtral-8x7B shape (HBM-resident, SwiGLU bf16)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

batches = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8,16,32,64").split(",")]
gamma = int(sys.argv[2]) if len(sys.argv) > 2 else 4
import os  # noqa: E402
SHAPE = os.environ.get("SHAPE", "c2")
if SHAPE == "c4":  # fine-grained E64 K6, layer 0 dense (C4)
    spec = ModelSpec(num_layers=28, experts=64, top_k=6, hidden=2048, ffn=1408, vocab=102400, expert_kind=SWIGLU3,
                     moe_mask=[0] + [1] * 27)
else:
    spec = ModelSpec(num_layers=32, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
N_DRAFT = 8 if SHAPE == "c4" else 4
e = Engine(spec, weight_type=BF16, max_batch=max(batches), max_gamma=gamma).init_device(0)
e.build_affinity_device()
st = torch.cuda.ExternalStream(e.stream)
rows = []
for B in batches:
    e.spec_begin(RunCfg(gamma=gamma, n_draft=N_DRAFT, max_new_tokens=1 << 30), make_prompts(1000, B, 8, spec.vocab))
    for _ in range(2):
        e.spec_step()
    e.counters(reset=True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(st)
    toks = sum(e.spec_step()[0] for _ in range(4))
    b.record(st)
    b.synchronize()
    ms = a.elapsed_time(b)
    # profiled copy of the region: per-launch events around the expert GEMMs (serialises PDL overlap)
    e.counters(reset=True)
    e.profile_reset()
    for _ in range(4):
        e.spec_step()
    c = e.counters()
    p = e.profile_read("expert_gemm")
    if p["ms"] <= 0:  # persistent pass kernel: the expert GEMMs run inside it
        p = e.profile_read("pass")
    other = {k: round(e.profile_read(k)["ms"] / 4, 3) for k in ("dense_gemm", "head_gemm", "gate", "combine", "pass")}
    r = e.spec_end()
    row = {"B": B, "gamma": gamma, "tokens_per_s": toks / ms * 1e3, "ms_per_step": ms / 4, "tau": r.metrics["tau_mean"],
           "expert_gemm_ms_per_step": p["ms"] / 4, "expert_hbm_GBps": c["alg_expert_bytes"] / (p["ms"] * 1e-3) / 1e9,
           "hbm_bytes_per_token": c["alg_expert_bytes"] / max(1, toks), "other_ms_per_step": other}
    rows.append(row)
    print(json.dumps(row), flush=True)
json.dump(rows, open(f"gpurun_out/sweep_g{gamma}.json", "w"), indent=1)
