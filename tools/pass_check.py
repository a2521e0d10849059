"""Pass kernel (pass_tc.cu) vs the per-layer launch sequence on the same weights and prompts:
logits of forward() and the greedy tokens of a short speculative run."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "small"
if shape == "c2l4":
    spec = ModelSpec(num_layers=4, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
elif shape == "c4l4":
    spec = ModelSpec(num_layers=4, experts=64, top_k=6, hidden=2048, ffn=1408, vocab=102400, expert_kind=SWIGLU3,
                     moe_mask=[0, 1, 1, 1])
else:
    spec = ModelSpec(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, expert_kind=SWIGLU3)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ND = 8 if shape == "c4l4" else 4
prompts = make_prompts(7, B, 8, spec.vocab)
out = {}
for pk in ("0", "1"):
    os.environ["SMOE_PASS_KERNEL"] = pk
    os.environ["SMOE_PASS_MIN_ROWS"] = "1"
    e = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=4).init_device(3)
    e.build_affinity_device()
    e.counters(reset=True)
    lg, raw, fin = e.forward(prompts[0])
    print("SMOE_PASS_KERNEL", pk, "launches per forward", e.counters()["launches"])
    r = e.run_specmoe(RunCfg(gamma=4, n_draft=ND, max_new_tokens=16, run_seed=1), prompts)
    od = e.run_ondemand(RunCfg(gamma=4, n_draft=ND, max_new_tokens=16, run_seed=1), prompts)
    out[pk] = (np.array(lg), raw, fin, r.tokens, od.tokens, r.metrics["tau_mean"])
    e.close()
a, b = out["0"], out["1"]
rel = float(np.max(np.abs(a[0] - b[0])) / np.max(np.abs(a[0])))
same_tok = sum(x == y for x, y in zip(a[3], b[3]))
print(f"{shape} B={B}: logits bit-identical {np.array_equal(a[0], b[0])}; max rel diff {rel:.3e}; routing raw equal {a[1] == b[1]}; spec tokens equal seqs {same_tok}/{B};"
      f" lossless(pass kernel) {b[3] == b[4]}; tau {a[5]:.3f} vs {b[5]:.3f}")
assert b[3] == b[4], "pass kernel: speculative != on-demand"
