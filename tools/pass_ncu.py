"""Workload for an ncu capture of the pass kernel: Mixtral-shape (C2) on-demand decode passes at batch B."""
import sys

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = int(sys.argv[2]) if len(sys.argv) > 2 else 32
spec = ModelSpec(num_layers=L, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
e = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=4).init_device(0)
e.build_affinity_device()
e.run_ondemand(RunCfg(gamma=4, n_draft=4, max_new_tokens=3), make_prompts(1000, B, 8, spec.vocab))
print("done")
