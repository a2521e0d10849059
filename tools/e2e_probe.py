"""Where the end-to-end (C ABI) run's wall time goes: spec_begin, each spec_step, spec_end (C2, B=64)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
NT = int(sys.argv[2]) if len(sys.argv) > 2 else 12
spec = ModelSpec(num_layers=32, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
e = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=4).init_device(0)
e.build_affinity_device()
prompts = make_prompts(1000, B, 8, spec.vocab)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = e.run_specmoe(RunCfg(gamma=4, n_draft=4, max_new_tokens=NT), prompts)
    torch.cuda.synchronize()
    tw = time.perf_counter() - t0
    print(f"run_specmoe: {tw*1e3:.1f} ms, tokens {r.metrics['tokens_total']}, phases {r.metrics['phases']}, "
          f"{r.metrics['tokens_total']/tw:.1f} tok/s, tau {r.metrics['tau_mean']:.3f}", flush=True)
    t0 = time.perf_counter()
    e.spec_begin(RunCfg(gamma=4, n_draft=4, max_new_tokens=NT), prompts)
    tb = time.perf_counter() - t0
    steps, toks = [], []
    while True:
        t1 = time.perf_counter()
        a, act = e.spec_step()
        steps.append(time.perf_counter() - t1)
        toks.append((a, act))
        if act == 0:
            break
    t2 = time.perf_counter()
    rr = e.spec_end()
    te = time.perf_counter() - t2
    print(f"stepped: begin {tb*1e3:.1f} ms, steps {len(steps)} x [{', '.join(f'{s*1e3:.1f}' for s in steps)}] ms, "
          f"end {te*1e3:.1f} ms, tokens/step {[t[0] for t in toks]}, active {[t[1] for t in toks]}", flush=True)
