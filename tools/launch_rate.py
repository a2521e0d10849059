"""Host launch rate vs device time of one speculative phase (SMOE_HOST_PROF breakdown on stderr).

A model with the C4 layer count but tiny widths: the device work per kernel is a few microseconds, so
the phase time measures how fast the host issues the phase's ~600 launches."""
import os
import sys
import time

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "tiny_c4"
if shape == "tiny_c4":
    spec = ModelSpec(num_layers=28, experts=64, top_k=6, hidden=256, ffn=128, vocab=512, moe_mask=[0] + [1] * 27,
                     expert_kind=SWIGLU3)
    B, nd = 32, 8
else:
    spec = ModelSpec(num_layers=32, experts=8, top_k=2, hidden=256, ffn=256, vocab=512, expert_kind=SWIGLU3)
    B, nd = 64, 4
e = Engine(spec, weight_type=BF16, max_batch=B, max_gamma=4).init_device(0)
e.build_affinity_device()
e.spec_begin(RunCfg(gamma=4, n_draft=nd, max_new_tokens=1 << 30), make_prompts(1, B, 8, spec.vocab))
for _ in range(3):
    e.spec_step()
e.counters(reset=True)
t0 = time.perf_counter()
n = 10
for _ in range(n):
    e.spec_step()
dt = (time.perf_counter() - t0) / n
c = e.counters()
print(f"{shape}: {dt * 1e3:.3f} ms per phase, {c['launches'] / n:.0f} launches per phase, "
      f"{dt / (c['launches'] / n) * 1e6:.2f} us per launch (wall)")
