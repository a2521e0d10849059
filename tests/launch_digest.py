"""Digest of one engine's results (logits, routing, token streams) for tests/test_engine_gpu.py::
test_launch_shape_switches_bitexact: run in a fresh process per environment, because the launch-shape
switches (row-kernel clusters, gate staging, pair units, L2 prefetch, PDL) are read once per process.
Prints one JSON line {shape: sha256}."""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

SHAPES = {
    # d=2048: 512-thread row trees (2-CTA row clusters), E=8 gate weights staged in shared memory
    "e8_d2048": (ModelSpec(num_layers=2, experts=8, top_k=2, hidden=2048, ffn=1024, vocab=512,
                           expert_kind=SWIGLU3, gate_skew=1.0), 4),
    # E=64 at d=1024: 1024-thread gate tree (4-CTA clusters), gate weights too large to stage
    "e64_d1024": (ModelSpec(num_layers=3, experts=64, top_k=6, hidden=1024, ffn=512, vocab=512,
                            expert_kind=SWIGLU3, moe_mask=[0, 1, 1], gate_skew=0.5), 8),
    # E=64 at B=32: verify passes of 160 rows > SMs (row-group gate without staged weights, 256-thread CTAs)
    "e64_b32": (ModelSpec(num_layers=2, experts=64, top_k=6, hidden=1024, ffn=256, vocab=512,
                          expert_kind=SWIGLU3, moe_mask=[0, 1], gate_skew=0.5), 8, 32),
    # B=64 verify passes of 320 rows over 4 experts: groups of > 128 tokens (unpaired launches)
    "e4_b64": (ModelSpec(num_layers=2, experts=4, top_k=2, hidden=1024, ffn=512, vocab=512,
                         expert_kind=SWIGLU3, gate_skew=1.0), 2, 64),
}


def digest(spec, nd, batch=8):
    h = hashlib.sha256()
    e = Engine(spec, weight_type=BF16, max_batch=batch, max_gamma=4).init_device(3)
    for prefix in ([1, 2, 3], list(range(40)), [100] * 9):
        lg, raw, fin = e.forward(prefix)
        for a in (lg, raw, fin):
            h.update(np.ascontiguousarray(a).tobytes())
    e.build_affinity_device()
    r = e.run_specmoe(RunCfg(gamma=4, n_draft=nd, max_new_tokens=24), make_prompts(11, batch, 8, spec.vocab))
    h.update(json.dumps([r.tokens, [list(x) for x in r.ledger]]).encode())
    e.close()
    return h.hexdigest()


if __name__ == "__main__":
    print(json.dumps({k: digest(*v) for k, v in SHAPES.items()}))
