"""Compare forward() outputs of the two gate kernels (SMOE_GATE_RG=0 vs 1) on the E=64 digest shape."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec
    E = int(os.environ.get("DBG_E", "64"))
    spec = ModelSpec(num_layers=3, experts=E, top_k=6 if E > 8 else 2, hidden=1024, ffn=512, vocab=512,
                     expert_kind=SWIGLU3, moe_mask=[0, 1, 1], gate_skew=0.5)
    e = Engine(spec, weight_type=BF16, max_batch=8, max_gamma=4).init_device(3)
    out = {}
    for n, prefix in enumerate(([1, 2, 3], list(range(40)), [100] * 9)):
        lg, raw, fin = e.forward(prefix)
        out[f"lg{n}"], out[f"raw{n}"], out[f"fin{n}"] = lg, raw, fin
    np.savez(sys.argv[2], **out)
else:
    for v in ("0", "1"):
        subprocess.run([sys.executable, __file__, "child", f"/tmp/gd{v}.npz"], env=dict(os.environ, SMOE_GATE_RG=v),
                       check=True)
    a, b = np.load("/tmp/gd0.npz"), np.load("/tmp/gd1.npz")
    for k in a.files:
        x, y = a[k], b[k]
        same = np.array_equal(x, y)
        print(k, "same" if same else f"DIFF max|d|={np.nanmax(np.abs(x.astype(np.float64) - y)):.3g}",
              "" if same else (x[:12], y[:12]))
