import sys, numpy as np
sys.path.insert(0, ".")
from oracle.oracle import Oracle, ModelSpec as OS
from paper_2604_10152_b200.engine import Engine, ModelSpec, F32
port = Oracle("port")
base = dict(num_layers=1, experts=8, top_k=2, hidden=32, ffn=64, vocab=64, seed=0)
cases = [{}, {"hidden": 64}, {"hidden": 128}, {"hidden": 256}, {"hidden": 512}, {"ffn": 1024}, {"vocab": 1024},
         {"hidden": 512, "ffn": 1024, "vocab": 1024}, {"num_layers": 4, "hidden": 512, "ffn": 1024, "vocab": 1024}]
for c in cases:
    s = dict(base, **c)
    m = port.build(OS(**s))
    e = Engine(ModelSpec(**s), weight_type=F32, max_batch=1, max_gamma=1).init_exact()
    for pre in ([3], [1, 2, 3, 4, 5, 6, 7, 8]):
        pre = [p % s["vocab"] for p in pre]
        lg, raw, _ = e.forward(pre)
        rl, rr, _ = m.forward(pre)
        print(c, len(pre), "err", float(np.max(np.abs(lg - rl))), "scale", float(np.max(np.abs(rl))), "raw_eq", raw.tolist() == rr.tolist(), flush=True)
    e.close()
