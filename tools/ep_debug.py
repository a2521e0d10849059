"""EP loopback debugging: run G virtual ranks on one GPU for a shape given on the command line."""
import sys
import threading

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, LoopbackGroup, ModelSpec, RunCfg  # noqa: E402
from paper_2604_10152_b200.prompts import make_prompts  # noqa: E402

G, E, K, dense0, B = (int(v) for v in sys.argv[1:6])
mask = [0, 1, 1] if dense0 else [1, 1, 1]
s = ModelSpec(num_layers=3, experts=E, top_k=K, hidden=256, ffn=256, vocab=512, expert_kind=SWIGLU3, moe_mask=mask,
              gate_skew=0.5, seed=4)
prompts = make_prompts(8, B, 8, s.vocab)
cfg = RunCfg(gamma=4, n_draft=max(K, min(E, 8)), max_new_tokens=6)
grp = LoopbackGroup(G)
engines = []
for r in range(G):
    e = Engine(s, weight_type=BF16, max_batch=B, max_gamma=4, ep_rank=r, ep_world=G).init_device(13)
    e.build_affinity_device()
    e.attach_loopback(grp)
    engines.append(e)
out, errs = [None] * G, []


def work(r):
    try:
        out[r] = engines[r].run_ondemand(cfg, prompts)
    except Exception as ex:
        errs.append((r, ex))


import os, time  # noqa: E401,E402
t0 = time.time()
th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
[t.start() for t in th]
[t.join(timeout=120) for t in th]
print(os.environ.get("SMOE_PDL", "-"), os.environ.get("SMOE_EP_MODE", "-"), "G", G, "E", E, "K", K, "dense0", dense0, "B", B,
      "errors", str(errs)[:400], "ok" if not errs else "FAIL", round(time.time() - t0, 2), "s", flush=True)
