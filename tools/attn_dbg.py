import sys, numpy as np
sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, F32, GEMM_SIMT, GEMM_TCGEN05, SWIGLU3, Engine, ModelSpec
from oracle.oracle import Oracle, ModelSpec as OSpec
for hd_cfg in [dict(attn_heads=8, kv_heads=2, head_dim=64), dict(attn_heads=0)]:
    sp = dict(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, seed=0, expert_kind=SWIGLU3, rope_theta=1e6, **hd_cfg)
    m = Oracle("port").build(OSpec(**sp))
    ms = ModelSpec(**sp)
    es = {n: Engine(ms, weight_type=wt, gemm=g, max_batch=1, max_gamma=1, max_seq_len=64).init_exact()
          for n, wt, g in (("f32", F32, GEMM_SIMT), ("bf16simt", BF16, GEMM_SIMT), ("bf16tc", BF16, GEMM_TCGEN05))}
    rng = np.random.RandomState(4)
    for _ in range(4):
        prefix = rng.randint(0, 1024, size=rng.randint(1, 16)).tolist()
        rl = m.forward(prefix)[0]
        out = {n: float(np.max(np.abs(e.forward(prefix)[0] - rl)) / np.max(np.abs(rl))) for n, e in es.items()}
        print(hd_cfg.get("attn_heads"), len(prefix), {k: round(v, 5) for k, v in out.items()}, round(float(np.max(np.abs(rl))), 3))
