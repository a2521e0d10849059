"""Expert GEMM timed alone on the Mixtral-8x7B shape (one MoE layer's up + down projections)."""
import json
import sys

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"]
spec = ModelSpec(num_layers=1, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
e = Engine(spec, weight_type=BF16, max_batch=64, max_gamma=4).init_device(0)
rows = []
for T in [1, 4, 8, 16, 32, 80, 160, 320]:
    r = e.bench_expert_gemm(T, 10)
    r["T"] = T
    r["up_frac"] = r["up_GBps"] / peak
    r["down_frac"] = r["down_GBps"] / peak
    rows.append(r)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
json.dump(rows, open("gpurun_out/gemm_bench.json", "w"), indent=1)
