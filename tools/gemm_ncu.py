"""One up + one down expert-GEMM launch (8 experts, T tokens) for an ncu --set full capture."""
import sys

sys.path.insert(0, ".")
from paper_2604_10152_b200.engine import BF16, SWIGLU3, Engine, ModelSpec  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 160
spec = ModelSpec(num_layers=1, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
e = Engine(spec, weight_type=BF16, max_batch=64, max_gamma=4).init_device(0)
print(e.bench_expert_gemm(T, 1))
