"""SwiGLU (expert_kind=1, the benchmarked expert) pinned to the oracle's independent restatement.

The reference expert is tanh2 (model.cpp:54-59); the north_star's Mixtral expert is SwiGLU, so the
only independent statement of its arithmetic is the plain-C port's swiglu3
(oracle/specmoe_oracle.c `expert_fwd`: h = silu(W1^T x) * (W3^T x), y = W2^T h, weights drawn w1, w3,
w2 per expert in the reference's polar stream order).  These tests compare the engine with it:

  * fp32 engine (CUDA-core GEMMs) vs the float64 port: routing, drafts, accepted counts, tokens,
    ledger, hotness and modeled metrics bit-exact; logits within 2e-5 of the logit scale.
  * bf16 tcgen05 engine (the benchmarked path: interleaved w1/w3 tiles, silu*mul epilogue in TMEM
    read-back) vs the port, margin-aware: every routing decision whose oracle gate margin exceeds
    0.05 and every greedy token whose logit margin exceeds 0.1 agree; logits within 3% of the scale.
    Near-tie rates are printed.
  * The same two checks at Mixtral-8x7B widths (d=4096, f=14336) on a one-MoE-layer slice with 4
    experts (the port's fp64 weights uploaded into both engines; the slice keeps the oracle build
    to ~30 s of single-threaded weight generation).
"""
import numpy as np
import pytest

from paper_2604_10152_b200.engine import BF16, F32, GEMM_TCGEN05, SWIGLU3, Engine, ModelSpec, RunCfg
from paper_2604_10152_b200.prompts import make_prompts

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-5


def _spec(d):
    return ModelSpec(**{k: v for k, v in d.items() if k in ModelSpec.__dataclass_fields__})


TOYS = [
    dict(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.5, seed=1),
    dict(num_layers=3, experts=8, top_k=2, hidden=48, ffn=40, vocab=96, gate_skew=0.5, seed=2),
    dict(num_layers=3, moe_mask=[0, 1, 1], experts=64, top_k=6, hidden=64, ffn=32, vocab=128, seed=3),
    dict(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, seed=0),        # C1 widths
]
RUNS = [
    dict(gamma=5, n_draft=4, max_new_tokens=20),
    dict(gamma=4, n_draft=3, max_new_tokens=16, policy="hot_global", warmup_steps=5),
    dict(gamma=4, n_draft=8, max_new_tokens=14),
    dict(gamma=4, n_draft=4, max_new_tokens=16),
]


def _equal_runs(got, want):
    assert got.tokens == want.tokens
    assert got.outcomes == want.outcomes
    assert got.trace == want.trace
    assert got.ledger == want.ledger
    assert got.hotness.tolist() == want.hotness.tolist()
    for k, v in want.metrics.items():
        if k != "wall_s":
            assert got.metrics[k] == v, k


@pytest.mark.parametrize("case", range(len(TOYS)))
def test_f32_swiglu_equals_port(case, port):
    from oracle.oracle import ModelSpec as OSpec, RunCfg as ORun
    sp = dict(TOYS[case], expert_kind=SWIGLU3)
    m = port.build(OSpec(**sp))
    B = 1 if sp["hidden"] >= 512 else 3
    e = Engine(_spec(sp), weight_type=F32, max_batch=B, max_gamma=5).init_exact()
    assert np.array_equal(e.affinity(), m.affinity())
    prompts = make_prompts(40 + case, B, 8, sp["vocab"])
    for p in (prompts[0], prompts[0] + [1, 2, 3], [sp["vocab"] - 1] * 3):
        lg, raw, _ = e.forward(p)
        rl, rr, _ = m.forward(p)
        assert raw.tolist() == rr.tolist()
        assert np.max(np.abs(lg - rl)) <= LOGIT_TOL * np.max(np.abs(rl))
    cfg = dict(RUNS[case], collect_trace=True, run_seed=case)
    _equal_runs(e.run_specmoe(RunCfg(**cfg), prompts), m.run_specmoe(ORun(**cfg), prompts))
    od_g, od_w = e.run_ondemand(RunCfg(**cfg), prompts), m.run_ondemand(ORun(**cfg), prompts)
    assert od_g.tokens == od_w.tokens and od_g.ledger == od_w.ledger and od_g.trace == od_w.trace
    e.close()


def _margin_aware(e, m, K, V, prefixes, label):
    """Compare a bf16 engine's forward() with the float64 port over prefixes; return the stats."""
    route_total = route_big = route_bad = tok_big = tok_bad = 0
    worst = 0.0
    for prefix in prefixes:
        lg, raw, _ = e.forward(prefix)
        rl, gates = m.forward_gates(prefix)
        rr = m.forward(prefix)[1]
        worst = max(worst, float(np.max(np.abs(lg - rl)) / np.max(np.abs(rl))))
        for l in range(gates.shape[0]):
            srt = np.sort(gates[l])[::-1]
            route_total += 1
            if srt[K - 1] - srt[K] > 0.05:
                route_big += 1
                route_bad += set(raw[l].tolist()) != set(rr[l].tolist())
        s2 = np.sort(rl)[::-1]
        if s2[0] - s2[1] > 0.1:
            tok_big += 1
            tok_bad += int(np.argmax(lg)) != int(np.argmax(rl))
    print(f"{label}: worst logit err {worst:.4f}; routing near-tie rate {1 - route_big / route_total:.3f}; "
          f"token near-tie rate {1 - tok_big / len(prefixes):.3f}; decisions checked {route_big}+{tok_big}")
    return worst, route_bad, tok_bad, route_big, tok_big


def test_bf16_tcgen05_swiglu_c1_vs_port(port):
    from oracle.oracle import ModelSpec as OSpec
    sp = dict(TOYS[3], expert_kind=SWIGLU3)
    m = port.build(OSpec(**sp))
    e = Engine(_spec(sp), weight_type=BF16, gemm=GEMM_TCGEN05, max_batch=1, max_gamma=1).init_exact()
    rng = np.random.RandomState(3)
    prefixes = [rng.randint(0, sp["vocab"], size=rng.randint(1, 24)).tolist() for _ in range(60)]
    worst, rbad, tbad, rbig, tbig = _margin_aware(e, m, sp["top_k"], sp["vocab"], prefixes, "C1 swiglu3 bf16")
    assert worst <= 0.03
    assert rbad == 0 and tbad == 0
    assert rbig >= 120 and tbig >= 20
    e.close()


SLICE = dict(num_layers=1, experts=4, top_k=2, hidden=4096, ffn=14336, vocab=1024, seed=7, expert_kind=SWIGLU3)


@pytest.fixture(scope="module")
def mixtral_slice(port):
    """Port model at Mixtral widths; its float64 tensors uploaded into an fp32 and a bf16 engine."""
    from oracle.oracle import ModelSpec as OSpec
    m = port.build(OSpec(**SLICE))
    engines = {}
    for wt in (F32, BF16):
        e = Engine(_spec(SLICE), weight_type=wt, max_batch=2, max_gamma=4)
        e.upload("embedding", m.tensor("embedding"))
        e.upload("head", m.tensor("head"))
        e.upload("mix", m.tensor("mix", 0), layer=0)
        e.upload("gate", m.tensor("gate", 0), layer=0)
        for x in range(SLICE["experts"]):
            for name in ("w1", "w3", "w2"):
                e.upload(name, m.tensor(name, 0, x), layer=0, expert=x)
        e.set_affinity(m.affinity())
        engines[wt] = e
    yield m, engines
    for e in engines.values():
        e.close()


def test_f32_swiglu_mixtral_width_slice_equals_port(mixtral_slice):
    from oracle.oracle import RunCfg as ORun
    m, engines = mixtral_slice
    e = engines[F32]
    prompts = make_prompts(11, 2, 8, SLICE["vocab"])
    lg, raw, _ = e.forward(prompts[0])
    rl, rr, _ = m.forward(prompts[0])
    assert raw.tolist() == rr.tolist()
    assert np.max(np.abs(lg - rl)) <= LOGIT_TOL * np.max(np.abs(rl))
    cfg = dict(gamma=4, n_draft=2, max_new_tokens=5, collect_trace=True, run_seed=1)
    got, want = e.run_specmoe(RunCfg(**cfg), prompts), m.run_specmoe(ORun(**cfg), prompts)
    assert got.tokens == want.tokens and got.outcomes == want.outcomes
    assert got.trace == want.trace and got.ledger == want.ledger


def test_bf16_tcgen05_swiglu_mixtral_width_vs_port(mixtral_slice):
    m, engines = mixtral_slice
    rng = np.random.RandomState(5)
    prefixes = [rng.randint(0, SLICE["vocab"], size=rng.randint(1, 16)).tolist() for _ in range(24)]
    worst, rbad, tbad, rbig, tbig = _margin_aware(engines[BF16], m, SLICE["top_k"], SLICE["vocab"], prefixes,
                                                  "Mixtral-width swiglu3 bf16")
    assert worst <= 0.03
    assert rbad == 0 and tbad == 0
    assert rbig >= 10 and tbig >= 6
