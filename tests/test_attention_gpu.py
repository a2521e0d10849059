"""Real GQA attention with a paged KV cache and rollback against its restatement.

The reference has no attention (model.cpp:211-224 is a prefix-mean surrogate), so the semantics are
pinned by the plain-C port's extension (oracle/specmoe_oracle.c fwd_attn): x0 = the token's embedding,
per layer x += Wo attn(RoPE(Wq rms x), RoPE(Wk rms x), Wv rms x) over every earlier position, the draft
model's k/v for a phase's draft positions and the target's for committed ones.  The engine keeps the k/v
in a paged cache (prefill of the prompts, draft passes write tentative k/v, the verify pass rewrites
them with the target's, acceptance advances the committed length = rollback of the rejected tail).

  * fp32 engine vs the float64 port: routing, drafts, accepted counts, tokens, ledger bit-exact; logits
    within 2e-5 of the logit scale.
  * bf16 tcgen05 engine: speculative == on-demand token for token (lossless), batch invariant, and
    margin-aware agreement with the port at C1 widths.
  * offloaded store and sampling mode with attention.
"""
import numpy as np
import pytest

from paper_2604_10152_b200.engine import BF16, F32, SWIGLU3, TANH2, Engine, ModelSpec, RunCfg
from paper_2604_10152_b200.prompts import make_prompts

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-5

TOYS = [
    dict(num_layers=3, experts=8, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.0, seed=3, attn_heads=4,
         kv_heads=2, head_dim=8, rope_theta=10000.0),
    dict(num_layers=4, experts=16, top_k=2, hidden=64, ffn=64, vocab=96, gate_skew=1.5, seed=5, attn_heads=8,
         kv_heads=2, head_dim=16, rope_theta=1e6, expert_kind=SWIGLU3),
    dict(num_layers=3, moe_mask=[0, 1, 1], experts=32, top_k=4, hidden=64, ffn=32, vocab=128, seed=7,
         attn_heads=4, kv_heads=4, head_dim=16, rope_theta=500.0),
]
RUNS = [
    dict(gamma=4, n_draft=4, max_new_tokens=14),
    dict(gamma=5, n_draft=4, max_new_tokens=16, policy="hot_global", warmup_steps=3),
    dict(gamma=3, n_draft=8, max_new_tokens=12, use_affinity=False),
]


def _spec(d):
    return ModelSpec(**{k: v for k, v in d.items() if k in ModelSpec.__dataclass_fields__})


@pytest.mark.parametrize("case", range(len(TOYS)))
def test_f32_attention_equals_port(case, port):
    from oracle.oracle import ModelSpec as OSpec, RunCfg as ORun
    sp = TOYS[case]
    m = port.build(OSpec(**sp))
    B = 3
    e = Engine(_spec(sp), weight_type=F32, max_batch=B, max_gamma=5, max_seq_len=64).init_exact()
    assert np.array_equal(e.affinity(), m.affinity())
    prompts = make_prompts(60 + case, B, 6, sp["vocab"])
    for p in (prompts[0], prompts[1][:1], prompts[2] + [5, 6, 7, 8, 9]):
        lg, raw, _ = e.forward(p)
        rl, rr, _ = m.forward(p)
        assert raw.tolist() == rr.tolist()
        assert np.max(np.abs(lg - rl)) <= LOGIT_TOL * np.max(np.abs(rl))
    sets = [sorted(np.random.RandomState(case).choice(sp["experts"], 4, replace=False).tolist())
            for _ in range(_spec(sp).moe_layers)]
    lg, raw, fin = e.forward(prompts[0], sets, use_affinity=True)
    rl, rr, rf = m.forward(prompts[0], sets, use_affinity=True)
    assert raw.tolist() == rr.tolist() and fin.tolist() == rf.tolist()
    assert np.max(np.abs(lg - rl)) <= LOGIT_TOL * np.max(np.abs(rl))
    cfg = dict(RUNS[case], collect_trace=True, run_seed=case)
    got, want = e.run_specmoe(RunCfg(**cfg), prompts), m.run_specmoe(ORun(**cfg), prompts)
    assert got.tokens == want.tokens
    assert got.outcomes == want.outcomes
    assert got.trace == want.trace and got.ledger == want.ledger
    od_g, od_w = e.run_ondemand(RunCfg(**cfg), prompts), m.run_ondemand(ORun(**cfg), prompts)
    assert od_g.tokens == od_w.tokens == want.tokens and od_g.ledger == od_w.ledger
    e.close()


def _c1_attn(kind=SWIGLU3, skew=1.0, seed=1):
    return ModelSpec(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, gate_skew=skew, seed=seed,
                     expert_kind=kind, attn_heads=8, kv_heads=2, head_dim=64, rope_theta=1e6)


@pytest.mark.parametrize("kind", [TANH2, SWIGLU3])
def test_bf16_attention_lossless_and_batch_invariant(kind):
    s = _c1_attn(kind)
    e = Engine(s, weight_type=BF16, max_batch=4, max_gamma=4, max_seq_len=128).init_device(3)
    e.build_affinity_device()
    prompts = make_prompts(5, 4, 8, s.vocab)
    od = e.run_ondemand(RunCfg(gamma=4, max_new_tokens=40), prompts)
    sp = e.run_specmoe(RunCfg(gamma=4, n_draft=4, max_new_tokens=40), prompts)
    assert sp.tokens == od.tokens
    one = e.run_specmoe(RunCfg(gamma=4, n_draft=4, max_new_tokens=40), prompts[1:2])
    assert one.tokens[0] == sp.tokens[1]
    assert sp.metrics["bytes_spec"] == 0
    e.close()


def test_bf16_attention_margin_aware_vs_port(port):
    """bf16 vs the float64 port at C1 widths.  Through attention a single token's embedding (not a
    prefix mean) feeds the residual stream, and bf16 rounding of K/V, the attention output and the GEMM
    operands moves the logits by up to ~10% of their scale -- the bf16 CUDA-core path shows the same
    error, so the tcgen05 path is held to it: within 3% of the bf16 CUDA-core logits, within 15% of the
    port's, and every decision whose port margin exceeds the observed error (tokens: twice the max logit
    error of that prefix; routing: gate margin > 0.25) agrees."""
    from oracle.oracle import ModelSpec as OSpec
    from paper_2604_10152_b200.engine import GEMM_SIMT, GEMM_TCGEN05
    sp = dict(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, seed=0, expert_kind=SWIGLU3,
              attn_heads=8, kv_heads=2, head_dim=64, rope_theta=1e6)
    m = port.build(OSpec(**sp))
    e = Engine(_spec(sp), weight_type=BF16, gemm=GEMM_TCGEN05, max_batch=1, max_gamma=1, max_seq_len=64).init_exact()
    c = Engine(_spec(sp), weight_type=BF16, gemm=GEMM_SIMT, max_batch=1, max_gamma=1, max_seq_len=64).init_exact()
    rng = np.random.RandomState(4)
    rbig = rbad = tbig = tbad = 0
    worst = worst_cc = 0.0
    for _ in range(24):
        prefix = rng.randint(0, sp["vocab"], size=rng.randint(1, 16)).tolist()
        lg, raw, _ = e.forward(prefix)
        lc = c.forward(prefix)[0]
        rl, gates = m.forward_gates(prefix)
        rr = m.forward(prefix)[1]
        scale = np.max(np.abs(rl))
        err = float(np.max(np.abs(lg - rl)))
        worst = max(worst, err / scale)
        worst_cc = max(worst_cc, float(np.max(np.abs(lg - lc)) / scale))
        for l in range(gates.shape[0]):
            srt = np.sort(gates[l])[::-1]
            if srt[1] - srt[2] > 0.25:
                rbig += 1
                rbad += set(raw[l].tolist()) != set(rr[l].tolist())
        s2 = np.sort(rl)[::-1]
        if s2[0] - s2[1] > 2 * err:
            tbig += 1
            tbad += int(np.argmax(lg)) != int(np.argmax(rl))
    print(f"attention bf16: worst logit err vs port {worst:.4f}, vs bf16 CUDA-core {worst_cc:.4f}; "
          f"decisions checked {rbig} routing + {tbig} tokens")
    assert worst_cc <= 0.03 and worst <= 0.15
    assert rbad == 0 and tbad == 0 and rbig >= 30
    e.close()
    c.close()


def test_attention_offloaded_store_and_sampling():
    s = _c1_attn(SWIGLU3, seed=2)
    a = Engine(s, weight_type=BF16, max_batch=4, max_gamma=4, max_seq_len=96).init_device(9)
    b = Engine(s, weight_type=BF16, max_batch=4, max_gamma=4, max_seq_len=96, offload=1).init_device(9)
    a.build_affinity_device()
    b.build_affinity_device()
    prompts = make_prompts(2, 4, 8, s.vocab)
    cfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=20)
    ra, rb = a.run_specmoe(cfg, prompts), b.run_specmoe(cfg, prompts)
    assert ra.tokens == rb.tokens and ra.ledger == rb.ledger
    assert rb.metrics["h2d_expert_bytes"] == len(rb.ledger) * b.info()["bytes_per_expert"]  # prefill excluded
    scfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=20, mode="sampling", temperature=0.8, run_seed=3)
    s1, s2 = a.run_specmoe(scfg, prompts), a.run_specmoe(scfg, prompts)
    assert s1.tokens == s2.tokens and all(len(t) == 20 for t in s1.tokens)   # deterministic, complete
    o1 = a.run_ondemand(scfg, prompts)
    assert all(len(t) == 20 for t in o1.tokens)
    a.close()
    b.close()
