"""GPU parity tests: the sm_100a engine (through the C ABI) against the reference oracle.

Bars:
  * P1/P2 -- fp32 mode: routing indices (raw and post-remap), accepted counts, outcomes, greedy
    tokens, ledger and the modeled metrics equal the float64 reference bit for bit; logits agree
    within 2e-5 of the logit scale (fp32 vs fp64 arithmetic).
  * P3 -- bf16 mode (tcgen05): losslessness (speculative == on-demand on the same engine, exact),
    batch invariance, and tcgen05 vs CUDA-core GEMMs within bf16 tolerance.
"""
import json
import os

import numpy as np
import pytest

from paper_2604_10152_b200.engine import BF16, F32, GEMM_SIMT, GEMM_TCGEN05, SWIGLU3, TANH2, Engine, ModelSpec, RunCfg
from paper_2604_10152_b200.prompts import make_prompts

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
LOGIT_TOL = 2e-5  # fp32 engine vs float64 reference, relative to max |logit|


def gold(name):
    with open(os.path.join(GOLD, name + ".json")) as f:
        return json.load(f)


def run_dict(r, drop=("wall_s", "gpu_s", "h2d_expert_bytes", "h2d_s", "prefetch_bytes",
                        "prefetch_wasted_bytes")):
    return {"tokens": r.tokens, "ledger": [list(x) for x in r.ledger],
            "outcomes": [list(o[:5]) + [list(o[5])] for o in r.outcomes],
            "trace": [[t[0], t[1], t[2], list(t[3])] for t in r.trace],
            "hotness": r.hotness.tolist(),
            "metrics": {k: v for k, v in r.metrics.items() if k not in drop}}


def spec_of(d):
    return ModelSpec(**{k: v for k, v in d.items() if k in ModelSpec.__dataclass_fields__})


@pytest.fixture(scope="module")
def toy_engines():
    out = []
    for g in gold("toy"):
        e = Engine(spec_of(g["spec"]), weight_type=F32, max_batch=8, max_gamma=10).init_exact()
        out.append((g, e))
    yield out
    for _, e in out:
        e.close()


def test_f32_forward_matches_reference(toy_engines):
    g = gold("spec_forward")
    e = Engine(spec_of(g["spec"]), weight_type=F32, max_batch=1, max_gamma=1).init_exact()
    lg, raw, _ = e.forward(g["prefix"])
    ref = np.asarray(g["logits"])
    assert np.max(np.abs(lg - ref)) <= LOGIT_TOL * np.max(np.abs(ref))
    assert raw.tolist() == g["raw"]
    assert int(np.argmax(lg)) == int(np.argmax(ref))


@pytest.mark.parametrize("i", range(5))
def test_f32_affinity_bitexact(toy_engines, i):
    g, e = toy_engines[i]
    assert e.affinity().tolist() == g["affinity"]


@pytest.mark.parametrize("i", range(5))
def test_f32_specmoe_equals_reference(toy_engines, i):
    """run_specmoe (specdec.cpp:190-397) on the GPU == the reference, field for field."""
    g, e = toy_engines[i]
    cfg = RunCfg(**g["cfg"])
    got = run_dict(e.run_specmoe(cfg, g["prompts"]))
    want = g["specmoe"]
    for key in ("tokens", "outcomes", "trace", "ledger", "hotness", "metrics"):
        assert got[key] == want[key], key


@pytest.mark.parametrize("i", range(5))
def test_f32_ondemand_equals_reference(toy_engines, i):
    g, e = toy_engines[i]
    got = run_dict(e.run_ondemand(RunCfg(**g["cfg"]), g["prompts"]))
    assert got == g["ondemand"]


def test_f32_restricted_forward_remap_equals_oracle(toy_engines, port):
    """Draft semantics (model.cpp:237-246): affinity and hash-surrogate remaps, exact."""
    g, e = toy_engines[1]
    m = port.build(spec_of(g["spec"]))
    rng = np.random.RandomState(0)
    for trial in range(12):
        nd = [2, 3, 4, 8][trial % 4]
        sets = [sorted(rng.choice(16, nd, replace=False).tolist()) for _ in range(4)]
        prefix = rng.randint(0, 64, size=rng.randint(1, 12)).tolist()
        for aff in (True, False):
            lg, raw, fin = e.forward(prefix, sets, use_affinity=aff)
            rl, rr, rf = m.forward(prefix, sets, use_affinity=aff)
            assert raw.tolist() == rr.tolist() and fin.tolist() == rf.tolist()
            assert np.max(np.abs(lg - rl)) <= LOGIT_TOL * np.max(np.abs(rl))


def test_c1_f32_parity():
    """BASELINE configs[0] (L4 E8 K2 d512): tokens / routing trace / ledger equal the reference."""
    g = gold("c1")
    e = Engine(spec_of(g["spec"]), weight_type=F32, max_batch=1, max_gamma=4).init_exact()
    lg, raw, _ = e.forward(g["prompts"][0])
    ref = np.asarray(g["forward_logits"])
    assert np.max(np.abs(lg - ref)) <= LOGIT_TOL * np.max(np.abs(ref))
    assert raw.tolist() == g["forward_raw"]
    assert e.affinity().tolist() == g["affinity"]
    got = run_dict(e.run_specmoe(RunCfg(**g["cfg"]), g["prompts"]))
    for key in ("tokens", "outcomes", "trace", "ledger", "metrics"):
        assert got[key] == g["specmoe"][key], key


def test_f32_losslessness_many_seeds():
    """SPEC.md:512 acceptance 1 on the GPU: spec == on-demand for N in {2,4,8,16}, gamma in {5,10}."""
    for seed in range(6):
        s = ModelSpec(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.5, seed=seed)
        e = Engine(s, weight_type=F32, max_batch=2, max_gamma=10).init_exact()
        prompts = make_prompts(seed, 2, 8, 64)
        od = e.run_ondemand(RunCfg(max_new_tokens=20, run_seed=seed), prompts)
        for nd, gm in [(2, 5), (4, 10), (8, 5), (16, 10)]:
            sp = e.run_specmoe(RunCfg(gamma=gm, n_draft=nd, max_new_tokens=20, run_seed=seed), prompts)
            assert sp.tokens == od.tokens
            if nd == 16:
                assert all(o[2] == gm for o in sp.outcomes)
        e.close()


# ---------------------------------------------------------------- bf16 / tcgen05
def _c1_like(kind, skew=0.0):
    return ModelSpec(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, gate_skew=skew, seed=1,
                     expert_kind=kind)


@pytest.mark.parametrize("kind", [TANH2, SWIGLU3])
def test_tcgen05_matches_cuda_core_gemm(kind):
    """Same bf16 weights through the tcgen05 path and the CUDA-core path: logits within bf16 noise."""
    s = _c1_like(kind)
    a = Engine(s, weight_type=BF16, gemm=GEMM_TCGEN05, max_batch=4, max_gamma=4).init_device(7)
    b = Engine(s, weight_type=BF16, gemm=GEMM_SIMT, max_batch=4, max_gamma=4).init_device(7)
    for prefix in ([1, 2, 3], list(range(40)), [1000] * 9):
        la, ra, _ = a.forward(prefix)
        lb, rb, _ = b.forward(prefix)
        scale = np.max(np.abs(lb))
        assert np.max(np.abs(la - lb)) <= 3e-2 * scale, (np.max(np.abs(la - lb)), scale)
        assert np.mean(ra == rb) >= 0.75


@pytest.mark.parametrize("kind", [TANH2, SWIGLU3])
def test_bf16_lossless_and_batch_invariant(kind):
    """P3: on the tcgen05 engine, speculative output == on-demand output exactly, and every
    sequence's output is independent of the batch it runs in."""
    s = _c1_like(kind, skew=1.0)
    e = Engine(s, weight_type=BF16, max_batch=4, max_gamma=4).init_device(3)
    e.build_affinity_device()
    prompts = make_prompts(5, 4, 8, s.vocab)
    od = e.run_ondemand(RunCfg(gamma=4, max_new_tokens=24), prompts)
    sp = e.run_specmoe(RunCfg(gamma=4, n_draft=4, max_new_tokens=24), prompts)
    assert sp.tokens == od.tokens
    one = e.run_specmoe(RunCfg(gamma=4, n_draft=4, max_new_tokens=24), prompts[2:3])
    assert one.tokens[0] == sp.tokens[2]
    assert sp.metrics["bytes_spec"] == 0


# ---------------------------------------------------------------- C3: expert store (pinned host -> HBM)
@pytest.mark.parametrize("i", [1, 4])
def test_offload_store_f32_equals_reference(i):
    """Experts in pinned host DRAM, migrated per layer during verify: tokens/ledger still equal the
    reference, and the bytes physically copied == ledger bytes (fp32 tanh2: real bytes per expert ==
    the reference's 2*d*f*4)."""
    g = gold("toy")[i]
    s = spec_of(g["spec"])
    e = Engine(s, weight_type=F32, max_batch=8, max_gamma=10, offload=1, hbm_expert_slots=40).init_exact()
    assert e.affinity().tolist() == g["affinity"]
    cfg = RunCfg(**g["cfg"])
    r = e.run_specmoe(cfg, g["prompts"])
    got = run_dict(r)
    for key in ("tokens", "outcomes", "trace", "ledger", "metrics"):
        assert got[key] == g["specmoe"][key], key
    assert r.metrics["h2d_expert_bytes"] == r.metrics["bytes_total"]
    od = e.run_ondemand(cfg, g["prompts"])
    assert run_dict(od) == g["ondemand"]
    assert od.metrics["h2d_expert_bytes"] == od.metrics["bytes_total"]


@pytest.mark.parametrize("policy", ["hot_temporal", "random", "hot_global"])
def test_offload_bf16_matches_resident(policy):
    """Same device-initialised weights, HBM-resident vs offloaded store: identical tokens and
    ledger; migrated bytes == ledger entries x real bytes per expert."""
    s = _c1_like(SWIGLU3, skew=1.0)
    a = Engine(s, weight_type=BF16, max_batch=4, max_gamma=4).init_device(9)
    b = Engine(s, weight_type=BF16, max_batch=4, max_gamma=4, offload=1).init_device(9)
    a.build_affinity_device()
    b.build_affinity_device()
    assert np.array_equal(a.affinity(), b.affinity())
    prompts = make_prompts(2, 4, 8, s.vocab)
    cfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=16, policy=policy, warmup_steps=4)
    ra, rb = a.run_specmoe(cfg, prompts), b.run_specmoe(cfg, prompts)
    assert ra.tokens == rb.tokens and ra.ledger == rb.ledger and ra.outcomes == rb.outcomes
    bpe = b.info()["bytes_per_expert"]
    assert rb.metrics["h2d_expert_bytes"] == len(rb.ledger) * bpe
    assert rb.metrics["h2d_s"] > 0
    oa, ob = a.run_ondemand(cfg, prompts), b.run_ondemand(cfg, prompts)
    assert oa.tokens == ob.tokens == ra.tokens
    assert ob.metrics["h2d_expert_bytes"] == len(ob.ledger) * bpe


def test_offload_slot_exhaustion_is_reported():
    s = _c1_like(TANH2)
    e = Engine(s, weight_type=BF16, max_batch=2, max_gamma=4, offload=1, hbm_expert_slots=8).init_device(1)
    e.build_affinity_device()
    from paper_2604_10152_b200.engine import EngineError
    with pytest.raises(EngineError) as ei:
        e.run_specmoe(RunCfg(gamma=4, n_draft=4, max_new_tokens=8), make_prompts(0, 2, 8, s.vocab))
    assert ei.value.code == 2


# ---------------------------------------------------------------- breadth: configs and edge cases vs the oracle
CASES = [
    # (spec overrides, run cfg overrides, batch)
    (dict(num_layers=3, moe_mask=[0, 1, 1], experts=64, top_k=6, hidden=64, ffn=32, vocab=128, seed=5),
     dict(gamma=4, n_draft=8, max_new_tokens=14), 3),                                  # C4-like: E64 K6, dense layer 0
    (dict(num_layers=2, experts=8, top_k=2, hidden=32, ffn=64, vocab=64, seed=6),
     dict(gamma=1, n_draft=2, max_new_tokens=1), 2),                                   # gamma=1, N=K, 1 new token
    (dict(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.5, seed=7),
     dict(gamma=5, n_draft=4, max_new_tokens=17, use_affinity=False), 2),             # hash-surrogate remap
    (dict(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.5, seed=8),
     dict(gamma=3, n_draft=4, max_new_tokens=13, policy="hot_global", warmup_steps=5), 2),
    (dict(num_layers=4, experts=16, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.5, seed=9),
     dict(gamma=3, n_draft=4, max_new_tokens=13, policy="random"), 3),
    (dict(num_layers=3, experts=8, top_k=3, hidden=48, ffn=40, vocab=96, gate_skew=0.5, seed=10),
     dict(gamma=6, n_draft=3, max_new_tokens=20), 4),                                  # K=3, N=K, odd dims
    (dict(num_layers=4, experts=8, top_k=2, hidden=32, ffn=64, vocab=64, gate_skew=1.0, seed=11),
     dict(gamma=4, n_draft=2, max_new_tokens=16, device_capacity_bytes=(4 * 2 + 3) * 2 * 32 * 64 * 4), 2),  # eviction
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_f32_configs_equal_oracle(case, port):
    from oracle.oracle import ModelSpec as OSpec, OracleError, RunCfg as ORun
    sp, rc, B = CASES[case]
    ospec = OSpec(**sp)
    m = port.build(ospec)
    prompts = make_prompts(100 + case, B, 6, sp["vocab"])
    cfg = dict(rc, collect_trace=True, run_seed=case)
    try:
        want = m.run_specmoe(ORun(**cfg), prompts)
    except OracleError as ex:
        want = ex
    e = Engine(spec_of(sp), weight_type=F32, max_batch=B, max_gamma=cfg["gamma"]).init_exact()
    if isinstance(want, Exception):
        from paper_2604_10152_b200.engine import EngineError
        with pytest.raises(EngineError) as ei:
            e.run_specmoe(RunCfg(**cfg), prompts)
        assert ei.value.code == want.code
        return
    got = e.run_specmoe(RunCfg(**cfg), prompts)
    assert got.tokens == want.tokens
    assert got.outcomes == want.outcomes
    assert got.trace == want.trace
    assert got.ledger == want.ledger
    assert got.hotness.tolist() == want.hotness.tolist()
    for k, v in want.metrics.items():
        if k != "wall_s":
            assert got.metrics[k] == v, k
    od_w = m.run_ondemand(ORun(**cfg), prompts)
    od_g = e.run_ondemand(RunCfg(**cfg), prompts)
    assert od_g.tokens == od_w.tokens and od_g.ledger == od_w.ledger and od_g.trace == od_w.trace


def test_bf16_fine_grained_lossless():
    """C4-like shape on the tcgen05 path (E=64, K=6, dense first layer): lossless + batch invariant."""
    s = ModelSpec(num_layers=3, moe_mask=[0, 1, 1], experts=64, top_k=6, hidden=256, ffn=128, vocab=512, seed=4,
                  expert_kind=SWIGLU3)
    e = Engine(s, weight_type=BF16, max_batch=4, max_gamma=4).init_device(4)
    e.build_affinity_device()
    prompts = make_prompts(9, 4, 8, s.vocab)
    sp = e.run_specmoe(RunCfg(gamma=4, n_draft=8, max_new_tokens=20), prompts)
    od = e.run_ondemand(RunCfg(gamma=4, max_new_tokens=20), prompts)
    assert sp.tokens == od.tokens
    one = e.run_specmoe(RunCfg(gamma=4, n_draft=8, max_new_tokens=20), prompts[1:2])
    assert one.tokens[0] == sp.tokens[1]


# ---------------------------------------------------------------- expert parallelism (virtual ranks)
def _run_ep(G, spec, init, cfg, prompts, weight_type=BF16, ondemand=False, work_fn=None, offload=0):
    import threading
    from paper_2604_10152_b200.engine import LoopbackGroup
    grp = LoopbackGroup(G)
    engines = []
    for r in range(G):
        e = Engine(spec, weight_type=weight_type, max_batch=len(prompts), max_gamma=cfg.gamma, ep_rank=r, ep_world=G,
                   offload=offload)
        init(e)
        e.attach_loopback(grp)
        engines.append(e)
    out, errs = [None] * G, []

    def work(r):
        try:
            eng = engines[r]
            if work_fn is not None:
                out[r] = work_fn(eng)
            else:
                out[r] = eng.run_ondemand(cfg, prompts) if ondemand else eng.run_specmoe(cfg, prompts)
        except Exception as ex:  # pragma: no cover - surfaced below
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join(timeout=300) for t in th]
    assert not errs, errs
    return out


@pytest.fixture(params=["p2p", "a2a"])
def ep_mode(request):
    """Both exchange paths: fused peer-memory stores (default) and the all-to-all collectives."""
    with _env(SMOE_EP_MODE=request.param):
        yield request.param


@pytest.mark.parametrize("G", [2, 4])
def test_expert_parallel_bitexact_bf16(G, ep_mode):
    """Experts sharded over G virtual ranks (loopback transport, one GPU): every rank produces the
    single-GPU token stream, routing trace and ledger bit for bit."""
    s = _c1_like(SWIGLU3, skew=1.0)
    prompts = make_prompts(3, 3, 8, s.vocab)
    cfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=16, collect_trace=True)

    def init(e):
        e.init_device(11)
        e.build_affinity_device()

    one = Engine(s, weight_type=BF16, max_batch=3, max_gamma=4)
    init(one)
    want = one.run_specmoe(cfg, prompts)
    for r in _run_ep(G, s, init, cfg, prompts):
        assert r.tokens == want.tokens and r.trace == want.trace and r.ledger == want.ledger
        assert r.outcomes == want.outcomes


@pytest.mark.parametrize("G", [2, 4, 8])
def test_expert_parallel_fine_grained_bitexact(G, ep_mode):
    """C4-like shape (64 experts top-6, dense layer 0) with rows split over G ranks and the experts'
    rows exchanged by all-to-all: token stream, routing trace, ledger and forward() logits equal G = 1."""
    s = ModelSpec(num_layers=3, experts=64, top_k=6, hidden=256, ffn=256, vocab=512, expert_kind=SWIGLU3,
                  moe_mask=[0, 1, 1], gate_skew=0.5, seed=4)
    prompts = make_prompts(8, 5, 8, s.vocab)  # B=5: ragged row blocks at every G
    cfg = RunCfg(gamma=4, n_draft=8, max_new_tokens=12, collect_trace=True)

    def init(e):
        e.init_device(13)
        e.build_affinity_device()

    one = Engine(s, weight_type=BF16, max_batch=5, max_gamma=4)
    init(one)
    want = one.run_specmoe(cfg, prompts)
    want_lg = one.forward(prompts[2] + [7, 9])

    def work(e):
        r = e.run_specmoe(cfg, prompts)
        return r, e.forward(prompts[2] + [7, 9])
    for r, lg in _run_ep(G, s, init, cfg, prompts, work_fn=work):
        assert r.tokens == want.tokens and r.trace == want.trace and r.ledger == want.ledger
        assert np.array_equal(lg[0], want_lg[0]) and np.array_equal(lg[1], want_lg[1])


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("policy", ["hot_temporal", "random"])
def test_expert_parallel_offloaded_store(G, policy, ep_mode):
    """Expert parallelism with the offloaded store: every rank keeps its experts in its own
    pinned host pool and fetches needed ∩ owned per verify layer over its own PCIe link; hot_temporal
    re-pins per layer from the all-gathered counts.  Tokens, routing trace and ledger equal the
    single-GPU offloaded (and resident) runs, and the ranks' migrated bytes add up to the ledger."""
    s = _c1_like(SWIGLU3, skew=1.0)
    prompts = make_prompts(4, 3, 8, s.vocab)
    cfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=14, collect_trace=True, policy=policy)

    def init(e):
        e.init_device(21)
        e.build_affinity_device()

    one = Engine(s, weight_type=BF16, max_batch=3, max_gamma=4, offload=1)
    init(one)
    want = one.run_specmoe(cfg, prompts)
    bpe = one.info()["bytes_per_expert"]
    assert want.metrics["h2d_expert_bytes"] == len(want.ledger) * bpe
    res = _run_ep(G, s, init, cfg, prompts, offload=1)
    for r in res:
        assert r.tokens == want.tokens and r.trace == want.trace and r.ledger == want.ledger
        assert r.outcomes == want.outcomes
    assert sum(r.metrics["h2d_expert_bytes"] for r in res) == len(want.ledger) * bpe
    od = _run_ep(G, s, init, cfg, prompts, offload=1, ondemand=True)
    od1 = one.run_ondemand(cfg, prompts)
    assert od[0].tokens == od1.tokens == want.tokens and od[0].ledger == od1.ledger
    assert sum(r.metrics["h2d_expert_bytes"] for r in od) == len(od1.ledger) * bpe


@pytest.mark.slow
@pytest.mark.parametrize("G", [2, 8])
def test_expert_parallel_c5_slice_bitexact(G, ep_mode):
    """Two-layer slice of the Mixtral-8x22B shape (C5: d=6144, f=16384, V=32768, SwiGLU bf16), B=16:
    expert-parallel runs over G virtual ranks equal the single-engine run token for token."""
    s = ModelSpec(num_layers=2, experts=8, top_k=2, hidden=6144, ffn=16384, vocab=32768, expert_kind=SWIGLU3, seed=5)
    prompts = make_prompts(21, 16, 8, s.vocab)
    cfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=6, collect_trace=True)

    def init(e):
        e.init_device(17)
        e.build_affinity_device()

    one = Engine(s, weight_type=BF16, max_batch=16, max_gamma=4)
    init(one)
    want = one.run_specmoe(cfg, prompts)
    one.close()
    for r in _run_ep(G, s, init, cfg, prompts):
        assert r.tokens == want.tokens and r.trace == want.trace and r.ledger == want.ledger


def test_expert_parallel_f32_equals_reference():
    """fp32 exact weights sharded over 2 ranks: still equal to the reference golden run."""
    g = gold("toy")[1]
    s = spec_of(g["spec"])
    cfg = RunCfg(**g["cfg"])
    res = _run_ep(2, s, lambda e: e.init_exact(), cfg, g["prompts"], weight_type=F32)
    for r in res:
        got = run_dict(r)
        for key in ("tokens", "outcomes", "trace", "ledger", "metrics"):
            assert got[key] == g["specmoe"][key], key
    od = _run_ep(2, s, lambda e: e.init_exact(), cfg, g["prompts"], weight_type=F32, ondemand=True)
    assert run_dict(od[0]) == g["ondemand"]


@pytest.mark.slow
def test_mixtral_shape_lossless_b64():
    """The benchmark configuration itself (Mixtral-8x7B shape, SwiGLU bf16, B=64, gamma=4): the
    speculative token stream equals plain greedy decoding on the same engine, token for token."""
    s = ModelSpec(num_layers=32, experts=8, top_k=2, hidden=4096, ffn=14336, vocab=32000, expert_kind=SWIGLU3)
    e = Engine(s, weight_type=BF16, max_batch=64, max_gamma=4).init_device(0)
    e.build_affinity_device()
    prompts = make_prompts(1000, 64, 8, s.vocab)
    sp = e.run_specmoe(RunCfg(gamma=4, n_draft=4, max_new_tokens=6), prompts)
    od = e.run_ondemand(RunCfg(gamma=4, max_new_tokens=6), prompts)
    assert sp.tokens == od.tokens
    assert sp.metrics["tokens_total"] == 64 * 6
    e.close()


def test_bf16_agreement_with_oracle_margin_aware(port):
    """P3 (ii)/(iii): the bf16 tcgen05 engine on the reference's own weights (C1 shape) agrees with the
    float64 oracle on every routing decision whose oracle gate margin (K-th minus (K+1)-th gate
    logit) exceeds 0.05, and on every greedy token whose logit margin exceeds 0.1; logits within 3% of
    the logit scale.  The near-tie rates are reported (bf16 rounding can flip genuine near-ties)."""
    from oracle.oracle import ModelSpec as OSpec
    sp = dict(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, seed=0)
    m = port.build(OSpec(**sp))
    e = Engine(spec_of(sp), weight_type=BF16, max_batch=1, max_gamma=1).init_exact()
    rng = np.random.RandomState(1)
    route_total = route_big = route_bad = tok_big = tok_bad = 0
    worst = 0.0
    for trial in range(60):
        prefix = rng.randint(0, sp["vocab"], size=rng.randint(1, 24)).tolist()
        lg, raw, _ = e.forward(prefix)
        rl, gates = m.forward_gates(prefix)
        rr = m.forward(prefix)[1]
        worst = max(worst, float(np.max(np.abs(lg - rl)) / np.max(np.abs(rl))))
        for l in range(gates.shape[0]):
            srt = np.sort(gates[l])[::-1]
            margin = srt[sp["top_k"] - 1] - srt[sp["top_k"]]
            route_total += 1
            if margin > 0.05:
                route_big += 1
                route_bad += set(raw[l].tolist()) != set(rr[l].tolist())
        s2 = np.sort(rl)[::-1]
        if s2[0] - s2[1] > 0.1:
            tok_big += 1
            tok_bad += int(np.argmax(lg)) != int(np.argmax(rl))
    print(f"bf16 vs oracle: worst logit err {worst:.4f}; routing near-tie rate {1 - route_big / route_total:.3f}; "
          f"token near-tie rate {1 - tok_big / 60:.3f}")
    assert worst <= 0.03
    assert route_bad == 0 and tok_bad == 0


# ---------------------------------------------------------------- launch-shape switches
class _env:
    """Set engine environment switches for the engines constructed inside the block."""

    def __init__(self, **kv):
        self.kv = {k: str(v) for k, v in kv.items()}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update(self.kv)

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("env", ["SMOE_ROW_CLUSTER=1", "SMOE_ROW_THREADS=256", "SMOE_GATE_STAGE=0",
                                 "SMOE_TC_PAIR=0", "SMOE_TC_PAIR_DOWN=0", "SMOE_TC_PAIR_SINGLE=2",
                                 "SMOE_TILED=0", "SMOE_W_EVICT_FIRST=0", "SMOE_PF_PRED=0", "SMOE_PDL=0",
                                 "SMOE_ROW_WIDE=0", "SMOE_GRAPH=0", "SMOE_GATE_RG=0", "SMOE_GATE_RG=2", "SMOE_STATIC_FIRST=0"])
def test_launch_shape_switches_bitexact(env):
    """Launch-shape switches change how the work is laid out on the GPU (row clusters with DSMEM
    reductions, fewer row threads playing the same reduction tree, gate weights staged in shared
    memory, pair units, L2 prefetch, PDL) but never the arithmetic: logits, routing and token streams
    are bit-identical to the default launch shapes."""
    import subprocess
    import sys
    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "launch_digest.py")

    def run(extra):
        env_ = dict(os.environ)
        env_.update(extra)
        out = subprocess.run([sys.executable, script], env=env_, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        return json.loads(out.stdout.strip().splitlines()[-1])

    k, v = env.split("=")
    if "base" not in _DIGEST_BASE:
        _DIGEST_BASE["base"] = run({})
    assert run({k: v}) == _DIGEST_BASE["base"]


_DIGEST_BASE = {}
