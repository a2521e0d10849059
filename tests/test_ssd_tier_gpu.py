"""The SSD tier of the expert store (offload=2; the reference's TierConfig.ssd_bandwidth regime,
memsim.hpp:31-37): every expert of the model in a file on local storage (O_DIRECT when
the filesystem allows), read through pinned staging chunks into the HBM slots.  Same token streams,
routing and ledger as the pinned-DRAM tier and the resident model; the bytes moved equal the ledger."""
import pytest

from paper_2604_10152_b200.engine import BF16, F32, SWIGLU3, Engine, ModelSpec, RunCfg
from paper_2604_10152_b200.prompts import make_prompts

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("wt", [F32, BF16])
def test_ssd_tier_equals_dram_tier_and_resident(wt):
    s = ModelSpec(num_layers=4, experts=8, top_k=2, hidden=512, ffn=1024, vocab=1024, gate_skew=1.0, seed=3,
                  expert_kind=SWIGLU3)
    engines = [Engine(s, weight_type=wt, max_batch=4, max_gamma=4, offload=o).init_device(7) for o in (0, 1, 2)]
    for e in engines:
        e.build_affinity_device()
    prompts = make_prompts(6, 4, 8, s.vocab)
    cfg = RunCfg(gamma=4, n_draft=4, max_new_tokens=16, collect_trace=True, ssd_bandwidth=7e9)
    res = [e.run_specmoe(cfg, prompts) for e in engines]
    for r in res[1:]:
        assert r.tokens == res[0].tokens and r.trace == res[0].trace and r.ledger == res[0].ledger
    bpe = engines[2].info()["bytes_per_expert"]
    assert res[2].metrics["h2d_expert_bytes"] == len(res[2].ledger) * bpe == res[1].metrics["h2d_expert_bytes"]
    assert res[2].metrics["modeled_seconds"] == res[0].metrics["modeled_seconds"]  # ssd_bandwidth cost model
    od = [e.run_ondemand(cfg, prompts) for e in engines[1:]]
    assert od[0].tokens == od[1].tokens == res[0].tokens and od[0].ledger == od[1].ledger
    for e in engines:
        e.close()
