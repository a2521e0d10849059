// caller.cpp -- a client of the reference C++ API (/root/reference/proj/core/include/specmoe).
//
// The SAME source is compiled twice:
//   * against the reference headers + sources      -> tests/golden/cpp_caller.json (make_golden.py)
//   * against include/specmoe/ + libspecmoe_b200.so -> run on the B200 (tests/test_cpp_dropin.py)
// and the two outputs must agree (integers exactly, logits within the fp32 tolerance): the drop-in
// claim of the B200 engine, exercised through the reference's own interface.
#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

#include "specmoe/baselines.hpp"
#include "specmoe/drafting.hpp"
#include "specmoe/memsim.hpp"
#include "specmoe/model.hpp"
#include "specmoe/specdec.hpp"

using namespace specmoe;

static std::string ints(const std::vector<int>& v) {
    std::string s = "[";
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    return s + "]";
}
static std::string nested(const std::vector<std::vector<int>>& v) {
    std::string s = "[";
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + ints(v[i]);
    return s + "]";
}
static std::string dbl(double x) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", x);
    return b;
}
static std::string run_json(const RunResult& r) {
    std::string s = "{\"tokens\":" + nested(r.tokens) + ",\"ledger\":[";
    for (size_t i = 0; i < r.ledger.entries().size(); ++i) {
        const auto& e = r.ledger.entries()[i];
        s += (i ? "," : "") + std::string("[\"") + to_string(e.phase) + "\"," + std::to_string(e.step) + "," +
             std::to_string(e.key.layer) + "," + std::to_string(e.key.expert) + "," + std::to_string(e.bytes) + "]";
    }
    s += "],\"outcomes\":[";
    for (size_t i = 0; i < r.outcomes.size(); ++i) {
        const auto& o = r.outcomes[i];
        s += (i ? "," : "") + std::string("[") + std::to_string(o.seq) + "," + std::to_string(o.phase) + "," +
             std::to_string(o.accepted) + "," + std::to_string(o.correction) + "," +
             std::to_string(o.tokens_generated) + "," + ints(o.drafts) + "]";
    }
    const RunMetrics& m = r.metrics;
    s += "],\"trace_rows\":" + std::to_string(r.trace.size()) + ",\"metrics\":{\"tau_mean\":" + dbl(m.tau_mean) +
         ",\"tokens_total\":" + std::to_string(m.tokens_total) + ",\"phases\":" + std::to_string(m.phases) +
         ",\"modeled_seconds\":" + dbl(m.modeled_seconds) + ",\"bytes_total\":" + std::to_string(m.bytes_total) +
         ",\"bytes_verify\":" + std::to_string(m.bytes_verify) + ",\"bytes_baseline\":" + std::to_string(m.bytes_baseline) +
         ",\"setup_bytes\":" + std::to_string(m.setup_bytes) + ",\"warmup_bytes\":" + std::to_string(m.warmup_bytes) +
         ",\"lambda\":" + dbl(m.lambda) + ",\"c_measured\":" + dbl(m.c_measured) + "}}";
    return s;
}

int main() {
    ModelSpec spec;  // SPEC.md toy defaults: L4 E16 K2 d32 f64 V64
    spec.gate_skew = 1.5;
    spec.seed = 21;
    ModelWeights w = build_model(spec);
    AffinityTable aff = build_affinity_table(w);
    std::stringstream csv;
    save_affinity_csv(aff, csv);
    AffinityTable aff2 = load_affinity_csv(csv);

    TierConfig tier;
    tier.bytes_per_expert = bytes_per_expert(spec);
    tier.device_capacity_bytes = (uint64_t)spec.moe_layer_count() * spec.experts_per_block * tier.bytes_per_expert;
    SpecConfig cfg;
    cfg.gamma = 5;
    cfg.n_draft = 4;
    cfg.max_new_tokens = 20;
    std::vector<std::vector<int>> prompts = {{1, 2, 3, 4, 5, 6, 7, 8}, {9, 8, 7, 6, 5, 4, 3, 2}, {63, 0, 17, 17, 4, 4, 40, 2}};
    cfg.batch = (int)prompts.size();

    std::printf("{");
    // forward: target and draft semantics
    ForwardResult f0 = forward(w, std::vector<int>{3, 1, 4, 1, 5});
    RestrictedExperts rx{{{0, 2, 5, 9}, {1, 3, 5, 7}, {2, 4, 6, 8}, {0, 1, 14, 15}}};
    ForwardResult f1 = forward(w, std::vector<int>{3, 1, 4, 1, 5}, &rx, &aff2);
    std::printf("\"forward\":{\"argmax\":%d,\"logits\":[", greedy_next(f0.logits));
    for (size_t i = 0; i < f0.logits.size(); ++i) std::printf("%s%.17g", i ? "," : "", f0.logits[i]);
    std::printf("],\"raw\":[");
    for (size_t l = 0; l < f0.activations.size(); ++l) std::printf("%s%s", l ? "," : "", ints(f0.activations[l].raw).c_str());
    std::printf("],\"restricted_final\":[");
    for (size_t l = 0; l < f1.activations.size(); ++l) std::printf("%s%s", l ? "," : "", ints(f1.activations[l].final).c_str());
    std::printf("],\"restricted_argmax\":%d},", greedy_next(f1.logits));
    // speculate / verify_greedy
    DraftState ds;
    ds.n_draft = 4;
    ds.sets = rx.per_layer;
    Rng rng(7);
    SpeculationResult sr = speculate(w, ds, &aff, prompts, 4, DecodeMode::greedy, 1.0, rng);
    std::printf("\"speculate\":{\"drafts\":%s,\"distinct\":[", nested(sr.drafts).c_str());
    for (size_t t = 0; t < sr.distinct_draft_experts.size(); ++t) std::printf("%s%llu", t ? "," : "", (unsigned long long)sr.distinct_draft_experts[t]);
    std::printf("]},");
    VerifyResult vr = verify_greedy(w, prompts[0], sr.drafts[0]);
    std::printf("\"verify\":{\"accepted\":%d,\"correction\":%d,\"pos0_raw\":%s},", vr.accepted, vr.correction,
                ints(vr.positions.rows[0][0].raw).c_str());
    // the loops
    for (DraftPolicy p : {DraftPolicy::hot_temporal, DraftPolicy::random, DraftPolicy::hot_global}) {
        SpecConfig c = cfg;
        c.warmup_steps = 6;
        std::printf("\"specmoe_%s\":%s,", to_string(p), run_json(run_specmoe(w, c, p, tier, prompts, 5, &aff, true)).c_str());
    }
    std::printf("\"ondemand\":%s,", run_json(run_ondemand(w, prompts, cfg, tier, 5, false)).c_str());
    std::printf("\"overlap\":%s,", run_json(run_overlap(w, prompts, cfg, tier, 5, false)).c_str());
    BaselineConfig bc;
    bc.kind = BaselineKind::caching;
    bc.cache_fraction = 0.25;
    bc.warmup_steps = 6;
    std::printf("\"caching\":%s,", run_json(run_caching(w, prompts, cfg, tier, bc, 5, false)).c_str());
    // error behaviour: ConfigError / InvariantError types
    int cfg_err = 0, inv_err = 0;
    try { SpecConfig bad = cfg; bad.gamma = 0; run_specmoe(w, bad, DraftPolicy::hot_temporal, tier, prompts, 0, &aff); }
    catch (const ConfigError&) { cfg_err = 1; }
    try { forward(w, std::vector<int>{}); } catch (const InvariantError&) { inv_err = 1; }
    std::printf("\"errors\":{\"config\":%d,\"invariant\":%d},", cfg_err, inv_err);
    std::printf("\"speedup\":%s}\n", dbl(speedup_eq2(7.265, 10, 0.05, 2.0)).c_str());
    return 0;
}
