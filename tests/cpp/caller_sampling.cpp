// caller_sampling.cpp -- sampling-mode client of the reference C++ API (specdec.cpp:82-157,
// model.cpp:178-190).  Compiled against the reference (tests/golden/cpp_caller_sampling.json) and
// against include/specmoe/ + libspecmoe_b200.so (tests/test_cpp_dropin.py): the draws follow the
// reference's RNG consumption order, so tokens, acceptances and the ledger must agree exactly.
#include <cstdio>
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
static std::string run_json(const RunResult& r) {
    std::string s = "{\"tokens\":" + nested(r.tokens) + ",\"outcomes\":[";
    for (size_t i = 0; i < r.outcomes.size(); ++i) {
        const auto& o = r.outcomes[i];
        s += (i ? "," : "") + std::string("[") + std::to_string(o.seq) + "," + std::to_string(o.phase) + "," +
             std::to_string(o.accepted) + "," + std::to_string(o.correction) + "," + ints(o.drafts) + "]";
    }
    s += "],\"bytes_total\":" + std::to_string(r.metrics.bytes_total) + ",\"ledger_entries\":" +
         std::to_string(r.ledger.entries().size()) + ",\"phases\":" + std::to_string(r.metrics.phases) + "}";
    return s;
}

int main() {
    ModelSpec spec;  // SPEC.md toy: L4 E16 K2 d32 f64 V64
    spec.gate_skew = 1.0;
    spec.seed = 33;
    ModelWeights w = build_model(spec);
    AffinityTable aff = build_affinity_table(w);
    TierConfig tier;
    tier.bytes_per_expert = bytes_per_expert(spec);
    tier.device_capacity_bytes = (uint64_t)spec.moe_layer_count() * spec.experts_per_block * tier.bytes_per_expert;
    std::vector<std::vector<int>> prompts = {{5, 6, 7, 8, 1, 2, 3, 4}, {40, 41, 42, 43, 44, 45, 46, 47},
                                             {0, 63, 0, 63, 0, 63, 0, 63}, {9, 9, 9, 9, 9, 9, 9, 9}};
    std::printf("{");
    // sample_next on a fixed distribution
    {
        Rng rng(123);
        std::vector<double> lg{0.5, -1.0, 2.0, 0.0, 1.5, -0.5};
        std::vector<int> draws;
        for (int i = 0; i < 24; ++i) draws.push_back(sample_next(lg, 0.8, rng));
        std::printf("\"sample_next\":%s,", ints(draws).c_str());
    }
    // speculate + verify_sampling for one batch
    {
        DraftState ds;
        ds.n_draft = 4;
        ds.sets = {{0, 2, 5, 9}, {1, 3, 5, 7}, {2, 4, 6, 8}, {0, 1, 14, 15}};
        Rng rng(9);
        SpeculationResult sr = speculate(w, ds, &aff, prompts, 4, DecodeMode::sampling, 1.0, rng);
        std::printf("\"spec_drafts\":%s,\"verify\":[", nested(sr.drafts).c_str());
        for (size_t s = 0; s < prompts.size(); ++s) {
            VerifyResult v = verify_sampling(w, prompts[s], sr.drafts[s], sr.draw_probs[s], 1.0, rng);
            std::printf("%s[%d,%d]", s ? "," : "", v.accepted, v.correction);
        }
        std::printf("],");
    }
    // the loops in sampling mode
    for (double temp : {1.0, 0.7}) {
        SpecConfig cfg;
        cfg.gamma = 4;
        cfg.n_draft = 4;
        cfg.max_new_tokens = 16;
        cfg.mode = DecodeMode::sampling;
        cfg.temperature = temp;
        cfg.batch = (int)prompts.size();
        cfg.warmup_steps = 4;
        const std::string t = temp == 1.0 ? "t10" : "t07";
        std::printf("\"specmoe_%s\":%s,", t.c_str(),
                    run_json(run_specmoe(w, cfg, DraftPolicy::hot_temporal, tier, prompts, 11, &aff)).c_str());
        std::printf("\"specmoe_hash_%s\":%s,", t.c_str(),
                    run_json(run_specmoe(w, [&] { SpecConfig c = cfg; c.use_affinity = false; return c; }(),
                                         DraftPolicy::random, tier, prompts, 12, nullptr)).c_str());
        std::printf("\"ondemand_%s\":%s%s", t.c_str(), run_json(run_ondemand(w, prompts, cfg, tier, 11)).c_str(),
                    temp == 1.0 ? "," : "");
    }
    std::printf("}\n");
    return 0;
}
