// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Flat C adapter (oracle/oracle_abi.h) over the reference's own C++ sources, which
// oracle/Makefile compiles directly from /root/reference/proj/core/src into
// oracle/_ref/libspecmoe_ref.so.  Nothing here re-implements the algorithm: every call
// forwards to the reference (specmoe::build_model, forward, run_specmoe, run_ondemand, ...)
// and only converts types.  It is the checker for the restatement (oracle/specmoe_oracle.c)
// and for the B200 engine, and the CPU baseline timed by bench.py.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <set>
#include <span>
#include <thread>
#include <vector>

#include "oracle_abi.h"
#include "specmoe/baselines.hpp"
#include "specmoe/drafting.hpp"
#include "specmoe/memsim.hpp"
#include "specmoe/model.hpp"
#include "specmoe/specdec.hpp"

using namespace specmoe;

namespace {

int report(const std::exception& e, char* err, int errlen) {
    if (err && errlen > 0) std::snprintf(err, errlen, "%s", e.what());
    if (dynamic_cast<const ConfigError*>(&e)) return 1;
    if (dynamic_cast<const InvariantError*>(&e)) return 2;
    return 3;
}

TierConfig tier_of(const om_run_cfg* c) {
    TierConfig t;
    t.device_capacity_bytes = c->device_capacity_bytes;
    t.host_bandwidth = c->host_bandwidth;
    t.ssd_bandwidth = c->ssd_bandwidth;
    t.bytes_per_expert = c->bytes_per_expert;
    t.compute_rate_tokens_per_s = c->compute_rate;
    t.compute_cost_per_active_expert_s = c->compute_cost_per_expert;
    return t;
}

SpecConfig spec_of(const om_run_cfg* c, int B, int plen) {
    SpecConfig s;
    s.gamma = c->gamma;
    s.n_draft = c->n_draft;
    s.mode = DecodeMode::greedy;
    s.batch = B;
    s.max_new_tokens = c->max_new_tokens;
    s.prompt_len = plen;
    s.use_affinity = c->use_affinity != 0;
    s.warmup_steps = c->warmup_steps;
    return s;
}

std::vector<std::vector<int>> prompts_of(const int* p, int B, int plen) {
    std::vector<std::vector<int>> v(B);
    for (int b = 0; b < B; ++b) v[b].assign(p + (size_t)b * plen, p + (size_t)(b + 1) * plen);
    return v;
}

om_result* flatten(const RunResult& rr, int B, int max_new, int M, int E, int K, int gamma, double wall) {
    om_result* r = static_cast<om_result*>(std::calloc(1, sizeof(om_result)));
    r->B = B; r->max_new = max_new; r->moe_layers = M; r->experts = E; r->top_k = K; r->gamma = gamma;
    r->tokens = static_cast<int*>(std::calloc((size_t)B * max_new + 1, sizeof(int)));
    r->n_tokens = static_cast<int*>(std::calloc((size_t)B, sizeof(int)));
    for (int b = 0; b < B; ++b) {
        r->n_tokens[b] = (int)rr.tokens[b].size();
        for (size_t i = 0; i < rr.tokens[b].size() && (int)i < max_new; ++i) r->tokens[(size_t)b * max_new + i] = rr.tokens[b][i];
    }
    const auto& le = rr.ledger.entries();
    r->n_ledger = (int)le.size();
    r->ledger = static_cast<om_ledger_entry*>(std::calloc(le.size() + 1, sizeof(om_ledger_entry)));
    for (size_t i = 0; i < le.size(); ++i)
        r->ledger[i] = om_ledger_entry{static_cast<int>(le[i].phase), le[i].step, le[i].key.layer, le[i].key.expert, le[i].bytes};
    r->n_outcomes = (int)rr.outcomes.size();
    r->outcomes = static_cast<om_outcome*>(std::calloc(rr.outcomes.size() + 1, sizeof(om_outcome)));
    r->outcome_drafts = static_cast<int*>(std::calloc(rr.outcomes.size() * (size_t)gamma + 1, sizeof(int)));
    for (size_t i = 0; i < rr.outcomes.size(); ++i) {
        const auto& o = rr.outcomes[i];
        r->outcomes[i] = om_outcome{o.seq, o.phase, o.accepted, o.correction, o.tokens_generated};
        for (int j = 0; j < gamma && j < (int)o.drafts.size(); ++j) r->outcome_drafts[i * gamma + j] = o.drafts[j];
    }
    r->n_trace = (int)rr.trace.size();
    r->trace = static_cast<int*>(std::calloc(rr.trace.size() * (3 + K) + 1, sizeof(int)));
    for (size_t i = 0; i < rr.trace.size(); ++i) {
        int* t = r->trace + i * (3 + K);
        t[0] = rr.trace[i].step; t[1] = rr.trace[i].seq; t[2] = rr.trace[i].layer;
        for (int k = 0; k < K; ++k) t[3 + k] = rr.trace[i].experts[k];
    }
    r->hotness = static_cast<uint64_t*>(std::calloc((size_t)M * E + 1, sizeof(uint64_t)));
    for (int l = 0; l < M && l < (int)rr.hotness.counts.size(); ++l)
        for (int e = 0; e < E; ++e) r->hotness[(size_t)l * E + e] = rr.hotness.counts[l][e];
    const RunMetrics& m = rr.metrics;
    r->tau_mean = m.tau_mean; r->tokens_total = m.tokens_total; r->phases = m.phases;
    r->speculation_s = m.speculation_s; r->verification_s = m.verification_s;
    r->modeled_seconds = m.modeled_seconds; r->tokens_per_sec = m.tokens_per_sec;
    r->bytes_spec = m.bytes_spec; r->bytes_verify = m.bytes_verify; r->bytes_baseline = m.bytes_baseline;
    r->bytes_total = m.bytes_total; r->setup_bytes = m.setup_bytes; r->warmup_bytes = m.warmup_bytes;
    r->lambda = m.lambda; r->c_measured = m.c_measured; r->wall_s = wall;
    return r;
}

}  // namespace

extern "C" {

void* om_build_model(const om_spec* s, char* err, int errlen) {
    try {
        if (s->expert_kind != 0) throw ConfigError("reference supports only the tanh2 expert");
        if (s->attn_heads > 0) throw ConfigError("reference has no attention (prefix-mean surrogate only)");
        ModelSpec spec;
        spec.num_layers = s->num_layers;
        if (s->moe_mask) spec.moe_layer_mask.assign(s->moe_mask, s->moe_mask + s->num_layers);
        spec.experts_per_block = s->experts;
        spec.top_k = s->top_k;
        spec.hidden_dim = s->hidden;
        spec.ffn_dim = s->ffn;
        spec.vocab_size = s->vocab;
        spec.gate_skew = s->gate_skew;
        spec.seed = s->seed;
        return new ModelWeights(build_model(spec));
    } catch (const std::exception& e) {
        report(e, err, errlen);
        return nullptr;
    }
}

void om_free_model(void* m) { delete static_cast<ModelWeights*>(m); }

long long om_get_tensor(void* model, const char* name, int layer, int expert, double* out, long long cap) {
    const ModelWeights& w = *static_cast<ModelWeights*>(model);
    const std::vector<double>* v = nullptr;
    if (!std::strcmp(name, "embedding")) v = &w.embedding;
    else if (!std::strcmp(name, "head")) v = &w.head;
    else {
        if (layer < 0 || layer >= (int)w.layers.size()) return -1;
        const LayerWeights& L = w.layers[layer];
        if (!std::strcmp(name, "mix")) v = &L.mix;
        else if (!std::strcmp(name, "gate")) v = &L.gate;
        else if (!std::strcmp(name, "gate_bias")) v = &L.gate_bias;
        else {
            const ExpertWeights* x = nullptr;
            if (expert < 0) x = L.is_moe ? nullptr : &L.ffn;
            else if (L.is_moe && expert < (int)L.experts.size()) x = &L.experts[expert];
            if (!x) return -1;
            if (!std::strcmp(name, "up")) v = &x->up;
            else if (!std::strcmp(name, "down")) v = &x->down;
        }
    }
    if (!v || v->empty()) return -1;
    if (out) {
        if (cap < (long long)v->size()) return -1;
        std::memcpy(out, v->data(), v->size() * sizeof(double));
    }
    return (long long)v->size();
}

void* om_build_affinity(void* model) { return new AffinityTable(build_affinity_table(*static_cast<ModelWeights*>(model))); }
void om_free_affinity(void* a) { delete static_cast<AffinityTable*>(a); }
int om_affinity_get(void* p, double* out, long long cap) {
    const AffinityTable& a = *static_cast<AffinityTable*>(p);
    long long n = 0;
    for (const auto& d : a.dist) n += (long long)d.size();
    if (cap < n) return -1;
    for (const auto& d : a.dist) {
        std::memcpy(out, d.data(), d.size() * sizeof(double));
        out += d.size();
    }
    return 0;
}

int om_forward(void* model, const int* prefix, int n, const int* restricted, int nd, void* aff, double* logits,
               int* raw_out, int* final_out, char* err, int errlen) {
    try {
        const ModelWeights& w = *static_cast<ModelWeights*>(model);
        RestrictedExperts rx;
        if (restricted) {
            int M = w.spec.moe_layer_count();
            rx.per_layer.resize(M);
            for (int l = 0; l < M; ++l) rx.per_layer[l].assign(restricted + (size_t)l * nd, restricted + (size_t)(l + 1) * nd);
        }
        ForwardResult fr = forward(w, std::span<const int>(prefix, (size_t)n), restricted ? &rx : nullptr,
                                   static_cast<const AffinityTable*>(aff));
        std::memcpy(logits, fr.logits.data(), fr.logits.size() * sizeof(double));
        const int K = w.spec.top_k;
        for (size_t l = 0; l < fr.activations.size(); ++l)
            for (int k = 0; k < K; ++k) {
                if (raw_out) raw_out[l * K + k] = fr.activations[l].raw[k];
                if (final_out) final_out[l * K + k] = fr.activations[l].final[k];
            }
        return 0;
    } catch (const std::exception& e) {
        return report(e, err, errlen);
    }
}

om_result* om_run_specmoe(void* model, const om_run_cfg* c, const int* prompts, int B, int plen, void* aff,
                          char* err, int errlen) {
    try {
        const ModelWeights& w = *static_cast<ModelWeights*>(model);
        auto t0 = std::chrono::steady_clock::now();
        RunResult rr = run_specmoe(w, spec_of(c, B, plen), static_cast<DraftPolicy>(c->policy), tier_of(c),
                                   prompts_of(prompts, B, plen), c->run_seed, static_cast<const AffinityTable*>(aff),
                                   c->collect_trace != 0);
        double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return flatten(rr, B, c->max_new_tokens, w.spec.moe_layer_count(), w.spec.experts_per_block, w.spec.top_k,
                       c->gamma, wall);
    } catch (const std::exception& e) {
        report(e, err, errlen);
        return nullptr;
    }
}

om_result* om_run_ondemand(void* model, const om_run_cfg* c, const int* prompts, int B, int plen, char* err,
                           int errlen) {
    try {
        const ModelWeights& w = *static_cast<ModelWeights*>(model);
        auto t0 = std::chrono::steady_clock::now();
        RunResult rr = run_ondemand(w, prompts_of(prompts, B, plen), spec_of(c, B, plen), tier_of(c), c->run_seed,
                                    c->collect_trace != 0);
        double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return flatten(rr, B, c->max_new_tokens, w.spec.moe_layer_count(), w.spec.experts_per_block, w.spec.top_k, 0,
                       wall);
    } catch (const std::exception& e) {
        report(e, err, errlen);
        return nullptr;
    }
}

om_result* om_run_overlap(void* model, const om_run_cfg* c, const int* prompts, int B, int plen, char* err,
                          int errlen) {
    try {
        const ModelWeights& w = *static_cast<ModelWeights*>(model);
        auto t0 = std::chrono::steady_clock::now();
        RunResult rr = run_overlap(w, prompts_of(prompts, B, plen), spec_of(c, B, plen), tier_of(c), c->run_seed,
                                   c->collect_trace != 0);
        double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return flatten(rr, B, c->max_new_tokens, w.spec.moe_layer_count(), w.spec.experts_per_block, w.spec.top_k, 0,
                       wall);
    } catch (const std::exception& e) {
        report(e, err, errlen);
        return nullptr;
    }
}

om_result* om_run_caching(void* model, const om_run_cfg* c, double cache_fraction, const int* prompts, int B,
                          int plen, char* err, int errlen) {
    try {
        const ModelWeights& w = *static_cast<ModelWeights*>(model);
        BaselineConfig bc;
        bc.kind = BaselineKind::caching;
        bc.cache_fraction = cache_fraction;
        bc.warmup_steps = c->warmup_steps;
        auto t0 = std::chrono::steady_clock::now();
        RunResult rr = run_caching(w, prompts_of(prompts, B, plen), spec_of(c, B, plen), tier_of(c), bc, c->run_seed,
                                   c->collect_trace != 0);
        double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return flatten(rr, B, c->max_new_tokens, w.spec.moe_layer_count(), w.spec.experts_per_block, w.spec.top_k, 0,
                       wall);
    } catch (const std::exception& e) {
        report(e, err, errlen);
        return nullptr;
    }
}

double om_time_forward(void* model, const int* prefix, int n, int threads, int iters) {
    try {
        const ModelWeights& w = *static_cast<ModelWeights*>(model);
        std::span<const int> p(prefix, (size_t)n);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int i = 0; i < threads; ++i)
            th.emplace_back([&] {
                for (int it = 0; it < iters; ++it) (void)forward(w, p);
            });
        for (auto& t : th) t.join();
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    } catch (const std::exception&) {
        return -1.0;
    }
}

void om_free_result(om_result* r) {
    if (!r) return;
    std::free(r->tokens); std::free(r->n_tokens); std::free(r->ledger); std::free(r->outcomes);
    std::free(r->outcome_drafts); std::free(r->trace); std::free(r->hotness);
    std::free(r);
}

int om_route_topk(const double* l, int n, int k, int* out) {
    try {
        auto v = route_topk(std::span<const double>(l, (size_t)n), k);
        std::memcpy(out, v.data(), v.size() * sizeof(int));
        return 0;
    } catch (const std::exception& e) { return -report(e, nullptr, 0); }
}
int om_greedy_next(const double* l, int n) {
    try { return greedy_next(std::span<const double>(l, (size_t)n)); }
    catch (const std::exception& e) { return -report(e, nullptr, 0); }
}
int om_softmax(const double* l, int n, double* out) {
    try {
        auto p = softmax(std::span<const double>(l, (size_t)n));
        std::memcpy(out, p.data(), p.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) { return -report(e, nullptr, 0); }
}
int om_nearest_draft_expert(const double* dist_l, int E, int raw, const int* ds, int nd, const int* ex, int nex) {
    try {
        AffinityTable t;
        t.experts = E;
        t.dist.emplace_back(dist_l, dist_l + (size_t)E * E);
        return nearest_draft_expert(t, 0, raw, std::span<const int>(ds, (size_t)nd), std::span<const int>(ex, (size_t)nex));
    } catch (const std::exception& e) { return -report(e, nullptr, 0); }
}
int om_select_draft_experts(int policy, const uint64_t* counts, int layers, int E, const int* cur, int n, uint64_t seed,
                            int* out) {
    try {
        HotnessCounter hc(layers, E);
        for (int l = 0; l < layers; ++l)
            for (int e = 0; e < E; ++e) hc.counts[l][e] = counts ? counts[(size_t)l * E + e] : 0;
        DraftState ds;
        ds.n_draft = n;
        if (cur) {
            ds.sets.resize(layers);
            for (int l = 0; l < layers; ++l) ds.sets[l].assign(cur + (size_t)l * n, cur + (size_t)(l + 1) * n);
        }
        Rng rng(seed);
        auto sets = select_draft_experts(static_cast<DraftPolicy>(policy), hc, ds, E, rng);
        for (int l = 0; l < layers; ++l) std::memcpy(out + (size_t)l * n, sets[l].data(), sizeof(int) * (size_t)n);
        return 0;
    } catch (const std::exception& e) { return -report(e, nullptr, 0); }
}
double om_skewness(const uint64_t* counts, int layers, int E, uint64_t routed, double frac) {
    try {
        HotnessCounter hc(layers, E);
        for (int l = 0; l < layers; ++l)
            for (int e = 0; e < E; ++e) hc.counts[l][e] = counts[(size_t)l * E + e];
        hc.routed_tokens = routed;
        return skewness(hc, frac);
    } catch (const std::exception&) { return -1.0; }
}

}  // extern "C"
