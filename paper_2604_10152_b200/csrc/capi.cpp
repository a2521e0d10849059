// capi.cpp -- extern "C" boundary (include/specmoe_b200.h).  Exceptions never cross it: every entry
// point converts smoe::Error / std::exception into a status code and a thread-local message.
#include <cstdlib>
#include <cstring>
#include <string>

#include "engine.h"
#include "specmoe/harness.hpp"

struct smoe_engine {
    std::unique_ptr<smoe::Engine> e;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return SMOE_OK;
    } catch (const smoe::Error& x) {
        g_err = x.what();
        return x.code;
    } catch (const std::exception& x) {
        g_err = x.what();
        return SMOE_INVARIANT;
    }
}

smoe::RunCfg cfg_of(const smoe_run_config* c) {
    smoe::RunCfg r;
    r.gamma = c->gamma;
    r.n_draft = c->n_draft;
    r.max_new_tokens = c->max_new_tokens;
    r.use_affinity = c->use_affinity;
    r.warmup_steps = c->warmup_steps;
    r.policy = c->policy;
    r.collect_trace = c->collect_trace;
    r.run_seed = c->run_seed;
    r.device_capacity_bytes = c->device_capacity_bytes;
    r.bytes_per_expert = c->bytes_per_expert;
    r.host_bandwidth = c->host_bandwidth;
    r.ssd_bandwidth = c->ssd_bandwidth;
    r.compute_rate = c->compute_rate;
    r.compute_cost_per_expert = c->compute_cost_per_expert;
    r.mode = c->mode;
    r.temperature = c->temperature;
    return r;
}

std::vector<std::vector<int>> prompts_of(const int* p, int B, int plen) {
    std::vector<std::vector<int>> v(B);
    for (int b = 0; b < B; ++b) v[b].assign(p + (size_t)b * plen, p + (size_t)(b + 1) * plen);
    return v;
}

template <typename T>
T* cdup(const T* src, size_t n) {
    T* p = static_cast<T*>(std::calloc(n + 1, sizeof(T)));
    if (n) std::memcpy(p, src, n * sizeof(T));
    return p;
}

smoe_run_result* flatten(const smoe::RunOut& r, int M, int E, int K) {
    auto* o = static_cast<smoe_run_result*>(std::calloc(1, sizeof(smoe_run_result)));
    o->B = r.B; o->max_new = r.max_new; o->moe_layers = M; o->experts = E; o->top_k = K; o->gamma = r.gamma;
    o->tokens = static_cast<int*>(std::calloc((size_t)r.B * r.max_new + 1, sizeof(int)));
    o->n_tokens = static_cast<int*>(std::calloc((size_t)r.B + 1, sizeof(int)));
    for (int b = 0; b < r.B; ++b) {
        o->n_tokens[b] = (int)r.tokens[b].size();
        for (size_t i = 0; i < r.tokens[b].size() && (int)i < r.max_new; ++i) o->tokens[(size_t)b * r.max_new + i] = r.tokens[b][i];
    }
    o->n_ledger = (int)r.ledger.size();
    o->ledger = static_cast<smoe_ledger_entry*>(std::calloc(r.ledger.size() + 1, sizeof(smoe_ledger_entry)));
    for (size_t i = 0; i < r.ledger.size(); ++i)
        o->ledger[i] = smoe_ledger_entry{r.ledger[i].phase, r.ledger[i].step, r.ledger[i].layer, r.ledger[i].expert,
                                         r.ledger[i].bytes};
    o->n_outcomes = (int)r.outcomes.size();
    o->outcomes = static_cast<smoe_outcome*>(std::calloc(r.outcomes.size() + 1, sizeof(smoe_outcome)));
    o->outcome_drafts = static_cast<int*>(std::calloc(r.outcomes.size() * (size_t)std::max(1, r.gamma) + 1, sizeof(int)));
    for (size_t i = 0; i < r.outcomes.size(); ++i) {
        const auto& x = r.outcomes[i];
        o->outcomes[i] = smoe_outcome{x.seq, x.phase, x.accepted, x.correction, x.generated};
        for (int j = 0; j < r.gamma && j < (int)x.drafts.size(); ++j) o->outcome_drafts[i * r.gamma + j] = x.drafts[j];
    }
    o->n_trace = (int)r.trace.size();
    o->trace = static_cast<int*>(std::calloc(r.trace.size() * (3 + K) + 1, sizeof(int)));
    for (size_t i = 0; i < r.trace.size(); ++i) {
        int* t = o->trace + i * (3 + K);
        t[0] = r.trace[i].step; t[1] = r.trace[i].seq; t[2] = r.trace[i].layer;
        for (int k = 0; k < K; ++k) t[3 + k] = r.trace[i].experts[k];
    }
    o->hotness = cdup(r.hotness.data(), r.hotness.size());
    o->tau_mean = r.tau_mean; o->tokens_total = r.tokens_total; o->phases = r.phases;
    o->speculation_s = r.speculation_s; o->verification_s = r.verification_s; o->modeled_seconds = r.modeled_seconds;
    o->tokens_per_sec = r.tokens_per_sec; o->bytes_spec = r.bytes_spec; o->bytes_verify = r.bytes_verify;
    o->bytes_baseline = r.bytes_baseline; o->bytes_total = r.bytes_total; o->setup_bytes = r.setup_bytes;
    o->warmup_bytes = r.warmup_bytes; o->lambda = r.lambda; o->c_measured = r.c_measured; o->wall_s = r.wall_s;
    o->gpu_s = r.gpu_s; o->h2d_expert_bytes = r.h2d_expert_bytes; o->h2d_s = r.h2d_s;
    o->prefetch_bytes = r.prefetch_bytes; o->prefetch_wasted_bytes = r.prefetch_wasted_bytes;
    return o;
}

}  // namespace

extern "C" {

const char* smoe_last_error(void) { return g_err.c_str(); }

int smoe_engine_create(const smoe_engine_config* cfg, smoe_engine** out) {
    return guarded([&] {
        auto* h = new smoe_engine;
        try {
            h->e = std::make_unique<smoe::Engine>(*cfg);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void smoe_engine_destroy(smoe_engine* e) { delete e; }

int smoe_engine_info(smoe_engine* h, uint64_t* device_bytes, uint64_t* bpe_real, int* moe_layers) {
    return guarded([&] {
        size_t fr = 0, tot = 0;
        SMOE_CUDA(cudaMemGetInfo(&fr, &tot));
        if (device_bytes) *device_bytes = tot - fr;
        if (bpe_real) *bpe_real = h->e->real_bytes_per_expert();
        if (moe_layers) *moe_layers = h->e->M;
    });
}

void* smoe_engine_stream(smoe_engine* h) { return h ? (void*)h->e->stream : nullptr; }

int smoe_init_weights_exact(smoe_engine* h) { return guarded([&] { h->e->init_exact(); }); }
int smoe_init_weights_device(smoe_engine* h, uint64_t seed) { return guarded([&] { h->e->init_device(seed); }); }
int smoe_upload_tensor(smoe_engine* h, const char* name, int layer, int expert, const double* src, long long n) {
    return guarded([&] { h->e->upload_tensor(name, layer, expert, src, n); });
}
int smoe_set_affinity(smoe_engine* h, const double* dist) {
    return guarded([&] {
        auto& e = *h->e;
        e.affinity.assign(dist, dist + (size_t)e.M * e.E * e.E);
        e.have_affinity = true;
        ++e.affinity_gen;
    });
}
int smoe_build_affinity_device(smoe_engine* h) { return guarded([&] { h->e->build_affinity_device(); }); }
int smoe_get_affinity(smoe_engine* h, double* out) {
    return guarded([&] {
        if (!h->e->have_affinity) throw smoe::Error(SMOE_INVARIANT, "affinity table not built");
        std::memcpy(out, h->e->affinity.data(), h->e->affinity.size() * sizeof(double));
    });
}

// A stepped run (smoe_spec_begin .. smoe_spec_end) owns the engine's per-sequence state and draft
// tables; any other entry point that resets them would silently corrupt the stepped run.
static void no_stepped_run(smoe_engine* h) {
    if (h->e->st) throw smoe::Error(SMOE_INVARIANT, "stepped run in progress; call smoe_spec_end first");
}

int smoe_forward(smoe_engine* h, const int* prefix, int n, const int* restricted, int n_draft, int use_affinity,
                 float* logits_out, int* raw_out, int* final_out) {
    return guarded([&] {
        no_stepped_run(h);
        if (restricted && (n_draft < 0 || n_draft > h->e->E))
            throw smoe::Error(SMOE_INVARIANT, "forward: restricted set larger than experts_per_block");
        std::vector<int> p(prefix, prefix + std::max(0, n));
        for (int t : p)
            if (t < 0 || t >= h->e->V) throw smoe::Error(SMOE_INVARIANT, "forward: token out of range");
        h->e->forward_one(p, restricted, n_draft, use_affinity, logits_out, raw_out, final_out);
    });
}

int smoe_run_specmoe(smoe_engine* h, const smoe_run_config* cfg, const int* prompts, int B, int plen,
                     smoe_run_result** out) {
    return guarded([&] {
        no_stepped_run(h);
        if (B < 1) throw smoe::Error(SMOE_CONFIG, "run_specmoe: no prompts");
        auto r = smoe::run_specmoe(*h->e, cfg_of(cfg), prompts_of(prompts, B, plen));
        *out = flatten(r, h->e->M, h->e->E, h->e->K);
    });
}

int smoe_run_ondemand(smoe_engine* h, const smoe_run_config* cfg, const int* prompts, int B, int plen,
                      smoe_run_result** out) {
    return guarded([&] {
        no_stepped_run(h);
        auto r = smoe::run_ondemand(*h->e, cfg_of(cfg), prompts_of(prompts, B, plen));
        *out = flatten(r, h->e->M, h->e->E, h->e->K);
    });
}

int smoe_run_overlap(smoe_engine* h, const smoe_run_config* cfg, const int* prompts, int B, int plen,
                     smoe_run_result** out) {
    return guarded([&] {
        no_stepped_run(h);
        smoe::RunCfg c = cfg_of(cfg);
        c.overlap = 1;
        auto r = smoe::run_ondemand(*h->e, c, prompts_of(prompts, B, plen));
        *out = flatten(r, h->e->M, h->e->E, h->e->K);
    });
}

int smoe_run_caching(smoe_engine* h, const smoe_run_config* cfg, double cache_fraction, const int* prompts, int B,
                     int plen, smoe_run_result** out) {
    return guarded([&] {
        no_stepped_run(h);
        if (!(cache_fraction > 0.0 && cache_fraction < 1.0))
            throw smoe::Error(SMOE_CONFIG, "baseline: 0 < cache_fraction < 1 violated");
        const auto P = prompts_of(prompts, B, plen);
        smoe::RunCfg c = cfg_of(cfg);
        c.policy = 1;  // hot_global profiling (baselines.cpp:119-145)
        uint64_t warm = 0;
        const auto cached = smoe::caching_sets(*h->e, c, P, cache_fraction, &warm);
        auto r = smoe::run_ondemand(*h->e, cfg_of(cfg), P, &cached);
        r.warmup_bytes = warm;
        *out = flatten(r, h->e->M, h->e->E, h->e->K);
    });
}

void smoe_free_result(smoe_run_result* r) {
    if (!r) return;
    std::free(r->tokens); std::free(r->n_tokens); std::free(r->ledger); std::free(r->outcomes);
    std::free(r->outcome_drafts); std::free(r->trace); std::free(r->hotness);
    std::free(r);
}

int smoe_spec_begin(smoe_engine* h, const smoe_run_config* cfg, const int* prompts, int B, int plen) {
    return guarded([&] {
        no_stepped_run(h);
        if (B < 1) throw smoe::Error(SMOE_CONFIG, "run_specmoe: no prompts");
        smoe::spec_begin(*h->e, cfg_of(cfg), prompts_of(prompts, B, plen));
    });
}
int smoe_spec_step(smoe_engine* h, int* tokens_accepted_out, int* active_out) {
    return guarded([&] {
        if (!h->e->st) throw smoe::Error(SMOE_INVARIANT, "spec_step without spec_begin");
        int n = smoe::spec_step(*h->e, tokens_accepted_out);
        if (active_out) *active_out = n;
    });
}
int smoe_spec_end(smoe_engine* h, smoe_run_result** out) {
    return guarded([&] {
        if (!h->e->st) throw smoe::Error(SMOE_INVARIANT, "spec_end without spec_begin");
        auto r = smoe::spec_end(*h->e);
        if (out) *out = flatten(r, h->e->M, h->e->E, h->e->K);
    });
}

int smoe_counters(smoe_engine* h, uint64_t* launches, double* alg_expert_bytes, double* alg_dense_bytes,
                  uint64_t* ctl_h2d, uint64_t* ctl_d2h, int reset) {
    return guarded([&] {
        auto& e = *h->e;
        if (launches) *launches = e.launches;
        if (alg_expert_bytes) *alg_expert_bytes = e.alg_expert_bytes;
        if (alg_dense_bytes) *alg_dense_bytes = e.alg_dense_bytes;
        if (ctl_h2d) *ctl_h2d = e.ctl_h2d;
        if (ctl_d2h) *ctl_d2h = e.ctl_d2h;
        if (reset) {
            e.launches = e.ctl_h2d = e.ctl_d2h = 0;
            e.alg_expert_bytes = e.alg_dense_bytes = 0;
            e.named.clear();
        }
    });
}

int smoe_bench_expert_gemm(smoe_engine* h, int T, int iters, double* up_ms, double* down_ms, double* bytes_up,
                           double* bytes_down) {
    return guarded([&] { h->e->bench_expert_gemm(T, iters, up_ms, down_ms, bytes_up, bytes_down); });
}

int smoe_ep_nccl_unique_id(void* out, int len) {
    int n = 0;
    int rc = guarded([&] { n = smoe::nccl_unique_id(out, len); });
    return rc ? -rc : n;
}
int smoe_ep_attach_nccl(smoe_engine* h, const void* id, int len) {
    return guarded([&] {
        auto& e = *h->e;
        if (e.ep_world < 2) throw smoe::Error(SMOE_CONFIG, "engine was not created with ep_world > 1");
        e.comm = smoe::make_nccl_comm(e.ep_rank, e.ep_world, id, len, e.device);
    });
}
int smoe_ep_attach_host(smoe_engine* h, smoe_host_allgather_fn fn, void* user) {
    return guarded([&] {
        auto& e = *h->e;
        if (e.ep_world < 2) throw smoe::Error(SMOE_CONFIG, "engine was not created with ep_world > 1");
        e.comm = smoe::make_host_comm(e.ep_rank, e.ep_world, fn, user);
    });
}
smoe_ep_loopback* smoe_ep_loopback_create(int world) {
    smoe::LoopbackGroup* g = nullptr;
    guarded([&] { g = smoe::loopback_create(world); });
    return reinterpret_cast<smoe_ep_loopback*>(g);
}
void smoe_ep_loopback_destroy(smoe_ep_loopback* g) { smoe::loopback_destroy(reinterpret_cast<smoe::LoopbackGroup*>(g)); }
int smoe_ep_attach_loopback(smoe_engine* h, smoe_ep_loopback* g) {
    return guarded([&] {
        auto& e = *h->e;
        if (e.ep_world < 2) throw smoe::Error(SMOE_CONFIG, "engine was not created with ep_world > 1");
        e.comm = smoe::make_loopback_comm(reinterpret_cast<smoe::LoopbackGroup*>(g), e.ep_rank);
    });
}

int smoe_profile_reset(smoe_engine* h) {
    return guarded([&] {
        h->e->prof_collect();
        h->e->prof.clear();
        h->e->profiling = true;
    });
}
int smoe_counter(smoe_engine* h, const char* name, double* value) {
    return guarded([&] {
        if (std::strcmp(name, "ssd_direct") == 0) {  // the SSD tier reads with O_DIRECT (1) or buffered (0)
            *value = h->e->ssd_direct();
            return;
        }
        auto it = h->e->named.find(name);
        *value = it == h->e->named.end() ? 0.0 : it->second;
    });
}
int smoe_profile_stop(smoe_engine* h) {
    return guarded([&] {
        h->e->prof_collect();
        h->e->profiling = false;
    });
}
int smoe_profile_read(smoe_engine* h, const char* cls, double* total_ms, long long* launches, double* bytes) {
    return guarded([&] {
        h->e->prof_collect();
        auto it = h->e->prof.find(cls);
        if (it == h->e->prof.end()) {
            *total_ms = 0; *launches = 0; *bytes = 0;
            return;
        }
        *total_ms = it->second.ms;
        *launches = it->second.n;
        *bytes = it->second.bytes;
    });
}

}  // extern "C"

int smoe_make_prompts(uint64_t seed, int batch, int prompt_len, int vocab, int* out) {
    try {
        const auto p = specmoe::make_prompts(seed, batch, prompt_len, vocab);
        for (int b = 0; b < batch; ++b) std::memcpy(out + (size_t)b * prompt_len, p[b].data(), sizeof(int) * prompt_len);
        return SMOE_OK;
    } catch (const specmoe::ConfigError& x) {
        g_err = x.what();
        return SMOE_CONFIG;
    } catch (const std::exception& x) {
        g_err = x.what();
        return SMOE_INVARIANT;
    }
}
