// loop.cpp -- the self-assisted speculative-decoding loop (specdec.cpp:190-397) and the on-demand
// comparator (baselines.cpp:29-99) on top of the device engine.
//
// Device side, per phase and without any host round trip in between: gamma restricted draft passes
// (T = active sequences), one unrestricted verify pass (T = active * (gamma+1)), the accept kernel.
// Host side, once per phase: read back accepted counts, corrections and the raw routing picks,
// then run the reference's bookkeeping -- coalesced ensure_resident, acceptance/truncation, hotness,
// hot_temporal selection + pin, flush -- exactly as the reference orders it, so tokens, ledger,
// outcomes and modeled metrics equal the oracle's.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <cmath>
#include <random>

#include "engine.h"

namespace smoe {

namespace {

// ------------------------------------------------------------------ memsim replica (memsim.cpp)
struct Ledger {
    std::vector<LedgerEntry> e;
    uint64_t tot[3] = {0, 0, 0}, total = 0;
    void add(int phase, int step, int key, int E, uint64_t bytes) {
        e.push_back(LedgerEntry{phase, step, key / E, key % E, bytes});
        tot[phase] += bytes;
        total += bytes;
    }
    void reset() {
        e.clear();
        tot[0] = tot[1] = tot[2] = 0;
        total = 0;
    }
};

void tier_check(const RunCfg& c, int n_draft, int M) {  // memsim.cpp:21-31
    if (c.host_bandwidth <= 0.0) throw Error(kConfig, "tier: host_bandwidth > 0 violated");
    if (c.ssd_bandwidth < 0.0) throw Error(kConfig, "tier: ssd_bandwidth >= 0 violated");
    if (c.bytes_per_expert == 0) throw Error(kConfig, "tier: bytes_per_expert > 0 violated");
    if (c.compute_rate <= 0.0) throw Error(kConfig, "tier: compute_rate > 0 violated");
    if (c.compute_cost_per_expert < 0.0) throw Error(kConfig, "tier: expert compute cost >= 0 violated");
    if (c.device_capacity_bytes < (uint64_t)n_draft * (uint64_t)M * c.bytes_per_expert)
        throw Error(kConfig, "tier: device capacity below N * moe_layers * bytes_per_expert");
}

double step_cost(uint64_t toks, uint64_t experts, uint64_t bytes, const RunCfg& c, bool overlap) {  // memsim.cpp:163-172
    const double comp = (double)toks / c.compute_rate + (double)experts * c.compute_cost_per_expert;
    const double mig = (double)bytes / (c.ssd_bandwidth > 0.0 ? c.ssd_bandwidth : c.host_bandwidth);
    return overlap ? std::max(comp, mig) : comp + mig;
}

// Residency: keys are (moe_layer * E + expert); iteration in key order == std::set<ExpertKey> order.
class Residency {
public:
    Residency(int M, int E, const RunCfg& c) : M_(M), E_(E), cap_(c.device_capacity_bytes), bpe_(c.bytes_per_expert) {
        tier_check(c, 0, M);
        arrival_.assign((size_t)M * E, -1);
        pinned_.assign((size_t)M * E, 0);
    }
    bool resident(int k) const { return arrival_[k] >= 0; }
    bool pinned(int k) const { return pinned_[k] != 0; }
    // memsim.cpp:102-113
    uint64_t ensure(const std::vector<uint8_t>& keys, int phase, int step, Ledger& lg) {
        uint64_t b = 0;
        for (int k = 0; k < M_ * E_; ++k) {
            if (!keys[k] || resident(k)) continue;
            admit(k, keys);
            lg.add(phase, step, k, E_, bpe_);
            b += bpe_;
        }
        return b;
    }
    // memsim.cpp:115-150
    uint64_t pin(const std::vector<std::vector<int>>& sets, Ledger& lg, int phase, int step) {
        if ((int)sets.size() != M_) throw Error(kInvariant, "pin_draft_experts: set count != MoE layer count");
        std::vector<uint8_t> target((size_t)M_ * E_, 0);
        for (int l = 0; l < M_; ++l)
            for (int e : sets[l]) {
                if (e < 0 || e >= E_) throw Error(kInvariant, "residency: expert key out of range");
                uint8_t& t = target[(size_t)l * E_ + e];
                if (t) throw Error(kInvariant, "pin_draft_experts: duplicate expert in draft set");
                t = 1;
            }
        for (int k = 0; k < M_ * E_; ++k)
            if (pinned_[k] && !target[k]) pinned_[k] = 0;
        uint64_t b = 0;
        for (int k = 0; k < M_ * E_; ++k) {
            if (!target[k]) continue;
            if (!resident(k)) {
                admit(k, target);
                lg.add(phase, step, k, E_, bpe_);
                b += bpe_;
            }
            pinned_[k] = 1;
        }
        return b;
    }
    void flush() {  // memsim.cpp:152-161
        for (int k = 0; k < M_ * E_; ++k)
            if (resident(k) && !pinned_[k]) { arrival_[k] = -1; used_ -= bpe_; }
    }

private:
    void admit(int key, const std::vector<uint8_t>& keep) {  // memsim.cpp:81-100
        while (used_ + bpe_ > cap_) {
            int victim = -1;
            for (int k = 0; k < M_ * E_; ++k) {
                if (!resident(k) || pinned_[k] || keep[k]) continue;
                if (victim < 0 || arrival_[k] < arrival_[victim]) victim = k;
            }
            if (victim < 0) throw Error(kInvariant, "residency: device capacity exhausted with no evictable expert");
            arrival_[victim] = -1;
            used_ -= bpe_;
        }
        arrival_[key] = (int64_t)seq_++;
        used_ += bpe_;
    }
    int M_, E_;
    uint64_t cap_, bpe_, used_ = 0, seq_ = 0;
    std::vector<int64_t> arrival_;
    std::vector<uint8_t> pinned_;
};

// ------------------------------------------------------------------ drafting replica (drafting.cpp:153-227)
double unif(std::mt19937_64& r) { return (double)(r() >> 11) * 0x1.0p-53; }

// hot_* selection for one layer (drafting.cpp:191-226): top-N by (count desc, index asc) among
// activated experts, filled from the current set in its order, sorted.
std::vector<int> select_layer_hot(const uint64_t* c, int E, const std::vector<int>* current, int n) {
    std::vector<int> idx(E);
    for (int i = 0; i < E; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return c[a] > c[b]; });
    std::vector<int> picked;
    for (int i = 0; i < std::min(n, E); ++i)
        if (c[idx[i]] > 0) picked.push_back(idx[i]);
    if ((int)picked.size() < n && current)
        for (int e : *current) {
            if ((int)picked.size() == n) break;
            if (std::find(picked.begin(), picked.end(), e) == picked.end()) picked.push_back(e);
        }
    if ((int)picked.size() != n) throw Error(kInvariant, "select_draft_experts: cannot assemble N draft experts");
    std::sort(picked.begin(), picked.end());
    return picked;
}

std::vector<std::vector<int>> select_sets(int policy, const std::vector<uint64_t>& counts, int M, int E,
                                          const std::vector<std::vector<int>>& current, int n, std::mt19937_64& rng) {
    if (n > E) throw Error(kConfig, "select_draft_experts: n_draft > experts_per_block");
    std::vector<std::vector<int>> out(M);
    for (int l = 0; l < M; ++l) {
        if (policy == SMOE_POLICY_RANDOM) {
            std::vector<int> pool(E);
            for (int i = 0; i < E; ++i) pool[i] = i;
            for (int i = 0; i < n; ++i) {
                size_t j = (size_t)i + (size_t)(unif(rng) * (double)((size_t)E - (size_t)i));
                std::swap(pool[i], pool[j]);
            }
            pool.resize(n);
            std::sort(pool.begin(), pool.end());
            out[l] = pool;
            continue;
        }
        out[l] = select_layer_hot(counts.data() + (size_t)l * E, E, l < (int)current.size() ? &current[l] : nullptr, n);
    }
    return out;
}

void validate_decode(const RunCfg& c, int B, int plen) {  // specdec.cpp:15-23
    if (c.gamma < 1) throw Error(kConfig, "spec: gamma >= 1 violated");
    if (B < 1) throw Error(kConfig, "spec: batch >= 1 violated");
    if (c.max_new_tokens < 1) throw Error(kConfig, "spec: max_new_tokens >= 1 violated");
    if (plen < 1) throw Error(kConfig, "spec: prompt_len >= 1 violated");
    if (c.warmup_steps < 1) throw Error(kConfig, "spec: warmup_steps >= 1 violated");
}

int prompt_len_of(const std::vector<std::vector<int>>& prompts) {
    size_t n = prompts.empty() ? 0 : prompts[0].size();
    for (auto& p : prompts)
        if (p.size() != n) throw Error(kConfig, "prompts must share one length");
    return (int)n;
}

// Copy the raw (or final) picks of `T` rows of pass slot `slot` to host: out[m][T*K].
void read_log(Engine& e, const int* log, int slot, int T, std::vector<int>& out) {
    out.resize((size_t)e.M * T * e.K);
    SMOE_CUDA(cudaMemcpy2DAsync(out.data(), sizeof(int) * T * e.K, log + (size_t)slot * e.M * e.Tmax * e.K,
                                sizeof(int) * e.Tmax * e.K, sizeof(int) * T * e.K, e.M, cudaMemcpyDeviceToHost,
                                e.stream));
}

struct Timer {
    cudaEvent_t a = nullptr, b = nullptr;
    std::chrono::steady_clock::time_point w0;
    void start(cudaStream_t s) {
        if (!a) { SMOE_CUDA(cudaEventCreate(&a)); SMOE_CUDA(cudaEventCreate(&b)); }
        w0 = std::chrono::steady_clock::now();
        SMOE_CUDA(cudaEventRecord(a, s));
    }
    void stop(cudaStream_t s, double* gpu_s, double* wall_s) {
        SMOE_CUDA(cudaEventRecord(b, s));
        SMOE_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        SMOE_CUDA(cudaEventElapsedTime(&ms, a, b));
        *gpu_s = ms * 1e-3;
        *wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    }
    ~Timer() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
};

}  // namespace

// uniform01 (common.hpp:40-42): one 64-bit output per draw
static double uniform01(std::mt19937_64& r) { return (double)(r() >> 11) * 0x1.0p-53; }

struct SpecState {
    RunCfg c;
    int B = 0, M = 0, E = 0, K = 0, g = 0, nd = 0;
    std::mt19937_64 prng;
    std::mt19937_64 srng;  // sample_rng (specdec.cpp:209): drafts and verify draws in sampling mode
    std::unique_ptr<Residency> res;
    Ledger led;
    std::vector<std::vector<int>> sets;
    bool sets_dirty = true;
    std::vector<uint64_t> pc;  // phase hotness counter [M][E]
    RunOut out;
    std::vector<int> gen;
    uint64_t tau_sum = 0, tau_cnt = 0;
    double spec_s = 0, ver_s = 0, step_s = 0;
    std::vector<uint64_t> lam;  // 4 per phase
    int phase = 0;
    Timer timer;
    // scratch
    std::vector<int> h_acc, h_corr, h_drafts, vraw, dfin, rows;
};

void SpecStateDeleter::operator()(SpecState* s) const { delete s; }

// hot_global warmup (specdec.cpp:223-245): greedy on-demand steps over the prompts.
static void hot_global_warmup(Engine& e, SpecState& S, const std::vector<std::vector<int>>& prompts) {
    const int B = S.B, M = S.M, E = S.E, K = S.K;
    std::vector<uint64_t> wc((size_t)M * E, 0);
    Ledger wl;
    Residency wr(M, E, S.c);
    if (e.offload) e.store_reset();  // the profiling pass starts from an empty device (no pins)
    e.reset_sequences(prompts);
    std::vector<int> rs(B), one(B, 1), raw, am(B);
    for (int b = 0; b < B; ++b) rs[b] = b;
    e.upload_ints(e.row_seq, rs.data(), B);
    e.upload_ints(e.seqs, rs.data(), B);
    e.upload_ints(e.commit_take, one.data(), B);
    for (int step = 0; step < S.c.warmup_steps; ++step) {
        e.pass(B, e.row_seq, nullptr, 0, false, 0, 0);
        read_log(e, e.raw_log, 0, B, raw);
        SMOE_CUDA(cudaMemcpyAsync(am.data(), e.amax, sizeof(int) * B, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
        e.check_flags();
        std::vector<uint8_t> need((size_t)M * E, 0);
        for (int m = 0; m < M; ++m)
            for (int b = 0; b < B; ++b)
                for (int k = 0; k < K; ++k) {
                    int key = m * E + raw[((size_t)m * B + b) * K + k];
                    need[key] = 1;
                    wc[key]++;
                }
        launch_commit(e.seq_sum, e.seq_len, e.emb64, e.seqs, e.amax, 1, e.commit_take, B, e.d, e.stream, e.last_tok);
        e.kv_advance(rs, one);
        wr.ensure(need, 2, step, wl);
        wr.flush();
    }
    S.out.warmup_bytes = wl.total;
    S.sets = select_sets(SMOE_POLICY_HOT_GLOBAL, wc, M, E, S.sets, S.nd, S.prng);
}

void spec_begin(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts) {
    std::unique_ptr<SpecState, SpecStateDeleter> S(new SpecState);
    S->c = c;
    const int plen = prompt_len_of(prompts);
    validate_decode(c, (int)prompts.size(), plen);
    S->B = (int)prompts.size();
    S->M = e.M; S->E = e.E; S->K = e.K; S->g = c.gamma; S->nd = c.n_draft;
    if (S->nd < e.K) throw Error(kConfig, "spec: n_draft >= top_k violated");
    if (S->nd > e.E) throw Error(kConfig, "spec: n_draft <= experts_per_block violated");
    tier_check(c, S->nd, e.M);
    if (c.use_affinity && !e.have_affinity) throw Error(kInvariant, "run_specmoe: affinity table required but missing");
    if (S->B > e.Bmax) throw Error(kConfig, "engine: batch exceeds max_batch");
    if (S->g > e.Gmax) throw Error(kConfig, "engine: gamma exceeds max_gamma");
    S->prng.seed(substream(c.run_seed, 0x706f6c69ull));
    S->srng.seed(substream(c.run_seed, 0x73616d70ull));
    if (c.mode == 1) {
        if (!(c.temperature > 0.0)) throw Error(kConfig, "spec: temperature > 0 violated in sampling mode");
        e.sampling_alloc();
    }
    S->res = std::make_unique<Residency>(e.M, e.E, c);
    S->pc.assign((size_t)e.M * e.E, 0);
    S->out.B = S->B; S->out.max_new = c.max_new_tokens; S->out.gamma = c.gamma;
    S->out.tokens.assign(S->B, {});
    S->out.hotness.assign((size_t)e.M * e.E, 0);
    S->sets = select_sets(SMOE_POLICY_RANDOM, S->pc, e.M, e.E, {}, S->nd, S->prng);
    if (c.policy == SMOE_POLICY_HOT_GLOBAL) hot_global_warmup(e, *S, prompts);
    S->res->pin(S->sets, S->led, 1, -1);
    S->out.setup_bytes = S->led.total;
    S->led.reset();
    if (e.offload) {  // initial pin = model setup, excluded like the reference's setup_bytes
        e.store_reset();
        e.store_pin_sets(S->sets);
        e.collect_h2d();
    }
    e.reset_sequences(prompts);
    S->gen.assign(S->B, 0);
    e.collect_h2d();  // copies of earlier runs (a caching warm-up) are not this run's
    e.h2d_bytes = 0;
    e.h2d_ms = 0;
    S->timer.start(e.stream);
    e.st = std::move(S);
}

// env SMOE_HOST_PROF=1: per phase, host time before the first launch / launching / waiting for the
// device / bookkeeping after the readback (stderr)
static const bool g_host_prof = [] {
    const char* v = std::getenv("SMOE_HOST_PROF");
    return v && v[0] == '1';
}();
static double host_now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int spec_step(Engine& e, int* accepted_tokens) {
    SpecState& S = *e.st;
    const int B = S.B, M = S.M, E = S.E, K = S.K, g = S.g;
    if (accepted_tokens) *accepted_tokens = 0;
    const double hp0 = g_host_prof ? host_now() : 0.0;
    double hp1 = 0.0, hp2 = 0.0, hp3 = 0.0;
    NvtxRange nv_phase("smoe speculative phase");
    std::vector<int> act;
    for (int b = 0; b < B; ++b)
        if (S.gen[b] < S.c.max_new_tokens) act.push_back(b);
    if (act.empty()) return 0;
    const int na = (int)act.size();
    for (int m = 0; m < M; ++m)
        for (int ex : S.sets[m])
            if (!S.res->pinned(m * E + ex) || !S.res->resident(m * E + ex))
                throw Error(kInvariant, "run_specmoe: draft expert not pinned on device");
    if (S.sets_dirty) {
        e.set_draft_sets(S.sets, S.nd, true);
        S.sets_dirty = false;
    }
    // rows: [0, na*(g+1)) verify (seq, i); [Tmax, Tmax+na) draft (seq)
    const int TV = na * (g + 1);
    S.rows.assign((size_t)2 * TV + na, 0);
    for (int s = 0; s < na; ++s)
        for (int i = 0; i <= g; ++i) {
            S.rows[(size_t)s * (g + 1) + i] = act[s];
            S.rows[(size_t)TV + s * (g + 1) + i] = i;
        }
    for (int s = 0; s < na; ++s) S.rows[(size_t)2 * TV + s] = act[s];
    // the phase's control uploads are queued without host syncs (engine.h upload_async)
    e.upload_async(e.row_seq, S.rows.data(), sizeof(int) * TV);
    e.upload_async(e.row_extra, S.rows.data() + TV, sizeof(int) * TV);
    int* drows = e.row_seq + e.Tmax;
    e.upload_async(drows, S.rows.data() + 2 * TV, sizeof(int) * na);
    e.upload_async(e.seqs, act.data(), sizeof(int) * na);

    // (a) speculation: gamma restricted passes, drafts stay on device.  Sampling mode: the draft token
    // of step t, sequence s is drawn with the (t*na + s)-th uniform of the phase (speculate's loop order,
    // specdec.cpp:38-50) from softmax(logits/T), whose rows are kept as the draw probabilities q.
    const bool samp = S.c.mode == 1;
    if (samp) {
        std::vector<double> u((size_t)g * na);
        for (double& x : u) x = uniform01(S.srng);
        e.upload_doubles(e.samp_u, u.data(), u.size());
    }
    if (g_host_prof) hp1 = host_now();
    // The phase's device work (gamma draft passes, the verify pass, the accept) has no host step inside:
    // on the HBM-resident greedy single-GPU path it is captured once per (rows, gamma, N) as a CUDA graph
    // and replayed (SMOE_GRAPH=0: direct launches).  The host-side counters the passes bump are re-applied
    // on each replay.  Bit-identical; it removes the per-launch CPU/front-end cost that small passes
    // expose (C4 B=32 14.07 -> 13.75 ms/step, C2 B=1 23.4 -> 23.2; C2 B=64 unchanged).
    static const bool use_graph = [] {
        const char* v = std::getenv("SMOE_GRAPH");
        return !(v && v[0] == '0');
    }();
    const bool graphable = use_graph && !samp && !e.offload && e.ep_world == 1 && !e.profiling && !e.attn();
    auto phase_device = [&]() {
        for (int t = 0; t < g; ++t) {
            e.pass(na, drows, nullptr, t, true, S.c.use_affinity, t);
            if (samp)
                launch_sample_rows(e.logits, na, e.V, S.c.temperature, e.samp_u + (size_t)t * na, e.amax,
                                   e.samp_q + (size_t)t * e.Bmax * e.V, e.V, e.stream);
            launch_scatter_tokens(e.amax, drows, nullptr, t, na, e.drafts, e.stride, e.stream);
        }
        // (b) verification: one pass over all gamma+1 positions of every active sequence.  Offloaded
        // experts are migrated layer by layer inside the pass; hot_temporal re-pins each layer as soon as
        // its routing over all verify rows is known (same rule and inputs as the phase-end selection).
        if (e.offload && S.c.policy == SMOE_POLICY_HOT_TEMPORAL) {
            e.repin_hook = [&S, E](int mo, const uint64_t* cnt, std::vector<int>& next) {
                next = select_layer_hot(cnt, E, &S.sets[mo], S.nd);
                return true;
            };
        }
        try {
            e.pass(TV, e.row_seq, e.row_extra, 0, false, 0, g);
        } catch (...) {
            e.repin_hook = nullptr;
            throw;
        }
        e.repin_hook = nullptr;
    };
    const uint64_t gkey = ((uint64_t)na << 32) | ((uint64_t)g << 20) | ((uint64_t)e.cur_n_draft << 4) |
                          (uint64_t)(S.c.use_affinity != 0);
    // capture on the second consecutive phase with the same key: a capture + instantiate costs tens of ms,
    // which only the steady state (the active count unchanged for many phases) repays -- not the tail of a
    // run, where sequences finish and the row count changes from phase to phase
    const bool repeat = gkey == e.last_phase_key;
    e.last_phase_key = gkey;
    // the graph is captured on a side stream while the GPU runs this phase's direct launches (capture +
    // instantiate of ~660 launches costs ~60 ms of host time, which the phase's device time hides)
    auto gi = graphable ? e.phase_graphs.find(gkey) : e.phase_graphs.end();
    const bool have_graph = graphable && gi != e.phase_graphs.end();
    const bool capture_after = graphable && !have_graph && repeat;
    if (have_graph) {
        SMOE_CUDA(cudaGraphLaunch(gi->second.exec, e.stream));
        e.launches += gi->second.launches;
        e.alg_dense_bytes += gi->second.dense_bytes;
    } else {
        phase_device();
    }
    auto capture_phase = [&]() {
        if (!e.capture_stream) SMOE_CUDA(cudaStreamCreateWithFlags(&e.capture_stream, cudaStreamNonBlocking));
        const uint64_t l0 = e.launches;
        const double b0 = e.alg_dense_bytes;
        cudaStream_t live = e.stream;
        e.stream = e.capture_stream;
        cudaGraph_t gr = nullptr;
        SMOE_CUDA(cudaStreamBeginCapture(e.stream, cudaStreamCaptureModeThreadLocal));
        try {
            phase_device();
        } catch (...) {
            cudaStreamEndCapture(e.stream, &gr);
            if (gr) cudaGraphDestroy(gr);
            e.stream = live;
            e.launches = l0;
            e.alg_dense_bytes = b0;
            throw;
        }
        e.stream = live;
        SMOE_CUDA(cudaStreamEndCapture(e.capture_stream, &gr));
        cudaGraphExec_t ex = nullptr;
        SMOE_CUDA(cudaGraphInstantiate(&ex, gr, 0));
        SMOE_CUDA(cudaGraphDestroy(gr));
        e.phase_graphs.emplace(gkey, Engine::PhaseGraph{ex, e.launches - l0, e.alg_dense_bytes - b0});
        e.launches = l0;
        e.alg_dense_bytes = b0;
    };
    // (c) accept: greedy (specdec.cpp:76-78) or Leviathan acceptance with the residual resample
    // (specdec.cpp:104-157) over a pool of na*(g+1) uniforms; the stream then advances by what was used
    std::mt19937_64 srng_before;
    int used = 0;
    if (samp) {
        srng_before = S.srng;
        std::vector<double> pool((size_t)na * (g + 1));
        for (double& x : pool) x = uniform01(S.srng);
        double* dpool = e.samp_u + (size_t)e.Gmax * e.Bmax;
        e.upload_doubles(dpool, pool.data(), pool.size());
        launch_verify_sampling(e.logits, e.V, S.c.temperature, e.samp_stats, e.samp_q, (long long)e.Bmax * e.V,
                               e.drafts, e.stride, e.seqs, na, g, dpool, e.acc, e.samp_i, e.samp_i + e.Bmax,
                               e.samp_i + 2 * e.Bmax, e.corr, e.flags, e.samp_ratio, e.stream);
        SMOE_CUDA(cudaMemcpyAsync(&used, e.samp_i + 2 * e.Bmax, sizeof(int), cudaMemcpyDeviceToHost, e.stream));
        e.launches += 3 + g;
    } else {
        launch_scatter_tokens(e.amax, e.row_seq, e.row_extra, 0, TV, e.vam, e.stride, e.stream);
        launch_accept(e.drafts, e.vam, e.seqs, na, g, e.stride, e.acc, e.corr, e.stream);
    }
    S.h_acc.resize(na); S.h_corr.resize(na); S.h_drafts.resize((size_t)e.Bmax * e.stride);
    // the phase's readbacks through the pinned arena: queued, one sync, then copied out
    e.download_async(S.h_acc.data(), e.acc, sizeof(int) * na);
    e.download_async(S.h_corr.data(), e.corr, sizeof(int) * na);
    e.download_async(S.h_drafts.data(), e.drafts, sizeof(int) * e.Bmax * e.stride);
    auto read_log_async = [&](const int* log, int slot, int T, std::vector<int>& out) {
        out.resize((size_t)e.M * T * e.K);
        e.download_async(out.data(), log + (size_t)slot * e.M * e.Tmax * e.K, sizeof(int) * T * e.K, (size_t)e.M,
                         sizeof(int) * e.Tmax * e.K);
    };
    read_log_async(e.raw_log, g, TV, S.vraw);
    std::vector<std::vector<int>> dfin(g);
    for (int t = 0; t < g; ++t) read_log_async(e.fin_log, t, na, dfin[t]);
    if (capture_after) {
        const double c0 = g_host_prof ? host_now() : 0.0;
        capture_phase();
        if (g_host_prof) fprintf(stderr, "smoe host: phase graph captured (rows %d): %.3f ms\n", na, (host_now() - c0) * 1e3);
    }
    if (g_host_prof) hp2 = host_now();
    {
        NvtxRange nv("smoe device wait");
        e.sync();
    }
    e.download_finish();
    e.upload_reset();  // the stream is idle: every queued control upload has been read
    if (g_host_prof) hp3 = host_now();
    NvtxRange nv_book("smoe bookkeeping (reference order)");
    e.check_flags();
    if (samp) {
        S.srng = srng_before;
        S.srng.discard((unsigned long long)used);
    }
    e.launches += (uint64_t)g + 2;  // scatters + accept (commit counted below)
    e.ctl_d2h += sizeof(int) * ((size_t)2 * na + (size_t)e.Bmax * e.stride + (size_t)M * K * (TV + (size_t)g * na));
    {  // algorithmic expert bytes: every distinct (layer, expert) a pass touches streams its weights once
        // (this rank's experts only under expert parallelism)
        const double bpe = (double)e.real_bytes_per_expert();
        const uint64_t mine = (e.e_hi - e.e_lo >= 64 ? ~0ull : ((1ull << (e.e_hi - e.e_lo)) - 1)) << e.e_lo;
        // and every routed (row, pick) on this rank's experts costs 2 * (U*d + d*f) flops
        const double fpp = 2.0 * ((double)e.U * e.d + (double)e.d * e.f);
        auto& ctr = e.named;
        for (int t = 0; t < g; ++t)
            for (int m = 0; m < M; ++m) {
                uint64_t seen = 0;
                long long picks = 0;
                for (int q = 0; q < na * K; ++q) {
                    const int x = dfin[t][(size_t)m * na * K + q];
                    seen |= 1ull << x;
                    picks += x >= e.e_lo && x < e.e_hi;
                }
                e.alg_expert_bytes += bpe * __builtin_popcountll(seen & mine);
                ctr["alg_expert_bytes:draft"] += bpe * __builtin_popcountll(seen & mine);
                ctr["expert_flops:draft"] += fpp * (double)picks;
            }
        for (int m = 0; m < M; ++m) {
            uint64_t seen = 0;
            long long picks = 0;
            for (int q = 0; q < TV * K; ++q) {
                const int x = S.vraw[(size_t)m * TV * K + q];
                seen |= 1ull << x;
                picks += x >= e.e_lo && x < e.e_hi;
            }
            e.alg_expert_bytes += bpe * __builtin_popcountll(seen & mine);
            ctr["alg_expert_bytes:verify"] += bpe * __builtin_popcountll(seen & mine);
            ctr["expert_flops:verify"] += fpp * (double)picks;
        }
    }

    // modeled speculation time (specdec.cpp:282-288)
    for (int t = 0; t < g; ++t) {
        std::vector<uint8_t> ex((size_t)M * E, 0);
        uint64_t distinct = 0;
        for (int m = 0; m < M; ++m)
            for (int q = 0; q < na * K; ++q) {
                int key = m * E + dfin[t][(size_t)m * na * K + q];
                if (!ex[key]) { ex[key] = 1; ++distinct; }
            }
        S.spec_s += step_cost((uint64_t)na, distinct, 0, S.c, false);
    }
    // coalesced union over the batch and all positions (specdec.cpp:303-317)
    auto vraw_at = [&](int s, int i, int m, int k) { return S.vraw[((size_t)m * TV + (size_t)s * (g + 1) + i) * K + k]; };
    std::vector<uint8_t> need((size_t)M * E, 0), first((size_t)M * E, 0);
    uint64_t n_need = 0, n_first = 0;
    for (int s = 0; s < na; ++s)
        for (int i = 0; i <= g; ++i)
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < K; ++k) {
                    int key = m * E + vraw_at(s, i, m, k);
                    if (!need[key]) { need[key] = 1; ++n_need; }
                    if (i == 0 && !first[key]) { first[key] = 1; ++n_first; }
                }
    uint64_t spec_before = S.led.tot[0];
    const uint64_t vb = S.res->ensure(need, 1, S.phase, S.led);
    if (S.led.tot[0] != spec_before) throw Error(kInvariant, "run_specmoe: speculation phase migrated bytes");
    const uint64_t vt = (uint64_t)na * (uint64_t)(g + 1);
    S.ver_s += step_cost(vt, n_need, vb, S.c, false);
    S.lam.insert(S.lam.end(), {vt, n_need, (uint64_t)na, n_first});
    S.step_s += step_cost((uint64_t)na, n_first, n_first * S.c.bytes_per_expert, S.c, false);

    // acceptance bookkeeping and per-sequence advance (specdec.cpp:330-362)
    std::vector<int> ctoks((size_t)na * e.stride, 0), ctake(na, 0);
    int total_take = 0;
    for (int s = 0; s < na; ++s) {
        const int b = act[s];
        const int a = S.h_acc[s];
        Outcome o{b, S.phase, a, S.h_corr[s], a + 1, {}};
        for (int i = 0; i < g; ++i) o.drafts.push_back(S.h_drafts[(size_t)b * e.stride + i]);
        S.tau_sum += (uint64_t)(a + 1);
        ++S.tau_cnt;
        const int take = std::min(a + 1, S.c.max_new_tokens - S.gen[b]);
        for (int t = 0; t < take; ++t) {
            const int tok = t < a ? o.drafts[t] : o.correction;
            ctoks[(size_t)s * e.stride + t] = tok;
            S.out.tokens[b].push_back(tok);
        }
        ctake[s] = take;
        total_take += take;
        S.gen[b] += take;
        S.out.outcomes.push_back(std::move(o));
        for (int i = 0; i <= g; ++i)
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < K; ++k) {
                    int key = m * E + vraw_at(s, i, m, k);
                    S.pc[key]++;
                    S.out.hotness[key]++;
                }
        if (S.c.collect_trace)
            for (int i = 0; i <= g; ++i)
                for (int m = 0; m < M; ++m) {
                    TraceRow tr{S.phase, b, m, {}};
                    for (int k = 0; k < K; ++k) tr.experts.push_back(vraw_at(s, i, m, k));
                    S.out.trace.push_back(std::move(tr));
                }
    }
    // rollback / advance of the device prefix state: only the taken tokens enter the running sums
    e.upload_async(e.commit_toks, ctoks.data(), sizeof(int) * ctoks.size());
    e.upload_async(e.commit_take, ctake.data(), sizeof(int) * na);
    launch_commit(e.seq_sum, e.seq_len, e.emb64, e.seqs, e.commit_toks, e.stride, e.commit_take, na, e.d, e.stream,
                  e.last_tok);
    e.kv_advance(act, ctake);
    e.launches += 1;

    if (S.c.policy == SMOE_POLICY_HOT_TEMPORAL) {
        auto next = select_sets(SMOE_POLICY_HOT_TEMPORAL, S.pc, M, E, S.sets, S.nd, S.prng);
        S.res->pin(next, S.led, 1, S.phase);
        if (e.offload)  // the store re-pinned layer by layer during verify: it must agree
            for (int m = 0; m < M; ++m)
                for (int ex = e.e_lo; ex < e.e_hi; ++ex)  // this rank's experts
                    if ((e.key_pinned[(size_t)m * E + ex] != 0) !=
                        (std::find(next[m].begin(), next[m].end(), ex) != next[m].end()))
                        throw Error(kInvariant, "expert store: per-layer re-pin diverged from the phase selection");
        if (next != S.sets) S.sets_dirty = true;
        S.sets = std::move(next);
    }
    std::fill(S.pc.begin(), S.pc.end(), 0);
    S.res->flush();
    ++S.phase;
    if (accepted_tokens) *accepted_tokens = total_take;
    if (g_host_prof)
        std::fprintf(stderr, "smoe host phase %d: prep %.3f ms, launch %.3f ms, device wait %.3f ms, bookkeeping %.3f ms\n",
                     S.phase, (hp1 - hp0) * 1e3, (hp2 - hp1) * 1e3, (hp3 - hp2) * 1e3, (host_now() - hp3) * 1e3);
    return na;
}

RunOut spec_end(Engine& e) {
    SpecState& S = *e.st;
    RunOut& R = S.out;
    S.timer.stop(e.stream, &R.gpu_s, &R.wall_s);
    R.phases = S.phase;
    R.tau_mean = S.tau_cnt ? (double)S.tau_sum / (double)S.tau_cnt : 1.0;
    R.tokens_total = 0;
    for (auto& t : R.tokens) R.tokens_total += t.size();
    R.speculation_s = S.spec_s;
    R.verification_s = S.ver_s;
    R.modeled_seconds = S.spec_s + S.ver_s;
    R.tokens_per_sec = R.modeled_seconds > 0.0 ? (double)R.tokens_total / R.modeled_seconds : 0.0;
    R.bytes_spec = S.led.tot[0];
    R.bytes_verify = S.led.tot[1];
    R.bytes_baseline = S.led.tot[2];
    R.bytes_total = S.led.total;
    if (S.lam.empty()) {
        R.lambda = 1.0;
    } else {  // specdec.cpp:159-172
        double vs = 0.0, ss = 0.0;
        for (size_t i = 0; i < S.lam.size(); i += 4) {
            vs += step_cost(S.lam[i], S.lam[i + 1], S.lam[i + 1] * S.c.bytes_per_expert, S.c, false);
            ss += step_cost(S.lam[i + 2], S.lam[i + 3], S.lam[i + 3] * S.c.bytes_per_expert, S.c, false);
        }
        if (ss <= 0.0) throw Error(kInvariant, "measure_lambda: zero single-step latency");
        R.lambda = vs / ss;
    }
    R.lambda_inputs = S.lam;
    R.c_measured = (S.phase > 0 && S.step_s > 0.0)
                       ? (S.spec_s / ((double)S.phase * S.g)) / (S.step_s / (double)S.phase)
                       : 0.0;
    R.ledger = S.led.e;
    e.collect_h2d();
    R.h2d_expert_bytes = e.h2d_bytes;
    R.h2d_s = e.h2d_ms * 1e-3;
    RunOut out = std::move(R);
    e.st.reset();
    return out;
}

RunOut run_specmoe(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts) {
    spec_begin(e, c, prompts);
    try {
        while (spec_step(e, nullptr) > 0) {
        }
    } catch (...) {
        e.st.reset();
        throw;
    }
    return spec_end(e);
}

// baselines.cpp:29-99 (greedy, no pinned set, no overlap)
RunOut run_ondemand(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts,
                    const std::vector<std::vector<int>>* pinned_sets) {
    const int plen = prompt_len_of(prompts);
    const int B = (int)prompts.size();
    if (c.gamma < 1) throw Error(kConfig, "spec: gamma >= 1 violated");
    if (c.max_new_tokens < 1) throw Error(kConfig, "spec: max_new_tokens >= 1 violated");
    if (c.warmup_steps < 1) throw Error(kConfig, "spec: warmup_steps >= 1 violated");
    if (plen < 1) throw Error(kConfig, "spec: prompt_len >= 1 violated");
    if (B < 1) throw Error(kConfig, "baseline run: no prompts");
    if (B > e.Bmax) throw Error(kConfig, "engine: batch exceeds max_batch");
    const int M = e.M, E = e.E, K = e.K;
    tier_check(c, 0, M);
    Residency res(M, E, c);
    Ledger led;
    RunOut R;
    R.B = B; R.max_new = c.max_new_tokens; R.gamma = 0;
    R.tokens.assign(B, {});
    R.hotness.assign((size_t)M * E, 0);
    if (e.offload) e.store_reset();
    if (pinned_sets) {  // MoE-Caching: cached experts pinned up front (baselines.cpp:60-65)
        res.pin(*pinned_sets, led, 2, -1);
        R.setup_bytes = led.total;
        led.reset();
        if (e.offload) e.store_pin_sets(*pinned_sets);
    }
    e.collect_h2d();  // copies of earlier runs (a caching warm-up) are not this run's
    e.h2d_bytes = 0;
    e.h2d_ms = 0;
    // overlap baseline on the physical store: prefetch the next layer's previous-step experts behind each
    // layer's fetch (the reference's oracle overlap, baselines.cpp:101-111, is a cost-model max())
    e.store_prefetch = e.offload && c.overlap != 0;
    e.reset_sequences(prompts);
    std::vector<int> rs(B), one(B, 1), raw, am(B);
    for (int b = 0; b < B; ++b) rs[b] = b;
    e.upload_ints(e.row_seq, rs.data(), B);
    e.upload_ints(e.seqs, rs.data(), B);
    e.upload_ints(e.commit_take, one.data(), B);
    // sampling mode: token of (step, b) drawn with the (step*B + b)-th uniform of sample_rng
    // (baselines.cpp:43, 59-64)
    const bool samp = c.mode == 1;
    std::mt19937_64 srng(substream(c.run_seed, 0x73616d70ull));
    if (samp) {
        if (!(c.temperature > 0.0)) throw Error(kConfig, "sample_next: temperature must be > 0");
        e.sampling_alloc();
    }
    Timer tm;
    tm.start(e.stream);
    double modeled = 0.0;
    for (int step = 0; step < c.max_new_tokens; ++step) {
        if (samp) {
            std::vector<double> u(B);
            for (double& x : u) x = uniform01(srng);
            e.upload_doubles(e.samp_u, u.data(), B);
        }
        e.pass(B, e.row_seq, nullptr, 0, false, 0, 0);
        if (samp) launch_sample_rows(e.logits, B, e.V, c.temperature, e.samp_u, e.amax, nullptr, 0, e.stream);
        launch_commit(e.seq_sum, e.seq_len, e.emb64, e.seqs, e.amax, 1, e.commit_take, B, e.d, e.stream, e.last_tok);
        e.kv_advance(rs, one);
        read_log(e, e.raw_log, 0, B, raw);
        SMOE_CUDA(cudaMemcpyAsync(am.data(), e.amax, sizeof(int) * B, cudaMemcpyDeviceToHost, e.stream));
        e.sync();
        e.check_flags();
        std::vector<uint8_t> need((size_t)M * E, 0);
        uint64_t n_need = 0;
        for (int b = 0; b < B; ++b) {
            for (int m = 0; m < M; ++m)
                for (int k = 0; k < K; ++k) {
                    int key = m * E + raw[((size_t)m * B + b) * K + k];
                    if (!need[key]) { need[key] = 1; ++n_need; }
                    R.hotness[key]++;
                }
            R.tokens[b].push_back(am[b]);
            if (c.collect_trace)
                for (int m = 0; m < M; ++m) {
                    TraceRow tr{step, b, m, {}};
                    for (int k = 0; k < K; ++k) tr.experts.push_back(raw[((size_t)m * B + b) * K + k]);
                    R.trace.push_back(std::move(tr));
                }
        }
        const uint64_t bytes = res.ensure(need, 2, step, led);
        modeled += step_cost((uint64_t)B, n_need, bytes, c, c.overlap != 0);
        res.flush();
        if (e.store_prefetch) e.prev_need = need;
    }
    tm.stop(e.stream, &R.gpu_s, &R.wall_s);
    e.store_prefetch = false;
    R.phases = c.max_new_tokens;
    R.tau_mean = 1.0;
    R.tokens_total = (uint64_t)B * c.max_new_tokens;
    R.modeled_seconds = modeled;
    R.verification_s = modeled;
    R.tokens_per_sec = modeled > 0.0 ? (double)R.tokens_total / modeled : 0.0;
    R.bytes_spec = led.tot[0];
    R.bytes_verify = led.tot[1];
    R.bytes_baseline = led.tot[2];
    R.bytes_total = led.total;
    R.lambda = 1.0;
    R.c_measured = 0.0;
    R.ledger = led.e;
    e.collect_h2d();
    R.h2d_expert_bytes = e.h2d_bytes;
    R.h2d_s = e.h2d_ms * 1e-3;
    R.prefetch_bytes = e.prefetch_bytes;
    R.prefetch_wasted_bytes = e.prefetch_wasted;
    return R;
}

std::vector<std::vector<int>> caching_sets(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts,
                                           double cache_fraction, uint64_t* warmup_bytes) {
    if (cache_fraction <= 0.0 || cache_fraction >= 1.0) throw Error(kConfig, "baseline: 0 < cache_fraction < 1 violated");
    if (c.warmup_steps < 1) throw Error(kConfig, "baseline: warmup_steps >= 1 violated");
    SpecState S;
    S.c = c;
    S.B = (int)prompts.size();
    S.M = e.M; S.E = e.E; S.K = e.K;
    S.nd = (int)std::ceil(cache_fraction * e.E);
    const uint64_t cache_bytes = (uint64_t)S.nd * e.M * c.bytes_per_expert;
    hot_global_warmup(e, S, prompts);  // fills S.sets from the warmup counts (empty current set)
    if (cache_bytes > c.device_capacity_bytes) throw Error(kConfig, "caching: cached experts exceed device capacity");
    if (warmup_bytes) *warmup_bytes = S.out.warmup_bytes;
    return S.sets;
}

}  // namespace smoe
