// api.cpp -- the reference's C++ API (include/specmoe/api.hpp) on top of the B200 engine.
//
// Host pieces (weights generation, affinity, policy, memsim, cost model) reproduce the reference's
// arithmetic order so their outputs are bit-identical; every forward computation (forward, speculate,
// verify_*, run_*) runs on the GPU engine.  One engine per ModelWeights object (fingerprinted), fp32
// storage by default so tokens/routing match the reference bit for bit (SPECMOE_B200_DTYPE=bf16 selects
// the tcgen05 path).
#include "../../include/specmoe/api.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <mutex>
#include <numeric>
#include <sstream>
#include <thread>
#include <atomic>

#include "engine.h"

namespace specmoe {

// ============================================================== common
double gaussian(Rng& rng) {  // Marsaglia polar, second variate dropped (reference common.hpp:46-55)
    while (true) {
        const double u = 2.0 * uniform01(rng) - 1.0;
        const double v = 2.0 * uniform01(rng) - 1.0;
        const double s = u * u + v * v;
        if (s > 0.0 && s < 1.0) return u * std::sqrt(-2.0 * std::log(s) / s);
    }
}
uint64_t fnv1a64(const void* data, size_t len, uint64_t h) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < len; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
    return h;
}
uint64_t hash_tokens(const std::vector<int>& tokens) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int t : tokens) {
        const uint32_t v = static_cast<uint32_t>(t);
        h = fnv1a64(&v, sizeof v, h);
    }
    return h;
}

namespace {

[[noreturn]] void rethrow(const smoe::Error& e) {
    if (e.code == smoe::kConfig) throw ConfigError(e.what());
    if (e.code == smoe::kInvariant) throw InvariantError(e.what());
    throw std::runtime_error(e.what());
}
template <typename F>
auto guard(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const smoe::Error& e) {
        rethrow(e);
    }
}

bool finite_all(std::span<const double> x) {
    return std::all_of(x.begin(), x.end(), [](double v) { return std::isfinite(v); });
}
bool has(std::span<const int> xs, int v) { return std::find(xs.begin(), xs.end(), v) != xs.end(); }

}  // namespace

// ============================================================== model spec + host weights
void ModelSpec::validate() const {  // reference model.cpp:68-80 (same messages)
    if (experts_per_block < 1) throw ConfigError("model: experts_per_block >= 1 violated");
    if (top_k < 1 || top_k > experts_per_block) throw ConfigError("model: 1 <= top_k <= experts_per_block violated");
    if (vocab_size < 2) throw ConfigError("model: vocab_size >= 2 violated");
    if (hidden_dim < 1) throw ConfigError("model: hidden_dim >= 1 violated");
    if (ffn_dim < 1) throw ConfigError("model: ffn_dim >= 1 violated");
    if (num_layers < 1) throw ConfigError("model: num_layers >= 1 violated");
    if (gate_skew < 0.0) throw ConfigError("model: gate_skew >= 0 violated");
    if (!moe_layer_mask.empty() && (int)moe_layer_mask.size() != num_layers)
        throw ConfigError("model: moe_layer_mask length must equal num_layers");
    const auto m = effective_mask();
    if (std::none_of(m.begin(), m.end(), [](uint8_t b) { return b != 0; }))
        throw ConfigError("model: at least one layer must be an MoE block");
}
std::vector<uint8_t> ModelSpec::effective_mask() const {
    return moe_layer_mask.empty() ? std::vector<uint8_t>((size_t)num_layers, 1) : moe_layer_mask;
}
int ModelSpec::moe_layer_count() const {
    const auto m = effective_mask();
    return (int)std::count_if(m.begin(), m.end(), [](uint8_t b) { return b != 0; });
}
int ModelSpec::moe_layer_index(int moe_ordinal) const {
    const auto m = effective_mask();
    for (int l = 0, seen = 0; l < num_layers; ++l)
        if (m[l] && seen++ == moe_ordinal) return l;
    throw InvariantError("moe_layer_index: ordinal out of range");
}

ModelWeights build_model(const ModelSpec& spec) {  // draw order of reference model.cpp:106-143
    spec.validate();
    ModelWeights w;
    w.spec = spec;
    const int d = spec.hidden_dim, f = spec.ffn_dim, E = spec.experts_per_block, V = spec.vocab_size;
    const double sd = 1.0 / std::sqrt((double)d);
    Rng rng(spec.seed);
    auto fill = [&](std::vector<double>& v, size_t n) {
        v.resize(n);
        for (auto& x : v) x = sd * gaussian(rng);
    };
    const auto mask = spec.effective_mask();
    fill(w.embedding, (size_t)V * d);
    w.layers.resize(spec.num_layers);
    for (int l = 0; l < spec.num_layers; ++l) {
        LayerWeights& L = w.layers[l];
        L.is_moe = mask[l] != 0;
        fill(L.mix, (size_t)d * d);
        if (L.is_moe) {
            fill(L.gate, (size_t)d * E);
            L.gate_bias.resize(E);
            for (int e = 0; e < E; ++e) L.gate_bias[e] = spec.gate_skew * (1.0 - (double)e / E);
            L.experts.resize(E);
            for (auto& x : L.experts) {
                fill(x.up, (size_t)d * f);
                fill(x.down, (size_t)f * d);
            }
        } else {
            fill(L.ffn.up, (size_t)d * f);
            fill(L.ffn.down, (size_t)f * d);
        }
    }
    fill(w.head, (size_t)d * V);
    return w;
}

std::vector<double> softmax(std::span<const double> logits) {
    if (logits.empty()) throw InvariantError("softmax: empty input");
    if (!finite_all(logits)) throw InvariantError("softmax: non-finite input");
    const double mx = *std::max_element(logits.begin(), logits.end());
    std::vector<double> p(logits.size());
    double sum = 0.0;
    for (size_t i = 0; i < p.size(); ++i) sum += (p[i] = std::exp(logits[i] - mx));
    for (double& v : p) v /= sum;
    return p;
}

std::vector<int> route_topk(std::span<const double> gate_logits, int k) {
    if (k > (int)gate_logits.size()) throw InvariantError("route_topk: k exceeds expert count");
    if (k < 0) throw InvariantError("route_topk: negative k");
    std::vector<int> idx(gate_logits.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return gate_logits[a] > gate_logits[b]; });
    idx.resize(k);
    return idx;
}

int greedy_next(std::span<const double> logits) {
    if (logits.empty()) throw InvariantError("greedy_next: empty logits");
    if (!finite_all(logits)) throw InvariantError("greedy_next: non-finite logits");
    return (int)(std::max_element(logits.begin(), logits.end()) - logits.begin());
}

int sample_next(std::span<const double> logits, double temperature, Rng& rng) {
    if (temperature <= 0.0) throw ConfigError("sample_next: temperature must be > 0");
    std::vector<double> sc(logits.begin(), logits.end());
    for (double& v : sc) v /= temperature;
    const auto p = softmax(sc);
    const double u = uniform01(rng);
    double cum = 0.0;
    for (size_t i = 0; i < p.size(); ++i)
        if (u < (cum += p[i])) return (int)i;
    return (int)p.size() - 1;
}

// ============================================================== engines per ModelWeights
namespace {

struct EngineSlot {
    std::unique_ptr<smoe::Engine> eng;
    uint64_t fingerprint = 0;
    int max_batch = 0, max_gamma = 0;
    const AffinityTable* aff_ptr = nullptr;
    uint64_t aff_fp = 0;
};
std::mutex g_mu;
std::map<const ModelWeights*, EngineSlot> g_engines;

// Content hash of every weight tensor (the drop-in API takes ModelWeights by reference every call, so a
// caller may refill it in place between calls; the device copy is rebuilt whenever any value changed).
// Four independent multiply-xor lanes per tensor, tensors hashed on all host threads, combined in order.
uint64_t hash_doubles(const std::vector<double>& v) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(v.data());
    const size_t n = v.size();
    uint64_t h[4] = {0x9e3779b97f4a7c15ull, 0xc2b2ae3d27d4eb4full, 0x165667b19e3779f9ull, 0x27d4eb2f165667c5ull};
    size_t i = 0;
    for (; i + 4 <= n; i += 4)
        for (int j = 0; j < 4; ++j) h[j] = ((h[j] ^ w[i + j]) * 0x100000001b3ull) ^ (h[j] >> 29);
    for (; i < n; ++i) h[0] = ((h[0] ^ w[i]) * 0x100000001b3ull) ^ (h[0] >> 29);
    uint64_t out = n;
    for (int j = 0; j < 4; ++j) out = fnv1a64(&h[j], sizeof h[j], out);
    return out;
}

uint64_t fingerprint(const ModelWeights& w) {
    std::vector<const std::vector<double>*> ts{&w.embedding, &w.head};
    for (const auto& L : w.layers) {
        ts.push_back(&L.mix);
        ts.push_back(&L.gate);
        for (const auto& x : L.experts) { ts.push_back(&x.up); ts.push_back(&x.down); }
        ts.push_back(&L.ffn.up);
        ts.push_back(&L.ffn.down);
    }
    std::vector<uint64_t> hs(ts.size());
    const size_t nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::atomic<size_t> next{0};
    auto work = [&] {
        for (size_t i; (i = next.fetch_add(1)) < ts.size();) hs[i] = hash_doubles(*ts[i]);
    };
    std::vector<std::thread> th;
    for (size_t t = 1; t < nth; ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    uint64_t h = 0xcbf29ce484222325ull;
    const ModelSpec& s = w.spec;
    const int dims[7] = {s.num_layers, s.experts_per_block, s.top_k, s.hidden_dim, s.ffn_dim, s.vocab_size,
                         (int)s.moe_layer_mask.size()};
    h = fnv1a64(dims, sizeof dims, h);
    h = fnv1a64(&s.gate_skew, sizeof s.gate_skew, h);
    return fnv1a64(hs.data(), hs.size() * sizeof(uint64_t), h);
}

uint64_t aff_fingerprint(const AffinityTable& a) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const auto& d : a.dist) h = fnv1a64(d.data(), d.size() * sizeof(double), h);
    return h;
}

// The engine for `w`, (re)built and uploaded when needed; affinity installed when given.
smoe::Engine& engine_for(const ModelWeights& w, int batch, int gamma, const AffinityTable* aff) {
    const uint64_t fp = fingerprint(w);
    EngineSlot& slot = g_engines[&w];
    if (!slot.eng || slot.fingerprint != fp || batch > slot.max_batch || gamma > slot.max_gamma) {
        const ModelSpec& s = w.spec;
        s.validate();
        const char* dt = std::getenv("SPECMOE_B200_DTYPE");
        const bool bf16 = dt && std::string(dt) == "bf16";
        smoe_engine_config c{};
        c.num_layers = s.num_layers;
        c.experts = s.experts_per_block;
        c.top_k = s.top_k;
        c.hidden = s.hidden_dim;
        c.ffn = s.ffn_dim;
        c.vocab = s.vocab_size;
        c.gate_skew = s.gate_skew;
        c.seed = s.seed;
        c.moe_mask = s.moe_layer_mask.empty() ? nullptr : s.moe_layer_mask.data();
        c.expert_kind = SMOE_EXPERT_TANH2;
        c.weight_type = bf16 ? SMOE_BF16 : SMOE_F32;
        c.max_batch = std::max({batch, slot.max_batch, 8});
        c.max_gamma = std::max({gamma, slot.max_gamma, 10});
        c.gemm_backend = SMOE_GEMM_AUTO;
        slot.eng.reset();
        slot.eng = std::make_unique<smoe::Engine>(c);
        smoe::Engine& e = *slot.eng;
        e.upload_tensor("embedding", -1, -1, w.embedding.data(), (long long)w.embedding.size());
        e.upload_tensor("head", -1, -1, w.head.data(), (long long)w.head.size());
        for (int l = 0; l < s.num_layers; ++l) {
            const LayerWeights& L = w.layers[l];
            e.upload_tensor("mix", l, -1, L.mix.data(), (long long)L.mix.size());
            if (L.is_moe) {
                e.upload_tensor("gate", l, -1, L.gate.data(), (long long)L.gate.size());
                e.upload_tensor("gate_bias", l, -1, L.gate_bias.data(), (long long)L.gate_bias.size());
                for (int x = 0; x < s.experts_per_block; ++x) {
                    e.upload_tensor("up", l, x, L.experts[x].up.data(), (long long)L.experts[x].up.size());
                    e.upload_tensor("down", l, x, L.experts[x].down.data(), (long long)L.experts[x].down.size());
                }
            } else {
                e.upload_tensor("up", l, -1, L.ffn.up.data(), (long long)L.ffn.up.size());
                e.upload_tensor("down", l, -1, L.ffn.down.data(), (long long)L.ffn.down.size());
            }
        }
        slot.fingerprint = fp;
        slot.max_batch = c.max_batch;
        slot.max_gamma = c.max_gamma;
        slot.aff_ptr = nullptr;
        slot.aff_fp = 0;
    }
    smoe::Engine& e = *slot.eng;
    if (aff) {
        const uint64_t afp = aff_fingerprint(*aff);
        if (slot.aff_ptr != aff || slot.aff_fp != afp) {
            if ((int)aff->dist.size() != e.M || aff->experts != e.E)
                throw InvariantError("affinity table shape does not match the model");
            e.affinity.clear();
            for (const auto& d : aff->dist) e.affinity.insert(e.affinity.end(), d.begin(), d.end());
            e.have_affinity = true;
            ++e.affinity_gen;
            slot.aff_ptr = aff;
            slot.aff_fp = afp;
        }
    }
    return e;
}

smoe::RunCfg run_cfg(const SpecConfig& c, DraftPolicy p, const TierConfig& t, uint64_t seed, bool trace) {
    smoe::RunCfg r;
    r.gamma = c.gamma;
    r.n_draft = c.n_draft;
    r.max_new_tokens = c.max_new_tokens;
    r.use_affinity = c.use_affinity ? 1 : 0;
    r.warmup_steps = c.warmup_steps;
    r.policy = static_cast<int>(p);
    r.collect_trace = trace ? 1 : 0;
    r.run_seed = seed;
    r.device_capacity_bytes = t.device_capacity_bytes;
    r.bytes_per_expert = t.bytes_per_expert;
    r.host_bandwidth = t.host_bandwidth;
    r.ssd_bandwidth = t.ssd_bandwidth;
    r.compute_rate = t.compute_rate_tokens_per_s;
    r.compute_cost_per_expert = t.compute_cost_per_active_expert_s;
    r.mode = c.mode == DecodeMode::sampling ? 1 : 0;  // device-side draws, host RNG order (sampling.cu)
    r.temperature = c.temperature;
    return r;
}

RunResult to_result(const smoe::RunOut& o, int M, int E) {
    RunResult r;
    r.tokens = o.tokens;
    RunMetrics& m = r.metrics;
    m.tau_mean = o.tau_mean;
    m.tokens_total = o.tokens_total;
    m.phases = o.phases;
    m.speculation_s = o.speculation_s;
    m.verification_s = o.verification_s;
    m.modeled_seconds = o.modeled_seconds;
    m.tokens_per_sec = o.tokens_per_sec;
    m.bytes_spec = o.bytes_spec;
    m.bytes_verify = o.bytes_verify;
    m.bytes_baseline = o.bytes_baseline;
    m.bytes_total = o.bytes_total;
    m.setup_bytes = o.setup_bytes;
    m.warmup_bytes = o.warmup_bytes;
    m.lambda = o.lambda;
    m.c_measured = o.c_measured;
    for (const auto& le : o.ledger)
        r.ledger.add(static_cast<Phase>(le.phase), le.step, ExpertKey{le.layer, le.expert}, le.bytes);
    for (const auto& oc : o.outcomes)
        r.outcomes.push_back(StepOutcome{oc.seq, oc.phase, oc.drafts, oc.accepted, oc.correction, oc.generated});
    for (const auto& t : o.trace) r.trace.push_back(TraceRow{t.step, t.seq, t.layer, t.experts});
    r.hotness = HotnessCounter(M, E);
    for (int l = 0; l < M; ++l)
        for (int e = 0; e < E; ++e) r.hotness.counts[l][e] = o.hotness[(size_t)l * E + e];
    for (size_t i = 0; i + 3 < o.lambda_inputs.size(); i += 4)
        r.lambda_inputs.push_back(
            LambdaInputs{o.lambda_inputs[i], o.lambda_inputs[i + 1], o.lambda_inputs[i + 2], o.lambda_inputs[i + 3]});
    return r;
}

ActivationRow activations_of(const smoe::Engine& e, const std::vector<int>& raw, const std::vector<int>& fin, int T,
                             int row) {
    ActivationRow out(e.M);
    for (int m = 0; m < e.M; ++m)
        for (int k = 0; k < e.K; ++k) {
            out[m].raw.push_back(raw[((size_t)m * T + row) * e.K + k]);
            out[m].final.push_back(fin.empty() ? raw[((size_t)m * T + row) * e.K + k]
                                               : fin[((size_t)m * T + row) * e.K + k]);
        }
    return out;
}

void read_log(smoe::Engine& e, const int* log, int slot, int T, std::vector<int>& out) {
    out.resize((size_t)e.M * T * e.K);
    SMOE_CUDA(cudaMemcpy2DAsync(out.data(), sizeof(int) * T * e.K, log + (size_t)slot * e.M * e.Tmax * e.K,
                                sizeof(int) * e.Tmax * e.K, sizeof(int) * T * e.K, e.M, cudaMemcpyDeviceToHost,
                                e.stream));
}

std::vector<std::vector<double>> read_logits(smoe::Engine& e, int T) {
    std::vector<float> buf((size_t)T * e.V);
    SMOE_CUDA(cudaMemcpyAsync(buf.data(), e.logits, buf.size() * sizeof(float), cudaMemcpyDeviceToHost, e.stream));
    e.sync();
    std::vector<std::vector<double>> out(T, std::vector<double>(e.V));
    for (int t = 0; t < T; ++t)
        for (int v = 0; v < e.V; ++v) out[t][v] = buf[(size_t)t * e.V + v];
    return out;
}

}  // namespace

ForwardResult forward(const ModelWeights& weights, std::span<const int> prefix, const RestrictedExperts* restricted,
                      const AffinityTable* affinity) {
    const ModelSpec& s = weights.spec;
    if (prefix.empty()) throw InvariantError("forward: empty prefix");
    for (int t : prefix)
        if (t < 0 || t >= s.vocab_size) throw InvariantError("forward: token out of range");
    if (restricted) {
        if ((int)restricted->per_layer.size() != s.moe_layer_count())
            throw InvariantError("forward: restricted set count != MoE layer count");
        for (const auto& st : restricted->per_layer)
            if ((int)st.size() < s.top_k) throw InvariantError("forward: restricted set smaller than top_k");
    }
    return guard([&] {
        std::lock_guard<std::mutex> lk(g_mu);
        smoe::Engine& e = engine_for(weights, 1, 1, affinity);
        const std::vector<int> p(prefix.begin(), prefix.end());
        ForwardResult fr;
        std::vector<float> lg(e.V);
        std::vector<int> raw((size_t)e.M * e.K), fin((size_t)e.M * e.K);
        if (restricted) {
            e.set_draft_sets(restricted->per_layer, 0);
            e.reset_sequences({p});
            int zero = 0;
            e.upload_ints(e.row_seq, &zero, 1);
            e.pass(1, e.row_seq, nullptr, 0, true, affinity ? 1 : 0, 0);
            e.sync();
            e.check_flags();
            SMOE_CUDA(cudaMemcpy(lg.data(), e.logits, sizeof(float) * e.V, cudaMemcpyDeviceToHost));
            std::vector<int> r, f;
            read_log(e, e.raw_log, 0, 1, r);
            read_log(e, e.fin_log, 0, 1, f);
            e.sync();
            raw = r;
            fin = f;
        } else {
            e.forward_one(p, nullptr, 0, 0, lg.data(), raw.data(), fin.data());
        }
        fr.logits.assign(lg.begin(), lg.end());
        for (int m = 0; m < e.M; ++m) {
            LayerActivation a;
            a.raw.assign(raw.begin() + (size_t)m * e.K, raw.begin() + (size_t)(m + 1) * e.K);
            a.final.assign(fin.begin() + (size_t)m * e.K, fin.begin() + (size_t)(m + 1) * e.K);
            fr.activations.push_back(std::move(a));
        }
        return fr;
    });
}

// ============================================================== drafting
AffinityTable build_affinity_table(const ModelWeights& weights) {  // reference drafting.cpp:28-57 order
    const int E = weights.spec.experts_per_block;
    AffinityTable t;
    t.experts = E;
    for (const LayerWeights& L : weights.layers) {
        if (!L.is_moe) continue;
        std::vector<double> D((size_t)E * E, 0.0);
        for (int i = 0; i < E; ++i)
            for (int j = i + 1; j < E; ++j) {
                double ss = 0.0;
                const auto& a = L.experts[i];
                const auto& b = L.experts[j];
                for (size_t k = 0; k < a.up.size(); ++k) ss += (a.up[k] - b.up[k]) * (a.up[k] - b.up[k]);
                for (size_t k = 0; k < a.down.size(); ++k) ss += (a.down[k] - b.down[k]) * (a.down[k] - b.down[k]);
                D[(size_t)i * E + j] = D[(size_t)j * E + i] = std::sqrt(ss);
            }
        t.dist.push_back(std::move(D));
    }
    return t;
}

void save_affinity_csv(const AffinityTable& t, std::ostream& out) {
    out << "# specmoe-affinity v1 layers=" << t.dist.size() << " experts=" << t.experts << "\n";
    out << "layer,i,j,distance\n";
    char buf[64];
    for (size_t l = 0; l < t.dist.size(); ++l)
        for (int i = 0; i < t.experts; ++i)
            for (int j = i + 1; j < t.experts; ++j) {
                std::snprintf(buf, sizeof buf, "%.17g", t.at((int)l, i, j));
                out << l << ',' << i << ',' << j << ',' << buf << "\n";
            }
}
void save_affinity_csv(const AffinityTable& t, const std::string& path) {
    std::ofstream out(path);
    if (!out) throw ConfigError("cannot open for writing: " + path);
    save_affinity_csv(t, out);
}
AffinityTable load_affinity_csv(std::istream& in) {
    std::string line;
    if (!std::getline(in, line)) throw ConfigError("affinity file: empty");
    int layers = 0, experts = 0;
    if (std::sscanf(line.c_str(), "# specmoe-affinity v1 layers=%d experts=%d", &layers, &experts) != 2)
        throw ConfigError("affinity file: bad or missing version header");
    if (!std::getline(in, line) || line != "layer,i,j,distance") throw ConfigError("affinity file: bad column header");
    AffinityTable t;
    t.experts = experts;
    t.dist.assign(layers, std::vector<double>((size_t)experts * experts, 0.0));
    for (int lineno = 3; std::getline(in, line); ++lineno) {
        if (line.empty()) continue;
        int l = 0, i = 0, j = 0;
        double d = 0.0;
        if (std::sscanf(line.c_str(), "%d,%d,%d,%lf", &l, &i, &j, &d) != 4)
            throw ConfigError("affinity file: parse error at line " + std::to_string(lineno));
        if (l < 0 || l >= layers || i < 0 || i >= experts || j < 0 || j >= experts)
            throw ConfigError("affinity file: index out of range at line " + std::to_string(lineno));
        t.dist[l][(size_t)i * experts + j] = t.dist[l][(size_t)j * experts + i] = d;
    }
    return t;
}
AffinityTable load_affinity_csv(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ConfigError("cannot open: " + path);
    return load_affinity_csv(in);
}

int nearest_draft_expert(const AffinityTable& t, int layer, int raw, std::span<const int> draft,
                         std::span<const int> excluded) {
    if (has(draft, raw) && !has(excluded, raw)) return raw;
    int best = -1;
    double bd = 0.0;
    for (int c : draft) {
        if (has(excluded, c)) continue;
        const double d = t.at(layer, raw, c);
        if (best < 0 || d < bd || (d == bd && c < best)) { best = c; bd = d; }
    }
    if (best < 0) throw InvariantError("nearest_draft_expert: empty candidate set");
    return best;
}

int surrogate_draft_expert(int layer, int raw, size_t prefix_len, std::span<const int> draft,
                           std::span<const int> excluded) {
    if (has(draft, raw) && !has(excluded, raw)) return raw;
    std::vector<int> cand;
    for (int c : draft)
        if (!has(excluded, c)) cand.push_back(c);
    if (cand.empty()) throw InvariantError("surrogate_draft_expert: empty candidate set");
    std::sort(cand.begin(), cand.end());
    const uint64_t h = substream(0x5eed5eedull, (uint64_t)layer << 32 | (uint32_t)raw, prefix_len);
    return cand[h % cand.size()];
}

const char* to_string(DraftPolicy p) {
    switch (p) {
        case DraftPolicy::random: return "random";
        case DraftPolicy::hot_global: return "hot_global";
        case DraftPolicy::hot_temporal: return "hot_temporal";
    }
    return "?";
}
DraftPolicy draft_policy_from_string(const std::string& n) {
    if (n == "random") return DraftPolicy::random;
    if (n == "hot_global") return DraftPolicy::hot_global;
    if (n == "hot_temporal") return DraftPolicy::hot_temporal;
    throw ConfigError("unknown draft policy: " + n);
}

void HotnessCounter::reset() {
    for (auto& c : counts) std::fill(c.begin(), c.end(), 0);
    routed_tokens = 0;
}

void record_activations(HotnessCounter& counter, const ActivationRecord& record) {
    for (const ActivationRow& row : record.rows) {
        if (row.size() != counter.counts.size()) throw InvariantError("record_activations: row layer count mismatch");
        for (size_t l = 0; l < row.size(); ++l)
            for (int e : row[l].raw) {
                if (e < 0 || e >= (int)counter.counts[l].size())
                    throw InvariantError("record_activations: expert index out of range");
                ++counter.counts[l][e];
            }
        ++counter.routed_tokens;
    }
}

std::vector<std::vector<int>> select_draft_experts(DraftPolicy policy, const HotnessCounter& counter,
                                                   const DraftState& current, int E, Rng& rng) {
    const int n = current.n_draft;
    if (n > E) throw ConfigError("select_draft_experts: n_draft > experts_per_block");
    const size_t layers = counter.counts.empty() ? current.sets.size() : counter.counts.size();
    std::vector<std::vector<int>> out(layers);
    for (size_t l = 0; l < layers; ++l) {
        if (policy == DraftPolicy::random) {
            std::vector<int> pool(E);
            std::iota(pool.begin(), pool.end(), 0);
            for (int i = 0; i < n; ++i) {
                const size_t j = (size_t)i + (size_t)(uniform01(rng) * (double)(pool.size() - (size_t)i));
                std::swap(pool[i], pool[j]);
            }
            pool.resize(n);
            std::sort(pool.begin(), pool.end());
            out[l] = std::move(pool);
            continue;
        }
        const auto& c = counter.counts[l];
        std::vector<int> idx(c.size());
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return c[a] > c[b]; });
        idx.resize(std::min<size_t>(idx.size(), (size_t)n));
        std::vector<int> picked;
        for (int e : idx)
            if (c[e] > 0) picked.push_back(e);
        if ((int)picked.size() < n && l < current.sets.size())
            for (int e : current.sets[l]) {
                if ((int)picked.size() == n) break;
                if (!has(picked, e)) picked.push_back(e);
            }
        if ((int)picked.size() != n) throw InvariantError("select_draft_experts: cannot assemble N draft experts");
        std::sort(picked.begin(), picked.end());
        out[l] = std::move(picked);
    }
    return out;
}

double skewness(const HotnessCounter& counter, double frac) {
    if (counter.counts.empty()) throw InvariantError("skewness: empty counter");
    if (counter.routed_tokens == 0) throw InvariantError("skewness: no routed tokens");
    double acc = 0.0;
    for (const auto& c : counter.counts) {
        const uint64_t tot = std::accumulate(c.begin(), c.end(), uint64_t{0});
        if (tot == 0) throw InvariantError("skewness: layer with no routed tokens");
        std::vector<uint64_t> s(c);
        std::sort(s.begin(), s.end(), std::greater<>());
        const auto top = (size_t)std::ceil(frac * (double)c.size());
        acc += (double)std::accumulate(s.begin(), s.begin() + top, uint64_t{0}) / (double)tot;
    }
    return acc / (double)counter.counts.size();
}

// ============================================================== memsim
const char* to_string(Phase p) {
    switch (p) {
        case Phase::speculation: return "speculation";
        case Phase::verification: return "verification";
        case Phase::baseline_step: return "baseline-step";
    }
    return "?";
}
uint64_t bytes_per_expert(const ModelSpec& s) { return 2ull * s.hidden_dim * s.ffn_dim * 4ull; }

void TierConfig::validate(int n_draft, int moe_layers) const {
    if (host_bandwidth <= 0.0) throw ConfigError("tier: host_bandwidth > 0 violated");
    if (ssd_bandwidth < 0.0) throw ConfigError("tier: ssd_bandwidth >= 0 violated");
    if (bytes_per_expert == 0) throw ConfigError("tier: bytes_per_expert > 0 violated");
    if (compute_rate_tokens_per_s <= 0.0) throw ConfigError("tier: compute_rate > 0 violated");
    if (compute_cost_per_active_expert_s < 0.0) throw ConfigError("tier: expert compute cost >= 0 violated");
    if (device_capacity_bytes < (uint64_t)n_draft * moe_layers * bytes_per_expert)
        throw ConfigError("tier: device capacity below N * moe_layers * bytes_per_expert");
}

void MigrationLedger::add(Phase phase, int step, ExpertKey key, uint64_t bytes) {
    entries_.push_back(LedgerEntry{phase, step, key, bytes});
    totals_.total += bytes;
    (phase == Phase::speculation ? totals_.speculation
                                 : phase == Phase::verification ? totals_.verification : totals_.baseline) += bytes;
    totals_.migrations = entries_.size();
}
uint64_t MigrationLedger::total(Phase phase) const {
    return phase == Phase::speculation ? totals_.speculation
           : phase == Phase::verification ? totals_.verification : totals_.baseline;
}
void MigrationLedger::reset() {
    entries_.clear();
    totals_ = Totals{};
}
void MigrationLedger::write_csv(std::ostream& out) const {
    out << "phase,step,layer,expert,bytes\n";
    for (const auto& e : entries_)
        out << to_string(e.phase) << ',' << e.step << ',' << e.key.layer << ',' << e.key.expert << ',' << e.bytes << "\n";
}

ResidencyState::ResidencyState(const ModelSpec& spec, const TierConfig& tier)
    : tier_(tier), moe_layers_(spec.moe_layer_count()), experts_(spec.experts_per_block) {
    tier_.validate(0, moe_layers_);
}
void ResidencyState::check_key(ExpertKey k) const {
    if (k.layer < 0 || k.layer >= moe_layers_ || k.expert < 0 || k.expert >= experts_)
        throw InvariantError("residency: expert key out of range");
}
bool ResidencyState::device_resident(ExpertKey k) const { return residents_.count(k) != 0; }
bool ResidencyState::pinned(ExpertKey k) const { return pinned_.count(k) != 0; }
void ResidencyState::admit(ExpertKey key, const std::set<ExpertKey>& keep) {
    while (device_bytes_ + tier_.bytes_per_expert > tier_.device_capacity_bytes) {
        auto victim = residents_.end();
        for (auto it = residents_.begin(); it != residents_.end(); ++it) {
            if (pinned_.count(it->first) || keep.count(it->first)) continue;
            if (victim == residents_.end() || it->second < victim->second) victim = it;
        }
        if (victim == residents_.end())
            throw InvariantError("residency: device capacity exhausted with no evictable expert");
        residents_.erase(victim);
        device_bytes_ -= tier_.bytes_per_expert;
    }
    residents_.emplace(key, arrival_seq_++);
    device_bytes_ += tier_.bytes_per_expert;
}
uint64_t ensure_resident(const std::set<ExpertKey>& keys, Phase phase, int step, MigrationLedger& ledger,
                         ResidencyState& r) {
    uint64_t bytes = 0;
    for (ExpertKey k : keys) {
        r.check_key(k);
        if (r.device_resident(k)) continue;
        r.admit(k, keys);
        ledger.add(phase, step, k, r.tier_.bytes_per_expert);
        bytes += r.tier_.bytes_per_expert;
    }
    return bytes;
}
uint64_t pin_draft_experts(const std::vector<std::vector<int>>& sets, ResidencyState& r, MigrationLedger& ledger,
                           Phase phase, int step) {
    if ((int)sets.size() != r.moe_layers_) throw InvariantError("pin_draft_experts: set count != MoE layer count");
    std::set<ExpertKey> target;
    for (int l = 0; l < r.moe_layers_; ++l)
        for (int e : sets[l]) {
            ExpertKey k{l, e};
            r.check_key(k);
            if (!target.insert(k).second) throw InvariantError("pin_draft_experts: duplicate expert in draft set");
        }
    for (auto it = r.pinned_.begin(); it != r.pinned_.end();) it = target.count(*it) ? std::next(it) : r.pinned_.erase(it);
    uint64_t bytes = 0;
    for (ExpertKey k : target) {
        if (!r.device_resident(k)) {
            r.admit(k, target);
            ledger.add(phase, step, k, r.tier_.bytes_per_expert);
            bytes += r.tier_.bytes_per_expert;
        }
        r.pinned_.insert(k);
    }
    return bytes;
}
void flush_transients(ResidencyState& r) {
    for (auto it = r.residents_.begin(); it != r.residents_.end();) {
        if (r.pinned_.count(it->first)) {
            ++it;
        } else {
            r.device_bytes_ -= r.tier_.bytes_per_expert;
            it = r.residents_.erase(it);
        }
    }
}
StepTiming step_latency(uint64_t toks, uint64_t experts, uint64_t bytes, const TierConfig& tier, bool overlap) {
    StepTiming t;
    t.overlap = overlap;
    t.compute_s = (double)toks / tier.compute_rate_tokens_per_s + (double)experts * tier.compute_cost_per_active_expert_s;
    t.migration_s = (double)bytes / tier.offload_bandwidth();
    t.total_s = overlap ? std::max(t.compute_s, t.migration_s) : t.compute_s + t.migration_s;
    return t;
}

// ============================================================== specdec
const char* to_string(DecodeMode m) { return m == DecodeMode::greedy ? "greedy" : "sampling"; }
void SpecConfig::validate() const {
    if (gamma < 1) throw ConfigError("spec: gamma >= 1 violated");
    if (batch < 1) throw ConfigError("spec: batch >= 1 violated");
    if (max_new_tokens < 1) throw ConfigError("spec: max_new_tokens >= 1 violated");
    if (prompt_len < 1) throw ConfigError("spec: prompt_len >= 1 violated");
    if (mode == DecodeMode::sampling && temperature <= 0.0)
        throw ConfigError("spec: temperature > 0 violated in sampling mode");
    if (warmup_steps < 1) throw ConfigError("spec: warmup_steps >= 1 violated");
}

// Draft generation: gamma restricted passes over all sequences at once; drafts stay on device in
// greedy mode, sampling draws on the host from the device logits with the reference's RNG order.
SpeculationResult speculate(const ModelWeights& weights, const DraftState& ds, const AffinityTable* affinity,
                            const std::vector<std::vector<int>>& prefixes, int gamma, DecodeMode mode,
                            double temperature, Rng& rng) {
    SpeculationResult res;
    const size_t n = prefixes.size();
    res.drafts.assign(n, {});
    res.draw_probs.assign(n, {});
    res.distinct_draft_experts.assign((size_t)std::max(0, gamma), 0);
    if (n == 0 || gamma <= 0) return res;
    return guard([&] {
        std::lock_guard<std::mutex> lk(g_mu);
        smoe::Engine& e = engine_for(weights, (int)n, gamma, affinity);
        e.set_draft_sets(ds.sets, ds.n_draft);
        e.reset_sequences(prefixes);
        std::vector<int> rows(n);
        std::iota(rows.begin(), rows.end(), 0);
        e.upload_ints(e.row_seq, rows.data(), n);
        std::vector<std::vector<int>> raw(gamma), fin(gamma);
        for (int t = 0; t < gamma; ++t) {
            e.pass((int)n, e.row_seq, nullptr, t, true, affinity ? 1 : 0, 0);
            read_log(e, e.raw_log, 0, (int)n, raw[t]);
            read_log(e, e.fin_log, 0, (int)n, fin[t]);
            if (mode == DecodeMode::greedy) {
                smoe::launch_scatter_tokens(e.amax, e.row_seq, nullptr, t, (int)n, e.drafts, e.stride, e.stream);
                std::vector<int> am(n);
                SMOE_CUDA(cudaMemcpyAsync(am.data(), e.amax, sizeof(int) * n, cudaMemcpyDeviceToHost, e.stream));
                e.sync();
                e.check_flags();
                for (size_t s = 0; s < n; ++s) res.drafts[s].push_back(am[s]);
            } else {
                auto lg = read_logits(e, (int)n);
                e.check_flags();
                std::vector<int> dr((size_t)e.Bmax * e.stride);
                SMOE_CUDA(cudaMemcpy(dr.data(), e.drafts, sizeof(int) * dr.size(), cudaMemcpyDeviceToHost));
                for (size_t s = 0; s < n; ++s) {
                    std::vector<double> sc(lg[s]);
                    for (double& v : sc) v /= temperature;
                    res.draw_probs[s].push_back(softmax(sc));
                    const int tok = sample_next(lg[s], temperature, rng);
                    res.drafts[s].push_back(tok);
                    dr[s * e.stride + t] = tok;
                }
                SMOE_CUDA(cudaMemcpy(e.drafts, dr.data(), sizeof(int) * dr.size(), cudaMemcpyHostToDevice));
            }
        }
        e.sync();
        for (int t = 0; t < gamma; ++t) {
            std::set<std::pair<int, int>> executed;
            for (size_t s = 0; s < n; ++s) {
                ActivationRow row = activations_of(e, raw[t], fin[t], (int)n, (int)s);
                for (size_t l = 0; l < row.size(); ++l)
                    for (int x : row[l].final) executed.insert({(int)l, x});
                res.activations.rows.push_back(std::move(row));
            }
            res.distinct_draft_experts[t] = executed.size();
        }
        return res;
    });
}

namespace {
// Target logits + raw routing of prefix ++ drafts[:i] for i = 0..gamma: one verify pass.
VerifyResult verify_pass(const ModelWeights& w, const std::vector<int>& prefix, const std::vector<int>& drafts) {
    std::lock_guard<std::mutex> lk(g_mu);
    const int g = (int)drafts.size();
    smoe::Engine& e = engine_for(w, 1, g, nullptr);
    if (prefix.empty()) throw InvariantError("forward: empty prefix");
    e.reset_sequences({prefix});
    std::vector<int> dr((size_t)e.stride, 0), rseq(g + 1, 0), rext(g + 1);
    for (int i = 0; i < g; ++i) {
        if (drafts[i] < 0 || drafts[i] >= e.V) throw InvariantError("forward: token out of range");
        dr[i] = drafts[i];
    }
    for (int i = 0; i <= g; ++i) rext[i] = i;
    e.upload_ints(e.drafts, dr.data(), dr.size());
    e.upload_ints(e.row_seq, rseq.data(), rseq.size());
    e.upload_ints(e.row_extra, rext.data(), rext.size());
    e.pass(g + 1, e.row_seq, e.row_extra, 0, false, 0, 0);
    std::vector<int> raw;
    read_log(e, e.raw_log, 0, g + 1, raw);
    VerifyResult vr;
    vr.logits = read_logits(e, g + 1);
    e.check_flags();
    for (int i = 0; i <= g; ++i) vr.positions.rows.push_back(activations_of(e, raw, {}, g + 1, i));
    return vr;
}
}  // namespace

VerifyResult verify_greedy(const ModelWeights& weights, const std::vector<int>& prefix, const std::vector<int>& drafts) {
    return guard([&] {
        VerifyResult vr = verify_pass(weights, prefix, drafts);
        const int g = (int)drafts.size();
        int a = 0;
        while (a < g && drafts[a] == greedy_next(vr.logits[a])) ++a;
        vr.accepted = a;
        vr.correction = greedy_next(vr.logits[a]);
        return vr;
    });
}

VerifyResult verify_sampling(const ModelWeights& weights, const std::vector<int>& prefix,
                             const std::vector<int>& drafts, const std::vector<std::vector<double>>& draw_probs,
                             double temperature, Rng& rng) {
    const int g = (int)drafts.size();
    if ((int)draw_probs.size() != g) throw InvariantError("verify_sampling: draw_probs size != drafts size");
    return guard([&] {
        VerifyResult vr = verify_pass(weights, prefix, drafts);
        std::vector<std::vector<double>> p(g + 1);
        for (int i = 0; i <= g; ++i) {
            std::vector<double> sc(vr.logits[i]);
            for (double& v : sc) v /= temperature;
            p[i] = softmax(sc);
        }
        auto draw = [&](const std::vector<double>& dist, double norm) {
            const double u = uniform01(rng) * norm;
            double cum = 0.0;
            for (size_t j = 0; j < dist.size(); ++j)
                if (u < (cum += dist[j])) return (int)j;
            return (int)dist.size() - 1;
        };
        int a = 0, tok = -1;
        for (; a < g; ++a) {  // Leviathan acceptance, residual resample on first rejection
            const int x = drafts[a];
            const auto& q = draw_probs[a];
            if (q[x] <= 0.0) throw InvariantError("verify_sampling: zero draw probability for proposed token");
            if (uniform01(rng) < std::min(1.0, p[a][x] / q[x])) continue;
            std::vector<double> res(p[a].size());
            double norm = 0.0;
            for (size_t j = 0; j < res.size(); ++j) norm += (res[j] = std::max(0.0, p[a][j] - q[j]));
            if (norm <= 0.0) {
                res = p[a];
                norm = 1.0;
            }
            tok = draw(res, norm);
            break;
        }
        if (a == g) tok = draw(p[g], 1.0);
        vr.accepted = a;
        vr.correction = tok;
        return vr;
    });
}

RunResult run_specmoe(const ModelWeights& weights, const SpecConfig& config, DraftPolicy policy, const TierConfig& tier,
                      const std::vector<std::vector<int>>& prompts, uint64_t run_seed, const AffinityTable* affinity,
                      bool collect_trace) {
    config.validate();
    const ModelSpec& s = weights.spec;
    const int M = s.moe_layer_count(), E = s.experts_per_block;
    if (config.n_draft < s.top_k) throw ConfigError("spec: n_draft >= top_k violated");
    if (config.n_draft > E) throw ConfigError("spec: n_draft <= experts_per_block violated");
    if (prompts.empty()) throw ConfigError("run_specmoe: no prompts");
    tier.validate(config.n_draft, M);
    if (config.use_affinity && !affinity) throw InvariantError("run_specmoe: affinity table required but missing");
    return guard([&] {
        std::lock_guard<std::mutex> lk(g_mu);
        smoe::Engine& e = engine_for(weights, (int)prompts.size(), config.gamma, config.use_affinity ? affinity : nullptr);
        smoe::RunOut o = smoe::run_specmoe(e, run_cfg(config, policy, tier, run_seed, collect_trace), prompts);
        return to_result(o, M, E);
    });
}

double speedup_eq1(double tau, int gamma, double c) {
    if (gamma < 1) throw ConfigError("speedup_eq1: gamma >= 1 violated");
    if (c < 0.0) throw ConfigError("speedup_eq1: c >= 0 violated");
    if (tau < 1.0 || tau > gamma + 1.0) throw ConfigError("speedup_eq1: tau outside [1, gamma+1]");
    return tau / (gamma * c + 1.0);
}
double speedup_eq2(double tau, int gamma, double c, double lambda) {
    if (gamma < 1) throw ConfigError("speedup_eq2: gamma >= 1 violated");
    if (c < 0.0) throw ConfigError("speedup_eq2: c >= 0 violated");
    if (lambda <= 0.0) throw ConfigError("speedup_eq2: lambda > 0 violated");
    if (tau < 1.0 || tau > gamma + 1.0) throw ConfigError("speedup_eq2: tau outside [1, gamma+1]");
    return tau / (gamma * c + lambda);
}
double measure_lambda(const std::vector<LambdaInputs>& phases, const TierConfig& tier) {
    if (phases.empty()) throw InvariantError("measure_lambda: empty run");
    double v = 0.0, s = 0.0;
    for (const auto& p : phases) {
        v += step_latency(p.verify_tokens, p.verify_experts, p.verify_experts * tier.bytes_per_expert, tier, false).total_s;
        s += step_latency(p.step_tokens, p.step_experts, p.step_experts * tier.bytes_per_expert, tier, false).total_s;
    }
    if (s <= 0.0) throw InvariantError("measure_lambda: zero single-step latency");
    return v / s;
}

// ============================================================== baselines
const char* to_string(BaselineKind k) {
    switch (k) {
        case BaselineKind::ondemand: return "ondemand";
        case BaselineKind::overlap: return "overlap";
        case BaselineKind::caching: return "caching";
    }
    return "?";
}
void BaselineConfig::validate() const {
    if (kind == BaselineKind::caching && (cache_fraction <= 0.0 || cache_fraction >= 1.0))
        throw ConfigError("baseline: 0 < cache_fraction < 1 violated");
    if (warmup_steps < 1) throw ConfigError("baseline: warmup_steps >= 1 violated");
}

namespace {
RunResult stepwise(const ModelWeights& w, const std::vector<std::vector<int>>& prompts, const SpecConfig& decode,
                   const TierConfig& tier, uint64_t run_seed, bool overlap, const std::vector<std::vector<int>>* pinned,
                   bool trace) {
    decode.validate();
    const ModelSpec& s = w.spec;
    const int M = s.moe_layer_count(), E = s.experts_per_block;
    if (prompts.empty()) throw ConfigError("baseline run: no prompts");
    tier.validate(0, M);
    return guard([&] {
        std::lock_guard<std::mutex> lk(g_mu);
        smoe::Engine& e = engine_for(w, (int)prompts.size(), decode.gamma, nullptr);
        smoe::RunCfg c = run_cfg(decode, DraftPolicy::hot_temporal, tier, run_seed, trace);
        c.overlap = overlap ? 1 : 0;
        smoe::RunOut o = smoe::run_ondemand(e, c, prompts, pinned);
        return to_result(o, M, E);
    });
}
}  // namespace

RunResult run_ondemand(const ModelWeights& w, const std::vector<std::vector<int>>& prompts, const SpecConfig& decode,
                       const TierConfig& tier, uint64_t run_seed, bool trace) {
    return stepwise(w, prompts, decode, tier, run_seed, false, nullptr, trace);
}
RunResult run_overlap(const ModelWeights& w, const std::vector<std::vector<int>>& prompts, const SpecConfig& decode,
                      const TierConfig& tier, uint64_t run_seed, bool trace) {
    return stepwise(w, prompts, decode, tier, run_seed, true, nullptr, trace);
}
RunResult run_caching(const ModelWeights& w, const std::vector<std::vector<int>>& prompts, const SpecConfig& decode,
                      const TierConfig& tier, const BaselineConfig& config, uint64_t run_seed, bool trace) {
    config.validate();
    std::vector<std::vector<int>> cached;
    uint64_t warm = 0;
    guard([&] {
        std::lock_guard<std::mutex> lk(g_mu);
        smoe::Engine& e = engine_for(w, (int)prompts.size(), decode.gamma, nullptr);
        smoe::RunCfg c = run_cfg(decode, DraftPolicy::hot_global, tier, run_seed, false);
        c.warmup_steps = config.warmup_steps;
        cached = smoe::caching_sets(e, c, prompts, config.cache_fraction, &warm);
        return 0;
    });
    RunResult r = stepwise(w, prompts, decode, tier, run_seed, false, &cached, trace);
    r.metrics.warmup_bytes = warm;
    return r;
}

}  // namespace specmoe
