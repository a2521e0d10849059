// harness.cpp -- experiment harness (reference harness.hpp:13-108, declared there but never defined;
// behaviour from SPEC.md:443-507): flat config parsing / serialisation, deterministic prompts,
// Cartesian sweeps over the B200 decode loop, CSV/JSON results, routing-trace I/O and analysis, and
// the selftest invariant suite.  Everything here is host C++; the cells run on the engine through
// the drop-in API (api.cpp).
#include "specmoe/harness.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <numeric>
#include <set>
#include <sstream>

namespace specmoe {

namespace {

// ------------------------------------------------------------------ value formatting / parsing
std::string fmt_double(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

std::string trim(const std::string& s) {
    size_t a = 0, b = s.size();
    while (a < b && std::isspace((unsigned char)s[a])) ++a;
    while (b > a && std::isspace((unsigned char)s[b - 1])) --b;
    return s.substr(a, b - a);
}

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == sep) {
            out.push_back(trim(cur));
            cur.clear();
        } else {
            cur.push_back(c);
        }
    }
    out.push_back(trim(cur));
    return out;
}

struct LineError {
    int line;
    std::string what;
};

long long parse_int(const std::string& v, int line) {
    if (v.empty()) throw LineError{line, "expected an integer"};
    size_t pos = 0;
    long long x = 0;
    try {
        x = std::stoll(v, &pos, 10);
    } catch (...) {
        throw LineError{line, "expected an integer, got '" + v + "'"};
    }
    if (pos != v.size()) throw LineError{line, "expected an integer, got '" + v + "'"};
    return x;
}

uint64_t parse_u64(const std::string& v, int line) {
    if (v.empty() || v[0] == '-') throw LineError{line, "expected a non-negative integer, got '" + v + "'"};
    size_t pos = 0;
    unsigned long long x = 0;
    try {
        x = std::stoull(v, &pos, 0);
    } catch (...) {
        throw LineError{line, "expected a non-negative integer, got '" + v + "'"};
    }
    if (pos != v.size()) throw LineError{line, "expected a non-negative integer, got '" + v + "'"};
    return x;
}

double parse_double(const std::string& v, int line) {
    if (v.empty()) throw LineError{line, "expected a number"};
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (end != v.c_str() + v.size() || !std::isfinite(x)) throw LineError{line, "expected a number, got '" + v + "'"};
    return x;
}

bool parse_bool(const std::string& v, int line) {
    if (v == "true" || v == "1" || v == "yes" || v == "on") return true;
    if (v == "false" || v == "0" || v == "no" || v == "off") return false;
    throw LineError{line, "expected a boolean, got '" + v + "'"};
}

// comma list of integers; each item may be a range a..b (inclusive)
template <typename T, typename F>
std::vector<T> parse_int_list(const std::string& v, int line, F one) {
    std::vector<T> out;
    for (const std::string& item : split(v, ',')) {
        const size_t dots = item.find("..");
        if (dots == std::string::npos) {
            out.push_back((T)one(item, line));
        } else {
            const long long a = (long long)one(trim(item.substr(0, dots)), line);
            const long long b = (long long)one(trim(item.substr(dots + 2)), line);
            if (b < a) throw LineError{line, "empty range '" + item + "'"};
            if (b - a > 1000000) throw LineError{line, "range too long '" + item + "'"};
            for (long long x = a; x <= b; ++x) out.push_back((T)x);
        }
    }
    return out;
}

template <typename T>
std::string join(const std::vector<T>& v, std::function<std::string(const T&)> f) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + f(v[i]);
    return s;
}

const char* engine_names[] = {"specmoe", "ondemand", "overlap", "caching"};

bool valid_engine(const std::string& e) {
    for (const char* n : engine_names)
        if (e == n) return true;
    return false;
}

// per-cell tier: derived bytes per expert / capacity when left at 0 (capacity for every expert of
// the model: a verify phase's coalesced fetch can touch all M*E keys at once)
TierConfig cell_tier(const ExperimentConfig& c, int n_draft, double bandwidth) {
    (void)n_draft;
    TierConfig t = c.tier;
    t.host_bandwidth = bandwidth;
    if (t.bytes_per_expert == 0) t.bytes_per_expert = bytes_per_expert(c.model);
    if (t.device_capacity_bytes == 0)
        t.device_capacity_bytes =
            (uint64_t)c.model.moe_layer_count() * (uint64_t)c.model.experts_per_block * t.bytes_per_expert;
    return t;
}

}  // namespace

// ================================================================== config
ExperimentConfig default_config() {
    ExperimentConfig c;  // SPEC.md:464 defaults: gamma 10, N 4, K 2, cache_fraction 0.10, host 64e9
    c.seeds.resize(20);
    std::iota(c.seeds.begin(), c.seeds.end(), 0);
    c.batch_list = {c.spec.batch};
    c.gamma_list = {c.spec.gamma};
    c.n_draft_list = {c.spec.n_draft};
    c.bandwidth_list = {c.tier.host_bandwidth};
    return c;
}

void ExperimentConfig::validate() const {
    model.validate();
    if (!valid_engine(engine)) throw ConfigError("config: engine must be specmoe|ondemand|overlap|caching");
    if (seeds.empty()) throw ConfigError("config: seeds must be non-empty");
    if (batch_list.empty() || gamma_list.empty() || n_draft_list.empty() || bandwidth_list.empty())
        throw ConfigError("config: sweep axes must be non-empty");
    const int M = model.moe_layer_count();
    for (int b : batch_list)
        for (int g : gamma_list)
            for (int n : n_draft_list)
                for (double bw : bandwidth_list) {
                    SpecConfig s = spec;
                    s.batch = b;
                    s.gamma = g;
                    s.n_draft = n;
                    s.validate();
                    if (n < model.top_k) throw ConfigError("config: n_draft >= top_k violated");
                    if (n > model.experts_per_block) throw ConfigError("config: n_draft <= experts violated");
                    cell_tier(*this, n, bw).validate(engine == "specmoe" ? n : 0, M);
                }
    if (engine != "specmoe") {
        BaselineConfig bc = baseline;
        bc.kind = engine == "ondemand" ? BaselineKind::ondemand
                  : engine == "overlap" ? BaselineKind::overlap
                                        : BaselineKind::caching;
        bc.validate();
    }
    const size_t cells = batch_list.size() * gamma_list.size() * n_draft_list.size() * bandwidth_list.size() *
                         seeds.size();
    if (!trace_out.empty() && cells != 1) throw ConfigError("config: trace_out needs a single-cell sweep");
}

ExperimentConfig parse_config_text(const std::string& text) {
    ExperimentConfig c = default_config();
    std::set<std::string> seen;
    bool batch_set = false, gamma_set = false, n_set = false, bw_set = false;
    std::istringstream in(text);
    std::string raw;
    int line = 0;
    try {
        while (std::getline(in, raw)) {
            ++line;
            const size_t hash = raw.find('#');
            const std::string s = trim(hash == std::string::npos ? raw : raw.substr(0, hash));
            if (s.empty()) continue;
            const size_t eq = s.find('=');
            if (eq == std::string::npos) throw LineError{line, "expected 'key = value'"};
            const std::string key = trim(s.substr(0, eq)), v = trim(s.substr(eq + 1));
            if (key.empty()) throw LineError{line, "missing key"};
            if (!seen.insert(key).second) throw LineError{line, "duplicate key '" + key + "'"};
            auto need = [&] {
                if (v.empty()) throw LineError{line, "missing value for '" + key + "'"};
            };
            // ---- model
            if (key == "num_layers") c.model.num_layers = (int)parse_int(v, line);
            else if (key == "moe_layer_mask") {
                c.model.moe_layer_mask.clear();
                for (char ch : v) {
                    if (ch == ',' || std::isspace((unsigned char)ch)) continue;
                    if (ch != '0' && ch != '1') throw LineError{line, "moe_layer_mask takes 0/1 digits"};
                    c.model.moe_layer_mask.push_back((uint8_t)(ch - '0'));
                }
            } else if (key == "experts") c.model.experts_per_block = (int)parse_int(v, line);
            else if (key == "top_k") c.model.top_k = (int)parse_int(v, line);
            else if (key == "hidden_dim") c.model.hidden_dim = (int)parse_int(v, line);
            else if (key == "ffn_dim") c.model.ffn_dim = (int)parse_int(v, line);
            else if (key == "vocab_size") c.model.vocab_size = (int)parse_int(v, line);
            else if (key == "gate_skew") c.model.gate_skew = parse_double(v, line);
            else if (key == "model_seed") c.model.seed = parse_u64(v, line);
            // ---- tier
            else if (key == "device_capacity_bytes") c.tier.device_capacity_bytes = parse_u64(v, line);
            else if (key == "host_bandwidth") {
                need();
                c.bandwidth_list.clear();
                for (const std::string& x : split(v, ',')) c.bandwidth_list.push_back(parse_double(x, line));
                c.tier.host_bandwidth = c.bandwidth_list[0];
                bw_set = true;
            } else if (key == "ssd_bandwidth") c.tier.ssd_bandwidth = parse_double(v, line);
            else if (key == "bytes_per_expert") c.tier.bytes_per_expert = parse_u64(v, line);
            else if (key == "compute_rate") c.tier.compute_rate_tokens_per_s = parse_double(v, line);
            else if (key == "compute_cost_per_expert") c.tier.compute_cost_per_active_expert_s = parse_double(v, line);
            // ---- decode
            else if (key == "batch") {
                need();
                c.batch_list = parse_int_list<int>(v, line, parse_int);
                c.spec.batch = c.batch_list[0];
                batch_set = true;
            } else if (key == "gamma") {
                need();
                c.gamma_list = parse_int_list<int>(v, line, parse_int);
                c.spec.gamma = c.gamma_list[0];
                gamma_set = true;
            } else if (key == "n_draft") {
                need();
                c.n_draft_list = parse_int_list<int>(v, line, parse_int);
                c.spec.n_draft = c.n_draft_list[0];
                n_set = true;
            } else if (key == "mode") {
                if (v == "greedy") c.spec.mode = DecodeMode::greedy;
                else if (v == "sampling") c.spec.mode = DecodeMode::sampling;
                else throw LineError{line, "mode must be greedy|sampling"};
            } else if (key == "temperature") c.spec.temperature = parse_double(v, line);
            else if (key == "max_new_tokens") c.spec.max_new_tokens = (int)parse_int(v, line);
            else if (key == "prompt_len") c.spec.prompt_len = (int)parse_int(v, line);
            else if (key == "use_affinity") c.spec.use_affinity = parse_bool(v, line);
            else if (key == "warmup_steps") c.spec.warmup_steps = (int)parse_int(v, line);
            // ---- engine
            else if (key == "engine") {
                if (!valid_engine(v)) throw LineError{line, "engine must be specmoe|ondemand|overlap|caching"};
                c.engine = v;
            } else if (key == "policy") {
                try {
                    c.policy = draft_policy_from_string(v);
                } catch (const ConfigError&) {
                    throw LineError{line, "policy must be random|hot_global|hot_temporal"};
                }
            } else if (key == "cache_fraction") c.baseline.cache_fraction = parse_double(v, line);
            else if (key == "baseline_warmup_steps") c.baseline.warmup_steps = (int)parse_int(v, line);
            // ---- run
            else if (key == "seeds") {
                need();
                c.seeds = parse_int_list<uint64_t>(v, line, parse_u64);
            } else if (key == "trace_out") c.trace_out = v;
            else if (key == "verbose") c.verbose = parse_bool(v, line);
            else throw LineError{line, "unknown key '" + key + "'"};
        }
    } catch (const LineError& e) {
        throw ConfigError("config line " + std::to_string(e.line) + ": " + e.what);
    }
    if (!batch_set) c.batch_list = {c.spec.batch};
    if (!gamma_set) c.gamma_list = {c.spec.gamma};
    if (!n_set) c.n_draft_list = {c.spec.n_draft};
    if (!bw_set) c.bandwidth_list = {c.tier.host_bandwidth};
    c.validate();
    return c;
}

ExperimentConfig parse_config(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw ConfigError("config: cannot open " + path);
    std::stringstream ss;
    ss << f.rdbuf();
    return parse_config_text(ss.str());
}

std::string serialize_config(const ExperimentConfig& c) {
    std::ostringstream o;
    auto I = [](const int& x) { return std::to_string(x); };
    auto U = [](const uint64_t& x) { return std::to_string(x); };
    auto D = [](const double& x) { return fmt_double(x); };
    o << "# specmoe-config v1\n";
    o << "num_layers = " << c.model.num_layers << "\n";
    o << "moe_layer_mask = ";
    for (uint8_t m : c.model.moe_layer_mask) o << (m ? '1' : '0');
    o << "\n";
    o << "experts = " << c.model.experts_per_block << "\n";
    o << "top_k = " << c.model.top_k << "\n";
    o << "hidden_dim = " << c.model.hidden_dim << "\n";
    o << "ffn_dim = " << c.model.ffn_dim << "\n";
    o << "vocab_size = " << c.model.vocab_size << "\n";
    o << "gate_skew = " << fmt_double(c.model.gate_skew) << "\n";
    o << "model_seed = " << c.model.seed << "\n";
    o << "device_capacity_bytes = " << c.tier.device_capacity_bytes << "\n";
    o << "host_bandwidth = " << join<double>(c.bandwidth_list, D) << "\n";
    o << "ssd_bandwidth = " << fmt_double(c.tier.ssd_bandwidth) << "\n";
    o << "bytes_per_expert = " << c.tier.bytes_per_expert << "\n";
    o << "compute_rate = " << fmt_double(c.tier.compute_rate_tokens_per_s) << "\n";
    o << "compute_cost_per_expert = " << fmt_double(c.tier.compute_cost_per_active_expert_s) << "\n";
    o << "batch = " << join<int>(c.batch_list, I) << "\n";
    o << "gamma = " << join<int>(c.gamma_list, I) << "\n";
    o << "n_draft = " << join<int>(c.n_draft_list, I) << "\n";
    o << "mode = " << to_string(c.spec.mode) << "\n";
    o << "temperature = " << fmt_double(c.spec.temperature) << "\n";
    o << "max_new_tokens = " << c.spec.max_new_tokens << "\n";
    o << "prompt_len = " << c.spec.prompt_len << "\n";
    o << "use_affinity = " << (c.spec.use_affinity ? "true" : "false") << "\n";
    o << "warmup_steps = " << c.spec.warmup_steps << "\n";
    o << "engine = " << c.engine << "\n";
    o << "policy = " << to_string(c.policy) << "\n";
    o << "cache_fraction = " << fmt_double(c.baseline.cache_fraction) << "\n";
    o << "baseline_warmup_steps = " << c.baseline.warmup_steps << "\n";
    o << "seeds = " << join<uint64_t>(c.seeds, U) << "\n";
    if (!c.trace_out.empty()) o << "trace_out = " << c.trace_out << "\n";
    o << "verbose = " << (c.verbose ? "true" : "false") << "\n";
    return o.str();
}

// ================================================================== prompts
std::vector<std::vector<int>> make_prompts(uint64_t seed, int batch, int prompt_len, int vocab) {
    if (batch < 0 || prompt_len < 1 || vocab < 1) throw ConfigError("make_prompts: bad shape");
    constexpr uint64_t kPromptTag = 0x70726f6dull;  // "prom"
    std::vector<std::vector<int>> out((size_t)batch);
    for (int b = 0; b < batch; ++b) {
        Rng rng(substream(seed, kPromptTag, (uint64_t)b));
        out[b].resize((size_t)prompt_len);
        for (int i = 0; i < prompt_len; ++i)
            out[b][i] = std::min(vocab - 1, (int)(uniform01(rng) * (double)vocab));
    }
    return out;
}

// ================================================================== sweep
std::vector<ResultRow> run_experiment(const ExperimentConfig& config) {
    config.validate();
    const ModelWeights weights = build_model(config.model);
    const bool spec = config.engine == "specmoe";
    AffinityTable affinity;
    const bool need_aff = spec && config.spec.use_affinity;
    if (need_aff) affinity = build_affinity_table(weights);
    std::vector<ResultRow> rows;
    for (double bw : config.bandwidth_list)
        for (int b : config.batch_list)
            for (int g : config.gamma_list)
                for (int n : config.n_draft_list)
                    for (uint64_t seed : config.seeds) {
                        SpecConfig sc = config.spec;
                        sc.batch = b;
                        sc.gamma = g;
                        sc.n_draft = n;
                        const TierConfig tier = cell_tier(config, n, bw);
                        const auto prompts = make_prompts(seed, b, sc.prompt_len, config.model.vocab_size);
                        const bool trace = !config.trace_out.empty();
                        const auto t0 = std::chrono::steady_clock::now();
                        RunResult r;
                        const std::string cell = "cell (bandwidth=" + fmt_double(bw) + ", batch=" +
                                                 std::to_string(b) + ", gamma=" + std::to_string(g) +
                                                 ", n_draft=" + std::to_string(n) + ", seed=" +
                                                 std::to_string(seed) + "): ";
                        try {
                            if (spec) {
                                r = run_specmoe(weights, sc, config.policy, tier, prompts, seed,
                                                need_aff ? &affinity : nullptr, trace);
                            } else if (config.engine == "ondemand") {
                                r = run_ondemand(weights, prompts, sc, tier, seed, trace);
                            } else if (config.engine == "overlap") {
                                r = run_overlap(weights, prompts, sc, tier, seed, trace);
                            } else {
                                BaselineConfig bc = config.baseline;
                                bc.kind = BaselineKind::caching;
                                r = run_caching(weights, prompts, sc, tier, bc, seed, trace);
                            }
                        } catch (const ConfigError& e) {
                            throw ConfigError(cell + e.what());
                        } catch (const InvariantError& e) {
                            throw InvariantError(cell + e.what());
                        }
                        const double wall =
                            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                        ResultRow row;
                        row.policy = spec ? to_string(config.policy) : config.engine;
                        row.batch = b;
                        row.gamma = g;
                        row.n_draft = n;
                        row.bandwidth = bw;
                        row.seed = seed;
                        row.tau = r.metrics.tau_mean;
                        row.tokens_per_sec = r.metrics.tokens_per_sec;
                        row.bytes_total = r.metrics.bytes_total;
                        row.bytes_spec = r.metrics.bytes_spec;
                        row.bytes_verify = r.metrics.bytes_verify;
                        row.lambda = r.metrics.lambda;
                        const double tau = std::clamp(row.tau, 1.0, (double)g + 1.0);
                        const double c = std::max(0.0, r.metrics.c_measured);
                        row.s_eq1 = speedup_eq1(tau, g, c);
                        row.s_eq2 = speedup_eq2(tau, g, c, row.lambda > 0.0 ? row.lambda : 1.0);
                        uint64_t h = 0xcbf29ce484222325ull;
                        for (const auto& seq : r.tokens) h = fnv1a64(seq.data(), seq.size() * sizeof(int), h);
                        row.text_hash = h;
                        row.sim_wall_s = wall;
                        rows.push_back(row);
                        if (trace) {
                            TraceFile tf;
                            tf.moe_layers = config.model.moe_layer_count();
                            tf.experts = config.model.experts_per_block;
                            tf.top_k = config.model.top_k;
                            tf.rows = r.trace;
                            write_trace(tf, config.trace_out);
                        }
                    }
    return rows;
}

// ================================================================== results
void emit_results(std::span<const ResultRow> rows, const std::string& format, std::ostream& out, bool verbose) {
    if (rows.empty()) throw ConfigError("emit_results: no rows");
    if (format != "csv" && format != "json") throw ConfigError("emit_results: format must be csv|json");
    if (format == "csv") {
        out << "policy,batch,gamma,n_draft,bandwidth,seed,tau,tokens_per_sec,bytes_total,bytes_spec,bytes_verify,"
               "lambda,s_eq1,s_eq2"
            << (verbose ? ",text_hash" : "") << "\n";
        for (const ResultRow& r : rows) {
            out << r.policy << ',' << r.batch << ',' << r.gamma << ',' << r.n_draft << ',' << fmt_double(r.bandwidth)
                << ',' << r.seed << ',' << fmt_double(r.tau) << ',' << fmt_double(r.tokens_per_sec) << ','
                << r.bytes_total << ',' << r.bytes_spec << ',' << r.bytes_verify << ',' << fmt_double(r.lambda) << ','
                << fmt_double(r.s_eq1) << ',' << fmt_double(r.s_eq2);
            if (verbose) out << ',' << r.text_hash;
            out << "\n";
        }
    } else {
        out << "[\n";
        for (size_t i = 0; i < rows.size(); ++i) {
            const ResultRow& r = rows[i];
            out << "  {\"policy\": \"" << r.policy << "\", \"batch\": " << r.batch << ", \"gamma\": " << r.gamma
                << ", \"n_draft\": " << r.n_draft << ", \"bandwidth\": " << fmt_double(r.bandwidth)
                << ", \"seed\": " << r.seed << ", \"tau\": " << fmt_double(r.tau)
                << ", \"tokens_per_sec\": " << fmt_double(r.tokens_per_sec) << ", \"bytes_total\": " << r.bytes_total
                << ", \"bytes_spec\": " << r.bytes_spec << ", \"bytes_verify\": " << r.bytes_verify
                << ", \"lambda\": " << fmt_double(r.lambda) << ", \"s_eq1\": " << fmt_double(r.s_eq1)
                << ", \"s_eq2\": " << fmt_double(r.s_eq2);
            if (verbose) out << ", \"text_hash\": " << r.text_hash;
            out << "}" << (i + 1 < rows.size() ? "," : "") << "\n";
        }
        out << "]\n";
    }
    if (!out) throw InvariantError("emit_results: I/O failure");
}

void emit_results(std::span<const ResultRow> rows, const std::string& format, const std::string& path, bool verbose) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw ConfigError("emit_results: cannot open " + path);
    emit_results(rows, format, f, verbose);
}

// ================================================================== traces
void write_trace(const TraceFile& t, std::ostream& out) {
    out << "# specmoe-trace v1 layers=" << t.moe_layers << " experts=" << t.experts << " top_k=" << t.top_k << "\n";
    out << "step,seq,layer,experts\n";
    for (const TraceRow& r : t.rows) {
        out << r.step << ',' << r.seq << ',' << r.layer;
        for (int e : r.experts) out << ',' << e;
        out << "\n";
    }
    if (!out) throw InvariantError("write_trace: I/O failure");
}

void write_trace(const TraceFile& t, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw ConfigError("write_trace: cannot open " + path);
    write_trace(t, f);
}

TraceFile read_trace(std::istream& in) {
    TraceFile t;
    std::string line;
    int ln = 0;
    auto bad = [&](const std::string& m) { return ConfigError("trace line " + std::to_string(ln) + ": " + m); };
    if (!std::getline(in, line)) throw ConfigError("trace: empty file");
    ++ln;
    if (std::sscanf(line.c_str(), "# specmoe-trace v1 layers=%d experts=%d top_k=%d", &t.moe_layers, &t.experts,
                    &t.top_k) != 3)
        throw bad("expected '# specmoe-trace v1 layers=<M> experts=<E> top_k=<K>'");
    if (t.moe_layers < 1 || t.experts < 1 || t.top_k < 1 || t.top_k > t.experts) throw bad("bad header values");
    if (!std::getline(in, line)) throw ConfigError("trace: missing column header");
    ++ln;
    if (trim(line) != "step,seq,layer,experts") throw bad("expected column header 'step,seq,layer,experts'");
    while (std::getline(in, line)) {
        ++ln;
        if (trim(line).empty()) continue;
        const auto f = split(line, ',');
        if ((int)f.size() != 3 + t.top_k) throw bad("expected " + std::to_string(3 + t.top_k) + " fields");
        TraceRow r;
        try {
            r.step = (int)parse_int(f[0], ln);
            r.seq = (int)parse_int(f[1], ln);
            r.layer = (int)parse_int(f[2], ln);
            for (int k = 0; k < t.top_k; ++k) r.experts.push_back((int)parse_int(f[3 + k], ln));
        } catch (const LineError& e) {
            throw bad(e.what);
        }
        if (r.step < 0 || r.seq < 0) throw bad("negative step / seq");
        if (r.layer < 0 || r.layer >= t.moe_layers) throw bad("layer out of range");
        for (int e : r.experts)
            if (e < 0 || e >= t.experts) throw bad("expert index out of range");
        t.rows.push_back(std::move(r));
    }
    return t;
}

TraceFile read_trace(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw ConfigError("read_trace: cannot open " + path);
    return read_trace(f);
}

// Each routed position contributes one row per MoE layer: counts as record_activations
// (reference drafting.cpp:158-171) would, one routed token per layer-0 row.
HotnessCounter ingest_trace(const TraceFile& t) {
    HotnessCounter h(t.moe_layers, t.experts);
    for (const TraceRow& r : t.rows) {
        if (r.layer < 0 || r.layer >= t.moe_layers) throw InvariantError("ingest_trace: layer out of range");
        for (int e : r.experts) {
            if (e < 0 || e >= t.experts) throw InvariantError("ingest_trace: expert index out of range");
            ++h.counts[r.layer][e];
        }
        if (r.layer == 0) ++h.routed_tokens;
    }
    return h;
}

HotnessCounter ingest_trace(const std::string& path) { return ingest_trace(read_trace(path)); }

TraceReport analyze_trace(const HotnessCounter& counter, int top_n) {
    TraceReport rep;
    rep.skewness = skewness(counter);
    rep.routed_tokens = counter.routed_tokens;
    rep.frequencies = counter.counts;
    for (const auto& counts : counter.counts) {
        std::vector<int> idx(counts.size());
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return counts[a] > counts[b]; });
        idx.resize(std::min<size_t>(idx.size(), (size_t)std::max(0, top_n)));
        rep.hottest.push_back(std::move(idx));
    }
    return rep;
}

void write_trace_report(const TraceReport& rep, std::ostream& out) {
    out << "layer,expert,count,fraction\n";
    for (size_t l = 0; l < rep.frequencies.size(); ++l) {
        const auto& c = rep.frequencies[l];
        const uint64_t tot = std::accumulate(c.begin(), c.end(), uint64_t{0});
        for (size_t e = 0; e < c.size(); ++e)
            out << l << ',' << e << ',' << c[e] << ',' << fmt_double(tot ? (double)c[e] / (double)tot : 0.0) << "\n";
    }
    if (!out) throw InvariantError("write_trace_report: I/O failure");
}

void write_trace_report(const TraceReport& rep, const std::string& path) {
    std::ofstream f(path, std::ios::binary);
    if (!f) throw ConfigError("write_trace_report: cannot open " + path);
    write_trace_report(rep, f);
}

// ================================================================== selftest
bool selftest(std::ostream& out) {
    int failed = 0;
    auto check = [&](const char* name, const std::function<bool(std::string&)>& fn) {
        std::string why;
        bool ok = false;
        try {
            ok = fn(why);
        } catch (const std::exception& e) {
            why = std::string("exception: ") + e.what();
        }
        out << (ok ? "ok   " : "FAIL ") << name << (ok || why.empty() ? "" : ": " + why) << "\n";
        failed += !ok;
    };
    auto near = [](double a, double b, double tol) { return std::fabs(a - b) <= tol; };
    // ---- model primitives
    check("softmax KATs", [&](std::string&) {
        const std::vector<double> a{0.0, 0.0}, b{std::log(2.0), 0.0}, c{1000.0, 0.0};
        const auto pa = softmax(a), pb = softmax(b), pc = softmax(c);
        return near(pa[0], 0.5, 1e-15) && near(pb[0], 2.0 / 3.0, 1e-12) && near(pb[1], 1.0 / 3.0, 1e-12) &&
               near(pc[0], 1.0, 1e-12) && near(pc[1], 0.0, 1e-12);
    });
    check("route_topk KATs", [&](std::string&) {
        const std::vector<double> a{3, 1, 2}, b{5, 5, 1};
        const auto ra = route_topk(a, 2), rb = route_topk(b, 1), rc = route_topk(a, 3);
        return ra == std::vector<int>{0, 2} && rb == std::vector<int>{0} && rc == std::vector<int>{0, 2, 1};
    });
    check("route_topk K > E rejected", [&](std::string&) {
        try {
            const std::vector<double> a{1, 2};
            route_topk(a, 3);
        } catch (const ConfigError&) {
            return true;
        } catch (const InvariantError&) {
            return true;
        }
        return false;
    });
    check("greedy_next KATs", [&](std::string&) {
        const std::vector<double> a{0.1, 0.9}, b{0.5, 0.5};
        bool ok = greedy_next(a) == 1 && greedy_next(b) == 0;
        for (int i = 0; i < 16; ++i) {
            std::vector<double> oh(16, 0.0);
            oh[i] = 1.0;
            ok &= greedy_next(oh) == i;
        }
        return ok;
    });
    // ---- store
    check("ensure_resident 3 keys d32 f64 -> 49152 B", [&](std::string& why) {
        ModelSpec ms;
        ms.num_layers = 2;
        ms.experts_per_block = 4;
        ms.top_k = 1;
        ms.hidden_dim = 32;
        ms.ffn_dim = 64;
        TierConfig t;
        t.bytes_per_expert = bytes_per_expert(ms);
        t.device_capacity_bytes = 8 * t.bytes_per_expert;
        ResidencyState rs(ms, t);
        MigrationLedger led;
        const std::set<ExpertKey> keys{{0, 1}, {0, 3}, {1, 2}};
        const uint64_t b1 = ensure_resident(keys, Phase::verification, 0, led, rs);
        const uint64_t b2 = ensure_resident(keys, Phase::verification, 0, led, rs);
        why = std::to_string(b1) + " / " + std::to_string(b2);
        return b1 == 49152 && b2 == 0 && led.migration_count() == 3;
    });
    check("pin: initial N*layers*bpe, re-pin 0", [&](std::string& why) {
        ModelSpec ms;
        ms.num_layers = 3;
        ms.experts_per_block = 8;
        ms.top_k = 2;
        TierConfig t;
        t.bytes_per_expert = bytes_per_expert(ms);
        t.device_capacity_bytes = 64 * t.bytes_per_expert;
        ResidencyState rs(ms, t);
        MigrationLedger led;
        const std::vector<std::vector<int>> sets{{0, 1}, {2, 3}, {4, 5}};
        const uint64_t a = pin_draft_experts(sets, rs, led, Phase::verification, 0);
        const uint64_t b = pin_draft_experts(sets, rs, led, Phase::verification, 1);
        why = std::to_string(a) + " / " + std::to_string(b);
        return a == 6 * t.bytes_per_expert && b == 0 && rs.pinned_set().size() == 6;
    });
    // ---- drafting
    check("nearest_draft_expert stub (raw 1, set {0,2} -> 2)", [&](std::string&) {
        AffinityTable at;
        at.experts = 3;
        at.dist = {{0.0, 5.0, 1.0, 5.0, 0.0, std::sqrt(18.0), 1.0, std::sqrt(18.0), 0.0}};
        const std::vector<int> set{0, 2}, none, self{1, 2}, one{0};
        return nearest_draft_expert(at, 0, 1, set, none) == 2 && nearest_draft_expert(at, 0, 1, self, none) == 1 &&
               nearest_draft_expert(at, 0, 2, one, none) == 0;
    });
    check("record_activations picks [3,5]", [&](std::string&) {
        HotnessCounter h(1, 8);
        ActivationRecord rec;
        rec.rows.push_back(ActivationRow{LayerActivation{{3, 5}, {3, 5}}});
        record_activations(h, rec);
        return h.counts[0][3] == 1 && h.counts[0][5] == 1 && h.routed_tokens == 1;
    });
    check("select_draft_experts counts [5,3,9,1] N=2 -> {2,0}", [&](std::string&) {
        HotnessCounter h(1, 4);
        h.counts[0] = {5, 3, 9, 1};
        h.routed_tokens = 9;
        DraftState cur;
        cur.n_draft = 2;
        cur.sets = {{1, 3}};
        Rng rng(0);
        const auto s = select_draft_experts(DraftPolicy::hot_temporal, h, cur, 4, rng);
        HotnessCounter z(1, 4);
        const auto s0 = select_draft_experts(DraftPolicy::hot_temporal, z, cur, 4, rng);
        std::vector<int> a = s[0], b = s0[0];
        std::sort(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        return a == std::vector<int>{0, 2} && b == std::vector<int>{1, 3};
    });
    check("skewness uniform 0.25 / one-hot 1.0 / [7,1,1,1] 0.70", [&](std::string& why) {
        HotnessCounter u(2, 8), o(2, 8), h(1, 4);
        for (int l = 0; l < 2; ++l)
            for (int e = 0; e < 8; ++e) u.counts[l][e] = 100;
        u.routed_tokens = 400;
        o.counts[0][3] = 50;
        o.counts[1][0] = 50;
        o.routed_tokens = 50;
        h.counts[0] = {7, 1, 1, 1};
        h.routed_tokens = 10;
        const double su = skewness(u), so = skewness(o), sh = skewness(h);
        why = fmt_double(su) + " " + fmt_double(so) + " " + fmt_double(sh);
        return near(su, 0.25, 1e-12) && so == 1.0 && near(sh, 0.70, 1e-15);
    });
    // ---- specdec math
    check("speedup eq1/eq2 KATs", [&](std::string&) {
        return near(speedup_eq1(11.0, 10, 0.0), 11.0, 1e-12) && near(speedup_eq2(1.0, 10, 0.0, 1.0), 1.0, 1e-12) &&
               near(speedup_eq2(7.265, 10, 0.05, 2.0), 2.906, 1e-12);
    });
    // ---- harness formats
    check("config defaults, round trip, gamma=0 rejected", [&](std::string& why) {
        const ExperimentConfig d = parse_config_text("");
        const ExperimentConfig c = parse_config_text("experts = 16\ntop_k = 2\nn_draft = 4\nbatch = 1, 8\n");
        const std::string s1 = serialize_config(c), s2 = serialize_config(parse_config_text(s1));
        bool rejected = false;
        try {
            parse_config_text("gamma = 0\n");
        } catch (const ConfigError& e) {
            rejected = std::string(e.what()).find("gamma") != std::string::npos;
            why = e.what();
        }
        return d.spec.gamma == 10 && d.spec.n_draft == 4 && d.model.top_k == 2 && d.seeds.size() == 20 &&
               s1 == s2 && rejected;
    });
    check("make_prompts batch transparency", [&](std::string&) {
        const auto a = make_prompts(7, 1, 8, 1000), b = make_prompts(7, 8, 8, 1000);
        return a[0] == b[0] && b[1] != b[0];
    });
    check("trace round trip + analysis", [&](std::string&) {
        TraceFile t;
        t.moe_layers = 2;
        t.experts = 4;
        t.top_k = 2;
        for (int s = 0; s < 3; ++s)
            for (int l = 0; l < 2; ++l) t.rows.push_back(TraceRow{s, 0, l, {l, 3}});
        std::stringstream ss;
        write_trace(t, ss);
        const TraceFile r = read_trace(ss);
        const HotnessCounter h = ingest_trace(r);
        const TraceReport rep = analyze_trace(h, 2);
        return r.rows.size() == 6 && h.routed_tokens == 3 && h.counts[1][1] == 3 && h.counts[0][3] == 3 &&
               rep.hottest[0] == std::vector<int>{0, 3} && near(rep.skewness, 0.5, 1e-15);
    });
    // ---- engine checks (SPEC.md:512-516 acceptance 1, 2, 4), only with a CUDA device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        out << "skip engine checks (no CUDA device)\n";
    } else {
        ModelSpec ms;  // acceptance-1 toy model: L4 E16 K2 d32 f64 V64
        const ModelWeights w = build_model(ms);
        const AffinityTable aff = build_affinity_table(w);
        TierConfig tier;
        tier.bytes_per_expert = bytes_per_expert(ms);
        tier.device_capacity_bytes = (uint64_t)(16 * 4 + 16) * tier.bytes_per_expert;
        check("forward: full draft set == unrestricted", [&](std::string&) {
            RestrictedExperts all;
            for (int l = 0; l < ms.moe_layer_count(); ++l) {
                all.per_layer.emplace_back(16);
                std::iota(all.per_layer.back().begin(), all.per_layer.back().end(), 0);
            }
            const std::vector<int> prefix{2, 7, 7};
            return forward(w, prefix, nullptr, nullptr).logits == forward(w, prefix, &all, &aff).logits;
        });
        check("lossless: specmoe == ondemand (N 2/4/8/16, gamma 5/10, 4 seeds)", [&](std::string& why) {
            for (int n : {2, 4, 8, 16})
                for (int g : {5, 10})
                    for (uint64_t seed = 0; seed < 4; ++seed) {
                        SpecConfig sc;
                        sc.gamma = g;
                        sc.n_draft = n;
                        sc.batch = 2;
                        const auto prompts = make_prompts(seed, 2, sc.prompt_len, ms.vocab_size);
                        const RunResult a = run_specmoe(w, sc, DraftPolicy::hot_temporal, tier, prompts, seed, &aff);
                        const RunResult b = run_ondemand(w, prompts, sc, tier, seed);
                        if (a.tokens != b.tokens) {
                            why = "N=" + std::to_string(n) + " gamma=" + std::to_string(g) + " seed=" +
                                  std::to_string(seed);
                            return false;
                        }
                        if (a.metrics.bytes_spec != 0) {
                            why = "speculation bytes != 0";
                            return false;
                        }
                    }
            return true;
        });
        check("identity limit: N=E -> tau = gamma+1", [&](std::string& why) {
            SpecConfig sc;
            sc.gamma = 5;
            sc.n_draft = 16;
            sc.max_new_tokens = 30;
            const auto prompts = make_prompts(3, 1, sc.prompt_len, ms.vocab_size);
            const RunResult a = run_specmoe(w, sc, DraftPolicy::hot_temporal, tier, prompts, 3, &aff);
            why = "tau " + fmt_double(a.metrics.tau_mean);
            return a.metrics.tau_mean == 6.0;
        });
    }
    out << (failed ? "selftest: FAILED " + std::to_string(failed) + " check(s)\n" : "selftest: all checks passed\n");
    return failed == 0;
}

}  // namespace specmoe
