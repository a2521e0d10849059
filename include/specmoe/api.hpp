// specmoe/api.hpp -- C++ drop-in for the reference's model/decoder API (/root/reference/proj/core,
// namespace specmoe), implemented on the B200 engine (libspecmoe_b200.so).
//
// Every declaration keeps the reference's name, signature, value types and error behaviour
// (ConfigError / InvariantError), so a caller written against the reference headers recompiles
// against include/specmoe/ unchanged.  The per-module headers (common.hpp, model.hpp, drafting.hpp,
// memsim.hpp, specdec.hpp, baselines.hpp) just include this file.
//
// What runs where:
//   * forward / speculate / verify_greedy / verify_sampling (target logits) / run_specmoe /
//     run_ondemand / run_overlap / run_caching: the sm_100a engine.  Weights are uploaded once per
//     ModelWeights object (fp32 storage -> routing/tokens bit-exact with the reference; set
//     SPECMOE_B200_DTYPE=bf16 for the tcgen05 path), draft sets as device rank tables.
//   * build_model, affinity, policy, residency/ledger, cost model: host C++, same arithmetic order as
//     the reference (bit-identical results).
#pragma once

#include <compare>
#include <cstdint>
#include <iosfwd>
#include <map>
#include <random>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace specmoe {

// ============================================================== errors, RNG (reference common.hpp:12-73)
struct ConfigError : std::runtime_error {     // exit code 1
    using std::runtime_error::runtime_error;
};
struct InvariantError : std::runtime_error {  // exit code 2
    using std::runtime_error::runtime_error;
};

using Rng = std::mt19937_64;

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline uint64_t substream(uint64_t seed, uint64_t tag0, uint64_t tag1 = 0) {
    return splitmix64(seed ^ splitmix64(tag0 ^ splitmix64(tag1)));
}
inline double uniform01(Rng& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
double gaussian(Rng& rng);
uint64_t fnv1a64(const void* data, size_t len, uint64_t h = 0xcbf29ce484222325ull);
uint64_t hash_tokens(const std::vector<int>& tokens);

// ============================================================== model (reference model.hpp)
struct AffinityTable;

struct ModelSpec {
    int num_layers = 4;
    std::vector<uint8_t> moe_layer_mask;  // empty: every layer is an MoE block
    int experts_per_block = 16;
    int top_k = 2;
    int hidden_dim = 32;
    int ffn_dim = 64;
    int vocab_size = 64;
    double gate_skew = 0.0;
    uint64_t seed = 0;

    void validate() const;
    std::vector<uint8_t> effective_mask() const;
    int moe_layer_count() const;
    int moe_layer_index(int moe_ordinal) const;
};

struct ExpertWeights {
    std::vector<double> up;    // d x f
    std::vector<double> down;  // f x d
};

struct LayerWeights {
    bool is_moe = false;
    std::vector<double> mix;        // d x d
    std::vector<double> gate;       // d x E
    std::vector<double> gate_bias;  // E
    std::vector<ExpertWeights> experts;
    ExpertWeights ffn;
};

struct ModelWeights {
    ModelSpec spec;
    std::vector<double> embedding;  // V x d
    std::vector<LayerWeights> layers;
    std::vector<double> head;       // d x V
};

ModelWeights build_model(const ModelSpec& spec);
std::vector<double> softmax(std::span<const double> logits);
std::vector<int> route_topk(std::span<const double> gate_logits, int k);
int greedy_next(std::span<const double> logits);
int sample_next(std::span<const double> logits, double temperature, Rng& rng);

struct LayerActivation {
    std::vector<int> raw;
    std::vector<int> final;
};
using ActivationRow = std::vector<LayerActivation>;
struct ActivationRecord {
    std::vector<ActivationRow> rows;
};
struct TraceRow {
    int step = 0;
    int seq = 0;
    int layer = 0;
    std::vector<int> experts;
};
struct ForwardResult {
    std::vector<double> logits;
    ActivationRow activations;
};
struct RestrictedExperts {
    std::vector<std::vector<int>> per_layer;
};

ForwardResult forward(const ModelWeights& weights, std::span<const int> prefix,
                      const RestrictedExperts* restricted = nullptr, const AffinityTable* affinity = nullptr);

// ============================================================== drafting (reference drafting.hpp)
struct AffinityTable {
    int experts = 0;
    std::vector<std::vector<double>> dist;  // per MoE block, E*E
    double at(int layer, int i, int j) const { return dist[layer][static_cast<size_t>(i) * experts + j]; }
};

AffinityTable build_affinity_table(const ModelWeights& weights);
void save_affinity_csv(const AffinityTable& table, std::ostream& out);
void save_affinity_csv(const AffinityTable& table, const std::string& path);
AffinityTable load_affinity_csv(std::istream& in);
AffinityTable load_affinity_csv(const std::string& path);
int nearest_draft_expert(const AffinityTable& table, int layer, int raw_pick, std::span<const int> draft_set,
                         std::span<const int> excluded);
int surrogate_draft_expert(int layer, int raw_pick, size_t prefix_len, std::span<const int> draft_set,
                           std::span<const int> excluded);

enum class DraftPolicy { random, hot_global, hot_temporal };
const char* to_string(DraftPolicy policy);
DraftPolicy draft_policy_from_string(const std::string& name);

struct DraftState {
    DraftPolicy policy = DraftPolicy::hot_temporal;
    int n_draft = 4;
    std::vector<std::vector<int>> sets;
};

struct HotnessCounter {
    std::vector<std::vector<uint64_t>> counts;
    uint64_t routed_tokens = 0;
    HotnessCounter() = default;
    HotnessCounter(int moe_layers, int experts) : counts(moe_layers, std::vector<uint64_t>(experts, 0)) {}
    void reset();
};

void record_activations(HotnessCounter& counter, const ActivationRecord& record);
std::vector<std::vector<int>> select_draft_experts(DraftPolicy policy, const HotnessCounter& counter,
                                                   const DraftState& current, int experts_per_block, Rng& rng);
double skewness(const HotnessCounter& counter, double top_fraction = 0.25);

// ============================================================== memsim (reference memsim.hpp)
struct ExpertKey {
    int layer = 0;
    int expert = 0;
    auto operator<=>(const ExpertKey&) const = default;
};

enum class Phase { speculation, verification, baseline_step };
const char* to_string(Phase phase);

struct TierConfig {
    uint64_t device_capacity_bytes = 0;
    double host_bandwidth = 64e9;
    double ssd_bandwidth = 0.0;
    uint64_t bytes_per_expert = 0;
    double compute_rate_tokens_per_s = 1e6;
    double compute_cost_per_active_expert_s = 2e-6;
    double offload_bandwidth() const { return ssd_bandwidth > 0.0 ? ssd_bandwidth : host_bandwidth; }
    void validate(int n_draft, int moe_layers) const;
};

uint64_t bytes_per_expert(const ModelSpec& spec);

struct LedgerEntry {
    Phase phase;
    int step;
    ExpertKey key;
    uint64_t bytes;
};

class MigrationLedger {
public:
    struct Totals {
        uint64_t total = 0;
        uint64_t speculation = 0;
        uint64_t verification = 0;
        uint64_t baseline = 0;
        size_t migrations = 0;
    };
    void add(Phase phase, int step, ExpertKey key, uint64_t bytes);
    const std::vector<LedgerEntry>& entries() const { return entries_; }
    uint64_t total() const { return totals_.total; }
    uint64_t total(Phase phase) const;
    size_t migration_count() const { return entries_.size(); }
    Totals snapshot() const { return totals_; }
    void reset();
    void write_csv(std::ostream& out) const;

private:
    std::vector<LedgerEntry> entries_;
    Totals totals_;
};

class ResidencyState {
public:
    ResidencyState(const ModelSpec& spec, const TierConfig& tier);
    bool device_resident(ExpertKey key) const;
    bool pinned(ExpertKey key) const;
    uint64_t device_bytes_used() const { return device_bytes_; }
    const std::set<ExpertKey>& pinned_set() const { return pinned_; }
    size_t transient_count() const { return residents_.size() - pinned_.size(); }
    const TierConfig& tier() const { return tier_; }
    int moe_layers() const { return moe_layers_; }
    int experts_per_block() const { return experts_; }

private:
    friend uint64_t ensure_resident(const std::set<ExpertKey>&, Phase, int, MigrationLedger&, ResidencyState&);
    friend uint64_t pin_draft_experts(const std::vector<std::vector<int>>&, ResidencyState&, MigrationLedger&, Phase,
                                      int);
    friend void flush_transients(ResidencyState& residency);
    void check_key(ExpertKey key) const;
    void admit(ExpertKey key, const std::set<ExpertKey>& keep);

    TierConfig tier_;
    int moe_layers_;
    int experts_;
    std::map<ExpertKey, uint64_t> residents_;  // key -> arrival order
    std::set<ExpertKey> pinned_;
    uint64_t device_bytes_ = 0;
    uint64_t arrival_seq_ = 0;
};

uint64_t ensure_resident(const std::set<ExpertKey>& keys, Phase phase, int step, MigrationLedger& ledger,
                         ResidencyState& residency);
uint64_t pin_draft_experts(const std::vector<std::vector<int>>& per_layer_sets, ResidencyState& residency,
                           MigrationLedger& ledger, Phase phase, int step);
void flush_transients(ResidencyState& residency);

struct StepTiming {
    double compute_s = 0.0;
    double migration_s = 0.0;
    double total_s = 0.0;
    bool overlap = false;
};
StepTiming step_latency(uint64_t active_tokens, uint64_t distinct_active_experts, uint64_t bytes_migrated,
                        const TierConfig& tier, bool overlap_mode);

// ============================================================== specdec (reference specdec.hpp)
enum class DecodeMode { greedy, sampling };
const char* to_string(DecodeMode mode);

struct SpecConfig {
    int gamma = 10;
    int n_draft = 4;
    DecodeMode mode = DecodeMode::greedy;
    double temperature = 1.0;
    int batch = 1;
    int max_new_tokens = 32;
    int prompt_len = 8;
    bool use_affinity = true;
    int warmup_steps = 64;
    void validate() const;
};

struct StepOutcome {
    int seq = 0;
    int phase = 0;
    std::vector<int> drafts;
    int accepted = 0;
    int correction = 0;
    int tokens_generated = 0;
};

struct RunMetrics {
    double tau_mean = 1.0;
    uint64_t tokens_total = 0;
    int phases = 0;
    double speculation_s = 0.0;
    double verification_s = 0.0;
    double modeled_seconds = 0.0;
    double tokens_per_sec = 0.0;
    uint64_t bytes_spec = 0;
    uint64_t bytes_verify = 0;
    uint64_t bytes_baseline = 0;
    uint64_t bytes_total = 0;
    uint64_t setup_bytes = 0;
    uint64_t warmup_bytes = 0;
    double lambda = 1.0;
    double c_measured = 0.0;
};

struct LambdaInputs {
    uint64_t verify_tokens = 0;
    uint64_t verify_experts = 0;
    uint64_t step_tokens = 0;
    uint64_t step_experts = 0;
};

struct RunResult {
    std::vector<std::vector<int>> tokens;
    RunMetrics metrics;
    MigrationLedger ledger;
    std::vector<StepOutcome> outcomes;
    std::vector<TraceRow> trace;
    HotnessCounter hotness;
    std::vector<LambdaInputs> lambda_inputs;
};

struct SpeculationResult {
    std::vector<std::vector<int>> drafts;
    std::vector<std::vector<std::vector<double>>> draw_probs;
    ActivationRecord activations;
    std::vector<uint64_t> distinct_draft_experts;
};

SpeculationResult speculate(const ModelWeights& weights, const DraftState& draft_state, const AffinityTable* affinity,
                            const std::vector<std::vector<int>>& prefixes, int gamma, DecodeMode mode,
                            double temperature, Rng& rng);

struct VerifyResult {
    int accepted = 0;
    int correction = 0;
    ActivationRecord positions;
    std::vector<std::vector<double>> logits;
};

VerifyResult verify_greedy(const ModelWeights& weights, const std::vector<int>& prefix, const std::vector<int>& drafts);
VerifyResult verify_sampling(const ModelWeights& weights, const std::vector<int>& prefix,
                             const std::vector<int>& drafts, const std::vector<std::vector<double>>& draw_probs,
                             double temperature, Rng& rng);

RunResult run_specmoe(const ModelWeights& weights, const SpecConfig& config, DraftPolicy policy, const TierConfig& tier,
                      const std::vector<std::vector<int>>& prompts, uint64_t run_seed, const AffinityTable* affinity,
                      bool collect_trace = false);

double speedup_eq1(double tau, int gamma, double c);
double speedup_eq2(double tau, int gamma, double c, double lambda);
double measure_lambda(const std::vector<LambdaInputs>& phases, const TierConfig& tier);

// ============================================================== baselines (reference baselines.hpp)
enum class BaselineKind { ondemand, overlap, caching };
const char* to_string(BaselineKind kind);

struct BaselineConfig {
    BaselineKind kind = BaselineKind::ondemand;
    double cache_fraction = 0.10;
    int warmup_steps = 64;
    void validate() const;
};

RunResult run_ondemand(const ModelWeights& weights, const std::vector<std::vector<int>>& prompts,
                       const SpecConfig& decode, const TierConfig& tier, uint64_t run_seed, bool collect_trace = false);
RunResult run_overlap(const ModelWeights& weights, const std::vector<std::vector<int>>& prompts,
                      const SpecConfig& decode, const TierConfig& tier, uint64_t run_seed, bool collect_trace = false);
RunResult run_caching(const ModelWeights& weights, const std::vector<std::vector<int>>& prompts,
                      const SpecConfig& decode, const TierConfig& tier, const BaselineConfig& config,
                      uint64_t run_seed, bool collect_trace = false);

}  // namespace specmoe
