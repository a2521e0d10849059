/* oracle_abi.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * One flat C interface implemented twice:
 *   - oracle/specmoe_oracle.c : a plain-C restatement of the reference algorithm
 *                               (built into oracle/liboracle_port.so);
 *   - oracle/ref_shim.cpp     : a thin adapter over the reference's own C++ sources
 *                               compiled from /root/reference/proj/core/src
 *                               (built into oracle/_ref/libspecmoe_ref.so).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load either library.
 *
 * All types mirror the reference's value types (proj/core/include/specmoe/ headers) in flat
 * form; see the comments next to each field.
 */
#ifndef SPECMOE_ORACLE_ABI_H
#define SPECMOE_ORACLE_ABI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ModelSpec (model.hpp:16-32).  expert_kind 1 (swiglu3) is an extension of the port only. */
typedef struct {
    int num_layers, experts, top_k, hidden, ffn, vocab;
    double gate_skew;
    uint64_t seed;
    const uint8_t* moe_mask; /* num_layers entries, or NULL = every layer MoE */
    int expert_kind;         /* 0 = tanh2 (reference), 1 = swiglu3 (port only) */
    /* Port-only extension: real GQA attention with RoPE replaces the reference's
     * prefix-mean + mix surrogate when attn_heads > 0 (x0 = embedding of the token at each position;
     * per layer x += Wo attn(RoPE(Wq rms x), RoPE(Wk rms x), Wv rms x)).  The reference rejects it. */
    int attn_heads, kv_heads, head_dim;
    double rope_theta;
} om_spec;

/* SpecConfig (specdec.hpp:17-29) + TierConfig (memsim.hpp:28-39) + policy + seed. */
typedef struct {
    int gamma, n_draft, max_new_tokens, use_affinity, warmup_steps;
    int policy; /* DraftPolicy: 0 random, 1 hot_global, 2 hot_temporal */
    int collect_trace;
    uint64_t run_seed;
    uint64_t device_capacity_bytes, bytes_per_expert;
    double host_bandwidth, ssd_bandwidth, compute_rate, compute_cost_per_expert;
} om_run_cfg;

/* LedgerEntry (memsim.hpp:44-49); phase: 0 speculation, 1 verification, 2 baseline-step */
typedef struct { int phase, step, layer, expert; uint64_t bytes; } om_ledger_entry;
/* StepOutcome (specdec.hpp:32-39) */
typedef struct { int seq, phase, accepted, correction, tokens_generated; } om_outcome;

/* RunResult (specdec.hpp:70-78) with RunMetrics (41-57) flattened. */
typedef struct {
    int B, max_new, moe_layers, experts, top_k, gamma;
    int* tokens;   /* [B*max_new], row b valid for n_tokens[b] */
    int* n_tokens; /* [B] */
    int n_ledger;
    om_ledger_entry* ledger;
    int n_outcomes;
    om_outcome* outcomes;
    int* outcome_drafts; /* [n_outcomes*gamma] */
    int n_trace;          /* TraceRow (model.hpp:91-96): step, seq, layer, K experts */
    int* trace;           /* [n_trace*(3+K)] */
    uint64_t* hotness;    /* whole-run HotnessCounter [moe_layers*experts] */
    double tau_mean;
    uint64_t tokens_total;
    int phases;
    double speculation_s, verification_s, modeled_seconds, tokens_per_sec;
    uint64_t bytes_spec, bytes_verify, bytes_baseline, bytes_total, setup_bytes, warmup_bytes;
    double lambda, c_measured;
    double wall_s; /* steady_clock around the phase loop (whole call) */
} om_result;

/* Opaque model / affinity handles. */
void* om_build_model(const om_spec* spec, char* err, int errlen);
void om_free_model(void* model);
/* Export a weight tensor as float64, reference layout (row-major as in model.hpp:34-55).
 * name: "embedding","head","mix","gate","gate_bias","up","down","w1","w3","w2" (ffn for dense layers:
 * expert = -1).  Returns element count, or -1. */
long long om_get_tensor(void* model, const char* name, int layer, int expert, double* out, long long cap);

void* om_build_affinity(void* model);
void om_free_affinity(void* aff);
/* dist[moe_layer][E][E] */
int om_affinity_get(void* aff, double* out, long long cap);

/* forward (model.hpp:114-116).  restricted: [moe_layers*n_draft] sorted sets or NULL.
 * logits_out [V]; raw_out/final_out [moe_layers*K].  Returns 0, 1 (config) or 2 (invariant). */
int om_forward(void* model, const int* prefix, int n, const int* restricted, int n_draft, void* aff,
               double* logits_out, int* raw_out, int* final_out, char* err, int errlen);

/* Port only: forward() plus every MoE layer's gate logits (+ bias) [moe_layers*E] -- the decision
 * margins for the bf16 agreement tests. */
int om_forward_gates(void* model, const int* prefix, int n, double* logits_out, double* gates_out, char* err,
                     int errlen);

/* run_specmoe (specdec.hpp:122-124) and run_ondemand (baselines.hpp:24-26). prompts [B*prompt_len]. */
om_result* om_run_specmoe(void* model, const om_run_cfg* cfg, const int* prompts, int B, int prompt_len,
                          void* aff, char* err, int errlen);
om_result* om_run_ondemand(void* model, const om_run_cfg* cfg, const int* prompts, int B, int prompt_len,
                           char* err, int errlen);
/* run_overlap (baselines.hpp:30-34) and run_caching (baselines.hpp:36-41; BaselineConfig.warmup_steps =
 * cfg->warmup_steps). */
om_result* om_run_overlap(void* model, const om_run_cfg* cfg, const int* prompts, int B, int prompt_len,
                          char* err, int errlen);
om_result* om_run_caching(void* model, const om_run_cfg* cfg, double cache_fraction, const int* prompts, int B,
                          int prompt_len, char* err, int errlen);
void om_free_result(om_result* r);

/* CPU-baseline timing (bench.py): `threads` host threads each run `iters` forward() calls on the
 * shared read-only weights.  Returns wall seconds, or < 0 on error. */
double om_time_forward(void* model, const int* prefix, int n, int threads, int iters);

/* Host primitives (SPEC KATs). */
int om_route_topk(const double* logits, int n, int k, int* out);
int om_greedy_next(const double* logits, int n);
int om_softmax(const double* logits, int n, double* out);
int om_nearest_draft_expert(const double* dist_layer, int E, int raw, const int* draft, int nd,
                            const int* excluded, int nex);
int om_select_draft_experts(int policy, const uint64_t* counts, int layers, int E, const int* current,
                            int n_draft, uint64_t rng_seed, int* out);
double om_skewness(const uint64_t* counts, int layers, int E, uint64_t routed, double top_fraction);

#ifdef __cplusplus
}
#endif
#endif
