/* specmoe_b200.h -- C ABI of the B200-native self-assisted speculative-decoding engine.
 *
 * This is the drop-in boundary below the reference's C++ API (/root/reference/proj/core):
 * plain pointers, sizes and status codes, no STL, no torch types.  Each entry point names the
 * reference interface it replaces.  The C++ drop-in headers (include/specmoe/ headers) and the Python
 * host mirror (paper_2604_10152_b200/engine.py) are both built on these calls.
 *
 * Status codes (reference common.hpp:12-21 exit codes + CUDA): 0 ok, 1 ConfigError,
 * 2 InvariantError, 3 CUDA/NCCL error.  smoe_last_error() returns the thread-local message.
 */
#ifndef SPECMOE_B200_H
#define SPECMOE_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SMOE_OK = 0, SMOE_CONFIG = 1, SMOE_INVARIANT = 2, SMOE_CUDA = 3 };
enum { SMOE_F32 = 0, SMOE_BF16 = 1 };                      /* weight / operand storage */
enum { SMOE_EXPERT_TANH2 = 0, SMOE_EXPERT_SWIGLU3 = 1 };   /* model.cpp:54-59 / Mixtral */
enum { SMOE_GEMM_AUTO = 0, SMOE_GEMM_SIMT = 1, SMOE_GEMM_TCGEN05 = 2 };
enum { SMOE_POLICY_RANDOM = 0, SMOE_POLICY_HOT_GLOBAL = 1, SMOE_POLICY_HOT_TEMPORAL = 2 }; /* drafting.hpp:40 */
enum { SMOE_PHASE_SPECULATION = 0, SMOE_PHASE_VERIFICATION = 1, SMOE_PHASE_BASELINE = 2 }; /* memsim.hpp:21 */

typedef struct smoe_engine smoe_engine;

/* ModelSpec (model.hpp:16-32) + device configuration. */
typedef struct {
    int num_layers, experts, top_k, hidden, ffn, vocab;
    double gate_skew;
    uint64_t seed;
    const uint8_t* moe_mask; /* num_layers entries or NULL (every layer MoE) */
    int expert_kind;         /* SMOE_EXPERT_* */
    int weight_type;         /* SMOE_F32 (parity) / SMOE_BF16 (perf) */
    int max_batch, max_gamma;
    int gemm_backend;        /* SMOE_GEMM_* ; AUTO = tcgen05 for bf16, SIMT for f32 */
    int device;
    int offload;             /* 0: all experts HBM-resident; 1: pinned host pool + HBM slots (C3); 2: SSD tier,
                                a file on local storage ($SMOE_SSD_DIR, default /tmp) read with O_DIRECT */
    int hbm_expert_slots;    /* offload: HBM slot count (0 = 4 pinned draft experts per layer + two layers' transients) */
    int ep_rank, ep_world;   /* expert parallelism: this rank holds experts [r*E/G, (r+1)*E/G) of every layer
                                (0, 0 or 0, 1 = single GPU); attach a transport before running */
    /* Extension (no reference counterpart): attn_heads > 0 replaces the reference's
     * prefix-mean + mix surrogate with real GQA attention (RoPE, paged KV cache of max_seq_len tokens per
     * sequence; 0 = 512).  Single GPU only. */
    int attn_heads, kv_heads, head_dim;
    double rope_theta;
    int max_seq_len;
} smoe_engine_config;

/* SpecConfig (specdec.hpp:17-29) + TierConfig (memsim.hpp:28-39) + policy/seed + decode mode. */
typedef struct {
    int gamma, n_draft, max_new_tokens, use_affinity, warmup_steps, policy, collect_trace;
    uint64_t run_seed;
    uint64_t device_capacity_bytes, bytes_per_expert; /* ledger accounting (reference units) */
    double host_bandwidth, ssd_bandwidth, compute_rate, compute_cost_per_expert;
    int mode;           /* DecodeMode (specdec.hpp:15): 0 greedy, 1 sampling (draws on the device from the
                           host's sample_rng stream, substream(run_seed, "samp"), in the reference's order) */
    double temperature; /* sampling temperature (> 0) */
} smoe_run_config;

typedef struct { int phase, step, layer, expert; uint64_t bytes; } smoe_ledger_entry; /* memsim.hpp:44-49 */
typedef struct { int seq, phase, accepted, correction, tokens_generated; } smoe_outcome; /* specdec.hpp:32-39 */

/* RunResult (specdec.hpp:70-78) with RunMetrics (41-57) flattened, plus measured device time. */
typedef struct {
    int B, max_new, moe_layers, experts, top_k, gamma;
    int* tokens;
    int* n_tokens;
    int n_ledger;
    smoe_ledger_entry* ledger;
    int n_outcomes;
    smoe_outcome* outcomes;
    int* outcome_drafts;
    int n_trace;
    int* trace;
    uint64_t* hotness;
    double tau_mean;
    uint64_t tokens_total;
    int phases;
    double speculation_s, verification_s, modeled_seconds, tokens_per_sec;
    uint64_t bytes_spec, bytes_verify, bytes_baseline, bytes_total, setup_bytes, warmup_bytes;
    double lambda, c_measured;
    double wall_s;          /* host wall time of the loop */
    double gpu_s;           /* CUDA-event time of the loop on the engine stream */
    uint64_t h2d_expert_bytes; /* real bytes migrated by the expert store (offload mode) */
    double h2d_s;           /* CUDA-event time spent in expert migration copies */
    uint64_t prefetch_bytes;        /* overlap baseline: bytes the store prefetched for the next layer */
    uint64_t prefetch_wasted_bytes; /* ... of which the next layer never routed to */
} smoe_run_result;

const char* smoe_last_error(void);

/* Engine lifetime.  Replaces the implicit state of build_model (model.hpp:61) + ResidencyState. */
int smoe_engine_create(const smoe_engine_config* cfg, smoe_engine** out);
void smoe_engine_destroy(smoe_engine* e);
int smoe_engine_info(smoe_engine* e, uint64_t* device_bytes, uint64_t* bytes_per_expert_real, int* moe_layers);
void* smoe_engine_stream(smoe_engine* e); /* the cudaStream_t every hot-path kernel is launched on */

/* Weights.  exact: the reference's mt19937_64 polar stream (model.cpp:106-143, common.hpp:46-55),
 * converted to the engine's storage type, with the affinity table computed in float64 exactly as
 * drafting.cpp:28-57.  device: counter-based normal RNG on the GPU (perf shapes).
 * upload: a float64 tensor in the reference layout (model.hpp:34-55). */
int smoe_init_weights_exact(smoe_engine* e);
int smoe_init_weights_device(smoe_engine* e, uint64_t seed);
int smoe_upload_tensor(smoe_engine* e, const char* name, int layer, int expert, const double* src, long long n);
/* AffinityTable (drafting.hpp:14-21): [moe_layers][E][E] float64. */
int smoe_set_affinity(smoe_engine* e, const double* dist);
int smoe_build_affinity_device(smoe_engine* e);
int smoe_get_affinity(smoe_engine* e, double* out);

/* forward (model.hpp:114-116) for one prefix: logits [V] f32, raw/final picks [moe_layers][K].
 * restricted: [moe_layers][n_draft] sorted draft sets or NULL. */
int smoe_forward(smoe_engine* e, const int* prefix, int n, const int* restricted, int n_draft, int use_affinity,
                 float* logits_out, int* raw_out, int* final_out);

/* run_specmoe (specdec.hpp:122-124) / run_ondemand (baselines.hpp:24-26), greedy. */
int smoe_run_specmoe(smoe_engine* e, const smoe_run_config* cfg, const int* prompts, int B, int prompt_len,
                     smoe_run_result** out);
int smoe_run_ondemand(smoe_engine* e, const smoe_run_config* cfg, const int* prompts, int B, int prompt_len,
                      smoe_run_result** out);
/* run_overlap (baselines.hpp:30-34): the on-demand token stream and ledger; on the offloaded store each
 * layer's fetch is followed by a prefetch of the next layer's experts of the previous step, so the copy
 * engine streams while the layer computes (misses are fetched on demand; unused prefetches counted).
 * run_caching (baselines.hpp:36-41): top ceil(cache_fraction*E) experts per layer by a hot_global
 * on-demand warmup profile (cfg->warmup_steps) pinned in HBM, then on-demand decoding. */
int smoe_run_overlap(smoe_engine* e, const smoe_run_config* cfg, const int* prompts, int B, int prompt_len,
                     smoe_run_result** out);
int smoe_run_caching(smoe_engine* e, const smoe_run_config* cfg, double cache_fraction, const int* prompts, int B,
                     int prompt_len, smoe_run_result** out);
void smoe_free_result(smoe_run_result* r);

/* Stepped interface for benchmarking one speculative phase at a time (a "step" = draft pass of
 * gamma tokens + batched verify + accept/rollback + expert store for all active sequences). */
int smoe_spec_begin(smoe_engine* e, const smoe_run_config* cfg, const int* prompts, int B, int prompt_len);
int smoe_spec_step(smoe_engine* e, int* tokens_accepted_out, int* active_out);
int smoe_spec_end(smoe_engine* e, smoe_run_result** out);

/* Expert parallelism.  Experts sharded in contiguous blocks, the rows of every pass split in
 * contiguous blocks of ceil(T/G); per MoE layer the gate kernel stores routed rows into the expert
 * owners' memory and the owners' down-projection epilogue stores the finished rows back (NVLink peer
 * memory, CUDA IPC handles exchanged on the first pass, per-layer flags); env SMOE_EP_MODE=a2a uses two
 * NCCL all-to-alls instead.  Argmax tokens and routing logs are all-gathered once per pass, so every
 * rank holds the same host state and the results are bit-identical at any G.  Every engine call is
 * collective across the ranks.
 * NCCL: rank 0 calls smoe_ep_nccl_unique_id, the id is broadcast out of band, every rank attaches.
 * Loopback: G engines on one device driven by G host threads (validation without a multi-GPU box). */
typedef struct smoe_ep_loopback smoe_ep_loopback;
/* Host transport: one process per rank and a blocking host all-gather supplied by the caller
 * (torch.distributed/gloo, MPI, sockets): recv[r * bytes ..) = rank r's send[0 .. bytes), return 0 on
 * success.  Collectives are staged through host memory; the fused exchange's peer buffers are CUDA IPC
 * handles all-gathered the same way, so ranks may share one GPU (tests) or sit on different GPUs. */
typedef int (*smoe_host_allgather_fn)(void* user, const void* send, void* recv, uint64_t bytes);
int smoe_ep_attach_host(smoe_engine* e, smoe_host_allgather_fn fn, void* user);
int smoe_ep_nccl_unique_id(void* out, int len);
int smoe_ep_attach_nccl(smoe_engine* e, const void* id, int len);
smoe_ep_loopback* smoe_ep_loopback_create(int world);
void smoe_ep_loopback_destroy(smoe_ep_loopback* g);
int smoe_ep_attach_loopback(smoe_engine* e, smoe_ep_loopback* g);

/* Counters since the last reset: hot-path kernel launches, algorithmic HBM bytes of the expert GEMMs
 * (distinct experts touched per pass x bytes per expert) and of the dense GEMMs, and control-path
 * host<->device bytes (rows, accepted counts, routing logs). */
int smoe_counters(smoe_engine* e, uint64_t* launches, double* alg_expert_bytes, double* alg_dense_bytes,
                  uint64_t* ctl_h2d, uint64_t* ctl_d2h, int reset);

/* Named counters since the last smoe_counters(reset): "alg_expert_bytes:draft" / ":verify" (the split of
 * alg_expert_bytes by pass kind) and "expert_flops:draft" / ":verify" (2 * (U*d + d*f) per routed
 * (row, pick) on this rank's experts).  "ssd_direct": 1 when the SSD tier reads with O_DIRECT, 0 buffered,
 * -1 no SSD tier.  Unknown names read 0. */
int smoe_counter(smoe_engine* e, const char* name, double* value);

/* Expert GEMMs timed alone (bench.py roofline): T tokens routed round-robin over every expert of
 * MoE layer 0; average CUDA-event ms per up (w1/w3 or up) and down launch, and the algorithmic bytes
 * each launch must move (weights of touched experts + activations). */
int smoe_bench_expert_gemm(smoe_engine* e, int T, int iters, double* up_ms, double* down_ms, double* bytes_up,
                           double* bytes_down);

/* Kernel timing hooks for bench.py: events recorded around each launch of a kernel class ("expert_gemm",
 * "dense_gemm", "head_gemm", "gate", "combine", "pass"), each also counted under "<class>:draft" or
 * "<class>:verify" by the kind of pass that launched it. */
int smoe_profile_reset(smoe_engine* e);  /* clears the records and starts recording */
int smoe_profile_stop(smoe_engine* e);   /* stops recording (records stay readable) */
int smoe_profile_read(smoe_engine* e, const char* kernel_class, double* total_ms, long long* launches,
                      double* bytes);

/* Harness prompts (reference harness.hpp:60-62): prompt b = floor(uniform01 * V) draws from
 * mt19937_64(substream(seed, "prom", b)); out is [batch][prompt_len].  Host only (no device). */
int smoe_make_prompts(uint64_t seed, int batch, int prompt_len, int vocab, int* out);

#ifdef __cplusplus
}
#endif
#endif
