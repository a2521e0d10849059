// engine.h -- the B200 engine: device-resident model, per-sequence prefix state, batched draft /
// verify passes, expert store and the speculative-decode loop.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/specmoe_b200.h"
#include "common.cuh"
#include "ep.h"
#include "kernels.h"

namespace smoe {

// NVTX range for profilers (nsys / ncu --nvtx): a no-op unless a tool is attached (header-only nvtx3).
struct NvtxRange {
    explicit NvtxRange(const char* name);
    ~NvtxRange();
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// tcgen05 grouped GEMM (gemm_tc.cu).  A = weights (TMA, K-major, 128-row tiles), B = activations.
struct TcOperand {
    const void* base;  // bf16, row-major [rows][K]
    long long rows;
    int K;
    bool tiled = false;  // [rows/256][K/64][256][64] chunks (kernels.h tiled_index): a 3D tensor map
};
struct TcGemmArgs {
    TcOperand A;        // weight pool, 2D [slots*rows_per_slot, K]
    long long a_rows_per_slot;
    TcOperand B;        // activations [rows, K]
    int Nout, K;
    const int* group_cnt;  // nullptr -> single group {0, single_rows} with slot single_slot
    const int* group_slot;
    int G, seg;            // group g = rows [g*seg, g*seg + group_cnt[g]) of B / Y
    int single_rows, single_slot;
    int rows_bound;
    void* Y;
    int ldy;
    Epi epi;
    int splits;               // K splits (kEpiStoreF32 only): partial ks written at Y + ks*split_stride
    long long split_stride;
    int* sched;               // device [3] zero-initialised work counters (self-resetting)
    int* done = nullptr;      // device [64] zeroed per-group completion counters (fused launches)
    void* const* peer_y = nullptr;  // EP fused return (see tc::Phase): device table of the ranks' return buffers
    int peer_eo = 0, peer_me = 0;
    // grouped launches of draft passes: the groups expected to have rows (device, ascending), whose first
    // weight boxes are prefetched into L2 before the dependency wait
    const int* pred_groups = nullptr;
    int n_pred = 0;
};
void launch_gemm_tc(const TcGemmArgs& a, cudaStream_t s);
// One launch for a MoE layer's grouped up- (tanh / SwiGLU) and down-projection (f32 split partials):
// down units of expert g start once g's up units have published (gemm_tc.cu).
void launch_moe_tc(const TcGemmArgs& up, const TcGemmArgs& down, cudaStream_t s);

struct RunCfg {
    int gamma = 10, n_draft = 4, max_new_tokens = 32, use_affinity = 1, warmup_steps = 64, policy = 2,
        collect_trace = 0;
    uint64_t run_seed = 0;
    uint64_t device_capacity_bytes = 0, bytes_per_expert = 0;
    double host_bandwidth = 64e9, ssd_bandwidth = 0.0, compute_rate = 1e6, compute_cost_per_expert = 2e-6;
    int overlap = 0;  // baselines: oracle overlap timing, total = max(compute, migration) (baselines.cpp:101-111)
    int mode = 0;              // DecodeMode: 0 greedy, 1 sampling (specdec.hpp:15)
    double temperature = 1.0;  // sampling temperature (SpecConfig.temperature)
};

struct LedgerEntry { int phase, step, layer, expert; uint64_t bytes; };
struct Outcome { int seq, phase, accepted, correction, generated; std::vector<int> drafts; };
struct TraceRow { int step, seq, layer; std::vector<int> experts; };

struct RunOut {
    int B = 0, max_new = 0, gamma = 0;
    std::vector<std::vector<int>> tokens;
    std::vector<LedgerEntry> ledger;
    std::vector<Outcome> outcomes;
    std::vector<TraceRow> trace;
    std::vector<uint64_t> hotness;  // [M][E]
    double tau_mean = 1.0;
    uint64_t tokens_total = 0;
    int phases = 0;
    double speculation_s = 0, verification_s = 0, modeled_seconds = 0, tokens_per_sec = 0;
    uint64_t bytes_spec = 0, bytes_verify = 0, bytes_baseline = 0, bytes_total = 0, setup_bytes = 0,
             warmup_bytes = 0;
    double lambda = 1.0, c_measured = 0.0;
    double wall_s = 0, gpu_s = 0, h2d_s = 0;
    uint64_t h2d_expert_bytes = 0;
    uint64_t prefetch_bytes = 0, prefetch_wasted_bytes = 0;  // overlap baseline (store prefetch)
    std::vector<uint64_t> lambda_inputs;  // 4 per phase: verify tokens, verify experts, step tokens, step experts
};

struct SpecState;  // stepped loop state (loop.cpp)
struct SpecStateDeleter {
    void operator()(SpecState* s) const;
};

class Engine {
public:
    explicit Engine(const smoe_engine_config& c);
    ~Engine();

    // ---- configuration
    int L, E, K, d, f, V, M;
    int kind;        // ExpertKind
    WType wt;        // storage / operand type
    int use_tc;      // tcgen05 path for GEMMs
    int Bmax, Gmax, Tmax, stride;
    double skew;
    uint64_t seed;
    std::vector<uint8_t> mask;
    std::vector<int> moe_index;   // ordinal -> raw layer
    std::vector<int> moe_ord;     // raw layer -> ordinal or -1
    int n_dense;
    int offload, n_slots;
    int U;                        // rows per slot in the up pool (f or 2f)
    // expert parallelism: this rank owns experts [e_lo, e_hi) of every MoE layer
    int ep_rank = 0, ep_world = 1, e_lo = 0, e_hi = 0;
    std::unique_ptr<Comm> comm;
    // EP buffers (pass_ep): received routed rows, finished rows to return / returned, received counts,
    // per-layer group slots of the (source rank, local expert) groups, gathered logs / argmax / logits
    void* xrecv = nullptr;        // [E*Tmax][d] operand type
    float* ysend = nullptr;       // [E*Tmax][d]
    float* yret = nullptr;        // [s_down][E*Tmax][d]
    int* rcnt = nullptr;          // [E]
    int* ep_gslot = nullptr;      // [M][E]
    int* ep_logs = nullptr;       // [2][M][Tmax][K] packed + [G][2][M][Tmax][K] gathered
    int* amax_loc = nullptr;      // [Tmax]
    float* logits_loc = nullptr;  // [Tmax][V]
    bool ep_gather_logits = false;  // forward(): every rank needs row 0's logits
    TcOperand op_xrecv{};
    // fused peer-memory exchange (default; env SMOE_EP_MODE=a2a selects the NCCL all-to-all path): the gate
    // stores routed rows into the owners' xrecv, the down-projection epilogue stores partials into the
    // senders' yret ([s_down][E][Tmax][d]); per-layer sequence flags replace the collectives
    bool ep_p2p = false;
    int* ep_flags = nullptr;      // [2][G]: dispatch flags from the senders, done flags from the owners
    void** ep_peer = nullptr;     // device [4][G]: every rank's xrecv, rcnt, yret, ep_flags
    std::vector<void*> ep_ipc_opened;  // peer allocations opened through CUDA IPC (closed at teardown)
    int ep_seq = 0;               // MoE layer-passes exchanged so far (identical on every rank)
    bool ep_peers_ready = false;
    void ep_setup_peers();
    bool dev_rng = false;         // weights came from init_device (regenerable anywhere)
    uint64_t dev_seed = 0;
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    int device = 0;

    // ---- weights (device)
    double* emb64 = nullptr;  // [V][d]
    void* mix = nullptr;      // [L][d][d]
    float* gate_w = nullptr;  // [M][E][d]
    float* gate_b = nullptr;  // [M][E]
    void* up_pool = nullptr;  // [S][U][d]
    void* down_pool = nullptr;  // [S][d][f]
    void* head = nullptr;     // [V][d]
    int* slot_of = nullptr;   // [M][E] device
    std::vector<int> h_slot_of;
    std::vector<int> dense_slot;  // raw layer -> slot in pools (dense layers)
    std::vector<double> affinity;  // [M][E][E]
    bool have_affinity = false;
    uint64_t affinity_gen = 0;    // bumped whenever `affinity` is rebuilt or replaced
    double* aff_dev = nullptr;    // [M][E][E] device copy for the rank-table kernel
    uint64_t aff_dev_gen = ~0ull;

    // ---- expert store (offload mode, store.cpp): pinned host pools, HBM slot pool
    // offload 1: pinned host DRAM pools.  offload 2 (SSD tier): one file on local storage holding every
    // expert of this rank (O_DIRECT when the filesystem allows), read through pinned staging chunks
    struct SsdDeleter {
        void operator()(struct SsdTier* t) const;
    };
    std::unique_ptr<struct SsdTier, SsdDeleter> ssd;
    void host_to_device(int key, int which, void* dst, cudaStream_t s);   // which: 0 up/w1w3, 1 down
    double ssd_direct() const;  // -1: no SSD tier; 1: O_DIRECT; 0: buffered reads
    void device_to_host(int key, int which, const void* src);             // (synchronous)
    void* host_up = nullptr;    // [M*eo][U][d] pinned: this rank's experts (eo = E / ep_world), hkey order
    void* host_down = nullptr;  // [M*eo][d][f] pinned
    void* stage_up = nullptr;   // device staging of one expert (offload init)
    void* stage_down = nullptr;
    int n_exp_slots = 0;
    std::vector<int> slot_key;       // slot -> key (moe_layer*E + expert) or -1
    std::vector<uint8_t> key_pinned;
    std::vector<int> free_slots;
    int* h_store = nullptr;          // pinned: slot_of mirror [M*E], group sizes, group slots, raw picks
    std::vector<uint64_t> store_counts;  // routed picks per expert of the layer being fetched (all ranks' rows)
    int* ep_cntg = nullptr;               // EP: [G][E] device, the ranks' per-expert counts of one layer
    // overlap baseline (run_overlap): prefetch of the next layer's previous-step experts
    bool store_prefetch = false;
    std::vector<uint8_t> key_prefetched;  // [M*E] resident because of a prefetch, not yet routed to
    std::vector<uint8_t> prev_need;       // [M*E] keys the previous step routed to
    uint64_t prefetch_bytes = 0, prefetch_wasted = 0, prefetch_hits = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> h2d_ev;
    // hot_temporal re-pin decided per layer during a verify pass: (layer, routed picks per expert over
    // every row of the pass [E]) -> next set
    std::function<bool(int, const uint64_t*, std::vector<int>&)> repin_hook;
    bool owns(int key) const { const int e = key % E; return e >= e_lo && e < e_hi; }
    size_t hkey(int key) const { return (size_t)(key / E) * (e_hi - e_lo) + (size_t)(key % E - e_lo); }
    void store_alloc(int exp_slots);
    void store_reset();
    void upload_slot_rows(int m0, int m1);
    size_t expert_bytes(int which) const;
    void store_copy_in(int key, int slot);
    int store_take_slot(int key);
    void store_release(int key);
    void store_pin_sets(const std::vector<std::vector<int>>& sets);
    void store_fetch_layer(int mo, const int* cnt_dev);
    void store_fetch_layer_ep(int mo, const int* cnt_dev);
    void store_issue_layer(int mo, const int* cnt, int* gslot_dev);
    void store_finish_layer(int mo);
    void collect_h2d();

    // ---- per-sequence state / buffers (device)
    double* seq_sum = nullptr;  // [Bmax][d]
    int* seq_len = nullptr;     // [Bmax]
    int* drafts = nullptr;      // [Bmax][stride]
    int* vam = nullptr;         // [Bmax][stride]
    int *row_seq = nullptr, *row_extra = nullptr, *row_plen = nullptr;  // row_seq/row_extra: [2*Tmax]
    float* x = nullptr;
    void* xa = nullptr;
    int *raw_log = nullptr, *fin_log = nullptr;  // [Gmax+1][M][Tmax][K]
    float* wgt = nullptr;
    int *pos = nullptr, *group_slot = nullptr;
    int* grp_cnt = nullptr;  // [M][E] rows dispatched to each expert in the current pass (zeroed per pass)
    void* xperm = nullptr;  // [E*Tmax][d] expert segments of T rows (gate dispatch)
    void* hbuf = nullptr;   // [E*Tmax][f]
    float* ybuf = nullptr;  // [s_down][E*Tmax][d] split-K partials of the down projection
    const int* pred_groups = nullptr;  // draft passes: this layer's draft experts (fused MoE launch prefetch)
    int n_pred = 0;
    float* pmix = nullptr;  // [s_mix][Tmax][d] split-K partials of the mix GEMM
    int s_mix = 1, s_down = 1;
    int tile_up = 0, tile_dn = 0;  // tiled expert pools: their K (d, f); 0 = row-major (kernels.h tiled_index)
    bool tile_mix = false, tile_head = false, tile_qkv = false, tile_wo = false;  // tiled dense matrices
    float* logits = nullptr;  // [Tmax][V]
    int* amax = nullptr;
    uint8_t* in_draft = nullptr;  // [M][E]
    int* draft_sorted = nullptr;  // [M][Nmax]
    int* rank = nullptr;          // [M][E][Nmax]
    int* acc = nullptr;
    int* corr = nullptr;
    // sampling mode (sampling.cu), allocated on first use: host-drawn uniforms, the draft passes'
    // probabilities [Gmax][Bmax][V] f64, verify row statistics, acceptance scratch
    double* samp_u = nullptr;      // [Gmax*Bmax + Bmax*(Gmax+1)]
    double* samp_q = nullptr;
    double* samp_stats = nullptr;  // [Tmax][2]
    double* samp_ratio = nullptr;  // [Bmax*Gmax]
    int* samp_i = nullptr;         // kind [Bmax], uidx [Bmax], used [1]
    void sampling_alloc();
    void upload_doubles(double* dst, const double* src, size_t n);
    int* commit_toks = nullptr;  // [Bmax][stride]
    int* commit_take = nullptr;  // [Bmax]
    int* seqs = nullptr;         // [Bmax]
    int* flags = nullptr;
    int* sched = nullptr;        // tcgen05 GEMM dynamic tile scheduler counters [2 slots][4]
    int* moe_done = nullptr;     // fused expert GEMM per-group completion counters [2 slots][64]
    int fuse_moe = 1;            // one launch per MoE layer for up+down (env SMOE_FUSED_MOE=0: two)
    unsigned gemm_launches = 0;
    double* scratch64 = nullptr;  // staging for exact uploads / affinity partials
    size_t scratch64_n = 0;
    // pinned host staging
    int* h_small = nullptr;  // generic pinned int staging
    size_t h_small_n = 0;

    // tcgen05 operands (tensor maps are built and cached per box shape by gemm_tc.cu)
    TcOperand op_mix, op_up, op_down, op_head, op_xa, op_xperm, op_h;

    // ---- profiling (CUDA events around kernel classes)
    bool profiling = false;
    struct Prof {
        double ms = 0;
        long long n = 0;
        double bytes = 0;
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
        std::vector<const char*> sub;  // per event pair: the pass kind it also counts under ("cls:draft" ...)
    };
    std::map<std::string, Prof> prof;
    std::map<std::string, double> named;  // named counters (smoe_counter), reset with smoe_counters(reset)
    const char* prof_pass = nullptr;  // "draft" / "verify" while a pass runs (sub-class of every record)
    void prof_begin(const char* cls, cudaEvent_t* a);
    void prof_end(const char* cls, cudaEvent_t a, double bytes);
    void prof_collect();

    // ---- weights init
    void init_exact();
    void init_device(uint64_t seed);
    void upload_tensor(const std::string& name, int layer, int expert, const double* src, long long n);
    void build_affinity_device();

    // ---- draft tables
    void set_draft_sets(const std::vector<std::vector<int>>& sets, int n_draft, bool async = false);  // sorted per layer
    // Control uploads of a stepped speculative run without a host sync each: staged in a pinned arena and
    // queued on the engine stream; the arena is recycled (upload_reset) once the phase's readback has
    // synchronised the stream, so no queued copy can still be reading a reused region.
    void upload_async(void* dst, const void* src, size_t bytes);
    void upload_reset() { up_arena_off = 0; }
    char* up_arena = nullptr;
    size_t up_arena_n = 0, up_arena_off = 0;
    // The phase's readbacks the same way: queued device -> pinned-arena copies (rows of `rows` x `row_bytes`
    // at a device pitch), one stream sync, then download_finish() moves them into the host vectors
    // (a device -> pageable copy blocks the host once per call).
    void download_async(void* host_dst, const void* dev_src, size_t row_bytes, size_t rows = 1,
                        size_t dev_pitch = 0);
    void download_finish();
    char* dn_arena = nullptr;
    size_t dn_arena_n = 0, dn_arena_off = 0;
    struct PendingDown {
        void* dst;
        size_t off, bytes;
    };
    std::vector<PendingDown> dn_pending;
    int cur_n_draft = 0;
    // ---- real GQA attention (attn.cu; attn_heads > 0)
    int Hq = 0, Hkv = 0, hd = 0, QD = 0, KD = 0, QKVD = 0, max_seq = 0, maxp = 0, s_qkv = 1;
    double theta = 1e4;
    void* wqkv = nullptr;    // [L][QKVD][d]: rows q (QD), k (KD), v (KD) -- K-major, like the Mix
    void* wo = nullptr;      // [L][d][QD]
    float* pqkv = nullptr;   // [s_qkv][Tmax][QKVD] split-K partials of the QKV projection
    float* qbuf = nullptr;   // [Tmax][QD] rotated queries
    void* attn_o = nullptr;  // [Tmax][QD] attention output (the Wo GEMM operand)
    void* kv = nullptr;      // KV pages [n_pages][L][2][Hkv][kKvPage][hd]
    int* ptab = nullptr;     // [Bmax][maxp] page table
    int* last_tok = nullptr; // [Bmax] last committed token (the input of the next row)
    int* row_pos = nullptr;  // [Tmax] position of each row of the pass
    float2* rope = nullptr;  // [maxp * kKvPage][hd/2] RoPE (cos, sin)
    int* pre_tok = nullptr;  // [Tmax] prefill rows: explicit tokens and positions
    int* pre_pos = nullptr;
    bool prefill_rows = false;
    TcOperand op_wqkv{}, op_wo{}, op_ao{};
    std::vector<std::vector<int>> kv_pages;  // host: pages of each sequence
    std::vector<int> kv_free, h_seq_len;
    bool attn() const { return Hq > 0; }
    void kv_fit(int b);     // pages for positions [0, h_seq_len[b] + Gmax] (and the table row uploaded)
    void kv_advance(const std::vector<int>& seqs, const std::vector<int>& takes);
    void attn_layer(int l, int T, const int* rseq);
    void prefill(const std::vector<std::vector<int>>& prompts);

    // ---- passes
    // rows r=0..T-1: sequence slot row_seq[r], pending-draft count row_extra[r] (or extra_uniform).
    // restricted = draft semantics.  log_slot selects where raw/fin picks are logged.
    void pass(int T, const int* rseq, const int* rextra, int extra_uniform, bool restricted, int use_aff,
              int log_slot);
    void gemm(const void* W, long long slot_stride, const TcOperand& aop, long long a_rows_per_slot, int Nout, int Kd,
              const int* gcnt, const int* gslot, int G, int seg, int single_rows, int single_slot, int rows_bound,
              const void* X, const TcOperand& bop, void* Y, int ldy, Epi epi, const char* cls, double bytes,
              int splits = 1, long long split_stride = 0);
    // a MoE layer's expert FFN (grouped up + down projection), fused into one launch on tcgen05; rows of
    // group g are [g*seg, g*seg + cnt[g]) of X (xperm, or the received rows under EP)
    void expert_ffn(int seg, const int* cnt, const int* slots, const char* cls, const void* X = nullptr,
                    const TcOperand* xop = nullptr, void* const* peer_y = nullptr);
    // expert-parallel pass: rows split across ranks, all-to-all dispatch / combine per MoE layer (ep.h)
    void pass_ep(int T, const int* rseq, const int* rextra, int extra_uniform, bool restricted, int use_aff,
                 int log_slot);

    // ---- host<->device helpers
    void upload_ints(int* dst, const int* src, size_t n);  // via pinned staging, async on stream
    void sync();
    void h2d(void* dst, const void* src, size_t bytes);
    void check_flags();

    // ---- public ops
    void forward_one(const std::vector<int>& prefix, const int* restricted, int n_draft, int use_aff,
                     float* logits_out, int* raw_out, int* fin_out);
    void reset_sequences(const std::vector<std::vector<int>>& prompts);

    // isolated expert-GEMM microbenchmark (bench.py roofline, kernel timed alone)
    void bench_expert_gemm(int T, int iters, double* up_ms, double* down_ms, double* bytes_up, double* bytes_down);

    // ---- counters (bench.py): kernel launches, algorithmic HBM bytes, control-path PCIe bytes
    uint64_t launches = 0, ctl_h2d = 0, ctl_d2h = 0;
    // captured speculative phases (loop.cpp spec_step, SMOE_GRAPH=1): key (rows, gamma, affinity)
    struct PhaseGraph {
        cudaGraphExec_t exec;
        uint64_t launches;
        double dense_bytes;
    };
    std::map<uint64_t, PhaseGraph> phase_graphs;
    uint64_t last_phase_key = ~0ull;
    cudaStream_t capture_stream = nullptr;  // phase graphs are recorded here while the engine stream runs
    double alg_expert_bytes = 0, alg_dense_bytes = 0;

    // ---- store (offload)
    uint64_t real_bytes_per_expert() const;
    uint64_t h2d_bytes = 0;
    double h2d_ms = 0;

    // stepped loop
    std::unique_ptr<SpecState, SpecStateDeleter> st;
};


// loop.cpp
RunOut run_specmoe(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts);
// pinned_sets != nullptr: MoE-Caching (baselines.cpp:117-145) -- those experts are pinned before the
// run (setup bytes, excluded from the ledger) and cost zero bytes afterwards.
RunOut run_ondemand(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts,
                    const std::vector<std::vector<int>>* pinned_sets = nullptr);
// baselines.cpp:117-145: greedy on-demand warmup profile -> top ceil(fraction*E) per layer.
std::vector<std::vector<int>> caching_sets(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts,
                                           double cache_fraction, uint64_t* warmup_bytes);
void spec_begin(Engine& e, const RunCfg& c, const std::vector<std::vector<int>>& prompts);
int spec_step(Engine& e, int* accepted_tokens);  // returns number of active sequences after the step
RunOut spec_end(Engine& e);

}  // namespace smoe
