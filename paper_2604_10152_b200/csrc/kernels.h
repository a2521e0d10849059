// kernels.h -- launchers for the sm_100a kernels of the spec-decode hot path.
// Every launcher enqueues on the given stream and never synchronises.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace smoe {

// K1 (model.cpp:212-217): x[r] = (sum[b] + sum_{j<e} emb[pend[b][j]]) / (len[b] + e), computed in
// float64 in the reference's sequential order, stored as f32.  e = row_extra[r] (or extra_uniform
// when row_extra == nullptr); also writes the row's prefix length (for the surrogate remap).
void launch_x0(const double* emb64, const double* seq_sum, const int* seq_len, const int* pend, int pend_stride,
               const int* row_seq, const int* row_extra, int extra_uniform, int T, int d, float* x, int* row_plen,
               cudaStream_t s);

// K1 + K2 fused: the first layer's rms (model.cpp:19-26) of x0 -> xa (operand type).
void launch_x0_rms(const double* emb64, const double* seq_sum, const int* seq_len, const int* pend, int pend_stride,
                   const int* row_seq, const int* row_extra, int extra_uniform, int T, int d, float* x, int* row_plen,
                   void* xa, WType op, cudaStream_t s);

// K2 (model.cpp:19-26): xa[r] = x[r] * (mean(x^2) + 1e-12)^-1/2 in the operand type.
void launch_rms(const float* x, int T, int d, void* xa, WType op, cudaStream_t s);

// Residual add of a split-K GEMM followed by rms (dense layers, model.cpp:222-226):
//   x[t] += sum_s P[s][t] (s in order);  xa[t] = rms(x[t]).
void launch_resid_rms(float* x, const float* P, int S, long long pstride, int T, int d, void* xa, WType op,
                      cudaStream_t s);

// K4+K5+K6 (model.cpp:229-246, drafting.cpp:123-151): fused rms + gate GEMV + bias + softmax +
// top-K + (restricted) remap + dispatch.  Writes raw/final picks [T][K], the combine weight p[raw]
// [T][K], and dispatches the normalised row (operand type) straight into its experts' segments of
// xperm: pick (t,k) of expert e lands in row e*T + slot, slot = atomicAdd(&cnt[e], 1), and
// pos[t*K+k] records it.  Row order inside a segment is arbitrary: every GEMM column depends only on
// its own row, so results do not depend on it.
struct GateArgs {
    float* x;                 // residual stream; the mix partials are added first (x += sum_s pmix[s])
    const float* pmix;
    int s_mix;
    long long pstride;
    int T, d, E, K;
    const float* gate_w;  // [E][d]
    const float* gate_b;  // [E]
    void* xperm;          // out [E*T][d] operand type (expert segments of T rows)
    int* cnt;             // in/out [E] rows dispatched per expert (zero on entry)
    int* pos;             // out [T][K] xperm row of pick (t,k)
    WType op;
    int* raw;             // out [T][K]
    int* fin;             // out [T][K]
    float* wgt;           // out [T][K]
    // restricted (draft) mode; in_draft == nullptr => target semantics
    const uint8_t* in_draft;  // [E]
    const int* draft_sorted;  // [N]
    const int* rank;          // [E][N] draft members ordered by (affinity distance, index)
    int N;
    int use_affinity;
    int moe_ordinal;
    int seg;                  // rows per expert segment of xperm (0: T)
    const int* row_plen;      // prefix length per row (surrogate hash)
    int* flags;
    // expert parallelism, fused dispatch: expert e's rows go straight into rank e / ep_eo's receive buffer
    // (device table peer_x) at rows (ep_me * ep_eo + e % ep_eo) * seg + slot; nullptr = local xperm
    void* const* peer_x = nullptr;
    int ep_eo = 0, ep_me = 0;
    int stage_gw = 0;  // set by launch_gate: gate weights staged into shared memory before the dependency wait
};
void launch_gate(const GateArgs& a, cudaStream_t s);


// K9 (model.cpp:248-257) + the next rms: y_k = sum_s P[s][pos[t,k]] (split-K partials, s in order;
// pos == nullptr: row t*K+k),
// x[t] += sum_k wgt[t,k] * y_k (k in order; dense: x[t] += y), then xa[t] = rms(x[t]).
void launch_combine_rms(float* x, const float* P, int S, long long pstride, const int* pos, const float* wgt, int T,
                        int K, int d, int dense, void* xa, WType op, cudaStream_t s);

// K10 (model.cpp:172-176): per-row argmax, first max wins; non-finite -> flag.
void launch_argmax(const float* logits, int T, int V, int* out, int* flags, cudaStream_t s);

// dst[row_seq[r]*stride + extra(r)] = src[r]
void launch_scatter_tokens(const int* src, const int* row_seq, const int* row_extra, int extra_uniform, int T,
                           int* dst, int stride, cudaStream_t s);

// K11 (specdec.cpp:63-80): a = longest prefix drafts[i] == vam[i]; corr = vam[a].
void launch_accept(const int* drafts, const int* vam, const int* seqs, int na, int gamma, int stride, int* acc,
                   int* corr, cudaStream_t s);

// State advance / rollback (F6): sum[b] += emb[tok] for the taken tokens, len[b] += take.
void launch_commit(double* seq_sum, int* seq_len, const double* emb64, const int* seqs, const int* toks,
                   int tok_stride, const int* take, int na, int d, cudaStream_t s, int* last_tok = nullptr);

// Grouped skinny GEMM on CUDA cores (f32 or bf16 weights, f32 accumulation):
//   for group g with slot s = group_slot[g] >= 0 and rows [g*seg, g*seg + group_cnt[g]):
//     acc[r][n] = sum_k W[s][n][k] * X[r][k]       (n < Nout)
//   epilogue per Epi.  For kEpiSwiglu, W[s] has 2*Nout rows, interleaved: 2n = w1, 2n+1 = w3.
struct GemmArgs {
    const void* W;
    long long slot_stride;  // elements between slots
    int Nout, K;
    const int* group_cnt;  // nullptr -> single group {0, single_rows} with slot single_slot
    const int* group_slot;
    int G, seg;            // G groups; group g's rows start at g*seg
    int single_rows, single_slot;
    int rows_bound;  // upper bound on rows in any group (host-known)
    const void* X;   // [rows][K] operand type
    void* Y;         // [rows][ldy]
    int ldy;
    Epi epi;
};
void launch_gemm_simt(const GemmArgs& a, WType wt, cudaStream_t s);

// Device init / conversion helpers.
// Counter-based N(0, stddev) fill; element i of dst draws the variate of global index index0 + i, so
// a tensor filled in pieces equals the tensor filled at once.
// tile_k > 0: dst is an expert pool region in the tiled layout (tiled_index below) with K = tile_k; the
// values are those of the row-major fill (the variate of logical element i lands at tiled_index(i)).
void launch_fill_normal(void* dst, WType t, long long n, double stddev, uint64_t seed, uint64_t tensor_id,
                        cudaStream_t s, long long index0 = 0, int tile_k = 0);
void launch_fill_normal_f64(double* dst, long long n, double stddev, uint64_t seed, uint64_t tensor_id,
                            cudaStream_t s);
// dst[c*mul+off][r] = (T)src[r][c] for a rows x cols float64 source (reference row-major -> K-major;
// mul=2 interleaves the SwiGLU w1/w3 rows).
void launch_convert_transpose(const double* src, int rows, int cols, void* dst, WType t, cudaStream_t s,
                              int mul = 1, int off = 0, bool tiled = false);

// Tiled expert-pool layout of the tcgen05 engines (engine.h `tiled`): the pool [rows][K] is stored as
// [rows/256][K/64] chunks of 256 rows x 64 columns, each chunk 32 KB contiguous, so one TMA weight box of a
// pair unit is one contiguous DRAM stream instead of 256 pieces of 128 B at a K*2-byte stride
// (tools/bw_probe2.cu: 7.40 vs 7.01 TB/s at K=4096 on 148 SMs, 7.41 vs 6.77 on 88).  Needs rows % 256 == 0.
__host__ __device__ __forceinline__ long long tiled_index(long long row, long long k, int K) {
    return (((row >> 8) * (K >> 6) + (k >> 6)) << 14) + ((row & 255) << 6) + (k & 63);
}
// tile_k > 0: dst is a tiled matrix base and element i lands at tiled_index(row0 + i / tile_k, i % tile_k)
void launch_convert(const double* src, long long n, void* dst, WType t, cudaStream_t s, int tile_k = 0,
                    long long row0 = 0);
void launch_cast_f64_to_f32(const double* src, long long n, float* dst, cudaStream_t s);

// Pairwise L2 distance of expert weights (drafting.cpp:28-57) accumulated in float64:
// out[i*E+j] += sum_k (a_i[k]-a_j[k])^2 over one matrix pool region, for all i<j.
// draft members of each (layer, raw expert) ordered by (affinity distance, index); aff null = index order
void launch_rank_tables(const double* aff, const int* sorted, int M, int E, int nmax, int* rank, cudaStream_t s);
void launch_pairwise_sqdist(const void* pool, WType t, long long slot_stride, long long n, const int* slots, int E,
                            double* out, cudaStream_t s);

// Temperature sampling (sampling.cu).  sample_rows: row r of logits -> tok[r] drawn with u[r] from
// softmax(logits/T) (model.cpp:178-190), q row r = those probabilities when q != nullptr.
void launch_sample_rows(const float* logits, int R, int V, double T, const double* u, int* tok, double* q,
                        long long q_stride, cudaStream_t s);
// verify_sampling (specdec.cpp:82-157) for na sequences at once: verify rows s*(g+1)+i, draft probabilities
// q + i*q_tstride + s*V, uniforms from `pool` in sequence order; acc/corr per sequence, used[0] = uniforms
// consumed.  stats [na*(g+1)][2], kind/uidx [na], ratio [na*g] are scratch.
void launch_verify_sampling(const float* logits, int V, double T, double* stats, const double* q, long long q_tstride,
                            const int* drafts, int dstride, const int* seqs, int na, int g, const double* pool,
                            int* acc, int* kind, int* uidx, int* used, int* corr, int* flags, double* ratio,
                            cudaStream_t s);

// Real GQA attention (attn.cu).  KV cache pages of kKvPage tokens: [page][L][k|v][Hkv][kKvPage][hd].
constexpr int kKvPage = 16;
// x0 = emb[token of the row] and its rms (attention models): token/position from the sequence state
// (position len-1+i, token = last committed or pending draft i-1) or explicit (rtok/rpos, the prefill)
void launch_x0_tok_rms(const double* emb64, const int* seq_len, const int* last_tok, const int* pend, int pend_stride,
                       const int* row_seq, const int* row_extra, int extra_uniform, const int* rtok, const int* rpos,
                       int T, int d, float* x, int* row_plen, int* row_pos, void* xa, WType op, cudaStream_t s);
struct AttnArgs {
    const float* P;  // QKV projection split-K partials [S][Tmax][Hq*hd + 2*Hkv*hd]
    int S;
    long long pstride;
    int T, Hq, Hkv, hd;
    const float2* rope;  // [positions][hd/2] (cos, sin), launch_rope_table
    const int *row_seq, *row_pos, *ptab;
    int maxp, layer, L;
    float* qbuf;   // [Tmax][Hq*hd]
    void* kv;      // cache pages
    WType kvt;     // cache / output element type
    int max_pos;   // longest sequence the scores scratch holds
    void* out;     // [Tmax][Hq*hd] -> the Wo GEMM operand
};
void launch_attention(const AttnArgs& a, cudaStream_t s);
void launch_rope_table(int npos, int hd, double theta, float2* rope, cudaStream_t s);

}  // namespace smoe
