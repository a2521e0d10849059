// attn.cu -- real GQA attention with RoPE over a paged KV cache (no reference counterpart:
// the reference's attention is a prefix-mean surrogate, model.cpp:211-224).  Enabled by attn_heads > 0;
// the layer becomes  x += Wo . attn(RoPE(Wq rms x), RoPE(Wk rms x), Wv rms x)  in place of  x += Mix rms x,
// and x0 is the embedding of the row's own token (the restatement: oracle/specmoe_oracle.c fwd_attn).
//
// Row r of a pass = (sequence b, position p): its token is the sequence's last committed token (p =
// len-1) or a pending draft (p = len-1+i), or an explicit (token, position) during the prompt prefill.
// The QKV projection is a tcgen05 (or CUDA-core) GEMM writing split-K partials; k_qkv_rope sums them,
// rotates q/k and stores k/v of (b, p) into the sequence's page of the cache; k_attn runs one CTA per
// (row, kv head) with one warp per query head of the group, over positions 0..p of the pages; its
// output is the Wo GEMM's operand, whose split-K partials the gate / residual kernels add to x exactly
// as they add the Mix partials.
//
// Every row's arithmetic is a fixed function of its inputs (fixed summation orders, no cross-row
// reductions), so draft, verify and on-demand passes compute a position identically (losslessness).
// Cache semantics: positions < len-1 hold the target model's k/v; a draft pass writes its own (draft
// model) k/v at len-1+t; the verify pass rewrites len-1..len-1+gamma with the target's; acceptance keeps
// the committed length (rollback = not advancing it), so stale draft k/v is never read.
#include "common.cuh"
#include "kernels.h"

namespace smoe {
namespace {

constexpr int kPage = kKvPage;

template <typename T>
__device__ __forceinline__ void store_op(void* base, long long idx, float v) {
    reinterpret_cast<T*>(base)[idx] = from_f<T>(v);
}
// fixed-order block reduction (warp butterflies, then warp 0), as the other row kernels
__device__ float block_sum(float v, float* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    float t = lane < nw ? red[lane] : 0.f;
    if (w == 0)
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[32] = t;
    __syncthreads();
    return red[32];
}

// x0 = emb[token] (float64 table -> f32) and its rms; row_plen = position + 1 (the remap hash's prefix
// length), row_pos = position.
template <typename OT>
__global__ void k_x0_tok_rms(const double* __restrict__ emb, const int* __restrict__ slen,
                             const int* __restrict__ last_tok, const int* __restrict__ pend, int pstride,
                             const int* __restrict__ row_seq, const int* __restrict__ row_extra, int extra_u,
                             const int* __restrict__ rtok, const int* __restrict__ rpos, int d, float* __restrict__ x,
                             int* __restrict__ row_plen, int* __restrict__ row_pos, void* __restrict__ xa) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float row[];
    __shared__ float red[33];
    const int r = blockIdx.x, b = row_seq[r];
    int tok, p;
    if (rtok) {
        tok = rtok[r];
        p = rpos[r];
    } else {
        const int e = row_extra ? row_extra[r] : extra_u;
        p = slen[b] - 1 + e;
        tok = e == 0 ? last_tok[b] : pend[(long long)b * pstride + e - 1];
    }
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        const float v = (float)emb[(long long)tok * d + i];
        x[(long long)r * d + i] = v;
        row[i] = v;
        ss += v * v;
    }
    if (threadIdx.x == 0) {
        row_plen[r] = p + 1;
        row_pos[r] = p;
    }
    ss = block_sum(ss, red);
    const float inv = 1.0f / sqrtf(ss / (float)d + 1e-12f);
    for (int i = threadIdx.x; i < d; i += blockDim.x) store_op<OT>(xa, (long long)r * d + i, row[i] * inv);
}

template <typename KT>
__device__ __forceinline__ long long kv_off(const int* ptab, int maxp, int b, int p, int l, int L, int kv, int h,
                                            int Hkv, int hd) {
    const long long page = ptab[(long long)b * maxp + p / kPage];
    return ((((page * L + l) * 2 + kv) * Hkv + h) * kPage + p % kPage) * (long long)hd;
}

// RoPE table: rope[p][j] = (cos, sin) of p * theta^(-2j/hd), evaluated in float64 and rounded once.
__global__ void k_rope_table(int npos, int half, int hd, double theta, float2* __restrict__ rope) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npos * half; i += gridDim.x * blockDim.x) {
        const int p = i / half, j = i % half;
        double sn, cs;
        sincos((double)p * pow(theta, -2.0 * j / hd), &sn, &cs);
        rope[i] = make_float2((float)cs, (float)sn);
    }
}

// qkv = sum_s P[s][r] (s in order); RoPE (rotate-half with the table) on the Hq query and Hkv key heads;
// q -> qbuf, k/v -> the cache page of (b, p).
template <typename KT>
__global__ void k_qkv_rope(const float* __restrict__ P, int S, long long pstride, int Hq, int Hkv, int hd,
                           const float2* __restrict__ rope, const int* __restrict__ row_seq,
                           const int* __restrict__ row_pos, const int* __restrict__ ptab, int maxp, int l, int L,
                           float* __restrict__ qbuf, KT* __restrict__ kv) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x, b = row_seq[r], p = row_pos[r];
    const int QD = Hq * hd, KD = Hkv * hd, W = QD + 2 * KD, half = hd / 2;
    const float* pr = P + (long long)r * W;
    auto sum = [&](int c) {
        float v = 0.f;
        for (int s = 0; s < S; ++s) v += pr[s * pstride + c];
        return v;
    };
    // rotated pairs (j, j + hd/2) of the query and key heads
    for (int i = threadIdx.x; i < (Hq + Hkv) * half; i += blockDim.x) {
        const int h = i / half, j = i % half;
        const int c0 = h * hd + j;  // heads are contiguous: q heads, then k heads
        const float x0 = sum(c0), x1 = sum(c0 + half);
        const float2 cs = rope[(long long)p * half + j];
        const float c = cs.x, s = cs.y;
        const float y0 = x0 * c - x1 * s, y1 = x1 * c + x0 * s;
        if (h < Hq) {
            qbuf[(long long)r * QD + c0] = y0;
            qbuf[(long long)r * QD + c0 + half] = y1;
        } else {
            const long long o = kv_off<KT>(ptab, maxp, b, p, l, L, 0, h - Hq, Hkv, hd);
            kv[o + j] = from_f<KT>(y0);
            kv[o + j + half] = from_f<KT>(y1);
        }
    }
    for (int c = threadIdx.x; c < KD; c += blockDim.x) {
        const long long o = kv_off<KT>(ptab, maxp, b, p, l, L, 1, c / hd, Hkv, hd);
        kv[o + c % hd] = from_f<KT>(sum(QD + KD + c));
    }
}

// One CTA per (row, kv head), one warp per query head of the group: scores q.k_t / sqrt(hd) over
// t = 0..p (lane-strided, each dot product in dimension order), max-subtracted exp, a butterfly sum,
// then o = sum_t (e_t / sum) v_t in position order (lanes over dimensions).  The K and V rows of the
// sequence are staged in shared memory kAttnChunk positions at a time with coalesced 16-byte loads (the
// CTA's warps share them); every per-lane loop keeps its order, so the result does not depend on the
// staging.  o -> the Wo GEMM operand.
constexpr int kAttnChunk = 64;
template <typename KT, typename OT>
__global__ void k_attn(const float* __restrict__ qbuf, int Hq, int Hkv, int hd, const int* __restrict__ row_seq,
                       const int* __restrict__ row_pos, const int* __restrict__ ptab, int maxp, int l, int L,
                       const KT* __restrict__ kv, int max_pos, void* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float sm[];
    const int r = blockIdx.x, kh = blockIdx.y, b = row_seq[r], p = row_pos[r];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, G = Hq / Hkv, h = kh * G + w;
    float* sq = sm + (size_t)w * hd;                        // this warp's query [hd]
    float* sc = sm + (size_t)G * hd + (size_t)w * max_pos;   // its scores / weights [p + 1]
    KT* stg = reinterpret_cast<KT*>(sm + (size_t)G * hd + (size_t)G * max_pos);  // [kAttnChunk][hd] K or V rows
    const int QD = Hq * hd;
    for (int j = lane; j < hd; j += 32) sq[j] = qbuf[(long long)r * QD + (long long)h * hd + j];
    // cooperative staging of positions [t0, t0 + n) of the k (kv = 0) or v (kv = 1) rows of this kv head:
    // a page holds kKvPage consecutive positions of one (layer, k|v, head) contiguously
    const int vec = 16 / (int)sizeof(KT), hv = hd / vec;  // 16-byte vectors per row
    auto stage = [&](int kvsel, int t0, int n) {
        __syncthreads();
        for (int i = threadIdx.x; i < n * hv; i += blockDim.x) {
            const int t = t0 + i / hv, c = i % hv;
            const KT* src = kv + kv_off<KT>(ptab, maxp, b, t, l, L, kvsel, kh, Hkv, hd);
            reinterpret_cast<uint4*>(stg + (size_t)(t - t0) * hd)[c] = reinterpret_cast<const uint4*>(src)[c];
        }
        __syncthreads();
    };
    const float inv = 1.0f / sqrtf((float)hd);
    float mx = -INFINITY;
    for (int t0 = 0; t0 <= p; t0 += kAttnChunk) {
        const int n = min(kAttnChunk, p + 1 - t0);
        stage(0, t0, n);
        for (int t = t0 + lane; t < t0 + n; t += 32) {
            const KT* kt = stg + (size_t)(t - t0) * hd;
            float s = 0.f;
            for (int j = 0; j < hd; ++j) s = fmaf(sq[j], to_f(kt[j]), s);
            s *= inv;
            sc[t] = s;
            mx = fmaxf(mx, s);
        }
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float part = 0.f;
    for (int t = lane; t <= p; t += 32) {
        const float e = expf(sc[t] - mx);
        sc[t] = e;
        part += e;
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    constexpr int kMaxDims = 8;  // hd <= 256: dimensions j = lane + 32 i of this lane
    float acc[kMaxDims];
#pragma unroll
    for (int i = 0; i < kMaxDims; ++i) acc[i] = 0.f;
    for (int t0 = 0; t0 <= p; t0 += kAttnChunk) {
        const int n = min(kAttnChunk, p + 1 - t0);
        stage(1, t0, n);
        for (int t = t0; t < t0 + n; ++t) {
            const float wgt = sc[t] / part;
            const KT* vt = stg + (size_t)(t - t0) * hd;
#pragma unroll
            for (int i = 0; i < kMaxDims; ++i)
                if (lane + 32 * i < hd) acc[i] = fmaf(wgt, to_f(vt[lane + 32 * i]), acc[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < kMaxDims; ++i)
        if (lane + 32 * i < hd) store_op<OT>(out, (long long)r * QD + (long long)h * hd + lane + 32 * i, acc[i]);
}

}  // namespace

void launch_x0_tok_rms(const double* emb64, const int* seq_len, const int* last_tok, const int* pend, int pend_stride,
                       const int* row_seq, const int* row_extra, int extra_uniform, const int* rtok, const int* rpos,
                       int T, int d, float* x, int* row_plen, int* row_pos, void* xa, WType op, cudaStream_t s) {
    if (T <= 0) return;
    const size_t sm = sizeof(float) * d;
    if (op == kF32)
        launch_k(k_x0_tok_rms<float>, T, row_threads(d), sm, s, emb64, seq_len, last_tok, pend, pend_stride, row_seq,
                 row_extra, extra_uniform, rtok, rpos, d, x, row_plen, row_pos, xa);
    else
        launch_k(k_x0_tok_rms<__nv_bfloat16>, T, row_threads(d), sm, s, emb64, seq_len, last_tok, pend, pend_stride,
                 row_seq, row_extra, extra_uniform, rtok, rpos, d, x, row_plen, row_pos, xa);
}

void launch_rope_table(int npos, int hd, double theta, float2* rope, cudaStream_t s) {
    launch_k(k_rope_table, 128, 256, 0, s, npos, hd / 2, hd, theta, rope);
}

void launch_attention(const AttnArgs& a, cudaStream_t s) {
    if (a.T <= 0) return;
    if (a.hd > 256 || a.hd % 8) throw Error(kConfig, "attention: head_dim must be a multiple of 8, at most 256");
    if (a.kvt == kF32)
        launch_k(k_qkv_rope<float>, a.T, 256, 0, s, a.P, a.S, a.pstride, a.Hq, a.Hkv, a.hd, a.rope, a.row_seq,
                 a.row_pos, a.ptab, a.maxp, a.layer, a.L, a.qbuf, reinterpret_cast<float*>(a.kv));
    else
        launch_k(k_qkv_rope<__nv_bfloat16>, a.T, 256, 0, s, a.P, a.S, a.pstride, a.Hq, a.Hkv, a.hd, a.rope,
                 a.row_seq, a.row_pos, a.ptab, a.maxp, a.layer, a.L, a.qbuf, reinterpret_cast<__nv_bfloat16*>(a.kv));
    const int G = a.Hq / a.Hkv;
    const size_t kvb = a.kvt == kF32 ? 4 : 2;
    const size_t sm = sizeof(float) * ((size_t)G * a.hd + (size_t)G * a.max_pos) + (size_t)kAttnChunk * a.hd * kvb;
    const dim3 grid(a.T, a.Hkv);
    if (a.kvt == kF32)
        launch_k(k_attn<float, float>, grid, 32 * G, sm, s, (const float*)a.qbuf, a.Hq, a.Hkv, a.hd, a.row_seq,
                 a.row_pos, a.ptab, a.maxp, a.layer, a.L, (const float*)a.kv, a.max_pos, a.out);
    else
        launch_k(k_attn<__nv_bfloat16, __nv_bfloat16>, grid, 32 * G, sm, s, (const float*)a.qbuf, a.Hq, a.Hkv, a.hd,
                 a.row_seq, a.row_pos, a.ptab, a.maxp, a.layer, a.L, (const __nv_bfloat16*)a.kv, a.max_pos, a.out);
}

}  // namespace smoe
