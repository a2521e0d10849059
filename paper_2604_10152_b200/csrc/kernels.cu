// kernels.cu -- state, normalisation, gating/routing, permutation, combine, argmax, accept and
// commit kernels of the spec-decode hot path (sm_100a).  These move a few MB per pass, so they
// are latency-bound; they are written as single-pass, coalesced, 16-byte-vectorised kernels.
#include <cooperative_groups.h>
#include <math.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.h"
#include "gate_dev.cuh"
#include "tc_common.cuh"

namespace smoe {

bool g_use_pdl = [] {
    const char* v = std::getenv("SMOE_PDL");
    return !(v && v[0] == '0');
}();

namespace {

constexpr int kPairChunks = 64;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Fixed-order block reduction (warp butterflies then warp 0): the result depends only on the
// block size, never on T, so every row is computed identically in every pass (batch invariance).
__device__ float block_sum(float v, float* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    float t = lane < nw ? red[lane] : 0.f;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) red[32] = t;
    __syncthreads();
    return red[32];
}

// In-step timeline of the row kernels (SMOE_TC_TRACE builds, read by tools/tc_trace.py): one record per
// block -- kernel id, block, entry, dependency wait released, end -- in a device ring.
#ifdef SMOE_TC_TRACE
struct RkRec {
    int kid, blk;
    long long t_in, t_wait, t_end, t_m[3];  // t_m: kernel-specific marks (gate: rms done, GEMV done, selected)
};
constexpr int kRkRing = 1 << 18;
__device__ RkRec g_rk[kRkRing];
__device__ unsigned g_rk_n;
__device__ __forceinline__ long long rk_now() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define RK_IN() \
    const long long rk_t0 = rk_now(); \
    long long rk_m[3] = {0, 0, 0}
#define RK_WAITED() const long long rk_t1 = rk_now()
#define RK_MARK(n) rk_m[n] = rk_now()
#define RK_END(kid)                                                                                      \
    do {                                                                                                 \
        if (threadIdx.x == 0) {                                                                          \
            const unsigned i = atomicAdd(&g_rk_n, 1u) % kRkRing;                                         \
            g_rk[i] = RkRec{kid, (int)blockIdx.x, rk_t0, rk_t1, rk_now(), {rk_m[0], rk_m[1], rk_m[2]}};  \
        }                                                                                                \
    } while (0)
#else
#define RK_IN()
#define RK_WAITED()
#define RK_MARK(n)
#define RK_END(kid)
#endif

template <typename T>
__device__ __forceinline__ void store_op(void* base, long long idx, float v) {
    reinterpret_cast<T*>(base)[idx] = from_f<T>(v);
}

// ------------------------------------------------------------------ K1 prefix state
__global__ void k_x0(const double* __restrict__ emb, const double* __restrict__ ssum, const int* __restrict__ slen,
                     const int* __restrict__ pend, int pstride, const int* __restrict__ row_seq,
                     const int* __restrict__ row_extra, int extra_u, int d, float* __restrict__ x,
                     int* __restrict__ row_plen) {
    const int r = blockIdx.x;
    const int b = row_seq[r];
    const int e = row_extra ? row_extra[r] : extra_u;
    const int n = slen[b] + e;
    const int* toks = pend + (long long)b * pstride;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        double acc = ssum[(long long)b * d + i];
        for (int j = 0; j < e; ++j) acc += emb[(long long)toks[j] * d + i];
        x[(long long)r * d + i] = (float)(acc / (double)n);
    }
    if (threadIdx.x == 0) row_plen[r] = n;
}

// ------------------------------------------------------------------ K2 rms
template <typename OT>
__global__ void k_rms(const float* __restrict__ x, int d, void* __restrict__ xa) {
    pdl_wait();
    pdl_trigger();
    __shared__ float red[33];
    const float* xr = x + (long long)blockIdx.x * d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) ss += xr[i] * xr[i];
    ss = block_sum(ss, red);
    const float inv = 1.0f / sqrtf(ss / (float)d + 1e-12f);
    for (int i = threadIdx.x; i < d; i += blockDim.x) store_op<OT>(xa, (long long)blockIdx.x * d + i, xr[i] * inv);
}

// Row kernels below keep one row in shared memory (d floats) and use float4 accesses (d % 4 == 0).
template <typename OT>
__device__ __forceinline__ void store_row_op(void* xa, long long base, const float* row, int d, float inv) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) store_op<OT>(xa, base + i, row[i] * inv);
}

// ---- virtual-block row kernels (resid+rms, gate, combine+rms)
// These kernels always evaluate exactly the reduction tree of a VB-thread block (VB = row_threads(d) or
// gate_threads(d, E), the trees the pass kernel and the tests pin), whatever the launch shape: a row is
// processed by a cluster of C CTAs of RT threads (RowCtx below), each real thread playing one or more
// virtual threads that accumulate their columns in order, and the virtual warps' butterflies feed the
// same final warp.  Default shape: C = VB/256 CTAs of 256 threads per row (SMOE_ROW_CLUSTER=0: one
// VB-thread block per row, or SMOE_ROW_THREADS fewer threads).  Small CTAs sit beside a GEMM CTA on an
// SM (a 1024-thread block at 64 registers fills the register file, so the next Mix launch's CTAs could
// not start on the SMs of the combine), and spread a draft pass's 64 rows over 4x the SMs.  Split-K
// partials are loaded four or eight at a time (the old loop issued one dependent load per partial).
int row_rt(int vb) {
    static const int rt = [] {
        const char* v = std::getenv("SMOE_ROW_THREADS");
        return v ? std::atoi(v) : 0;
    }();
    return rt >= 256 && rt < vb && vb % rt == 0 ? rt : vb;
}
struct RowShape {
    int C, RT;
};
RowShape row_shape(int vb, int T = 0) {
    static const bool cl = [] {
        const char* v = std::getenv("SMOE_ROW_CLUSTER");
        return v && v[0] == '1';
    }();
    static const int wide = [] {  // SMOE_ROW_WIDE=0: off
        const char* v = std::getenv("SMOE_ROW_WIDE");
        return v ? std::atoi(v) : 1;
    }();
    if (cl && vb > 256) return {vb / 256, 256};
    // A VB-thread row block fills an SM's register file (1024 x 64), so a pass with T rows takes
    // ceil(T / SMs) waves; with more rows than SMs (a verify pass: 320 at B=64) 256-thread blocks playing
    // the same VB-thread tree put four rows on an SM and finish in one wave (the gate of a C2 verify pass:
    // 26.7 -> 18.8 us, bit-identical)
    if (wide && T > tc::sm_count() && vb > 256 && vb % 256 == 0 && row_rt(vb) == vb) return {1, 256};
    return {1, row_rt(vb)};
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void add4(float4& a, const float4 b) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}
// sum_{s=0..S-1} P[s][off..off+4) in order from zero; loads issued B at a time
template <int B>
__device__ __forceinline__ float4 sum_splits(const float* __restrict__ P, long long pstride, int S, long long off) {
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s0 = 0; s0 < S; s0 += B) {
        float4 q[B];
#pragma unroll
        for (int j = 0; j < B; ++j)
            if (s0 + j < S) q[j] = ld4(P + (s0 + j) * pstride + off);
#pragma unroll
        for (int j = 0; j < B; ++j)
            if (s0 + j < S) add4(y, q[j]);
    }
    return y;
}
// Row layout of these kernels: a row is processed by a cluster of C CTAs (C = 1: no cluster) of RT
// threads each; CTA c, thread t plays virtual threads vt = c*RT + t + j*C*RT (j < VB / (C*RT)).
struct RowCtx {
    int C, c, RT, VB, nv;
    __device__ RowCtx(int vb) : VB(vb) {
        C = (int)cooperative_groups::this_cluster().num_blocks();
        c = C > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
        RT = blockDim.x;
        nv = VB / (C * RT);
    }
    __device__ int vt(int j) const { return c * RT + (int)threadIdx.x + j * C * RT; }
    __device__ int row() const { return (int)blockIdx.x / C; }
    __device__ void sync() const {
        if (C > 1) cooperative_groups::this_cluster().sync();
        else __syncthreads();
    }
    // value v -> dst[idx] of every CTA of the row's cluster (shared memory)
    template <typename V>
    __device__ void put_all(V* dst, int idx, V v) const {
        if (C == 1) {
            dst[idx] = v;
            return;
        }
        auto cl = cooperative_groups::this_cluster();
        for (int q = 0; q < C; ++q) cl.map_shared_rank(dst, q)[idx] = v;
    }
    template <typename V>
    __device__ void put0(V* dst, int idx, V v) const {  // -> CTA 0 of the cluster
        if (C == 1) dst[idx] = v;
        else cooperative_groups::this_cluster().map_shared_rank(dst, 0)[idx] = v;
    }
};
// Virtual-block reduction (block_sum's tree over VB threads), stage 1: the butterfly of virtual warp
// vt(j)/32 -> red[] in every CTA of the cluster (all lanes call)
__device__ __forceinline__ void vwarp_put(const RowCtx& rc, float v, int j, float* red) {
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) rc.put_all(red, rc.vt(j) >> 5, v);
}
// stage 2 (after rc.sync()): block_sum's final butterfly over the VB/32 virtual-warp partials, evaluated
// by every warp (identical inputs, identical result)
__device__ __forceinline__ float vblock_total(int nvw, const float* red) {
    const int lane = threadIdx.x & 31;
    return warp_sum(lane < nvw ? red[lane] : 0.f);
}
template <typename OT>
__device__ __forceinline__ void store4_op(void* base, long long idx, const float4 v, float s);
template <>
__device__ __forceinline__ void store4_op<float>(void* base, long long idx, const float4 v, float s) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + idx) = make_float4(v.x * s, v.y * s, v.z * s, v.w * s);
}
template <>
__device__ __forceinline__ void store4_op<__nv_bfloat16>(void* base, long long idx, const float4 v, float s) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x * s, v.y * s), hi = __floats2bfloat162_rn(v.z * s, v.w * s);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(base) + idx) = u;
}
// dst row = row * s (the operand-type store of a finished row)
template <typename OT>
__device__ __forceinline__ void store_row4(void* dst, long long base, const float4* row, int d4, float s) {
    for (int i = threadIdx.x; i < d4; i += blockDim.x) store4_op<OT>(dst, base + 4ll * i, row[i], s);
}

template <typename OT>
__global__ void k_x0_rms(const double* __restrict__ emb, const double* __restrict__ ssum, const int* __restrict__ slen,
                         const int* __restrict__ pend, int pstride, const int* __restrict__ row_seq,
                         const int* __restrict__ row_extra, int extra_u, int d, float* __restrict__ x,
                         int* __restrict__ row_plen, void* __restrict__ xa) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float row[];
    __shared__ float red[33];
    const int r = blockIdx.x;
    const int b = row_seq[r];
    const int e = row_extra ? row_extra[r] : extra_u;
    const int n = slen[b] + e;
    const int* toks = pend + (long long)b * pstride;
    float ss = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        double acc = ssum[(long long)b * d + i];
        for (int j = 0; j < e; ++j) acc += emb[(long long)toks[j] * d + i];
        const float v = (float)(acc / (double)n);
        x[(long long)r * d + i] = v;
        row[i] = v;
        ss += v * v;
    }
    if (threadIdx.x == 0) row_plen[r] = n;
    ss = block_sum(ss, red);
    store_row_op<OT>(xa, (long long)r * d, row, d, 1.0f / sqrtf(ss / (float)d + 1e-12f));
}

template <typename OT>
__global__ void __launch_bounds__(1024) k_resid_rms(float* __restrict__ x, const float* __restrict__ P, int S, long long pstride, int d,
                            void* __restrict__ xa) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float4 row4[];
    __shared__ float red[33];
    const RowCtx rc(row_threads(d));
    const long long base = (long long)rc.row() * d;
    const int d4 = d >> 2;
#pragma unroll 1
    for (int j = 0; j < rc.nv; ++j) {
        float ss = 0.f;
        for (int i = rc.vt(j); i < d4; i += rc.VB) {
            float4 v = ld4(x + base + 4ll * i);
            add4(v, sum_splits<8>(P, pstride, S, base + 4ll * i));
            *reinterpret_cast<float4*>(x + base + 4ll * i) = v;
            row4[i] = v;
            ss = __fadd_rn(ss, sumsq4(v));
        }
        vwarp_put(rc, ss, j, red);
    }
    rc.sync();
    const float inv = 1.0f / sqrtf(vblock_total(rc.VB >> 5, red) / (float)d + 1e-12f);
#pragma unroll 1
    for (int j = 0; j < rc.nv; ++j)
        for (int i = rc.vt(j); i < d4; i += rc.VB) store4_op<OT>(xa, base + 4ll * i, row4[i], inv);
}

// ------------------------------------------------------------------ K4/K5 gate + remap
template <typename OT>
__global__ void __launch_bounds__(1024) k_gate(GateArgs a) {
    RK_IN();
    extern __shared__ float sm[];  // [gw[E*d] when staged], xf[d], gl[E], p[E], red[8*32 + 33]
    __shared__ uint64_t gw_bar;
    float* gw = sm;
    const int gw_rows = a.stage_gw == 2 ? (a.E / (gate_threads(a.d, a.E) >> 5)) * (int)(blockDim.x >> 5)
                                        : (a.stage_gw ? a.E : 0);
    float* xf = sm + (size_t)gw_rows * a.d;
    float* gl = xf + a.d;
    float* red = gl + 2 * a.E + 8 * 32;
    // Gate weights staged per CTA: one CTA per row stages all E rows; a row cluster (SMOE_ROW_CLUSTER,
    // one virtual thread per real thread) stages only its CTA's experts -- its virtual warps
    // w0 = c*RT/32 .. +RT/32 own experts w0 + k*nvw, i.e. E/nvw chunks of RT/32 contiguous rows.
    const int gw_wpc = (int)(blockDim.x >> 5), gw_nvw = gate_threads(a.d, a.E) >> 5;
    const int gw_c = a.stage_gw == 2 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
    if (a.stage_gw && threadIdx.x == 0) {
        // the layer's gate weights do not depend on earlier kernels: copy them into shared memory while
        // this block waits for the Mix GEMM (the GEMV then reads shared memory, not four L2 round trips)
        tc::mbar_init(&gw_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t row_b = (uint32_t)a.d * 4;
        const int chunks = a.stage_gw == 2 ? a.E / gw_nvw : 1;
        const uint32_t chunk_b = a.stage_gw == 2 ? (uint32_t)gw_wpc * row_b : (uint32_t)a.E * row_b;
        tc::mbar_expect_tx(&gw_bar, chunk_b * chunks);
        for (int k = 0; k < chunks; ++k) {
            const char* src = reinterpret_cast<const char*>(a.gate_w) +
                              (size_t)(a.stage_gw == 2 ? k * gw_nvw + gw_c * gw_wpc : 0) * row_b;
            char* dst = reinterpret_cast<char*>(gw) + (size_t)k * chunk_b;
            for (uint32_t off = 0; off < chunk_b; off += 32768)
                tc::bulk_g2s(dst + off, src + off, min(32768u, chunk_b - off), &gw_bar);
        }
    }
    pdl_wait();
    pdl_trigger();
    RK_WAITED();
    const RowCtx rc(gate_threads(a.d, a.E));
    const int r = rc.row(), d = a.d, E = a.E, K = a.K, d4 = d >> 2;
    const long long base = (long long)r * d;
    float4* xf4 = reinterpret_cast<float4*>(xf);
    // restricted passes: the draft tables the remap reads per pick (two dependent global loads per pick
    // otherwise) go to shared memory now, next to the row loads below
    int* s_rank = reinterpret_cast<int*>(red + 33);
    int* s_sorted = s_rank + E * a.N;
    uint8_t* s_in = reinterpret_cast<uint8_t*>(s_sorted + a.N);
    if (a.in_draft) {
        for (int i = threadIdx.x; i < E * a.N; i += blockDim.x) s_rank[i] = a.rank[i];
        for (int i = threadIdx.x; i < a.N; i += blockDim.x) s_sorted[i] = a.draft_sorted[i];
        for (int i = threadIdx.x; i < E; i += blockDim.x) s_in[i] = a.in_draft[i];
    }
    // residual add of the mix GEMM's split-K partials (model.cpp:224), then rms (model.cpp:226)
#pragma unroll 1
    for (int j = 0; j < rc.nv; ++j) {
        float ss = 0.f;
        for (int i = rc.vt(j); i < d4; i += rc.VB) {
            float4 v = ld4(a.x + base + 4ll * i);
            add4(v, sum_splits<4>(a.pmix, a.pstride, a.s_mix, base + 4ll * i));
            *reinterpret_cast<float4*>(a.x + base + 4ll * i) = v;
            xf4[i] = v;
            ss = __fadd_rn(ss, sumsq4(v));
        }
        vwarp_put(rc, ss, j, red);
    }
    rc.sync();
    const float inv = 1.0f / sqrtf(vblock_total(rc.VB >> 5, red) / (float)d + 1e-12f);
    RK_MARK(0);
    // the normalised row, whole, in every CTA of the cluster
#pragma unroll 1
    for (int j = 0; j < rc.nv; ++j)
        for (int i = rc.vt(j); i < d4; i += rc.VB) {
            const float4 v = xf4[i];
            rc.put_all(xf4, i, make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv));
        }
    rc.sync();
    // gate GEMV (model.cpp:229-230): virtual warp vw owns experts vw, vw + VB/32, ...; each lane strides
    // d in float4s (fixed order, then a butterfly), so every row's logits are computed identically in
    // any pass.  The logits are gathered in CTA 0 of the cluster.
    const int lane = threadIdx.x & 31, nvw = rc.VB >> 5;
    if (a.stage_gw) tc::mbar_wait(&gw_bar, 0);
    const float* gsrc = a.stage_gw ? gw : a.gate_w;
#pragma unroll 1
    for (int j = 0; j < rc.nv; ++j) {
        for (int e = rc.vt(j) >> 5; e < E; e += nvw) {
            // staged per cluster CTA: chunk e / nvw, row e % nvw - c*wpc within it
            const long long gr = a.stage_gw == 2 ? (long long)(e / gw_nvw) * gw_wpc + (e % gw_nvw - gw_c * gw_wpc) : e;
            const float4* g = reinterpret_cast<const float4*>(gsrc + gr * d);
            float acc = 0.f;
#pragma unroll 8
            for (int i = lane; i < d4; i += 32) {
                acc = __fadd_rn(acc, dot4f(g[i], xf4[i]));
            }
            acc = warp_sum(acc);
            if (lane == 0) rc.put0(gl, e, acc + a.gate_b[e]);
        }
    }
    rc.sync();
    RK_MARK(1);
    if (rc.c != 0) return;  // CTA 0 selects and dispatches the row
    // ---- selection on warp 0 (E <= 64: lane l holds experts l and l+32)
    __shared__ int dst[16];
    if (threadIdx.x < 32) {
        gate_select_warp(a, r, gl, dst, s_rank, s_sorted, a.in_draft ? s_in : nullptr);
    }
    __syncthreads();
    RK_MARK(2);
    const int sg = a.seg > 0 ? a.seg : a.T;
    for (int k = 0; k < K; ++k) {
        void* base = a.xperm;
        long long row = dst[k];
        if (a.peer_x) {  // fused EP dispatch over peer memory
            const int e = (int)(row / sg);
            base = a.peer_x[e / a.ep_eo];
            row = (long long)(a.ep_me * a.ep_eo + e % a.ep_eo) * sg + (row - (long long)e * sg);
        }
        store_row4<OT>(base, row * d, xf4, d4, 1.0f);
    }
    if (a.peer_x) __threadfence_system();
    RK_END(1);
}

// ---- K4/K5 gate, row-group form for many experts (C4: E=64, 512 KB of f32 gate weights).  k_gate reads
// all E x d weights once per row (from L2: one SM pulls 512 KB per row, the GEMV's bound); here a
// cluster of kGateRG CTAs takes kGateRG rows and CTA c owns row c (residual + rms, selection,
// dispatch) and experts [c*E/kGateRG, (c+1)*E/kGateRG) of every row of the cluster, so the weights
// are read once per cluster.  Every reduction is k_gate's: the row tree over VB virtual threads (each
// of the RT real threads plays VB/RT of them) and, per (row, expert), the lane-strided float4 chain +
// butterfly -- a row's logits and picks are bit-identical to k_gate's.
constexpr int kGateRG = 8;

template <typename OT>
__global__ void __launch_bounds__(512, 1) k_gate_rg(GateArgs a) {
    RK_IN();
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ float4 sm4[];
    __shared__ uint64_t gw_bar;
    __shared__ float red[33];
    __shared__ int dst[16];
    const int d = a.d, d4 = d >> 2, E = a.E, K = a.K, Ec = E / kGateRG;
    const int c = (int)cl.block_rank();
    const int row0 = (int)(blockIdx.x / kGateRG) * kGateRG;
    const int nrows = min(kGateRG, a.T - row0);
    const int r = row0 + c;
    float4* gw4 = sm4;                                               // [Ec][d4] when staged
    float4* xall = gw4 + (a.stage_gw ? (size_t)Ec * d4 : 0);         // [kGateRG][d4] the cluster's rows
    float* gl = reinterpret_cast<float*>(xall + (size_t)kGateRG * d4);  // [2E] own row's logits + scratch
    int* s_rank = reinterpret_cast<int*>(gl + 2 * E);
    int* s_sorted = s_rank + E * a.N;
    uint8_t* s_in = reinterpret_cast<uint8_t*>(s_sorted + a.N);
    if (a.stage_gw && threadIdx.x == 0) {  // this CTA's expert rows: independent of the Mix, fetched now
        tc::mbar_init(&gw_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t bytes = (uint32_t)Ec * d * 4;
        tc::mbar_expect_tx(&gw_bar, bytes);
        const char* src = reinterpret_cast<const char*>(a.gate_w + (size_t)c * Ec * d);
        for (uint32_t off = 0; off < bytes; off += 32768)
            tc::bulk_g2s(reinterpret_cast<char*>(gw4) + off, src + off, min(32768u, bytes - off), &gw_bar);
    }
    cl.sync();  // every CTA of the cluster is running before any writes into its shared memory
    pdl_wait();
    pdl_trigger();
    RK_WAITED();
    if (a.in_draft) {
        for (int i = threadIdx.x; i < E * a.N; i += blockDim.x) s_rank[i] = a.rank[i];
        for (int i = threadIdx.x; i < a.N; i += blockDim.x) s_sorted[i] = a.draft_sorted[i];
        for (int i = threadIdx.x; i < E; i += blockDim.x) s_in[i] = a.in_draft[i];
    }
    const int VB = gate_threads(d, E), RT = blockDim.x, nv = VB / RT;
    const long long base = (long long)r * d;
    float4* own = xall + (size_t)c * d4;
    if (c < nrows) {
        // residual add of the mix partials + rms (k_gate's tree: virtual thread vt = t + j*RT)
#pragma unroll 1
        for (int j = 0; j < nv; ++j) {
            float ss = 0.f;
            for (int i = (int)threadIdx.x + j * RT; i < d4; i += VB) {
                float4 v = ld4(a.x + base + 4ll * i);
                add4(v, sum_splits<8>(a.pmix, a.pstride, a.s_mix, base + 4ll * i));
                *reinterpret_cast<float4*>(a.x + base + 4ll * i) = v;
                own[i] = v;
                ss = __fadd_rn(ss, sumsq4(v));
            }
            ss = warp_sum(ss);
            if ((threadIdx.x & 31) == 0) red[((int)threadIdx.x + j * RT) >> 5] = ss;
        }
        __syncthreads();
        const float inv = 1.0f / sqrtf(vblock_total(VB >> 5, red) / (float)d + 1e-12f);
        RK_MARK(0);
        // the normalised row into slot c of every CTA of the cluster (each computes its experts for all rows)
#pragma unroll 1
        for (int i = threadIdx.x; i < d4; i += RT) {
            const float4 v = own[i];
            const float4 xn = make_float4(v.x * inv, v.y * inv, v.z * inv, v.w * inv);
#pragma unroll
            for (int q = 0; q < kGateRG; ++q) cl.map_shared_rank(xall, q)[(size_t)c * d4 + i] = xn;
        }
    }
    cl.sync();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = RT >> 5;
    if (a.stage_gw) tc::mbar_wait(&gw_bar, 0);
    // GEMV: warp w takes expert c*Ec + w % Ec for rows w / Ec, + rstep, ... four rows per weight load
    const int rstep = max(1, nw / Ec);
#pragma unroll 1
    for (int task = w; task < Ec * rstep; task += nw) {
        const int el = task % Ec, e = c * Ec + el;
        const float4* g = a.stage_gw ? gw4 + (size_t)el * d4 : reinterpret_cast<const float4*>(a.gate_w + (size_t)e * d);
#pragma unroll 1
        for (int qb = task / Ec; qb < nrows; qb += 4 * rstep) {
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            const float4* x0 = xall + (size_t)qb * d4;
            const int nq = min(4, (nrows - qb + rstep - 1) / rstep);
            if (nq == 4) {
#pragma unroll 4
                for (int i = lane; i < d4; i += 32) {
                    const float4 gv = g[i];
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[k] = __fadd_rn(acc[k], dot4f(gv, x0[(size_t)k * rstep * d4 + i]));
                }
            } else {
                for (int i = lane; i < d4; i += 32) {
                    const float4 gv = g[i];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k < nq) acc[k] = __fadd_rn(acc[k], dot4f(gv, x0[(size_t)k * rstep * d4 + i]));
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float v = warp_sum(acc[k]);
                if (k < nq && lane == 0) cl.map_shared_rank(gl, qb + k * rstep)[e] = v + a.gate_b[e];
            }
        }
    }
    cl.sync();
    RK_MARK(1);
    if (c >= nrows) return;
    if (threadIdx.x < 32) {
        gate_select_warp(a, r, gl, dst, s_rank, s_sorted, a.in_draft ? s_in : nullptr);
    }
    __syncthreads();
    RK_MARK(2);
    const int sg = a.seg > 0 ? a.seg : a.T;
    for (int k = 0; k < K; ++k) {
        void* obase = a.xperm;
        long long row = dst[k];
        if (a.peer_x) {  // fused EP dispatch over peer memory (as k_gate)
            const int e = (int)(row / sg);
            obase = a.peer_x[e / a.ep_eo];
            row = (long long)(a.ep_me * a.ep_eo + e % a.ep_eo) * sg + (row - (long long)e * sg);
        }
        store_row4<OT>(obase, row * d, own, d4, 1.0f);
    }
    if (a.peer_x) __threadfence_system();
    RK_END(1);
}

// ------------------------------------------------------------------ K9 combine (+ next rms)
template <typename OT>
__global__ void __launch_bounds__(1024) k_combine_rms(float* __restrict__ x, const float* __restrict__ P, int S, long long pstride,
                              const int* __restrict__ pos, const float* __restrict__ wgt, int K, int d, int dense,
                              void* __restrict__ xa) {
    RK_IN();
    pdl_wait();
    pdl_trigger();
    RK_WAITED();
    extern __shared__ float4 row4[];
    __shared__ float red[33];
    __shared__ long long src_s[16];
    __shared__ float w_s[16];
    const RowCtx rc(row_threads(d));
    const int t = rc.row(), d4 = d >> 2;
    const int nk = dense ? 1 : K;
    const long long base = (long long)t * d;
    if (threadIdx.x < nk) {  // the K picks' partial rows and weights, read once per block
        const int k = threadIdx.x;
        src_s[k] = (dense ? (long long)t : pos ? (long long)pos[t * K + k] : (long long)t * K + k) * d;
        w_s[k] = dense ? 1.f : wgt[t * K + k];
    }
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < rc.nv; ++j) {
        float ss = 0.f;
        for (int i = rc.vt(j); i < d4; i += rc.VB) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int k = 0; k < nk; ++k) {
                const float4 y = sum_splits<4>(P, pstride, S, src_s[k] + 4ll * i);
                if (dense) acc = y;
                else axpy4(acc, w_s[k], y);
            }
            float4 v = ld4(x + base + 4ll * i);
            add4(v, acc);
            *reinterpret_cast<float4*>(x + base + 4ll * i) = v;
            row4[i] = v;
            ss = __fadd_rn(ss, sumsq4(v));
        }
        vwarp_put(rc, ss, j, red);
    }
    rc.sync();
    const float inv = 1.0f / sqrtf(vblock_total(rc.VB >> 5, red) / (float)d + 1e-12f);
#pragma unroll 1
    for (int j = 0; j < rc.nv; ++j)
        for (int i = rc.vt(j); i < d4; i += rc.VB) store4_op<OT>(xa, base + 4ll * i, row4[i], inv);
    RK_END(2);
}

// ------------------------------------------------------------------ K10 argmax
__global__ void k_argmax(const float* __restrict__ lg, int V, int* __restrict__ out, int* flags) {
    pdl_wait();
    pdl_trigger();
    __shared__ float sv[32];
    __shared__ int si[32];
    const float* row = lg + (long long)blockIdx.x * V;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    bool fin = true;
    // (value, -index) is a total order, so the scan order does not matter: first max wins
    auto upd = [&](float v, int i) {
        fin &= isfinite(v);
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    };
    if ((V & 3) == 0) {  // 16-byte rows: float4 loads, four in flight per thread (was one dependent load per step)
        const float4* r4 = reinterpret_cast<const float4*>(row);
#pragma unroll 4
        for (int i = threadIdx.x; i < (V >> 2); i += blockDim.x) {
            const float4 q = r4[i];
            upd(q.x, 4 * i);
            upd(q.y, 4 * i + 1);
            upd(q.z, 4 * i + 2);
            upd(q.w, 4 * i + 3);
        }
    } else {
        for (int i = threadIdx.x; i < V; i += blockDim.x) upd(row[i], i);
    }
    if (!fin) atomicOr(flags, kFlagNonFiniteLogits);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) { sv[w] = bv; si[w] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 1; j < (int)(blockDim.x >> 5); ++j)
            if (sv[j] > bv || (sv[j] == bv && si[j] < bi)) { bv = sv[j]; bi = si[j]; }
        out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
    }
}

__global__ void k_scatter_tokens(const int* src, const int* row_seq, const int* row_extra, int extra_u, int T,
                                 int* dst, int stride) {
    pdl_wait();
    pdl_trigger();
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= T) return;
    int e = row_extra ? row_extra[r] : extra_u;
    dst[(long long)row_seq[r] * stride + e] = src[r];
}

__global__ void k_accept(const int* drafts, const int* vam, const int* seqs, int na, int gamma, int stride, int* acc,
                         int* corr) {
    pdl_wait();
    pdl_trigger();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= na) return;
    const int b = seqs[i];
    const int* dr = drafts + (long long)b * stride;
    const int* am = vam + (long long)b * stride;
    int a = 0;
    while (a < gamma && dr[a] == am[a]) ++a;
    acc[i] = a;
    corr[i] = am[a];
}

__global__ void k_commit(double* ssum, int* slen, const double* emb, const int* seqs, const int* toks, int tstride,
                         const int* take, int d, int* last_tok) {
    pdl_wait();
    pdl_trigger();
    const int j = blockIdx.x;
    const int b = seqs[j];
    const int n = take[j];
#pragma unroll 4
    for (int i = threadIdx.x; i < d; i += blockDim.x) {  // columns independent; per column in token order
        double s = ssum[(long long)b * d + i];
        for (int t = 0; t < n; ++t) s += emb[(long long)toks[(long long)j * tstride + t] * d + i];
        ssum[(long long)b * d + i] = s;
    }
    if (threadIdx.x == 0) {
        slen[b] += n;
        if (last_tok && n > 0) last_tok[b] = toks[(long long)j * tstride + n - 1];  // attention models' next input
    }
}

// ------------------------------------------------------------------ init / conversion
__device__ __forceinline__ double normal_at(uint64_t seed, uint64_t tid, long long i) {
    uint64_t h = splitmix64(seed ^ splitmix64(tid * 0x9E3779B97F4A7C15ull + (uint64_t)i));
    uint64_t h2 = splitmix64(h ^ 0xD1B54A32D192ED03ull);
    double u1 = ((double)(h >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    double u2 = (double)(h2 >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

template <typename T>
__global__ void k_fill_normal(T* dst, long long n, double sd, uint64_t seed, uint64_t tid, long long idx0, int tile_k) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[tile_k ? tiled_index(i / tile_k, i % tile_k, tile_k) : i] = from_f<T>((float)(sd * normal_at(seed, tid, idx0 + i)));
}
__global__ void k_fill_normal_f64(double* dst, long long n, double sd, uint64_t seed, uint64_t tid) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = sd * normal_at(seed, tid, i);
}

template <typename T>
__global__ void k_convert_transpose(const double* __restrict__ src, int rows, int cols, T* __restrict__ dst, int mul,
                                    int off, int tiled) {
    __shared__ double tile[32][33];
    int c = blockIdx.x * 32 + threadIdx.x;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int r = blockIdx.y * 32 + j;
        if (r < rows && c < cols) tile[j][threadIdx.x] = src[(long long)r * cols + c];
    }
    __syncthreads();
    int r = blockIdx.y * 32 + threadIdx.x;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int cc = blockIdx.x * 32 + j;
        if (r < rows && cc < cols) {
            const long long orow = (long long)cc * mul + off;
            dst[tiled ? tiled_index(orow, r, rows) : orow * rows + r] = from_f<T>((float)tile[threadIdx.x][j]);
        }
    }
}
template <typename T>
__global__ void k_convert(const double* __restrict__ src, long long n, T* __restrict__ dst, int tile_k, long long row0) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[tile_k ? tiled_index(row0 + i / tile_k, i % tile_k, tile_k) : i] = from_f<T>((float)src[i]);
}

template <typename T>
__global__ void k_pair_sqdist(const T* __restrict__ pool, long long stride, long long n, const int* __restrict__ slots,
                              int E, double* __restrict__ out) {
    // blockIdx.x = pair (i,j) with i<j enumerated row-major; blockIdx.y = chunk
    int p = blockIdx.x, i = 0;
    while (p >= E - 1 - i) { p -= E - 1 - i; ++i; }
    const int j = i + 1 + p;
    const T* a = pool + (long long)slots[i] * stride;
    const T* b = pool + (long long)slots[j] * stride;
    const long long per = (n + gridDim.y - 1) / gridDim.y;
    const long long s0 = per * blockIdx.y, s1 = min(n, s0 + per);
    double acc = 0.0;
    for (long long k = s0 + threadIdx.x; k < s1; k += blockDim.x) {
        double df = (double)to_f<T>(a[k]) - (double)to_f<T>(b[k]);
        acc += df * df;
    }
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        out[((long long)i * E + j) * gridDim.y + blockIdx.y] += t;
    }
}

}  // namespace

void launch_x0(const double* emb64, const double* seq_sum, const int* seq_len, const int* pend, int pend_stride,
               const int* row_seq, const int* row_extra, int extra_uniform, int T, int d, float* x, int* row_plen,
               cudaStream_t s) {
    if (T <= 0) return;
    k_x0<<<T, 128, 0, s>>>(emb64, seq_sum, seq_len, pend, pend_stride, row_seq, row_extra, extra_uniform, d, x,
                           row_plen);
}


void launch_x0_rms(const double* emb64, const double* seq_sum, const int* seq_len, const int* pend, int pend_stride,
                   const int* row_seq, const int* row_extra, int extra_uniform, int T, int d, float* x, int* row_plen,
                   void* xa, WType op, cudaStream_t s) {
    if (T <= 0) return;
    const size_t sm = sizeof(float) * d;
    if (op == kF32)
        launch_k(k_x0_rms<float>, T, row_threads(d), sm, s, emb64, seq_sum, seq_len, pend, pend_stride, row_seq,
                 row_extra, extra_uniform, d, x, row_plen, xa);
    else
        launch_k(k_x0_rms<__nv_bfloat16>, T, row_threads(d), sm, s, emb64, seq_sum, seq_len, pend, pend_stride,
                 row_seq, row_extra, extra_uniform, d, x, row_plen, xa);
}

void launch_resid_rms(float* x, const float* P, int S, long long pstride, int T, int d, void* xa, WType op,
                      cudaStream_t s) {
    if (T <= 0) return;
    const size_t sm = sizeof(float) * d;
    const RowShape rs = row_shape(row_threads(d));
    if (op == kF32) launch_kc(k_resid_rms<float>, T * rs.C, rs.RT, sm, s, rs.C, x, P, S, pstride, d, xa);
    else launch_kc(k_resid_rms<__nv_bfloat16>, T * rs.C, rs.RT, sm, s, rs.C, x, P, S, pstride, d, xa);
}

void launch_rms(const float* x, int T, int d, void* xa, WType op, cudaStream_t s) {
    if (T <= 0) return;
    if (op == kF32) k_rms<float><<<T, 256, 0, s>>>(x, d, xa);
    else k_rms<__nv_bfloat16><<<T, 256, 0, s>>>(x, d, xa);
}

void launch_gate(const GateArgs& a0, cudaStream_t s) {
    if (a0.T <= 0) return;
    GateArgs a = a0;
    static const int rg_env = [] {  // SMOE_GATE_RG: 0 off, 1 many-expert gates (default), 2 every gate
        const char* v = std::getenv("SMOE_GATE_RG");
        return v ? std::atoi(v) : 1;
    }();
    if (rg_env && (a.E > 16 || rg_env == 2) && a.E % kGateRG == 0 && a.E <= 64 && a.K <= 16 && a.d % 4 == 0 &&
        (reinterpret_cast<uintptr_t>(a.gate_w) & 15) == 0) {
        const int clusters = (a.T + kGateRG - 1) / kGateRG;
        // staged expert rows hold one CTA per SM: only when the pass's CTAs fit in one wave; otherwise
        // 256-thread CTAs, two per SM, read their expert rows from L2
        a.stage_gw = clusters * kGateRG <= tc::sm_count() ? 1 : 0;
        const int vb = gate_threads(a.d, a.E), rt = std::min(a.stage_gw ? 512 : 256, vb);
        const size_t smem = sizeof(float4) * ((size_t)(a.stage_gw ? a.E / kGateRG : 0) + kGateRG) * (a.d / 4) +
                            sizeof(float) * 2 * a.E + (a.in_draft ? sizeof(int) * ((size_t)a.E * a.N + a.N) + a.E : 0);
        static std::atomic<uint64_t> configured_rg{0};
        if (first_use_on_device(configured_rg)) {
            SMOE_CUDA(cudaFuncSetAttribute(k_gate_rg<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            SMOE_CUDA(cudaFuncSetAttribute(k_gate_rg<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        }
        if (smem <= 200 * 1024 && vb % rt == 0) {
            if (a.op == kF32) launch_kc(k_gate_rg<float>, clusters * kGateRG, rt, smem, s, kGateRG, a);
            else launch_kc(k_gate_rg<__nv_bfloat16>, clusters * kGateRG, rt, smem, s, kGateRG, a);
            return;
        }
        a.stage_gw = 0;
    }
    static const bool stage_env = [] {
        const char* v = std::getenv("SMOE_GATE_STAGE");
        return !(v && v[0] == '0');
    }();
    // stage the gate weights (E x d f32) in shared memory when they fit beside one row (C2: 128 KB); a row
    // cluster with one virtual thread per real thread stages only each CTA's experts (C4: 128 KB of 512)
    // (wide row blocks only with few experts: the GEMV's virtual warps per expert shrink to a quarter)
    const RowShape rs0 = row_shape(gate_threads(a.d, a.E), a.E <= 16 ? a.T : 0);
    const int vb = gate_threads(a.d, a.E), nvw = vb >> 5;
    const bool per_cta = rs0.C > 1 && rs0.C * rs0.RT == vb && a.E % nvw == 0;
    const size_t gw_bytes = sizeof(float) * (size_t)(per_cta ? (rs0.RT >> 5) * (a.E / nvw) : a.E) * a.d;
    // wide passes read the gate weights from L2 (a staged copy per block would hold one block per SM again)
    const bool wide = rs0.C == 1 && rs0.RT < vb && a.T > tc::sm_count();
    a.stage_gw = stage_env && !wide && gw_bytes <= 160 * 1024 && (reinterpret_cast<uintptr_t>(a.gate_w) & 15) == 0
                     ? (per_cta ? 2 : 1) : 0;
    size_t smem = sizeof(float) * (a.d + 2 * a.E + 8 * 32 + 33) + (a.stage_gw ? gw_bytes : 0) +
                  (a.in_draft ? sizeof(int) * ((size_t)a.E * a.N + a.N) + a.E : 0);
    static std::atomic<uint64_t> configured{0};
    if (first_use_on_device(configured)) {
        SMOE_CUDA(cudaFuncSetAttribute(k_gate<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        SMOE_CUDA(cudaFuncSetAttribute(k_gate<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    }
    const RowShape rs = rs0;  // a row per cluster, a (virtual) warp per expert
    if (a.op == kF32) launch_kc(k_gate<float>, a.T * rs.C, rs.RT, smem, s, rs.C, a);
    else launch_kc(k_gate<__nv_bfloat16>, a.T * rs.C, rs.RT, smem, s, rs.C, a);
}


void launch_combine_rms(float* x, const float* P, int S, long long pstride, const int* pos, const float* wgt, int T,
                        int K, int d, int dense, void* xa, WType op, cudaStream_t s) {
    if (T <= 0) return;
    const size_t sm = sizeof(float) * d;
    const RowShape rs = row_shape(row_threads(d));  // (wide blocks measured no faster for the combine)
    if (op == kF32)
        launch_kc(k_combine_rms<float>, T * rs.C, rs.RT, sm, s, rs.C, x, P, S, pstride, pos, wgt, K, d, dense, xa);
    else
        launch_kc(k_combine_rms<__nv_bfloat16>, T * rs.C, rs.RT, sm, s, rs.C, x, P, S, pstride, pos, wgt, K, d, dense,
                  xa);
}

void launch_argmax(const float* logits, int T, int V, int* out, int* flags, cudaStream_t s) {
    if (T <= 0) return;
    launch_k(k_argmax, T, 512, 0, s, logits, V, out, flags);
}

void launch_scatter_tokens(const int* src, const int* row_seq, const int* row_extra, int extra_uniform, int T, int* dst,
                           int stride, cudaStream_t s) {
    if (T <= 0) return;
    launch_k(k_scatter_tokens, ceil_div(T, 128), 128, 0, s, src, row_seq, row_extra, extra_uniform, T, dst, stride);
}

void launch_accept(const int* drafts, const int* vam, const int* seqs, int na, int gamma, int stride, int* acc,
                   int* corr, cudaStream_t s) {
    if (na <= 0) return;
    launch_k(k_accept, ceil_div(na, 128), 128, 0, s, drafts, vam, seqs, na, gamma, stride, acc, corr);
}

void launch_commit(double* seq_sum, int* seq_len, const double* emb64, const int* seqs, const int* toks,
                   int tok_stride, const int* take, int na, int d, cudaStream_t s, int* last_tok) {
    if (na <= 0) return;
    launch_k(k_commit, na, 1024, 0, s, seq_sum, seq_len, emb64, seqs, toks, tok_stride, take, d, last_tok);
}

void launch_fill_normal(void* dst, WType t, long long n, double stddev, uint64_t seed, uint64_t tensor_id,
                        cudaStream_t s, long long index0, int tile_k) {
    int grid = (int)std::min<long long>(148LL * 16, (n + 255) / 256);
    if (grid <= 0) return;
    if (t == kF32) k_fill_normal<float><<<grid, 256, 0, s>>>((float*)dst, n, stddev, seed, tensor_id, index0, tile_k);
    else k_fill_normal<__nv_bfloat16><<<grid, 256, 0, s>>>((__nv_bfloat16*)dst, n, stddev, seed, tensor_id, index0, tile_k);
}
void launch_fill_normal_f64(double* dst, long long n, double stddev, uint64_t seed, uint64_t tensor_id,
                            cudaStream_t s) {
    int grid = (int)std::min<long long>(148LL * 16, (n + 255) / 256);
    if (grid <= 0) return;
    k_fill_normal_f64<<<grid, 256, 0, s>>>(dst, n, stddev, seed, tensor_id);
}

void launch_convert_transpose(const double* src, int rows, int cols, void* dst, WType t, cudaStream_t s, int mul,
                              int off, bool tiled) {
    dim3 grid(ceil_div(cols, 32), ceil_div(rows, 32)), block(32, 8);
    if (t == kF32) k_convert_transpose<float><<<grid, block, 0, s>>>(src, rows, cols, (float*)dst, mul, off, (int)tiled);
    else k_convert_transpose<__nv_bfloat16><<<grid, block, 0, s>>>(src, rows, cols, (__nv_bfloat16*)dst, mul, off, (int)tiled);
}
void launch_convert(const double* src, long long n, void* dst, WType t, cudaStream_t s, int tile_k, long long row0) {
    int grid = (int)std::min<long long>(148LL * 16, (n + 255) / 256);
    if (grid <= 0) return;
    if (t == kF32) k_convert<float><<<grid, 256, 0, s>>>(src, n, (float*)dst, tile_k, row0);
    else k_convert<__nv_bfloat16><<<grid, 256, 0, s>>>(src, n, (__nv_bfloat16*)dst, tile_k, row0);
}
void launch_cast_f64_to_f32(const double* src, long long n, float* dst, cudaStream_t s) {
    launch_convert(src, n, dst, kF32, s);
}

void launch_pairwise_sqdist(const void* pool, WType t, long long slot_stride, long long n, const int* slots, int E,
                            double* out, cudaStream_t s) {
    if (E < 2) return;
    dim3 grid(E * (E - 1) / 2, kPairChunks);
    if (t == kF32)
        k_pair_sqdist<float><<<grid, 512, 0, s>>>((const float*)pool, slot_stride, n, slots, E, out);
    else
        k_pair_sqdist<__nv_bfloat16><<<grid, 512, 0, s>>>((const __nv_bfloat16*)pool, slot_stride, n, slots, E, out);
}

// Draft rank tables (engine.cpp set_draft_sets): thread (m, r) orders layer m's draft members by
// (affinity distance to raw expert r, index) -- a stable insertion sort of the ascending member list,
// the same total order the host's stable_sort used (drafting.cpp:123-138 nearest_draft_expert).
__global__ void k_rank_tables(const double* __restrict__ aff, const int* __restrict__ sorted, int M, int E, int nmax,
                              int* __restrict__ rank) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M * E) return;
    const int m = i / E;
    const int* srt = sorted + (size_t)m * E;
    const double* D = aff ? aff + (size_t)i * E : nullptr;
    int* o = rank + (size_t)i * nmax;
    int n = 0;
    for (int j = 0; j < nmax; ++j) {
        const int v = srt[j];
        if (v < 0) {
            o[j] = -1;
            continue;
        }
        int q = n++;
        if (D) {
            const double dv = D[v];
            while (q > 0) {
                const int u = o[q - 1];
                const double du = D[u];
                if (du < dv || (du == dv && u <= v)) break;
                o[q] = u;
                --q;
            }
        }
        o[q] = v;
    }
}

void launch_rank_tables(const double* aff, const int* sorted, int M, int E, int nmax, int* rank, cudaStream_t s) {
    const int n = M * E;
    if (n == 0 || nmax == 0) return;
    k_rank_tables<<<(n + 127) / 128, 128, 0, s>>>(aff, sorted, M, E, nmax, rank);
}

}  // namespace smoe

extern "C" int smoe_rk_trace_dump(const char* path) {
#ifdef SMOE_TC_TRACE
    using namespace smoe;
    std::vector<RkRec> r(kRkRing);
    unsigned n = 0;
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    cudaMemcpyFromSymbol(r.data(), g_rk, r.size() * sizeof(RkRec));
    cudaMemcpyFromSymbol(&n, g_rk_n, sizeof(n));
    FILE* fp = fopen(path, "wb");
    if (!fp) return -3;
    const int cnt = (int)std::min<unsigned>(n, kRkRing);
    fwrite(&cnt, sizeof(int), 1, fp);
    fwrite(r.data(), sizeof(RkRec), cnt, fp);
    fclose(fp);
    return 0;
#else
    (void)path;
    return -1;
#endif
}
