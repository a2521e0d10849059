// pass_tc.cu -- the whole forward pass (every layer of model.cpp:221-258 for T rows) as ONE persistent
// tcgen05 kernel: one CTA per SM, weights streamed by TMA, accumulators in TMEM.
//
// Per layer l the pass has four dependent phases; their work items are claimed dynamically by the CTAs
// and ordered by per-layer device counters instead of kernel boundaries:
//   A  mix GEMM units        pmix[s] = Mix_l . xa  (split-K partials)              (model.cpp:222-224)
//   B  row tasks             MoE layer: x += sum_s pmix[s]; rms; gate GEMV + bias; softmax; top-K;
//                            restricted remap; dispatch into the experts' segments of xperm
//                            (model.cpp:226-246, drafting.cpp:123-151); dense layer: x += ...; xa = rms(x)
//   C  expert FFN units      grouped up (tanh | SwiGLU) then down (f32 split partials), a down unit of
//                            expert g loads H once g's up units have published       (model.cpp:248)
//   D  row tasks             x += sum_k p[raw_k] y_k; xa = rms(x) for the next layer (model.cpp:249-257)
// Roles inside a CTA (192 threads) are those of gemm_tc.cu: warp 0 = scheduler + TMA producer, warp 1 =
// TMEM owner + MMA issuer, warps 2-5 = epilogue AND row-task workers.  The producer publishes GEMM units
// and two markers per layer (B, D) through a ring; the workers run the epilogues in ring order and, at a
// marker, join that layer's row tasks once the phase before it is complete everywhere.
//
// What the fusion buys (profiles/r02_*): the weight stream never stops at a layer boundary.  While the
// workers finish layer l's combine rows, the producer is already streaming layer l+1's Mix weights into
// the ring (its activation boxes are held back until layer l's D phase has published); the gate no
// longer costs a launch plus a ramp of every MoE kernel; 4 launches per layer become 1 per pass.
//
// Ordering: every cross-CTA hand-off is "stores; __threadfence; fence.proxy.async (if TMA reads it);
// counter += 1" on the writer side and "ld.acquire counter; fence.proxy.async" on the reader side.
// Counters are per pass and self-resetting (the last CTA out zeroes them); nothing is claimed before
// griddepcontrol.wait, so a pass kernel launched early under PDL never touches the previous pass's
// counters.  Results are batch invariant: every row task is computed by 128 threads in a fixed order
// and GEMM columns never depend on other columns.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gate_dev.cuh"
#include "tc_common.cuh"

namespace smoe {
namespace {
using namespace tc;

constexpr int kMaxLayers = 128;
constexpr int kCtr = 8 + kMaxGroups;  // per-layer counters
enum : int { cClaimA = 0, cClaimC, cClaimB, cClaimD, cDoneA, cDoneB, cDoneC, cDoneD, cUp };
enum : int { kEnd = -1, kA = 0, kC = 1, kMarkB = 2, kMarkD = 3 };
constexpr int kWorkers = 128;  // warps 2..5
constexpr int kMaxE = 64;

struct PassParams {
    int T, d, E, K, L, U;
    int pf;                     // L2 prefetch bits: 1 = next layer's Mix tiles, 2 = next gate weights
    int n_tiles;                // token tiles of BN_MAX rows
    int stages, b_region;
    Phase mix, up, down;
    short lay_mo[kMaxLayers];   // MoE ordinal or -1
    short lay_slot[kMaxLayers]; // dense FFN slot (dense layers)
    float* x;
    const float* pmix;
    int s_mix;
    long long pm_stride;
    const float* ybuf;
    int s_down;
    long long yd_stride;
    __nv_bfloat16* xa;
    __nv_bfloat16* xperm;
    const float* gate_w;
    const float* gate_b;
    int* grp_cnt;               // [M][E]
    const int* slot_of;         // [M][E]
    int* pos;
    float* wgt;
    int* raw_log;               // [M][Tmax][K] of this pass's log slot
    int* fin_log;
    long long log_stride;       // Tmax*K
    const uint8_t* in_draft;    // [M][E] or nullptr (target semantics)
    const int* draft_sorted;    // [M][E]
    const int* rank;            // [M][E][rank_n]
    int rank_n, N, use_aff;
    const int* row_plen;
    int* flags;
    int* ctr;                   // [L][kCtr] + exit counter
};

struct RingItem {
    int kind, layer;
    Unit w;
};

// Worker scratch: the stage ring, which is idle during the B and D row phases (the producer streams
// nothing between publishing a B / D marker and that phase's completion), filled by 1D bulk copies.
struct Scratch {
    uint8_t* base;
    uint32_t bytes;
    uint64_t* mb;  // completion barrier (one arrival + tx bytes per fill)
    int phase;     // parity of the next fill (tracked identically by all workers)
};

struct RowSmem {
    uint64_t mb;  // scratch fill barrier
    float vred[32];  // per-virtual-warp partials (vblock_sum)
    float red[4][kMaxE];
    float gl[2 * kMaxE];
    float ss[4];
    int dst[32];
};

#ifdef SMOE_PASS_TRACE
// Phase timeline of the last pass (tools/pass_trace.py): per CTA, per layer, 8 globaltimer stamps:
// 0 producer enters layer, 1 producer sees B done, 2 producer out of C claims, 3 workers see A done,
// 4 workers leave B rows, 5 workers see C done, 6 workers leave D rows, 7 workers reach marker D.
__device__ long long g_ptr_ev[160][kMaxLayers][24];
__device__ __forceinline__ void pev(int l, int k) {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_ptr_ev[blockIdx.x % 160][l][k] = t;
}
#define PEV(l, k) pev(l, k)
#else
#define PEV(l, k)
#endif

__device__ __forceinline__ int* lctr(const PassParams& p, int l) { return p.ctr + (size_t)l * kCtr; }

__device__ __forceinline__ void wbar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// ---- unit geometry
// first Mix unit statically owned by CTA b (unit u belongs to CTA (u + T) % grid)
__device__ __forceinline__ int a_first(const PassParams& p, int b) {
    const int g = (int)gridDim.x;
    return ((b - p.T) % g + g) % g;
}
__device__ __forceinline__ int units_A(const PassParams& p) { return p.n_tiles * p.mix.m_tiles * p.mix.splits; }
__device__ __forceinline__ int groups_C(const PassParams& p, int l) { return p.lay_mo[l] >= 0 ? p.E : 1; }
__device__ __forceinline__ int units_C0(const PassParams& p, int l) {
    return groups_C(p, l) * p.n_tiles * p.up.m_tiles * p.up.splits;
}
__device__ __forceinline__ int units_C(const PassParams& p, int l) {
    return units_C0(p, l) + groups_C(p, l) * p.n_tiles * p.down.m_tiles * p.down.splits;
}
// group g of layer l: weight slot and rows [r0, r1) (counts are final once the layer's B phase is done)
__device__ __forceinline__ void group_rows(const PassParams& p, int l, int g, int& slot, int& r0, int& r1) {
    const int mo = p.lay_mo[l];
    if (mo >= 0) {
        slot = __ldcg(p.slot_of + mo * p.E + g);
        r0 = g * p.T;
        r1 = r0 + __ldcg(p.grp_cnt + mo * p.E + g);
    } else {
        slot = p.lay_slot[l];
        r0 = 0;
        r1 = p.T;
    }
}
__device__ __forceinline__ void split_unit(const Phase& P, int u, int& ks, int& mt, int& rest) {
    ks = u % P.splits;
    u /= P.splits;
    mt = u % P.m_tiles;
    rest = u / P.m_tiles;
}
__device__ __forceinline__ bool decode_A(const PassParams& p, int l, int u, Unit& w) {
    int ks, mt, nt;
    split_unit(p.mix, u, ks, mt, nt);
    w.phase = 0;
    w.g = 0;
    w.slot = l;
    w.n0 = nt * BN_MAX;
    if (w.n0 >= p.T) return false;
    w.n_valid = min(BN_MAX, p.T - w.n0);
    w.m0 = mt * BM;
    w.ks = ks;
    w.kb0 = ks * p.mix.kb_per_split;
    w.kb1 = min(p.mix.num_kb, w.kb0 + p.mix.kb_per_split);
    w.id = u;
    return w.kb0 < w.kb1;
}
__device__ __forceinline__ bool decode_C(const PassParams& p, int l, int u, Unit& w) {
    const int u0 = units_C0(p, l);
    const int ph = u >= u0;
    const Phase& P = ph ? p.down : p.up;
    int ks, mt, rest;
    split_unit(P, ph ? u - u0 : u, ks, mt, rest);
    const int G = groups_C(p, l);
    const int g = rest % G, nt = rest / G;
    int slot, r0, r1;
    group_rows(p, l, g, slot, r0, r1);
    w.n0 = r0 + nt * BN_MAX;
    if (slot < 0 || w.n0 >= r1) return false;
    w.phase = ph;
    w.g = g;
    w.slot = slot;
    w.n_valid = min(BN_MAX, r1 - w.n0);
    w.m0 = mt * BM;
    w.ks = ks;
    w.kb0 = ks * P.kb_per_split;
    w.kb1 = min(P.num_kb, w.kb0 + P.kb_per_split);
    w.id = u;
    return w.kb0 < w.kb1;
}
__device__ __forceinline__ int up_units_of_group(const PassParams& p, int l, int g) {
    int slot, r0, r1;
    group_rows(p, l, g, slot, r0, r1);
    if (slot < 0 || r1 <= r0) return 0;
    return (r1 - r0 + BN_MAX - 1) / BN_MAX * p.up.m_tiles * p.up.splits;
}
__device__ __forceinline__ int valid_C(const PassParams& p, int l) {
    const int per = p.up.m_tiles * p.up.splits + p.down.m_tiles * p.down.splits;
    int n = 0;
    for (int g = 0; g < groups_C(p, l); ++g) {
        int slot, r0, r1;
        group_rows(p, l, g, slot, r0, r1);
        if (slot >= 0 && r1 > r0) n += (r1 - r0 + BN_MAX - 1) / BN_MAX;
    }
    return n * per;
}

// ---- row tasks (128 worker threads; wt = 0..127).  Element i4 = (wt + 128 j) * 4 of the row.

// Row tasks.  A row task is latency-bound (about one row per CTA at decode sizes) and runs once per
// layer, i.e. always from a cold instruction cache, so the code is kept compact: every operand row
// arrives in the scratch through bulk copies (one round trip), and the compute loops stay rolled
// (shared-memory latency needs no unrolling).  Worker wt owns float4 columns i = wt + 128 j.
__device__ __forceinline__ void add4(float4& a, const float4 b) {
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}
__device__ __forceinline__ void store_bf16x4(__nv_bfloat16* dst, float4 a, float s) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(a.x * s, a.y * s), hi = __floats2bfloat162_rn(a.z * s, a.w * s);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dst) = pk;
}

// Scratch fills (thread 0): any number of scratch_add() calls, then scratch_commit() arrives with the
// last batch; every worker then scratch_wait()s.  The first add of a fill must follow a worker barrier
// that retired all generic reads of the region it overwrites.
__device__ __forceinline__ void scratch_add(Scratch& sc, uint32_t off, const void* src, uint32_t bytes) {
    proxy_fence_async_smem();
    mbar_add_tx(sc.mb, bytes);
    for (uint32_t o = 0; o < bytes; o += 32768) bulk_g2s(sc.base + off + o, (const char*)src + o, min(32768u, bytes - o), sc.mb);
}
__device__ __forceinline__ void scratch_commit(Scratch& sc) { mbar_arrive(sc.mb); }
__device__ __forceinline__ void scratch_wait(Scratch& sc) {
    mbar_wait(sc.mb, (uint32_t)sc.phase);
    sc.phase ^= 1;
}
// scratch rows of d floats: [0, EC) gate chunk, [EC] x row, [EC+1, EC+1+S) mix partials
__device__ __forceinline__ int gate_chunk(const PassParams& p, const Scratch& sc) {
    const int nrow = (int)(sc.bytes / (uint32_t)(p.d * 4));
    return max(1, min(p.E, nrow - 1 - p.s_mix));
}
__device__ __forceinline__ void gate_add(const PassParams& p, int mo, int e0, Scratch& sc) {
    const int n = min(gate_chunk(p, sc), p.E - e0);
    scratch_add(sc, 0, p.gate_w + ((size_t)mo * p.E + e0) * p.d, (uint32_t)n * p.d * 4);
}

// Sum of squares of a row exactly as the per-layer row kernels with blockDim = VB compute it (kernels.cu:
// row_threads(d), or gate_threads(d, E) for the gate kernel)
// compute it: virtual thread v accumulates float4 columns v, v + VB, ... in order, each virtual warp
// butterflies, and warp 0 butterflies the virtual-warp partials; thread 0's value is the result.  The
// 128 workers play the VB virtual threads (worker wt = virtual threads wt + 128 m, which own columns
// that the worker itself wrote to `row`).
__device__ __forceinline__ float vblock_sumsq(const float4* row, int d4, int VB, RowSmem& rs, int wt) {
    const int nw = VB >> 5;
#pragma unroll 1
    for (int v = wt; v < VB; v += kWorkers) {
        float t = 0.f;
        for (int i = v; i < d4; i += VB) t = __fadd_rn(t, sumsq4(row[i]));
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if ((wt & 31) == 0) rs.vred[v >> 5] = t;
    }
    wbar();
    if (wt < 32) {
        float t = wt < nw ? rs.vred[wt] : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (wt == 0) rs.ss[0] = t;
    }
    wbar();
    const float t = rs.ss[0];
    wbar();
    return t;
}

// Phase B for row r: x += sum_s pmix[s][r] (split order); MoE layer: rms; gate GEMV + bias; softmax,
// top-K, restricted remap and dispatch into xperm (K2 + K4/K5/K6, same semantics as kernels.cu);
// dense layer: xa = rms(x).  `pre`: gate chunk 0 was added before phase A completed.
__device__ __noinline__ void row_B(const PassParams& p, int l, int r, float4* row, RowSmem& rs, int wt, Scratch& sc,
                                   bool pre) {
    const int d = p.d, d4 = d >> 2, E = p.E, S = p.s_mix, mo = p.lay_mo[l];
    const bool moe = mo >= 0;
    const int EC = moe ? gate_chunk(p, sc) : 0;
    float4* sg = reinterpret_cast<float4*>(sc.base);
    float4* sx = sg + (size_t)EC * d4;
    if (wt == 0) PEV(l, 8);
    if (wt == 0) {
        if (moe && !pre) gate_add(p, mo, 0, sc);
        scratch_add(sc, (uint32_t)EC * d * 4, p.x + (long long)r * d, (uint32_t)d * 4);
        for (int s2 = 0; s2 < S; ++s2)
            scratch_add(sc, (uint32_t)(EC + 1 + s2) * d * 4, p.pmix + s2 * p.pm_stride + (long long)r * d, (uint32_t)d * 4);
        scratch_commit(sc);
    }
    scratch_wait(sc);
    float* xr = p.x + (long long)r * d;
#pragma unroll 1
    for (int i = wt; i < d4; i += kWorkers) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);  // x += (sum_s partials), partials summed first
        for (int s2 = 0; s2 < S; ++s2) add4(acc, sx[(size_t)(1 + s2) * d4 + i]);
        float4 v = sx[i];
        add4(v, acc);
        reinterpret_cast<float4*>(xr)[i] = v;
        row[i] = v;
    }
    const float ss = vblock_sumsq(row, d4, moe ? gate_threads(d, E) : row_threads(d), rs, wt);
    const float inv = 1.0f / sqrtf(ss / (float)d + 1e-12f);
    if (wt == 0) PEV(l, 9);
    if (!moe) {
#pragma unroll 1
        for (int i = wt; i < d4; i += kWorkers) store_bf16x4(p.xa + (long long)r * d + i * 4, row[i], inv);
        return;
    }
#pragma unroll 1
    for (int i = wt; i < d4; i += kWorkers) {
        const float4 a = row[i];
        row[i] = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
    }
    wbar();  // the GEMV below reads every worker's elements (lane-stride order of the per-layer kernel)
    // gate GEMV over the scratch chunks: per-thread partial dots, then a fixed-order reduction (lanes,
    // then the 4 worker warps in order)
    for (int e0 = 0; e0 < E; e0 += EC) {
        if (e0 > 0) {
            wbar();  // previous chunk fully read
            if (wt == 0) {
                gate_add(p, mo, e0, sc);
                scratch_commit(sc);
            }
            scratch_wait(sc);
        }
        // k_gate's GEMV: one warp per expert, lane l accumulates columns l, l+32, ... in order, then a
        // butterfly; lane 0's value + bias is the logit
        const int ne = min(EC, E - e0), lane = wt & 31;
#pragma unroll 1
        for (int e = wt >> 5; e < ne; e += 4) {
            float t = 0.f;
#pragma unroll 4
            for (int i = lane; i < d4; i += 32) t = __fadd_rn(t, dot4f(sg[(size_t)e * d4 + i], row[i]));
#pragma unroll
            for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) rs.red[0][e0 + e] = t;
        }
    }
    wbar();
    if (wt == 0) PEV(l, 10);
    if (wt < E) rs.gl[wt] = rs.red[0][wt] + p.gate_b[mo * E + wt];
    wbar();
    if (wt < 32) {
        GateArgs a{};
        a.T = p.T;
        a.d = d;
        a.E = E;
        a.K = p.K;
        a.cnt = p.grp_cnt + mo * E;
        a.pos = p.pos;
        a.raw = p.raw_log + mo * p.log_stride;
        a.fin = p.fin_log + mo * p.log_stride;
        a.wgt = p.wgt;
        a.in_draft = p.in_draft ? p.in_draft + mo * E : nullptr;
        a.draft_sorted = p.draft_sorted + mo * E;
        a.rank = p.rank + (size_t)mo * E * p.rank_n;
        a.N = p.N;
        a.use_affinity = p.use_aff;
        a.moe_ordinal = mo;
        a.row_plen = p.row_plen;
        a.flags = p.flags;
        gate_select_warp(a, r, rs.gl, rs.dst);
    }
    wbar();
    if (wt == 0) PEV(l, 11);
    for (int k = 0; k < p.K; ++k) {
        __nv_bfloat16* dst = p.xperm + (long long)rs.dst[k] * d;
#pragma unroll 1
        for (int i = wt; i < d4; i += kWorkers) store_bf16x4(dst + i * 4, row[i], 1.0f);
    }
    if (wt == 0) PEV(l, 12);
}

// Phase D for row r: y_k = sum_s ybuf[s][pos[r,k]] (s in order), x += sum_k p_k y_k (k in order)
// (dense layer: x += sum_s ybuf[s][r]); xa = rms(x).  Scratch rows: [0] x, [1 + k*S + s] partials.
__device__ __noinline__ void row_D(const PassParams& p, int l, int r, float4* row, RowSmem& rs, int wt, Scratch& sc) {
    const int d = p.d, d4 = d >> 2, S = p.s_down;
    const bool moe = p.lay_mo[l] >= 0;
    const int K = moe ? p.K : 1;
    if (wt < K) {
        rs.dst[wt] = moe ? __ldcg(p.pos + r * p.K + wt) : r;
        rs.gl[wt] = moe ? __ldcg(p.wgt + r * p.K + wt) : 1.f;
    }
    if (wt == 0) PEV(l, 16);
    wbar();
    if (wt == 0) PEV(l, 17);
    float* xr = p.x + (long long)r * d;
    const uint32_t rb = (uint32_t)d * 4;
    if (wt == 0) {
        scratch_add(sc, 0, xr, rb);
        for (int k = 0; k < K; ++k)
            for (int s2 = 0; s2 < S; ++s2)
                scratch_add(sc, rb * (1 + k * S + s2), p.ybuf + s2 * p.yd_stride + (long long)rs.dst[k] * d, rb);
        scratch_commit(sc);
    }
    if (wt == 0) PEV(l, 18);
    scratch_wait(sc);
    if (wt == 0) PEV(l, 19);
    const float4* sv = reinterpret_cast<const float4*>(sc.base);
#pragma unroll 1
    for (int i = wt; i < d4; i += kWorkers) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k = 0; k < K; ++k) {
            float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s2 = 0; s2 < S; ++s2) add4(y, sv[(size_t)(1 + k * S + s2) * d4 + i]);
            if (moe) axpy4(acc, rs.gl[k], y);
            else acc = y;
        }
        float4 v = sv[i];
        add4(v, acc);
        reinterpret_cast<float4*>(xr)[i] = v;
        row[i] = v;
    }
    const float ss = vblock_sumsq(row, d4, row_threads(d), rs, wt);
    const float inv = 1.0f / sqrtf(ss / (float)d + 1e-12f);
#pragma unroll 1
    for (int i = wt; i < d4; i += kWorkers) store_bf16x4(p.xa + (long long)r * d + i * 4, row[i], inv);
}

template <int PH>
__device__ void row_phase(const PassParams& p, int l, float4* row, RowSmem& rs, int wt, Scratch& sc) {
    int* c = lctr(p, l);
    if (wt == 0 && PH == kMarkD) PEV(l, 7);
    // a MoE layer's gate weights do not depend on phase A: start their copy before waiting for it
    const bool pre = PH == kMarkB && p.lay_mo[l] >= 0 && (int)blockIdx.x < p.T;
    if (wt == 0 && pre) gate_add(p, p.lay_mo[l], 0, sc);  // committed by row_B with the row's operands
    if (wt == 0) {
        spin_until(c + (PH == kMarkB ? cDoneA : cDoneC), PH == kMarkB ? units_A(p) : valid_C(p, l));
        proxy_fence_async();  // rows written by other CTAs are read by bulk copies (async proxy)
    }
    if (wt == 0) PEV(l, PH == kMarkB ? 3 : 5);
    wbar();
    // static assignment: row r -> CTA r % grid.  Every CTA's workers are free at this point (the counter
    // above counts finished epilogues), so a dynamic claim would only add an atomic per row.
    for (int r = blockIdx.x;; r += gridDim.x) {
        if (r >= p.T) {
            if (wt == 0) PEV(l, PH == kMarkB ? 4 : 6);
            break;
        }
        const bool pre_now = pre && r == (int)blockIdx.x;
        if (PH == kMarkB) row_B(p, l, r, row, rs, wt, sc, pre_now);
        else row_D(p, l, r, row, rs, wt, sc);
        // xperm / xa rows are read by TMA (async proxy) in other CTAs
        if (wt == 0 && PH == kMarkD) PEV(l, 14);
        __threadfence();
        proxy_fence_async();
        wbar();
        if (wt == 0) PEV(l, PH == kMarkB ? 13 : 15);
        if (wt == 0) atomicAdd(c + (PH == kMarkB ? cDoneB : cDoneD), 1);
    }
}

__device__ __forceinline__ bool ring_next(uint64_t* ring_full, uint64_t* ring_empty, const RingItem* ring, int& cons,
                                          bool whole_warp, RingItem& it) {
    const int r = cons % kRing;
    mbar_wait(&ring_full[r], (uint32_t)((cons / kRing) & 1));
    it = ring[r];
    ++cons;
    if (whole_warp) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&ring_empty[r]);
    } else {
        mbar_arrive(&ring_empty[r]);
    }
    return it.kind != kEnd;
}

template <int EPI_UP>
__global__ void __launch_bounds__(kThreads, 1)
    k_pass_tc(const __grid_constant__ CUtensorMap mapMix, const __grid_constant__ CUtensorMap mapXa,
              const __grid_constant__ CUtensorMap mapUp, const __grid_constant__ CUtensorMap mapXperm,
              const __grid_constant__ CUtensorMap mapDown, const __grid_constant__ CUtensorMap mapH,
              const __grid_constant__ PassParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int stages = p.stages;
    const int stage_bytes = kABytes + p.b_region;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + kMaxStages;
    uint64_t* acc_full = empty + kMaxStages;  // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint64_t* ring_full = acc_empty + 2;      // [kRing]
    uint64_t* ring_empty = ring_full + kRing; // [kRing]
    RingItem* ring = reinterpret_cast<RingItem*>(ring_empty + kRing);
    RowSmem* rs = reinterpret_cast<RowSmem*>(ring + kRing);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rs + 1);
    float4* rowbuf = reinterpret_cast<float4*>((reinterpret_cast<uintptr_t>(tmem_slot + 1) + 15) & ~uintptr_t(15));  // [d/4]
    __shared__ int s_last;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 4);
        }
        for (int r = 0; r < kRing; ++r) {
            mbar_init(&ring_full[r], 1);
            mbar_init(&ring_empty[r], 5);
        }
        mbar_init(&rs->mb, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapMix) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapXa) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapUp) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapXperm) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapDown) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapH) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {  // ---------------- scheduler + TMA producer
            int it = 0, pub = 0;
            bool kdep = false;  // griddepcontrol.wait done
            auto publish = [&](int kind, int l, const Unit* w) {
                const int r = pub % kRing;
                mbar_wait(&ring_empty[r], (uint32_t)(((pub / kRing) & 1) ^ 1));
                ring[r].kind = kind;
                ring[r].layer = l;
                if (w) ring[r].w = *w;
                mbar_arrive(&ring_full[r]);
                ++pub;
            };
            // Stream one unit: weight boxes at once; activation boxes once `dep` holds (at most `stages`
            // weight boxes are issued ahead of it).  dep_kind: 0 none, 1 kernel dependency, 2 counter.
            auto stream = [&](const Unit& w, const CUtensorMap* mA, const CUtensorMap* mB, long long a_rows_per_slot,
                              int dep_kind, const int* dep_ctr, int dep_target) {
                const int arow = (int)((long long)w.slot * a_rows_per_slot + w.m0);
                const int nb = (w.n_valid + BOX_N - 1) / BOX_N;
                const uint32_t bytes = kABytes + nb * kBoxBytes;
                bool ready = dep_kind == 0 || (dep_kind == 1 && kdep) ||
                             (dep_kind == 2 && ld_relaxed(dep_ctr) >= dep_target);
                if (ready && dep_kind == 2) {
                    fence_acquire();
                    proxy_fence_async();
                }
                const int pend_it = it;
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                    const int s = it % stages;
                    mbar_wait(&empty[s], (uint32_t)(((it / stages) & 1) ^ 1));
                    uint8_t* st = smem + s * stage_bytes;
                    mbar_expect_tx(&full[s], bytes);
                    tma_load_2d(mA, &full[s], st, kb * BK, arow);
                    if (ready) {
                        for (int j = 0; j < nb; ++j)
                            tma_load_2d(mB, &full[s], st + kABytes + j * kBoxBytes, kb * BK, w.n0 + j * BOX_N);
                        continue;
                    }
                    if (it + 1 - pend_it < stages && kb + 1 < w.kb1) continue;  // keep streaming weights
                    if (dep_kind == 1) {
                        pdl_wait();
                        kdep = true;
                    } else {
                        spin_until(dep_ctr, dep_target);
                        proxy_fence_async();
                    }
                    ready = true;
                    for (int j2 = pend_it; j2 <= it; ++j2) {
                        uint8_t* sp = smem + (j2 % stages) * stage_bytes + kABytes;
                        const int k2 = w.kb0 + (j2 - pend_it);
                        for (int j = 0; j < nb; ++j)
                            tma_load_2d(mB, &full[j2 % stages], sp + j * kBoxBytes, k2 * BK, w.n0 + j * BOX_N);
                    }
                }
            };
            const int nA = units_A(p);
            for (int l = 0; l < p.L; ++l) {
                int* c = lctr(p, l);
                PEV(l, 0);
                // ---- A: Mix units, statically owned: unit u -> CTA (u + T) % grid, so the first units go to
                // CTAs without row tasks (b >= T), whose ring is never worker scratch: they stream weights
                // at once and hold the activation boxes until layer l-1's D phase has published.  CTAs with
                // row tasks wait for D first (their ring is the D rows' scratch); idle CTAs prefetched
                // those units' tiles into L2 meanwhile (below).  Layer 0: weights before the kernel wait.
                const bool idle = (int)blockIdx.x >= p.T;
                if (l > 0 && !idle) {
                    spin_until(lctr(p, l - 1) + cDoneD, p.T);
                    proxy_fence_async();  // xa rows of other CTAs are read by TMA
                }
                for (int u = a_first(p, blockIdx.x); u < nA; u += gridDim.x) {
                    Unit w;
                    decode_A(p, l, u, w);
                    publish(kA, l, &w);
                    if (l == 0) stream(w, &mapMix, &mapXa, p.d, 1, nullptr, 0);
                    else if (idle) stream(w, &mapMix, &mapXa, p.d, 2, lctr(p, l - 1) + cDoneD, p.T);
                    else stream(w, &mapMix, &mapXa, p.d, 0, nullptr, 0);
                }
                if (!kdep) {
                    pdl_wait();
                    kdep = true;
                }
                publish(kMarkB, l, nullptr);
                // ---- C: expert (or dense) FFN units; the geometry is final once B has published
                spin_until(c + cDoneB, p.T);
                proxy_fence_async();
                PEV(l, 1);
                const bool moe = p.lay_mo[l] >= 0;
                const int nC = units_C(p, l);
                while (true) {
                    const int u = atomicAdd(c + cClaimC, 1);
                    if (u >= nC) break;
                    Unit w;
                    if (!decode_C(p, l, u, w)) continue;
                    publish(kC, l, &w);
                    if (w.phase == 0)
                        stream(w, &mapUp, moe ? &mapXperm : &mapXa, p.U, 0, nullptr, 0);
                    else
                        stream(w, &mapDown, &mapH, p.d, 2, c + cUp + w.g, up_units_of_group(p, l, w.g));
                }
                PEV(l, 2);
                publish(kMarkD, l, nullptr);
                // while layer l's D rows run, idle CTAs prefetch into L2 the next layer's Mix tiles owned by
                // CTAs with rows; every CTA prefetches one slice of the next MoE layer's gate weights
                if (l + 1 < p.L) {
                    const int n_idle = (int)gridDim.x - p.T;
                    if ((p.pf & 1) && n_idle > 0 && (int)blockIdx.x >= p.T)
                        for (int u = n_idle + ((int)blockIdx.x - p.T); u < nA; u += n_idle) {
                            if ((u + p.T) % (int)gridDim.x >= p.T) continue;  // owned by an idle CTA
                            Unit w;
                            decode_A(p, l + 1, u, w);
                            for (int kb = w.kb0; kb < w.kb1; ++kb) tma_prefetch_2d(&mapMix, kb * BK, (l + 1) * p.d + w.m0);
                        }
                    for (int l2 = l + 1; l2 < p.L && (p.pf & 2); ++l2)
                        if (p.lay_mo[l2] >= 0) {
                            const long long bytes = (long long)p.E * p.d * 4;
                            const long long chunk = ((bytes + gridDim.x - 1) / gridDim.x + 4095) / 4096 * 4096;
                            const long long off = (long long)blockIdx.x * chunk;
                            if (off < bytes) {
                                const char* src = reinterpret_cast<const char*>(p.gate_w + (size_t)p.lay_mo[l2] * p.E * p.d) + off;
                                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"((uint32_t)min(chunk, bytes - off))
                                             : "memory");
                            }
                            break;
                        }
                }
            }
            publish(kEnd, 0, nullptr);
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            int it = 0, cnt = 0, cons = 0;
            RingItem ri;
            while (ring_next(ring_full, ring_empty, ring, cons, false, ri)) {
                if (ri.kind != kA && ri.kind != kC) continue;
                const Unit& w = ri.w;
                const int acc = cnt & 1;
                mbar_wait(&acc_empty[acc], (uint32_t)(((cnt >> 1) & 1) ^ 1));
                tc_fence_after();
                const uint32_t d_tmem = tmem + (uint32_t)(acc * BN_MAX);
                const uint32_t idesc = idesc_bf16(BM, (w.n_valid + 15) & ~15);
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
                    const int s = it % stages;
                    mbar_wait(&full[s], (uint32_t)((it / stages) & 1));
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(smem + s * stage_bytes);
                    const uint32_t b_base = a_base + kABytes;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        mma_bf16(d_tmem, smem_desc(a_base + kk * 32), smem_desc(b_base + kk * 32), idesc,
                                 (kb > w.kb0 || kk) ? 1u : 0u);
                    mma_commit(&empty[s]);
                }
                mma_commit(&acc_full[acc]);
                ++cnt;
            }
        }
        __syncwarp();
    } else {  // -------------------------- warps 2..5: epilogues + row tasks
        const int q = warp & 3, wt = threadIdx.x - 64;
        Scratch sc{smem, (uint32_t)(stages * stage_bytes), &rs->mb, 0};
        int cnt = 0, cons = 0;
        RingItem ri;
        while (ring_next(ring_full, ring_empty, ring, cons, true, ri)) {
            if (ri.kind == kMarkB) {
                row_phase<kMarkB>(p, ri.layer, rowbuf, *rs, wt, sc);
                continue;
            }
            if (ri.kind == kMarkD) {
                row_phase<kMarkD>(p, ri.layer, rowbuf, *rs, wt, sc);
                continue;
            }
            const Unit& w = ri.w;
            const int acc = cnt & 1;
            mbar_wait(&acc_full[acc], (uint32_t)((cnt >> 1) & 1));
            tc_fence_after();
            const int row = w.m0 + q * 32 + lane;
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN_MAX);
            const bool up = ri.kind == kC && w.phase == 0;
            const Phase& P = ri.kind == kA ? p.mix : (w.phase ? p.down : p.up);
            for (int c0 = 0; c0 < w.n_valid; c0 += 16) {
                uint32_t v[16];
                tmem_ld16(taddr + c0, v);
                tmem_wait_ld();
                if (up) epilogue_store<EPI_UP>(P, w, row, lane, c0, v);
                else epilogue_store<kEpiStoreF32>(P, w, row, lane, c0, v);
            }
            tc_fence_before();
            // publish: all four warps' stores of this unit, then the counters
            __threadfence();
            if (up) proxy_fence_async();  // H is read by TMA
            wbar();
            if (wt == 0) {
                int* c = lctr(p, ri.layer);
                if (ri.kind == kA) {
                    atomicAdd(c + cDoneA, 1);
                } else {
                    if (up) atomicAdd(c + cUp + w.g, 1);
                    atomicAdd(c + cDoneC, 1);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
            ++cnt;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {  // last CTA out resets the pass counters for the next launch
        __threadfence();
        s_last = atomicAdd(p.ctr + (size_t)p.L * kCtr, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        for (int i = threadIdx.x; i < p.L * kCtr; i += blockDim.x) p.ctr[i] = 0;
        __syncthreads();
        if (threadIdx.x == 0) {
            p.ctr[(size_t)p.L * kCtr] = 0;
            __threadfence();
        }
    }
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

}  // namespace

bool pass_kernel_supported(const Engine& e) {
    // row tasks stage 2 + s_mix (B) and 1 + K*s_down (D) rows of d floats in the (>= 120 KB) stage ring
    const long long need = (long long)std::max(2 + e.s_mix, 1 + e.K * e.s_down) * e.d * 4;
    return e.use_tc && e.wt == kBF16 && !e.offload && e.ep_world == 1 && e.E <= kMaxE && e.K <= 32 &&
           e.L <= kMaxLayers && e.d % 4 == 0 && need <= 120 * 1024;
}

void launch_pass_tc(Engine& e, int T, bool restricted, int use_aff, int log_slot) {
    if (!e.pass_ctr) {
        SMOE_CUDA(cudaMalloc(&e.pass_ctr, sizeof(int) * ((size_t)e.L * kCtr + 1)));
        SMOE_CUDA(cudaMemset(e.pass_ctr, 0, sizeof(int) * ((size_t)e.L * kCtr + 1)));
        SMOE_CUDA(cudaDeviceSynchronize());
    }
    const Epi up_epi = e.kind == kSwiglu3 ? kEpiSwiglu : kEpiTanh;
    PassParams p{};
    p.T = T;
    p.d = e.d;
    p.E = e.E;
    p.K = e.K;
    p.L = e.L;
    p.U = e.U;
    static const int pf = [] {
        const char* v = getenv("SMOE_PASS_PREFETCH");
        return v ? atoi(v) : 3;
    }();
    p.pf = pf;
    p.n_tiles = (T + BN_MAX - 1) / BN_MAX;
    const long long yd_stride = (long long)e.E * e.Tmax * e.d, pm_stride = (long long)e.Tmax * e.d;
    p.mix = make_phase(TcGemmArgs{e.op_mix, e.d, e.op_xa, e.d, e.d, nullptr, nullptr, 1, 0, T, 0, T, e.pmix, e.d,
                                  kEpiStoreF32, e.s_mix, pm_stride, nullptr, nullptr});
    p.up = make_phase(TcGemmArgs{e.op_up, e.U, e.op_xperm, e.f, e.d, nullptr, nullptr, 1, 0, T, 0, T, e.hbuf, e.f, up_epi,
                                 1, 0, nullptr, nullptr});
    p.down = make_phase(TcGemmArgs{e.op_down, e.d, e.op_h, e.d, e.f, nullptr, nullptr, 1, 0, T, 0, T, e.ybuf, e.d,
                                   kEpiStoreF32, e.s_down, yd_stride, nullptr, nullptr});
    for (int l = 0; l < e.L; ++l) {
        p.lay_mo[l] = (short)e.moe_ord[l];
        p.lay_slot[l] = (short)e.dense_slot[l];
    }
    p.x = e.x;
    p.pmix = e.pmix;
    p.s_mix = e.s_mix;
    p.pm_stride = pm_stride;
    p.ybuf = e.ybuf;
    p.s_down = e.s_down;
    p.yd_stride = yd_stride;
    p.xa = reinterpret_cast<__nv_bfloat16*>(e.xa);
    p.xperm = reinterpret_cast<__nv_bfloat16*>(e.xperm);
    p.gate_w = e.gate_w;
    p.gate_b = e.gate_b;
    p.grp_cnt = e.grp_cnt;
    p.slot_of = e.slot_of;
    p.pos = e.pos;
    p.wgt = e.wgt;
    p.log_stride = (long long)e.Tmax * e.K;
    p.raw_log = e.raw_log + (size_t)log_slot * e.M * p.log_stride;
    p.fin_log = e.fin_log + (size_t)log_slot * e.M * p.log_stride;
    p.in_draft = restricted ? e.in_draft : nullptr;
    p.draft_sorted = e.draft_sorted;
    p.rank = e.rank;
    p.rank_n = std::max(1, e.cur_n_draft);
    p.N = e.cur_n_draft;
    p.use_aff = use_aff;
    p.row_plen = e.row_plen;
    p.flags = e.flags;
    p.ctr = e.pass_ctr;

    const int nb_max = (std::min(T, BN_MAX) + BOX_N - 1) / BOX_N;
    p.b_region = nb_max * kBoxBytes;
    const int stage_bytes = kABytes + p.b_region;
    const int ctrl = (int)(2 * kMaxStages + 4 + 2 * kRing) * 8 + kRing * (int)sizeof(RingItem) + (int)sizeof(RowSmem) +
                     32 + std::max(e.d, 4 * kWorkers) * 4;
    constexpr int kSmemBudget = 220 * 1024;
    p.stages = std::max(2, std::min(kMaxStages, (kSmemBudget - 1024 - ctrl) / stage_bytes));
    const size_t smem = (size_t)p.stages * stage_bytes + 1024 + ctrl;
    if ((long long)std::max(2 + e.s_mix, 1 + e.K * e.s_down) * e.d * 4 > (long long)p.stages * stage_bytes)
        throw Error(kInvariant, "pass kernel: row-task operands exceed the stage ring");

    const CUtensorMap& mMix = tensor_map(e.op_mix, BM);
    const CUtensorMap& mXa = tensor_map(e.op_xa, BOX_N);
    const CUtensorMap& mUp = tensor_map(e.op_up, BM);
    const CUtensorMap& mXp = tensor_map(e.op_xperm, BOX_N);
    const CUtensorMap& mDn = tensor_map(e.op_down, BM);
    const CUtensorMap& mH = tensor_map(e.op_h, BOX_N);
    auto go = [&](auto kern, size_t& configured) {
        if (smem > configured) {
            SMOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            configured = smem;
        }
        launch_k(kern, sm_count(), kThreads, smem, e.stream, mMix, mXa, mUp, mXp, mDn, mH, p);
    };
    static size_t configured[2] = {0, 0};  // per instantiation (same function-pointer type)
    if (up_epi == kEpiSwiglu) go(k_pass_tc<kEpiSwiglu>, configured[0]);
    else go(k_pass_tc<kEpiTanh>, configured[1]);
}

}  // namespace smoe

extern "C" int smoe_pass_trace_dump(const char* path) {
#ifdef SMOE_PASS_TRACE
    std::vector<long long> v((size_t)160 * smoe::kMaxLayers * 24);
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    cudaMemcpyFromSymbol(v.data(), smoe::g_ptr_ev, v.size() * sizeof(long long));
    FILE* fp = fopen(path, "wb");
    if (!fp) return -3;
    fwrite(v.data(), sizeof(long long), v.size(), fp);
    fclose(fp);
    return 0;
#else
    (void)path;
    return -1;
#endif
}
