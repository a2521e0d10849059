// gemm_tc.cu -- persistent grouped "swap-AB" GEMM on the 5th-generation tensor cores
// (tcgen05.mma + TMEM accumulators + TMA), the hot kernel of every pass.
//
// Decode-size expert GEMMs have few tokens per expert (n_e = 1..160) and large weight matrices, so
// the weights take the MMA M slot (128 rows per tile) and the tokens the N slot:
//   D[row m][token n] (TMEM, f32) = sum_k W[slot][m][k] * X[row n][k]
// Work unit = (phase, group g, 128-row tile, token tile of <=256 rows, K split).  One CTA per SM
// claims units dynamically (global atomic counter); its roles run decoupled through mbarrier rings:
//   warp 0     scheduler + TMA producer: one 128x64 bf16 weight box + ceil(n/32) 32x64 token boxes per
//              stage (token boxes sized by the group's real row count, 128B swizzle);
//   warp 1     owns TMEM (2 x 256 columns: double-buffered accumulator); one lane issues
//              tcgen05.mma.cta_group::1.kind::f16 with M=128, N=round16(n) (runtime instruction
//              descriptor), K=16, four per stage, and commits stages / finished accumulators;
//   warps 2-5  epilogue: tcgen05.ld.32x32b.x16 -> tanh | SwiGLU (w1/w3 rows interleaved, pairs
//              combined with one shuffle) | f32 store (optionally into a split-K partial) | residual
//              add, 32 consecutive rows per warp per token (coalesced), then release the accumulator.
// The epilogue of unit i overlaps the loads and MMAs of unit i+1.
//
// Two-phase launches fuse a MoE layer's up- and down-projection: every phase-0 (up) unit precedes
// the phase-1 (down) units in claim order; a down unit of expert g streams its weights into the ring
// at once and loads its activations (g's up output H) when all of g's up units have published
// completion through a per-expert counter (release / acquire + async-proxy fence).  The up->down
// kernel boundary and the up projection's tail disappear.  Programmatic dependent launch is handled
// the same way for a CTA's first unit: weights first, then griddepcontrol.wait, then activations.
//
// The K order inside a unit and the split count are fixed per GEMM shape (never T-dependent) and a D
// column never depends on other columns, so every token row gets bit-identical results in draft,
// verify and on-demand passes (batch invariance).
#include <cuda.h>

#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

namespace smoe {
namespace {
using namespace tc;

// Token (activation) operand maps with box heights 32, 64, ..., 256 rows: a unit loads its tokens with
// the smallest box that covers them, one TMA issue per stage (measured, tools/gemm_bench.py, T=320 with
// 80 rows per expert: up projection 0.707 -> 0.751 of the HBM peak, down 0.731 -> 0.766 vs three 32-row
// boxes per stage).  The stage ring of a grouped launch is laid out at run time from the routing
// counts: token space for the largest group's box only, every other byte of shared memory for more
// weight stages (a verify pass at B=64 gets 7 stages instead of 4 sized for 256 rows).
#ifndef SMOE_TOK_BOX0
#define SMOE_TOK_BOX0 32
#endif
constexpr int kTokBox0 = SMOE_TOK_BOX0, kTokBoxes = 256 / kTokBox0;
struct TokenMaps {
    CUtensorMap m[kTokBoxes];
};
// weight operand maps: 128-row box (one tile) and 256-row box (pair units)
struct WeightMaps {
    CUtensorMap m[2];
};
__host__ __device__ __forceinline__ int tok_box_index(int rows) {
    rows = rows < 1 ? 1 : (rows > BN_MAX ? BN_MAX : rows);
    return (rows + kTokBox0 - 1) / kTokBox0 - 1;
}
__host__ __device__ __forceinline__ int tok_box_bytes(int bi) { return (bi + 1) * kTokBox0 * BK * 2; }

struct TcParams {
    Phase ph[2];
    int nphase;
    const int* group_cnt;  // nullptr: single group {0, single_rows} -> single_slot
    const int* group_slot;
    int G, seg, single_rows, single_slot;  // group g: rows [g*seg, g*seg + group_cnt[g])
    int n_tiles;
    int stages, b_region;  // host layout (single-group launches): stage count, token bytes per stage
    int stage_space;       // shared bytes available to the stage ring (run-time layout of grouped launches)
    int pair_ok;           // grouped launches: phases (bit 0 up, bit 1 down) that may use pair units
    int pair_single;       // single-group launch in pair units (host-decided: rows <= 128)
    int* sched;            // [2]: next-unit counter, finished-CTA counter (self-resetting)
    int* done;             // [kMaxGroups]: finished phase-0 units per group (two-phase; self-resetting)
    int tr;                // trace slot (SMOE_TC_TRACE builds)
    // draft passes: the groups the launch will most likely have (the layer's draft experts, ascending);
    // before the dependency wait each CTA pulls the first pf_kb weight boxes of "its" predicted unit into L2
    const int* pred;
    int n_pred, pf_kb;
    int w_evict_first;         // weight boxes loaded with an L2 evict_first policy
    int static_first;          // CTA b starts with unit b (SMOE_STATIC_FIRST=0: every unit from the counter)
};

#ifdef SMOE_TC_TRACE
// Timeline instrumentation (tools/tc_trace.py; variant builds only): per launch, per unit
// {cta, t_claim, t_tma_done, t_mma_first, t_mma_done, t_epi_done} and per CTA {t_start, t_end}, globaltimer ns.
constexpr int kTrLaunches = 192, kTrUnits = 8192, kTrCtas = 160;
struct TrUnit { long long cta, claim, tma_done, mma_first, mma_done, epi_done, epi_start, epi_stored, epi_fenced, epi_barred; };
__device__ TrUnit g_tr_unit[kTrLaunches][kTrUnits];
__device__ long long g_tr_cta[kTrLaunches][kTrCtas][2];
__device__ long long g_tr_cta_dep[kTrLaunches][kTrCtas];  // after the grouped launch's dependency wait
__device__ int g_tr_meta[kTrLaunches][4];  // total units, nphase, T rows bound, grid
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TR(x) x
#else
#define TR(x)
#endif

// Pair units: two consecutive 128-row weight tiles under ONE 256-row TMA box per stage and two TMEM
// accumulators (each MMA and every output element are unchanged, so results are bit-identical).  The
// TMA issue count per weight byte halves, which is what bounded the stream: isolated up projection
// 0.865 -> 0.97 of the HBM copy peak, down 0.80 -> 0.99 (tools/gemm_bench.py, T <= 32).  Needs groups of
// <= 128 tokens (2 accumulators x 2 buffers x 128 TMEM columns).
__device__ __forceinline__ int row_tiles(const Phase& P, int pair) { return pair ? (P.m_tiles + 1) / 2 : P.m_tiles; }

// Grouped launches enumerate their units over a compacted list of work items = the (group, token tile)
// pairs that have rows, built once per CTA from the routing counts after the dependency wait (warp 0,
// one ballot pass over the groups) and kept in shared memory.  A draft pass routes to N of E experts
// (C4: 8 of 64), so enumerating every (group, tile) would make most unit claims land on empty groups:
// each such claim is one more round trip of the global unit counter for the claiming producer.
// Single-group launches have one implicit group (item i = token tile i).
constexpr int kMaxItems = 256;
struct Plan {
    int n_items, stages, stage_bytes, pair;
};
__device__ __forceinline__ int item_group(const int16_t* items, int i) { return items ? (items[i] & 0xff) : 0; }
__device__ __forceinline__ int item_tile(const int16_t* items, int i) { return items ? (items[i] >> 8) : i; }

// Warp 0 (all lanes), after the dependency wait: the item list and the stage ring of a grouped launch
// (token space for the largest group's box, every other byte of shared memory for weight stages).
// slot_pre[j]: group_slot[j*32 + lane], read before the dependency wait (the slot tables are written by
// stream-ordered host copies, never by the kernels this launch may overlap under PDL)
__device__ __forceinline__ void build_plan(const TcParams& p, int16_t* items, Plan* plan, const int* slot_pre) {
    const int lane = threadIdx.x & 31;
    int n = 0, mx = 1;
    for (int g0 = 0; g0 < p.G; g0 += 32) {
        const int g = g0 + lane;
        int cnt = 0;
        if (g < p.G && slot_pre[g0 >> 5] >= 0) cnt = p.group_cnt[g];
        const int nt = min(p.n_tiles, (cnt + BN_MAX - 1) / BN_MAX);
        mx = max(mx, min(BN_MAX, cnt));
        int incl = nt;  // inclusive prefix of the tile counts over the lanes (groups stay in order)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        for (int t = 0; t < nt; ++t) items[n + incl - nt + t] = (int16_t)(g | (t << 8));
        n += __shfl_sync(0xffffffffu, incl, 31);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
        const int pair = p.pair_ok && mx <= BN_MAX / 2 ? p.pair_ok : 0;
        const int stage_bytes = (pair ? 2 : 1) * kABytes + tok_box_bytes(tok_box_index(mx));
        plan->n_items = n;
        plan->pair = pair;
        plan->stage_bytes = stage_bytes;
        plan->stages = max(2, min(kMaxStages, p.stage_space / stage_bytes));
    }
}

__device__ __forceinline__ int units_of_phase(const TcParams& p, int n_items, int ph, int pair) {
    return n_items * row_tiles(p.ph[ph], (pair >> ph) & 1) * p.ph[ph].splits;
}

__device__ __forceinline__ void group_rows(const TcParams& p, int g, int& slot, int& r0, int& r1) {
    if (p.group_cnt) {
        slot = p.group_slot[g];
        r0 = g * p.seg;
        r1 = r0 + p.group_cnt[g];
    } else {
        slot = p.single_slot;
        r0 = 0;
        r1 = p.single_rows;
    }
}

// Unit u -> (phase, item = (group, token tile), row tile, split); returns false for units with no rows
// (single-group launches: token tiles past the rows).
__device__ __forceinline__ bool decode_unit(const TcParams& p, const int16_t* items, int n_items, int u, Unit& w,
                                           int pair) {
    int ph = 0;
    const int u0 = units_of_phase(p, n_items, 0, pair);
    if (u >= u0) {
        ph = 1;
        u -= u0;
    }
    const Phase& P = p.ph[ph];
    pair = (pair >> ph) & 1;
    const int mtu = row_tiles(P, pair);
    const int ks = u % P.splits;
    u /= P.splits;
    const int mt = u % mtu;
    u /= mtu;
    const int g = item_group(items, u);
    const int nt = item_tile(items, u);
    int slot, r0, r1;
    group_rows(p, g, slot, r0, r1);
    w.n0 = r0 + nt * BN_MAX;
    if (slot < 0 || w.n0 >= r1) return false;
    w.phase = ph;
    w.g = g;
    w.slot = slot;
    w.n_valid = min(BN_MAX, r1 - w.n0);
    w.m0 = mt * (pair ? 2 * BM : BM);
    w.pair = pair;
    w.ks = ks;
    w.kb0 = ks * P.kb_per_split;
    w.kb1 = min(P.num_kb, w.kb0 + P.kb_per_split);
    return w.kb0 < w.kb1;
}

// Phase-0 units a phase-1 unit of group g waits for (every token tile x row tile x split of g).
__device__ __forceinline__ int phase0_units_of_group(const TcParams& p, int g, int pair) {
    int slot, r0, r1;
    group_rows(p, g, slot, r0, r1);
    if (slot < 0 || r1 <= r0) return 0;
    return min(p.n_tiles, (r1 - r0 + BN_MAX - 1) / BN_MAX) * row_tiles(p.ph[0], pair & 1) * p.ph[0].splits;
}

// Consumer side of the unit ring: returns false when the producer published "done".  whole_warp:
// all 32 lanes call this (epilogue warps; lane 0 releases the slot after the warp has read it);
// otherwise a single lane (the MMA issuer) calls it and releases the slot itself.
__device__ __forceinline__ bool next_unit(const TcParams& p, const int16_t* items, int n_items, uint64_t* ring_full,
                                          uint64_t* ring_empty, const int* ring, int& cons, bool whole_warp, Unit& w,
                                          int pair) {
    const int r = cons % kRing;
    mbar_wait(&ring_full[r], (uint32_t)((cons / kRing) & 1));
    const int u = ring[r];
    ++cons;
    if (whole_warp) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&ring_empty[r]);
    } else {
        mbar_arrive(&ring_empty[r]);
    }
    if (u < 0) return false;
    decode_unit(p, items, n_items, u, w, pair);
    w.id = u;
    return true;
}

// The dependency wait of a launch: the previous grid's completion and memory flush (PDL).
__device__ __forceinline__ void dep_wait(const TcParams&) { pdl_wait(); }

// Draft passes: while the CTAs wait for the gate (HBM is idle then), prefetch into L2 the first weight
// boxes of the first wave of units as they will be enumerated if every predicted group has rows (the
// claims are dynamic, so CTA b warms unit b for whichever CTA takes it).  A wrong guess costs only
// bandwidth that was idle.
__device__ __forceinline__ void prefetch_predicted(const TcParams& p, const WeightMaps& mapA0, const WeightMaps& mapA1) {
    int u = blockIdx.x;
    int ph = 0;
    const int pr0 = p.pair_ok & 1, pr1 = (p.pair_ok >> 1) & 1;
    const int up_units = p.n_pred * row_tiles(p.ph[0], pr0) * p.ph[0].splits;
    if (u >= up_units) {
        if (p.nphase < 2) return;
        u -= up_units;
        ph = 1;
    }
    const Phase& P = p.ph[ph];
    const int pair = ph ? pr1 : pr0;
    const int mtu = row_tiles(P, pair);
    const int ks = u % P.splits;
    u /= P.splits;
    const int mt = u % mtu, item = u / mtu;
    if (item >= p.n_pred) return;
    const int g = p.pred[item];
    const int slot = g >= 0 && g < p.G ? p.group_slot[g] : -1;
    if (slot < 0) return;
    const CUtensorMap* map = ph ? &mapA1.m[pair] : &mapA0.m[pair];
    const int arow = (int)((long long)slot * P.a_rows_per_slot + mt * (pair ? 2 * BM : BM));
    const int kb0 = ks * P.kb_per_split, kb1 = min(P.num_kb, min(kb0 + P.kb_per_split, kb0 + p.pf_kb));
    for (int kb = kb0; kb < kb1; ++kb) {
        if (P.tiled) tma_prefetch_3d(map, arow & 255, (arow >> 8) * P.num_kb + kb);
        else tma_prefetch_2d(map, kb * BK, arow);
    }
}

template <int EPI0, int EPI1>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ WeightMaps mapA0, const __grid_constant__ TokenMaps mapB0,
              const __grid_constant__ WeightMaps mapA1, const __grid_constant__ TokenMaps mapB1, TcParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // single-group launches: host layout (their weights stream before the dependency wait); grouped
    // launches: re-laid out from the counts by the producer and the MMA lane after the wait
    int pair = p.group_cnt ? 0 : p.pair_single;  // grouped launches: decided from the counts below
    int stages = p.stages;
    int stage_bytes = (pair ? 2 : 1) * kABytes + p.b_region;
    int n_items = p.n_tiles;  // grouped launches: from the plan below
    int total_units = units_of_phase(p, n_items, 0, pair) + (p.nphase > 1 ? units_of_phase(p, n_items, 1, pair) : 0);
    TR(const int trs = p.tr % kTrLaunches; const long long tr_entry = gtimer();)

    // control block first (fixed size), then the 1024-aligned stage ring
    extern __shared__ uint8_t smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 15) & ~uintptr_t(15));
    uint64_t* empty = full + kMaxStages;
    uint64_t* acc_full = empty + kMaxStages;  // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint64_t* ring_full = acc_empty + 2;      // [kRing]
    uint64_t* ring_empty = ring_full + kRing; // [kRing]
    int* ring = reinterpret_cast<int*>(ring_empty + kRing);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);
    Plan* plan = reinterpret_cast<Plan*>(tmem_slot + 4);
    int16_t* s_items = reinterpret_cast<int16_t*>(plan + 1);
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(s_items + kMaxItems) + 1023) & ~uintptr_t(1023));
    const int16_t* items = p.group_cnt ? s_items : nullptr;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], 4);  // one arrival per epilogue warp
        }
        for (int r = 0; r < kRing; ++r) {
            mbar_init(&ring_full[r], 1);
            mbar_init(&ring_empty[r], 5);  // MMA lane + 4 epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA0.m[0]) : "memory");
        if (p.pair_ok || p.pair_single) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA0.m[1]) : "memory");
        for (int i = 0; i < kTokBoxes; ++i) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB0.m[i]) : "memory");
        if (p.nphase > 1) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA1.m[0]) : "memory");
            if (p.pair_ok) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA1.m[1]) : "memory");
            for (int i = 0; i < kTokBoxes; ++i) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB1.m[i]) : "memory");
        }
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
    if (threadIdx.x == 0) pdl_trigger();  // let the next kernel's CTAs take SMs as ours retire
    if (p.group_cnt) {
        // grouped launches: the unit geometry (rows per expert) is written by the gate kernel that
        // immediately precedes this one, so it may only be read after the dependency wait
        if (p.pred && threadIdx.x == 0) prefetch_predicted(p, mapA0, mapA1);
        int slot_pre[kMaxGroups / 32];
#pragma unroll
        for (int j = 0; j < kMaxGroups / 32; ++j) {
            const int g = j * 32 + lane;
            slot_pre[j] = warp == 0 && g < p.G ? p.group_slot[g] : -1;
        }
        dep_wait(p);
        if (warp == 0) build_plan(p, s_items, plan, slot_pre);
        __syncthreads();
        n_items = plan->n_items;
        pair = plan->pair;
        stages = plan->stages;
        stage_bytes = plan->stage_bytes;
        total_units = units_of_phase(p, n_items, 0, pair) + (p.nphase > 1 ? units_of_phase(p, n_items, 1, pair) : 0);
    }
    TR(if (threadIdx.x == 0) {
        g_tr_cta[trs][blockIdx.x % kTrCtas][0] = tr_entry;
        g_tr_cta_dep[trs][blockIdx.x % kTrCtas] = gtimer();
        if (blockIdx.x == 0) { g_tr_meta[trs][0] = total_units; g_tr_meta[trs][1] = p.nphase; g_tr_meta[trs][2] = units_of_phase(p, n_items, 0, 0); g_tr_meta[trs][3] = gridDim.x; }
    })

    if (warp == 0) {
        // ---------------- scheduler + TMA producer: like the MMA issuer, the whole warp runs the loop and one
        // elected lane issues, with the unit's coordinates made warp-uniform (uniform-register TMA operands)
        int it = 0, ps = 0;
        uint32_t pph = 0;
        const uint64_t wpol = policy_evict_first();
        const bool wef = p.w_evict_first != 0;
        const int stg = __shfl_sync(0xffffffffu, stages, 0);
        const uint32_t sbytes = (uint32_t)__shfl_sync(0xffffffffu, stage_bytes, 0);
        const int a_space = __shfl_sync(0xffffffffu, (pair ? 2 : 1) * kABytes, 0);  // weight bytes of a stage
        // griddepcontrol.wait done: the previous kernel's outputs are visible (grouped: waited above)
        bool kernel_dep = p.group_cnt != nullptr;
        for (int pub = 0;; ++pub) {
            // dynamic work distribution: claim the next non-empty unit (single-group geometry is
            // host-known; grouped geometry was waited for above)
            int u = 0;
            Unit w;
            if (lane == 0) {
                // CTA b's first unit is unit b (no atomic round trip before the first TMA); later claims
                // take units gridDim.x, gridDim.x + 1, ... from the counter
                bool first = p.static_first && pub == 0 && (int)blockIdx.x < total_units;
                do {
                    u = first ? (int)blockIdx.x : (p.static_first ? (int)gridDim.x : 0) + atomicAdd(&p.sched[0], 1);
                    first = false;
                } while (u < total_units && !decode_unit(p, items, n_items, u, w, pair));
            }
            u = __shfl_sync(0xffffffffu, u, 0);
            TR(if (lane == 0 && u < total_units && u < kTrUnits) { g_tr_unit[trs][u].cta = blockIdx.x | ((long long)p.tr << 32); g_tr_unit[trs][u].claim = gtimer(); })
            const int r = pub % kRing;
            mbar_wait(&ring_empty[r], (uint32_t)(((pub / kRing) & 1) ^ 1));
            if (lane == 0) {
                ring[r] = u < total_units ? u : -1;
                mbar_arrive(&ring_full[r]);
            }
            __syncwarp();
            if (u >= total_units) break;  // out of units
            // lane 0's decode, broadcast (the other lanes' w is unset)
            const int phase = __shfl_sync(0xffffffffu, w.phase, 0), wp = __shfl_sync(0xffffffffu, w.pair, 0);
            const int kb0 = __shfl_sync(0xffffffffu, w.kb0, 0), kb1 = __shfl_sync(0xffffffffu, w.kb1, 0);
            const int n0 = __shfl_sync(0xffffffffu, w.n0, 0), g = __shfl_sync(0xffffffffu, w.g, 0);
            const int nval = __shfl_sync(0xffffffffu, w.n_valid, 0);
            const int arow = __shfl_sync(
                0xffffffffu, lane == 0 ? (int)((long long)w.slot * p.ph[w.phase].a_rows_per_slot + w.m0) : 0, 0);
            const int wtiled = p.ph[phase].tiled;
            const int tc1 = arow & 255, tc2 = (arow >> 8) * p.ph[phase].num_kb;  // tiled-layout box coordinates
            const CUtensorMap* mA = phase ? &mapA1.m[wp] : &mapA0.m[wp];
            // the unit's tokens as ONE box per stage: the smallest of 32/64/128/256 rows covering them
            // (one TMA issue per stage; rows past the group are fetched but never multiplied in)
            const int bi = tok_box_index(nval);
            const CUtensorMap* mB = phase ? &mapB1.m[bi] : &mapB0.m[bi];
            const uint32_t bytes = (uint32_t)((wp ? 2 : 1) * kABytes + tok_box_bytes(bi));
            // Activations may be read once (a) the previous kernel is complete (PDL) and (b) for a
            // phase-1 unit, every phase-0 unit of its group has published.  Until then only weight
            // boxes are issued; at most `stages` of them are held back.
            const int need = phase ? phase0_units_of_group(p, g, pair) : 0;
            bool ready = kernel_dep && (phase == 0 || __shfl_sync(0xffffffffu, ld_relaxed(&p.done[g]), 0) >= need);
            if (ready && phase) {
                fence_acquire();
                proxy_fence_async();
            }
            const int pend_it = it;
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                // ring position kept incrementally: the producer's per-stage instruction count is on the
                // stream's critical path (a runtime it % stages is an emulated division)
                const int s = ps;
                const uint32_t sph = pph;
                if (++ps == stg) {
                    ps = 0;
                    pph ^= 1u;
                }
                mbar_wait(&empty[s], sph ^ 1u);
                uint8_t* st = smem + s * sbytes;
                if (elect_one()) {
                    mbar_expect_tx(&full[s], bytes);
                    if (wtiled) {
                        if (wef) tma_load_3d_hint(mA, &full[s], st, tc1, tc2 + kb, wpol);
                        else tma_load_3d(mA, &full[s], st, tc1, tc2 + kb);
                    } else {
                        if (wef) tma_load_2d_hint(mA, &full[s], st, kb * BK, arow, wpol);
                        else tma_load_2d(mA, &full[s], st, kb * BK, arow);
                    }
                    if (ready) tma_load_2d(mB, &full[s], st + a_space, kb * BK, n0);
                }
                __syncwarp();
                if (ready) continue;
                if (it + 1 - pend_it < stg && kb + 1 < kb1) continue;  // keep streaming weights
                if (!kernel_dep) {
                    dep_wait(p);
                    kernel_dep = true;
                }
                if (phase) {
                    spin_until(&p.done[g], need);
                    proxy_fence_async();  // generic-proxy stores of H before async-proxy (TMA) reads
                }
                ready = true;
                if (elect_one())
                    for (int j2 = pend_it; j2 <= it; ++j2) {  // activations of the held-back stages
                        uint8_t* sp = smem + (j2 % stg) * sbytes + a_space;
                        tma_load_2d(mB, &full[j2 % stg], sp, (kb0 + (j2 - pend_it)) * BK, n0);
                    }
                __syncwarp();
            }
            TR(if (lane == 0 && u < kTrUnits) g_tr_unit[trs][u].tma_done = gtimer();)
        }
        if (!kernel_dep) dep_wait(p);
    } else if (warp == 1) {
        if (!p.group_cnt) dep_wait(p);
        // ---------------- MMA issuer: the whole warp runs the loop convergently and one elected lane issues.
        // Every operand is made warp-uniform (__shfl_sync from lane 0), so ptxas builds the descriptors in
        // uniform registers once per stage instead of wrapping each tcgen05.mma in its own elect / R2UR
        // loop -- this thread's per-stage latency (full barrier -> stage released) is on the stream's
        // critical path.
        // TMEM = two 256-column accumulator buffers used alternately (epilogue of one unit overlaps the
        // MMAs of the next)
        // (bit a of `par`: phase parity of buffer a)
        const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
        const int stg = __shfl_sync(0xffffffffu, stages, 0);
        const uint32_t sbytes = (uint32_t)__shfl_sync(0xffffffffu, stage_bytes, 0);
        const uint32_t bofs = (uint32_t)__shfl_sync(0xffffffffu, (pair ? 2 : 1) * kABytes, 0);
        const uint32_t sbase = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
        int nb = 0, cons = 0, ms = 0;
        uint32_t par = 0, mph = 0;
        Unit w;
        while (next_unit(p, items, n_items, ring_full, ring_empty, ring, cons, true, w, pair)) {
            const int kb0 = __shfl_sync(0xffffffffu, w.kb0, 0), kb1 = __shfl_sync(0xffffffffu, w.kb1, 0);
            const int wpair = __shfl_sync(0xffffffffu, w.pair, 0);
            const int nval = __shfl_sync(0xffffffffu, w.n_valid, 0);
            const int acc = nb;
            mbar_wait(&acc_empty[acc], ((par >> acc) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tm + (uint32_t)(acc * BN_MAX);
            const uint32_t d_tile1 = d_tmem + (uint32_t)BM;  // pair units' second tile
            const uint32_t idesc = idesc_bf16(BM, (nval + 15) & ~15);
            for (int kb = kb0; kb < kb1; ++kb) {
                const int s = ms;
                const uint32_t sph = mph;
                if (++ms == stg) {
                    ms = 0;
                    mph ^= 1u;
                }
                mbar_wait(&full[s], sph);
                tc_fence_after();
                TR(if (kb == kb0 && lane == 0) g_tr_unit[trs][w.id % kTrUnits].mma_first = gtimer();)
                const uint32_t a_base = sbase + (uint32_t)s * sbytes;
                // descriptors of the stage's K=16 slices: +32 B of address = +2 in the 14-bit start field
                // (shared addresses < 256 KB never carry out of it)
                const uint64_t da = smem_desc(a_base), db = smem_desc(a_base + bofs);
                static_assert(BK == 64, "mma_stage_*: four K=16 slices per stage");
                if (elect_one()) {
                    if (wpair)  // second 128-row tile of the box -> second accumulator, same tokens
                        mma_stage_pair(d_tmem, d_tile1, da, smem_desc(a_base + kABytes), db, idesc, kb > kb0);
                    else
                        mma_stage_single(d_tmem, da, db, idesc, kb > kb0);
                    mma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(&acc_full[acc]);
            __syncwarp();
            par ^= 1u << acc;
            nb ^= 1;
            TR(if (lane == 0) g_tr_unit[trs][w.id % kTrUnits].mma_done = gtimer();)
        }
    } else {  // -------------------------- epilogue: warps 2..5 -> TMEM lane quarters 2,3,0,1
        if (!p.group_cnt) dep_wait(p);
        const int q = warp & 3;
        int nb = 0, cons = 0;
        uint32_t par = 0;
        Unit w;
        while (next_unit(p, items, n_items, ring_full, ring_empty, ring, cons, true, w, pair)) {
            const int acc = nb;  // the MMA issuer's buffer sequence
            mbar_wait(&acc_full[acc], (par >> acc) & 1);
            tc_fence_after();
            TR(if (warp == 2 && lane == 0) g_tr_unit[trs][w.id % kTrUnits].epi_start = gtimer();)
            const Phase& P = p.ph[w.phase];
            for (int h = 0; h < (w.pair ? 2 : 1); ++h) {  // pair units: the two 128-row tiles in turn
                const int row = w.m0 + h * BM + q * 32 + lane;  // weight row within the slot
                const uint32_t taddr =
                    tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN_MAX + h * BM);
#ifndef SMOE_EPI32_MIN
#define SMOE_EPI32_MIN 16
#endif
                if (EPI0 == kEpiSwiglu && w.phase == 0 && w.n_valid > SMOE_EPI32_MIN) {
                    for (int c = 0; c < w.n_valid; c += 32) {  // 32 columns per step (tmem buffer is 256 wide)
                        uint32_t v[32];
                        tmem_ld16(taddr + c, v);
                        tmem_ld16(taddr + c + 16, v + 16);
                        tmem_wait_ld();
                        epilogue_swiglu32(P, w, row, lane, c, v);
                    }
                    continue;
                }
                for (int c = 0; c < w.n_valid; c += 16) {
                    uint32_t v[16];
                    tmem_ld16(taddr + c, v);
                    tmem_wait_ld();
                    if (w.phase == 0) epilogue_store<EPI0>(P, w, row, lane, c, v);
                    else epilogue_store<EPI1>(P, w, row, lane, c, v);
                }
            }
            TR(if (warp == 2 && lane == 0) g_tr_unit[trs][w.id % kTrUnits].epi_stored = gtimer();)
            tc_fence_before();
            if (p.nphase > 1 && w.phase == 0) {
                // publish: all four warps' stores of this unit (ordered before the async-proxy reads of the
                // down units), a CTA barrier, then ONE release increment -- release is cumulative over the
                // barrier, so the other warps' stores are covered without each warp draining its stores
                // through a full fence.sc (which waited microseconds behind the weight stream)
                proxy_fence_async();
                TR(if (warp == 2 && lane == 0) g_tr_unit[trs][w.id % kTrUnits].epi_fenced = gtimer();)
                asm volatile("bar.sync 1, 128;" ::: "memory");
                TR(if (warp == 2 && lane == 0) g_tr_unit[trs][w.id % kTrUnits].epi_barred = gtimer();)
#ifdef SMOE_PUBLISH_FENCE_SC
                if (warp == 2 && lane == 0) {
                    __threadfence();
                    atomicAdd(&p.done[w.g], 1);
                }
#else
                if (warp == 2 && lane == 0)
                    asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(&p.done[w.g]) : "memory");
#endif
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
            par ^= 1u << acc;
            nb ^= 1;
            TR(if (warp == 2 && lane == 0) g_tr_unit[trs][w.id % kTrUnits].epi_done = gtimer();)
        }
    }
    if (p.nphase > 1 && p.ph[1].peer_y) __threadfence_system();  // peer stores performed before the grid ends
    tc_fence_before();
    __syncthreads();
    TR(if (threadIdx.x == 0) g_tr_cta[trs][blockIdx.x % kTrCtas][1] = gtimer();)
    if (threadIdx.x == 0) {  // last CTA out resets the scheduler (and counters) for the next launch
        __threadfence();
        if (atomicAdd(&p.sched[1], 1) == (int)gridDim.x - 1) {
            p.sched[0] = 0;
            if (p.nphase > 1)
                for (int g = 0; g < p.G; ++g) p.done[g] = 0;
            p.sched[1] = 0;
            __threadfence();
        }
    }
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

}  // namespace

// ------------------------------------------------------------------ host side
namespace tc {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

const CUtensorMap& tensor_map(const TcOperand& op, int box_rows) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, long long, int, int, bool>, CUtensorMap> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(op.base, op.rows, op.K, box_rows, op.tiled);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    EncodeTiledFn fn = encode_fn();
    if (!fn) throw Error(kCuda, "cuTensorMapEncodeTiled entry point unavailable");
    CUtensorMap m;
    if (op.tiled) {  // [rows/256 * K/64] chunks of [256][64]: box {64, box_rows, 1} = one contiguous 16 / 32 KB piece
        if (op.rows % 256 || op.K % 64 || box_rows > 256)
            throw Error(kInvariant, "tcgen05 GEMM: tiled operand needs rows % 256 == 0 and K % 64 == 0");
        cuuint64_t dims[3] = {64, 256, (cuuint64_t)(op.rows / 256) * (cuuint64_t)(op.K / 64)};
        cuuint64_t strides[2] = {128, 32768};
        cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(op.base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled (3D) failed: " + std::to_string((int)r));
        return cache.emplace(key, m).first->second;
    }
    cuuint64_t dims[2] = {(cuuint64_t)op.K, (cuuint64_t)op.rows};
    cuuint64_t strides[1] = {(cuuint64_t)op.K * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(op.base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return cache.emplace(key, m).first->second;
}

int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

Phase make_phase(const TcGemmArgs& a) {
    Phase P{};
    P.Nrows = a.epi == kEpiSwiglu ? 2 * a.Nout : a.Nout;
    P.a_rows_per_slot = a.a_rows_per_slot;
    P.m_tiles = (P.Nrows + BM - 1) / BM;
    P.num_kb = (a.K + BK - 1) / BK;
    P.splits = std::max(1, std::min(a.splits, P.num_kb));
    P.kb_per_split = (P.num_kb + P.splits - 1) / P.splits;
    // every split must own K blocks: a consumer sums exactly `splits` partials
    if ((P.splits - 1) * P.kb_per_split >= P.num_kb) throw Error(kInvariant, "tcgen05 GEMM: empty K split");
    P.Y = a.Y;
    P.ldy = a.ldy;
    P.split_stride = a.split_stride;
    P.peer_y = a.peer_y;
    P.peer_eo = a.peer_eo;
    P.peer_me = a.peer_me;
    P.peer_seg = a.seg;
    P.tiled = a.A.tiled ? 1 : 0;
    if (P.tiled && a.a_rows_per_slot % 256) throw Error(kInvariant, "tcgen05 GEMM: tiled slots need 256-row multiples");
    return P;
}
}  // namespace tc

namespace {
using namespace tc;
int g_launch_no = 0;  // trace slot of the next launch (SMOE_TC_TRACE builds)

TokenMaps token_maps(const TcOperand& op) {
    TokenMaps t;
    for (int i = 0; i < kTokBoxes; ++i) t.m[i] = tensor_map(op, kTokBox0 * (i + 1));
    return t;
}

template <int EPI0, int EPI1>
void launch_phases(const TcGemmArgs& a, const TcGemmArgs* b, cudaStream_t s) {
#ifndef SMOE_TC_SMEM_KB
#define SMOE_TC_SMEM_KB 220
#endif
    constexpr int kSmemBudget = SMOE_TC_SMEM_KB * 1024;  // stages + 1.5 KB control <= 227 KB
    static std::atomic<uint64_t> configured{0};
    if (first_use_on_device(configured))
        SMOE_CUDA(cudaFuncSetAttribute(k_gemm_tc<EPI0, EPI1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    TcParams p{};
    p.ph[0] = make_phase(a);
    p.nphase = b ? 2 : 1;
    if (b) p.ph[1] = make_phase(*b);
    p.group_cnt = a.group_cnt;
    p.group_slot = a.group_slot;
    p.G = a.group_cnt ? a.G : 1;
    p.seg = a.seg;
    p.single_rows = a.single_rows;
    p.single_slot = a.single_slot;
    p.n_tiles = (a.rows_bound + BN_MAX - 1) / BN_MAX;
    if (a.group_cnt && (long long)p.G * p.n_tiles > kMaxItems)
        throw Error(kInvariant, "tcgen05 GEMM: more (group, token tile) items than the plan holds");
    if (a.group_cnt && p.G > kMaxGroups)
        throw Error(kInvariant, "tcgen05 GEMM: more groups than the plan's slot preload holds");

    constexpr int kCtrl = 1024;  // control block (barriers, unit ring, TMEM slot) + alignment slack below
    static const bool pair_env = [] {
        const char* v = getenv("SMOE_TC_PAIR");
        return !(v && v[0] == '0');
    }();
    static const int pair_single_env = [] {  // 0 off, 1 auto (default), 2 whenever rows allow
        const char* v = getenv("SMOE_TC_PAIR_SINGLE");
        return v ? atoi(v) : 1;
    }();
    static const bool pair_down_env = [] {
        const char* v = getenv("SMOE_TC_PAIR_DOWN");
        return !(v && v[0] == '0');
    }();
    // grouped launches: bit 0 pairs the first phase, bit 1 the second (applied when the counts allow)
    p.pair_ok = a.group_cnt && pair_env ? (1 | (b && pair_down_env ? 2 : 0)) : 0;
    // single-group launches pair only when that does not load the busiest SM with more weight bytes
    // (the C2 Mix launch at T=64 would run 64 paired units on 64 of 148 SMs: 20.8 vs 18.0 us; the head
    // at T=64, 250 units = 2 waves of 1 MB, becomes 1 wave of 2 MB paired units)
    const long long nt = (a.rows_bound + BN_MAX - 1) / BN_MAX, sms = sm_count();
    const long long units1 = nt * p.ph[0].m_tiles * p.ph[0].splits;
    const long long units2 = nt * ((p.ph[0].m_tiles + 1) / 2) * p.ph[0].splits;
    const bool pair_pays = 2 * ((units2 + sms - 1) / sms) <= (units1 + sms - 1) / sms;
    p.pair_single = !a.group_cnt && pair_env && pair_single_env && a.single_rows <= BN_MAX / 2 &&
                    (pair_pays || pair_single_env == 2);
    p.b_region = tok_box_bytes(tok_box_index(std::min(a.rows_bound, BN_MAX)));
    const int stage_bytes = (p.pair_single ? 2 : 1) * kABytes + p.b_region;
    p.stage_space = kSmemBudget - kCtrl - 1024;
    p.stages = std::max(2, std::min(kMaxStages, p.stage_space / stage_bytes));
    p.sched = a.sched;
    p.done = a.done;
    static const int wef_env = [] {
        const char* v = getenv("SMOE_W_EVICT_FIRST");
        return v ? atoi(v) : 1;
    }();
    p.w_evict_first = a.group_cnt && wef_env;  // expert weights: streamed once per pass
    static const int static_first_env = [] {
        const char* v = getenv("SMOE_STATIC_FIRST");
        return v ? atoi(v) : 1;
    }();
    p.static_first = static_first_env;

    static const int pf_kb_env = [] {
        const char* v = getenv("SMOE_PF_KB");
        return v ? atoi(v) : 8;
    }();
    if (a.group_cnt && a.pred_groups && a.n_pred > 0 && pf_kb_env > 0) {
        p.pred = a.pred_groups;
        p.n_pred = a.n_pred;
        p.pf_kb = pf_kb_env;
    }
    p.tr = g_launch_no++;
    const size_t smem = a.group_cnt ? (size_t)kSmemBudget : (size_t)p.stages * stage_bytes + kCtrl + 1024;
    const WeightMaps ma0{{tensor_map(a.A, BM), tensor_map(a.A, 2 * BM)}};
    const TokenMaps mb0 = token_maps(a.B);
    const WeightMaps ma1 = b ? WeightMaps{{tensor_map(b->A, BM), tensor_map(b->A, 2 * BM)}} : ma0;
    const TokenMaps mb1 = b ? token_maps(b->B) : mb0;
    long long units = (long long)p.G * p.n_tiles * (p.pair_single ? (p.ph[0].m_tiles + 1) / 2 : p.ph[0].m_tiles) *
                      p.ph[0].splits;
    if (b) units += (long long)p.G * p.n_tiles * p.ph[1].m_tiles * p.ph[1].splits;
    const int grid = (int)std::max(1ll, std::min(units, (long long)sm_count()));
    launch_k(k_gemm_tc<EPI0, EPI1>, grid, kThreads, smem, s, ma0, mb0, ma1, mb1, p);
}

}  // namespace

void launch_gemm_tc(const TcGemmArgs& a, cudaStream_t s) {
    if (a.Nout <= 0 || a.rows_bound <= 0) return;
    switch (a.epi) {
        case kEpiStoreF32: launch_phases<kEpiStoreF32, kEpiStoreF32>(a, nullptr, s); break;
        case kEpiResidAdd: launch_phases<kEpiResidAdd, kEpiStoreF32>(a, nullptr, s); break;
        case kEpiTanh: launch_phases<kEpiTanh, kEpiStoreF32>(a, nullptr, s); break;
        case kEpiSwiglu: launch_phases<kEpiSwiglu, kEpiStoreF32>(a, nullptr, s); break;
    }
}

void launch_moe_tc(const TcGemmArgs& up, const TcGemmArgs& down, cudaStream_t s) {
    if (up.Nout <= 0 || up.rows_bound <= 0) return;
    if (!up.group_cnt || !up.done || up.G > kMaxGroups)
        throw Error(kInvariant, "fused expert GEMM: needs <= 64 groups and completion counters");
    if (down.epi != kEpiStoreF32 || down.group_cnt != up.group_cnt || down.seg != up.seg ||
        down.rows_bound != up.rows_bound)
        throw Error(kInvariant, "fused expert GEMM: down projection must share the up projection's groups");
    if (up.epi == kEpiSwiglu) launch_phases<kEpiSwiglu, kEpiStoreF32>(up, &down, s);
    else if (up.epi == kEpiTanh) launch_phases<kEpiTanh, kEpiStoreF32>(up, &down, s);
    else throw Error(kInvariant, "fused expert GEMM: up projection epilogue must be tanh or SwiGLU");
}

}  // namespace smoe

// Trace dump for tools/tc_trace.py (SMOE_TC_TRACE variant builds; returns -1 otherwise).
extern "C" int smoe_tc_trace_dump(const char* path) {
#ifdef SMOE_TC_TRACE
    using namespace smoe;
    std::vector<TrUnit> u((size_t)kTrLaunches * kTrUnits);
    std::vector<long long> c((size_t)kTrLaunches * kTrCtas * 2);
    std::vector<int> m((size_t)kTrLaunches * 4);
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    cudaMemcpyFromSymbol(u.data(), g_tr_unit, u.size() * sizeof(TrUnit));
    cudaMemcpyFromSymbol(c.data(), g_tr_cta, c.size() * sizeof(long long));
    cudaMemcpyFromSymbol(m.data(), g_tr_meta, m.size() * sizeof(int));
    std::vector<long long> dep((size_t)kTrLaunches * kTrCtas);
    cudaMemcpyFromSymbol(dep.data(), g_tr_cta_dep, dep.size() * sizeof(long long));
    FILE* fp = fopen(path, "wb");
    if (!fp) return -3;
    int hdr[3] = {kTrLaunches, kTrUnits, kTrCtas};
    fwrite(hdr, sizeof(hdr), 1, fp);
    fwrite(m.data(), sizeof(int), m.size(), fp);
    fwrite(c.data(), sizeof(long long), c.size(), fp);
    fwrite(u.data(), sizeof(TrUnit), u.size(), fp);
    fwrite(dep.data(), sizeof(long long), dep.size(), fp);
    fclose(fp);
    return 0;
#else
    (void)path;
    return -1;
#endif
}
