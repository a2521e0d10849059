// gate_dev.cuh -- K5/K6 selection shared by k_gate (kernels.cu) and the pass kernel (pass_tc.cu):
// softmax (model.cpp:145-157), top-K with ties -> lower index (model.cpp:159-170), restricted-mode
// remap (drafting.cpp:123-151) and the dispatch of each pick into its expert's segment.
#pragma once
#include "kernels.h"

namespace smoe {

// Called by ONE full warp for row r.  gl[0..E) = gate logits incl. bias; gl[E..2E) is scratch for
// the softmax numerators.  Writes raw/fin/wgt/pos of row r and dst[k] = the xperm row of pick k.
// The draft tables come as shared-memory copies (in_draft == nullptr: target semantics); `a` stays the
// kernel parameter (a local copy of GateArgs would turn every field read into a local-memory load).
__device__ __forceinline__ void gate_select_warp(const GateArgs& a, int r, float* gl, int* dst, const int* s_rank,
                                                 const int* s_sorted, const uint8_t* in_draft) {
    const int lane = threadIdx.x & 31, E = a.E, K = a.K;
    {
        const unsigned FULL = 0xffffffffu;
        const int l0 = lane, l1 = lane + 32;
        const float g0 = l0 < E ? gl[l0] : 0.f, g1 = l1 < E ? gl[l1] : 0.f;
        const bool fin_ok = (l0 >= E || isfinite(g0)) && (l1 >= E || isfinite(g1));
        if (!__all_sync(FULL, fin_ok) && lane == 0) atomicOr(a.flags, kFlagNonFiniteGate);
        // softmax (model.cpp:145-157), max-subtracted; the max is exact in any order, the sum runs in
        // expert order on lane 0
        float mx = fmaxf(l0 < E ? g0 : -INFINITY, l1 < E ? g1 : -INFINITY);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
        float* p = gl + E;
        if (l0 < E) p[l0] = expf(g0 - mx);
        if (l1 < E) p[l1] = expf(g1 - mx);
        __syncwarp();
        // the sum in expert order on lane 0, its loads issued ahead of the dependent adds
        float sum = 0.f;
        if (lane == 0) {
            int e = 0;
            for (; e + 8 <= E; e += 8) {
                float q[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) q[j] = p[e + j];
#pragma unroll
                for (int j = 0; j < 8; ++j) sum += q[j];
            }
            for (; e < E; ++e) sum += p[e];
        }
        sum = __shfl_sync(FULL, sum, 0);
        // top-K (model.cpp:159-170: K rounds of first-max, ties -> lower index) as ranks: expert e is pick
        // rank(e) = #{e' : g[e'] > g[e] or (g[e'] == g[e] and e' < e)} -- the same order, found with one
        // pass of independent compares instead of K dependent warp reductions.  (Non-finite logits have
        // raised the flag above, which fails the pass; their picks only need to be in range.)
        int r0 = 0, r1 = 0;
        int e = 0;
        for (; e + 8 <= E; e += 8) {
            float q[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) q[j] = gl[e + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                r0 += (q[j] > g0) | ((q[j] == g0) & (e + j < l0));
                r1 += (q[j] > g1) | ((q[j] == g1) & (e + j < l1));
            }
        }
        for (; e < E; ++e) {
            const float ge = gl[e];
            r0 += (ge > g0) | ((ge == g0) & (e < l0));
            r1 += (ge > g1) | ((ge == g1) & (e < l1));
        }
        unsigned long long chosen = 0ull;
        int my_pick = 0, my_ex = 0;  // lane k keeps pick k
        for (int k = 0; k < K; ++k) {
            const unsigned b0 = __ballot_sync(FULL, l0 < E && r0 == k), b1 = __ballot_sync(FULL, l1 < E && r1 == k);
            const int pick = b0 ? __ffs(b0) - 1 : (b1 ? 32 + __ffs(b1) - 1 : k);
            int ex = pick;
            if (in_draft && !(in_draft[pick] && !((chosen >> pick) & 1ull))) {
                // restricted (draft) semantics: remap into draft \ chosen (drafting.cpp:123-151)
                ex = -1;
                if (a.use_affinity) {
                    // nearest by (distance, index) = first rank entry not yet chosen; -1 pads short sets
                    for (int j0 = 0; j0 < a.N && ex < 0; j0 += 32) {
                        const int j = j0 + lane;
                        const int c = j < a.N ? s_rank[pick * a.N + j] : -1;
                        const unsigned pad = __ballot_sync(FULL, j < a.N && c < 0);
                        const unsigned ok = __ballot_sync(FULL, j < a.N && c >= 0 && !((chosen >> c) & 1ull));
                        const unsigned before_pad = pad ? (1u << (__ffs(pad) - 1)) - 1u : FULL;
                        const unsigned m = ok & before_pad;
                        if (m) ex = __shfl_sync(FULL, c, __ffs(m) - 1);
                        if (pad) break;
                    }
                } else {  // hash surrogate (drafting.cpp:140-151): want-th non-chosen draft member
                    int total = 0;
                    for (int j0 = 0; j0 < a.N; j0 += 32) {
                        const int j = j0 + lane;
                        const int c = j < a.N ? s_sorted[j] : -1;
                        total += __popc(__ballot_sync(FULL, c >= 0 && !((chosen >> c) & 1ull)));
                    }
                    if (total > 0) {
                        const uint64_t h = substream(0x5eed5eedull, ((uint64_t)a.moe_ordinal << 32) | (uint32_t)pick,
                                                     (uint64_t)a.row_plen[r]);
                        int want = (int)(h % (uint64_t)total);
                        for (int j0 = 0; j0 < a.N && ex < 0; j0 += 32) {
                            const int j = j0 + lane;
                            const int c = j < a.N ? s_sorted[j] : -1;
                            unsigned m = __ballot_sync(FULL, c >= 0 && !((chosen >> c) & 1ull));
                            const int n = __popc(m);
                            if (want < n) {
                                for (int q = 0; q < want; ++q) m &= m - 1;  // drop the lowest `want` members
                                ex = __shfl_sync(FULL, c, __ffs(m) - 1);
                            } else {
                                want -= n;
                            }
                        }
                    }
                }
                if (ex < 0) {
                    if (lane == 0) atomicOr(a.flags, kFlagEmptyRemap);
                    ex = pick;
                }
            }
            chosen |= 1ull << ex;
            if (lane == k) {
                my_pick = pick;
                my_ex = ex;
            }
        }
        if (lane < K) {
            a.raw[r * K + lane] = my_pick;
            a.fin[r * K + lane] = my_ex;
            a.wgt[r * K + lane] = p[my_pick] / sum;  // the raw pick's weight, no renormalisation (model.cpp:249)
            // dispatch: lanes 0..K-1 claim their rows of the experts' segments concurrently
            const int row = my_ex * (a.seg > 0 ? a.seg : a.T) + atomicAdd(&a.cnt[my_ex], 1);
            a.pos[r * K + lane] = row;
            dst[lane] = row;
        }
        }
}

}  // namespace smoe
