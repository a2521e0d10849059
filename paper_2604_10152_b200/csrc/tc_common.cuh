// tc_common.cuh -- tcgen05 / TMEM / TMA / mbarrier building blocks shared by the grouped GEMM
// (gemm_tc.cu) and the persistent pass kernel (pass_tc.cu).  sm_100a only.
#pragma once
#include <cuda.h>

#include <cstdio>

#include "engine.h"

namespace smoe {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;        // 64 bf16 = 128 B = one swizzle-atom row
constexpr int BN_MAX = 256;   // max tokens per unit (MMA N)
#ifndef SMOE_BOX_N
#define SMOE_BOX_N 32  // 16 measured: no gain in the bench, slower at T=320 (profiles/r02_pass_kernel.md)
#endif
constexpr int BOX_N = SMOE_BOX_N;  // token rows per TMA box
constexpr int kThreads = 192;
constexpr int kMaxStages = 12;
constexpr int kABytes = BM * BK * 2;
constexpr int kBoxBytes = BOX_N * BK * 2;
constexpr int kTmemCols = 512;  // 2 accumulators x BN_MAX

constexpr int kRing = 8;        // unit ids published by the producer to the MMA / epilogue roles
constexpr int kMaxGroups = 64;  // completion counters per two-phase launch

struct Phase {
    int Nrows;  // valid weight rows per slot to compute (Nout, or 2*Nout for SwiGLU)
    long long a_rows_per_slot;
    int m_tiles, splits, kb_per_split, num_kb;
    void* Y;
    int ldy;
    long long split_stride;  // elements between split-K partial outputs
    // expert parallelism, fused return (kEpiStoreF32): group g's rows go straight into the return buffer
    // of rank g / peer_eo over peer memory, at the rows [(me*eo + g % eo) * seg, ...) it dispatched them from
    void* const* peer_y;
    int peer_eo, peer_me, peer_seg;
    int tiled;  // weight operand in the tiled layout (3D maps; coordinates {0, row & 255, (row >> 8) * num_kb + kb})
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// add tx bytes to the current phase without arriving (several fills, one arrive.expect_tx commits)
__device__ __forceinline__ void mbar_add_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: a pipeline bug traps (context error) instead of hanging the GPU.
__device__ __forceinline__ bool mbar_try(uint32_t addr, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    if (mbar_try(addr, parity)) return;  // fast path: no clock reads
    uint32_t done = 0;
    const long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 4000000000ll) {  // ~2 s
            printf("smoe mbar_wait timeout: block %d thread %d parity %u\n", (int)blockIdx.x, (int)threadIdx.x, parity);
            __trap();
        }
    }
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// same with an L2 eviction-priority policy (createpolicy): streamed-once weights as evict_first keep the
// L2 for what is re-read (activations, partials, the next layer's prefetched Mix weights)
__device__ __forceinline__ void tma_load_2d_hint(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
        "%4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
// 3D box of a tiled pool (kernels.h tiled_index): {0, row within the 256-row tile, chunk}
__device__ __forceinline__ void tma_load_3d_hint(const CUtensorMap* map, uint64_t* bar, void* dst, int c1, int c2,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, "
        "%4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(0), "r"(c1), "r"(c2), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(map), "r"(0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0), "r"(c1)
                 : "memory");
}
// 1D bulk copy global -> shared (async proxy), completion on an mbarrier; bytes % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void proxy_fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void proxy_fence_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ int ld_relaxed(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Wait until *c >= target.  Polls with relaxed loads (an acquire load costs an L1 invalidate per poll,
// which stalls the whole SM's memory pipe) and acquires once; traps after ~2 s (a lost publication).
__device__ __forceinline__ void spin_until(const int* c, int target) {
    const long long t0 = clock64();
    while (ld_relaxed(c) < target) {
        __nanosleep(32);
        if (clock64() - t0 > 4000000000ll) {
            printf("smoe spin_until timeout: block %d counter %d < %d\n", (int)blockIdx.x, ld_relaxed(c), target);
            __trap();
        }
    }
    fence_acquire();
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// K-major operand tile, 128-byte swizzle: 128-B rows, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, K-major, N>>3 at [17,23), M>>4 at [24,29).
__device__ __forceinline__ uint32_t idesc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}
// One 64-K stage of a pair unit in a single asm block: 2 tiles x 4 K=16 slices sharing the token operand
// (descriptors advance by 2 per slice).  One block lets ptxas move each operand into the uniform
// registers once instead of wrapping every tcgen05.mma in its own elect / R2UR sequence.
__device__ __forceinline__ void mma_stage_pair(uint32_t d0, uint32_t d1, uint64_t da, uint64_t da1, uint64_t db,
                                               uint32_t idesc, uint32_t accum_first) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 a1, a2, a3, c1, c2, c3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "add.s64 a1, %2, 2;\n\tadd.s64 a2, %2, 4;\n\tadd.s64 a3, %2, 6;\n\t"
        "add.s64 c1, %3, 2;\n\tadd.s64 c2, %3, 4;\n\tadd.s64 c3, %3, 6;\n\t"
        "add.s64 b1, %4, 2;\n\tadd.s64 b2, %4, 4;\n\tadd.s64 b3, %4, 6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %5, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %5, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, 1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %5, 1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %5, 1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c2, b2, %5, 1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %5, 1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c3, b3, %5, 1;\n\t}"
        ::"r"(d0), "r"(d1), "l"(da), "l"(da1), "l"(db), "r"(idesc), "r"(accum_first)
        : "memory");
}
__device__ __forceinline__ void mma_stage_single(uint32_t d0, uint64_t da, uint64_t db, uint32_t idesc,
                                                 uint32_t accum_first) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}"
        ::"r"(d0), "l"(da), "l"(db), "r"(idesc), "r"(accum_first)
        : "memory");
}
// One lane of a converged warp (the lowest active lane: lane 0 of a full warp, every time).
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred)
        :
        : "memory");
    return pred != 0;
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

struct Unit {
    int phase, g, slot, n0, n_valid, m0, kb0, kb1, ks, id;
    int pair;  // two 128-row tiles (gemm_tc.cu pair units)
};

// SwiGLU over a 32-column TMEM chunk (two x16 loads in flight).  Rows 2i / 2i+1 of the slot hold w1 / w3 of
// feature i: lanes 2i and 2i+1 split the chunk's tokens (even lane: tokens 0-15, odd lane: 16-31), trading the
// half they do not finish through one shuffle per token, so every lane computes 16 independent silu products
// (the 16-column form left the odd lanes idle and ran one dependent MUFU chain per token on the even lanes).
// Same fast-intrinsic formula per element as epilogue_store<kEpiSwiglu> (bit-identical H).
__device__ __forceinline__ void epilogue_swiglu32(const Phase& P, const Unit& w, int row, int lane, int c,
                                                  const uint32_t* v) {
    const bool odd = lane & 1;
    float a[16], b[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float mine_keep = __uint_as_float(odd ? v[16 + j] : v[j]);
        const float mine_send = __uint_as_float(odd ? v[j] : v[16 + j]);
        const float other = __shfl_xor_sync(0xffffffffu, mine_send, 1);
        a[j] = odd ? other : mine_keep;  // w1 (even row)
        b[j] = odd ? mine_keep : other;  // w3 (odd row)
    }
    if (row >= P.Nrows) return;
    const int t0 = c + (odd ? 16 : 0);
    __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(P.Y) + (long long)(w.n0 + t0) * P.ldy + (row >> 1);
    float h[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) h[j] = __fdividef(a[j], 1.0f + __expf(-a[j])) * b[j];
#pragma unroll
    for (int j = 0; j < 16; ++j)
        if (t0 + j < w.n_valid) y[(long long)j * P.ldy] = __float2bfloat16_rn(h[j]);
}

// One 16-column TMEM chunk of a finished accumulator -> the phase's output.
template <int EPI>
__device__ __forceinline__ void epilogue_store(const Phase& P, const Unit& w, int row, int lane, int c,
                                               const uint32_t* v) {
    if (EPI == kEpiSwiglu) {
        // rows 2j / 2j+1 of the slot hold w1 / w3 of feature j: pair up adjacent lanes.  silu with the
        // fast intrinsics (ex2.approx, approximate divide): each element is a fixed function of its
        // accumulator, so every pass computes it identically, and H is rounded to bf16 right after (the
        // <= 2-ulp f32 differences from expf/IEEE division vanish there).  The accurate-division path
        // serialised the 16 columns and made this epilogue the up->down critical path (9.7 us per C4
        // draft unit, tools/tc_trace.py).
        float other[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) other[j] = __shfl_xor_sync(0xffffffffu, __uint_as_float(v[j]), 1);
        if (!(lane & 1) && row < P.Nrows) {
            __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(P.Y) + (long long)(w.n0 + c) * P.ldy + (row >> 1);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float a = __uint_as_float(v[j]);
                const float h = __fdividef(a, 1.0f + __expf(-a)) * other[j];
                if (c + j < w.n_valid) y[(long long)j * P.ldy] = __float2bfloat16_rn(h);
            }
        }
    } else if (row < P.Nrows) {
        float* yf = reinterpret_cast<float*>(P.Y);
        long long n0 = w.n0;
        if (EPI == kEpiStoreF32 && P.peer_y) {
            yf = reinterpret_cast<float*>(P.peer_y[w.g / P.peer_eo]);
            n0 = (long long)(P.peer_me * P.peer_eo + w.g % P.peer_eo) * P.peer_seg + (w.n0 - (long long)w.g * P.peer_seg);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (c + j >= w.n_valid) break;
            const long long o = (long long)(w.n0 + c + j) * P.ldy + row;
            const float a = __uint_as_float(v[j]);
            if (EPI == kEpiStoreF32)
                yf[(n0 + c + j) * P.ldy + row + (long long)w.ks * P.split_stride] = a;
            else if (EPI == kEpiResidAdd)
                reinterpret_cast<float*>(P.Y)[o] += a;
            else
                reinterpret_cast<__nv_bfloat16*>(P.Y)[o] = __float2bfloat16_rn(tanhf(a));
        }
    }
}


// host: cached 2D tensor map (K-major bf16, 128B swizzle, box BK x box_rows); SM count
const CUtensorMap& tensor_map(const TcOperand& op, int box_rows);
int sm_count();
Phase make_phase(const TcGemmArgs& a);

}  // namespace tc
}  // namespace smoe
