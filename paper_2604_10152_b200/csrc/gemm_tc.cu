// gemm_tc.cu -- persistent grouped "swap-AB" GEMM on the 5th-generation tensor cores
// (tcgen05.mma + TMEM accumulators + TMA), the hot kernel of every pass.
//
// Decode-size expert GEMMs have few tokens per expert (n_e = 1..160) and large weight matrices, so
// the weights take the MMA M slot (128 rows per tile) and the tokens the N slot:
//   D[row m][token n] (TMEM, f32) = sum_k W[slot][m][k] * X[row n][k]
// Work unit = (group g, 128-row tile, token tile of <=256 rows, K split).  One CTA per SM walks the
// units round-robin; its roles run decoupled through mbarrier rings:
//   warp 0     TMA producer: one 128x64 bf16 weight box + ceil(n/32) 32x64 token boxes per stage
//              (token boxes sized by the group's real row count, 128B swizzle), multi-stage ring;
//   warp 1     owns TMEM (2 x 256 columns: double-buffered accumulator); one lane issues
//              tcgen05.mma.cta_group::1.kind::f16 with M=128, N=round16(n) (runtime instruction
//              descriptor), K=16, four per stage, and commits stages / finished accumulators;
//   warps 2-5  epilogue: tcgen05.ld.32x32b.x16 -> tanh | SwiGLU (w1/w3 rows interleaved, pairs
//              combined with one shuffle) | f32 store (optionally into a split-K partial) | residual
//              add, 32 consecutive rows per warp per token (coalesced), then release the accumulator.
// The epilogue of unit i overlaps the loads and MMAs of unit i+1.  The K order inside a unit and the
// split count are fixed per GEMM shape (never T-dependent) and a D column never depends on other
// columns, so every token row gets bit-identical results in draft, verify and on-demand passes.
#include <cuda.h>

#include <map>
#include <mutex>
#include <tuple>

#include "engine.h"

namespace smoe {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;        // 64 bf16 = 128 B = one swizzle-atom row
constexpr int BN_MAX = 256;   // max tokens per unit (MMA N)
constexpr int BOX_N = 32;     // token rows per TMA box
constexpr int kThreads = 192;
constexpr int kMaxStages = 12;
constexpr int kABytes = BM * BK * 2;
constexpr int kBoxBytes = BOX_N * BK * 2;
constexpr int kTmemCols = 512;  // 2 accumulators x BN_MAX

struct TcParams {
    int Nrows;  // valid weight rows per slot to compute (Nout, or 2*Nout for SwiGLU)
    int K;
    long long a_rows_per_slot;
    const int* group_off;
    const int* group_slot;
    int G, single_rows, single_slot;
    int m_tiles, n_tiles, splits, kb_per_split, num_kb;
    void* Y;
    int ldy;
    long long split_stride;  // elements between split-K partial outputs
    int stages, b_region;    // b_region = bytes of token boxes per stage
    int* sched;              // [2]: next-unit counter, finished-CTA counter (self-resetting)
};

constexpr int kRing = 8;  // unit ids published by the producer to the MMA / epilogue roles

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Bounded wait: a pipeline bug traps (context error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
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
        if (clock64() - t0 > 4000000000ll) __trap();  // ~2 s
    }
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

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

// Unit u -> (group, token tile, row tile, split); returns false for units with no rows.
struct Unit {
    int slot, n0, n_valid, m0, kb0, kb1, ks;
};
__device__ __forceinline__ bool decode_unit(const TcParams& p, int u, Unit& w) {
    int ks = u % p.splits;
    u /= p.splits;
    const int mt = u % p.m_tiles;
    u /= p.m_tiles;
    const int g = u % p.G;
    const int nt = u / p.G;
    int slot, r0, r1;
    if (p.group_off) {
        slot = p.group_slot[g];
        r0 = p.group_off[g];
        r1 = p.group_off[g + 1];
    } else {
        slot = p.single_slot;
        r0 = 0;
        r1 = p.single_rows;
    }
    w.n0 = r0 + nt * BN_MAX;
    if (slot < 0 || w.n0 >= r1) return false;
    w.slot = slot;
    w.n_valid = min(BN_MAX, r1 - w.n0);
    w.m0 = mt * BM;
    w.ks = ks;
    w.kb0 = ks * p.kb_per_split;
    w.kb1 = min(p.num_kb, w.kb0 + p.kb_per_split);
    return w.kb0 < w.kb1;
}

// Consumer side of the unit ring: returns false when the producer published "done".  whole_warp:
// all 32 lanes call this (epilogue warps; lane 0 releases the slot after the warp has read it);
// otherwise a single lane (the MMA issuer) calls it and releases the slot itself.
__device__ __forceinline__ bool next_unit(const TcParams& p, uint64_t* ring_full, uint64_t* ring_empty, const int* ring,
                                          int& cons, bool whole_warp, Unit& w) {
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
    decode_unit(p, u, w);
    return true;
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TcParams p) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int stages = p.stages;
    const int stage_bytes = kABytes + p.b_region;
    const int total_units = p.G * p.n_tiles * p.m_tiles * p.splits;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
    uint64_t* empty = full + kMaxStages;
    uint64_t* acc_full = empty + kMaxStages;  // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint64_t* ring_full = acc_empty + 2;      // [kRing]
    uint64_t* ring_empty = ring_full + kRing; // [kRing]
    int* ring = reinterpret_cast<int*>(ring_empty + kRing);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
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
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
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

    if (warp == 0) {
        if (lane == 0) {  // ---------------- scheduler + TMA producer
            int it = 0;
            bool first = true;
            for (int pub = 0;; ++pub) {
                // dynamic work distribution: claim the next non-empty unit (unit geometry comes from the
                // routing kernels, which completed before the kernel preceding this one could trigger)
                int u;
                Unit w;
                do {
                    u = atomicAdd(&p.sched[0], 1);
                } while (u < total_units && !decode_unit(p, u, w));
                const int r = pub % kRing;
                mbar_wait(&ring_empty[r], (uint32_t)(((pub / kRing) & 1) ^ 1));
                ring[r] = u < total_units ? u : -1;
                mbar_arrive(&ring_full[r]);
                if (u >= total_units) break;
                const int arow = (int)((long long)w.slot * p.a_rows_per_slot + w.m0);
                const int nb = (w.n_valid + BOX_N - 1) / BOX_N;
                const uint32_t bytes = kABytes + nb * kBoxBytes;
                int kb = w.kb0;
                if (first) {
                    // PDL: weights do not depend on the previous kernel -- stream the first stages' weight
                    // boxes while it drains, then wait for it before loading its activations.
                    const int pre = min(stages, w.kb1 - w.kb0);
                    for (int j = 0; j < pre; ++j) {
                        const int s = (it + j) % stages;
                        mbar_expect_tx(&full[s], bytes);
                        tma_load_2d(&mapA, &full[s], smem + s * stage_bytes, (kb + j) * BK, arow);
                    }
                    pdl_wait();
                    for (int j = 0; j < pre; ++j) {
                        const int s = (it + j) % stages;
                        uint8_t* st = smem + s * stage_bytes;
                        for (int q = 0; q < nb; ++q)
                            tma_load_2d(&mapB, &full[s], st + kABytes + q * kBoxBytes, (kb + j) * BK, w.n0 + q * BOX_N);
                    }
                    it += pre;
                    kb += pre;
                    first = false;
                }
                for (; kb < w.kb1; ++kb, ++it) {
                    const int s = it % stages;
                    mbar_wait(&empty[s], (uint32_t)(((it / stages) & 1) ^ 1));
                    uint8_t* st = smem + s * stage_bytes;
                    mbar_expect_tx(&full[s], bytes);
                    tma_load_2d(&mapA, &full[s], st, kb * BK, arow);
                    for (int j = 0; j < nb; ++j)
                        tma_load_2d(&mapB, &full[s], st + kABytes + j * kBoxBytes, kb * BK, w.n0 + j * BOX_N);
                }
            }
            if (first) pdl_wait();
        }
    } else if (warp == 1) {
        pdl_wait();
        if (lane == 0) {  // ---------------- MMA issuer
            int it = 0, cnt = 0, cons = 0;
            Unit w;
            while (next_unit(p, ring_full, ring_empty, ring, cons, false, w)) {
                const int acc = cnt & 1;
                mbar_wait(&acc_empty[acc], (uint32_t)(((cnt >> 1) & 1) ^ 1));
                tc_fence_after();
                const uint32_t d_tmem = tmem + (uint32_t)(acc * BN_MAX);
                const int nmma = (w.n_valid + 15) & ~15;
                const uint32_t idesc = idesc_bf16(BM, nmma);
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
    } else {  // -------------------------- epilogue: warps 2..5 -> TMEM lane quarters 2,3,0,1
        pdl_wait();
        const int q = warp & 3;
        int cnt = 0, cons = 0;
        Unit w;
        while (next_unit(p, ring_full, ring_empty, ring, cons, true, w)) {
            const int acc = cnt & 1;
            mbar_wait(&acc_full[acc], (uint32_t)((cnt >> 1) & 1));
            tc_fence_after();
            const int row = w.m0 + q * 32 + lane;  // weight row within the slot
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN_MAX);
            for (int c = 0; c < w.n_valid; c += 16) {
                uint32_t v[16];
                tmem_ld16(taddr + c, v);
                tmem_wait_ld();
                if (EPI == kEpiSwiglu) {
                    // rows 2j / 2j+1 of the slot hold w1 / w3 of feature j: pair up adjacent lanes
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float mine = __uint_as_float(v[j]);
                        const float other = __shfl_xor_sync(0xffffffffu, mine, 1);
                        if (!(lane & 1) && row < p.Nrows && c + j < w.n_valid) {
                            const float h = mine / (1.0f + expf(-mine)) * other;
                            reinterpret_cast<__nv_bfloat16*>(p.Y)[(long long)(w.n0 + c + j) * p.ldy + (row >> 1)] =
                                __float2bfloat16_rn(h);
                        }
                    }
                } else if (row < p.Nrows) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        if (c + j >= w.n_valid) break;
                        const long long o = (long long)(w.n0 + c + j) * p.ldy + row;
                        const float a = __uint_as_float(v[j]);
                        if (EPI == kEpiStoreF32)
                            reinterpret_cast<float*>(p.Y)[o + (long long)w.ks * p.split_stride] = a;
                        else if (EPI == kEpiResidAdd)
                            reinterpret_cast<float*>(p.Y)[o] += a;
                        else
                            reinterpret_cast<__nv_bfloat16*>(p.Y)[o] = __float2bfloat16_rn(tanhf(a));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
            ++cnt;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {  // last CTA out resets the scheduler for the next launch on this stream
        __threadfence();
        if (atomicAdd(&p.sched[1], 1) == (int)gridDim.x - 1) {
            p.sched[0] = 0;
            p.sched[1] = 0;
            __threadfence();
        }
    }
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// ------------------------------------------------------------------ host side
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
    static std::map<std::tuple<const void*, long long, int, int>, CUtensorMap> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(op.base, op.rows, op.K, box_rows);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    EncodeTiledFn fn = encode_fn();
    if (!fn) throw Error(kCuda, "cuTensorMapEncodeTiled entry point unavailable");
    CUtensorMap m;
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

template <int EPI>
void launch_epi(const TcGemmArgs& a, cudaStream_t s) {
    constexpr int kSmemBudget = 220 * 1024;
    static bool configured = false;
    if (!configured) {
        SMOE_CUDA(cudaFuncSetAttribute(k_gemm_tc<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        configured = true;
    }
    TcParams p{};
    p.Nrows = EPI == kEpiSwiglu ? 2 * a.Nout : a.Nout;
    p.K = a.K;
    p.a_rows_per_slot = a.a_rows_per_slot;
    p.group_off = a.group_off;
    p.group_slot = a.group_slot;
    p.G = a.group_off ? a.G : 1;
    p.single_rows = a.single_rows;
    p.single_slot = a.single_slot;
    p.m_tiles = (p.Nrows + BM - 1) / BM;
    p.n_tiles = (a.rows_bound + BN_MAX - 1) / BN_MAX;
    p.num_kb = (a.K + BK - 1) / BK;
    p.splits = std::max(1, std::min(a.splits, p.num_kb));
    p.kb_per_split = (p.num_kb + p.splits - 1) / p.splits;
    p.Y = a.Y;
    p.ldy = a.ldy;
    p.split_stride = a.split_stride;
    const int nb_max = (std::min(a.rows_bound, BN_MAX) + BOX_N - 1) / BOX_N;
    p.b_region = nb_max * kBoxBytes;
    const int stage_bytes = kABytes + p.b_region;
    p.stages = std::max(2, std::min(kMaxStages, (kSmemBudget - 1024 - 512) / stage_bytes));
    p.sched = a.sched;
    const size_t smem = (size_t)p.stages * stage_bytes + 1024 + 512;
    const CUtensorMap& ma = tensor_map(a.A, BM);
    const CUtensorMap& mb = tensor_map(a.B, BOX_N);
    const int units = p.G * p.n_tiles * p.m_tiles * p.splits;
    const int grid = std::max(1, std::min(units, sm_count()));
    launch_k(k_gemm_tc<EPI>, grid, kThreads, smem, s, ma, mb, p);
}

}  // namespace

void launch_gemm_tc(const TcGemmArgs& a, cudaStream_t s) {
    if (a.Nout <= 0 || a.rows_bound <= 0) return;
    switch (a.epi) {
        case kEpiStoreF32: launch_epi<kEpiStoreF32>(a, s); break;
        case kEpiResidAdd: launch_epi<kEpiResidAdd>(a, s); break;
        case kEpiTanh: launch_epi<kEpiTanh>(a, s); break;
        case kEpiSwiglu: launch_epi<kEpiSwiglu>(a, s); break;
    }
}

}  // namespace smoe
