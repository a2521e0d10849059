// gemm_tc.cu -- grouped "swap-AB" GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Decode-size expert GEMMs have few tokens per expert (n_e = 1..160) and a huge weight matrix, so
// the weights take the MMA M slot (128 rows per tile) and the tokens the N slot (BN = 32..256):
//   D[feature m][token n] (TMEM, f32) = sum_k W[slot][m][k] * X[row n][k]
// One CTA computes one (expert group, 128-feature tile, BN-token tile):
//   warp 0     : TMA producer -- 128x64 bf16 weight box (+ the matching w3 box for SwiGLU) and a
//                BNx64 activation box per stage, 128B-swizzled, multi-stage mbarrier ring;
//   warp 1     : allocates TMEM; one elected lane issues tcgen05.mma.kind::f16 (M=128, N=BN, K=16)
//                four times per stage and commits each stage back to the producer;
//   warps 2..5 : epilogue -- tcgen05.ld 32x32b.x16 from TMEM, activation (tanh / silu*mul) or
//                residual add, coalesced stores (32 consecutive features per warp per token).
// The K loop order is fixed and independent of T, and a column of D never depends on other columns,
// so every token row is computed identically in draft, verify and on-demand passes.
#include <cuda.h>

#include <map>
#include <mutex>
#include <tuple>

#include "engine.h"

namespace smoe {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 bytes = one swizzle atom row
constexpr int kThreads = 192;
constexpr int kMaxStages = 8;
constexpr int kABytes = BM * BK * 2;

struct TcParams {
    int Nout, K;
    long long a_rows_per_slot;
    const int* group_off;
    const int* group_slot;
    int single_rows, single_slot;
    void* Y;
    int ldy;
    int gate_off;  // SwiGLU: row offset of w3 inside a slot
    int stages;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Bounded wait: a descriptor or pipeline bug traps (kills the context with an error) instead of
// hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 20000000000ll) __trap();
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

// K-major operand tile in shared memory, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);  // start address
    d |= (uint64_t)1 << 16;                 // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;       // stride byte offset: next 8-row group
    d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
    return d;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
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

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TcParams p) {
    constexpr bool kGated = EPI == kEpiSwiglu;
    constexpr int kATiles = kGated ? 2 : 1;
    constexpr int kBBytes = BN * BK * 2;
    constexpr int kStageBytes = kATiles * kABytes + kBBytes;
    constexpr int kAccCols = kATiles * BN;
    constexpr int kTmemCols = kAccCols <= 32 ? 32 : kAccCols <= 64 ? 64 : kAccCols <= 128 ? 128 : kAccCols <= 256 ? 256 : 512;

    // ---- work item (uniform per CTA; empty tiles leave before touching any barrier)
    const int g = blockIdx.y;
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
    const int n0 = r0 + blockIdx.z * BN;
    if (slot < 0 || n0 >= r1) return;
    const int n_valid = min(BN, r1 - n0);
    const int m0 = blockIdx.x * BM;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int stages = p.stages;
    const int num_kb = (p.K + BK - 1) / BK;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStageBytes);
    uint64_t* empty = full + kMaxStages;
    uint64_t* acc_full = empty + kMaxStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
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

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            const int arow = (int)((long long)slot * p.a_rows_per_slot + m0);
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % stages;
                const uint32_t ph = (uint32_t)((kb / stages) & 1);
                mbar_wait(&empty[s], ph ^ 1u);
                uint8_t* st = smem + s * kStageBytes;
                mbar_expect_tx(&full[s], kStageBytes);
                tma_load_2d(&mapA, &full[s], st, kb * BK, arow);
                if (kGated) tma_load_2d(&mapA, &full[s], st + kABytes, kb * BK, arow + p.gate_off);
                tma_load_2d(&mapB, &full[s], st + kATiles * kABytes, kb * BK, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % stages;
                const uint32_t ph = (uint32_t)((kb / stages) & 1);
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a_base = smem_u32(smem + s * kStageBytes);
                const uint32_t b_base = a_base + kATiles * kABytes;
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk) {
                    const uint64_t bd = smem_desc(b_base + kk * 32);
                    const uint32_t accum = (kb | kk) ? 1u : 0u;
                    mma_bf16(tmem, smem_desc(a_base + kk * 32), bd, idesc, accum);
                    if (kGated) mma_bf16(tmem + BN, smem_desc(a_base + kABytes + kk * 32), bd, idesc, accum);
                }
                mma_commit(&empty[s]);  // stage free once these MMAs have read it
            }
            mma_commit(acc_full);  // accumulator complete
        }
        __syncwarp();
    } else {  // ---- epilogue: warps 2..5 cover TMEM lane quarters 2,3,0,1
        mbar_wait(acc_full, 0);
        tc_fence_after();
        const int q = warp & 3;
        const int m = m0 + q * 32 + lane;
        const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
        for (int c = 0; c < n_valid; c += 16) {
            uint32_t v[16], v3[16];
            tmem_ld16(lane_addr + c, v);
            if (kGated) tmem_ld16(lane_addr + BN + c, v3);
            tmem_wait_ld();
            if (m < p.Nout) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (c + j >= n_valid) break;
                    const long long o = (long long)(n0 + c + j) * p.ldy + m;
                    const float a = __uint_as_float(v[j]);
                    if (EPI == kEpiStoreF32) {
                        reinterpret_cast<float*>(p.Y)[o] = a;
                    } else if (EPI == kEpiResidAdd) {
                        reinterpret_cast<float*>(p.Y)[o] += a;
                    } else if (EPI == kEpiTanh) {
                        reinterpret_cast<__nv_bfloat16*>(p.Y)[o] = __float2bfloat16_rn(tanhf(a));
                    } else {
                        const float b = __uint_as_float(v3[j]);
                        reinterpret_cast<__nv_bfloat16*>(p.Y)[o] = __float2bfloat16_rn(a / (1.0f + expf(-a)) * b);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
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

template <int BN, int EPI>
void launch_bn_epi(const TcGemmArgs& a, cudaStream_t s) {
    constexpr int kATiles = EPI == kEpiSwiglu ? 2 : 1;
    constexpr int kStageBytes = kATiles * kABytes + BN * BK * 2;
    const int budget = 224 * 1024 - 1024 - 256;
    int stages = std::min(kMaxStages, budget / kStageBytes);
    const int num_kb = (a.K + BK - 1) / BK;
    stages = std::max(2, std::min(stages, std::max(2, num_kb)));
    const size_t smem = (size_t)stages * kStageBytes + 1024 + 256;
    static bool configured = false;
    if (!configured) {
        SMOE_CUDA(cudaFuncSetAttribute(k_gemm_tc<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       224 * 1024));
        configured = true;
    }
    TcParams p{a.Nout, a.K, a.a_rows_per_slot, a.group_off, a.group_slot, a.single_rows, a.single_slot, a.Y, a.ldy,
               a.Nout, stages};
    const CUtensorMap& ma = tensor_map(a.A, BM);
    const CUtensorMap& mb = tensor_map(a.B, BN);
    dim3 grid((a.Nout + BM - 1) / BM, a.group_off ? a.G : 1, (a.rows_bound + BN - 1) / BN);
    k_gemm_tc<BN, EPI><<<grid, kThreads, smem, s>>>(ma, mb, p);
}

template <int BN>
void launch_bn(const TcGemmArgs& a, cudaStream_t s) {
    switch (a.epi) {
        case kEpiStoreF32: launch_bn_epi<BN, kEpiStoreF32>(a, s); break;
        case kEpiResidAdd: launch_bn_epi<BN, kEpiResidAdd>(a, s); break;
        case kEpiTanh: launch_bn_epi<BN, kEpiTanh>(a, s); break;
        case kEpiSwiglu: launch_bn_epi<BN, kEpiSwiglu>(a, s); break;
    }
}

}  // namespace

void launch_gemm_tc(const TcGemmArgs& a, cudaStream_t s) {
    if (a.Nout <= 0 || a.rows_bound <= 0) return;
    // token tile: smallest of 32/64/128/256 covering the largest possible group (<= T rows)
    const int rb = a.rows_bound;
    if (rb <= 32) launch_bn<32>(a, s);
    else if (rb <= 64) launch_bn<64>(a, s);
    else if (rb <= 128) launch_bn<128>(a, s);
    else launch_bn<256>(a, s);
}

}  // namespace smoe
