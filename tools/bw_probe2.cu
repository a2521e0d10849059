// bw_probe2.cu -- does a pre-tiled expert-weight layout stream faster than the row-major one?
// One persistent CTA per SM, one producer thread, a ring of S stages of 32 KB (the fused MoE kernel's
// pair-unit weight box: 256 rows x 64 bf16), each CTA walking whole units of 256 rows x K (a slab):
//   (a) 2D TMA box {64, 256} over a row-major [rows][K] pool       -- the current layout
//   (b) 3D TMA box {64, 256, 1} over a pre-tiled pool, box = 32 KB contiguous ([unit][kb][256][64])
//   (c) 1D cp.async.bulk of the same contiguous 32 KB boxes
// Both TMA variants use the 128B swizzle, so (b) lands in shared memory exactly like (a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/bw_probe2 tools/bw_probe2.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    uint32_t d = 0;
    while (!d) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory");
}

constexpr int kBox = 32768;

template <int MODE>
__global__ void __launch_bounds__(32, 1) k_stream(const __grid_constant__ CUtensorMap map, const char* base, int nkb,
                                                  int units, int stages, int* ctr) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint64_t* full = (uint64_t*)(buf + stages * kBox);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) mb_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    long long it = 0;
    for (;;) {
        const int u = atomicAdd(ctr, 1);  // dynamic unit claims, like the GEMM
        if (u >= units) break;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = (int)(it % stages);
            if (it >= stages) mb_wait(&full[s], ((it / stages) - 1) & 1);  // slot's previous load landed
            mb_tx(&full[s], kBox);
            if (MODE == 0) {
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(su(buf + s * kBox)), "l"(&map), "r"(su(&full[s])), "r"(kb * 64), "r"(u * 256) : "memory");
            } else if (MODE == 1) {
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                             ::"r"(su(buf + s * kBox)), "l"(&map), "r"(su(&full[s])), "r"(0), "r"(0), "r"(u * nkb + kb) : "memory");
            } else {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %3, [%2];"
                             ::"r"(su(buf + s * kBox)), "l"(base + ((long long)u * nkb + kb) * kBox), "r"(su(&full[s])), "r"(kBox) : "memory");
            }
        }
    }
    for (long long j = it - stages; j < it; ++j) if (j >= 0) mb_wait(&full[j % stages], (j / stages) & 1);
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t bytes = 4ull << 30;
    char* pool;
    int* ctr;
    CK(cudaMalloc(&pool, bytes));
    CK(cudaMalloc(&ctr, 4));
    CK(cudaMemset(pool, 1, bytes));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int K : {4096, 2048, 14336}) {
        const long long rows = bytes / 2 / K;
        const int nkb = K / 64;
        const int units = (int)(rows / 256);
        CUtensorMap m2, m3;
        {
            cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
            cuuint64_t str[1] = {(cuuint64_t)K * 2};
            cuuint32_t box[2] = {64, 256}, es[2] = {1, 1};
            ((Enc)fn)(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        {
            const long long chunks = (long long)units * nkb;
            cuuint64_t dims[3] = {64, 256, (cuuint64_t)chunks};
            cuuint64_t str[2] = {128, kBox};
            cuuint32_t box[3] = {64, 256, 1}, es[3] = {1, 1, 1};
            CUresult r = ((Enc)fn)(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, pool, dims, str, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) printf("3D map encode failed %d\n", (int)r);
        }
        for (int stages : {4, 6}) {
            const size_t smem = (size_t)stages * kBox + 2048;
            CK(cudaFuncSetAttribute(k_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            for (int grid : {sms, 88}) {
                for (int mode = 0; mode < 3; ++mode) {
                    cudaEvent_t a, b;
                    cudaEventCreate(&a);
                    cudaEventCreate(&b);
                    float best = 1e9;
                    for (int rep = 0; rep < 5; ++rep) {
                        CK(cudaMemset(ctr, 0, 4));
                        cudaEventRecord(a);
                        if (mode == 0) k_stream<0><<<grid, 32, smem>>>(m2, pool, nkb, units, stages, ctr);
                        else if (mode == 1) k_stream<1><<<grid, 32, smem>>>(m3, pool, nkb, units, stages, ctr);
                        else k_stream<2><<<grid, 32, smem>>>(m3, pool, nkb, units, stages, ctr);
                        cudaEventRecord(b);
                        CK(cudaEventSynchronize(b));
                        float ms;
                        cudaEventElapsedTime(&ms, a, b);
                        if (ms < best) best = ms;
                    }
                    const char* names[3] = {"2D TMA {64,256} row-major", "3D TMA pre-tiled 32KB", "bulk pre-tiled 32KB"};
                    printf("K=%5d stages=%d grid=%3d %-28s %.1f GB/s\n", K, stages, grid, names[mode],
                           (double)units * nkb * kBox / (best * 1e-3) / 1e9);
                }
            }
        }
    }
    return 0;
}
