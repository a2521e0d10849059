// bw_probe.cu -- does the weight layout limit HBM streaming?  Streams a 4 GiB bf16 "weight pool"
// into shared memory with a persistent 1-CTA-per-SM producer ring (no compute), two ways:
//   (a) 2D TMA boxes of 128 rows x 64 bf16 (128 B per row, rows K*2 bytes apart) -- current layout
//   (b) cp.async.bulk of contiguous 16 KB chunks                             -- pre-tiled layout
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
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

template <int MODE>
__global__ void __launch_bounds__(32, 1) k_stream(const __grid_constant__ CUtensorMap map, const char* base, int K,
                                                  long long tiles, int stages, int G = 1) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    uint64_t* full = (uint64_t*)(buf + (stages < 0 ? -stages : stages) * 16384);
    if (threadIdx.x == 0) {
        for (int s = 0; s < (stages < 0 ? -stages : stages); ++s) mb_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int kb_per_row = K / 64;
    const int nst = stages < 0 ? -stages : stages;
    long long it = 0;
    const long long slabs = tiles / kb_per_row;
    for (long long i = 0;; ++i, ++it) {
        long long t;
        if (MODE == 9) {  // wave-interleaved tiled layout of width W=G; CTA c owns slabs c, c+grid, ...; optional holes
            const long long slab = blockIdx.x + (i / kb_per_row) * gridDim.x;
            if (slab >= slabs) break;
            const int j = (int)(i % kb_per_row);
            if (stages < 0 && ((slab / 224) & 1)) { --it; continue; }  // (holes: every other 224-slab "expert")
            t = ((slab / G) * kb_per_row * G) + (long long)j * G + (slab % G);
        } else if (MODE == 8) {  // each CTA streams G slabs at once, k-blocks alternating between them
            const long long grp = i / ((long long)kb_per_row * G);           // which group of G slabs
            const int within = (int)(i % ((long long)kb_per_row * G));
            const int which = within % G, kb = within / G;
            const long long slab = ((long long)blockIdx.x + grp * gridDim.x) * G + which;
            if (((long long)blockIdx.x + grp * gridDim.x) * G >= slabs) break;
            if (slab >= slabs) { --it; continue; }  // no ring slot consumed
            t = slab * kb_per_row + kb;
        } else if (MODE == 7) {  // slab per CTA, k-blocks visited with stride P (0, P, 2P, ..., 1, P+1, ...)
            const long long slab = blockIdx.x + (i / kb_per_row) * gridDim.x;
            if (slab >= slabs) break;
            const int j = (int)(i % kb_per_row), per = kb_per_row / G;
            t = slab * kb_per_row + (j % per) * G + j / per;
        } else if (MODE == 6) {  // groups of G CTAs share a slab; member m streams k-blocks m, m+G, m+2G, ...
            const int per = kb_per_row / G;
            const long long groups = gridDim.x / G;
            const long long g = blockIdx.x / G, m = blockIdx.x % G;
            const long long slab = g + (i / per) * groups;
            if (g >= groups || slab >= slabs) break;
            t = slab * kb_per_row + m + (i % per) * G;
        } else if (MODE == 5) {  // groups of G CTAs share a slab; member m streams k-blocks [m*kb/G, (m+1)*kb/G)
            const int per = kb_per_row / G;
            const long long groups = gridDim.x / G;
            const long long g = blockIdx.x / G, m = blockIdx.x % G;
            const long long slab = g + (i / per) * groups;
            if (g >= groups || slab >= slabs) break;
            t = slab * kb_per_row + m * per + (i % per);
        } else if (MODE == 4) {  // slab per CTA, but chunk j of slab u stored at (j * slabs + u) * 16 KB
            const long long slab = blockIdx.x + (i / kb_per_row) * gridDim.x;
            if (slab >= slabs) break;
            t = (i % kb_per_row) * slabs + slab;
        } else if (MODE <= 1) {  // interleaved: consecutive tiles on consecutive CTAs
            t = blockIdx.x + i * gridDim.x;
            if (t >= tiles) break;
        } else {          // GEMM order: CTA walks whole 128-row slabs along K
            const long long slab = blockIdx.x + (i / kb_per_row) * gridDim.x;
            if (slab >= slabs) break;
            t = slab * kb_per_row + (i % kb_per_row);
        }
        const int s = it % (stages < 0 ? -stages : stages);
        if (it >= nst) mb_wait(&full[s], ((it / nst) - 1) & 1);  // slot consumed (data landed)
        mb_tx(&full[s], 16384);
        if (MODE == 0 || MODE == 2 || MODE == 5 || MODE == 6 || MODE == 7 || MODE == 8) {  // 2D box (else bulk)
            const int kb = (int)(t % kb_per_row), rt = (int)(t / kb_per_row);
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                         ::"r"(su(buf + s * 16384)), "l"(&map), "r"(su(&full[s])), "r"(kb * 64), "r"(rt * 128) : "memory");
        } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];"
                         ::"r"(su(buf + s * 16384)), "l"(base + t * 16384), "r"(su(&full[s])) : "memory");
        }
    }
    for (long long j = it - nst; j < it; ++j) if (j >= 0) mb_wait(&full[j % nst], (j / nst) & 1);
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t bytes = 4ull << 30;
    char* pool;
    CK(cudaMalloc(&pool, bytes));
    CK(cudaMemset(pool, 1, bytes));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int prom = 0; prom < 1; ++prom)
    for (int K : {4096, 14336}) {
        const long long rows = bytes / 2 / K;
        CUtensorMap map;
        printf("--- L2 promotion %s\n", prom == 0 ? "256B" : prom == 1 ? "128B" : "none");
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
        cuuint64_t str[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
        ((Enc)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, pool, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B,
                  prom == 0 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : prom == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                            : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const long long tiles = (rows / 128) * (K / 64);
        for (int stages : {8}) {
            size_t smem = stages * 16384 + 1024 + 256;
            CK(cudaFuncSetAttribute(k_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            CK(cudaFuncSetAttribute(k_stream<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            for (int G : {1, 8, 16, 64, 128, -8, -16, -128}) {
                const int W = G < 0 ? -G : G;
                const int st = G < 0 ? -stages : stages;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaEventRecord(a);
                    k_stream<9><<<sms, 32, smem>>>(map, pool, K, tiles, st, W);
                    cudaEventRecord(b);
                    CK(cudaEventSynchronize(b));
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                const double frac = G < 0 ? 0.5 : 1.0;  // holes skip every other 224-slab block (approx.)
                printf("K=%5d stages=%2d bulk wave-interleaved W=%3d%s %.1f GB/s\n", K, stages, W, G < 0 ? " (half experts idle)" : "",
                       frac * tiles * 16384.0 / (best * 1e-3) / 1e9);
            }
            for (int G : {2}) { if (G) break;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                float best = 1e9;
                const int grid = (sms / G) * G;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaEventRecord(a);
                    k_stream<6><<<grid, 32, smem>>>(map, pool, K, tiles, stages, G);
                    cudaEventRecord(b);
                    CK(cudaEventSynchronize(b));
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                const long long per = (K / 64) / G, done = ((tiles / (K / 64)) / (grid / G)) * (grid / G) * per * G;
                printf("K=%5d stages=%2d 2D TMA, %2d CTAs/slab k-interleaved %.1f GB/s\n", K, stages, G,
                       done * 16384.0 / (best * 1e-3) / 1e9);
            }
            for (int mode = 1; mode < 4; mode += 2) {
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaEventRecord(a);
                    if (mode == 0) k_stream<0><<<sms, 32, smem>>>(map, pool, K, tiles, stages);
                    else if (mode == 1) k_stream<1><<<sms, 32, smem>>>(map, pool, K, tiles, stages);
                    else if (mode == 2) k_stream<2><<<sms, 32, smem>>>(map, pool, K, tiles, stages);
                    else if (mode == 3) k_stream<3><<<sms, 32, smem>>>(map, pool, K, tiles, stages);
                    else k_stream<4><<<sms, 32, smem>>>(map, pool, K, tiles, stages);
                    cudaEventRecord(b);
                    CK(cudaEventSynchronize(b));
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (ms < best) best = ms;
                }
                const char* names[5] = {"2D TMA, interleaved", "bulk 16KB, interleaved", "2D TMA, slab per CTA",
                                        "bulk 16KB, slab per CTA", "bulk, kb-major, slab/CTA"};
                printf("K=%5d stages=%2d %-24s %.1f GB/s\n", K, stages, names[mode],
                       tiles * 16384.0 / (best * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
