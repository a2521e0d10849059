// common.cuh -- shared device/host definitions for the B200 spec-decode engine.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>
#include <utility>

namespace smoe {

// Status codes returned through the C ABI: mirror the reference's exit codes
// (common.hpp:12-21: ConfigError -> 1, InvariantError -> 2) plus 3 for CUDA/NCCL failures.
enum Status : int { kOk = 0, kConfig = 1, kInvariant = 2, kCuda = 3 };

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SMOE_CUDA(x)                                                                               \
    do {                                                                                           \
        cudaError_t e__ = (x);                                                                     \
        if (e__ != cudaSuccess)                                                                    \
            throw ::smoe::Error(::smoe::kCuda, std::string(#x) + ": " + cudaGetErrorString(e__) + \
                                                   " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

// Weight / operand storage types.
enum WType : int { kF32 = 0, kBF16 = 1 };

// Expert FFN forms: tanh2 = reference (model.cpp:54-59), swiglu3 = Mixtral.
enum ExpertKind : int { kTanh2 = 0, kSwiglu3 = 1 };

// GEMM epilogues.
enum Epi : int {
    kEpiStoreF32 = 0,   // Y[f32] = acc
    kEpiResidAdd = 1,   // Y[f32] += acc                    (mix: x += Mix rms(x))
    kEpiTanh = 2,       // Y[op]  = tanh(acc)               (tanh2 up projection)
    kEpiSwiglu = 3,     // Y[op]  = silu(acc_w1) * acc_w3   (swiglu3 gated up projection)
};

// Device-resident error flag bits (checked once per phase, SURVEY 5 failure detection).
enum Flag : int { kFlagNonFiniteLogits = 1, kFlagEmptyRemap = 2, kFlagNonFiniteGate = 4, kFlagZeroDrawProb = 8 };

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {  // common.hpp:27-32
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__host__ __device__ inline uint64_t substream(uint64_t seed, uint64_t t0, uint64_t t1 = 0) {  // common.hpp:35-37
    return splitmix64(seed ^ splitmix64(t0 ^ splitmix64(t1)));
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Pinned float arithmetic for the row reductions shared by the per-layer kernels (kernels.cu) and the
// pass kernel (pass_tc.cu): both evaluate exactly these operations in exactly the same reduction tree,
// so a row's results are bit-identical whichever launch strategy computed it.
#ifdef __CUDACC__
__device__ __forceinline__ float sumsq4(const float4 v) {
    return __fmaf_rn(v.w, v.w, __fmaf_rn(v.z, v.z, __fmaf_rn(v.y, v.y, __fmul_rn(v.x, v.x))));
}
__device__ __forceinline__ float dot4f(const float4 a, const float4 b) {
    return __fmaf_rn(a.w, b.w, __fmaf_rn(a.z, b.z, __fmaf_rn(a.y, b.y, __fmul_rn(a.x, b.x))));
}
__device__ __forceinline__ void axpy4(float4& acc, float w, const float4 y) {
    acc.x = __fmaf_rn(w, y.x, acc.x);
    acc.y = __fmaf_rn(w, y.y, acc.y);
    acc.z = __fmaf_rn(w, y.z, acc.z);
    acc.w = __fmaf_rn(w, y.w, acc.w);
}
#endif
// threads per row of the per-layer row kernels (and the virtual block the pass kernel emulates)
__host__ __device__ inline int row_threads(int d) { return d >= 4096 ? 1024 : d >= 1024 ? 512 : 256; }
// threads of the gate kernel (K4-K6): at least one warp per expert (up to 1024), so each warp computes one
// gate logit instead of several in sequence (E=64 at d=2048: 1024 instead of 512)
__host__ __device__ inline int gate_threads(int d, int E) {
    const int t = E * 32 < 1024 ? E * 32 : 1024;
    return t > row_threads(d) ? t : row_threads(d);
}

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Kernel attributes (cudaFuncSetAttribute) are per device: true the first time the calling thread's
// current device asks, so a launch helper configures each kernel once on every device it runs on.
inline bool first_use_on_device(std::atomic<uint64_t>& seen) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (seen.load(std::memory_order_acquire) & bit) return false;
    seen.fetch_or(bit, std::memory_order_acq_rel);
    return true;
}

// Programmatic dependent launch (PDL).  Every hot-path kernel starts with pdl_wait() (no-op when not
// launched with the PDL attribute) before touching memory written by earlier kernels, then
// pdl_trigger() so the next kernel's CTAs may be scheduled as SMs free up and run their prologue
// (barrier init, TMEM alloc, static weight prefetch) under this kernel's tail.  Triggering before the
// wait would let a kernel two launches later become resident while an earlier one still runs (the
// GEMM launches alternate between two scheduler slots, which relies on at most two in flight).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

extern bool g_use_pdl;  // engine-wide switch (env SMOE_PDL=0 disables), defined in kernels.cu

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// launch_k with a thread-block cluster of `cluster` CTAs along x (1: none)
template <typename... KArgs, typename... Args>
inline void launch_kc(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                      Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (g_use_pdl) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (cluster > 1) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = cluster;
        at[n].val.clusterDim.y = 1;
        at[n++].val.clusterDim.z = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace smoe
