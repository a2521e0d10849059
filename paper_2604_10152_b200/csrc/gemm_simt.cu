// gemm_simt.cu -- grouped skinny GEMM on CUDA cores.
//
// Used for the fp32 parity mode (fp32 weights and activations, FFMA, sequential
// per-lane reductions -- the mode whose routing/tokens are compared bit-exactly with the float64
// reference) and as the independent cross-check of the tcgen05 kernel in bf16 mode.  One warp owns
// RPW output features and walks K with 16-byte weight loads; lane partial sums are combined by a
// fixed butterfly, so every output element is reduced in the same order whatever T is (batch
// invariance).
#include <math.h>

#include "kernels.h"

namespace smoe {
namespace {

constexpr int kWarps = 8;
constexpr int kRPW = 2;  // output features per warp
constexpr int kTok = 4;  // tokens per pass over the weights

template <typename T>
__device__ __forceinline__ void load_vec(const T* p, float* out);
template <>
__device__ __forceinline__ void load_vec<float>(const float* p, float* out) {
    float4 v = *reinterpret_cast<const float4*>(p);
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
}
template <>
__device__ __forceinline__ void load_vec<__nv_bfloat16>(const __nv_bfloat16* p, float* out) {
    uint4 v = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 f = __bfloat1622float2(h[i]);
        out[2 * i] = f.x;
        out[2 * i + 1] = f.y;
    }
}

template <typename T, int EPI>
__global__ void __launch_bounds__(kWarps * 32) k_gemm_simt(GemmArgs a) {
    constexpr int VEC = 16 / sizeof(T);
    constexpr bool kGated = EPI == kEpiSwiglu;
    pdl_wait();
    pdl_trigger();
    const int g = blockIdx.y;
    const int slot = a.group_cnt ? a.group_slot[g] : a.single_slot;
    if (slot < 0) return;
    const int r0 = a.group_cnt ? g * a.seg : 0;
    const int r1 = a.group_cnt ? r0 + a.group_cnt[g] : a.single_rows;
    if (r1 <= r0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = (blockIdx.x * kWarps + warp) * kRPW;
    if (n0 >= a.Nout) return;
    const T* Wb = reinterpret_cast<const T*>(a.W) + (long long)slot * a.slot_stride;
    const T* X = reinterpret_cast<const T*>(a.X);
    const int K = a.K;

    for (int t0 = r0; t0 < r1; t0 += kTok) {
        float acc[kRPW][kTok];
        float acc3[kGated ? kRPW : 1][kTok];
#pragma unroll
        for (int i = 0; i < kRPW; ++i)
#pragma unroll
            for (int j = 0; j < kTok; ++j) {
                acc[i][j] = 0.f;
                if (kGated) acc3[i][j] = 0.f;
            }
        for (int k = lane * VEC; k < K; k += 32 * VEC) {
            float xv[kTok][VEC];
#pragma unroll
            for (int j = 0; j < kTok; ++j) {
                if (t0 + j < r1) load_vec<T>(X + (long long)(t0 + j) * K + k, xv[j]);
                else
#pragma unroll
                    for (int v = 0; v < VEC; ++v) xv[j][v] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < kRPW; ++i) {
                const int n = n0 + i;
                if (n >= a.Nout) break;
                float wv[VEC];
                load_vec<T>(Wb + (long long)(kGated ? 2 * n : n) * K + k, wv);
#pragma unroll
                for (int j = 0; j < kTok; ++j)
#pragma unroll
                    for (int v = 0; v < VEC; ++v) acc[i][j] += wv[v] * xv[j][v];
                if (kGated) {  // SwiGLU slot rows are interleaved: 2n = w1, 2n+1 = w3
                    float w3[VEC];
                    load_vec<T>(Wb + (long long)(2 * n + 1) * K + k, w3);
#pragma unroll
                    for (int j = 0; j < kTok; ++j)
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc3[i][j] += w3[v] * xv[j][v];
                }
            }
        }
#pragma unroll
        for (int i = 0; i < kRPW; ++i)
#pragma unroll
            for (int j = 0; j < kTok; ++j) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    acc[i][j] += __shfl_xor_sync(0xffffffffu, acc[i][j], o);
                    if (kGated) acc3[i][j] += __shfl_xor_sync(0xffffffffu, acc3[i][j], o);
                }
            }
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < kRPW; ++i) {
                const int n = n0 + i;
                if (n >= a.Nout) break;
#pragma unroll
                for (int j = 0; j < kTok; ++j) {
                    const int r = t0 + j;
                    if (r >= r1) break;
                    const long long o = (long long)r * a.ldy + n;
                    const float v = acc[i][j];
                    if (EPI == kEpiStoreF32) reinterpret_cast<float*>(a.Y)[o] = v;
                    else if (EPI == kEpiResidAdd) reinterpret_cast<float*>(a.Y)[o] += v;
                    else if (EPI == kEpiTanh) reinterpret_cast<T*>(a.Y)[o] = from_f<T>(tanhf(v));
                    else reinterpret_cast<T*>(a.Y)[o] = from_f<T>(v / (1.0f + expf(-v)) * acc3[kGated ? i : 0][j]);
                }
            }
        }
    }
}

template <typename T>
void dispatch(const GemmArgs& a, cudaStream_t s) {
    dim3 grid(ceil_div(a.Nout, kWarps * kRPW), a.G);
    switch (a.epi) {
        case kEpiStoreF32: launch_k(k_gemm_simt<T, kEpiStoreF32>, grid, kWarps * 32, 0, s, a); break;
        case kEpiResidAdd: launch_k(k_gemm_simt<T, kEpiResidAdd>, grid, kWarps * 32, 0, s, a); break;
        case kEpiTanh: launch_k(k_gemm_simt<T, kEpiTanh>, grid, kWarps * 32, 0, s, a); break;
        case kEpiSwiglu: launch_k(k_gemm_simt<T, kEpiSwiglu>, grid, kWarps * 32, 0, s, a); break;
    }
}

}  // namespace

void launch_gemm_simt(const GemmArgs& a, WType wt, cudaStream_t s) {
    if (a.G <= 0 || a.Nout <= 0) return;
    if (wt == kF32) dispatch<float>(a, s);
    else dispatch<__nv_bfloat16>(a, s);
}

}  // namespace smoe
