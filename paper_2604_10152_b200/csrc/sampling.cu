// sampling.cu -- temperature sampling on the device: the draft draws of speculate()
// (specdec.cpp:38-50 -> sample_next, model.cpp:178-190), the batched verify_sampling acceptance and
// residual resample (specdec.cpp:82-157) and the on-demand draws (baselines.cpp:59-64).
//
// The reference draws every uniform from ONE host mt19937_64 stream in a fixed order; the host still
// draws them (uniform01, common.hpp:40-42) and ships them, so the device never owns RNG state:
//   * draft step t of a phase consumes one uniform per active sequence (speculate's t-major loop);
//   * verify consumes, per active sequence in order, one uniform per acceptance test and one for the
//     residual / bonus draw -- a data-dependent count, so the host ships a pool of na*(gamma+1) (the most
//     a sequence can use), k_verify_accept walks the sequences in order assigning pool offsets, and the
//     host advances its stream by exactly the number consumed.
// All probabilities are float64 from the float32 logits, as the reference computes them from its logits:
// p_j = exp(l_j/T - max) / sum (model.cpp:145-157), draws by the first cumulative sum exceeding u
// (inverse CDF, the rounding tail -> V-1).  Sums run as per-thread sequential chunks combined in a tree.
#include "common.cuh"
#include "kernels.h"

namespace smoe {
namespace {

constexpr int kST = 1024;  // threads per row block

// Block-wide fp64 sum / max over kST threads (warp shuffles, then warp 0).
__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (l == 0) red[32] = v;
    }
    __syncthreads();
    return red[32];
}
__device__ __forceinline__ double block_max(double v, double* red) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = l < (int)(blockDim.x >> 5) ? red[l] : -INFINITY;
        for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (l == 0) red[32] = v;
    }
    __syncthreads();
    return red[32];
}
// Exclusive prefix over the block of per-thread values (fp64), in thread order.
__device__ __forceinline__ double block_exclusive_scan(double v, double* red) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    double incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += t;
    }
    __syncthreads();
    if (l == 31) red[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        double t = l < nw ? red[l] : 0.0, s = t;
        for (int o = 1; o < 32; o <<= 1) {
            const double q = __shfl_up_sync(0xffffffffu, s, o);
            if (l >= o) s += q;
        }
        if (l < nw) red[l] = s - t;  // exclusive warp offsets
    }
    __syncthreads();
    return red[w] + incl - v;
}

// Row statistics of softmax(logits / T) in float64: max and sum of exp(x - max).
__device__ void row_stats(const float* lg, int V, double T, double* red, double& mx, double& sum) {
    double m = -INFINITY;
    for (int j = threadIdx.x; j < V; j += blockDim.x) m = fmax(m, (double)lg[j] / T);
    mx = block_max(m, red);
    double s = 0.0;
    for (int j = threadIdx.x; j < V; j += blockDim.x) s += exp((double)lg[j] / T - mx);
    sum = block_sum(s, red);
}

// First j with u < cum_j of the (unnormalised) weights w_j = f(j), thread-contiguous chunks; V-1 when
// u lands in the rounding tail.  Every thread returns the same j.
template <typename F>
__device__ int inverse_cdf(int V, double u, F f, double* red, int* s_pick) {
    const int chunk = (V + blockDim.x - 1) / blockDim.x;
    const int j0 = threadIdx.x * chunk, j1 = min(V, j0 + chunk);
    double part = 0.0;
    for (int j = j0; j < j1; ++j) part += f(j);
    const double before = block_exclusive_scan(part, red);
    if (threadIdx.x == 0) *s_pick = V - 1;
    __syncthreads();
    // every chunk ending past u scans to its first crossing; the smallest wins (robust to the chunk sums
    // and the running sum rounding differently)
    if (u < before + part) {
        double cum = before;
        for (int j = j0; j < j1; ++j) {
            cum += f(j);
            if (u < cum) {
                atomicMin(s_pick, j);
                break;
            }
        }
    }
    __syncthreads();
    return *s_pick;
}

// One block per row: q = softmax(logits/T) (optionally stored) and a draw with the row's uniform.
__global__ void __launch_bounds__(kST) k_sample_rows(const float* __restrict__ logits, int V, double T,
                                                      const double* __restrict__ u, int* __restrict__ tok,
                                                      double* __restrict__ q, long long q_stride) {
    __shared__ double red[33];
    __shared__ int pick;
    const int r = blockIdx.x;
    const float* lg = logits + (long long)r * V;
    double mx, sum;
    row_stats(lg, V, T, red, mx, sum);
    auto p = [&](int j) { return exp((double)lg[j] / T - mx) / sum; };
    if (q)
        for (int j = threadIdx.x; j < V; j += blockDim.x) q[r * q_stride + j] = p(j);
    const int t = inverse_cdf(V, u[r], p, red, &pick);
    if (threadIdx.x == 0) tok[r] = t;
}

// Verify rows: per-row softmax statistics (max, sum) for the acceptance ratios and the final draws.
__global__ void __launch_bounds__(kST) k_row_stats(const float* __restrict__ logits, int V, double T,
                                                    double* __restrict__ stats) {
    __shared__ double red[33];
    double mx, sum;
    row_stats(logits + (long long)blockIdx.x * V, V, T, red, mx, sum);
    if (threadIdx.x == 0) {
        stats[2 * blockIdx.x] = mx;
        stats[2 * blockIdx.x + 1] = sum;
    }
}

// Acceptance of every active sequence (specdec.cpp:104-118), in order: sequence s (verify rows
// s*(g+1) + i, drafts[seqs[s]][i], draft probabilities q[i][s]) uses the pool from the running offset.
// kind[s]: 0 = rejected at acc[s] (residual draw), 1 = all accepted (bonus draw); uidx[s] = the pool
// index of that draw; used[0] = uniforms consumed by the phase.  One block.
__global__ void k_verify_accept(const float* __restrict__ logits, int V, double T, const double* __restrict__ stats,
                                const double* __restrict__ q, long long q_tstride, const int* __restrict__ drafts,
                                int dstride, const int* __restrict__ seqs, int na, int g,
                                const double* __restrict__ pool, int* __restrict__ acc, int* __restrict__ kind,
                                int* __restrict__ uidx, int* __restrict__ used, int* __restrict__ flags,
                                double* __restrict__ ratio /* [na][g] scratch */) {
    // ratios min(1, p/q) in parallel
    for (int k = threadIdx.x; k < na * g; k += blockDim.x) {
        const int s = k / g, i = k % g, row = s * (g + 1) + i;
        const int x = drafts[(long long)seqs[s] * dstride + i];
        const double p = exp((double)logits[(long long)row * V + x] / T - stats[2 * row]) / stats[2 * row + 1];
        const double qq = q[i * q_tstride + (long long)s * V + x];
        if (qq <= 0.0) atomicOr(flags, kFlagZeroDrawProb);
        ratio[k] = qq > 0.0 ? fmin(1.0, p / qq) : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int off = 0;
        for (int s = 0; s < na; ++s) {
            int a = 0;
            while (a < g && pool[off++] < ratio[s * g + a]) ++a;
            acc[s] = a;
            kind[s] = a == g;
            uidx[s] = off++;
        }
        used[0] = off;
    }
}

// The draw that ends each sequence's verification: the residual max(0, p - q) at the rejected position
// (renormalised; p itself when the residual vanishes), or the bonus token from p at position g.
__global__ void __launch_bounds__(kST) k_verify_draw(const float* __restrict__ logits, int V, double T,
                                                      const double* __restrict__ stats, const double* __restrict__ q,
                                                      long long q_tstride, int g, const double* __restrict__ pool,
                                                      const int* __restrict__ acc, const int* __restrict__ kind,
                                                      const int* __restrict__ uidx, int* __restrict__ corr) {
    __shared__ double red[33];
    __shared__ int pick;
    const int s = blockIdx.x, a = acc[s];
    const int row = s * (g + 1) + a;
    const float* lg = logits + (long long)row * V;
    const double mx = stats[2 * row], sum = stats[2 * row + 1];
    auto p = [&](int j) { return exp((double)lg[j] / T - mx) / sum; };
    const double u = pool[uidx[s]];
    int t;
    if (kind[s]) {
        t = inverse_cdf(V, u, p, red, &pick);
    } else {
        const double* qq = q + a * q_tstride + (long long)s * V;
        auto res = [&](int j) { return fmax(0.0, p(j) - qq[j]); };
        double n = 0.0;
        for (int j = threadIdx.x; j < V; j += blockDim.x) n += res(j);
        const double norm = block_sum(n, red);
        if (norm > 0.0) t = inverse_cdf(V, u * norm, res, red, &pick);
        else t = inverse_cdf(V, u, p, red, &pick);  // p == q everywhere: any draw from p is exact
    }
    if (threadIdx.x == 0) corr[s] = t;
}

}  // namespace

void launch_sample_rows(const float* logits, int R, int V, double T, const double* u, int* tok, double* q,
                        long long q_stride, cudaStream_t s) {
    if (R <= 0) return;
    launch_k(k_sample_rows, R, kST, 0, s, logits, V, T, u, tok, q, q_stride);
}

void launch_verify_sampling(const float* logits, int V, double T, double* stats, const double* q, long long q_tstride,
                            const int* drafts, int dstride, const int* seqs, int na, int g, const double* pool,
                            int* acc, int* kind, int* uidx, int* used, int* corr, int* flags, double* ratio,
                            cudaStream_t s) {
    if (na <= 0) return;
    launch_k(k_row_stats, na * (g + 1), kST, 0, s, logits, V, T, stats);
    launch_k(k_verify_accept, 1, 256, 0, s, logits, V, T, (const double*)stats, q, q_tstride, drafts, dstride, seqs,
             na, g, pool, acc, kind, uidx, used, flags, ratio);
    launch_k(k_verify_draw, na, kST, 0, s, logits, V, T, (const double*)stats, q, q_tstride, g, pool,
             (const int*)acc, (const int*)kind, (const int*)uidx, corr);
}

}  // namespace smoe
