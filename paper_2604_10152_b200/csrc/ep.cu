// ep.cu -- expert-parallel transports (NCCL over NVLink/NVSwitch; loopback for virtual ranks) and the
// pack kernel that prepares a rank's disjoint expert-output contribution.
#include <dlfcn.h>
#include <cstring>
#include <nccl.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "ep.h"

namespace smoe {

namespace {

// y[j] = sum_s P[s][pos[j]] for picks j of this rank's experts (fin[j] in [e0, e1)), else 0: the
// rank's contribution in pick order, so the sum over ranks is exact and feeds the combine directly.
__global__ void k_ep_pack(const float* __restrict__ P, int S, long long pstride, const int* __restrict__ pos,
                          const int* __restrict__ fin, int e0, int e1, int d, float* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    const int j = blockIdx.x;
    const int e = fin[j];
    const bool mine = e >= e0 && e < e1;
    const long long src = (long long)pos[j] * d, dst = (long long)j * d;
    for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (mine)
            for (int s = 0; s < S; ++s) {
                const float4 q = *reinterpret_cast<const float4*>(P + s * pstride + src + i);
                a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
            }
        *reinterpret_cast<float4*>(y + dst + i) = a;
    }
}

struct Ptrs {
    const float* p[16];
};
__global__ void k_sum_ranks(Ptrs in, int world, size_t n, float* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float a = 0.f;
        for (int r = 0; r < world; ++r) a += in.p[r][i];  // rank order (exact: disjoint supports)
        out[i] = a;
    }
}

// ---------------------------------------------------------------- NCCL via dlopen
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.h, "ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.h || !api.get_unique_id || !api.comm_init_rank || !api.all_reduce)
        throw Error(kCuda, "NCCL (libnccl.so.2) not loadable");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(kCuda, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}

class NcclComm : public Comm {
public:
    NcclComm(int rank, int world, const ncclUniqueId& id, int device) : rank_(rank), world_(world) {
        SMOE_CUDA(cudaSetDevice(device));
        nccl_check(nccl().comm_init_rank(&comm_, world, id, rank), "ncclCommInitRank");
    }
    ~NcclComm() override {
        if (comm_ && nccl().comm_destroy) nccl().comm_destroy(comm_);
    }
    int rank() const override { return rank_; }
    int world() const override { return world_; }
    void allreduce_sum(float* buf, size_t n, cudaStream_t s) override {
        nccl_check(nccl().all_reduce(buf, buf, n, ncclFloat32, ncclSum, comm_, s), "ncclAllReduce");
    }

private:
    int rank_, world_;
    ncclComm_t comm_ = nullptr;
};

}  // namespace

int nccl_unique_id(void* out, int len) {
    if (len < (int)sizeof(ncclUniqueId)) throw Error(kConfig, "nccl unique id buffer too small");
    ncclUniqueId id;
    nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof id);
    return (int)sizeof id;
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id, int len, int device) {
    if (len < (int)sizeof(ncclUniqueId)) throw Error(kConfig, "nccl unique id too short");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    return std::make_unique<NcclComm>(rank, world, u, device);
}

// ---------------------------------------------------------------- loopback (virtual ranks)
struct LoopbackGroup {
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<float*> bufs;
    explicit LoopbackGroup(int w) : world(w), bufs(w, nullptr) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

LoopbackGroup* loopback_create(int world) {
    if (world < 1 || world > 16) throw Error(kConfig, "loopback world must be in [1, 16]");
    return new LoopbackGroup(world);
}
void loopback_destroy(LoopbackGroup* g) { delete g; }

namespace {
class LoopbackComm : public Comm {
public:
    LoopbackComm(LoopbackGroup* g, int rank) : g_(g), rank_(rank) {}
    ~LoopbackComm() override {
        if (scratch_) cudaFree(scratch_);
    }
    int rank() const override { return rank_; }
    int world() const override { return g_->world; }
    void allreduce_sum(float* buf, size_t n, cudaStream_t s) override {
        if (n > cap_) {
            if (scratch_) SMOE_CUDA(cudaFree(scratch_));
            SMOE_CUDA(cudaMalloc(&scratch_, n * sizeof(float)));
            cap_ = n;
        }
        SMOE_CUDA(cudaStreamSynchronize(s));
        g_->bufs[rank_] = buf;
        g_->barrier();  // every rank's contribution is ready
        Ptrs p{};
        for (int r = 0; r < g_->world; ++r) p.p[r] = g_->bufs[r];
        k_sum_ranks<<<148 * 4, 256, 0, s>>>(p, g_->world, n, scratch_);
        SMOE_CUDA(cudaGetLastError());
        SMOE_CUDA(cudaStreamSynchronize(s));
        g_->barrier();  // every rank has read every buffer
        SMOE_CUDA(cudaMemcpyAsync(buf, scratch_, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
    }

private:
    LoopbackGroup* g_;
    int rank_;
    float* scratch_ = nullptr;
    size_t cap_ = 0;
};
}  // namespace

std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* g, int rank) {
    if (!g || rank < 0 || rank >= g->world) throw Error(kConfig, "loopback rank out of range");
    return std::make_unique<LoopbackComm>(g, rank);
}

void launch_ep_pack(const float* P, int S, long long pstride, const int* pos, const int* fin, int e0, int e1, int picks,
                    int d, float* y_red, cudaStream_t s) {
    if (picks <= 0) return;
    launch_k(k_ep_pack, picks, 256, 0, s, P, S, pstride, pos, fin, e0, e1, d, y_red);
}

}  // namespace smoe
