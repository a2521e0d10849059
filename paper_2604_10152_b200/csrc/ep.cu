// ep.cu -- expert-parallel transports (NCCL over NVLink/NVSwitch; loopback for virtual ranks) and the
// pack kernel that prepares a rank's disjoint expert-output contribution.
#include <dlfcn.h>
#include <cstdio>
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

__global__ void k_ep_sum_partials(const float* __restrict__ P, int S, long long pstride, const int* __restrict__ cnt,
                                  int seg, int d, float* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    const int g = blockIdx.y, t = blockIdx.x;
    if (t >= cnt[g]) return;
    const long long row = ((long long)g * seg + t) * d;
    for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < S; ++s) {
            const float4 q = *reinterpret_cast<const float4*>(P + s * pstride + row + i);
            a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
        }
        *reinterpret_cast<float4*>(y + row + i) = a;
    }
}

__global__ void k_ep_signal(const int* __restrict__ cnt, int E, int eo, int me, int G, void* const* peer_cnt,
                            void* const* peer_flags, int slot, int seq) {
    pdl_wait();
    pdl_trigger();
    if (cnt)
        for (int e = threadIdx.x; e < E; e += blockDim.x)
            reinterpret_cast<int*>(peer_cnt[e / eo])[me * eo + e % eo] = cnt[e];
    __threadfence_system();
    __syncthreads();
    for (int r = threadIdx.x; r < G; r += blockDim.x) {
        int* f = reinterpret_cast<int*>(peer_flags[r]) + slot * G + me;
        asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(seq) : "memory");
    }
}

__global__ void k_ep_wait(const int* flags, int G, int slot, int seq) {
    pdl_wait();
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        for (int r = 0; r < G; ++r) {
            while (true) {
                int v;
                asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + slot * G + r) : "memory");
                if (v - seq >= 0) break;
                __nanosleep(64);
                if (clock64() - t0 > 40000000000ll) {  // ~20 s: a peer stopped exchanging
                    printf("smoe ep wait timeout: slot %d seq %d, flag of rank %d = %d (G %d)\n", slot, seq, r, v, G);
                    __trap();
                }
            }
        }
        asm volatile("fence.acq_rel.sys;" ::: "memory");
    }
    __syncthreads();
    pdl_trigger();
}

__global__ void k_ep_pack_logs(const int* __restrict__ raw, const int* __restrict__ fin, int M, int Tmax, int K,
                               int Tl, int seg, int* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int n = M * seg * K;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n; i += gridDim.x * blockDim.x) {
        const int w = i / n, j = i % n, m = j / (seg * K), t = (j / K) % seg, k = j % K;
        out[i] = t < Tl ? (w ? fin : raw)[((long long)m * Tmax + t) * K + k] : -1;
    }
}

__global__ void k_ep_unpack_logs(const int* __restrict__ in, int G, int M, int Tmax, int K, int T, int seg,
                                 int* __restrict__ raw, int* __restrict__ fin) {
    pdl_wait();
    pdl_trigger();
    const int n = M * seg * K;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < G * 2 * n; i += gridDim.x * blockDim.x) {
        const int r = i / (2 * n), w = (i / n) % 2, j = i % n, m = j / (seg * K), t = (j / K) % seg, k = j % K;
        const int row = r * seg + t;
        if (row < T) (w ? fin : raw)[((long long)m * Tmax + row) * K + k] = in[i];
    }
}

// ---------------------------------------------------------------- NCCL via dlopen
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
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
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.h, "ncclAllGather"));
        a.send = reinterpret_cast<decltype(a.send)>(dlsym(a.h, "ncclSend"));
        a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(a.h, "ncclRecv"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(a.h, "ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(a.h, "ncclGroupEnd"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.h || !api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.send || !api.recv ||
        !api.group_start || !api.group_end)
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
    void alltoall(const void* send, void* recv, size_t chunk, cudaStream_t s) override {
        // grouped point-to-point: one send and one receive per peer (self included), fixed-size chunks,
        // so no counts ever travel to the host
        nccl_check(nccl().group_start(), "ncclGroupStart");
        for (int r = 0; r < world_; ++r) {
            nccl_check(nccl().send(static_cast<const char*>(send) + r * chunk, chunk, ncclInt8, r, comm_, s), "ncclSend");
            nccl_check(nccl().recv(static_cast<char*>(recv) + r * chunk, chunk, ncclInt8, r, comm_, s), "ncclRecv");
        }
        nccl_check(nccl().group_end(), "ncclGroupEnd");
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        nccl_check(nccl().all_gather(send, recv, bytes, ncclInt8, comm_, s), "ncclAllGather");
    }
    void share_buffers(void* const* mine, int n, std::vector<void*>& all, std::vector<void*>& opened) override {
        std::vector<cudaIpcMemHandle_t> h(n);
        for (int i = 0; i < n; ++i) SMOE_CUDA(cudaIpcGetMemHandle(&h[i], mine[i]));
        const size_t bytes = sizeof(cudaIpcMemHandle_t) * n;
        char* dev = nullptr;
        SMOE_CUDA(cudaMalloc(&dev, bytes * (world_ + 1)));
        SMOE_CUDA(cudaMemcpy(dev, h.data(), bytes, cudaMemcpyHostToDevice));
        allgather(dev, dev + bytes, bytes, nullptr);
        std::vector<cudaIpcMemHandle_t> every((size_t)n * world_);
        SMOE_CUDA(cudaStreamSynchronize(nullptr));
        SMOE_CUDA(cudaMemcpy(every.data(), dev + bytes, bytes * world_, cudaMemcpyDeviceToHost));
        SMOE_CUDA(cudaFree(dev));
        all.assign((size_t)n * world_, nullptr);
        for (int r = 0; r < world_; ++r)
            for (int i = 0; i < n; ++i) {
                if (r == rank_) {
                    all[(size_t)r * n + i] = mine[i];
                    continue;
                }
                void* p = nullptr;
                SMOE_CUDA(cudaIpcOpenMemHandle(&p, every[(size_t)r * n + i], cudaIpcMemLazyEnablePeerAccess));
                all[(size_t)r * n + i] = p;
                opened.push_back(p);
            }
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
    std::vector<const void*> bufs;
    std::vector<void*> shared;  // share_buffers table
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
    int rank() const override { return rank_; }
    int world() const override { return g_->world; }
    // Every virtual rank publishes its send buffer; after a barrier each copies its chunks out of the
    // others' buffers on its own stream; a second barrier keeps senders from reusing their buffers early.
    void alltoall(const void* send, void* recv, size_t chunk, cudaStream_t s) override {
        exchange(send, [&](int r, const char* peer) {
            SMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + r * chunk, peer + rank_ * chunk, chunk,
                                      cudaMemcpyDeviceToDevice, s));
        }, s);
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        exchange(send, [&](int r, const char* peer) {
            SMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + r * bytes, peer, bytes, cudaMemcpyDeviceToDevice, s));
        }, s);
    }

    void fence(cudaStream_t s) override {
        SMOE_CUDA(cudaStreamSynchronize(s));
        g_->barrier();
    }
    void share_buffers(void* const* mine, int n, std::vector<void*>& all, std::vector<void*>& opened) override {
        (void)opened;
        {
            std::lock_guard<std::mutex> lk(g_->mu);
            g_->shared.resize((size_t)g_->world * n);
            for (int i = 0; i < n; ++i) g_->shared[(size_t)rank_ * n + i] = mine[i];
        }
        g_->barrier();
        {
            std::lock_guard<std::mutex> lk(g_->mu);
            all.assign(g_->shared.begin(), g_->shared.begin() + (size_t)g_->world * n);
        }
        g_->barrier();
    }

private:
    template <typename F>
    void exchange(const void* send, F copy_from, cudaStream_t s) {
        SMOE_CUDA(cudaStreamSynchronize(s));
        g_->bufs[rank_] = send;
        g_->barrier();  // every rank's send buffer is ready
        for (int r = 0; r < g_->world; ++r) copy_from(r, static_cast<const char*>(g_->bufs[r]));
        SMOE_CUDA(cudaStreamSynchronize(s));
        g_->barrier();  // every rank has read every buffer
    }
    LoopbackGroup* g_;
    int rank_;
};
}  // namespace

// ---------------------------------------------------------------- host transport (caller's all-gather)
// One process per rank, any device placement (several processes may share one GPU): the only thing the
// caller provides is a blocking host all-gather (gloo, MPI, sockets ...).  Every collective is staged
// through host memory, and the fused exchange's peer tables are CUDA IPC handles all-gathered the same
// way.  Unlike the loopback group there is no host fence: the device-side flag protocol (k_ep_signal /
// k_ep_wait) is what orders the ranks.
namespace {
class HostComm : public Comm {
public:
    HostComm(int rank, int world, HostAllgatherFn fn, void* user) : rank_(rank), world_(world), fn_(fn), user_(user) {}
    int rank() const override { return rank_; }
    int world() const override { return world_; }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        std::vector<char> hs(bytes), hr(bytes * world_);
        SMOE_CUDA(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, s));
        SMOE_CUDA(cudaStreamSynchronize(s));
        host_allgather(hs.data(), hr.data(), bytes);
        SMOE_CUDA(cudaMemcpyAsync(recv, hr.data(), bytes * world_, cudaMemcpyHostToDevice, s));
        SMOE_CUDA(cudaStreamSynchronize(s));
    }
    void alltoall(const void* send, void* recv, size_t chunk, cudaStream_t s) override {
        // every rank's whole send buffer travels to every rank; each keeps the chunks addressed to it
        const size_t row = chunk * world_;
        std::vector<char> hs(row), hr(row * world_);
        SMOE_CUDA(cudaMemcpyAsync(hs.data(), send, row, cudaMemcpyDeviceToHost, s));
        SMOE_CUDA(cudaStreamSynchronize(s));
        host_allgather(hs.data(), hr.data(), row);
        for (int r = 0; r < world_; ++r)
            SMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + r * chunk, hr.data() + r * row + rank_ * chunk, chunk,
                                      cudaMemcpyHostToDevice, s));
        SMOE_CUDA(cudaStreamSynchronize(s));
    }
    void share_buffers(void* const* mine, int n, std::vector<void*>& all, std::vector<void*>& opened) override {
        std::vector<cudaIpcMemHandle_t> h(n), every((size_t)n * world_);
        for (int i = 0; i < n; ++i) SMOE_CUDA(cudaIpcGetMemHandle(&h[i], mine[i]));
        host_allgather(h.data(), every.data(), sizeof(cudaIpcMemHandle_t) * n);
        all.assign((size_t)n * world_, nullptr);
        for (int r = 0; r < world_; ++r)
            for (int i = 0; i < n; ++i) {
                if (r == rank_) {
                    all[(size_t)r * n + i] = mine[i];
                    continue;
                }
                void* p = nullptr;
                SMOE_CUDA(cudaIpcOpenMemHandle(&p, every[(size_t)r * n + i], cudaIpcMemLazyEnablePeerAccess));
                all[(size_t)r * n + i] = p;
                opened.push_back(p);
            }
    }

private:
    void host_allgather(const void* send, void* recv, size_t bytes) {
        const int rc = fn_(user_, send, recv, (uint64_t)bytes);
        if (rc != 0) throw Error(kCuda, "host transport: all-gather callback failed (" + std::to_string(rc) + ")");
    }
    int rank_, world_;
    HostAllgatherFn fn_;
    void* user_;
};
}  // namespace

std::unique_ptr<Comm> make_host_comm(int rank, int world, HostAllgatherFn fn, void* user) {
    if (!fn) throw Error(kConfig, "host transport: no all-gather callback");
    if (world < 2 || rank < 0 || rank >= world) throw Error(kConfig, "host transport: rank out of range");
    return std::make_unique<HostComm>(rank, world, fn, user);
}

std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* g, int rank) {
    if (!g || rank < 0 || rank >= g->world) throw Error(kConfig, "loopback rank out of range");
    return std::make_unique<LoopbackComm>(g, rank);
}

void launch_ep_sum_partials(const float* P, int S, long long pstride, const int* cnt, int groups, int seg, int d,
                            float* y, cudaStream_t s) {
    if (groups <= 0 || seg <= 0) return;
    launch_k(k_ep_sum_partials, dim3(seg, groups), 256, 0, s, P, S, pstride, cnt, seg, d, y);
}
void launch_ep_signal(const int* cnt, int E, int eo, int me, int G, void* const* peer_cnt, void* const* peer_flags,
                      int slot, int seq, cudaStream_t s) {
    launch_k(k_ep_signal, 1, 64, 0, s, cnt, E, eo, me, G, peer_cnt, peer_flags, slot, seq);
}
void launch_ep_wait(const int* flags, int G, int slot, int seq, cudaStream_t s) {
    launch_k(k_ep_wait, 1, 32, 0, s, flags, G, slot, seq);
}
void launch_ep_pack_logs(const int* raw, const int* fin, int M, int Tmax, int K, int Tl, int seg, int* out,
                         cudaStream_t s) {
    if (M <= 0 || seg <= 0) return;
    launch_k(k_ep_pack_logs, 64, 256, 0, s, raw, fin, M, Tmax, K, Tl, seg, out);
}
void launch_ep_unpack_logs(const int* in, int G, int M, int Tmax, int K, int T, int seg, int* raw, int* fin,
                           cudaStream_t s) {
    if (M <= 0 || seg <= 0) return;
    launch_k(k_ep_unpack_logs, 128, 256, 0, s, in, G, M, Tmax, K, T, seg, raw, fin);
}

}  // namespace smoe
