// ep.h -- expert-parallel communication.
//
// Experts are sharded across G ranks in contiguous blocks (owner(e) = e / (E/G)); the rows of every
// pass are split across the ranks in contiguous blocks of seg = ceil(T/G) (the dense path, gate, head
// and argmax of a row run on its rank).  Per MoE layer the gate writes a rank's routed rows into
// expert-major segments [E][seg][d], which IS the all-to-all send buffer (chunk r = rank r's experts):
// dispatch = all-to-all of those rows and of the per-expert counts, the owners run one grouped GEMM over
// (source rank, local expert) groups, and combine = all-to-all of the finished rows back into the same
// [E][seg][d] layout, which the combine kernel reads through the unchanged pick positions.  Every row is
// computed by the same kernels in the same order as at G = 1, and routing logs and argmax tokens are
// all-gathered once per pass so the host bookkeeping is replicated, hence token streams, routing and
// ledger are bit-identical at G = 1, 2, 4, 8 (tested with the loopback transport on one GPU).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <memory>
#include <vector>

namespace smoe {

class Comm {
public:
    virtual ~Comm() = default;
    virtual int rank() const = 0;
    virtual int world() const = 0;
    // send[r * chunk .. (r+1) * chunk) -> rank r's recv[me * chunk ..), all ranks at once, ordered on `s`
    virtual void alltoall(const void* send, void* recv, size_t chunk_bytes, cudaStream_t s) = 0;
    // recv[r * bytes ..) = rank r's send[0 .. bytes)
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
    // every rank's n device buffers, addressable from this rank: all[r * n + i] (own: mine[i]).  NCCL:
    // CUDA IPC handles exchanged by an all-gather and opened with peer access; opened pointers are
    // appended to `opened` for the caller to close.  Loopback: the buffers of the other virtual ranks.
    virtual void share_buffers(void* const* mine, int n, std::vector<void*>& all, std::vector<void*>& opened) = 0;
    // After a fused-exchange signal: no-op with one process per GPU.  Virtual ranks sharing one device
    // must not let a device-side wait spin for a peer whose host thread is blocked in a device-wide
    // synchronisation (cudaFree, cudaMalloc, ...) queued behind that very wait; the loopback transport
    // therefore drains its stream and meets the other ranks here, so every wait finds its flags set.
    virtual void fence(cudaStream_t s) { (void)s; }
};

// NCCL (dlopen'ed libnccl.so.2, so the engine shares whichever NCCL the process already loaded)
int nccl_unique_id(void* out, int len);
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id, int len, int device);

// One process per rank with a caller-provided blocking host all-gather (recv[r * bytes ..) = rank r's
// send); device placement is free, several ranks may share a GPU.  Returns non-zero on failure.
typedef int (*HostAllgatherFn)(void* user, const void* send, void* recv, uint64_t bytes);
std::unique_ptr<Comm> make_host_comm(int rank, int world, HostAllgatherFn fn, void* user);

// G virtual ranks on one device (tests): each rank is an engine driven by its own host thread.
struct LoopbackGroup;
LoopbackGroup* loopback_create(int world);
void loopback_destroy(LoopbackGroup* g);
std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* g, int rank);

// y[r] = sum_s P[s][r] (s in order from 0, as the combine sums split partials) for the rows r of the
// groups g with rows [g*seg, g*seg + cnt[g]): the owner's finished expert rows, ready to be returned
void launch_ep_sum_partials(const float* P, int S, long long pstride, const int* cnt, int groups, int seg, int d,
                            float* y, cudaStream_t s);
// routing logs of a pass: pack this rank's rows [0, Tl) of raw/fin [M][Tmax][K] into [2][M][seg][K]
// and, after the all-gather, unpack rank r's block into rows [r*seg, min(T, (r+1)*seg)) of the logs
void launch_ep_pack_logs(const int* raw, const int* fin, int M, int Tmax, int K, int Tl, int seg, int* out,
                         cudaStream_t s);
// Fused exchange signalling (peer memory).  signal: rank `me` publishes its per-expert counts into the
// owners' receive-count arrays (cnt != nullptr), makes every prior store system-visible and sets its
// flag flags[r][slot * G + me] = seq on every rank r.  wait: until flags[slot * G + r] == seq for all r.
void launch_ep_signal(const int* cnt, int E, int eo, int me, int G, void* const* peer_cnt, void* const* peer_flags,
                      int slot, int seq, cudaStream_t s);
void launch_ep_wait(const int* flags, int G, int slot, int seq, cudaStream_t s);
void launch_ep_unpack_logs(const int* in, int G, int M, int Tmax, int K, int T, int seg, int* raw, int* fin,
                           cudaStream_t s);

}  // namespace smoe
