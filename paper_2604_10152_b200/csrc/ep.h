// ep.h -- expert-parallel communication.
//
// Experts are sharded across G ranks in contiguous blocks (owner(e) = e / (E/G)); every rank runs the
// dense path and the routing for all rows, computes only its own experts' rows, and the per-layer
// expert outputs -- one row per pick, zeros for other ranks' picks -- are summed across ranks.  A sum in
// which every element has one non-zero term is exact in any order, so the token stream, routing and
// ledger are bit-identical at G = 1, 2, 4, 8 (tested with the loopback transport on one GPU).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <memory>

namespace smoe {

class Comm {
public:
    virtual ~Comm() = default;
    virtual int rank() const = 0;
    virtual int world() const = 0;
    // in-place sum over ranks of a device f32 buffer, ordered on `s`
    virtual void allreduce_sum(float* buf, size_t n, cudaStream_t s) = 0;
};

// NCCL (dlopen'ed libnccl.so.2, so the engine shares whichever NCCL the process already loaded)
int nccl_unique_id(void* out, int len);
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id, int len, int device);

// G virtual ranks on one device (tests): each rank is an engine driven by its own host thread.
struct LoopbackGroup;
LoopbackGroup* loopback_create(int world);
void loopback_destroy(LoopbackGroup* g);
std::unique_ptr<Comm> make_loopback_comm(LoopbackGroup* g, int rank);

// y_red[j] = (e0 <= fin[j] < e1) ? sum_s P[s][pos[j]] : 0 for the T*K picks j (pick order)
void launch_ep_pack(const float* P, int S, long long pstride, const int* pos, const int* fin, int e0, int e1, int picks,
                    int d, float* y_red, cudaStream_t s);

}  // namespace smoe
