// store.cpp -- the real expert store for CPU-offloaded MoE (memsim.cpp:81-161 made
// physical).
//
// Every expert lives in pinned host DRAM (host_up / host_down, one key = (MoE layer, expert)).  HBM
// holds a pool of expert slots: the N pinned draft experts of every layer plus transients.  During an
// unrestricted pass (verify / on-demand / warmup) each MoE layer's routing is known only after its gate,
// so per layer: gate + route -> tiny D2H of the group sizes -> the host issues cudaMemcpyAsync of the
// non-resident experts on the copy stream -> the compute stream waits on an event -> expert GEMMs.
// The dense part of the next layer (mix, gate) cannot start before this layer's experts, so PCIe is
// kept busy back to back across layers (the copy of layer l+1 is issued ~0.5 ms after layer l's).
// After a layer's GEMMs: hot_temporal re-pin for that layer (its counts are complete once its gate
// ran over every verify row), relabelling slots in place -- zero bytes, the paper's zero-cost
// replacement -- then the layer's remaining transients are released (the reference's per-phase flush).
// HBM therefore needs only M*N pinned slots + (E - N) transient slots, not the whole model.
// The reference-semantics ledger is kept separately by loop.cpp; the bytes this store moves are
// exactly (ledger entries) x (real bytes per expert).
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <string>
#include <thread>

#include "engine.h"

namespace smoe {

// ------------------------------------------------------------------ SSD tier (offload = 2)
// The reference's third tier is a bandwidth scalar (TierConfig.ssd_bandwidth, memsim.hpp:31-37).  Here
// it is a file on local storage: every expert of this rank at a 4 KB-aligned record, read with O_DIRECT
// (page cache bypassed, so each migration really streams from the device; buffered reads + DONTNEED when
// the filesystem refuses O_DIRECT) by a small reader pool into pinned staging chunks, each chunk copied
// to its HBM slot on the copy stream as soon as it lands.  GPUDirect Storage (cuFile) would skip the
// staging copy; without the nvidia-fs module it degrades to this same bounce-buffer path.
struct SsdTier {
    static constexpr size_t kChunk = 8u << 20, kAlign = 4096;
    static constexpr int kSlots = 8, kReaders = 4;
    int fd = -1;
    bool direct = false;
    size_t rec_up = 0, rec = 0;
    char* stage[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    int next = 0;
    std::vector<std::thread> pool;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::function<void()>> q;
    bool stop = false;
    uint64_t read_bytes = 0;

    static size_t ru(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
    SsdTier(size_t up_b, size_t dn_b, size_t keys) {
        rec_up = ru(up_b);
        rec = rec_up + ru(dn_b);
        const char* dir = std::getenv("SMOE_SSD_DIR");
        std::string path = std::string(dir && *dir ? dir : "/tmp") + "/specmoe_ssd_" + std::to_string(getpid()) + "_" +
                           std::to_string(reinterpret_cast<uintptr_t>(this)) + ".bin";
        fd = open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC | O_DIRECT, 0600);
        direct = fd >= 0;
        if (fd < 0) fd = open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
        if (fd < 0) throw Error(kConfig, "expert store: cannot create the SSD-tier file " + path);
        unlink(path.c_str());  // removed when the engine closes it
        if (ftruncate(fd, (off_t)(rec * keys)) != 0) throw Error(kConfig, "expert store: SSD-tier file too large");
        for (int i = 0; i < kSlots; ++i) {
            SMOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stage[i]), kChunk, cudaHostAllocDefault));
            SMOE_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
        for (int i = 0; i < kReaders; ++i)
            pool.emplace_back([this] {
                for (;;) {
                    std::function<void()> job;
                    {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [&] { return stop || !q.empty(); });
                        if (stop && q.empty()) return;
                        job = std::move(q.front());
                        q.pop_front();
                    }
                    job();
                }
            });
    }
    ~SsdTier() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : pool) t.join();
        for (int i = 0; i < kSlots; ++i) {
            if (ev[i]) cudaEventDestroy(ev[i]);
            if (stage[i]) cudaFreeHost(stage[i]);
        }
        if (fd >= 0) close(fd);
    }
    void submit(std::function<void()> job) {
        {
            std::lock_guard<std::mutex> lk(mu);
            q.push_back(std::move(job));
        }
        cv.notify_one();
    }
    static void pread_all(int fd, char* buf, size_t n, off_t off, bool direct) {
        size_t done = 0;
        while (done < n) {
            const ssize_t r = pread(fd, buf + done, n - done, off + (off_t)done);
            if (r <= 0) throw Error(kCuda, "expert store: SSD-tier read failed");
            done += (size_t)r;
        }
        if (!direct) posix_fadvise(fd, off, (off_t)n, POSIX_FADV_DONTNEED);  // the next migration reads the device
    }
    // file region [off, off + n) -> device dst on stream s, chunk by chunk, kSlots - 1 reads ahead
    void read_to_device(size_t off, size_t n, char* dst, cudaStream_t s) {
        const size_t nch = (n + kChunk - 1) / kChunk;
        std::vector<std::atomic<int>> done(nch);
        std::vector<int> slot_of(nch);
        auto issue = [&](size_t i) {
            const int sl = next++ % kSlots;
            SMOE_CUDA(cudaEventSynchronize(ev[sl]));  // its previous chunk has left for the GPU
            slot_of[i] = sl;
            done[i] = 0;
            const size_t o = i * kChunk, len = ru(std::min(kChunk, n - o));
            char* buf = stage[sl];
            std::atomic<int>* flag = &done[i];
            const int f = fd;
            const bool dio = direct;
            submit([=] {
                try {
                    pread_all(f, buf, len, (off_t)(off + o), dio);
                    flag->store(1);
                } catch (...) {
                    flag->store(-1);
                }
            });
        };
        size_t issued = 0;
        for (; issued < nch && issued < (size_t)kSlots - 1; ++issued) issue(issued);
        for (size_t i = 0; i < nch; ++i) {
            while (done[i].load() == 0) std::this_thread::yield();
            if (done[i].load() < 0) throw Error(kCuda, "expert store: SSD-tier read failed");
            const size_t o = i * kChunk, len = std::min(kChunk, n - o);
            SMOE_CUDA(cudaMemcpyAsync(dst + o, stage[slot_of[i]], len, cudaMemcpyHostToDevice, s));
            SMOE_CUDA(cudaEventRecord(ev[slot_of[i]], s));
            read_bytes += len;
            if (issued < nch) issue(issued++);
        }
    }
    void write_from_device(size_t off, size_t n, const char* src, cudaStream_t s) {
        for (size_t o = 0; o < n; o += kChunk) {
            const size_t len = std::min(kChunk, n - o);
            SMOE_CUDA(cudaMemcpyAsync(stage[0], src + o, len, cudaMemcpyDeviceToHost, s));
            SMOE_CUDA(cudaStreamSynchronize(s));
            const size_t wl = ru(len);
            if (pwrite(fd, stage[0], wl, (off_t)(off + o)) != (ssize_t)wl)
                throw Error(kCuda, "expert store: SSD-tier write failed");
        }
    }
};

void Engine::SsdDeleter::operator()(SsdTier* t) const { delete t; }
double Engine::ssd_direct() const { return ssd ? (ssd->direct ? 1.0 : 0.0) : -1.0; }

void Engine::host_to_device(int key, int which, void* dst, cudaStream_t s) {
    const size_t bytes = expert_bytes(which), hk = hkey(key);
    if (ssd) {
        ssd->read_to_device(hk * ssd->rec + (which ? ssd->rec_up : 0), bytes, static_cast<char*>(dst), s);
        return;
    }
    const char* src = static_cast<const char*>(which ? host_down : host_up) + hk * bytes;
    SMOE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
}

void Engine::device_to_host(int key, int which, const void* src) {
    const size_t bytes = expert_bytes(which), hk = hkey(key);
    if (ssd) {
        ssd->write_from_device(hk * ssd->rec + (which ? ssd->rec_up : 0), bytes, static_cast<const char*>(src), stream);
        return;
    }
    char* dst = static_cast<char*>(which ? host_down : host_up) + hk * bytes;
    SMOE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream));
    sync();
}

void Engine::store_alloc(int exp_slots) {
    n_exp_slots = exp_slots;
    slot_key.assign(n_exp_slots, -1);
    key_pinned.assign((size_t)M * E, 0);
    key_prefetched.assign((size_t)M * E, 0);
    h_slot_of.assign((size_t)M * E, -1);
    free_slots.clear();
    for (int s = n_exp_slots - 1; s >= 0; --s) free_slots.push_back(s);
    const size_t ws = wt == kF32 ? 4 : 2;
    const size_t up_b = (size_t)U * d * ws, dn_b = (size_t)d * f * ws, owned = (size_t)M * (e_hi - e_lo);
    if (offload == 2) {
        ssd.reset(new SsdTier(up_b, dn_b, owned));
    } else {
        SMOE_CUDA(cudaHostAlloc(&host_up, owned * up_b, cudaHostAllocDefault));
        SMOE_CUDA(cudaHostAlloc(&host_down, owned * dn_b, cudaHostAllocDefault));
    }
    SMOE_CUDA(cudaMallocHost(&h_store, sizeof(int) * ((size_t)M * E + (4 + (size_t)ep_world) * E + 8)));
}

void Engine::store_reset() {
    std::fill(slot_key.begin(), slot_key.end(), -1);
    std::fill(key_pinned.begin(), key_pinned.end(), 0);
    std::fill(key_prefetched.begin(), key_prefetched.end(), 0);
    prev_need.clear();
    prefetch_bytes = prefetch_wasted = 0;
    prefetch_hits = 0;
    std::fill(h_slot_of.begin(), h_slot_of.end(), -1);
    free_slots.clear();
    for (int s = n_exp_slots - 1; s >= 0; --s) free_slots.push_back(s);
    upload_slot_rows(0, M);
}

// slot_of rows [m0, m1) -> device, ordered on the compute stream (pinned source region per layer).
// Under expert parallelism the GEMM groups are (source rank, local expert): their slot table ep_gslot
// is rebuilt from the same rows (group g -> this rank's expert e_lo + g % eo).
void Engine::upload_slot_rows(int m0, int m1) {
    int* hp = h_store;  // first M*E ints: pinned mirror of h_slot_of (or of the EP group slots)
    const size_t a = (size_t)m0 * E, n = (size_t)(m1 - m0) * E;
    if (ep_world > 1) {
        const int eo = e_hi - e_lo;
        for (int m = m0; m < m1; ++m)
            for (int g = 0; g < E; ++g) hp[(size_t)m * E + g] = h_slot_of[(size_t)m * E + e_lo + g % eo];
        SMOE_CUDA(cudaMemcpyAsync(ep_gslot + a, hp + a, n * sizeof(int), cudaMemcpyHostToDevice, stream));
        return;
    }
    std::memcpy(hp + a, h_slot_of.data() + a, n * sizeof(int));
    SMOE_CUDA(cudaMemcpyAsync(slot_of + a, hp + a, n * sizeof(int), cudaMemcpyHostToDevice, stream));
}

size_t Engine::expert_bytes(int which) const {
    const size_t ws = wt == kF32 ? 4 : 2;
    return which == 0 ? (size_t)U * d * ws : (size_t)d * f * ws;
}

// Copy one expert host -> HBM slot on the copy stream.
void Engine::store_copy_in(int key, int slot) {
    const size_t ub = expert_bytes(0), db = expert_bytes(1);
    host_to_device(key, 0, static_cast<char*>(up_pool) + (size_t)slot * ub, copy_stream);
    host_to_device(key, 1, static_cast<char*>(down_pool) + (size_t)slot * db, copy_stream);
    h2d_bytes += ub + db;
}

int Engine::store_take_slot(int key) {
    if (free_slots.empty())
        throw Error(kInvariant, "expert store: HBM slots exhausted (raise hbm_expert_slots to >= M*N + E - N)");
    const int s = free_slots.back();
    free_slots.pop_back();
    slot_key[s] = key;
    h_slot_of[key] = s;
    return s;
}

void Engine::store_release(int key) {
    const int s = h_slot_of[key];
    if (s < 0) return;
    slot_key[s] = -1;
    h_slot_of[key] = -1;
    free_slots.push_back(s);
}

// pin_draft_experts (memsim.cpp:115-150) made physical: used at setup (initial pin) and by
// forward() with explicit draft sets.
void Engine::store_pin_sets(const std::vector<std::vector<int>>& sets) {
    if (!offload) return;
    std::vector<uint8_t> target((size_t)M * E, 0);
    for (int m = 0; m < M; ++m)
        for (int e : sets[m])
            if (e >= e_lo && e < e_hi) target[(size_t)m * E + e] = 1;  // this rank's share of the sets
    for (int k = 0; k < M * E; ++k)
        if (key_pinned[k] && !target[k]) {
            key_pinned[k] = 0;
            store_release(k);
        }
    for (int k = 0; k < M * E; ++k) {
        if (!target[k]) continue;
        if (h_slot_of[k] < 0) store_copy_in(k, store_take_slot(k));
        key_pinned[k] = 1;
    }
    SMOE_CUDA(cudaStreamSynchronize(copy_stream));
    upload_slot_rows(0, M);
    sync();
}

// Inside an unrestricted pass, after route(mo): fetch this layer's missing experts.  With the
// overlap baseline's prefetch on (store_prefetch), the next layer's experts of the previous step are
// queued right behind them, so the copy engine keeps streaming while this layer computes and the host
// waits for the next gate; the next layer then copies only what the prefetch missed.  Prefetched
// experts the next layer does not route to are released unused at its finish (wasted bytes, counted).
void Engine::store_fetch_layer(int mo, const int* cnt_dev) {
    int* cnt = h_store + (size_t)M * E;
    SMOE_CUDA(cudaMemcpyAsync(cnt, cnt_dev, sizeof(int) * E, cudaMemcpyDeviceToHost, stream));
    sync();
    store_counts.assign(cnt, cnt + E);  // picks per expert over every row (unrestricted: final == raw)
    store_issue_layer(mo, cnt, group_slot);
}

// Expert parallelism: this rank owns experts [e_lo, e_hi); the counts every sender routed to them have
// arrived (rcnt, group g = (source rank g / eo, local expert g % eo)), so the rank fetches exactly
// needed ∩ owned over its own PCIe link.  The re-pin needs the layer's counts over all experts: one
// all-gather of every rank's per-expert counts of its own rows.
void Engine::store_fetch_layer_ep(int mo, const int* cnt_dev) {
    const int G = ep_world, eo = e_hi - e_lo;
    int* rc = h_store + (size_t)M * E;          // [E] received group counts
    int* all = rc + 3 * E + 8;                  // [G][E] gathered per-expert counts
    if (repin_hook) comm->allgather(cnt_dev, ep_cntg, sizeof(int) * E, stream);
    SMOE_CUDA(cudaMemcpyAsync(rc, rcnt, sizeof(int) * E, cudaMemcpyDeviceToHost, stream));
    if (repin_hook) SMOE_CUDA(cudaMemcpyAsync(all, ep_cntg, sizeof(int) * G * E, cudaMemcpyDeviceToHost, stream));
    sync();
    store_counts.assign(E, 0);
    if (repin_hook)
        for (int r = 0; r < G; ++r)
            for (int e = 0; e < E; ++e) store_counts[e] += (uint64_t)all[(size_t)r * E + e];
    std::vector<int> need(E, 0);  // owned experts' totals, indexed by the global expert id
    for (int g = 0; g < E; ++g) need[e_lo + g % eo] += rc[g];
    int* gs = rc + E;  // [E] group slots, staged after the fetch
    store_issue_layer(mo, need.data(), nullptr);
    for (int g = 0; g < E; ++g) gs[g] = rc[g] > 0 ? h_slot_of[(size_t)mo * E + e_lo + g % eo] : -1;
    SMOE_CUDA(cudaMemcpyAsync(ep_gslot + (size_t)mo * E, gs, sizeof(int) * E, cudaMemcpyHostToDevice, stream));
}

// Issue the copies of layer mo's needed (cnt[e] > 0), owned, non-resident experts on the copy stream
// (+ the overlap baseline's prefetch of the next layer), make the compute stream wait for them, and
// (single GPU) stage the layer's group slots into gslot_dev.
void Engine::store_issue_layer(int mo, const int* cnt, int* gslot_dev) {
    int* gslot = h_store + (size_t)M * E + E + 1;
    cudaEvent_t a, b;
    SMOE_CUDA(cudaEventCreate(&a));
    SMOE_CUDA(cudaEventCreate(&b));
    SMOE_CUDA(cudaEventRecord(a, copy_stream));
    for (int e = e_lo; e < e_hi; ++e) {
        const int key = mo * E + e;
        if (cnt[e] > 0) {
            if (h_slot_of[key] < 0) store_copy_in(key, store_take_slot(key));
            else if (key_prefetched[key]) ++prefetch_hits;
        } else if (key_prefetched[key]) {
            prefetch_wasted += expert_bytes(0) + expert_bytes(1);  // released unused at the layer's finish
        }
        key_prefetched[key] = 0;
    }
    // the copy stream is in order: this event also covers every earlier prefetch of this layer
    SMOE_CUDA(cudaEventRecord(b, copy_stream));
    SMOE_CUDA(cudaStreamWaitEvent(stream, b, 0));
    h2d_ev.emplace_back(a, b);
    if (store_prefetch && mo + 1 < M) {
        cudaEvent_t pa, pb;
        SMOE_CUDA(cudaEventCreate(&pa));
        SMOE_CUDA(cudaEventCreate(&pb));
        SMOE_CUDA(cudaEventRecord(pa, copy_stream));
        for (int e = e_lo; e < e_hi; ++e) {
            const int key = (mo + 1) * E + e;
            if (!prev_need.empty() && prev_need[key] && h_slot_of[key] < 0 && !free_slots.empty()) {
                const uint64_t before = h2d_bytes;
                store_copy_in(key, store_take_slot(key));
                prefetch_bytes += h2d_bytes - before;
                key_prefetched[key] = 1;
            }
        }
        SMOE_CUDA(cudaEventRecord(pb, copy_stream));
        h2d_ev.emplace_back(pa, pb);
    }
    if (gslot_dev) {
        for (int e = 0; e < E; ++e) gslot[e] = cnt[e] > 0 ? h_slot_of[(size_t)mo * E + e] : -1;
        SMOE_CUDA(cudaMemcpyAsync(gslot_dev, gslot, sizeof(int) * E, cudaMemcpyHostToDevice, stream));
    }
}

// After the layer's expert GEMMs are enqueued: optional re-pin (hot_temporal), then flush.
void Engine::store_finish_layer(int mo) {
    if (repin_hook) {
        std::vector<int> next;
        if (repin_hook(mo, store_counts.data(), next)) {
            std::vector<uint8_t> want(E, 0);
            for (int e : next) want[e] = 1;
            for (int e = e_lo; e < e_hi; ++e) {
                const int key = mo * E + e;
                if (want[e]) {
                    if (h_slot_of[key] < 0)
                        throw Error(kInvariant, "expert store: re-pinned expert not resident (replacement must be free)");
                    key_pinned[key] = 1;
                } else {
                    key_pinned[key] = 0;
                }
            }
        }
    }
    for (int e = e_lo; e < e_hi; ++e) {
        const int key = mo * E + e;
        if (!key_pinned[key]) store_release(key);
    }
    upload_slot_rows(mo, mo + 1);
}

void Engine::collect_h2d() {
    for (auto& p : h2d_ev) {
        float ms = 0.f;
        SMOE_CUDA(cudaEventSynchronize(p.second));
        SMOE_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
        h2d_ms += ms;
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    h2d_ev.clear();
}

}  // namespace smoe
