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
#include <algorithm>
#include <cstring>

#include "engine.h"

namespace smoe {

void Engine::store_alloc(int exp_slots) {
    n_exp_slots = exp_slots;
    slot_key.assign(n_exp_slots, -1);
    key_pinned.assign((size_t)M * E, 0);
    key_prefetched.assign((size_t)M * E, 0);
    h_slot_of.assign((size_t)M * E, -1);
    free_slots.clear();
    for (int s = n_exp_slots - 1; s >= 0; --s) free_slots.push_back(s);
    const size_t ws = wt == kF32 ? 4 : 2;
    const size_t up_b = (size_t)U * d * ws, dn_b = (size_t)d * f * ws;
    SMOE_CUDA(cudaHostAlloc(&host_up, (size_t)M * E * up_b, cudaHostAllocDefault));
    SMOE_CUDA(cudaHostAlloc(&host_down, (size_t)M * E * dn_b, cudaHostAllocDefault));
    SMOE_CUDA(cudaMallocHost(&h_store, sizeof(int) * ((size_t)M * E + 4 * (size_t)E + 8 + (size_t)Tmax * K)));
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
void Engine::upload_slot_rows(int m0, int m1) {
    int* hp = h_store;  // first M*E ints: pinned mirror of h_slot_of
    const size_t a = (size_t)m0 * E, n = (size_t)(m1 - m0) * E;
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
    SMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(up_pool) + (size_t)slot * ub, static_cast<char*>(host_up) + (size_t)key * ub,
                              ub, cudaMemcpyHostToDevice, copy_stream));
    SMOE_CUDA(cudaMemcpyAsync(static_cast<char*>(down_pool) + (size_t)slot * db,
                              static_cast<char*>(host_down) + (size_t)key * db, db, cudaMemcpyHostToDevice, copy_stream));
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
        for (int e : sets[m]) target[(size_t)m * E + e] = 1;
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
void Engine::store_fetch_layer(int mo, int T, const int* raw_dev, const int* cnt_dev) {
    int* cnt = h_store + (size_t)M * E;
    int* gslot = cnt + E + 1;
    int* raw = gslot + E;
    SMOE_CUDA(cudaMemcpyAsync(cnt, cnt_dev, sizeof(int) * E, cudaMemcpyDeviceToHost, stream));
    SMOE_CUDA(cudaMemcpyAsync(raw, raw_dev, sizeof(int) * T * K, cudaMemcpyDeviceToHost, stream));
    sync();
    cudaEvent_t a, b;
    SMOE_CUDA(cudaEventCreate(&a));
    SMOE_CUDA(cudaEventCreate(&b));
    SMOE_CUDA(cudaEventRecord(a, copy_stream));
    for (int e = 0; e < E; ++e) {
        const int key = mo * E + e;
        if (cnt[e] > 0) {
            if (h_slot_of[key] < 0) store_copy_in(key, store_take_slot(key));
            else if (key_prefetched[key]) ++prefetch_hits;
        } else if (key_prefetched[key]) {
            prefetch_wasted += expert_bytes(0) + expert_bytes(1);  // released unused at the layer's finish
        }
        key_prefetched[key] = 0;
        gslot[e] = cnt[e] > 0 ? h_slot_of[key] : -1;
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
        for (int e = 0; e < E; ++e) {
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
    SMOE_CUDA(cudaMemcpyAsync(group_slot, gslot, sizeof(int) * E, cudaMemcpyHostToDevice, stream));
    store_last_T = T;
}

// After the layer's expert GEMMs are enqueued: optional re-pin (hot_temporal), then flush.
void Engine::store_finish_layer(int mo) {
    if (repin_hook) {
        const int* raw = h_store + (size_t)M * E + 2 * E + 1;
        std::vector<int> next;
        if (repin_hook(mo, raw, store_last_T, next)) {
            std::vector<uint8_t> want(E, 0);
            for (int e : next) want[e] = 1;
            for (int e = 0; e < E; ++e) {
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
    for (int e = 0; e < E; ++e) {
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
