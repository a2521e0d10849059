// engine.cpp -- device model, weights, draft tables and the batched forward pass.
//
// Data layout in HBM: every GEMM weight is stored K-major with the
// output feature as the row ("out x in"), so a 128-row tile is one TMA box for tcgen05 and one
// 16-byte-vector row walk for the CUDA-core path:
//   mix  [L][d][d]           (reference mix is already out x in, model.cpp:29-39)
//   up   [S][U][d]           (reference up is d x f -> transposed; swiglu3: rows [0,f) w1, [f,2f) w3)
//   down [S][d][f]           (reference down is f x d -> transposed)
//   head [V][d]              (reference head is d x V -> transposed)
//   gate [M][E][d] f32, bias [M][E] f32, embedding [V][d] float64 (prefix sums stay float64)
// S = one slot per (MoE layer, expert) plus one per dense layer.
#include "engine.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>

#include <nvtx3/nvToolsExt.h>

namespace smoe {

NvtxRange::NvtxRange(const char* name) { nvtxRangePushA(name); }
NvtxRange::~NvtxRange() { nvtxRangePop(); }

namespace {

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    SMOE_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
}
void* dalloc_bytes(size_t n) {
    void* p = nullptr;
    SMOE_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1)));
    return p;
}

// Reference seeded normal stream: std::mt19937_64 + Marsaglia polar, second variate discarded
// (common.hpp:40-55).  Kept in the engine so exact-weight init never touches the oracle.
struct PolarStream {
    std::mt19937_64 rng;
    explicit PolarStream(uint64_t s) : rng(s) {}
    double u01() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
    double next() {
        for (;;) {
            double u = 2.0 * u01() - 1.0;
            double v = 2.0 * u01() - 1.0;
            double s = u * u + v * v;
            if (s > 0.0 && s < 1.0) return u * std::sqrt(-2.0 * std::log(s) / s);
        }
    }
    void fill(std::vector<double>& out, size_t n, double sd) {
        out.resize(n);
        for (size_t i = 0; i < n; ++i) out[i] = sd * next();
    }
};

}  // namespace

Engine::Engine(const smoe_engine_config& c) {
    L = c.num_layers; E = c.experts; K = c.top_k; d = c.hidden; f = c.ffn; V = c.vocab;
    skew = c.gate_skew; seed = c.seed; kind = c.expert_kind;
    wt = c.weight_type == SMOE_F32 ? kF32 : kBF16;
    Bmax = std::max(1, c.max_batch);
    Gmax = std::max(1, c.max_gamma);
    stride = Gmax + 1;
    Tmax = Bmax * (Gmax + 1);
    Hq = std::max(0, c.attn_heads);
    if (Hq > 0) {
        Hkv = c.kv_heads;
        hd = c.head_dim;
        theta = c.rope_theta;
        if (Hkv < 1 || Hq % Hkv || Hq / Hkv > 32 || hd < 2 || hd % 2 || !(theta > 0.0))
            throw Error(kConfig, "model: attention needs kv_heads | attn_heads (<= 32 per group), an even head_dim and rope_theta > 0");
        if (c.ep_world > 1) throw Error(kConfig, "engine: attention with expert parallelism is not supported");
        QD = Hq * hd;
        KD = Hkv * hd;
        QKVD = QD + 2 * KD;
        max_seq = c.max_seq_len > 0 ? c.max_seq_len : 512;
        maxp = (max_seq + Gmax + 1 + kKvPage - 1) / kKvPage;
    }
    device = c.device;
    offload = c.offload;
    if (E < 1 || K < 1 || K > E) throw Error(kConfig, "model: 1 <= top_k <= experts_per_block violated");
    if (E > 64) throw Error(kConfig, "engine: experts_per_block <= 64 (gate kernel bitmask) violated");
    if (K > 16) throw Error(kConfig, "engine: top_k <= 16 violated");
    if (V < 2) throw Error(kConfig, "model: vocab_size >= 2 violated");
    if (d < 1 || f < 1 || L < 1) throw Error(kConfig, "model: dims >= 1 violated");
    if (skew < 0.0) throw Error(kConfig, "model: gate_skew >= 0 violated");
    if (d % 8 || f % 8) throw Error(kConfig, "engine: hidden_dim and ffn_dim must be multiples of 8 (16-byte rows)");
    if (kind != kTanh2 && kind != kSwiglu3) throw Error(kConfig, "engine: unknown expert kind");
    mask.assign(L, 1);
    if (c.moe_mask)
        for (int l = 0; l < L; ++l) mask[l] = c.moe_mask[l] ? 1 : 0;
    moe_ord.assign(L, -1);
    for (int l = 0; l < L; ++l)
        if (mask[l]) { moe_ord[l] = (int)moe_index.size(); moe_index.push_back(l); }
    M = (int)moe_index.size();
    if (M == 0) throw Error(kConfig, "model: at least one layer must be an MoE block");
    n_dense = L - M;
    U = kind == kSwiglu3 ? 2 * f : f;
    if (c.gemm_backend == SMOE_GEMM_SIMT) use_tc = 0;
    else if (c.gemm_backend == SMOE_GEMM_TCGEN05) use_tc = 1;
    else use_tc = wt == kBF16 ? 1 : 0;
    if (use_tc && wt != kBF16) throw Error(kConfig, "engine: the tcgen05 path needs bf16 weights");
    {  // tiled weight layout (kernels.h tiled_index) for tcgen05 engines, per matrix whose rows come in 256s
        const char* v = getenv("SMOE_TILED");
        const bool want = use_tc && !(v && v[0] == '0');
        if (want && U % 256 == 0 && d % 256 == 0 && f % 64 == 0) {
            tile_up = d;
            tile_dn = f;
        }
        tile_mix = want && d % 256 == 0;
        tile_head = want && V % 256 == 0 && d % 64 == 0;
    }

    SMOE_CUDA(cudaSetDevice(device));
    SMOE_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    SMOE_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));

    const size_t ws = wt == kF32 ? 4 : 2;
    ep_world = std::max(1, c.ep_world);
    ep_rank = c.ep_rank;
    if (ep_rank < 0 || ep_rank >= ep_world) throw Error(kConfig, "engine: ep_rank outside [0, ep_world)");
    if (E % ep_world) throw Error(kConfig, "engine: experts_per_block must be divisible by ep_world");
    e_lo = ep_rank * (E / ep_world);
    e_hi = e_lo + E / ep_world;
    const int eo = E / ep_world;
    int exp_slots = M * eo;
    if (offload) {  // each rank stores its own experts: pinned draft share + two layers' transients
        exp_slots = c.hbm_expert_slots > 0 ? c.hbm_expert_slots : std::min(M * eo, M * std::min(4, eo) + 2 * eo);
        if (exp_slots < eo) throw Error(kConfig, "engine: hbm_expert_slots must be >= experts_per_block / ep_world");
    }
    n_slots = exp_slots + n_dense;
    emb64 = dalloc<double>((size_t)V * d);
    if (!attn()) mix = dalloc_bytes((size_t)L * d * d * ws);
    gate_w = dalloc<float>((size_t)M * E * d);
    gate_b = dalloc<float>((size_t)M * E);
    up_pool = dalloc_bytes((size_t)n_slots * U * d * ws);
    down_pool = dalloc_bytes((size_t)n_slots * d * f * ws);
    head = dalloc_bytes((size_t)V * d * ws);
    h_slot_of.assign((size_t)M * E, -1);  // experts of other EP ranks stay -1 (their GEMM groups are skipped)
    for (int m = 0; m < M; ++m)
        for (int e = e_lo; e < e_hi; ++e) h_slot_of[(size_t)m * E + e] = m * (e_hi - e_lo) + (e - e_lo);
    dense_slot.assign(L, -1);
    for (int l = 0, k = 0; l < L; ++l)
        if (!mask[l]) dense_slot[l] = exp_slots + k++;
    slot_of = dalloc<int>((size_t)M * E);
    if (offload) {
        stage_up = dalloc_bytes((size_t)U * d * ws);
        stage_down = dalloc_bytes((size_t)d * f * ws);
        store_alloc(exp_slots);  // everything starts in host DRAM; slot_of = -1
    }
    h2d(slot_of, h_slot_of.data(), sizeof(int) * M * E);
    std::vector<float> bias((size_t)M * E);
    for (int m = 0; m < M; ++m)
        for (int e = 0; e < E; ++e) bias[(size_t)m * E + e] = (float)(skew * (1.0 - (double)e / E));  // model.cpp:128-130
    h2d(gate_b, bias.data(), sizeof(float) * bias.size());

    if (attn()) {
        wqkv = dalloc_bytes((size_t)L * QKVD * d * ws);
        wo = dalloc_bytes((size_t)L * d * QD * ws);
        qbuf = dalloc<float>((size_t)Tmax * QD);
        attn_o = dalloc_bytes((size_t)Tmax * QD * ws);
        const size_t n_pages = (size_t)Bmax * maxp;
        kv = dalloc_bytes(n_pages * L * 2 * KD * kKvPage * ws);
        ptab = dalloc<int>((size_t)Bmax * maxp);
        SMOE_CUDA(cudaMemset(ptab, 0, sizeof(int) * Bmax * maxp));
        last_tok = dalloc<int>(Bmax);
        row_pos = dalloc<int>(Tmax);
        rope = dalloc<float2>((size_t)maxp * kKvPage * (hd / 2));
        launch_rope_table(maxp * kKvPage, hd, theta, rope, stream);
        pre_tok = dalloc<int>(Tmax);
        pre_pos = dalloc<int>(Tmax);
        kv_pages.assign(Bmax, {});
        for (int pg = (int)n_pages - 1; pg >= 0; --pg) kv_free.push_back(pg);
        h_seq_len.assign(Bmax, 0);
        tile_qkv = tile_mix && QKVD % 256 == 0;
        tile_wo = tile_mix && QD % 64 == 0;
        op_wqkv = {wqkv, (long long)L * QKVD, d, tile_qkv};
        op_wo = {wo, (long long)L * d, QD, tile_wo};
        op_ao = {attn_o, (long long)Tmax, QD};
    }
    seq_sum = dalloc<double>((size_t)Bmax * d);
    seq_len = dalloc<int>(Bmax);
    drafts = dalloc<int>((size_t)Bmax * stride);
    vam = dalloc<int>((size_t)Bmax * stride);
    SMOE_CUDA(cudaMemset(drafts, 0, sizeof(int) * Bmax * stride));
    SMOE_CUDA(cudaMemset(vam, 0, sizeof(int) * Bmax * stride));
    row_seq = dalloc<int>(2 * (size_t)Tmax);
    row_extra = dalloc<int>(2 * (size_t)Tmax);
    row_plen = dalloc<int>(Tmax);
    x = dalloc<float>((size_t)Tmax * d);
    xa = dalloc_bytes((size_t)Tmax * d * ws);
    raw_log = dalloc<int>((size_t)(Gmax + 1) * M * Tmax * K);
    fin_log = dalloc<int>((size_t)(Gmax + 1) * M * Tmax * K);
    wgt = dalloc<float>((size_t)Tmax * K);
    pos = dalloc<int>((size_t)Tmax * K);
    group_slot = dalloc<int>(E);
    grp_cnt = dalloc<int>((size_t)std::max(1, M) * E);
    SMOE_CUDA(cudaMemset(grp_cnt, 0, sizeof(int) * std::max(1, M) * E));
    const size_t seg_rows = (size_t)E * Tmax;  // expert segments of Tmax rows (gate dispatch)
    xperm = dalloc_bytes(seg_rows * d * ws);
    hbuf = dalloc_bytes(seg_rows * f * ws);
    // split-K counts are fixed per GEMM shape (never T-dependent) so results stay batch invariant
    if (use_tc) {
        const int nkb_d = (d + 63) / 64, nkb_f = (f + 63) / 64;
        auto pick = [](int nkb, int want) {  // effective split count: ceil(nkb / ceil(nkb / want))
            want = std::max(1, std::min(want, nkb));
            const int per = (nkb + want - 1) / want;
            return (nkb + per - 1) / per;
        };
        // mix: about one unit per SM at T <= 256 (measured best on the C2 shape: s_mix 4 > 8 > 2);
        // down: at least 2 splits, more until a pair unit (256 weight rows) streams <= 2 MB.  At C2 a
        // 2-split down unit streams 3.7 MB and a draft pass's last down units left a 44 us tail: B=64
        // 54.1 ms/step at 4 splits vs 57.0 at 2, 54.0-54.3 at 6/8, 56.2 at 16 (tools/ab_env.sh, same
        // box).  C4 (f=1408): 2 splits, 16.8 vs 17.4 ms/step at 4.
        const long long pair_unit_bytes = 256ll * f * 2;  // 256 weight rows x f bf16
        // (attention: the Wo GEMM, K = Hq*hd, produces the partials the gate kernel adds in the Mix's place)
        s_mix = pick(attn() ? (QD + 63) / 64 : nkb_d, std::max(1, 148 / std::max(1, (d + 127) / 128)));
        if (attn()) s_qkv = pick(nkb_d, std::max(1, 148 / std::max(1, (QKVD + 127) / 128)));
        s_down = pick(nkb_f, std::max(2, (int)((pair_unit_bytes + (2 << 20) - 1) / (2 << 20))));
        if (const char* v = getenv("SMOE_S_MIX")) s_mix = pick(attn() ? (QD + 63) / 64 : nkb_d, atoi(v));  // tuning overrides
        if (const char* v = getenv("SMOE_S_DOWN")) s_down = pick(nkb_f, atoi(v));
    }
    ybuf = dalloc<float>((size_t)s_down * seg_rows * d);
    if (ep_world > 1) {
        xrecv = dalloc_bytes(seg_rows * d * ws);
        ysend = dalloc<float>(seg_rows * d);
        yret = dalloc<float>((size_t)s_down * seg_rows * d);
        ep_flags = dalloc<int>(2 * (size_t)ep_world);
        SMOE_CUDA(cudaMemset(ep_flags, 0, sizeof(int) * 2 * ep_world));
        ep_peer = dalloc<void*>(4 * (size_t)ep_world);
        const char* mode = getenv("SMOE_EP_MODE");
        ep_p2p = use_tc && fuse_moe && E <= 64 && !(mode && std::string(mode) == "a2a");
        rcnt = dalloc<int>(E);
        ep_gslot = dalloc<int>((size_t)std::max(1, M) * E);
        ep_cntg = dalloc<int>((size_t)ep_world * E);
        ep_logs = dalloc<int>((size_t)(1 + ep_world) * 2 * std::max(1, M) * Tmax * K);
        amax_loc = dalloc<int>(Tmax);
        logits_loc = dalloc<float>((size_t)Tmax * V);
        // group g = (source rank g / (E/G), local expert g % (E/G)) -> this rank's weight slot
        std::vector<int> gs((size_t)std::max(1, M) * E);
        for (int m = 0; m < M; ++m)
            for (int g = 0; g < E; ++g) gs[(size_t)m * E + g] = h_slot_of[(size_t)m * E + e_lo + g % eo];
        h2d(ep_gslot, gs.data(), sizeof(int) * gs.size());
    }
    pmix = dalloc<float>((size_t)s_mix * Tmax * d);
    if (attn()) pqkv = dalloc<float>((size_t)s_qkv * Tmax * QKVD);
    // + ep_world rows: an EP all-gather writes G * ceil(T/G) >= T rows
    logits = dalloc<float>((size_t)(Tmax + ep_world) * V);
    amax = dalloc<int>(Tmax + ep_world);
    in_draft = dalloc<uint8_t>((size_t)M * E);
    draft_sorted = dalloc<int>((size_t)M * E);
    rank = dalloc<int>((size_t)M * E * E);
    acc = dalloc<int>(Bmax);
    corr = dalloc<int>(Bmax);
    commit_toks = dalloc<int>((size_t)Bmax * stride);
    commit_take = dalloc<int>(Bmax);
    seqs = dalloc<int>(Bmax);
    flags = dalloc<int>(1);
    SMOE_CUDA(cudaMemset(flags, 0, sizeof(int)));
    sched = dalloc<int>(8);  // two counter slots: consecutive GEMM launches may overlap under PDL
    SMOE_CUDA(cudaMemset(sched, 0, 8 * sizeof(int)));
    moe_done = dalloc<int>(128);
    SMOE_CUDA(cudaMemset(moe_done, 0, 128 * sizeof(int)));
    if (const char* v = getenv("SMOE_FUSED_MOE")) fuse_moe = atoi(v) != 0;

    h_small_n = (size_t)Tmax * 8 + (size_t)M * E * (E + 2) + 4096;
    SMOE_CUDA(cudaMallocHost(&h_small, h_small_n * sizeof(int)));

    op_mix = {mix, (long long)L * d, d, tile_mix};
    op_up = {up_pool, (long long)n_slots * U, d, tile_up > 0};
    op_down = {down_pool, (long long)n_slots * d, f, tile_dn > 0};
    op_head = {head, (long long)V, d, tile_head};
    op_xa = {xa, (long long)Tmax, d};
    op_xperm = {xperm, (long long)seg_rows, d};
    if (xrecv) op_xrecv = {xrecv, (long long)seg_rows, d};
    op_h = {hbuf, (long long)seg_rows, f};
    SMOE_CUDA(cudaDeviceSynchronize());  // legacy-stream memsets above vs. the non-blocking engine stream
}

Engine::~Engine() {
    auto fr = [](void* p) { if (p) cudaFree(p); };
    if (stream) cudaStreamSynchronize(stream);
    for (auto& kv : phase_graphs) cudaGraphExecDestroy(kv.second.exec);
    if (capture_stream) cudaStreamDestroy(capture_stream);
    fr(emb64); fr(mix); fr(gate_w); fr(gate_b); fr(up_pool); fr(down_pool); fr(head); fr(slot_of);
    fr(seq_sum); fr(seq_len); fr(drafts); fr(vam); fr(row_seq); fr(row_extra); fr(row_plen); fr(x); fr(xa);
    fr(raw_log); fr(fin_log); fr(wgt); fr(pos); fr(group_slot); fr(grp_cnt); fr(xperm); fr(hbuf); fr(ybuf); fr(pmix);
    for (void* q : ep_ipc_opened) cudaIpcCloseMemHandle(q);
    fr(xrecv); fr(ysend); fr(yret); fr(rcnt); fr(ep_gslot); fr(ep_logs); fr(amax_loc); fr(logits_loc);
    fr(ep_flags); fr(ep_peer); fr(aff_dev);
    fr(ep_cntg); fr(wqkv); fr(wo); fr(pqkv); fr(qbuf); fr(attn_o); fr(kv); fr(ptab); fr(last_tok); fr(row_pos); fr(rope);
    fr(pre_tok); fr(pre_pos); fr(samp_u); fr(samp_q); fr(samp_stats); fr(samp_ratio); fr(samp_i);
    fr(logits); fr(amax); fr(in_draft); fr(draft_sorted); fr(rank); fr(acc); fr(corr); fr(commit_toks);
    if (up_arena) cudaFreeHost(up_arena);
    if (dn_arena) cudaFreeHost(dn_arena);
    fr(commit_take); fr(seqs); fr(flags); fr(sched); fr(moe_done); fr(scratch64);
    if (h_small) cudaFreeHost(h_small);
    if (h_store) cudaFreeHost(h_store);
    fr(stage_up); fr(stage_down);
    for (auto& p : h2d_ev) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    if (host_up) cudaFreeHost(host_up);
    if (host_down) cudaFreeHost(host_down);
    for (auto& kv : prof)
        for (auto& p : kv.second.ev) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
}

uint64_t Engine::real_bytes_per_expert() const {
    return (uint64_t)(kind == kSwiglu3 ? 3 : 2) * d * f * (wt == kF32 ? 4 : 2);
}

void Engine::sync() { SMOE_CUDA(cudaStreamSynchronize(stream)); }

// Host->device copy ordered on the engine stream.  (A plain cudaMemcpy from pageable memory may
// return before its DMA lands and is not ordered with a non-blocking stream.)
void Engine::h2d(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    SMOE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
    sync();
}

void Engine::sampling_alloc() {
    if (samp_u) return;
    samp_u = dalloc<double>((size_t)Gmax * Bmax + (size_t)Bmax * (Gmax + 1));
    samp_q = dalloc<double>((size_t)Gmax * Bmax * V);
    samp_stats = dalloc<double>((size_t)Tmax * 2);
    samp_ratio = dalloc<double>((size_t)Bmax * Gmax);
    samp_i = dalloc<int>((size_t)2 * Bmax + 1);
}

void Engine::upload_doubles(double* dst, const double* src, size_t n) {
    if (n == 0) return;
    std::vector<int> as_ints(n * 2);
    std::memcpy(as_ints.data(), src, n * sizeof(double));
    upload_ints(reinterpret_cast<int*>(dst), as_ints.data(), as_ints.size());
}

void Engine::check_flags() {
    int h = 0;
    SMOE_CUDA(cudaMemcpy(&h, flags, sizeof(int), cudaMemcpyDeviceToHost));
    if (h) {
        SMOE_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), stream));
        sync();
        if (h & kFlagNonFiniteLogits) throw Error(kInvariant, "greedy_next: non-finite logits");
        if (h & kFlagNonFiniteGate) throw Error(kInvariant, "softmax: non-finite input");
        if (h & kFlagEmptyRemap) throw Error(kInvariant, "nearest_draft_expert: empty candidate set");
        if (h & kFlagZeroDrawProb) throw Error(kInvariant, "verify_sampling: zero draw probability for proposed token");
    }
}

void Engine::upload_async(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    const size_t need = (up_arena_off + bytes + 255) & ~size_t(255);
    if (need > up_arena_n) {  // grow: drain the queued copies first (they read the old arena)
        SMOE_CUDA(cudaStreamSynchronize(stream));
        if (up_arena) SMOE_CUDA(cudaFreeHost(up_arena));
        up_arena_n = std::max<size_t>(2 * need, 1 << 20);
        SMOE_CUDA(cudaMallocHost(&up_arena, up_arena_n));
        up_arena_off = 0;
    }
    char* slot = up_arena + up_arena_off;
    std::memcpy(slot, src, bytes);
    up_arena_off = (up_arena_off + bytes + 255) & ~size_t(255);
    ctl_h2d += bytes;
    SMOE_CUDA(cudaMemcpyAsync(dst, slot, bytes, cudaMemcpyHostToDevice, stream));
}
void Engine::download_async(void* host_dst, const void* dev_src, size_t row_bytes, size_t rows, size_t dev_pitch) {
    const size_t bytes = row_bytes * rows;
    if (!bytes) return;
    const size_t need = (dn_arena_off + bytes + 255) & ~size_t(255);
    if (need > dn_arena_n) {  // grow: complete the queued readbacks out of the old arena first
        SMOE_CUDA(cudaStreamSynchronize(stream));
        download_finish();
        if (dn_arena) SMOE_CUDA(cudaFreeHost(dn_arena));
        dn_arena_n = std::max<size_t>(2 * need, 1 << 20);
        SMOE_CUDA(cudaMallocHost(&dn_arena, dn_arena_n));
    }
    char* slot = dn_arena + dn_arena_off;
    if (rows == 1)
        SMOE_CUDA(cudaMemcpyAsync(slot, dev_src, bytes, cudaMemcpyDeviceToHost, stream));
    else
        SMOE_CUDA(cudaMemcpy2DAsync(slot, row_bytes, dev_src, dev_pitch, row_bytes, rows, cudaMemcpyDeviceToHost,
                                    stream));
    dn_pending.push_back({host_dst, dn_arena_off, bytes});
    dn_arena_off = (dn_arena_off + bytes + 255) & ~size_t(255);
}
void Engine::download_finish() {  // the stream must be synchronised
    for (const auto& pd : dn_pending) std::memcpy(pd.dst, dn_arena + pd.off, pd.bytes);
    dn_pending.clear();
    dn_arena_off = 0;
}
void Engine::upload_ints(int* dst, const int* src, size_t n) {
    // synchronous-safe: stage through pinned memory then wait, so callers may reuse src at once
    if (n == 0) return;
    SMOE_CUDA(cudaStreamSynchronize(stream));
    if (n > h_small_n) {
        SMOE_CUDA(cudaFreeHost(h_small));
        h_small_n = n * 2;
        SMOE_CUDA(cudaMallocHost(&h_small, h_small_n * sizeof(int)));
    }
    std::memcpy(h_small, src, n * sizeof(int));
    ctl_h2d += n * sizeof(int);
    SMOE_CUDA(cudaMemcpyAsync(dst, h_small, n * sizeof(int), cudaMemcpyHostToDevice, stream));
    SMOE_CUDA(cudaStreamSynchronize(stream));
}

// ------------------------------------------------------------------ weights
void Engine::upload_tensor(const std::string& name, int layer, int expert, const double* src, long long n) {
    auto need = [&](long long want) {
        if (n != want) throw Error(kConfig, "upload_tensor: " + name + " size mismatch");
    };
    auto stage = [&](long long cnt) -> double* {
        if ((size_t)cnt > scratch64_n) {
            if (scratch64) SMOE_CUDA(cudaFree(scratch64));
            scratch64_n = (size_t)cnt;
            scratch64 = dalloc<double>(scratch64_n);
        }
        h2d(scratch64, src, sizeof(double) * cnt);
        return scratch64;
    };
    const size_t ws = wt == kF32 ? 4 : 2;
    auto at = [&](void* base, size_t elems) { return static_cast<char*>(base) + elems * ws; };
    // Destination of an expert matrix: its HBM slot, or (offload) a device staging buffer that is
    // read-modified-written against the key's region of the pinned host pool.
    int off_key = -1;
    if ((name == "up" || name == "w1" || name == "w3" || name == "down" || name == "w2") && layer >= 0 && layer < L &&
        mask[layer] && expert >= 0 && expert < E && (expert < e_lo || expert >= e_hi)) {
        if (n != (long long)d * f) throw Error(kConfig, "upload_tensor: " + name + " size mismatch");
        return;  // another EP rank owns this expert
    }
    auto slot_for = [&]() -> int {
        if (layer < 0 || layer >= L) throw Error(kConfig, "upload_tensor: layer out of range");
        if (mask[layer]) {
            if (expert < 0 || expert >= E) throw Error(kConfig, "upload_tensor: expert out of range");
            if (offload) {
                off_key = moe_ord[layer] * E + expert;
                return -1;
            }
            return h_slot_of[(size_t)moe_ord[layer] * E + expert];
        }
        return dense_slot[layer];
    };
    auto up_dst = [&]() -> void* {
        const int sl = slot_for();
        if (sl >= 0) return at(up_pool, (size_t)sl * U * d);
        host_to_device(off_key, 0, stage_up, stream);  // read-modify-write of the w1/w3 rows
        return stage_up;
    };
    auto down_dst = [&]() -> void* {
        const int sl = slot_for();
        if (sl >= 0) return at(down_pool, (size_t)sl * d * f);
        return stage_down;
    };
    if (name == "embedding") {
        need((long long)V * d);
        h2d(emb64, src, sizeof(double) * n);
    } else if (name == "head") {
        need((long long)d * V);
        launch_convert_transpose(stage(n), d, V, head, wt, stream, 1, 0, tile_head);
    } else if (name == "mix") {
        need((long long)d * d);
        if (attn()) throw Error(kConfig, "upload_tensor: an attention model has no mix (wq/wk/wv/wo)");
        if (tile_mix) launch_convert(stage(n), n, mix, wt, stream, d, (long long)layer * d);
        else launch_convert(stage(n), n, at(mix, (size_t)layer * d * d), wt, stream);
    } else if (name == "wq" || name == "wk" || name == "wv" || name == "wo") {
        if (!attn()) throw Error(kConfig, "upload_tensor: " + name + " needs an attention model");
        if (layer < 0 || layer >= L) throw Error(kConfig, "upload_tensor: layer out of range");
        if (name == "wo") {
            need((long long)d * QD);
            if (tile_wo) launch_convert(stage(n), n, wo, wt, stream, QD, (long long)layer * d);
            else launch_convert(stage(n), n, at(wo, (size_t)layer * d * QD), wt, stream);
        } else {
            const int row0 = name == "wq" ? 0 : name == "wk" ? QD : QD + KD;
            need((long long)(name == "wq" ? QD : KD) * d);
            if (tile_qkv) launch_convert(stage(n), n, wqkv, wt, stream, d, (long long)layer * QKVD + row0);
            else launch_convert(stage(n), n, at(wqkv, ((size_t)layer * QKVD + row0) * d), wt, stream);
        }
    } else if (name == "gate") {
        need((long long)d * E);
        if (layer < 0 || layer >= L || !mask[layer]) throw Error(kConfig, "upload_tensor: gate on a dense layer");
        launch_convert_transpose(stage(n), d, E, gate_w + (size_t)moe_ord[layer] * E * d, kF32, stream);
    } else if (name == "gate_bias") {
        need(E);
        launch_convert(stage(n), n, gate_b + (size_t)moe_ord[layer] * E, kF32, stream);
    } else if (name == "up" || name == "w1") {
        need((long long)d * f);
        // SwiGLU: w1 feature j -> pool row 2j, w3 feature j -> row 2j+1 (one 128-row tile = 64 features)
        launch_convert_transpose(stage(n), d, f, up_dst(), wt, stream, kind == kSwiglu3 ? 2 : 1, 0, tile_up > 0);
    } else if (name == "w3") {
        need((long long)d * f);
        if (kind != kSwiglu3) throw Error(kConfig, "upload_tensor: w3 needs the swiglu3 expert kind");
        launch_convert_transpose(stage(n), d, f, up_dst(), wt, stream, 2, 1, tile_up > 0);
    } else if (name == "down" || name == "w2") {
        need((long long)f * d);
        launch_convert_transpose(stage(n), f, d, down_dst(), wt, stream, 1, 0, tile_dn > 0);
    } else {
        throw Error(kConfig, "upload_tensor: unknown tensor " + name);
    }
    SMOE_CUDA(cudaGetLastError());
    if (off_key >= 0) {  // write the converted expert matrix back to the pinned host pool
        const bool is_down = name == "down" || name == "w2";
        sync();
        device_to_host(off_key, is_down ? 1 : 0, is_down ? stage_down : stage_up);
    }
    sync();
}

// model.cpp:106-143 draw order; affinity (drafting.cpp:28-57) from the same float64 values.
void Engine::init_exact() {
    PolarStream ps(seed);
    const double sd = 1.0 / std::sqrt((double)d);
    std::vector<double> buf;
    ps.fill(buf, (size_t)V * d, sd);
    upload_tensor("embedding", -1, -1, buf.data(), (long long)buf.size());
    affinity.assign((size_t)M * E * E, 0.0);
    const int nmat = kind == kSwiglu3 ? 3 : 2;
    std::vector<std::vector<double>> ex((size_t)E * nmat);
    for (int l = 0; l < L; ++l) {
        if (attn()) {  // the attention weights take the mix's place in the draw order (oracle fwd_attn)
            const char* names[4] = {"wq", "wk", "wv", "wo"};
            const size_t cnt[4] = {(size_t)QD * d, (size_t)KD * d, (size_t)KD * d, (size_t)d * QD};
            for (int q = 0; q < 4; ++q) {
                ps.fill(buf, cnt[q], sd);
                upload_tensor(names[q], l, -1, buf.data(), (long long)buf.size());
            }
        } else {
            ps.fill(buf, (size_t)d * d, sd);
            upload_tensor("mix", l, -1, buf.data(), (long long)buf.size());
        }
        if (mask[l]) {
            ps.fill(buf, (size_t)d * E, sd);
            upload_tensor("gate", l, -1, buf.data(), (long long)buf.size());
            for (int e = 0; e < E; ++e) {
                const char* names3[3] = {"w1", "w3", "w2"};
                const char* names2[2] = {"up", "down"};
                for (int q = 0; q < nmat; ++q) {
                    auto& v = ex[(size_t)e * nmat + q];
                    ps.fill(v, (size_t)d * f, sd);
                    upload_tensor(nmat == 3 ? names3[q] : names2[q], l, e, v.data(), (long long)v.size());
                }
            }
            double* D = affinity.data() + (size_t)moe_ord[l] * E * E;
            for (int i = 0; i < E; ++i)
                for (int j = i + 1; j < E; ++j) {
                    double ss = 0.0;
                    for (int q = 0; q < nmat; ++q) {
                        const double* a = ex[(size_t)i * nmat + q].data();
                        const double* b = ex[(size_t)j * nmat + q].data();
                        const size_t n = (size_t)d * f;
                        for (size_t k = 0; k < n; ++k) {
                            double df = a[k] - b[k];
                            ss += df * df;
                        }
                    }
                    D[(size_t)i * E + j] = D[(size_t)j * E + i] = std::sqrt(ss);
                }
        } else {
            const char* names3[3] = {"w1", "w3", "w2"};
            const char* names2[2] = {"up", "down"};
            for (int q = 0; q < nmat; ++q) {
                ps.fill(buf, (size_t)d * f, sd);
                upload_tensor(nmat == 3 ? names3[q] : names2[q], l, -1, buf.data(), (long long)buf.size());
            }
        }
    }
    ps.fill(buf, (size_t)d * V, sd);
    upload_tensor("head", -1, -1, buf.data(), (long long)buf.size());
    have_affinity = true;
    ++affinity_gen;
}

void Engine::init_device(uint64_t s) {
    const double sd = 1.0 / std::sqrt((double)d);
    uint64_t tid = 1;
    launch_fill_normal_f64(emb64, (long long)V * d, sd, s, tid++, stream);
    if (attn()) {  // tensor ids 7, 8 (after the head's): the other tensors keep their streams
        launch_fill_normal(wqkv, wt, (long long)L * QKVD * d, sd, s, 7, stream, 0, tile_qkv ? d : 0);
        launch_fill_normal(wo, wt, (long long)L * d * QD, sd, s, 8, stream, 0, tile_wo ? QD : 0);
        ++tid;
    } else {
        launch_fill_normal(mix, wt, (long long)L * d * d, sd, s, tid++, stream, 0, tile_mix ? d : 0);
    }
    launch_fill_normal(gate_w, kF32, (long long)M * E * d, sd, s, tid++, stream);
    const uint64_t tid_up = tid++, tid_down = tid++;
    dev_rng = true;
    dev_seed = s;
    if (!offload && ep_world > 1) {  // this rank's experts, same values as the single-GPU layout
        const size_t ws = wt == kF32 ? 4 : 2;
        for (int m = 0; m < M; ++m)
            for (int e = e_lo; e < e_hi; ++e) {
                const int key = m * E + e, slot = h_slot_of[key];
                launch_fill_normal(static_cast<char*>(up_pool) + (size_t)slot * U * d * ws, wt, (long long)U * d, sd, s,
                                   tid_up, stream, (long long)key * U * d, tile_up);
                launch_fill_normal(static_cast<char*>(down_pool) + (size_t)slot * d * f * ws, wt, (long long)d * f, sd,
                                   s, tid_down, stream, (long long)key * d * f, tile_dn);
            }
        for (int l = 0, k = 0; l < L; ++l)
            if (!mask[l]) {
                const long long gi = (long long)(M * E + k);
                launch_fill_normal(static_cast<char*>(up_pool) + (size_t)dense_slot[l] * U * d * ws, wt, (long long)U * d,
                                   sd, s, tid_up, stream, gi * U * d, tile_up);
                launch_fill_normal(static_cast<char*>(down_pool) + (size_t)dense_slot[l] * d * f * ws, wt,
                                   (long long)d * f, sd, s, tid_down, stream, gi * d * f, tile_dn);
                ++k;
            }
    } else if (!offload) {
        launch_fill_normal(up_pool, wt, (long long)n_slots * U * d, sd, s, tid_up, stream, 0, tile_up);
        launch_fill_normal(down_pool, wt, (long long)n_slots * d * f, sd, s, tid_down, stream, 0, tile_dn);
    } else {
        // identical values to the HBM-resident layout (element index = key*U*d + j), staged per expert;
        // under expert parallelism only this rank's experts
        const size_t ws = wt == kF32 ? 4 : 2;
        for (int key = 0; key < M * E; ++key) {
            if (!owns(key)) continue;
            launch_fill_normal(stage_up, wt, (long long)U * d, sd, s, tid_up, stream, (long long)key * U * d, tile_up);
            launch_fill_normal(stage_down, wt, (long long)d * f, sd, s, tid_down, stream, (long long)key * d * f, tile_dn);
            device_to_host(key, 0, stage_up);
            device_to_host(key, 1, stage_down);
        }
        for (int l = 0, k = 0; l < L; ++l)
            if (!mask[l]) {
                const long long gi = (long long)(M * E + k);
                launch_fill_normal(static_cast<char*>(up_pool) + (size_t)dense_slot[l] * U * d * ws, wt, (long long)U * d,
                                   sd, s, tid_up, stream, gi * U * d, tile_up);
                launch_fill_normal(static_cast<char*>(down_pool) + (size_t)dense_slot[l] * d * f * ws, wt,
                                   (long long)d * f, sd, s, tid_down, stream, gi * d * f, tile_dn);
                ++k;
            }
    }
    launch_fill_normal(head, wt, (long long)V * d, sd, s, tid++, stream, 0, tile_head ? d : 0);
    SMOE_CUDA(cudaGetLastError());
    sync();
    have_affinity = false;
}

void Engine::build_affinity_device() {
    constexpr int kChunks = 64;  // matches kernels.cu kPairChunks
    const size_t need = (size_t)E * E * kChunks;
    if (need > scratch64_n) {
        if (scratch64) SMOE_CUDA(cudaFree(scratch64));
        scratch64_n = need;
        scratch64 = dalloc<double>(need);
    }
    affinity.assign((size_t)M * E * E, 0.0);
    std::vector<double> part(need);
    const size_t ws = wt == kF32 ? 4 : 2;
    if (offload) store_reset();
    std::vector<int> ident(E);
    for (int e = 0; e < E; ++e) ident[e] = e;
    void *tmp_up = nullptr, *tmp_down = nullptr;
    if (ep_world > 1) {  // experts of other ranks are not resident: regenerate each layer's E experts
        if (!dev_rng)
            throw Error(kConfig, "expert parallelism: build the affinity on the host (smoe_set_affinity) for uploaded weights");
        tmp_up = dalloc_bytes((size_t)E * U * d * ws);
        tmp_down = dalloc_bytes((size_t)E * d * f * ws);
    }
    for (int m = 0; m < M; ++m) {
        SMOE_CUDA(cudaMemsetAsync(scratch64, 0, need * sizeof(double), stream));
        const int* slots = slot_of + (size_t)m * E;
        if (offload && ep_world == 1) {  // bring the layer's experts into slots 0..E-1 for the pairwise pass
            for (int e = 0; e < E; ++e) store_copy_in(m * E + e, e);
            SMOE_CUDA(cudaStreamSynchronize(copy_stream));
            upload_ints(group_slot, ident.data(), E);
            slots = group_slot;
        }
        if (tmp_up) {
            const double sd = 1.0 / std::sqrt((double)d);
            for (int e = 0; e < E; ++e) {
                const long long key = (long long)m * E + e;
                launch_fill_normal(static_cast<char*>(tmp_up) + (size_t)e * U * d * ws, wt, (long long)U * d, sd, dev_seed,
                                   4, stream, key * U * d, tile_up);
                launch_fill_normal(static_cast<char*>(tmp_down) + (size_t)e * d * f * ws, wt, (long long)d * f, sd,
                                   dev_seed, 5, stream, key * d * f, tile_dn);
            }
            upload_ints(group_slot, ident.data(), E);
            slots = group_slot;
        }
        const void* pool_up = tmp_up ? tmp_up : up_pool;
        const void* pool_down = tmp_down ? tmp_down : down_pool;
        launch_pairwise_sqdist(pool_up, wt, (long long)U * d, (long long)U * d, slots, E, scratch64, stream);
        launch_pairwise_sqdist(pool_down, wt, (long long)d * f, (long long)d * f, slots, E, scratch64, stream);
        (void)ws;
        SMOE_CUDA(cudaMemcpyAsync(part.data(), scratch64, need * sizeof(double), cudaMemcpyDeviceToHost, stream));
        sync();
        double* D = affinity.data() + (size_t)m * E * E;
        for (int i = 0; i < E; ++i)
            for (int j = i + 1; j < E; ++j) {
                double s = 0.0;
                for (int c = 0; c < kChunks; ++c) s += part[((size_t)i * E + j) * kChunks + c];
                D[(size_t)i * E + j] = D[(size_t)j * E + i] = std::sqrt(s);
            }
    }
    if (tmp_up) SMOE_CUDA(cudaFree(tmp_up));
    if (tmp_down) SMOE_CUDA(cudaFree(tmp_down));
    if (offload) h2d_bytes = 0;
    have_affinity = true;
    ++affinity_gen;
}

// ------------------------------------------------------------------ draft tables
// For each MoE layer and raw expert r: the draft members ordered by (affinity distance to r, index)
// -- the order nearest_draft_expert (drafting.cpp:123-138) scans implicitly.  The device walks this
// list and takes the first member not already chosen, so no float64 compare happens on the GPU.
void Engine::set_draft_sets(const std::vector<std::vector<int>>& sets, int n_draft, bool async) {
    if ((int)sets.size() != M) throw Error(kInvariant, "forward: restricted set count != MoE layer count");
    // per-layer sizes may differ (RestrictedExperts allows it); rows are padded with -1 to the widest
    // Duplicates are kept: the reference's candidate lists are multisets (drafting.cpp:140-151 sizes
    // the surrogate's modulus by them), and the device walks the sorted multiset the same way.  The
    // per-layer tables hold E entries, so a set longer than E (necessarily with repeats) is refused.
    int nmax = 0;
    for (const auto& st : sets) {
        if ((int)st.size() < K) throw Error(kInvariant, "forward: restricted set smaller than top_k");
        if ((int)st.size() > E) throw Error(kInvariant, "forward: restricted set larger than experts_per_block");
        for (int x : st)
            if (x < 0 || x >= E) throw Error(kInvariant, "forward: draft expert out of range");
        nmax = std::max(nmax, (int)st.size());
    }
    (void)n_draft;
    std::vector<uint8_t> ind((size_t)M * E, 0);
    std::vector<int> sorted((size_t)M * E, -1);
    for (int m = 0; m < M; ++m) {
        std::vector<int> srt(sets[m]);
        std::sort(srt.begin(), srt.end());
        for (size_t i = 0; i < srt.size(); ++i) {
            ind[(size_t)m * E + srt[i]] = 1;
            sorted[(size_t)m * E + i] = srt[i];
        }
    }
    // the per-(layer, raw expert) orders are built on the device from a resident copy of the affinity
    if (have_affinity && aff_dev_gen != affinity_gen) {
        if (!aff_dev) aff_dev = dalloc<double>((size_t)M * E * E);
        if (affinity.size() != (size_t)M * E * E) throw Error(kInvariant, "affinity table shape does not match the model");
        SMOE_CUDA(cudaMemcpyAsync(aff_dev, affinity.data(), affinity.size() * sizeof(double), cudaMemcpyHostToDevice,
                                  stream));
        sync();
        aff_dev_gen = affinity_gen;
    }
    if (async) {
        upload_async(in_draft, ind.data(), ind.size());
        upload_async(draft_sorted, sorted.data(), sorted.size() * sizeof(int));
    } else {
        h2d(in_draft, ind.data(), ind.size());
        upload_ints(draft_sorted, sorted.data(), sorted.size());
    }
    launch_rank_tables(have_affinity ? aff_dev : nullptr, draft_sorted, M, E, nmax, rank, stream);
    SMOE_CUDA(cudaGetLastError());
    ++launches;
    cur_n_draft = nmax;
}

// ------------------------------------------------------------------ profiling
void Engine::prof_begin(const char* cls, cudaEvent_t* a) {
    *a = nullptr;
    if (!profiling) return;
    SMOE_CUDA(cudaEventCreate(a));
    SMOE_CUDA(cudaEventRecord(*a, stream));
    (void)cls;
}
void Engine::prof_end(const char* cls, cudaEvent_t a, double bytes) {
    if (!profiling || !a) return;
    cudaEvent_t b;
    SMOE_CUDA(cudaEventCreate(&b));
    SMOE_CUDA(cudaEventRecord(b, stream));
    Prof& p = prof[cls];
    p.ev.emplace_back(a, b);
    p.sub.push_back(prof_pass);
    p.n += 1;
    p.bytes += bytes;
    if (prof_pass) {
        Prof& q = prof[std::string(cls) + ":" + prof_pass];
        q.n += 1;
        q.bytes += bytes;
    }
}
void Engine::prof_collect() {
    sync();
    for (auto& kv : prof) {
        for (size_t i = 0; i < kv.second.ev.size(); ++i) {
            auto& pr = kv.second.ev[i];
            float ms = 0.f;
            SMOE_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
            kv.second.ms += ms;
            if (kv.second.sub[i]) prof[kv.first + ":" + kv.second.sub[i]].ms += ms;  // inserts never invalidate kv
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
        kv.second.ev.clear();
        kv.second.sub.clear();
    }
}

// ------------------------------------------------------------------ GEMM dispatch
void Engine::gemm(const void* W, long long slot_stride, const TcOperand& amap, long long a_rows_per_slot, int Nout,
                  int Kd, const int* gcnt, const int* gslot, int G, int seg, int single_rows, int single_slot,
                  int rows_bound,
                  const void* X, const TcOperand& bmap, void* Y, int ldy, Epi epi, const char* cls, double bytes,
                  int splits, long long split_stride) {
    cudaEvent_t ev;
    prof_begin(cls, &ev);
    if (use_tc) {
        if (splits > 1 && epi != kEpiStoreF32) throw Error(kInvariant, "split-K needs the f32 store epilogue");
        TcGemmArgs a{amap, a_rows_per_slot, bmap, Nout, Kd, gcnt, gslot, G, seg, single_rows, single_slot, rows_bound,
                     Y, ldy, epi, splits, split_stride, sched + 4 * (gemm_launches++ & 1)};
        launch_gemm_tc(a, stream);
    } else {
        if (splits != 1) throw Error(kInvariant, "the CUDA-core GEMM has no split-K");
        GemmArgs a{W, slot_stride, Nout, Kd, gcnt, gslot, G, seg, single_rows, single_slot, rows_bound, X, Y, ldy, epi};
        launch_gemm_simt(a, wt, stream);
    }
    prof_end(cls, ev, bytes);
}

// Grouped expert FFN of the current MoE layer: xperm segments -> hbuf (up) -> ybuf split partials
// (down).  Group e = rows [e*T, e*T + cnt[e]) in weight slot slots[e].
void Engine::expert_ffn(int T, const int* cnt, const int* slots, const char* cls, const void* X, const TcOperand* xop,
                        void* const* peer_y) {
    const size_t ws = wt == kF32 ? 4 : 2;
    const Epi up_epi = kind == kSwiglu3 ? kEpiSwiglu : kEpiTanh;
    const long long yd_stride = (long long)E * Tmax * d;
    if (!X) {
        X = xperm;
        xop = &op_xperm;
    }
    if (!(use_tc && fuse_moe && E <= 64)) {
        gemm(up_pool, (long long)U * d, op_up, U, f, d, cnt, slots, E, T, 0, 0, T, X, *xop, hbuf, f, up_epi,
             cls, (double)U * d * ws);
        gemm(down_pool, (long long)d * f, op_down, d, d, f, cnt, slots, E, T, 0, 0, T, hbuf, op_h, ybuf, d,
             kEpiStoreF32, cls, (double)d * f * ws, s_down, yd_stride);
        return;
    }
    cudaEvent_t ev;
    prof_begin(cls, &ev);
    const unsigned slot = gemm_launches++ & 1;
    TcGemmArgs up{op_up, U, *xop, f, d, cnt, slots, E, T, 0, 0, T, hbuf, f, up_epi, 1, 0, sched + 4 * slot,
                  moe_done + 64 * slot};
    TcGemmArgs dn{op_down, d, op_h, d, f, cnt, slots, E, T, 0, 0, T, ybuf, d, kEpiStoreF32, s_down, yd_stride,
                  sched + 4 * slot, moe_done + 64 * slot};
    up.pred_groups = pred_groups;
    up.n_pred = n_pred;
    if (peer_y) {
        dn.peer_y = peer_y;
        dn.peer_eo = E / ep_world;
        dn.peer_me = ep_rank;
    }
    launch_moe_tc(up, dn, stream);
    prof_end(cls, ev, (double)(U + d) * f * ws);
}

// Event scope for the non-GEMM kernel classes (profiling runs only).
struct ProfScope {
    Engine& e;
    const char* cls;
    cudaEvent_t ev;
    ProfScope(Engine& eng, const char* c) : e(eng), cls(c) { e.prof_begin(c, &ev); }
    ~ProfScope() { e.prof_end(cls, ev, 0); }
};

// ------------------------------------------------------------------ the batched forward pass
// One pass over T rows (model.cpp:192-263 applied to every row at once).
void Engine::pass(int T, const int* rseq, const int* rextra, int extra_uniform, bool restricted, int use_aff,
                  int log_slot) {
    if (T <= 0) return;
    NvtxRange nv(restricted ? "smoe draft pass" : "smoe pass");
    if (T > Tmax) throw Error(kConfig, "engine: rows per pass exceed max_batch*(max_gamma+1)");
    struct PassKind {
        const char*& slot;
        PassKind(const char*& s, bool restricted) : slot(s) { slot = restricted ? "draft" : "verify"; }
        ~PassKind() { slot = nullptr; }
    } pass_kind(prof_pass, restricted);
    if (ep_world > 1) return pass_ep(T, rseq, rextra, extra_uniform, restricted, use_aff, log_slot);
    const size_t ws = wt == kF32 ? 4 : 2;
    const long long pm_stride = (long long)Tmax * d, yd_stride = (long long)E * Tmax * d;
    if (M > 0) SMOE_CUDA(cudaMemsetAsync(grp_cnt, 0, sizeof(int) * (size_t)M * E, stream));  // dispatch counters
    // K1+K2: x0 and the first rms (attention models: the row's own token embedding)
    if (attn())
        launch_x0_tok_rms(emb64, seq_len, last_tok, drafts, stride, rseq, rextra, extra_uniform,
                          prefill_rows ? pre_tok : nullptr, prefill_rows ? pre_pos : nullptr, T, d, x, row_plen,
                          row_pos, xa, wt, stream);
    else
        launch_x0_rms(emb64, seq_sum, seq_len, drafts, stride, rseq, rextra, extra_uniform, T, d, x, row_plen, xa, wt,
                      stream);
    const double wbytes_dd = (double)d * d * ws;
    const double ebytes_up = (double)U * d * ws, ebytes_dn = (double)d * f * ws;
    const Epi up_epi = kind == kSwiglu3 ? kEpiSwiglu : kEpiTanh;
    for (int l = 0; l < L; ++l) {
        // K3: a = Mix rms(x) (or attention's Wo o) as split-K partials; the residual add happens in the next kernel
        if (attn())
            attn_layer(l, T, rseq);
        else
            gemm(mix, (long long)d * d, op_mix, d, d, d, nullptr, nullptr, 1, 0, T, l, T, xa, op_xa, pmix, d,
                 kEpiStoreF32, "dense_gemm", wbytes_dd, s_mix, pm_stride);
        const int mo = moe_ord[l];
        if (mo >= 0) {
            int* rl = raw_log + ((size_t)log_slot * M + mo) * Tmax * K;
            int* fl = fin_log + ((size_t)log_slot * M + mo) * Tmax * K;
            int* cnt = grp_cnt + (size_t)mo * E;
            GateArgs g{x, pmix, s_mix, pm_stride, T, d, E, K, gate_w + (size_t)mo * E * d, gate_b + (size_t)mo * E,
                       xperm, cnt, pos, wt, rl, fl, wgt, restricted ? in_draft + (size_t)mo * E : nullptr,
                       draft_sorted + (size_t)mo * E, rank + (size_t)mo * E * std::max(1, cur_n_draft), cur_n_draft,
                       use_aff, mo, 0, row_plen, flags};
            const bool fetch = offload && !restricted;
            {
                ProfScope ps(*this, "gate");
                launch_gate(g, stream);  // x += a; rms; gate, top-K, remap; dispatch rows into xperm
            }
            if (fetch) store_fetch_layer(mo, cnt);  // expert store: migrate this layer's missing experts
            // weight slots: the store's table for this layer's fetch, else the resident slot map (draft
            // passes touch only pinned draft experts)
            static const bool pf_pred = [] {
                const char* v = getenv("SMOE_PF_PRED");
                return !(v && v[0] == '0');
            }();
            if (restricted && !fetch && pf_pred) {
                pred_groups = draft_sorted + (size_t)mo * E;
                n_pred = cur_n_draft;
            }
            expert_ffn(T, cnt, fetch ? group_slot : slot_of + (size_t)mo * E, "expert_gemm");
            pred_groups = nullptr;
            n_pred = 0;
            if (fetch) store_finish_layer(mo);
            {
                // K9 combine + residual + the next layer's (or the head's) rms
                ProfScope ps(*this, "combine");
                launch_combine_rms(x, ybuf, s_down, yd_stride, pos, wgt, T, K, d, 0, xa, wt, stream);
            }
        } else {
            launch_resid_rms(x, pmix, s_mix, pm_stride, T, d, xa, wt, stream);
            gemm(up_pool, (long long)U * d, op_up, U, f, d, nullptr, nullptr, 1, 0, T, dense_slot[l], T, xa, op_xa,
                 hbuf, f, up_epi, "dense_gemm", ebytes_up);
            gemm(down_pool, (long long)d * f, op_down, d, d, f, nullptr, nullptr, 1, 0, T, dense_slot[l], T, hbuf,
                 op_h, ybuf, d, kEpiStoreF32, "dense_gemm", ebytes_dn, s_down, yd_stride);
            launch_combine_rms(x, ybuf, s_down, yd_stride, nullptr, nullptr, T, 1, d, 1, xa, wt, stream);
        }
    }
    gemm(head, 0, op_head, V, V, d, nullptr, nullptr, 1, 0, T, 0, T, xa, op_xa, logits, V, kEpiStoreF32,
         "head_gemm", (double)V * d * ws);
    launch_argmax(logits, T, V, amax, flags, stream);
    SMOE_CUDA(cudaGetLastError());
    launches += 3 + (uint64_t)M * ((use_tc && fuse_moe && E <= 64) ? 4 : 5) + (uint64_t)n_dense * 5 +
                (attn() ? 3ull * L : 0ull);
    alg_dense_bytes += (double)L * (attn() ? (double)(QKVD + QD) * d : (double)d * d) * ws + (double)V * d * ws +
                       (double)n_dense * (U + d) * (double)f * ws;
}

// ------------------------------------------------------------------ real attention (attn.cu)
// One layer's attention for the T rows of a pass: QKV projection (split-K partials), RoPE + k/v into the
// sequences' cache pages + attention (k_qkv_rope, k_attn), Wo projection into the Mix's partial buffer.
void Engine::attn_layer(int l, int T, const int* rseq) {
    const size_t ws = wt == kF32 ? 4 : 2;
    gemm(wqkv, (long long)QKVD * d, op_wqkv, QKVD, QKVD, d, nullptr, nullptr, 1, 0, T, l, T, xa, op_xa, pqkv, QKVD,
         kEpiStoreF32, "dense_gemm", (double)QKVD * d * ws, s_qkv, (long long)Tmax * QKVD);
    {
        ProfScope ps(*this, "attention");
        AttnArgs a{pqkv, s_qkv, (long long)Tmax * QKVD, T, Hq, Hkv, hd, rope, rseq, row_pos, ptab, maxp, l, L,
                   qbuf, kv, wt, maxp * kKvPage, attn_o};
        launch_attention(a, stream);
    }
    gemm(wo, (long long)d * QD, op_wo, d, d, QD, nullptr, nullptr, 1, 0, T, l, T, attn_o, op_ao, pmix, d,
         kEpiStoreF32, "dense_gemm", (double)d * QD * ws, s_mix, (long long)Tmax * d);
}

// Pages for positions [0, len + Gmax] of sequence b (the rows of the next draft / verify pass), the
// rest returned to the pool -- the cache of a rolled-back sequence shrinks with its committed length.
void Engine::kv_fit(int b) {
    const int need = (h_seq_len[b] + Gmax + kKvPage) / kKvPage;
    if (need > maxp) throw Error(kConfig, "attention: sequence longer than max_seq_len");
    auto& pg = kv_pages[b];
    if ((int)pg.size() == need) return;  // the table row is current (pages change every kKvPage tokens)
    while ((int)pg.size() > need) {
        kv_free.push_back(pg.back());
        pg.pop_back();
    }
    while ((int)pg.size() < need) {
        if (kv_free.empty()) throw Error(kInvariant, "attention: KV page pool exhausted");
        pg.push_back(kv_free.back());
        kv_free.pop_back();
    }
    std::vector<int> row(maxp, 0);
    std::copy(pg.begin(), pg.end(), row.begin());
    upload_ints(ptab + (size_t)b * maxp, row.data(), row.size());
}

void Engine::kv_advance(const std::vector<int>& seqs, const std::vector<int>& takes) {
    if (!attn()) return;
    for (size_t i = 0; i < seqs.size(); ++i) {
        h_seq_len[seqs[i]] += takes[i];
        kv_fit(seqs[i]);
    }
}

// The prompts' k/v: positions 0..len-2 of every sequence (the last prompt token is the next pass's input),
// as unrestricted passes of explicit (token, position) rows, position-major in chunks of Tmax rows so
// every row's earlier positions are in the cache before its attention runs.
void Engine::prefill(const std::vector<std::vector<int>>& prompts) {
    std::vector<int> rs, tk, ps;
    size_t longest = 0;
    for (auto& p : prompts) longest = std::max(longest, p.size());
    for (size_t p = 0; p + 1 < longest; ++p)
        for (size_t b = 0; b < prompts.size(); ++b)
            if (p + 1 < prompts[b].size()) {
                rs.push_back((int)b);
                tk.push_back(prompts[b][p]);
                ps.push_back((int)p);
            }
    const uint64_t hb = h2d_bytes;  // expert fetches of the prefill are setup, not ledger traffic
    const double hm = h2d_ms;
    prefill_rows = true;
    for (size_t r0 = 0; r0 < rs.size(); r0 += (size_t)Tmax) {
        const int n = (int)std::min((size_t)Tmax, rs.size() - r0);
        upload_ints(row_seq, rs.data() + r0, n);
        upload_ints(pre_tok, tk.data() + r0, n);
        upload_ints(pre_pos, ps.data() + r0, n);
        try {
            pass(n, row_seq, nullptr, 0, false, 0, 0);
        } catch (...) {
            prefill_rows = false;
            throw;
        }
    }
    prefill_rows = false;
    sync();
    if (offload) {
        collect_h2d();
        h2d_bytes = hb;
        h2d_ms = hm;
    }
}

// Peer tables for the fused exchange: every rank's xrecv, rcnt, yret and flag array, addressable from
// this rank (CUDA IPC under NCCL, shared pointers under the loopback group).
void Engine::ep_setup_peers() {
    if (ep_world < 2 || !comm || ep_peers_ready) return;
    ep_peers_ready = true;
    void* mine[4] = {xrecv, rcnt, yret, ep_flags};
    std::vector<void*> all;
    comm->share_buffers(mine, 4, all, ep_ipc_opened);
    std::vector<void*> tab(4 * (size_t)ep_world);
    for (int r = 0; r < ep_world; ++r)
        for (int i = 0; i < 4; ++i) tab[(size_t)i * ep_world + r] = all[(size_t)r * 4 + i];
    h2d(ep_peer, tab.data(), sizeof(void*) * tab.size());
    sync();
}

// Expert-parallel pass (ep.h): this rank runs rows [r0, r0 + Tl) of the pass (contiguous blocks of
// seg = ceil(T/G)) through the dense path, gate, head and argmax; per MoE layer its routed rows go to
// the expert owners and come back finished through two all-to-alls; the pass's argmax tokens and
// routing logs are all-gathered, so every rank ends the pass with the same host-visible state as G = 1.
// Every rank issues the same collectives in the same order (a rank with no rows sends empty segments).
void Engine::pass_ep(int T, const int* rseq, const int* rextra, int extra_uniform, bool restricted, int use_aff,
                     int log_slot) {
    if (!comm) throw Error(kInvariant, "expert parallelism: no transport attached");
    if (ep_p2p) ep_setup_peers();  // collective: the first pass of every rank exchanges the peer tables
    const int G = ep_world, eo = E / G;
    const int seg = (T + G - 1) / G, r0 = ep_rank * seg, Tl = std::max(0, std::min(seg, T - r0));
    const size_t ws = wt == kF32 ? 4 : 2;
    const long long pm_stride = (long long)Tmax * d, yd_stride = (long long)E * Tmax * d;
    if (M > 0) SMOE_CUDA(cudaMemsetAsync(grp_cnt, 0, sizeof(int) * (size_t)M * E, stream));
    if (Tl > 0)
        launch_x0_rms(emb64, seq_sum, seq_len, drafts, stride, rseq + r0, rextra ? rextra + r0 : nullptr, extra_uniform,
                      Tl, d, x, row_plen, xa, wt, stream);
    const Epi up_epi = kind == kSwiglu3 ? kEpiSwiglu : kEpiTanh;
    for (int l = 0; l < L; ++l) {
        if (Tl > 0)
            gemm(mix, (long long)d * d, op_mix, d, d, d, nullptr, nullptr, 1, 0, Tl, l, Tl, xa, op_xa, pmix, d,
                 kEpiStoreF32, "dense_gemm", (double)d * d * ws, s_mix, pm_stride);
        const int mo = moe_ord[l];
        if (mo < 0) {  // dense layer: local rows only
            if (Tl > 0) {
                launch_resid_rms(x, pmix, s_mix, pm_stride, Tl, d, xa, wt, stream);
                gemm(up_pool, (long long)U * d, op_up, U, f, d, nullptr, nullptr, 1, 0, Tl, dense_slot[l], Tl, xa,
                     op_xa, hbuf, f, up_epi, "dense_gemm", (double)U * d * ws);
                gemm(down_pool, (long long)d * f, op_down, d, d, f, nullptr, nullptr, 1, 0, Tl, dense_slot[l], Tl, hbuf,
                     op_h, ybuf, d, kEpiStoreF32, "dense_gemm", (double)d * f * ws, s_down, yd_stride);
                launch_combine_rms(x, ybuf, s_down, yd_stride, nullptr, nullptr, Tl, 1, d, 1, xa, wt, stream);
            }
            continue;
        }
        int* rl = raw_log + ((size_t)log_slot * M + mo) * Tmax * K;
        int* fl = fin_log + ((size_t)log_slot * M + mo) * Tmax * K;
        int* cnt = grp_cnt + (size_t)mo * E;
        const bool fetch = offload && !restricted;
        if (Tl > 0) {
            GateArgs g{x, pmix, s_mix, pm_stride, Tl, d, E, K, gate_w + (size_t)mo * E * d, gate_b + (size_t)mo * E,
                       xperm, cnt, pos, wt, rl, fl, wgt, restricted ? in_draft + (size_t)mo * E : nullptr,
                       draft_sorted + (size_t)mo * E, rank + (size_t)mo * E * std::max(1, cur_n_draft), cur_n_draft,
                       use_aff, mo, seg, row_plen, flags};
            if (ep_p2p) {
                g.peer_x = const_cast<void* const*>(ep_peer);
                g.ep_eo = eo;
                g.ep_me = ep_rank;
            }
            ProfScope ps(*this, "gate");
            launch_gate(g, stream);  // rows of expert e land in xperm rows [e*seg, e*seg + cnt[e])
        }
        if (ep_p2p) {
            // fused exchange over peer memory: the gate has stored this rank's routed rows into the owners'
            // xrecv; counts + flag -> owners; the owners' down-projection epilogues store the finished
            // split partials into the senders' yret; done flags -> senders; the combine reads yret
            const int seq = ++ep_seq;
            void* const* peer = const_cast<void* const*>(ep_peer);
            launch_ep_signal(cnt, E, eo, ep_rank, G, peer + G, peer + 3 * G, 0, seq, stream);
            comm->fence(stream);
            launch_ep_wait(ep_flags, G, 0, seq, stream);
            if (fetch) store_fetch_layer_ep(mo, cnt);  // needed ∩ owned, over this rank's PCIe link
            expert_ffn(seg, rcnt, ep_gslot + (size_t)mo * E, "expert_gemm", xrecv, &op_xrecv, peer + 2 * G);
            if (fetch) store_finish_layer(mo);
            launch_ep_signal(nullptr, E, eo, ep_rank, G, peer + G, peer + 3 * G, 1, seq, stream);
            comm->fence(stream);
            launch_ep_wait(ep_flags, G, 1, seq, stream);
            if (Tl > 0) {
                ProfScope ps(*this, "combine");
                launch_combine_rms(x, yret, s_down, yd_stride, pos, wgt, Tl, K, d, 0, xa, wt, stream);
            }
            continue;
        }
        // dispatch: chunk r of the expert-major segments = rank r's experts
        comm->alltoall(xperm, xrecv, (size_t)eo * seg * d * ws, stream);
        comm->alltoall(cnt, rcnt, sizeof(int) * eo, stream);
        if (fetch) store_fetch_layer_ep(mo, cnt);
        // owner: one grouped FFN over the (source rank, local expert) groups, finished rows summed over the
        // split-K partials exactly as the combine would, then returned into the senders' [E][seg] layout
        expert_ffn(seg, rcnt, ep_gslot + (size_t)mo * E, "expert_gemm", xrecv, &op_xrecv);
        if (fetch) store_finish_layer(mo);
        launch_ep_sum_partials(ybuf, s_down, yd_stride, rcnt, E, seg, d, ysend, stream);
        comm->alltoall(ysend, yret, (size_t)eo * seg * d * sizeof(float), stream);
        if (Tl > 0) {
            ProfScope ps(*this, "combine");
            launch_combine_rms(x, yret, 1, 0, pos, wgt, Tl, K, d, 0, xa, wt, stream);
        }
    }
    if (Tl > 0) {
        gemm(head, 0, op_head, V, V, d, nullptr, nullptr, 1, 0, Tl, 0, Tl, xa, op_xa, ep_gather_logits ? logits_loc : logits,
             V, kEpiStoreF32, "head_gemm", (double)V * d * ws);
        launch_argmax(ep_gather_logits ? logits_loc : logits, Tl, V, amax_loc, flags, stream);
    }
    // replicate the pass outputs: argmax tokens, routing logs of this log slot, optionally the logits
    comm->allgather(amax_loc, amax, sizeof(int) * seg, stream);
    if (M > 0) {
        int* pk = ep_logs;
        int* gathered = ep_logs + (size_t)2 * M * Tmax * K;
        launch_ep_pack_logs(raw_log + (size_t)log_slot * M * Tmax * K, fin_log + (size_t)log_slot * M * Tmax * K, M,
                            Tmax, K, Tl, seg, pk, stream);
        comm->allgather(pk, gathered, sizeof(int) * 2 * M * seg * K, stream);
        launch_ep_unpack_logs(gathered, G, M, Tmax, K, T, seg, raw_log + (size_t)log_slot * M * Tmax * K,
                              fin_log + (size_t)log_slot * M * Tmax * K, stream);
    }
    if (ep_gather_logits) comm->allgather(logits_loc, logits, sizeof(float) * seg * V, stream);
    SMOE_CUDA(cudaGetLastError());
    launches += 2 + (uint64_t)M * 5 + (uint64_t)n_dense * 5 + 2;
    alg_dense_bytes += (double)L * d * d * ws + (double)V * d * ws + (double)n_dense * (U + d) * (double)f * ws;
}

// Kernel timed alone: T tokens routed round-robin over all E experts of MoE layer 0 (every expert
// touched), up-projection then down-projection, `iters` times each with CUDA events.
void Engine::bench_expert_gemm(int T, int iters, double* up_ms, double* down_ms, double* bytes_up, double* bytes_down) {
    if (offload || ep_world > 1) throw Error(kConfig, "bench_expert_gemm: single-GPU HBM-resident engines only");
    if (T > Tmax) throw Error(kConfig, "bench_expert_gemm: T exceeds max_batch*(max_gamma+1)");
    // round-robin routing: expert e gets the picks (t,k) with (t*K+k) % E == e
    std::vector<int> cnt(E, 0);
    for (int j = 0; j < T * K; ++j) ++cnt[j % E];
    upload_ints(grp_cnt, cnt.data(), E);
    const long long yd_stride = (long long)E * Tmax * d;
    const Epi up_epi = kind == kSwiglu3 ? kEpiSwiglu : kEpiTanh;
    cudaEvent_t a, b, c;
    SMOE_CUDA(cudaEventCreate(&a)); SMOE_CUDA(cudaEventCreate(&b)); SMOE_CUDA(cudaEventCreate(&c));
    float t_up = 0, t_dn = 0;
    for (int pass = 0; pass < 2; ++pass) {  // pass 0 = warm-up
        SMOE_CUDA(cudaEventRecord(a, stream));
        for (int i = 0; i < iters; ++i)
            gemm(up_pool, (long long)U * d, op_up, U, f, d, grp_cnt, slot_of, E, T, 0, 0, T, xperm, op_xperm, hbuf, f,
                 up_epi, "bench", 0);
        SMOE_CUDA(cudaEventRecord(b, stream));
        for (int i = 0; i < iters; ++i)
            gemm(down_pool, (long long)d * f, op_down, d, d, f, grp_cnt, slot_of, E, T, 0, 0, T, hbuf, op_h, ybuf, d,
                 kEpiStoreF32, "bench", 0, s_down, yd_stride);
        SMOE_CUDA(cudaEventRecord(c, stream));
        SMOE_CUDA(cudaEventSynchronize(c));
        SMOE_CUDA(cudaEventElapsedTime(&t_up, a, b));
        SMOE_CUDA(cudaEventElapsedTime(&t_dn, b, c));
    }
    cudaEventDestroy(a); cudaEventDestroy(b); cudaEventDestroy(c);
    const size_t ws = wt == kF32 ? 4 : 2;
    const int touched = std::min(E, T * K);
    *up_ms = t_up / iters;
    *down_ms = t_dn / iters;
    *bytes_up = (double)touched * U * d * ws + (double)T * K * (d + f) * ws;
    *bytes_down = (double)touched * d * f * ws + (double)T * K * (f * ws + (double)d * 4 * s_down);
}

void Engine::reset_sequences(const std::vector<std::vector<int>>& prompts) {
    const int B = (int)prompts.size();
    if (B > Bmax) throw Error(kConfig, "engine: batch exceeds max_batch");
    SMOE_CUDA(cudaMemsetAsync(seq_sum, 0, sizeof(double) * Bmax * d, stream));
    SMOE_CUDA(cudaMemsetAsync(seq_len, 0, sizeof(int) * Bmax, stream));
    size_t plen = 0;
    for (auto& p : prompts) plen = std::max(plen, p.size());
    std::vector<int> toks((size_t)B * plen, 0), take(B), sq(B);
    for (int b = 0; b < B; ++b) {
        for (int v : prompts[b])
            if (v < 0 || v >= V) throw Error(kInvariant, "forward: token out of range");
        std::copy(prompts[b].begin(), prompts[b].end(), toks.begin() + (size_t)b * plen);
        take[b] = (int)prompts[b].size();
        sq[b] = b;
    }
    int* dtoks = dalloc<int>(toks.size());
    upload_ints(dtoks, toks.data(), toks.size());
    upload_ints(commit_take, take.data(), B);
    upload_ints(seqs, sq.data(), B);
    launch_commit(seq_sum, seq_len, emb64, seqs, dtoks, (int)plen, commit_take, B, d, stream, last_tok);
    sync();
    SMOE_CUDA(cudaFree(dtoks));
    if (attn()) {  // a fresh paged cache holding the prompts' k/v
        for (int b = 0; b < Bmax; ++b) {
            for (int pg : kv_pages[b]) kv_free.push_back(pg);
            kv_pages[b].clear();
            h_seq_len[b] = b < B ? (int)prompts[b].size() : 0;
        }
        for (int b = 0; b < B; ++b) kv_fit(b);
        prefill(prompts);
    }
}

void Engine::forward_one(const std::vector<int>& prefix, const int* restricted, int n_draft, int use_aff,
                         float* logits_out, int* raw_out, int* fin_out) {
    if (prefix.empty()) throw Error(kInvariant, "forward: empty prefix");
    if (use_aff && !have_affinity) throw Error(kInvariant, "forward: affinity table required but missing");
    if (restricted) {
        std::vector<std::vector<int>> sets(M);
        for (int m = 0; m < M; ++m) sets[m].assign(restricted + (size_t)m * n_draft, restricted + (size_t)(m + 1) * n_draft);
        set_draft_sets(sets, n_draft);
        store_pin_sets(sets);
    } else if (offload) {
        store_reset();
    }
    reset_sequences({prefix});
    int zero = 0;
    upload_ints(row_seq, &zero, 1);
    ep_gather_logits = true;  // under expert parallelism row 0 lives on rank 0 only
    pass(1, row_seq, nullptr, 0, restricted != nullptr, use_aff, 0);
    ep_gather_logits = false;
    sync();
    check_flags();
    if (logits_out) SMOE_CUDA(cudaMemcpy(logits_out, logits, sizeof(float) * V, cudaMemcpyDeviceToHost));
    for (int m = 0; m < M; ++m) {
        if (raw_out) SMOE_CUDA(cudaMemcpy(raw_out + (size_t)m * K, raw_log + (size_t)m * Tmax * K, sizeof(int) * K,
                                          cudaMemcpyDeviceToHost));
        if (fin_out) SMOE_CUDA(cudaMemcpy(fin_out + (size_t)m * K, fin_log + (size_t)m * Tmax * K, sizeof(int) * K,
                                          cudaMemcpyDeviceToHost));
    }
}

}  // namespace smoe
