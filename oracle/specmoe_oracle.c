/* specmoe_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker, never the product.
 *
 * A plain-C, float64, single-threaded restatement of the reference's self-assisted
 * speculative-decoding path (arxiv/paper_2604_10152, /root/reference/proj/core).  Every
 * function cites the reference file:line it follows; arithmetic is performed in the same
 * order as the reference so that logits agree with oracle/_ref bit for bit (pinned by
 * tests/test_oracle.py against the compiled reference and tests/golden/).
 *
 * Extension (parity unpinned by the reference): expert_kind = 1 (swiglu3) replaces the
 * reference's 2-matrix tanh expert with down^T (silu(w1^T x) * (w3^T x)), weights drawn
 * per expert in the order w1, w3, w2.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
 * may load the library built from this file.
 */
#define _POSIX_C_SOURCE 200809L
#include "oracle_abi.h"

#include <math.h>
#include <pthread.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ errors & arena */
/* ConfigError -> 1, InvariantError -> 2 (common.hpp:12-21). */
static __thread jmp_buf* g_jmp;
static __thread char g_msg[256];
static __thread int g_code;

static void fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_msg, sizeof g_msg, fmt, ap);
    va_end(ap);
    g_code = code;
    longjmp(*g_jmp, 1);
}

typedef struct blk { struct blk* next; } blk;
static __thread blk* g_arena;
static void* amalloc(size_t n) {
    blk* b = (blk*)calloc(1, sizeof(blk) + n + 16);
    if (!b) fail(2, "oracle: out of memory");
    b->next = g_arena;
    g_arena = b;
    return (char*)(b + 1);
}
static void arena_release(blk* upto) {
    while (g_arena && g_arena != upto) {
        blk* n = g_arena->next;
        free(g_arena);
        g_arena = n;
    }
}
#define ENTER(errbuf, errlen, failret)            \
    jmp_buf jb__;                                 \
    jmp_buf* prev__ = g_jmp;                      \
    blk* mark__ = g_arena;                        \
    g_jmp = &jb__;                                \
    if (setjmp(jb__)) {                           \
        arena_release(mark__);                    \
        g_jmp = prev__;                           \
        if (errbuf && errlen > 0) snprintf(errbuf, errlen, "%s", g_msg); \
        return failret;                           \
    }
#define LEAVE()               \
    do {                      \
        arena_release(mark__); \
        g_jmp = prev__;       \
    } while (0)

/* ------------------------------------------------------------------ RNG (common.hpp:23-55) */
typedef struct { uint64_t s[312]; int i; } mt64;
static void mt_seed(mt64* r, uint64_t seed) { /* std::mt19937_64 seeding, fixed by the C++ standard */
    r->s[0] = seed;
    for (int k = 1; k < 312; ++k) r->s[k] = 6364136223846793005ULL * (r->s[k - 1] ^ (r->s[k - 1] >> 62)) + (uint64_t)k;
    r->i = 312;
}
static uint64_t mt_next(mt64* r) {
    if (r->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            uint64_t y = (r->s[k] & 0xFFFFFFFF80000000ULL) | (r->s[(k + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = r->s[(k + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->s[k] = v;
        }
        r->i = 0;
    }
    uint64_t x = r->s[r->i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}
static uint64_t splitmix(uint64_t x) { /* common.hpp:27-32 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static uint64_t substream2(uint64_t seed, uint64_t t0, uint64_t t1) { /* common.hpp:35-37 */
    return splitmix(seed ^ splitmix(t0 ^ splitmix(t1)));
}
static double unif(mt64* r) { return (double)(mt_next(r) >> 11) * 0x1.0p-53; } /* common.hpp:40-42 */
static double gauss(mt64* r) {                                                  /* common.hpp:46-55 */
    for (;;) {
        double u = 2.0 * unif(r) - 1.0, v = 2.0 * unif(r) - 1.0, s = u * u + v * v;
        if (s > 0.0 && s < 1.0) return u * sqrt(-2.0 * log(s) / s);
    }
}

/* ------------------------------------------------------------------ model (model.cpp) */
typedef struct {
    double *up, *down, *w3; /* tanh2: up d*f, down f*d.  swiglu3: up=w1, w3, down=w2 */
} oexpert;
typedef struct {
    int is_moe;
    double *mix, *gate, *bias; /* mix d*d, gate d*E, bias E */
    double *wq, *wk, *wv, *wo; /* attention: [Hq*hd][d], [Hkv*hd][d] x2, [d][Hq*hd] (y = W x) */
    oexpert* experts;          /* E */
    oexpert ffn;
} olayer;
typedef struct {
    int L, E, K, d, f, V, M, kind;
    int Hq, Hkv, hd; /* attention extension (Hq = 0: the reference's surrogate) */
    double theta;
    double skew;
    uint64_t seed;
    uint8_t* mask;
    int* moe_index; /* ordinal -> raw layer */
    double *emb, *head;
    olayer* layers;
} omodel;

static double* gfill(size_t n, double sd, mt64* r) { /* model.cpp:64-67 (fill_gaussian) */
    double* p = (double*)malloc(n * sizeof(double));
    if (!p) return NULL;
    for (size_t i = 0; i < n; ++i) p[i] = sd * gauss(r);
    return p;
}

static void free_model(omodel* m) {
    if (!m) return;
    free(m->emb);
    free(m->head);
    if (m->layers)
        for (int l = 0; l < m->L; ++l) {
            olayer* ly = &m->layers[l];
            free(ly->mix); free(ly->gate); free(ly->bias);
            free(ly->wq); free(ly->wk); free(ly->wv); free(ly->wo);
            if (ly->experts)
                for (int e = 0; e < m->E; ++e) { free(ly->experts[e].up); free(ly->experts[e].down); free(ly->experts[e].w3); }
            free(ly->experts);
            free(ly->ffn.up); free(ly->ffn.down); free(ly->ffn.w3);
        }
    free(m->layers); free(m->mask); free(m->moe_index);
    free(m);
}

static void fill_expert(oexpert* x, int kind, int d, int f, double sd, mt64* r) {
    if (kind == 0) { /* model.cpp:131-135: up then down */
        x->up = gfill((size_t)d * f, sd, r);
        x->down = gfill((size_t)f * d, sd, r);
    } else { /* extension: w1, w3, w2 */
        x->up = gfill((size_t)d * f, sd, r);
        x->w3 = gfill((size_t)d * f, sd, r);
        x->down = gfill((size_t)f * d, sd, r);
    }
}

void* om_build_model(const om_spec* sp, char* err, int errlen) { /* model.cpp:106-143, validate 68-87 */
    const char* bad = NULL;
    if (sp->experts < 1) bad = "model: experts_per_block >= 1 violated";
    else if (sp->top_k < 1 || sp->top_k > sp->experts) bad = "model: 1 <= top_k <= experts_per_block violated";
    else if (sp->vocab < 2) bad = "model: vocab_size >= 2 violated";
    else if (sp->hidden < 1) bad = "model: hidden_dim >= 1 violated";
    else if (sp->ffn < 1) bad = "model: ffn_dim >= 1 violated";
    else if (sp->num_layers < 1) bad = "model: num_layers >= 1 violated";
    else if (sp->gate_skew < 0.0) bad = "model: gate_skew >= 0 violated";
    else if (sp->attn_heads > 0 && (sp->kv_heads < 1 || sp->attn_heads % sp->kv_heads || sp->head_dim < 2 ||
                                    sp->head_dim % 2 || sp->rope_theta <= 0.0))
        bad = "model: attention needs kv_heads | attn_heads, an even head_dim and rope_theta > 0";
    int any = 0;
    if (!bad) {
        for (int l = 0; l < sp->num_layers; ++l) any |= sp->moe_mask ? sp->moe_mask[l] != 0 : 1;
        if (!any) bad = "model: at least one layer must be an MoE block";
    }
    if (bad) {
        if (err) snprintf(err, errlen, "%s", bad);
        return NULL;
    }
    omodel* m = (omodel*)calloc(1, sizeof(omodel));
    m->L = sp->num_layers; m->E = sp->experts; m->K = sp->top_k; m->d = sp->hidden; m->f = sp->ffn;
    m->V = sp->vocab; m->skew = sp->gate_skew; m->seed = sp->seed; m->kind = sp->expert_kind;
    m->Hq = sp->attn_heads; m->Hkv = sp->kv_heads; m->hd = sp->head_dim; m->theta = sp->rope_theta;
    m->mask = (uint8_t*)malloc(m->L);
    m->moe_index = (int*)malloc(sizeof(int) * m->L);
    m->M = 0;
    for (int l = 0; l < m->L; ++l) {
        m->mask[l] = sp->moe_mask ? (sp->moe_mask[l] != 0) : 1;
        if (m->mask[l]) m->moe_index[m->M++] = l;
    }
    const int d = m->d, f = m->f, E = m->E, V = m->V;
    const double sd = 1.0 / sqrt((double)d);
    mt64* r = (mt64*)malloc(sizeof(mt64));
    mt_seed(r, m->seed);
    m->emb = gfill((size_t)V * d, sd, r);
    m->layers = (olayer*)calloc((size_t)m->L, sizeof(olayer));
    for (int l = 0; l < m->L; ++l) {
        olayer* ly = &m->layers[l];
        ly->is_moe = m->mask[l];
        if (m->Hq > 0) { /* extension: the attention weights take the mix's place in the draw order */
            const size_t qd = (size_t)m->Hq * m->hd, kd = (size_t)m->Hkv * m->hd;
            ly->wq = gfill(qd * d, sd, r);
            ly->wk = gfill(kd * d, sd, r);
            ly->wv = gfill(kd * d, sd, r);
            ly->wo = gfill((size_t)d * qd, sd, r);
        } else {
            ly->mix = gfill((size_t)d * d, sd, r);
        }
        if (ly->is_moe) {
            ly->gate = gfill((size_t)d * E, sd, r);
            ly->bias = (double*)malloc(sizeof(double) * E);
            for (int e = 0; e < E; ++e) ly->bias[e] = m->skew * (1.0 - (double)e / E);
            ly->experts = (oexpert*)calloc((size_t)E, sizeof(oexpert));
            for (int e = 0; e < E; ++e) fill_expert(&ly->experts[e], m->kind, d, f, sd, r);
        } else {
            fill_expert(&ly->ffn, m->kind, d, f, sd, r);
        }
    }
    m->head = gfill((size_t)d * V, sd, r);
    free(r);
    return m;
}

void om_free_model(void* model) { free_model((omodel*)model); }

long long om_get_tensor(void* model, const char* name, int layer, int expert, double* out, long long cap) {
    omodel* m = (omodel*)model;
    const double* src = NULL;
    long long n = 0;
    const long long d = m->d, f = m->f, E = m->E, V = m->V;
    if (!strcmp(name, "embedding")) { src = m->emb; n = V * d; }
    else if (!strcmp(name, "head")) { src = m->head; n = d * V; }
    else {
        if (layer < 0 || layer >= m->L) return -1;
        olayer* ly = &m->layers[layer];
        if (!strcmp(name, "mix")) { src = ly->mix; n = ly->mix ? d * d : 0; }
        else if (!strcmp(name, "wq")) { src = ly->wq; n = (long long)m->Hq * m->hd * d; }
        else if (!strcmp(name, "wk")) { src = ly->wk; n = (long long)m->Hkv * m->hd * d; }
        else if (!strcmp(name, "wv")) { src = ly->wv; n = (long long)m->Hkv * m->hd * d; }
        else if (!strcmp(name, "wo")) { src = ly->wo; n = (long long)m->Hq * m->hd * d; }
        else if (!strcmp(name, "gate")) { src = ly->gate; n = ly->is_moe ? d * E : 0; }
        else if (!strcmp(name, "gate_bias")) { src = ly->bias; n = ly->is_moe ? E : 0; }
        else {
            oexpert* x = NULL;
            if (expert < 0) x = ly->is_moe ? NULL : &ly->ffn;
            else if (ly->is_moe && expert < E) x = &ly->experts[expert];
            if (!x) return -1;
            if (!strcmp(name, "up") || !strcmp(name, "w1")) { src = x->up; n = d * f; }
            else if (!strcmp(name, "down") || !strcmp(name, "w2")) { src = x->down; n = f * d; }
            else if (!strcmp(name, "w3")) { src = x->w3; n = x->w3 ? d * f : 0; }
        }
    }
    if (!src || n == 0) return -1;
    if (out) {
        if (cap < n) return -1;
        memcpy(out, src, sizeof(double) * (size_t)n);
    }
    return n;
}

/* model.cpp:19-26 */
static void rms(const double* x, int n, double* out) {
    double ss = 0.0;
    for (int i = 0; i < n; ++i) ss += x[i] * x[i];
    double inv = 1.0 / sqrt(ss / (double)n + 1e-12);
    for (int i = 0; i < n; ++i) out[i] = x[i] * inv;
}
/* model.cpp:29-39: y = M x */
static void mv(const double* m, const double* x, int rows, int cols, double* y) {
    for (int r = 0; r < rows; ++r) {
        double acc = 0.0;
        const double* row = m + (size_t)r * cols;
        for (int c = 0; c < cols; ++c) acc += row[c] * x[c];
        y[r] = acc;
    }
}
/* model.cpp:42-52: y = M^T x */
static void mtv(const double* m, const double* x, int rows, int cols, double* y) {
    for (int c = 0; c < cols; ++c) y[c] = 0.0;
    for (int r = 0; r < rows; ++r) {
        const double* row = m + (size_t)r * cols;
        double xv = x[r];
        for (int c = 0; c < cols; ++c) y[c] += row[c] * xv;
    }
}
/* model.cpp:54-59 (tanh2) and the swiglu3 extension */
static void expert_fwd(const omodel* m, const oexpert* x, const double* in, double* out) {
    const int d = m->d, f = m->f;
    double* h = (double*)amalloc(sizeof(double) * f);
    mtv(x->up, in, d, f, h);
    if (m->kind == 0) {
        for (int i = 0; i < f; ++i) h[i] = tanh(h[i]);
    } else {
        double* g = (double*)amalloc(sizeof(double) * f);
        mtv(x->w3, in, d, f, g);
        for (int i = 0; i < f; ++i) h[i] = h[i] / (1.0 + exp(-h[i])) * g[i];
    }
    mtv(x->down, h, f, d, out);
}

static int finite_all(const double* x, int n) {
    for (int i = 0; i < n; ++i)
        if (!isfinite(x[i])) return 0;
    return 1;
}
/* model.cpp:145-157 */
static void softmax_(const double* l, int n, double* p) {
    if (n <= 0) fail(2, "softmax: empty input");
    if (!finite_all(l, n)) fail(2, "softmax: non-finite input");
    double mx = l[0];
    for (int i = 1; i < n; ++i)
        if (l[i] > mx) mx = l[i];
    double sum = 0.0;
    for (int i = 0; i < n; ++i) { p[i] = exp(l[i] - mx); sum += p[i]; }
    for (int i = 0; i < n; ++i) p[i] /= sum;
}
/* model.cpp:159-170: stable sort descending == repeated first-max selection */
static void topk_(const double* l, int n, int k, int* out) {
    if (k > n) fail(2, "route_topk: k exceeds expert count");
    if (k < 0) fail(2, "route_topk: negative k");
    uint8_t* taken = (uint8_t*)amalloc((size_t)n);
    for (int j = 0; j < k; ++j) {
        int best = -1;
        for (int i = 0; i < n; ++i)
            if (!taken[i] && (best < 0 || l[i] > l[best])) best = i;
        taken[best] = 1;
        out[j] = best;
    }
}
/* model.cpp:172-176 */
static int greedy_(const double* l, int n) {
    if (n <= 0) fail(2, "greedy_next: empty logits");
    if (!finite_all(l, n)) fail(2, "greedy_next: non-finite logits");
    int b = 0;
    for (int i = 1; i < n; ++i)
        if (l[i] > l[b]) b = i;
    return b;
}

static int contains(const int* xs, int n, int v) {
    for (int i = 0; i < n; ++i)
        if (xs[i] == v) return 1;
    return 0;
}
/* drafting.cpp:123-138 */
static int nearest_(const double* dist_l, int E, int raw, const int* ds, int nd, const int* ex, int nex) {
    if (contains(ds, nd, raw) && !contains(ex, nex, raw)) return raw;
    int best = -1;
    double bd = 0.0;
    for (int i = 0; i < nd; ++i) {
        int c = ds[i];
        if (contains(ex, nex, c)) continue;
        double dd = dist_l[(size_t)raw * E + c];
        if (best < 0 || dd < bd || (dd == bd && c < best)) { best = c; bd = dd; }
    }
    if (best < 0) fail(2, "nearest_draft_expert: empty candidate set");
    return best;
}
static int cmp_int(const void* a, const void* b) { return (*(const int*)a > *(const int*)b) - (*(const int*)a < *(const int*)b); }
/* drafting.cpp:140-151 */
static int surrogate_(int layer, int raw, size_t plen, const int* ds, int nd, const int* ex, int nex) {
    if (contains(ds, nd, raw) && !contains(ex, nex, raw)) return raw;
    int* c = (int*)amalloc(sizeof(int) * (size_t)(nd + 1));
    int nc = 0;
    for (int i = 0; i < nd; ++i)
        if (!contains(ex, nex, ds[i])) c[nc++] = ds[i];
    if (nc == 0) fail(2, "surrogate_draft_expert: empty candidate set");
    qsort(c, (size_t)nc, sizeof(int), cmp_int);
    uint64_t h = substream2(0x5eed5eedULL, ((uint64_t)layer << 32) | (uint32_t)raw, (uint64_t)plen);
    return c[h % (uint64_t)nc];
}

typedef struct { double* dist; int E, M; } oaff; /* drafting.hpp:14-19 */

/* model.cpp:192-263.  restricted: [M*nd] or NULL. */
static __thread double* g_gate_dump;  /* om_forward_gates: per-layer gate logits destination */
static __thread int g_committed;      /* attention extension: committed prefix length of a draft forward */

/* The MoE half of a layer (model.cpp:226-258): xf = rms(x); x += sum_k p[raw_k] expert_final_k(xf). */
static void moe_half(const omodel* m, const olayer* ly, int mo, double* x, int plen, const int* restricted, int nd,
                     const oaff* aff, int last, int* raw_out, int* fin_out);

/* Real-attention extension (no reference counterpart): positions 0..n-1 are run in order,
 * each attending causally to every earlier position's K/V of the same layer.  Positions < nc-1 (the
 * committed prefix except its last token) use the target model; with draft sets, positions >= nc-1 use
 * the restricted model (their K/V are the draft model's) -- the engine's KV cache after a phase's draft
 * passes.  Without draft sets every position is the target's.  RoPE: rotate-half, angle = p * theta^(-2j/hd).
 * Routing outputs and logits are those of the last position. */
static void fwd_attn(const omodel* m, const int* prefix, int n, const int* restricted, int nd, const oaff* aff,
                     int nc, double* logits, int* raw_out, int* fin_out) {
    const int d = m->d, Hq = m->Hq, Hkv = m->Hkv, hd = m->hd, G = Hq / Hkv;
    const size_t qd = (size_t)Hq * hd, kd = (size_t)Hkv * hd;
    blk* mark = g_arena;
    double* kc = (double*)amalloc(sizeof(double) * (size_t)m->L * n * kd); /* [L][n][kd] */
    double* vc = (double*)amalloc(sizeof(double) * (size_t)m->L * n * kd);
    double* x = (double*)amalloc(sizeof(double) * d);
    double* xn = (double*)amalloc(sizeof(double) * d);
    double* q = (double*)amalloc(sizeof(double) * qd);
    double* o = (double*)amalloc(sizeof(double) * qd);
    double* a = (double*)amalloc(sizeof(double) * d);
    double* sc = (double*)amalloc(sizeof(double) * n);
    const double inv_sqrt = 1.0 / sqrt((double)hd);
    for (int p = 0; p < n; ++p) {
        const int last = p == n - 1;
        const int draft = restricted && p >= nc - 1;
        const double* e = m->emb + (size_t)prefix[p] * d;
        for (int j = 0; j < d; ++j) x[j] = e[j];
        int mo = 0;
        for (int l = 0; l < m->L; ++l) {
            const olayer* ly = &m->layers[l];
            double* kp = kc + ((size_t)l * n + p) * kd;
            double* vp = vc + ((size_t)l * n + p) * kd;
            rms(x, d, xn);
            mv(ly->wq, xn, (int)qd, d, q);
            mv(ly->wk, xn, (int)kd, d, kp);
            mv(ly->wv, xn, (int)kd, d, vp);
            for (int h = 0; h < Hq + Hkv; ++h) { /* RoPE on every query and key head */
                double* v = h < Hq ? q + (size_t)h * hd : kp + (size_t)(h - Hq) * hd;
                for (int j = 0; j < hd / 2; ++j) {
                    const double ang = (double)p * pow(m->theta, -2.0 * j / hd);
                    const double c = cos(ang), s = sin(ang), x0 = v[j], x1 = v[j + hd / 2];
                    v[j] = x0 * c - x1 * s;
                    v[j + hd / 2] = x1 * c + x0 * s;
                }
            }
            for (int h = 0; h < Hq; ++h) { /* softmax(q k^T / sqrt(hd)) v over positions 0..p */
                const double* qh = q + (size_t)h * hd;
                const int kh = h / G;
                double mx = -INFINITY;
                for (int t = 0; t <= p; ++t) {
                    const double* kt = kc + ((size_t)l * n + t) * kd + (size_t)kh * hd;
                    double s = 0.0;
                    for (int j = 0; j < hd; ++j) s += qh[j] * kt[j];
                    sc[t] = s * inv_sqrt;
                    if (sc[t] > mx) mx = sc[t];
                }
                double sum = 0.0;
                for (int t = 0; t <= p; ++t) { sc[t] = exp(sc[t] - mx); sum += sc[t]; }
                double* oh = o + (size_t)h * hd;
                for (int j = 0; j < hd; ++j) oh[j] = 0.0;
                for (int t = 0; t <= p; ++t) {
                    const double* vt = vc + ((size_t)l * n + t) * kd + (size_t)kh * hd;
                    const double w = sc[t] / sum;
                    for (int j = 0; j < hd; ++j) oh[j] += w * vt[j];
                }
            }
            mv(ly->wo, o, d, (int)qd, a);
            for (int j = 0; j < d; ++j) x[j] += a[j];
            if (ly->is_moe) {
                moe_half(m, ly, mo, x, p + 1, draft ? restricted : NULL, nd, aff, last, last ? raw_out : NULL,
                         last ? fin_out : NULL);
                ++mo;
            } else {
                moe_half(m, ly, -1, x, p + 1, NULL, 0, NULL, 0, NULL, NULL);
            }
        }
        if (last) {
            rms(x, d, xn);
            mtv(m->head, xn, d, m->V, logits);
        }
    }
    arena_release(mark);
}

static void fwd(const omodel* m, const int* prefix, int n, const int* restricted, int nd, const oaff* aff,
                double* logits, int* raw_out, int* fin_out) {
    const int d = m->d, E = m->E, K = m->K;
    if (n <= 0) fail(2, "forward: empty prefix");
    for (int i = 0; i < n; ++i)
        if (prefix[i] < 0 || prefix[i] >= m->V) fail(2, "forward: token out of range");
    if (restricted && nd < K) fail(2, "forward: restricted set smaller than top_k");
    if (m->Hq > 0) {
        fwd_attn(m, prefix, n, restricted, nd, aff, g_committed > 0 ? g_committed : n, logits, raw_out, fin_out);
        return;
    }
    blk* mark = g_arena;
    double* x = (double*)amalloc(sizeof(double) * d);
    double* xn = (double*)amalloc(sizeof(double) * d);
    double* a = (double*)amalloc(sizeof(double) * d);
    double* y = (double*)amalloc(sizeof(double) * d);
    double* eo = (double*)amalloc(sizeof(double) * d);
    double* gl = (double*)amalloc(sizeof(double) * E);
    double* pr = (double*)amalloc(sizeof(double) * E);
    int* raw = (int*)amalloc(sizeof(int) * K);
    int* chosen = (int*)amalloc(sizeof(int) * K);
    for (int i = 0; i < n; ++i) {
        const double* e = m->emb + (size_t)prefix[i] * d;
        for (int j = 0; j < d; ++j) x[j] += e[j];
    }
    for (int j = 0; j < d; ++j) x[j] /= (double)n;
    int mo = 0;
    for (int l = 0; l < m->L; ++l) {
        const olayer* ly = &m->layers[l];
        rms(x, d, xn);
        mv(ly->mix, xn, d, d, a);
        for (int j = 0; j < d; ++j) x[j] += a[j];
        rms(x, d, xn); /* xn now holds xf */
        for (int j = 0; j < d; ++j) y[j] = 0.0;
        if (ly->is_moe) {
            mtv(ly->gate, xn, d, E, gl);
            for (int e = 0; e < E; ++e) gl[e] += ly->bias[e];
            if (g_gate_dump) memcpy(g_gate_dump + (size_t)mo * E, gl, sizeof(double) * E);
            softmax_(gl, E, pr);
            topk_(gl, E, K, raw);
            for (int k = 0; k < K; ++k) {
                int pick = raw[k], ex = pick;
                if (restricted) {
                    const int* ds = restricted + (size_t)mo * nd;
                    ex = aff ? nearest_(aff->dist + (size_t)mo * E * E, E, pick, ds, nd, chosen, k)
                             : surrogate_(mo, pick, (size_t)n, ds, nd, chosen, k);
                }
                chosen[k] = ex;
                expert_fwd(m, &ly->experts[ex], xn, eo);
                for (int j = 0; j < d; ++j) y[j] += pr[pick] * eo[j];
            }
            if (raw_out) memcpy(raw_out + (size_t)mo * K, raw, sizeof(int) * K);
            if (fin_out) memcpy(fin_out + (size_t)mo * K, chosen, sizeof(int) * K);
            ++mo;
        } else {
            expert_fwd(m, &ly->ffn, xn, y);
        }
        for (int j = 0; j < d; ++j) x[j] += y[j];
    }
    rms(x, d, xn);
    mtv(m->head, xn, d, m->V, logits);
    arena_release(mark);
}

static void moe_half(const omodel* m, const olayer* ly, int mo, double* x, int plen, const int* restricted, int nd,
                     const oaff* aff, int last, int* raw_out, int* fin_out) {
    const int d = m->d, E = m->E, K = m->K;
    blk* mark = g_arena;
    double* xn = (double*)amalloc(sizeof(double) * d);
    double* y = (double*)amalloc(sizeof(double) * d);
    double* eo = (double*)amalloc(sizeof(double) * d);
    double* gl = (double*)amalloc(sizeof(double) * E);
    double* pr = (double*)amalloc(sizeof(double) * E);
    int* raw = (int*)amalloc(sizeof(int) * K);
    int* chosen = (int*)amalloc(sizeof(int) * K);
    rms(x, d, xn);
    for (int j = 0; j < d; ++j) y[j] = 0.0;
    if (mo >= 0) {
        mtv(ly->gate, xn, d, E, gl);
        for (int e = 0; e < E; ++e) gl[e] += ly->bias[e];
        if (g_gate_dump && last) memcpy(g_gate_dump + (size_t)mo * E, gl, sizeof(double) * E);
        softmax_(gl, E, pr);
        topk_(gl, E, K, raw);
        for (int k = 0; k < K; ++k) {
            int pick = raw[k], ex = pick;
            if (restricted) {
                const int* ds = restricted + (size_t)mo * nd;
                ex = aff ? nearest_(aff->dist + (size_t)mo * E * E, E, pick, ds, nd, chosen, k)
                         : surrogate_(mo, pick, (size_t)plen, ds, nd, chosen, k);
            }
            chosen[k] = ex;
            expert_fwd(m, &ly->experts[ex], xn, eo);
            for (int j = 0; j < d; ++j) y[j] += pr[pick] * eo[j];
        }
        if (raw_out) memcpy(raw_out + (size_t)mo * K, raw, sizeof(int) * K);
        if (fin_out) memcpy(fin_out + (size_t)mo * K, chosen, sizeof(int) * K);
    } else {
        expert_fwd(m, &ly->ffn, xn, y);
    }
    for (int j = 0; j < d; ++j) x[j] += y[j];
    arena_release(mark);
}

int om_forward(void* model, const int* prefix, int n, const int* restricted, int nd, void* aff, double* logits,
               int* raw_out, int* final_out, char* err, int errlen) {
    ENTER(err, errlen, g_code);
    g_committed = 0;
    fwd((omodel*)model, prefix, n, restricted, nd, (oaff*)aff, logits, raw_out, final_out);
    LEAVE();
    return 0;
}

int om_forward_gates(void* model, const int* prefix, int n, double* logits, double* gates, char* err, int errlen) {
    ENTER(err, errlen, (g_gate_dump = NULL, g_code));
    g_gate_dump = gates;
    fwd((omodel*)model, prefix, n, NULL, 0, NULL, logits, NULL, NULL);
    g_gate_dump = NULL;
    LEAVE();
    return 0;
}

/* drafting.cpp:28-57 */
void* om_build_affinity(void* model) {
    omodel* m = (omodel*)model;
    oaff* a = (oaff*)calloc(1, sizeof(oaff));
    a->E = m->E; a->M = m->M;
    a->dist = (double*)calloc((size_t)m->M * m->E * m->E, sizeof(double));
    const size_t nu = (size_t)m->d * m->f;
    for (int mo = 0; mo < m->M; ++mo) {
        const olayer* ly = &m->layers[m->moe_index[mo]];
        double* D = a->dist + (size_t)mo * m->E * m->E;
        for (int i = 0; i < m->E; ++i)
            for (int j = i + 1; j < m->E; ++j) {
                const oexpert *x = &ly->experts[i], *y = &ly->experts[j];
                double ss = 0.0;
                for (size_t k = 0; k < nu; ++k) { double df = x->up[k] - y->up[k]; ss += df * df; }
                if (m->kind == 1)
                    for (size_t k = 0; k < nu; ++k) { double df = x->w3[k] - y->w3[k]; ss += df * df; }
                for (size_t k = 0; k < nu; ++k) { double df = x->down[k] - y->down[k]; ss += df * df; }
                double dd = sqrt(ss);
                D[(size_t)i * m->E + j] = dd;
                D[(size_t)j * m->E + i] = dd;
            }
    }
    return a;
}
void om_free_affinity(void* p) {
    oaff* a = (oaff*)p;
    if (a) free(a->dist);
    free(a);
}
int om_affinity_get(void* p, double* out, long long cap) {
    oaff* a = (oaff*)p;
    long long n = (long long)a->M * a->E * a->E;
    if (cap < n) return -1;
    memcpy(out, a->dist, sizeof(double) * (size_t)n);
    return 0;
}

/* ------------------------------------------------------------------ drafting policy (drafting.cpp:153-246) */
/* top_by_count (drafting.cpp:183-190): stable sort by count desc == first-max selection */
static void select_sets(int policy, const uint64_t* counts, int layers, int E, const int* cur, int ncur_layers,
                        int n, mt64* rng, int* out) {
    if (n > E) fail(1, "select_draft_experts: n_draft > experts_per_block");
    for (int l = 0; l < layers; ++l) {
        int* o = out + (size_t)l * n;
        if (policy == 0) { /* random: partial Fisher-Yates (drafting.cpp:203-214) */
            int* pool = (int*)amalloc(sizeof(int) * (size_t)E);
            for (int i = 0; i < E; ++i) pool[i] = i;
            for (int i = 0; i < n; ++i) {
                size_t j = (size_t)i + (size_t)(unif(rng) * (double)((size_t)E - (size_t)i));
                int t = pool[i]; pool[i] = pool[j]; pool[j] = t;
            }
            qsort(pool, (size_t)n, sizeof(int), cmp_int);
            memcpy(o, pool, sizeof(int) * (size_t)n);
            continue;
        }
        const uint64_t* c = counts + (size_t)l * E;
        uint8_t* taken = (uint8_t*)amalloc((size_t)E);
        int np = 0;
        int lim = n < E ? n : E;
        for (int j = 0; j < lim; ++j) {
            int best = -1;
            for (int i = 0; i < E; ++i)
                if (!taken[i] && (best < 0 || c[i] > c[best])) best = i;
            taken[best] = 1;
            if (c[best] > 0) o[np++] = best;
        }
        if (np < n && l < ncur_layers) {
            const int* cs = cur + (size_t)l * n;
            for (int i = 0; i < n; ++i) {
                if (np == n) break;
                if (!contains(o, np, cs[i])) o[np++] = cs[i];
            }
        }
        if (np != n) fail(2, "select_draft_experts: cannot assemble N draft experts");
        qsort(o, (size_t)n, sizeof(int), cmp_int);
    }
}

/* ------------------------------------------------------------------ memsim (memsim.cpp) */
typedef struct {
    int M, E;
    uint64_t cap, bpe;
    int64_t* arrival; /* -1 = not resident */
    uint8_t* pinned;
    uint64_t used, seq;
} ores;
typedef struct {
    om_ledger_entry* e;
    int n, capn;
    uint64_t tot[3], total;
} oledger;

static void ledger_add(oledger* lg, int phase, int step, int layer, int expert, uint64_t bytes) { /* memsim.cpp:33-43 */
    if (lg->n == lg->capn) {
        int nc = lg->capn ? lg->capn * 2 : 256;
        om_ledger_entry* ne = (om_ledger_entry*)realloc(lg->e, sizeof(om_ledger_entry) * (size_t)nc);
        if (!ne) fail(2, "oracle: out of memory");
        lg->e = ne; lg->capn = nc;
    }
    om_ledger_entry x = {phase, step, layer, expert, bytes};
    lg->e[lg->n++] = x;
    lg->total += bytes;
    lg->tot[phase] += bytes;
}
static void ledger_reset(oledger* lg) { lg->n = 0; lg->total = 0; lg->tot[0] = lg->tot[1] = lg->tot[2] = 0; }

static void tier_validate(const om_run_cfg* t, int nd, int M) { /* memsim.cpp:21-31 */
    if (t->host_bandwidth <= 0.0) fail(1, "tier: host_bandwidth > 0 violated");
    if (t->ssd_bandwidth < 0.0) fail(1, "tier: ssd_bandwidth >= 0 violated");
    if (t->bytes_per_expert == 0) fail(1, "tier: bytes_per_expert > 0 violated");
    if (t->compute_rate <= 0.0) fail(1, "tier: compute_rate > 0 violated");
    if (t->compute_cost_per_expert < 0.0) fail(1, "tier: expert compute cost >= 0 violated");
    uint64_t need = (uint64_t)nd * (uint64_t)M * t->bytes_per_expert;
    if (t->device_capacity_bytes < need) fail(1, "tier: device capacity below N * moe_layers * bytes_per_expert");
}
static void res_init(ores* r, int M, int E, const om_run_cfg* t) { /* memsim.cpp:67-70 */
    tier_validate(t, 0, M);
    r->M = M; r->E = E; r->cap = t->device_capacity_bytes; r->bpe = t->bytes_per_expert;
    r->arrival = (int64_t*)amalloc(sizeof(int64_t) * (size_t)M * E);
    r->pinned = (uint8_t*)amalloc((size_t)M * E);
    for (int i = 0; i < M * E; ++i) r->arrival[i] = -1;
    r->used = 0; r->seq = 0;
}
static void admit(ores* r, int key, const uint8_t* keep) { /* memsim.cpp:81-100 */
    while (r->used + r->bpe > r->cap) {
        int victim = -1;
        for (int k = 0; k < r->M * r->E; ++k) {
            if (r->arrival[k] < 0 || r->pinned[k] || keep[k]) continue;
            if (victim < 0 || r->arrival[k] < r->arrival[victim]) victim = k;
        }
        if (victim < 0) fail(2, "residency: device capacity exhausted with no evictable expert");
        r->arrival[victim] = -1;
        r->used -= r->bpe;
    }
    r->arrival[key] = (int64_t)r->seq++;
    r->used += r->bpe;
}
/* memsim.cpp:102-113; keys is a bitmap over (layer, expert), iterated in std::set order */
static uint64_t ensure(ores* r, const uint8_t* keys, int phase, int step, oledger* lg) {
    uint64_t b = 0;
    for (int k = 0; k < r->M * r->E; ++k) {
        if (!keys[k] || r->arrival[k] >= 0) continue;
        admit(r, k, keys);
        ledger_add(lg, phase, step, k / r->E, k % r->E, r->bpe);
        b += r->bpe;
    }
    return b;
}
/* memsim.cpp:115-150 */
static uint64_t pin(ores* r, const int* sets, int layers, int n, oledger* lg, int phase, int step) {
    if (layers != r->M) fail(2, "pin_draft_experts: set count != MoE layer count");
    uint8_t* target = (uint8_t*)amalloc((size_t)r->M * r->E);
    for (int l = 0; l < r->M; ++l)
        for (int i = 0; i < n; ++i) {
            int e = sets[(size_t)l * n + i];
            if (e < 0 || e >= r->E) fail(2, "residency: expert key out of range");
            if (target[l * r->E + e]) fail(2, "pin_draft_experts: duplicate expert in draft set");
            target[l * r->E + e] = 1;
        }
    for (int k = 0; k < r->M * r->E; ++k)
        if (r->pinned[k] && !target[k]) r->pinned[k] = 0;
    uint64_t b = 0;
    for (int k = 0; k < r->M * r->E; ++k) {
        if (!target[k]) continue;
        if (r->arrival[k] < 0) {
            admit(r, k, target);
            ledger_add(lg, phase, step, k / r->E, k % r->E, r->bpe);
            b += r->bpe;
        }
        r->pinned[k] = 1;
    }
    return b;
}
static void flush(ores* r) { /* memsim.cpp:152-161 */
    for (int k = 0; k < r->M * r->E; ++k)
        if (r->arrival[k] >= 0 && !r->pinned[k]) { r->arrival[k] = -1; r->used -= r->bpe; }
}
/* memsim.cpp:163-172 */
static double step_lat(uint64_t toks, uint64_t experts, uint64_t bytes, const om_run_cfg* t, int overlap) {
    double c = (double)toks / t->compute_rate + (double)experts * t->compute_cost_per_expert;
    double bw = t->ssd_bandwidth > 0.0 ? t->ssd_bandwidth : t->host_bandwidth;
    double mg = (double)bytes / bw;
    return overlap ? (c > mg ? c : mg) : c + mg;
}

/* ------------------------------------------------------------------ result helpers */
typedef struct { int* v; int n, cap; } ivec;
static void ipush(ivec* a, int x) {
    if (a->n == a->cap) {
        a->cap = a->cap ? a->cap * 2 : 1024;
        a->v = (int*)realloc(a->v, sizeof(int) * (size_t)a->cap);
        if (!a->v) fail(2, "oracle: out of memory");
    }
    a->v[a->n++] = x;
}

void om_free_result(om_result* r) {
    if (!r) return;
    free(r->tokens); free(r->n_tokens); free(r->ledger); free(r->outcomes); free(r->outcome_drafts);
    free(r->trace); free(r->hotness);
    free(r);
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void validate_decode(const om_run_cfg* c) { /* specdec.cpp:15-23 (greedy; batch/prompt_len from args) */
    if (c->gamma < 1) fail(1, "spec: gamma >= 1 violated");
    if (c->max_new_tokens < 1) fail(1, "spec: max_new_tokens >= 1 violated");
    if (c->warmup_steps < 1) fail(1, "spec: warmup_steps >= 1 violated");
}

/* Thread-safe owner of heap results that must be freed on failure. */
static __thread om_result* g_pending;
static __thread ivec g_iv[3];
static __thread oledger g_lg;
static void pending_cleanup(void) {
    om_free_result(g_pending); g_pending = NULL;
    for (int i = 0; i < 3; ++i) { free(g_iv[i].v); g_iv[i].v = NULL; g_iv[i].n = g_iv[i].cap = 0; }
    free(g_lg.e); memset(&g_lg, 0, sizeof g_lg);
}

static om_result* new_result(int B, int max_new, int M, int E, int K, int gamma) {
    om_result* r = (om_result*)calloc(1, sizeof(om_result));
    r->B = B; r->max_new = max_new; r->moe_layers = M; r->experts = E; r->top_k = K; r->gamma = gamma;
    r->tokens = (int*)calloc((size_t)B * (size_t)max_new + 1, sizeof(int));
    r->n_tokens = (int*)calloc((size_t)B, sizeof(int));
    r->hotness = (uint64_t*)calloc((size_t)M * E, sizeof(uint64_t));
    return r;
}

/* A growable sequence per batch row. */
typedef struct { int* t; int n, cap; } seqv;
static void spush(seqv* s, int x) {
    if (s->n == s->cap) {
        int nc = s->cap * 2 + 16;
        int* nt = (int*)amalloc(sizeof(int) * (size_t)nc);
        if (s->n) memcpy(nt, s->t, sizeof(int) * (size_t)s->n);
        s->t = nt; s->cap = nc;
    }
    s->t[s->n++] = x;
}

/* specdec.cpp:190-397 (greedy mode) */
static om_result* run_spec_(omodel* m, const om_run_cfg* cfg, const int* prompts, int B, int plen, oaff* aff) {
    validate_decode(cfg);
    if (B < 1) fail(1, "spec: batch >= 1 violated");
    if (plen < 1) fail(1, "spec: prompt_len >= 1 violated");
    const int M = m->M, E = m->E, K = m->K, g = cfg->gamma, nd = cfg->n_draft;
    if (nd < K) fail(1, "spec: n_draft >= top_k violated");
    if (nd > E) fail(1, "spec: n_draft <= experts_per_block violated");
    tier_validate(cfg, nd, M);
    if (cfg->use_affinity && !aff) fail(2, "run_specmoe: affinity table required but missing");
    const oaff* remap = cfg->use_affinity ? aff : NULL;
    double t0 = now_s();

    mt64* prng = (mt64*)amalloc(sizeof(mt64));
    mt_seed(prng, substream2(cfg->run_seed, 0x706f6c69ULL, 0));
    om_result* R = g_pending = new_result(B, cfg->max_new_tokens, M, E, K, g);
    ores res;
    res_init(&res, M, E, cfg);
    uint64_t* pc = (uint64_t*)amalloc(sizeof(uint64_t) * (size_t)M * E); /* phase counter */
    int* sets = (int*)amalloc(sizeof(int) * (size_t)M * nd);
    int* nsets = (int*)amalloc(sizeof(int) * (size_t)M * nd);
    select_sets(0, pc, M, E, sets, 0, nd, prng, sets);

    if (cfg->policy == 1) { /* hot_global warmup (specdec.cpp:223-245) */
        uint64_t* wc = (uint64_t*)amalloc(sizeof(uint64_t) * (size_t)M * E);
        oledger wl = {0};
        ores wr;
        res_init(&wr, M, E, cfg);
        seqv* work = (seqv*)amalloc(sizeof(seqv) * (size_t)B);
        for (int b = 0; b < B; ++b)
            for (int i = 0; i < plen; ++i) spush(&work[b], prompts[(size_t)b * plen + i]);
        double* lg = (double*)amalloc(sizeof(double) * m->V);
        int* raw = (int*)amalloc(sizeof(int) * (size_t)M * K);
        uint8_t* need = (uint8_t*)amalloc((size_t)M * E);
        for (int st = 0; st < cfg->warmup_steps; ++st) {
            memset(need, 0, (size_t)M * E);
            for (int b = 0; b < B; ++b) {
                fwd(m, work[b].t, work[b].n, NULL, 0, NULL, lg, raw, NULL);
                for (int i = 0; i < M * K; ++i) need[(i / K) * E + raw[i]] = 1;
                spush(&work[b], greedy_(lg, m->V));
                for (int i = 0; i < M * K; ++i) wc[(i / K) * E + raw[i]]++;
            }
            ensure(&wr, need, 2, st, &wl);
            flush(&wr);
        }
        R->warmup_bytes = wl.total;
        free(wl.e);
        memcpy(nsets, sets, sizeof(int) * (size_t)M * nd);
        select_sets(1, wc, M, E, nsets, M, nd, prng, sets);
    }
    oledger* L = &g_lg;
    memset(L, 0, sizeof *L);
    pin(&res, sets, M, nd, L, 1, -1);
    R->setup_bytes = L->total;
    ledger_reset(L);

    seqv* seq = (seqv*)amalloc(sizeof(seqv) * (size_t)B);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < plen; ++i) spush(&seq[b], prompts[(size_t)b * plen + i]);
    int* gen = (int*)amalloc(sizeof(int) * (size_t)B);
    uint64_t tau_sum = 0, tau_cnt = 0;
    double spec_s = 0.0, ver_s = 0.0, step_s = 0.0;
    ivec* oc = &g_iv[0];   /* outcomes: seq, phase, accepted, correction, generated, drafts... */
    ivec* tr = &g_iv[1];   /* trace */
    ivec* lam = &g_iv[2];  /* lambda inputs as 4 ints each (fits: counts < 2^31) */
    int* actives = (int*)amalloc(sizeof(int) * (size_t)B);
    int* drafts = (int*)amalloc(sizeof(int) * (size_t)B * g);
    double* lg = (double*)amalloc(sizeof(double) * m->V);
    int* raw = (int*)amalloc(sizeof(int) * (size_t)M * K);
    int* fin = (int*)amalloc(sizeof(int) * (size_t)M * K);
    int* vraw = (int*)amalloc(sizeof(int) * (size_t)B * (g + 1) * M * K);
    int* acc = (int*)amalloc(sizeof(int) * (size_t)B);
    int* corr = (int*)amalloc(sizeof(int) * (size_t)B);
    uint8_t* exec = (uint8_t*)amalloc((size_t)M * E);
    uint8_t* need = (uint8_t*)amalloc((size_t)M * E);
    uint8_t* first = (uint8_t*)amalloc((size_t)M * E);
    int* amax = (int*)amalloc(sizeof(int) * (size_t)(g + 1));
    seqv work = {0};
    int phase = 0;
    for (;;) {
        int na = 0;
        for (int b = 0; b < B; ++b)
            if (gen[b] < cfg->max_new_tokens) actives[na++] = b;
        if (na == 0) break;
        for (int l = 0; l < M; ++l)
            for (int i = 0; i < nd; ++i) {
                int k = l * E + sets[(size_t)l * nd + i];
                if (!res.pinned[k] || res.arrival[k] < 0) fail(2, "run_specmoe: draft expert not pinned on device");
            }
        /* (a) speculate (specdec.cpp:25-61) */
        uint64_t spec_before = L->tot[0];
        for (int t = 0; t < g; ++t) {
            memset(exec, 0, (size_t)M * E);
            uint64_t distinct = 0;
            for (int s = 0; s < na; ++s) {
                int b = actives[s];
                work.n = 0;
                for (int i = 0; i < seq[b].n; ++i) spush(&work, seq[b].t[i]);
                for (int i = 0; i < t; ++i) spush(&work, drafts[(size_t)s * g + i]);
                g_committed = seq[b].n; /* attention extension: the committed part of work */
                fwd(m, work.t, work.n, sets, nd, remap, lg, raw, fin);
                g_committed = 0;
                drafts[(size_t)s * g + t] = greedy_(lg, m->V);
                for (int i = 0; i < M * K; ++i) {
                    int k = (i / K) * E + fin[i];
                    if (!exec[k]) { exec[k] = 1; ++distinct; }
                }
            }
            spec_s += step_lat((uint64_t)na, distinct, 0, cfg, 0);
        }
        if (L->tot[0] != spec_before) fail(2, "run_specmoe: speculation phase migrated bytes");
        /* (b) verify_greedy per active sequence (specdec.cpp:63-80) */
        for (int s = 0; s < na; ++s) {
            int b = actives[s];
            work.n = 0;
            for (int i = 0; i < seq[b].n; ++i) spush(&work, seq[b].t[i]);
            for (int i = 0; i <= g; ++i) {
                fwd(m, work.t, work.n, NULL, 0, NULL, lg, vraw + ((size_t)s * (g + 1) + i) * M * K, NULL);
                amax[i] = greedy_(lg, m->V);
                if (i < g) spush(&work, drafts[(size_t)s * g + i]);
            }
            int a = 0;
            while (a < g && drafts[(size_t)s * g + a] == amax[a]) ++a;
            acc[s] = a;
            corr[s] = amax[a];
        }
        /* coalesced union (specdec.cpp:303-315) */
        memset(need, 0, (size_t)M * E);
        memset(first, 0, (size_t)M * E);
        uint64_t n_need = 0, n_first = 0;
        for (int s = 0; s < na; ++s)
            for (int i = 0; i <= g; ++i)
                for (int q = 0; q < M * K; ++q) {
                    int k = (q / K) * E + vraw[((size_t)s * (g + 1) + i) * M * K + q];
                    if (!need[k]) { need[k] = 1; ++n_need; }
                    if (i == 0 && !first[k]) { first[k] = 1; ++n_first; }
                }
        uint64_t vb = ensure(&res, need, 1, phase, L);
        uint64_t vt = (uint64_t)na * (uint64_t)(g + 1);
        ver_s += step_lat(vt, n_need, vb, cfg, 0);
        ipush(lam, (int)vt); ipush(lam, (int)n_need); ipush(lam, na); ipush(lam, (int)n_first);
        step_s += step_lat((uint64_t)na, n_first, n_first * cfg->bytes_per_expert, cfg, 0);
        /* acceptance bookkeeping (specdec.cpp:330-362) */
        for (int s = 0; s < na; ++s) {
            int b = actives[s];
            ipush(oc, b); ipush(oc, phase); ipush(oc, acc[s]); ipush(oc, corr[s]); ipush(oc, acc[s] + 1);
            for (int i = 0; i < g; ++i) ipush(oc, drafts[(size_t)s * g + i]);
            tau_sum += (uint64_t)(acc[s] + 1);
            ++tau_cnt;
            int room = cfg->max_new_tokens - gen[b];
            int take = acc[s] + 1 < room ? acc[s] + 1 : room;
            for (int t = 0; t < take; ++t) {
                int tok = t < acc[s] ? drafts[(size_t)s * g + t] : corr[s];
                spush(&seq[b], tok);
                R->tokens[(size_t)b * R->max_new + R->n_tokens[b]++] = tok;
            }
            gen[b] += take;
            for (int i = 0; i <= g; ++i)
                for (int q = 0; q < M * K; ++q) {
                    int k = (q / K) * E + vraw[((size_t)s * (g + 1) + i) * M * K + q];
                    pc[k]++;
                    R->hotness[k]++;
                }
            if (cfg->collect_trace)
                for (int i = 0; i <= g; ++i)
                    for (int l = 0; l < M; ++l) {
                        ipush(tr, phase); ipush(tr, b); ipush(tr, l);
                        for (int q = 0; q < K; ++q) ipush(tr, vraw[((size_t)s * (g + 1) + i) * M * K + (size_t)l * K + q]);
                    }
        }
        if (cfg->policy == 2) {
            select_sets(2, pc, M, E, sets, M, nd, prng, nsets);
            pin(&res, nsets, M, nd, L, 1, phase);
            memcpy(sets, nsets, sizeof(int) * (size_t)M * nd);
        }
        memset(pc, 0, sizeof(uint64_t) * (size_t)M * E);
        flush(&res);
        ++phase;
    }
    R->wall_s = now_s() - t0;
    R->phases = phase;
    R->tau_mean = tau_cnt ? (double)tau_sum / (double)tau_cnt : 1.0;
    R->tokens_total = 0;
    for (int b = 0; b < B; ++b) R->tokens_total += (uint64_t)R->n_tokens[b];
    R->speculation_s = spec_s;
    R->verification_s = ver_s;
    R->modeled_seconds = spec_s + ver_s;
    R->tokens_per_sec = R->modeled_seconds > 0.0 ? (double)R->tokens_total / R->modeled_seconds : 0.0;
    R->bytes_spec = L->tot[0]; R->bytes_verify = L->tot[1]; R->bytes_baseline = L->tot[2]; R->bytes_total = L->total;
    if (lam->n == 0) R->lambda = 1.0;
    else { /* specdec.cpp:159-172 */
        double vs = 0.0, ss = 0.0;
        for (int i = 0; i < lam->n; i += 4) {
            vs += step_lat((uint64_t)lam->v[i], (uint64_t)lam->v[i + 1], (uint64_t)lam->v[i + 1] * cfg->bytes_per_expert, cfg, 0);
            ss += step_lat((uint64_t)lam->v[i + 2], (uint64_t)lam->v[i + 3], (uint64_t)lam->v[i + 3] * cfg->bytes_per_expert, cfg, 0);
        }
        if (ss <= 0.0) fail(2, "measure_lambda: zero single-step latency");
        R->lambda = vs / ss;
    }
    R->c_measured = (phase > 0 && step_s > 0.0) ? (spec_s / ((double)phase * g)) / (step_s / (double)phase) : 0.0;
    /* move vectors into the result */
    const int per = 5 + g;
    R->n_outcomes = oc->n / per;
    R->outcomes = (om_outcome*)calloc((size_t)R->n_outcomes + 1, sizeof(om_outcome));
    R->outcome_drafts = (int*)calloc((size_t)R->n_outcomes * g + 1, sizeof(int));
    for (int i = 0; i < R->n_outcomes; ++i) {
        const int* v = oc->v + (size_t)i * per;
        om_outcome o = {v[0], v[1], v[2], v[3], v[4]};
        R->outcomes[i] = o;
        memcpy(R->outcome_drafts + (size_t)i * g, v + 5, sizeof(int) * (size_t)g);
    }
    R->n_trace = tr->n / (3 + K);
    R->trace = tr->v; tr->v = NULL; tr->n = tr->cap = 0;
    R->n_ledger = L->n;
    R->ledger = L->e; L->e = NULL;
    free(oc->v); oc->v = NULL; oc->n = oc->cap = 0;
    free(lam->v); lam->v = NULL; lam->n = lam->cap = 0;
    memset(L, 0, sizeof *L);
    g_pending = NULL;
    return R;
}

/* baselines.cpp:29-99 (run_stepwise, greedy).  overlap: modeled step time max(compute, migration)
 * (baselines.cpp:101-105); pinned [M][npin] sets pinned before the loop (run_caching, 41-46). */
static om_result* run_stepwise_(omodel* m, const om_run_cfg* cfg, const int* prompts, int B, int plen, int overlap,
                                const int* pinned, int npin) {
    validate_decode(cfg);
    if (B < 1) fail(1, "baseline run: no prompts");
    const int M = m->M, E = m->E, K = m->K;
    tier_validate(cfg, 0, M);
    double t0 = now_s();
    om_result* R = g_pending = new_result(B, cfg->max_new_tokens, M, E, K, 0);
    ores res;
    res_init(&res, M, E, cfg);
    oledger* L = &g_lg;
    memset(L, 0, sizeof *L);
    if (pinned) {
        pin(&res, pinned, M, npin, L, 2, -1);
        R->setup_bytes = L->total;
        ledger_reset(L);
    }
    seqv* seq = (seqv*)amalloc(sizeof(seqv) * (size_t)B);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < plen; ++i) spush(&seq[b], prompts[(size_t)b * plen + i]);
    double* lg = (double*)amalloc(sizeof(double) * m->V);
    int* raw = (int*)amalloc(sizeof(int) * (size_t)M * K);
    uint8_t* need = (uint8_t*)amalloc((size_t)M * E);
    ivec* tr = &g_iv[1];
    double modeled = 0.0;
    for (int st = 0; st < cfg->max_new_tokens; ++st) {
        memset(need, 0, (size_t)M * E);
        uint64_t n_need = 0;
        for (int b = 0; b < B; ++b) {
            fwd(m, seq[b].t, seq[b].n, NULL, 0, NULL, lg, raw, NULL);
            for (int q = 0; q < M * K; ++q) {
                int k = (q / K) * E + raw[q];
                if (!need[k]) { need[k] = 1; ++n_need; }
            }
            int tok = greedy_(lg, m->V);
            spush(&seq[b], tok);
            R->tokens[(size_t)b * R->max_new + R->n_tokens[b]++] = tok;
            if (cfg->collect_trace)
                for (int l = 0; l < M; ++l) {
                    ipush(tr, st); ipush(tr, b); ipush(tr, l);
                    for (int q = 0; q < K; ++q) ipush(tr, raw[l * K + q]);
                }
            for (int q = 0; q < M * K; ++q) R->hotness[(q / K) * E + raw[q]]++;
        }
        uint64_t bytes = ensure(&res, need, 2, st, L);
        modeled += step_lat((uint64_t)B, n_need, bytes, cfg, overlap);
        flush(&res);
    }
    R->wall_s = now_s() - t0;
    R->phases = cfg->max_new_tokens;
    R->tau_mean = 1.0;
    R->tokens_total = (uint64_t)B * (uint64_t)cfg->max_new_tokens;
    R->modeled_seconds = modeled;
    R->verification_s = modeled;
    R->tokens_per_sec = modeled > 0.0 ? (double)R->tokens_total / modeled : 0.0;
    R->bytes_spec = L->tot[0]; R->bytes_verify = L->tot[1]; R->bytes_baseline = L->tot[2]; R->bytes_total = L->total;
    R->lambda = 1.0;
    R->c_measured = 0.0;
    R->n_trace = tr->n / (3 + K);
    R->trace = tr->v; tr->v = NULL; tr->n = tr->cap = 0;
    R->n_ledger = L->n;
    R->ledger = L->e; L->e = NULL;
    memset(L, 0, sizeof *L);
    g_pending = NULL;
    return R;
}

static om_result* run_ondemand_(omodel* m, const om_run_cfg* cfg, const int* prompts, int B, int plen) {
    return run_stepwise_(m, cfg, prompts, B, plen, 0, NULL, 0);
}

/* baselines.cpp:113-157: greedy on-demand profiling warmup over the same prompts (its ledger reported
 * as warmup_bytes), top ceil(cache_fraction * E) experts per block by hot_global, pinned, on-demand. */
static om_result* run_caching_(omodel* m, const om_run_cfg* cfg, double cache_fraction, const int* prompts, int B,
                               int plen) {
    if (!(cache_fraction > 0.0 && cache_fraction < 1.0)) fail(1, "baseline: 0 < cache_fraction < 1 violated");
    if (cfg->warmup_steps < 1) fail(1, "baseline: warmup_steps >= 1 violated");
    const int M = m->M, E = m->E, K = m->K;
    uint64_t* wc = (uint64_t*)amalloc(sizeof(uint64_t) * (size_t)M * E);
    oledger wl = {0};
    ores wr;
    res_init(&wr, M, E, cfg);
    seqv* work = (seqv*)amalloc(sizeof(seqv) * (size_t)B);
    for (int b = 0; b < B; ++b)
        for (int i = 0; i < plen; ++i) spush(&work[b], prompts[(size_t)b * plen + i]);
    double* lg = (double*)amalloc(sizeof(double) * m->V);
    int* raw = (int*)amalloc(sizeof(int) * (size_t)M * K);
    uint8_t* need = (uint8_t*)amalloc((size_t)M * E);
    for (int st = 0; st < cfg->warmup_steps; ++st) {
        memset(need, 0, (size_t)M * E);
        for (int b = 0; b < B; ++b) {
            fwd(m, work[b].t, work[b].n, NULL, 0, NULL, lg, raw, NULL);
            for (int i = 0; i < M * K; ++i) need[(i / K) * E + raw[i]] = 1;
            spush(&work[b], greedy_(lg, m->V));
            for (int i = 0; i < M * K; ++i) wc[(i / K) * E + raw[i]]++;
        }
        ensure(&wr, need, 2, st, &wl);
        flush(&wr);
    }
    const uint64_t warm = wl.total;
    free(wl.e);
    const int cpl = (int)ceil(cache_fraction * (double)E);
    if ((uint64_t)cpl * (uint64_t)M * cfg->bytes_per_expert > cfg->device_capacity_bytes)
        fail(1, "caching: cached experts exceed device capacity");
    int* cached = (int*)amalloc(sizeof(int) * (size_t)M * cpl);
    select_sets(1, wc, M, E, NULL, 0, cpl, NULL, cached);
    om_result* R = run_stepwise_(m, cfg, prompts, B, plen, 0, cached, cpl);
    R->warmup_bytes = warm;
    return R;
}

om_result* om_run_specmoe(void* model, const om_run_cfg* cfg, const int* prompts, int B, int plen, void* aff,
                          char* err, int errlen) {
    ENTER(err, errlen, (pending_cleanup(), (om_result*)NULL));
    om_result* r = run_spec_((omodel*)model, cfg, prompts, B, plen, (oaff*)aff);
    LEAVE();
    return r;
}
om_result* om_run_ondemand(void* model, const om_run_cfg* cfg, const int* prompts, int B, int plen, char* err,
                           int errlen) {
    ENTER(err, errlen, (pending_cleanup(), (om_result*)NULL));
    om_result* r = run_ondemand_((omodel*)model, cfg, prompts, B, plen);
    LEAVE();
    return r;
}

om_result* om_run_overlap(void* model, const om_run_cfg* cfg, const int* prompts, int B, int plen, char* err,
                          int errlen) {
    ENTER(err, errlen, (pending_cleanup(), (om_result*)NULL));
    om_result* r = run_stepwise_((omodel*)model, cfg, prompts, B, plen, 1, NULL, 0);
    LEAVE();
    return r;
}
om_result* om_run_caching(void* model, const om_run_cfg* cfg, double cache_fraction, const int* prompts, int B,
                          int plen, char* err, int errlen) {
    ENTER(err, errlen, (pending_cleanup(), (om_result*)NULL));
    om_result* r = run_caching_((omodel*)model, cfg, cache_fraction, prompts, B, plen);
    LEAVE();
    return r;
}

/* ------------------------------------------------------------------ CPU-baseline timing */
typedef struct { omodel* m; const int* p; int n, iters; } fwd_job;
static void* fwd_worker(void* arg) {
    fwd_job* j = (fwd_job*)arg;
    double* lg = (double*)malloc(sizeof(double) * (size_t)j->m->V);
    char err[64];
    for (int i = 0; i < j->iters; ++i) om_forward(j->m, j->p, j->n, NULL, 0, NULL, lg, NULL, NULL, err, 64);
    free(lg);
    return NULL;
}
double om_time_forward(void* model, const int* prefix, int n, int threads, int iters) {
    fwd_job job = {(omodel*)model, prefix, n, iters};
    pthread_t th[256];
    if (threads > 256) threads = 256;
    double t0 = now_s();
    for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, fwd_worker, &job);
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    return now_s() - t0;
}

/* ------------------------------------------------------------------ host primitives */
int om_route_topk(const double* l, int n, int k, int* out) {
    ENTER(NULL, 0, -g_code);
    topk_(l, n, k, out);
    LEAVE();
    return 0;
}
int om_greedy_next(const double* l, int n) {
    ENTER(NULL, 0, -g_code);
    int r = greedy_(l, n);
    LEAVE();
    return r;
}
int om_softmax(const double* l, int n, double* out) {
    ENTER(NULL, 0, -g_code);
    softmax_(l, n, out);
    LEAVE();
    return 0;
}
int om_nearest_draft_expert(const double* dist_l, int E, int raw, const int* ds, int nd, const int* ex, int nex) {
    ENTER(NULL, 0, -g_code);
    int r = nearest_(dist_l, E, raw, ds, nd, ex, nex);
    LEAVE();
    return r;
}
int om_select_draft_experts(int policy, const uint64_t* counts, int layers, int E, const int* cur, int n,
                            uint64_t seed, int* out) {
    ENTER(NULL, 0, -g_code);
    mt64* r = (mt64*)amalloc(sizeof(mt64));
    mt_seed(r, seed);
    select_sets(policy, counts, layers, E, cur, cur ? layers : 0, n, r, out);
    LEAVE();
    return 0;
}
/* drafting.cpp:229-246 */
double om_skewness(const uint64_t* counts, int layers, int E, uint64_t routed, double frac) {
    if (layers <= 0 || routed == 0) return -1.0;
    double acc = 0.0;
    for (int l = 0; l < layers; ++l) {
        const uint64_t* c = counts + (size_t)l * E;
        uint64_t tot = 0;
        for (int e = 0; e < E; ++e) tot += c[e];
        if (tot == 0) return -1.0;
        uint64_t* s = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)E);
        memcpy(s, c, sizeof(uint64_t) * (size_t)E);
        for (int i = 0; i < E; ++i) /* selection sort descending */
            for (int j = i + 1; j < E; ++j)
                if (s[j] > s[i]) { uint64_t t = s[i]; s[i] = s[j]; s[j] = t; }
        size_t top = (size_t)ceil(frac * (double)E);
        uint64_t hot = 0;
        for (size_t i = 0; i < top; ++i) hot += s[i];
        free(s);
        acc += (double)hot / (double)tot;
    }
    return acc / layers;
}
