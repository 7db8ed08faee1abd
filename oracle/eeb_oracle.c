/*
 * eeb_oracle.c — straight-line CPU oracle of the batched early-exit decode
 * step.  TEST INFRASTRUCTURE ONLY (see eeb_oracle.h for what it restates and
 * the reference file:line anchors of every rule).
 *
 * Compiled with -ffp-contract=off so the weight definition (two correctly
 * rounded f32 multiplies per element) reproduces the device bit-for-bit.
 */
#include "eeb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
const char* orc_last_error(void) { return g_err; }
static int fail(const char* m) {
    snprintf(g_err, sizeof g_err, "%s", m);
    return -1;
}

/* ---------------------------------------------------------------------------
 * The reference's per-token decision over one complete record (every head
 * observed, ascending layers, last = final head):
 *   flat          observation_for_depth  trace.hpp:86-97, exit = depth, breached = conf < th  engine.hpp:350-354
 *   introspective earliest_confident_obs trace.hpp:69-76 (>=), exit = obs.layer               engine.hpp:355-359
 *   full depth    observations.back(), exit = num_layers, never breached                      engine.hpp:360-364
 *   unchanged     obs.token == final token                                                    engine.hpp:366
 * Returns the index of the observation used, or -1 (DomainError) when flat
 * finds no head at or below the depth (trace.hpp:92-93).
 * ------------------------------------------------------------------------- */
int orc_decide(int policy, int n, const int32_t* layers, const int32_t* toks, const float* confs, float th,
               int depth, int num_layers, orc_decision* out) {
    int idx = -1;
    if (n <= 0) return fail("token record has no observations");
    if (policy == 0) {
        for (int k = 0; k < n; ++k) {
            if (layers[k] == depth) { idx = k; break; }
            if (layers[k] < depth) idx = k;
        }
        if (idx < 0) return fail("no observation at or below the serving depth");
        out->exit_layer = depth;
        out->breached = confs[idx] < th;
    } else if (policy == 2) {
        idx = n - 1;
        out->exit_layer = num_layers;
        out->breached = 0;
    } else {
        idx = n - 1;
        for (int k = 0; k < n; ++k)
            if (confs[k] >= th) { idx = k; break; }
        out->exit_layer = layers[idx];
        out->breached = confs[idx] < th;
    }
    out->index = idx;
    out->unchanged = toks[idx] == toks[n - 1];
    return idx;
}

/* ---------------------------------------------------------------------------
 * Synthetic model definition (restated).
 * ------------------------------------------------------------------------- */
#define U_SCALE 3.46410161513775f /* 2*sqrt(3): unit variance */
#define SIGMA 0.02f
#define AMP_A 0.25f
#define AMP_B 1.0f
#define BETA 0.02f
#define JITTER 0.1f
#define LAYER_VAR 2e-3

static uint64_t fin64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static float draw(uint64_t seed, int tid, uint64_t idx) {
    uint64_t h = fin64(seed + 0x9E3779B97F4A7C15ULL * (uint64_t)(tid + 1));
    h = fin64(h ^ (idx * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
    return (float)(uint32_t)(h >> 40) * 0x1p-24f - 0.5f;
}
static float unitv(uint64_t seed, int tid, uint64_t idx) { return draw(seed, tid, idx) * U_SCALE; }
static int tid_layer(int l, int kind) { return l * 16 + kind; }
static int tid_base(int kind, int e) { return 8192 + kind * 64 + e; }

static float bf16_round(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    memcpy(&f, &u, 4);
    return f;
}

struct orc_model {
    orc_desc d;
    int threads;
    int hd, dq, dkv, up_rows;
    float alpha[64];
    float rsig;
    uint32_t pmul;
    int loaded;
    float* emb;
    float* head[64];
    float* head_norm[64];
    float** attn_norm; float** mlp_norm; float** wqkv; float** wo; float** wup; float** wdown;
    float* kc; float* vc;     /* [L][slots][Hkv][S][hd] */
    uint8_t* kv_depth;        /* [slots][S] */
    float* rcos; float* rsin; /* [S][hd/2] */
};

static float rnd(const orc_model* m, float v) { return m->d.dtype == 1 ? bf16_round(v) : v; }

static uint32_t coprime_mul(uint32_t vocab) {
    for (uint32_t p = 7919u;; ++p) {
        uint32_t a = p, b = vocab;
        while (b) { uint32_t t = a % b; a = b; b = t; }
        if (a == 1) return p;
    }
}

/* Head gains: target logit k*d/2 at the boundary amplitude A(1-c) must beat
 * the log-sum-exp of V-1 Gaussian logits (ln(V-1) + var/2) by logit(th). */
static void solve_alphas(orc_model* m) {
    const orc_desc* d = &m->d;
    double th = d->design_th;
    double thc = d->design_th <= 0.0f ? 1e-6 : (d->design_th >= 1.0f ? 1.0 - 1e-6 : th);
    double C = log((double)d->vocab - 1.0) + (double)BETA * BETA * d->d_model / 2.0 + log(thc / (1.0 - thc));
    double disc = 1.0 - 4.0 * C / d->d_model;
    if (disc < 0.05) disc = 0.05;
    double k = 1.0 - sqrt(disc);
    for (int e = 0; e < d->n_exits; ++e) {
        double c = d->exit_coverage[e];
        if (c > 0.99) c = 0.99;
        if (c < 0.01) c = 0.01;
        double a_star = (double)AMP_A * (1.0 - c);
        double n2 = LAYER_VAR * d->exit_layers[e];
        double rms = sqrt((a_star * a_star + (double)AMP_B * AMP_B + n2) / 2.0);
        m->alpha[e] = (float)(k * rms / a_star);
    }
}

static float z_tok(const orc_model* m, int t) { return draw(m->d.seed, tid_base(1, 0), (uint64_t)t) + 0.5f; }

static float emb_el(const orc_model* m, int t, int i) {
    const int dd = m->d.d_model;
    float g = unitv(m->d.seed, tid_base(0, 0), (uint64_t)t * dd + i);
    float amp = i < dd / 2 ? AMP_A * (1.0f - z_tok(m, t)) : AMP_B;
    return g * amp;
}
static float head_el(const orc_model* m, int e, int v, int i) {
    const int dd = m->d.d_model;
    float noise = unitv(m->d.seed, tid_base(2, e), (uint64_t)v * dd + i) * BETA;
    if (i >= dd / 2) return noise;
    int src = (int)(((uint64_t)v * m->pmul + 17u) % (uint32_t)m->d.vocab);
    float sig = unitv(m->d.seed, tid_base(0, 0), (uint64_t)src * dd + i) * m->alpha[e];
    return sig + noise;
}
static float gain_el(const orc_model* m, int tid, int i) { return 1.0f + draw(m->d.seed, tid, (uint64_t)i) * (2.0f * JITTER); }
static float lin_el(const orc_model* m, int tid, int r, int c, int cols, float scale, int zero_sig) {
    if (zero_sig && r < m->d.d_model / 2) return 0.0f;
    return unitv(m->d.seed, tid, (uint64_t)r * cols + c) * scale;
}

/* ---------------------------------------------------------------------------
 * Parallel-for over [0, n) (pthreads; the CPU baseline uses all host cores).
 * ------------------------------------------------------------------------- */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void* ctx; int64_t lo, hi; } job_t;
static void* job_run(void* p) { job_t* j = (job_t*)p; j->fn(j->ctx, j->lo, j->hi); return NULL; }
static void par_for(int threads, int64_t n, range_fn fn, void* ctx) {
    if (threads <= 1 || n < 64) { fn(ctx, 0, n); return; }
    pthread_t th[256];
    job_t jobs[256];
    if (threads > 256) threads = 256;
    int64_t per = (n + threads - 1) / threads;
    int k = 0;
    for (int t = 0; t < threads; ++t) {
        int64_t lo = t * per, hi = lo + per < n ? lo + per : n;
        if (lo >= hi) break;
        jobs[k] = (job_t){fn, ctx, lo, hi};
        pthread_create(&th[k], NULL, job_run, &jobs[k]);
        ++k;
    }
    for (int t = 0; t < k; ++t) pthread_join(th[t], NULL);
}

/* Tensor materialisation. */
typedef struct { orc_model* m; float* dst; int kind, tid, e, rows, cols, zero_sig; float scale; } fill_ctx;
static void fill_range(void* p, int64_t lo, int64_t hi) {
    fill_ctx* f = (fill_ctx*)p;
    for (int64_t idx = lo; idx < hi; ++idx) {
        int r = (int)(idx / f->cols), c = (int)(idx % f->cols);
        float v;
        switch (f->kind) {
            case 0: v = lin_el(f->m, f->tid, r, c, f->cols, f->scale, f->zero_sig); break;
            case 1: v = gain_el(f->m, f->tid, c); break;
            case 2: v = emb_el(f->m, r, c); break;
            default: v = head_el(f->m, f->e, r, c); break;
        }
        f->dst[idx] = f->kind == 1 ? v : rnd(f->m, v);
    }
}
static float* make_tensor(orc_model* m, int kind, int tid, int e, int rows, int cols, float scale, int zero_sig) {
    float* p = (float*)malloc(sizeof(float) * (size_t)rows * cols);
    if (!p) return NULL;
    fill_ctx f = {m, p, kind, tid, e, rows, cols, zero_sig, scale};
    par_for(m->threads, (int64_t)rows * cols, fill_range, &f);
    return p;
}

orc_model* orc_create(const orc_desc* d, int threads) {
    orc_model* m = (orc_model*)calloc(1, sizeof(orc_model));
    if (!m) return NULL;
    m->d = *d;
    if (m->d.norm_eps <= 0.f) m->d.norm_eps = 1e-5f;
    if (m->d.rope_theta <= 0.f) m->d.rope_theta = 10000.f;
    m->threads = threads > 0 ? threads : 1;
    m->hd = d->d_model / d->n_heads;
    m->dq = d->n_heads * m->hd;
    m->dkv = d->n_kv_heads * m->hd;
    m->up_rows = d->mlp_kind == 1 ? 2 * d->d_ffn : d->d_ffn;
    m->pmul = coprime_mul((uint32_t)d->vocab);
    solve_alphas(m);
    {
        double var_h = (double)d->d_model * SIGMA * SIGMA / 2.0;
        m->rsig = (float)sqrt(LAYER_VAR / ((double)d->d_ffn * var_h));
    }
    const int L = d->num_layers;
    m->attn_norm = (float**)calloc(L, sizeof(float*));
    m->mlp_norm = (float**)calloc(L, sizeof(float*));
    m->wqkv = (float**)calloc(L, sizeof(float*));
    m->wo = (float**)calloc(L, sizeof(float*));
    m->wup = (float**)calloc(L, sizeof(float*));
    m->wdown = (float**)calloc(L, sizeof(float*));
    size_t kv = (size_t)L * d->max_slots * d->n_kv_heads * d->max_seq_len * m->hd;
    m->kc = (float*)calloc(kv, sizeof(float));
    m->vc = (float*)calloc(kv, sizeof(float));
    m->kv_depth = (uint8_t*)calloc((size_t)d->max_slots * d->max_seq_len, 1);
    int half = m->hd / 2;
    m->rcos = (float*)malloc(sizeof(float) * (size_t)d->max_seq_len * half);
    m->rsin = (float*)malloc(sizeof(float) * (size_t)d->max_seq_len * half);
    if (!m->kc || !m->vc || !m->kv_depth || !m->rcos || !m->rsin) { orc_destroy(m); return NULL; }
    for (int p = 0; p < d->max_seq_len; ++p)
        for (int j = 0; j < half; ++j) {
            double inv = pow((double)m->d.rope_theta, -2.0 * j / (double)m->hd);
            double ang = (double)p * inv;
            m->rcos[(size_t)p * half + j] = (float)cos(ang);
            m->rsin[(size_t)p * half + j] = (float)sin(ang);
        }
    return m;
}

void orc_destroy(orc_model* m) {
    if (!m) return;
    free(m->emb);
    for (int e = 0; e < 64; ++e) { free(m->head[e]); free(m->head_norm[e]); }
    for (int l = 0; l < m->d.num_layers; ++l) {
        if (m->attn_norm) free(m->attn_norm[l]);
        if (m->mlp_norm) free(m->mlp_norm[l]);
        if (m->wqkv) free(m->wqkv[l]);
        if (m->wo) free(m->wo[l]);
        if (m->wup) free(m->wup[l]);
        if (m->wdown) free(m->wdown[l]);
    }
    free(m->attn_norm); free(m->mlp_norm); free(m->wqkv); free(m->wo); free(m->wup); free(m->wdown);
    free(m->kc); free(m->vc); free(m->kv_depth); free(m->rcos); free(m->rsin);
    free(m);
}

int orc_load(orc_model* m, int depth) {
    const orc_desc* d = &m->d;
    const int D = d->d_model;
    if (depth < 0 || depth > d->num_layers) return fail("depth out of range");
    if (!m->emb) {
        m->emb = make_tensor(m, 2, 0, 0, d->vocab, D, 0.f, 0);
        for (int e = 0; e < d->n_exits; ++e) {
            m->head[e] = make_tensor(m, 3, 0, e, d->vocab, D, 0.f, 0);
            m->head_norm[e] = make_tensor(m, 1, tid_base(3, e), e, 1, D, 0.f, 0);
        }
    }
    for (int l = m->loaded + 1; l <= depth; ++l) {
        const int i = l - 1;
        m->attn_norm[i] = make_tensor(m, 1, tid_layer(l, 0), 0, 1, D, 0.f, 0);
        m->mlp_norm[i] = make_tensor(m, 1, tid_layer(l, 3), 0, 1, D, 0.f, 0);
        m->wqkv[i] = make_tensor(m, 0, tid_layer(l, 1), 0, m->dq + 2 * m->dkv, D, SIGMA, 0);
        m->wo[i] = make_tensor(m, 0, tid_layer(l, 2), 0, D, m->dq, m->rsig, 1);
        m->wup[i] = make_tensor(m, 0, tid_layer(l, 4), 0, m->up_rows, D, SIGMA, 0);
        m->wdown[i] = make_tensor(m, 0, tid_layer(l, 5), 0, D, d->d_ffn, m->rsig, 1);
    }
    if (depth > m->loaded) m->loaded = depth;
    return 0;
}

float orc_alpha(const orc_model* m, int e) { return m->alpha[e]; }

float orc_weight(const orc_model* m, int tensor, int layer, int64_t index) {
    const float* p = NULL;
    if (tensor == 100) p = m->emb;
    else if (tensor >= 300) p = m->head_norm[tensor - 300];
    else if (tensor >= 200) p = m->head[tensor - 200];
    else {
        int i = layer - 1;
        switch (tensor) {
            case 0: p = m->attn_norm[i]; break;
            case 1: p = m->wqkv[i]; break;
            case 2: p = m->wo[i]; break;
            case 3: p = m->mlp_norm[i]; break;
            case 4: p = m->wup[i]; break;
            default: p = m->wdown[i]; break;
        }
    }
    return p ? p[index] : NAN;
}

/* Whole-tensor access (test hooks: caller-supplied weights).  Element counts
 * per kind: 0/3 norms [D]; 1 Wqkv [dq+2dkv][D]; 2 Wo [D][dq]; 4 Wup [up_rows][D];
 * 5 Wdown [D][F]; 100 embedding [V][D]; 200+e head [V][D]; 300+e head norm [D]. */
static float* tensor_ptr(orc_model* m, int tensor, int layer, int64_t* n) {
    const orc_desc* d = &m->d;
    const int64_t D = d->d_model;
    if (tensor == 100) { *n = (int64_t)d->vocab * D; return m->emb; }
    if (tensor >= 300 && tensor - 300 < d->n_exits) { *n = D; return m->head_norm[tensor - 300]; }
    if (tensor >= 200 && tensor - 200 < d->n_exits) { *n = (int64_t)d->vocab * D; return m->head[tensor - 200]; }
    if (layer < 1 || layer > m->loaded) return NULL;
    const int i = layer - 1;
    switch (tensor) {
        case 0: *n = D; return m->attn_norm[i];
        case 1: *n = (int64_t)(m->dq + 2 * m->dkv) * D; return m->wqkv[i];
        case 2: *n = D * m->dq; return m->wo[i];
        case 3: *n = D; return m->mlp_norm[i];
        case 4: *n = (int64_t)m->up_rows * D; return m->wup[i];
        case 5: *n = D * d->d_ffn; return m->wdown[i];
        default: return NULL;
    }
}

int64_t orc_tensor_get(orc_model* m, int tensor, int layer, float* out, int64_t n) {
    int64_t have = 0;
    const float* p = tensor_ptr(m, tensor, layer, &have);
    if (!p) return fail("no such tensor (or layer not loaded)");
    if (out) memcpy(out, p, sizeof(float) * (size_t)(n < have ? n : have));
    return have;
}

/* Replace a tensor (values rounded to the model dtype, as the device stores them). */
int orc_tensor_set(orc_model* m, int tensor, int layer, const float* src, int64_t n) {
    int64_t have = 0;
    float* p = tensor_ptr(m, tensor, layer, &have);
    if (!p) return fail("no such tensor (or layer not loaded)");
    if (n != have) return fail("tensor size mismatch");
    const int norm = tensor == 0 || tensor == 3 || tensor >= 300;
    for (int64_t i = 0; i < n; ++i) p[i] = norm ? src[i] : rnd(m, src[i]);
    return 0;
}

/* ---------------------------------------------------------------------------
 * The step.
 * ------------------------------------------------------------------------- */
/* y[r][n] = sum_k W[n][k] * X[r][k] for the live rows, f64 accumulation. */
typedef struct { const float* W; const float* X; float* Y; int N, K, rows; } mv_ctx;
static void mv_range(void* p, int64_t lo, int64_t hi) {
    mv_ctx* c = (mv_ctx*)p;
    for (int64_t n = lo; n < hi; ++n) {
        const float* w = c->W + (size_t)n * c->K;
        for (int r = 0; r < c->rows; ++r) {
            const float* x = c->X + (size_t)r * c->K;
            double s = 0.0;
            for (int k = 0; k < c->K; ++k) s += (double)w[k] * (double)x[k];
            c->Y[(size_t)r * c->N + n] = (float)s;
        }
    }
}
static void matvec(const orc_model* m, const float* W, const float* X, float* Y, int N, int K, int rows) {
    mv_ctx c = {W, X, Y, N, K, rows};
    par_for(m->threads, N, mv_range, &c);
}

static void rmsnorm(const orc_model* m, const float* x, const float* g, float* out) {
    const int D = m->d.d_model;
    double ss = 0.0;
    for (int c = 0; c < D; ++c) ss += (double)x[c] * x[c];
    float inv = (float)(1.0 / sqrt(ss / D + (double)m->d.norm_eps));
    for (int c = 0; c < D; ++c) out[c] = rnd(m, x[c] * inv * g[c]);
}

static void rope(const orc_model* m, const float* in, float* out, int pos) {
    const int hd = m->hd, half = hd / 2;
    const float* cs = m->rcos + (size_t)pos * half;
    const float* sn = m->rsin + (size_t)pos * half;
    for (int j = 0; j < half; ++j) {
        out[j] = in[j] * cs[j] - in[j + half] * sn[j];
        out[j + half] = in[j] * sn[j] + in[j + half] * cs[j];
    }
}

/* attention for one row at layer l (1-indexed); qkv row in, attn row out. */
static void attend(orc_model* m, int l, int slot, int pos, const float* qkv, float* out) {
    const orc_desc* d = &m->d;
    const int hd = m->hd, H = d->n_heads, Hkv = d->n_kv_heads, G = H / Hkv, S = d->max_seq_len;
    const size_t layer_off = (size_t)(l - 1) * d->max_slots * Hkv * S * hd;
    float q[128], k[128];
    double* sc = (double*)malloc(sizeof(double) * (size_t)(pos + 1));
    for (int g = 0; g < Hkv; ++g) {
        float* kc = m->kc + layer_off + ((size_t)slot * Hkv + g) * S * hd;
        float* vc = m->vc + layer_off + ((size_t)slot * Hkv + g) * S * hd;
        rope(m, qkv + m->dq + g * hd, k, pos);
        for (int j = 0; j < hd; ++j) {
            kc[(size_t)pos * hd + j] = rnd(m, k[j]);
            vc[(size_t)pos * hd + j] = rnd(m, qkv[m->dq + m->dkv + g * hd + j]);
        }
        for (int h = g * G; h < (g + 1) * G; ++h) {
            rope(m, qkv + h * hd, q, pos);
            double mx = -INFINITY;
            for (int p = 0; p <= pos; ++p) {
                int valid = p == pos || m->kv_depth[(size_t)slot * S + p] >= l;
                if (!valid) { sc[p] = -INFINITY; continue; }
                double s = 0.0;
                for (int j = 0; j < hd; ++j) s += (double)q[j] * kc[(size_t)p * hd + j];
                s /= sqrt((double)hd);
                sc[p] = s;
                if (s > mx) mx = s;
            }
            double lsum = 0.0;
            for (int p = 0; p <= pos; ++p) { sc[p] = sc[p] == -INFINITY ? 0.0 : exp(sc[p] - mx); lsum += sc[p]; }
            for (int j = 0; j < hd; ++j) {
                double o = 0.0;
                for (int p = 0; p <= pos; ++p) if (sc[p] != 0.0) o += sc[p] * vc[(size_t)p * hd + j];
                out[h * hd + j] = rnd(m, (float)(o / lsum));
            }
        }
    }
    free(sc);
}

typedef struct { int tok; float conf, logp; } head_obs;

static head_obs reduce_logits(const float* lg, int V) {
    float mx = lg[0];
    int am = 0;
    for (int v = 1; v < V; ++v) if (lg[v] > mx) { mx = lg[v]; am = v; }  /* ties -> lowest id */
    double s = 0.0;
    for (int v = 0; v < V; ++v) s += exp((double)lg[v] - mx);
    head_obs o = {am, (float)(1.0 / s), (float)(-log(s))};
    return o;
}

int orc_decode_step(orc_model* m, int depth, int policy, float th, int batch, const int32_t* slots,
                    const int32_t* tokens, const int32_t* positions, orc_out* out) {
    const orc_desc* d = &m->d;
    const int L = d->num_layers, D = d->d_model, F = d->d_ffn, V = d->vocab, NE = d->n_exits;
    const int S = d->max_seq_len;
    if (batch <= 0) return fail("empty batch");
    int run = L, heads[64], nh = 0;
    if (policy == 0) {
        int e_used = -1;
        for (int e = 0; e < NE; ++e) if (d->exit_layers[e] <= depth) e_used = e;
        if (e_used < 0) return fail("no observation at or below the serving depth");
        heads[nh++] = e_used;
        run = depth;
    } else if (policy == 2) {
        heads[nh++] = NE - 1;
    } else {
        for (int e = 0; e < NE; ++e) heads[nh++] = e;
    }
    if (m->loaded < run) return fail("layers not loaded");

    float* x = (float*)malloc(sizeof(float) * (size_t)batch * D);
    float* hn = (float*)malloc(sizeof(float) * (size_t)batch * (F > D ? F : D) * 2);
    float* qkv = (float*)malloc(sizeof(float) * (size_t)batch * (m->dq + 2 * m->dkv));
    float* att = (float*)malloc(sizeof(float) * (size_t)batch * m->dq);
    float* up = (float*)malloc(sizeof(float) * (size_t)batch * m->up_rows);
    float* y = (float*)malloc(sizeof(float) * (size_t)batch * (D > V ? D : V));
    int* live = (int*)malloc(sizeof(int) * batch);   /* compact index -> caller row */
    int* bin = (int*)malloc(sizeof(int) * batch);
    int nl = batch;
    for (int i = 0; i < batch; ++i) {
        live[i] = i;
        for (int c = 0; c < D; ++c) x[(size_t)i * D + c] = m->emb[(size_t)tokens[i] * D + c];
    }
    int hi = 0;
    for (int l = 1; l <= run && nl > 0; ++l) {
        const int li = l - 1;
        for (int i = 0; i < nl; ++i) rmsnorm(m, x + (size_t)i * D, m->attn_norm[li], hn + (size_t)i * D);
        matvec(m, m->wqkv[li], hn, qkv, m->dq + 2 * m->dkv, D, nl);
        for (int i = 0; i < nl; ++i) {
            int r = live[i];
            attend(m, l, slots[r], positions[r], qkv + (size_t)i * (m->dq + 2 * m->dkv), att + (size_t)i * m->dq);
        }
        matvec(m, m->wo[li], att, y, D, m->dq, nl);
        for (size_t t = 0; t < (size_t)nl * D; ++t) x[t] += y[t];
        for (int i = 0; i < nl; ++i) rmsnorm(m, x + (size_t)i * D, m->mlp_norm[li], hn + (size_t)i * D);
        matvec(m, m->wup[li], hn, up, m->up_rows, D, nl);
        for (int i = 0; i < nl; ++i) {
            float* u = up + (size_t)i * m->up_rows;
            float* h = hn + (size_t)i * F;   /* reuse hn as the [nl, F] hidden buffer */
            for (int j = 0; j < F; ++j) {
                if (d->mlp_kind == 1) {
                    float g = u[2 * j], v = u[2 * j + 1];
                    h[j] = rnd(m, (float)(g / (1.0 + exp(-(double)g))) * v);
                } else {
                    h[j] = rnd(m, u[j] > 0.f ? u[j] : 0.f);
                }
            }
        }
        matvec(m, m->wdown[li], hn, y, D, F, nl);
        for (size_t t = 0; t < (size_t)nl * D; ++t) x[t] += y[t];

        while (hi < nh && d->exit_layers[heads[hi]] == l) {
            const int e = heads[hi];
            const int is_final = hi + 1 == nh;
            for (int i = 0; i < nl; ++i) rmsnorm(m, x + (size_t)i * D, m->head_norm[e], hn + (size_t)i * D);
            matvec(m, m->head[e], hn, y, V, D, nl);
            int keep = 0;
            for (int i = 0; i < nl; ++i) {
                const int r = live[i];
                const float* lg = y + (size_t)i * V;
                if (out->logits_out) memcpy(out->logits_out + ((size_t)e * batch + r) * V, lg, sizeof(float) * V);
                head_obs o = reduce_logits(lg, V);
                int exit_layer = 0, brd = 0, unch = 2, done = 1;
                head_obs used = o;
                switch (policy) {
                    case 0: exit_layer = depth; brd = o.conf < th; unch = (is_final && d->exit_layers[e] == L) ? 1 : 2; break;
                    case 2: exit_layer = L; brd = 0; unch = 1; break;
                    case 1:
                        if (is_final) { exit_layer = d->exit_layers[e]; brd = o.conf < th; unch = 1; }
                        else if (o.conf >= th) { exit_layer = d->exit_layers[e]; brd = 0; unch = 2; }
                        else done = 0;
                        break;
                    default: {
                        out->head_token[(size_t)r * NE + e] = o.tok;
                        out->head_confidence[(size_t)r * NE + e] = o.conf;
                        out->head_logprob[(size_t)r * NE + e] = o.logp;
                        if (!is_final) { done = 0; break; }
                        orc_decision dec;
                        const int ex = orc_decide(1, NE, d->exit_layers, out->head_token + (size_t)r * NE,
                                                  out->head_confidence + (size_t)r * NE, th, depth, L, &dec);
                        used.tok = out->head_token[(size_t)r * NE + ex];
                        used.conf = out->head_confidence[(size_t)r * NE + ex];
                        used.logp = out->head_logprob[(size_t)r * NE + ex];
                        exit_layer = dec.exit_layer;
                        brd = dec.breached;
                        unch = dec.unchanged;
                        bin[r] = ex;
                        break;
                    }
                }
                if (policy == 3 && !is_final) { live[keep] = live[i]; memmove(x + (size_t)keep * D, x + (size_t)i * D, sizeof(float) * D); ++keep; continue; }
                if (!done) { live[keep] = live[i]; memmove(x + (size_t)keep * D, x + (size_t)i * D, sizeof(float) * D); ++keep; continue; }
                out->exit_layer[r] = exit_layer;
                out->token_id[r] = used.tok;
                out->confidence[r] = used.conf;
                out->logprob[r] = used.logp;
                out->breached[r] = (uint8_t)brd;
                out->unchanged[r] = (uint8_t)unch;
                if (policy != 3) bin[r] = e;
                if (policy != 1 || !is_final) { /* flat / full: rows continue to the serving depth */ }
                if (policy == 0 || policy == 2) { live[keep] = live[i]; memmove(x + (size_t)keep * D, x + (size_t)i * D, sizeof(float) * D); ++keep; }
            }
            nl = keep;
            ++hi;
        }
    }
    /* K4 restated: histogram over head bins, breach count, ordered logprob sum; KV depth map. */
    for (int e = 0; e < NE; ++e) out->hist[e] = 0;
    int64_t nb = 0;
    double sl = 0.0;
    for (int r = 0; r < batch; ++r) {
        out->hist[bin[r]] += 1;
        nb += out->breached[r];
        sl += (double)out->logprob[r];
        m->kv_depth[(size_t)slots[r] * S + positions[r]] = (uint8_t)(policy == 3 ? L : out->exit_layer[r]);
    }
    *out->n_breached = nb;
    *out->sum_logprob = sl;
    free(x); free(hn); free(qkv); free(att); free(up); free(y); free(live); free(bin);
    return 0;
}

int orc_read_kv(const orc_model* m, int layer, int slot, int pos, float* k, float* v) {
    const orc_desc* d = &m->d;
    const int hd = m->hd, Hkv = d->n_kv_heads, S = d->max_seq_len;
    const size_t layer_off = (size_t)(layer - 1) * d->max_slots * Hkv * S * hd;
    for (int g = 0; g < Hkv; ++g)
        for (int j = 0; j < hd; ++j) {
            size_t o = layer_off + (((size_t)slot * Hkv + g) * S + pos) * hd + j;
            if (k) k[g * hd + j] = m->kc[o];
            if (v) v[g * hd + j] = m->vc[o];
        }
    return 0;
}

/* Test hook: import K/V for positions [pos0, pos0 + n) of one slot at one
 * layer ([n][Hkv*hd] each, rounded to the model dtype) and raise those
 * positions' KV depth to `layer`.  Used to start the oracle from the GPU's
 * prefilled KV (tests/test_gpu_bench_parity.py) — the prefill itself is
 * checked independently on its first positions. */
int orc_write_kv(orc_model* m, int layer, int slot, int pos0, int n, const float* k, const float* v) {
    const orc_desc* d = &m->d;
    const int hd = m->hd, Hkv = d->n_kv_heads, S = d->max_seq_len;
    if (layer < 1 || layer > d->num_layers || slot < 0 || slot >= d->max_slots || pos0 < 0 || pos0 + n > S)
        return fail("kv coordinate out of range");
    const size_t layer_off = (size_t)(layer - 1) * d->max_slots * Hkv * S * hd;
    for (int q = 0; q < n; ++q) {
        for (int g = 0; g < Hkv; ++g)
            for (int j = 0; j < hd; ++j) {
                const size_t o = layer_off + (((size_t)slot * Hkv + g) * S + pos0 + q) * hd + j;
                const size_t i = (size_t)q * Hkv * hd + (size_t)g * hd + j;
                m->kc[o] = rnd(m, k[i]);
                m->vc[o] = rnd(m, v[i]);
            }
        uint8_t* dep = &m->kv_depth[(size_t)slot * S + pos0 + q];
        if (*dep < layer) *dep = (uint8_t)layer;
    }
    return 0;
}

/* CPU-baseline hook: fill positions [0, n) of one slot at every layer with
 * deterministic pseudo-random K/V in [-1, 1) (rounded to the dtype) computed
 * to full depth — a prompt's KV without running the prompt, so a timed decode
 * step attends over the same context length as the GPU workload. */
int orc_fill_kv_synthetic(orc_model* m, int slot, int n, uint64_t seed) {
    const orc_desc* d = &m->d;
    const int hd = m->hd, Hkv = d->n_kv_heads, S = d->max_seq_len, L = d->num_layers;
    if (slot < 0 || slot >= d->max_slots || n < 0 || n > S) return fail("kv coordinate out of range");
    for (int l = 0; l < L; ++l)
        for (int g = 0; g < Hkv; ++g)
            for (int p = 0; p < n; ++p)
                for (int j = 0; j < hd; ++j) {
                    const size_t o = (((size_t)l * d->max_slots + slot) * Hkv + g) * S * hd + (size_t)p * hd + j;
                    const uint64_t h = fin64(seed ^ (o * 0x9E3779B97F4A7C15ull));
                    m->kc[o] = rnd(m, (float)((h >> 40) * (1.0 / 8388608.0) - 1.0));
                    m->vc[o] = rnd(m, (float)(((h >> 16) & 0xFFFFFF) * (1.0 / 8388608.0) - 1.0));
                }
    for (int p = 0; p < n; ++p) m->kv_depth[(size_t)slot * S + p] = (uint8_t)L;
    return 0;
}
