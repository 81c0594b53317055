/* cascade_oracle.c — CPU oracle of the MoE verification step.
 *
 * TEST INFRASTRUCTURE ONLY (see cascade_oracle.h): loaded by tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline legs as the checker;
 * never linked into or called by the product library.
 *
 * fp64 accumulation everywhere; bf16 rounding exactly where the device
 * rounds; ties to the lower index.  Reference anchors (all under
 * /root/reference/proj/include/specsim/):
 *   top-k distinct experts per token ........ expert_model.hpp:100-112
 *   union popcount + shared ................. expert_model.hpp:120-139
 *   causal-prefix acceptance ................ workload.hpp:80-86
 *   truncation to the offered K ............. trace.hpp:69-74
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off -pthread).
 */
#include "cascade_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "cascade_weights.h"

#define NKINDS 15

struct orc_model {
    cascade_geometry g;
    uint64_t seed;
    int nthreads;
    int L, E, k, S, d, f, H, KV, hd, V, hq, nexp;
    uint16_t** cache; /* [NKINDS][L][nexp] */
    uint64_t cached;
};

/* ------------------------------------------------------------ threads */
typedef void (*range_fn)(void* ctx, long lo, long hi);
typedef struct {
    range_fn fn;
    void* ctx;
    long lo, hi;
} job_t;

static void* job_main(void* a) {
    job_t* j = (job_t*)a;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

static void parallel_for(int nthreads, long n, range_fn fn, void* ctx) {
    if (nthreads <= 1 || n < 2) {
        fn(ctx, 0, n);
        return;
    }
    if (nthreads > n) nthreads = (int)n;
    pthread_t th[256];
    job_t jobs[256];
    if (nthreads > 256) nthreads = 256;
    for (int i = 0; i < nthreads; ++i) {
        jobs[i].fn = fn;
        jobs[i].ctx = ctx;
        jobs[i].lo = n * i / nthreads;
        jobs[i].hi = n * (i + 1) / nthreads;
        if (i > 0) pthread_create(&th[i], NULL, job_main, &jobs[i]);
    }
    job_main(&jobs[0]);
    for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------ numerics */
static inline double bf(uint16_t b) { return (double)cascade_bf16_to_f32(b); }

/* correctly rounded double -> bf16 (RNE) */
static uint16_t d2bf(double v) {
    float f = (float)v;
    union { float f; uint32_t u; } c;
    c.f = f;
    if ((c.u & 0xFFFFu) == 0x8000u) {
        const double diff = v - (double)f;
        if (diff != 0.0) {
            const int away = (diff > 0.0) == (f > 0.0);
            return (uint16_t)((c.u >> 16) + (away ? 1u : 0u));
        }
    }
    return cascade_f32_to_bf16(f);
}

/* ------------------------------------------------------------ weights */
static void shape_of(const orc_model* m, int kind, int* rows, int* cols) {
    switch (kind) {
    case CASCADE_T_EMBED: *rows = m->V; *cols = m->d; break;
    case CASCADE_T_ATTN_NORM:
    case CASCADE_T_FFN_NORM:
    case CASCADE_T_FINAL_NORM: *rows = 1; *cols = m->d; break;
    case CASCADE_T_WQ: *rows = m->hq; *cols = m->d; break;
    case CASCADE_T_WK:
    case CASCADE_T_WV: *rows = m->KV * m->hd; *cols = m->d; break;
    case CASCADE_T_WO: *rows = m->d; *cols = m->hq; break;
    case CASCADE_T_ROUTER: *rows = m->E; *cols = m->d; break;
    case CASCADE_T_SHARED_GATE: *rows = 1; *cols = m->d; break;
    case CASCADE_T_W_GATE:
    case CASCADE_T_W_UP: *rows = m->f; *cols = m->d; break;
    case CASCADE_T_W_DOWN: *rows = m->d; *cols = m->f; break;
    case CASCADE_T_LM_HEAD: *rows = m->V; *cols = m->d; break;
    default: *rows = 0; *cols = 0;
    }
}

typedef struct {
    uint16_t* out;
    uint64_t key;
    float scale;
    int cols;
    long row0;
} gen_ctx;

static void gen_range(void* c, long lo, long hi) {
    gen_ctx* g = (gen_ctx*)c;
    for (long r = lo; r < hi; ++r) {
        uint16_t* o = g->out + r * g->cols;
        const uint64_t base = (uint64_t)(g->row0 + r) * (uint64_t)g->cols;
        for (int c2 = 0; c2 < g->cols; ++c2) o[c2] = cascade_weight_bits(g->key, base + (uint64_t)c2, g->scale);
    }
}

static int gen_rows(orc_model* m, int kind, int layer, int expert, int row0, int nrows, uint16_t* out) {
    int rows, cols;
    shape_of(m, kind, &rows, &cols);
    if (rows == 0 || row0 < 0 || row0 + nrows > rows) return -1;
    gen_ctx c;
    c.out = out;
    c.key = cascade_tensor_key(m->seed, cascade_tensor_id(kind, layer, expert));
    c.scale = cascade_kind_scale(kind, cols, m->g.router_scale);
    c.cols = cols;
    c.row0 = row0;
    parallel_for(m->nthreads, nrows, gen_range, &c);
    return 0;
}

static const uint16_t* W(orc_model* m, int kind, int layer, int expert) {
    if (kind == CASCADE_T_EMBED || kind == CASCADE_T_FINAL_NORM || kind == CASCADE_T_LM_HEAD) layer = 0;
    if (kind != CASCADE_T_W_GATE && kind != CASCADE_T_W_UP && kind != CASCADE_T_W_DOWN) expert = 0;
    const long idx = ((long)kind * m->L + layer) * m->nexp + expert;
    if (m->cache[idx]) return m->cache[idx];
    int rows, cols;
    shape_of(m, kind, &rows, &cols);
    uint16_t* p = (uint16_t*)malloc((size_t)rows * cols * 2);
    if (!p) return NULL;
    gen_rows(m, kind, layer, expert, 0, rows, p);
    m->cache[idx] = p;
    m->cached += (uint64_t)rows * cols * 2;
    return p;
}

orc_model* orc_model_create(const cascade_geometry* g, uint64_t seed, int nthreads) {
    if (!g || g->num_layers < 1 || g->experts_per_layer < 1 || g->top_k < 1 || g->top_k > g->experts_per_layer ||
        g->experts_per_layer > 128 || g->top_k > 16 || g->shared_experts < 0 || g->d_model < 1 || g->d_ff < 1 ||
        g->n_heads < 1 || g->n_kv_heads < 1 || g->n_heads % g->n_kv_heads || g->head_dim < 2 || g->head_dim % 2 ||
        g->vocab < 2)
        return NULL;
    orc_model* m = (orc_model*)calloc(1, sizeof(orc_model));
    m->g = *g;
    m->seed = seed;
    m->nthreads = nthreads < 1 ? 1 : nthreads;
    m->L = g->num_layers;
    m->E = g->experts_per_layer;
    m->k = g->top_k;
    m->S = g->shared_experts;
    m->d = g->d_model;
    m->f = g->d_ff;
    m->H = g->n_heads;
    m->KV = g->n_kv_heads;
    m->hd = g->head_dim;
    m->V = g->vocab;
    m->hq = m->H * m->hd;
    m->nexp = m->E + m->S;
    m->cache = (uint16_t**)calloc((size_t)NKINDS * m->L * m->nexp, sizeof(uint16_t*));
    return m;
}

void orc_model_drop_cache(orc_model* m) {
    if (!m) return;
    const long n = (long)NKINDS * m->L * m->nexp;
    for (long i = 0; i < n; ++i) {
        free(m->cache[i]);
        m->cache[i] = NULL;
    }
    m->cached = 0;
}

void orc_model_destroy(orc_model* m) {
    if (!m) return;
    orc_model_drop_cache(m);
    free(m->cache);
    free(m);
}

uint64_t orc_cached_bytes(const orc_model* m) { return m ? m->cached : 0; }

int orc_tensor(orc_model* m, int kind, int layer, int expert, int row0, int nrows, uint16_t* out) {
    if (!m || !out) return -1;
    if (kind == CASCADE_T_EMBED || kind == CASCADE_T_FINAL_NORM || kind == CASCADE_T_LM_HEAD) layer = 0;
    if (kind != CASCADE_T_W_GATE && kind != CASCADE_T_W_UP && kind != CASCADE_T_W_DOWN) expert = 0;
    return gen_rows(m, kind, layer, expert, row0, nrows, out);
}

int orc_prepare_layer(orc_model* m, int layer, const int32_t* experts, int n) {
    if (!m || layer < 0 || layer >= m->L) return -1;
    const int kinds[] = {CASCADE_T_ATTN_NORM, CASCADE_T_FFN_NORM, CASCADE_T_WQ, CASCADE_T_WK,
                         CASCADE_T_WV, CASCADE_T_WO, CASCADE_T_ROUTER};
    for (unsigned i = 0; i < sizeof(kinds) / sizeof(kinds[0]); ++i)
        if (!W(m, kinds[i], layer, 0)) return -2;
    for (int i = 0; i < n; ++i) {
        if (experts[i] < 0 || experts[i] >= m->nexp) return -1;
        if (!W(m, CASCADE_T_W_GATE, layer, experts[i]) || !W(m, CASCADE_T_W_UP, layer, experts[i]) ||
            !W(m, CASCADE_T_W_DOWN, layer, experts[i]))
            return -2;
    }
    return 0;
}

/* ------------------------------------------------------------ linear */
/* y[t][r] = sum_c Wm[r][c] * x[t][c]   (Wm bf16 [rows][cols], x double [T][cols]) */
typedef struct {
    const uint16_t* w;
    const double* x;
    double* y;
    int rows, cols, T;
} lin_ctx;

static void lin_range(void* c, long lo, long hi) {
    lin_ctx* l = (lin_ctx*)c;
    double* wr = (double*)malloc((size_t)l->cols * sizeof(double));
    for (long r = lo; r < hi; ++r) {
        const uint16_t* w = l->w + r * l->cols;
        for (int c2 = 0; c2 < l->cols; ++c2) wr[c2] = bf(w[c2]);
        for (int t = 0; t < l->T; ++t) {
            const double* x = l->x + (long)t * l->cols;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            int c2 = 0;
            for (; c2 + 4 <= l->cols; c2 += 4) {
                a0 += wr[c2] * x[c2];
                a1 += wr[c2 + 1] * x[c2 + 1];
                a2 += wr[c2 + 2] * x[c2 + 2];
                a3 += wr[c2 + 3] * x[c2 + 3];
            }
            for (; c2 < l->cols; ++c2) a0 += wr[c2] * x[c2];
            l->y[(long)t * l->rows + r] = (a0 + a1) + (a2 + a3);
        }
    }
    free(wr);
}

static void linear(orc_model* m, const uint16_t* w, int rows, int cols, const double* x, int T, double* y) {
    lin_ctx c = {w, x, y, rows, cols, T};
    parallel_for(m->nthreads, rows, lin_range, &c);
}

/* ------------------------------------------------------------ stages */
static void rmsnorm_d(const orc_model* m, const uint16_t* w, const double* x, int T, uint16_t* out) {
    (void)m;
    const int d = m->d;
    for (int t = 0; t < T; ++t) {
        const double* xr = x + (long)t * d;
        double ss = 0;
        for (int i = 0; i < d; ++i) ss += xr[i] * xr[i];
        const double r = 1.0 / sqrt(ss / d + (double)m->g.norm_eps);
        for (int i = 0; i < d; ++i) out[(long)t * d + i] = d2bf(xr[i] * r * bf(w[i]));
    }
}

int orc_rmsnorm(orc_model* m, int kind, int layer, const float* x, int T, uint16_t* out) {
    if (!m || !x || !out || T < 1) return -1;
    if (kind != CASCADE_T_ATTN_NORM && kind != CASCADE_T_FFN_NORM && kind != CASCADE_T_FINAL_NORM) return -1;
    const uint16_t* w = W(m, kind, layer, 0);
    double* xd = (double*)malloc((size_t)T * m->d * sizeof(double));
    for (long i = 0; i < (long)T * m->d; ++i) xd[i] = x[i];
    rmsnorm_d(m, w, xd, T, out);
    free(xd);
    return 0;
}

static double* bf_to_d(const uint16_t* a, long n) {
    double* o = (double*)malloc((size_t)n * sizeof(double));
    for (long i = 0; i < n; ++i) o[i] = bf(a[i]);
    return o;
}

int orc_router(orc_model* m, int layer, const uint16_t* xn, int T, double* logits, int32_t* topk, double* topw,
               double* gsh, double* margin) {
    if (!m || !xn || T < 1) return -1;
    const int E = m->E, k = m->k, ne = E + 1;
    double* x = bf_to_d(xn, (long)T * m->d);
    double* lg = (double*)malloc((size_t)T * E * sizeof(double));
    linear(m, W(m, CASCADE_T_ROUTER, layer, 0), E, m->d, x, T, lg);
    double* sg = NULL;
    if (m->g.shared_gate) {
        sg = (double*)malloc((size_t)T * sizeof(double));
        linear(m, W(m, CASCADE_T_SHARED_GATE, layer, 0), 1, m->d, x, T, sg);
    }
    for (int t = 0; t < T; ++t) {
        const double* l = lg + (long)t * E;
        if (logits) {
            for (int e = 0; e < E; ++e) logits[(long)t * ne + e] = l[e];
            logits[(long)t * ne + E] = sg ? sg[t] : 0.0;
        }
        double mx = l[0];
        for (int e = 1; e < E; ++e) mx = l[e] > mx ? l[e] : mx;
        double z = 0;
        for (int e = 0; e < E; ++e) z += exp(l[e] - mx);
        unsigned char taken[128] = {0};
        int ids[16];
        double zk = 0;
        for (int r = 0; r < k; ++r) {
            int bi = -1;
            for (int e = 0; e < E; ++e)
                if (!taken[e] && (bi < 0 || l[e] > l[bi])) bi = e; /* strict > keeps the lower index */
            taken[bi] = 1;
            ids[r] = bi;
            zk += exp(l[bi] - mx);
        }
        for (int r = 0; r < k; ++r) {
            if (topk) topk[t * k + r] = ids[r];
            if (topw) topw[t * k + r] = exp(l[ids[r]] - mx) / (m->g.renormalize_topk ? zk : z);
        }
        if (gsh) gsh[t] = sg ? 1.0 / (1.0 + exp(-sg[t])) : 1.0;
        if (margin) {
            /* smallest logit gap that decides the set or the rank order */
            double mg = INFINITY;
            for (int r = 0; r + 1 < k; ++r) {
                const double gp = l[ids[r]] - l[ids[r + 1]];
                mg = gp < mg ? gp : mg;
            }
            int bo = -1;
            for (int e = 0; e < E; ++e)
                if (!taken[e] && (bo < 0 || l[e] > l[bo])) bo = e;
            if (bo >= 0) {
                const double gp = l[ids[k - 1]] - l[bo];
                mg = gp < mg ? gp : mg;
            }
            margin[t] = mg;
        }
    }
    free(sg);
    free(lg);
    free(x);
    return 0;
}

int orc_union(const int32_t* topk, int T, int k, int32_t* uniq) {
    uint64_t m0 = 0, m1 = 0;
    for (int i = 0; i < T * k; ++i) {
        const int e = topk[i];
        if (e < 64) m0 |= 1ull << e;
        else m1 |= 1ull << (e - 64);
    }
    int n = 0;
    for (int e = 0; e < 128; ++e)
        if (e < 64 ? ((m0 >> e) & 1ull) : ((m1 >> (e - 64)) & 1ull)) {
            if (uniq) uniq[n] = e;
            ++n;
        }
    return n;
}

/* one expert block over the tokens routed to it: y[n][d] */
static void expert_ffn(orc_model* m, int layer, int e, const double* x, int n, double* y) {
    const int f = m->f, d = m->d;
    double* g = (double*)malloc((size_t)n * f * sizeof(double));
    double* u = (double*)malloc((size_t)n * f * sizeof(double));
    linear(m, W(m, CASCADE_T_W_GATE, layer, e), f, d, x, n, g);
    linear(m, W(m, CASCADE_T_W_UP, layer, e), f, d, x, n, u);
    for (long i = 0; i < (long)n * f; ++i) {
        const double s = g[i] / (1.0 + exp(-g[i]));
        g[i] = bf(d2bf(s * u[i]));
    }
    linear(m, W(m, CASCADE_T_W_DOWN, layer, e), d, f, g, n, y);
    free(g);
    free(u);
}

int orc_moe(orc_model* m, int layer, const uint16_t* xn, int T, const int32_t* topk, const double* topw,
            const double* gsh, double* out) {
    if (!m || !xn || !topk || !topw || !out || T < 1) return -1;
    const int d = m->d, k = m->k;
    double* x = bf_to_d(xn, (long)T * d);
    double* xs = (double*)malloc((size_t)T * k * d * sizeof(double));
    double* ys = (double*)malloc((size_t)T * k * d * sizeof(double));
    double* routed = (double*)calloc((size_t)T * k * d, sizeof(double)); /* [t][r][d] */
    int32_t uniq[128];
    const int U = orc_union(topk, T, k, uniq);
    for (int ui = 0; ui < U; ++ui) {
        const int e = uniq[ui];
        int* toks = (int*)malloc((size_t)T * k * sizeof(int));
        int* ranks = (int*)malloc((size_t)T * k * sizeof(int));
        int n = 0;
        for (int t = 0; t < T; ++t)
            for (int r = 0; r < k; ++r)
                if (topk[t * k + r] == e) {
                    toks[n] = t;
                    ranks[n] = r;
                    memcpy(xs + (long)n * d, x + (long)t * d, d * sizeof(double));
                    ++n;
                }
        expert_ffn(m, layer, e, xs, n, ys);
        for (int i = 0; i < n; ++i)
            memcpy(routed + ((long)toks[i] * k + ranks[i]) * d, ys + (long)i * d, d * sizeof(double));
        free(toks);
        free(ranks);
    }
    double* shared = NULL;
    if (m->S > 0) {
        shared = (double*)calloc((size_t)T * d, sizeof(double));
        for (int b = 0; b < m->S; ++b) {
            expert_ffn(m, layer, m->E + b, x, T, ys);
            for (long i = 0; i < (long)T * d; ++i) shared[i] += ys[i];
        }
    }
    for (int t = 0; t < T; ++t)
        for (int i = 0; i < d; ++i) {
            double a = 0;
            for (int r = 0; r < k; ++r) a += topw[t * k + r] * routed[((long)t * k + r) * d + i];
            if (shared) a += (gsh ? gsh[t] : 1.0) * shared[(long)t * d + i];
            out[(long)t * d + i] = a;
        }
    free(shared);
    free(routed);
    free(ys);
    free(xs);
    free(x);
    return 0;
}

static void rope(double* v, int hd, int pos, double theta) {
    const int h = hd / 2;
    for (int i = 0; i < h; ++i) {
        const double inv = pow(theta, -2.0 * (double)i / (double)hd);
        const double a = (double)pos * inv;
        const double c = cos(a), s = sin(a);
        const double x0 = v[i], x1 = v[i + h];
        v[i] = x0 * c - x1 * s;
        v[i + h] = x1 * c + x0 * s;
    }
}

static int attention_d(orc_model* m, int layer, const double* xd, int T, int ctx, const uint16_t* kc,
                       const uint16_t* vc, int kc_stride, double* out, uint16_t* k_new, uint16_t* v_new) {
    const int d = m->d, H = m->H, KV = m->KV, hd = m->hd, G = H / KV;
    uint16_t* xn = (uint16_t*)malloc((size_t)T * d * 2);
    rmsnorm_d(m, W(m, CASCADE_T_ATTN_NORM, layer, 0), xd, T, xn);
    double* x = bf_to_d(xn, (long)T * d);
    double* q = (double*)malloc((size_t)T * H * hd * sizeof(double));
    double* kk = (double*)malloc((size_t)T * KV * hd * sizeof(double));
    double* vv = (double*)malloc((size_t)T * KV * hd * sizeof(double));
    linear(m, W(m, CASCADE_T_WQ, layer, 0), H * hd, d, x, T, q);
    linear(m, W(m, CASCADE_T_WK, layer, 0), KV * hd, d, x, T, kk);
    linear(m, W(m, CASCADE_T_WV, layer, 0), KV * hd, d, x, T, vv);
    const double theta = (double)m->g.rope_theta;
    for (int t = 0; t < T; ++t) {
        for (int h = 0; h < H; ++h) rope(q + ((long)t * H + h) * hd, hd, ctx + t, theta);
        for (int h = 0; h < KV; ++h) {
            rope(kk + ((long)t * KV + h) * hd, hd, ctx + t, theta);
            for (int i = 0; i < hd; ++i) {
                const uint16_t kb = d2bf(kk[((long)t * KV + h) * hd + i]);
                const uint16_t vb = d2bf(vv[((long)t * KV + h) * hd + i]);
                kk[((long)t * KV + h) * hd + i] = bf(kb);
                vv[((long)t * KV + h) * hd + i] = bf(vb);
                if (k_new) k_new[((long)h * T + t) * hd + i] = kb;
                if (v_new) v_new[((long)h * T + t) * hd + i] = vb;
            }
        }
    }
    /* Device precision contract (attention.cuh): K/V are bf16 in the cache,
     * q and P enter the tensor cores as two-term (hi + lo) bf16 pairs, i.e.
     * the softmax is fp32-accurate; the attention output is rounded to bf16
     * for the O projection.  The oracle therefore computes an exact (fp64)
     * softmax over the bf16 keys/values and rounds only the output. */
    const double scale = 1.0 / sqrt((double)hd);
    double* o = (double*)malloc((size_t)T * H * hd * sizeof(double));
    double* sc = (double*)malloc((size_t)(ctx + T) * sizeof(double));
    for (int t = 0; t < T; ++t)
        for (int h = 0; h < H; ++h) {
            const int kvh = h / G;
            const double* qv = q + ((long)t * H + h) * hd;
            const int n = ctx + t + 1;
            double mx = -INFINITY;
            for (int j = 0; j < n; ++j) {
                double s2 = 0;
                if (j < ctx) {
                    const uint16_t* kr = kc + ((long)kvh * kc_stride + j) * hd;
                    for (int i = 0; i < hd; ++i) s2 += qv[i] * bf(kr[i]);
                } else {
                    const double* kr = kk + ((long)(j - ctx) * KV + kvh) * hd;
                    for (int i = 0; i < hd; ++i) s2 += qv[i] * kr[i];
                }
                sc[j] = s2 * scale;
                mx = sc[j] > mx ? sc[j] : mx;
            }
            double z = 0;
            for (int j = 0; j < n; ++j) {
                sc[j] = exp(sc[j] - mx);
                z += sc[j];
            }
            double* ov = o + ((long)t * H + h) * hd;
            for (int i = 0; i < hd; ++i) ov[i] = 0;
            for (int j = 0; j < n; ++j) {
                const double pj = sc[j] / z;
                if (j < ctx) {
                    const uint16_t* vr = vc + ((long)kvh * kc_stride + j) * hd;
                    for (int i = 0; i < hd; ++i) ov[i] += pj * bf(vr[i]);
                } else {
                    const double* vr = vv + ((long)(j - ctx) * KV + kvh) * hd;
                    for (int i = 0; i < hd; ++i) ov[i] += pj * vr[i];
                }
            }
            for (int i = 0; i < hd; ++i) ov[i] = bf(d2bf(ov[i])); /* O-proj input is bf16 */
        }
    linear(m, W(m, CASCADE_T_WO, layer, 0), d, H * hd, o, T, out);
    free(o);
    free(sc);
    free(vv);
    free(kk);
    free(q);
    free(x);
    free(xn);
    return 0;
}

int orc_attention(orc_model* m, int layer, const float* x, int T, int ctx, const uint16_t* kcache,
                  const uint16_t* vcache, double* out, uint16_t* k_new, uint16_t* v_new) {
    if (!m || !x || !out || T < 1 || ctx < 0 || (ctx > 0 && (!kcache || !vcache))) return -1;
    double* xd = (double*)malloc((size_t)T * m->d * sizeof(double));
    for (long i = 0; i < (long)T * m->d; ++i) xd[i] = x[i];
    const int rc = attention_d(m, layer, xd, T, ctx, kcache, vcache, ctx, out, k_new, v_new);
    free(xd);
    return rc;
}

static void argmax_rows(const double* lg, int T, int V, int32_t* am, double* margin) {
    for (int t = 0; t < T; ++t) {
        const double* l = lg + (long)t * V;
        int b = 0;
        for (int v = 1; v < V; ++v)
            if (l[v] > l[b]) b = v;
        if (am) am[t] = b;
        if (margin) {
            double s = -INFINITY;
            for (int v = 0; v < V; ++v)
                if (v != b && l[v] > s) s = l[v];
            margin[t] = l[b] - s;
        }
    }
}

int orc_lm_head(orc_model* m, const uint16_t* xn, int T, double* logits, int32_t* argmax, double* margin) {
    if (!m || !xn || T < 1) return -1;
    double* x = bf_to_d(xn, (long)T * m->d);
    double* lg = logits ? logits : (double*)malloc((size_t)T * m->V * sizeof(double));
    linear(m, W(m, CASCADE_T_LM_HEAD, 0, 0), m->V, m->d, x, T, lg);
    argmax_rows(lg, T, m->V, argmax, margin);
    if (!logits) free(lg);
    free(x);
    return 0;
}

int orc_greedy_accept(const int32_t* argmax, const int32_t* drafts, int K, int32_t* emitted) {
    int acc = 0;
    while (acc < K && argmax[acc] == drafts[acc]) {
        if (emitted) emitted[acc] = drafts[acc];
        ++acc;
    }
    if (emitted) emitted[acc] = argmax[acc];
    return acc;
}

/* ------------------------------------------------------------ session */
struct orc_session {
    orc_model* m;
    int max_ctx, len, pending;
    uint16_t* kc; /* [L][KV][max_ctx][hd] */
    uint16_t* vc;
    double min_router_margin; /* smallest router decision gap seen (flags near-ties) */
    int last_T;               /* routing of the last forward: [L][T][k] ids, [L][T] margins */
    int32_t* last_topk;
    double* last_margin;
};

orc_session* orc_session_create(orc_model* m, int max_ctx) {
    if (!m || max_ctx < 1) return NULL;
    orc_session* s = (orc_session*)calloc(1, sizeof(orc_session));
    s->m = m;
    s->max_ctx = max_ctx + 16;
    const size_t n = (size_t)m->L * m->KV * s->max_ctx * m->hd;
    s->kc = (uint16_t*)calloc(n, 2);
    s->vc = (uint16_t*)calloc(n, 2);
    s->min_router_margin = INFINITY;
    s->last_topk = (int32_t*)calloc((size_t)m->L * 64 * m->k, sizeof(int32_t));
    s->last_margin = (double*)calloc((size_t)m->L * 64, sizeof(double));
    return s;
}

void orc_session_destroy(orc_session* s) {
    if (!s) return;
    free(s->last_topk);
    free(s->last_margin);
    free(s->kc);
    free(s->vc);
    free(s);
}

int orc_cache_len(const orc_session* s) { return s ? s->len : -1; }

int orc_last_routing(const orc_session* s, int32_t* topk, double* margin) {
    if (!s) return -1;
    const int n = s->m->L * s->last_T;
    if (topk) memcpy(topk, s->last_topk, (size_t)n * s->m->k * sizeof(int32_t));
    if (margin) memcpy(margin, s->last_margin, (size_t)n * sizeof(double));
    return s->last_T;
}

double orc_min_router_margin(orc_session* s, int reset) {
    if (!s) return -1.0;
    const double v = s->min_router_margin;
    if (reset) s->min_router_margin = INFINITY;
    return v;
}

/* forward T tokens at positions len..len+T-1; writes their KV rows; logits
 * [T][V] of the final norm output */
static int forward(orc_session* s, const int32_t* toks, int T, double* logits, int32_t* union_sizes) {
    orc_model* m = s->m;
    const int d = m->d, hd = m->hd, KV = m->KV;
    if (s->len + T > s->max_ctx) return -1;
    double* x = (double*)malloc((size_t)T * d * sizeof(double));
    const uint16_t* emb = W(m, CASCADE_T_EMBED, 0, 0);
    for (int t = 0; t < T; ++t)
        for (int i = 0; i < d; ++i) x[(long)t * d + i] = bf(emb[(long)toks[t] * d + i]);
    double* a = (double*)malloc((size_t)T * d * sizeof(double));
    uint16_t* xn = (uint16_t*)malloc((size_t)T * d * 2);
    uint16_t* kn = (uint16_t*)malloc((size_t)KV * T * hd * 2);
    uint16_t* vn = (uint16_t*)malloc((size_t)KV * T * hd * 2);
    int32_t* topk = (int32_t*)malloc((size_t)T * m->k * sizeof(int32_t));
    double* topw = (double*)malloc((size_t)T * m->k * sizeof(double));
    double* gsh = (double*)malloc((size_t)T * sizeof(double));
    double* rmg = (double*)malloc((size_t)T * sizeof(double));
    for (int l = 0; l < m->L; ++l) {
        uint16_t* kc = s->kc + (size_t)l * KV * s->max_ctx * hd;
        uint16_t* vc = s->vc + (size_t)l * KV * s->max_ctx * hd;
        attention_d(m, l, x, T, s->len, kc, vc, s->max_ctx, a, kn, vn);
        for (int h = 0; h < KV; ++h)
            for (int t = 0; t < T; ++t) {
                memcpy(kc + ((size_t)h * s->max_ctx + s->len + t) * hd, kn + ((size_t)h * T + t) * hd, hd * 2);
                memcpy(vc + ((size_t)h * s->max_ctx + s->len + t) * hd, vn + ((size_t)h * T + t) * hd, hd * 2);
            }
        for (long i = 0; i < (long)T * d; ++i) x[i] += a[i];
        rmsnorm_d(m, W(m, CASCADE_T_FFN_NORM, l, 0), x, T, xn);
        orc_router(m, l, xn, T, NULL, topk, topw, gsh, rmg);
        for (int t = 0; t < T; ++t)
            if (rmg[t] < s->min_router_margin) s->min_router_margin = rmg[t];
        if (T <= 64) {
            s->last_T = T;
            memcpy(s->last_topk + (size_t)l * T * m->k, topk, (size_t)T * m->k * sizeof(int32_t));
            memcpy(s->last_margin + (size_t)l * T, rmg, (size_t)T * sizeof(double));
        }
        if (union_sizes) union_sizes[l] = orc_union(topk, T, m->k, NULL);
        orc_moe(m, l, xn, T, topk, topw, gsh, a);
        for (long i = 0; i < (long)T * d; ++i) x[i] += a[i];
    }
    rmsnorm_d(m, W(m, CASCADE_T_FINAL_NORM, 0, 0), x, T, xn);
    if (logits) {
        double* xx = bf_to_d(xn, (long)T * d);
        linear(m, W(m, CASCADE_T_LM_HEAD, 0, 0), m->V, d, xx, T, logits);
        free(xx);
    }
    free(rmg);
    free(gsh);
    free(topw);
    free(topk);
    free(vn);
    free(kn);
    free(xn);
    free(a);
    free(x);
    return 0;
}

int orc_prefill(orc_session* s, const int32_t* prompt, int n) {
    if (!s || !prompt || n < 1) return -1;
    int pos = 0;
    while (pos < n - 1) {
        const int T = (n - 1 - pos) < 16 ? (n - 1 - pos) : 16;
        if (forward(s, prompt + pos, T, NULL, NULL)) return -1;
        s->len += T;
        pos += T;
    }
    s->pending = prompt[n - 1];
    return 0;
}

int orc_verify(orc_session* s, const int32_t* drafts, int K, double* logits, int32_t* argmax, double* margin,
               int32_t* union_sizes) {
    if (!s || K < 0 || (K > 0 && !drafts)) return -1;
    const int T = K + 1;
    int32_t toks[64];
    if (T > 64) return -1;
    toks[0] = s->pending;
    for (int i = 0; i < K; ++i) toks[i + 1] = drafts[i];
    double* lg = logits ? logits : (double*)malloc((size_t)T * s->m->V * sizeof(double));
    if (forward(s, toks, T, lg, union_sizes)) {
        if (!logits) free(lg);
        return -1;
    }
    int32_t am[64];
    argmax_rows(lg, T, s->m->V, am, margin);
    if (argmax) memcpy(argmax, am, (size_t)T * sizeof(int32_t));
    const int acc = orc_greedy_accept(am, drafts, K, NULL);
    s->len += acc + 1;
    s->pending = am[acc];
    if (!logits) free(lg);
    return acc;
}
