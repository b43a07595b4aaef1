/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
 *
 * A plain-C, fp64 restatement of the reference hot path
 *   Pipeline::train_microbatch (shared-prompt branch)
 *   /root/reference/proj/src/pipeline.cpp:97-141
 * i.e. pack -> tri-model log-prob -> GRPO terms -> policy backward -> accumulate.
 *
 * Every function below cites the reference file:line whose arithmetic it
 * restates.  Loop orders mirror the reference so that, on the same libm, the
 * results are bit-identical to the reference build in oracle/_ref (checked by
 * tests/test_oracle.py); the reference's own known-answer tests are pinned by
 * tests/golden/ (see oracle/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "parl_oracle.h"

#ifndef M_SQRT1_2
#define M_SQRT1_2 0.70710678118654752440
#endif

/* ------------------------------------------------------------------------ */
/* RNG: splitmix64 / mix_seed / mt19937_64 / uniform / Box-Muller normal.   */
/* Restates proj/include/parl/rng.hpp:11-63 (std::mt19937_64 is specified   */
/* by the C++ standard; we implement the same recurrence).                  */

static uint64_t sm64(uint64_t x) { /* rng.hpp:13-18 */
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

uint64_t orc_mix_seed(uint64_t a, uint64_t b) { /* rng.hpp:20-22 */
    return sm64(sm64(a) ^ (0x9e3779b97f4a7c15ull + b));
}

typedef struct {
    uint64_t mt[312];
    int idx;
    double spare;
    int has_spare;
} orc_rng;

static void mt_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
    r->has_spare = 0;
    r->spare = 0.0;
}

static uint64_t mt_next(orc_rng* r) {
    const uint64_t UM = 0xffffffff80000000ull, LM = 0x7fffffffull;
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= 0xb5026f5aa96619e9ull;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71d67fffeda60000ull;
    y ^= (y << 37) & 0xfff7eee000000000ull;
    y ^= (y >> 43);
    return y;
}

static void rng_init(orc_rng* r, uint64_t seed) { mt_seed(r, sm64(seed)); } /* rng.hpp:31 */

static double rng_uniform(orc_rng* r) { /* rng.hpp:36 */
    return (double)(mt_next(r) >> 11) * 0x1.0p-53;
}

static double rng_normal(orc_rng* r) { /* rng.hpp:39-50 */
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = 1.0 - rng_uniform(r);
    double u2 = rng_uniform(r);
    double rad = sqrt(-2.0 * log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    r->spare = rad * sin(a);
    r->has_spare = 1;
    return rad * cos(a);
}



/* Deterministic stream helpers exposed for fixture generation. */
void orc_rng_stream(uint64_t seed, int n, int kind, double* out) {
    orc_rng r;
    rng_init(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = kind == 0 ? rng_uniform(&r) : rng_normal(&r);
}

/* ------------------------------------------------------------------------ */
/* Parameter layout: proj/src/model.cpp:86-114                               */

static int cfg_ok(const orc_cfg* c) { /* model.cpp:19-31 */
    if (c->vocab < 4 || c->d_model <= 0 || c->n_layers <= 0 || c->n_heads <= 0 || c->d_ff <= 0 ||
        c->max_seq <= 0 || c->d_model % c->n_heads != 0)
        return 0;
    return 1;
}

void orc_layout(const orc_cfg* c, orc_layout_t* L) {
    size_t o = 0;
    const size_t d = (size_t)c->d_model, F = (size_t)c->d_ff, V = (size_t)c->vocab;
    L->tok_emb = o; o += V * d;
    L->pos_emb = o; o += (size_t)c->max_seq * d;
    L->layer0 = o;
    /* per-layer block in declaration order: ln1.g ln1.b wq bq wk bk wv bv wo bo ln2.g ln2.b w1 b1 w2 b2 */
    L->layer_stride = 2 * d + 4 * (d * d + d) + 2 * d + (d * F + F) + (F * d + d);
    o += L->layer_stride * (size_t)c->n_layers;
    L->lnf_g = o; o += d;
    L->lnf_b = o; o += d;
    L->head_w = o; o += d * V;
    L->head_b = o; o += V;
    L->total = o;
}

size_t orc_param_count(const orc_cfg* c) {
    orc_layout_t L;
    orc_layout(c, &L);
    return L.total;
}

typedef struct {
    size_t ln1g, ln1b, wq, bq, wk, bk, wv, bv, wo, bo, ln2g, ln2b, w1, b1, w2, b2;
} layer_off;

static layer_off layer_offsets(const orc_cfg* c, const orc_layout_t* L, int l) {
    const size_t d = (size_t)c->d_model, F = (size_t)c->d_ff;
    layer_off r;
    size_t o = L->layer0 + L->layer_stride * (size_t)l;
    r.ln1g = o; o += d;
    r.ln1b = o; o += d;
    r.wq = o; o += d * d;
    r.bq = o; o += d;
    r.wk = o; o += d * d;
    r.bk = o; o += d;
    r.wv = o; o += d * d;
    r.bv = o; o += d;
    r.wo = o; o += d * d;
    r.bo = o; o += d;
    r.ln2g = o; o += d;
    r.ln2b = o; o += d;
    r.w1 = o; o += d * F;
    r.b1 = o; o += F;
    r.w2 = o; o += F * d;
    r.b2 = o; o += d;
    return r;
}

/* ModelParams::init, model.cpp:142-164: gammas 1, biases/betas 0, matrices
 * 0.08*N(0,1) drawn in layout order from Rng(mix_seed(seed, "model")). */
int orc_init_params(const orc_cfg* c, uint64_t seed, double* w) {
    if (!cfg_ok(c)) return -ORC_E_CONFIG;
    orc_layout_t L;
    orc_layout(c, &L);
    memset(w, 0, L.total * sizeof(double));
    orc_rng r;
    rng_init(&r, orc_mix_seed(seed, 0x6d6f64656cull));
    const size_t d = (size_t)c->d_model, F = (size_t)c->d_ff, V = (size_t)c->vocab;
#define FILL_N(off, n)                                                   \
    do {                                                                 \
        for (size_t i_ = 0; i_ < (n); ++i_) w[(off) + i_] = 0.08 * rng_normal(&r); \
    } while (0)
#define FILL_1(off, n)                                       \
    do {                                                     \
        for (size_t i_ = 0; i_ < (n); ++i_) w[(off) + i_] = 1.0; \
    } while (0)
    FILL_N(L.tok_emb, V * d);
    FILL_N(L.pos_emb, (size_t)c->max_seq * d);
    for (int l = 0; l < c->n_layers; ++l) {
        layer_off o = layer_offsets(c, &L, l);
        FILL_1(o.ln1g, d);
        FILL_N(o.wq, d * d);
        FILL_N(o.wk, d * d);
        FILL_N(o.wv, d * d);
        FILL_N(o.wo, d * d);
        FILL_1(o.ln2g, d);
        FILL_N(o.w1, d * F);
        FILL_N(o.w2, F * d);
    }
    FILL_1(L.lnf_g, d);
    FILL_N(L.head_w, d * V);
#undef FILL_N
#undef FILL_1
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Packing: proj/src/packing.cpp:7-45 plus segments/predecessors,            */
/* proj/src/model.cpp:230-253.                                               */

int orc_pack(const int* prompt, int P, const int* resp_flat, const int* resp_lens, int G,
             int max_seq, int* tokens, int* labels, int* positions, int* span_start, int* seg,
             int* pred) {
    if (P < 1) return -ORC_E_SHAPE;                /* packing.cpp:9 */
    if (G < 1) return -ORC_E_SHAPE;                /* packing.cpp:10 */
    long total = P;
    for (int g = 0; g < G; ++g) {
        if (resp_lens[g] < 1) return -ORC_E_SHAPE; /* packing.cpp:13 */
        total += resp_lens[g];
    }
    if (total > max_seq) return -ORC_E_SHAPE;      /* packing.cpp:16-19 */
    int t = 0, src = 0;
    for (int i = 0; i < P; ++i, ++t) {
        tokens[t] = prompt[i];
        labels[t] = -1;
        positions[t] = i;
        seg[t] = 0;
        pred[t] = t - 1;
    }
    for (int g = 0; g < G; ++g) {
        span_start[g] = t;
        for (int i = 0; i < resp_lens[g]; ++i, ++t, ++src) {
            tokens[t] = resp_flat[src];
            labels[t] = resp_flat[src]; /* self-aligned, packing.cpp:37 */
            positions[t] = P + i;
            seg[t] = g + 1;
            pred[t] = (i == 0) ? P - 1 : t - 1; /* model.cpp:249-253 */
        }
    }
    return t;
}

/* Dense mask oracle: packing.cpp:47-72. */
int orc_shared_prompt_mask(int P, const int* resp_lens, int G, unsigned char* mask) {
    if (P < 1) return -ORC_E_SHAPE;
    int n = P;
    for (int g = 0; g < G; ++g) {
        if (resp_lens[g] < 1) return -ORC_E_SHAPE;
        n += resp_lens[g];
    }
    int* seg = (int*)malloc(sizeof(int) * (size_t)n);
    int idx = 0;
    for (int i = 0; i < P; ++i) seg[idx++] = 0;
    for (int g = 0; g < G; ++g)
        for (int i = 0; i < resp_lens[g]; ++i) seg[idx++] = g + 1;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            int ok = seg[i] == 0 ? (seg[j] == 0 && j <= i) : (seg[j] == 0 || (seg[j] == seg[i] && j <= i));
            mask[(size_t)i * n + j] = (unsigned char)ok;
        }
    free(seg);
    return n;
}

/* ------------------------------------------------------------------------ */
/* Dense helpers (model.cpp:255-369).                                        */

static double gelu(double x) { return 0.5 * x * erfc(-x * M_SQRT1_2); } /* model.cpp:255 */
static double gelu_grad(double x) {                                      /* model.cpp:257-260 */
    const double inv_sqrt_2pi = 0.3989422804014326779399460599344;
    return 0.5 * erfc(-x * M_SQRT1_2) + x * inv_sqrt_2pi * exp(-0.5 * x * x);
}

/* out[T x N] = x[T x M] w[M x N] + b  (model.cpp:301-314; same loop order). */
static void linear(const double* x, int T, int M, const double* w, const double* b, int N,
                   double* out) {
    memset(out, 0, sizeof(double) * (size_t)T * N);
    for (int t = 0; t < T; ++t) {
        const double* xt = x + (size_t)t * M;
        double* ot = out + (size_t)t * N;
        for (int m = 0; m < M; ++m) {
            const double xv = xt[m];
            const double* wr = w + (size_t)m * N;
            for (int n = 0; n < N; ++n) ot[n] += xv * wr[n];
        }
        for (int n = 0; n < N; ++n) ot[n] += b[n];
    }
}

/* model.cpp:317-343 */
static void layer_norm(const double* x, int T, int D, const double* g, const double* b,
                       double* xhat, double* rstd, double* y) {
    for (int t = 0; t < T; ++t) {
        const double* xt = x + (size_t)t * D;
        double mean = 0.0;
        for (int i = 0; i < D; ++i) mean += xt[i];
        mean /= D;
        double var = 0.0;
        for (int i = 0; i < D; ++i) {
            double c = xt[i] - mean;
            var += c * c;
        }
        var /= D;
        double r = 1.0 / sqrt(var + 1e-5);
        rstd[t] = r;
        for (int i = 0; i < D; ++i) {
            xhat[(size_t)t * D + i] = (xt[i] - mean) * r;
            y[(size_t)t * D + i] = g[i] * xhat[(size_t)t * D + i] + b[i];
        }
    }
}

/* model.cpp:347-369 (adds into dx). */
static void layer_norm_bwd(const double* dy, const double* xhat, const double* rstd, int T, int D,
                           const double* g, double* dg, double* db, double* dx) {
    for (int t = 0; t < T; ++t) {
        const double* dyt = dy + (size_t)t * D;
        const double* xh = xhat + (size_t)t * D;
        double m1 = 0.0, m2 = 0.0;
        for (int i = 0; i < D; ++i) {
            double dxh = dyt[i] * g[i];
            m1 += dxh;
            m2 += dxh * xh[i];
        }
        m1 /= D;
        m2 /= D;
        for (int i = 0; i < D; ++i) {
            double dxh = dyt[i] * g[i];
            dx[(size_t)t * D + i] += rstd[t] * (dxh - m1 - xh[i] * m2);
            dg[i] += dyt[i] * xh[i];
            db[i] += dyt[i];
        }
    }
}

static double lse_row(const double* row, int n) { /* model.cpp:523-530 */
    double m = row[0];
    for (int i = 1; i < n; ++i)
        if (row[i] > m) m = row[i];
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += exp(row[i] - m);
    return m + log(s);
}

static int allowed(const int* seg, int i, int j) { /* model.cpp:242-245 */
    if (seg[i] == 0) return seg[j] == 0 && j <= i;
    return seg[j] == 0 || (seg[j] == seg[i] && j <= i);
}

/* ------------------------------------------------------------------------ */
/* Forward (+ optional backward).                                            */

typedef struct {
    double *x_in, *ln1_xhat, *ln1_rstd, *a, *q, *k, *v, *probs, *ctx, *x_mid, *ln2_xhat, *ln2_rstd,
        *bn, *pre, *act;
} lcache;

static void* xcalloc(size_t n, size_t s) {
    void* p = calloc(n ? n : 1, s);
    return p;
}

/* validate_forward_inputs, model.cpp:404-426, same check order. */
static int validate(const orc_cfg* c, const int* tokens, const int* positions, int T, int P,
                    const int* resp_lens, int G, const int* labels) {
    if (T <= 0) return -ORC_E_SHAPE;
    if (T > c->max_seq) return -ORC_E_SHAPE;
    for (int t = 0; t < T; ++t)
        if (tokens[t] < 0 || tokens[t] >= c->vocab) return -ORC_E_VOCAB;
    for (int t = 0; t < T; ++t)
        if (positions[t] < 0 || positions[t] >= c->max_seq) return -ORC_E_SHAPE;
    if (labels)
        for (int t = 0; t < T; ++t)
            if (labels[t] != -1 && (labels[t] < 0 || labels[t] >= c->vocab)) return -ORC_E_VOCAB;
    if (P > 0) { /* AttentionMaskSpec::validate, model.cpp:53-61 */
        if (G < 1) return -ORC_E_SHAPE;
        long tot = P;
        for (int g = 0; g < G; ++g) {
            if (resp_lens[g] < 1) return -ORC_E_SHAPE;
            tot += resp_lens[g];
        }
        if (tot != T) return -ORC_E_SHAPE;
    }
    return 0;
}

/*
 * orc_forward: forward_logprobs (model.cpp:534-567) over one sequence; when
 * `upstream` is non-NULL also runs backward (model.cpp:587-838) and ADDS the
 * gradient into grad_acc (GradBuffer::accumulate, model.cpp:189-194).
 * P == 0 selects the causal mask; P >= 1 the shared-prompt mask.
 * Returns the number of scored labels, or -error.
 * If rows_out != NULL it receives [T x V] log-softmax rows
 * (forward_logprob_rows, model.cpp:569-585) and labels may be NULL.
 */
int orc_forward(const orc_cfg* c, const double* w, const int* tokens, const int* positions, int T,
                int P, const int* resp_lens, int G, const int* labels, double* logprobs_out,
                int* scored_pos_out, const double* upstream, double* grad_acc, double* rows_out) {
    if (!cfg_ok(c)) return -ORC_E_CONFIG;
    int rc = validate(c, tokens, positions, T, P, resp_lens, G, labels);
    if (rc) return rc;
    if (!labels && !rows_out) return -ORC_E_SHAPE;

    const int D = c->d_model, H = c->n_heads, Dh = D / H, F = c->d_ff, V = c->vocab, NL = c->n_layers;
    const double scale = 1.0 / sqrt((double)Dh);
    orc_layout_t Lo;
    orc_layout(c, &Lo);

    int* seg = (int*)xcalloc((size_t)T, sizeof(int));
    if (P > 0) {
        int idx = P;
        for (int g = 0; g < G; ++g)
            for (int i = 0; i < resp_lens[g]; ++i) seg[idx++] = g + 1;
    }
    /* scored list + predecessor (model.cpp:545-556, 249-253) */
    int* spos = (int*)xcalloc((size_t)T, sizeof(int));
    int* sprd = (int*)xcalloc((size_t)T, sizeof(int));
    int S = 0;
    if (labels) {
        for (int t = 0; t < T; ++t) {
            if (labels[t] == -1) continue;
            int p;
            if (P == 0) p = t - 1;
            else p = (seg[t] != 0 && seg[t - 1] != seg[t]) ? P - 1 : t - 1;
            if (p < 0) {
                free(seg); free(spos); free(sprd);
                return -ORC_E_SHAPE; /* model.cpp:548-549 */
            }
            spos[S] = t;
            sprd[S] = p;
            ++S;
        }
    }

    const size_t TD = (size_t)T * D, TF = (size_t)T * F;
    lcache* LC = (lcache*)xcalloc((size_t)NL, sizeof(lcache));
    double* x = (double*)xcalloc(TD, sizeof(double));
    for (int t = 0; t < T; ++t) /* model.cpp:449-455 */
        for (int i = 0; i < D; ++i)
            x[(size_t)t * D + i] = w[Lo.tok_emb + (size_t)tokens[t] * D + i] +
                                   w[Lo.pos_emb + (size_t)positions[t] * D + i];
    double* tmp = (double*)xcalloc(TD > TF ? TD : TF, sizeof(double));
    double* scores = (double*)xcalloc((size_t)T, sizeof(double));

    for (int l = 0; l < NL; ++l) { /* model.cpp:458-516 */
        lcache* C = &LC[l];
        layer_off o = layer_offsets(c, &Lo, l);
        C->x_in = (double*)xcalloc(TD, sizeof(double));
        memcpy(C->x_in, x, TD * sizeof(double));
        C->ln1_xhat = (double*)xcalloc(TD, sizeof(double));
        C->ln1_rstd = (double*)xcalloc((size_t)T, sizeof(double));
        C->a = (double*)xcalloc(TD, sizeof(double));
        layer_norm(C->x_in, T, D, w + o.ln1g, w + o.ln1b, C->ln1_xhat, C->ln1_rstd, C->a);
        C->q = (double*)xcalloc(TD, sizeof(double));
        C->k = (double*)xcalloc(TD, sizeof(double));
        C->v = (double*)xcalloc(TD, sizeof(double));
        linear(C->a, T, D, w + o.wq, w + o.bq, D, C->q);
        linear(C->a, T, D, w + o.wk, w + o.bk, D, C->k);
        linear(C->a, T, D, w + o.wv, w + o.bv, D, C->v);
        C->probs = (double*)xcalloc((size_t)H * T * T, sizeof(double));
        C->ctx = (double*)xcalloc(TD, sizeof(double));
        for (int h = 0; h < H; ++h) { /* model.cpp:471-501 */
            const int ho = h * Dh;
            for (int i = 0; i < T; ++i) {
                const double* qi = C->q + (size_t)i * D + ho;
                double mx = -INFINITY;
                for (int j = 0; j <= i; ++j) {
                    if (!allowed(seg, i, j)) continue;
                    const double* kj = C->k + (size_t)j * D + ho;
                    double s = 0.0;
                    for (int e = 0; e < Dh; ++e) s += qi[e] * kj[e];
                    s *= scale;
                    scores[j] = s;
                    if (s > mx) mx = s;
                }
                double den = 0.0;
                for (int j = 0; j <= i; ++j)
                    if (allowed(seg, i, j)) den += exp(scores[j] - mx);
                double* pr = C->probs + ((size_t)h * T + i) * T;
                double* ci = C->ctx + (size_t)i * D + ho;
                for (int j = 0; j <= i; ++j) {
                    if (!allowed(seg, i, j)) continue;
                    double pw = exp(scores[j] - mx) / den;
                    pr[j] = pw;
                    const double* vj = C->v + (size_t)j * D + ho;
                    for (int e = 0; e < Dh; ++e) ci[e] += pw * vj[e];
                }
            }
        }
        /* Note: model.cpp:477 iterates j <= i even for responses attending to
         * the prompt; prompt keys always precede response queries, so the
         * bound never cuts an allowed pair. */
        linear(C->ctx, T, D, w + o.wo, w + o.bo, D, tmp);
        C->x_mid = (double*)xcalloc(TD, sizeof(double));
        for (size_t i = 0; i < TD; ++i) C->x_mid[i] = C->x_in[i] + tmp[i];
        C->ln2_xhat = (double*)xcalloc(TD, sizeof(double));
        C->ln2_rstd = (double*)xcalloc((size_t)T, sizeof(double));
        C->bn = (double*)xcalloc(TD, sizeof(double));
        layer_norm(C->x_mid, T, D, w + o.ln2g, w + o.ln2b, C->ln2_xhat, C->ln2_rstd, C->bn);
        C->pre = (double*)xcalloc(TF, sizeof(double));
        C->act = (double*)xcalloc(TF, sizeof(double));
        linear(C->bn, T, D, w + o.w1, w + o.b1, F, C->pre);
        for (size_t i = 0; i < TF; ++i) C->act[i] = gelu(C->pre[i]);
        linear(C->act, T, F, w + o.w2, w + o.b2, D, tmp);
        for (size_t i = 0; i < TD; ++i) x[i] = C->x_mid[i] + tmp[i];
    }
    double* lnf_xhat = (double*)xcalloc(TD, sizeof(double));
    double* lnf_rstd = (double*)xcalloc((size_t)T, sizeof(double));
    double* hf = (double*)xcalloc(TD, sizeof(double));
    layer_norm(x, T, D, w + Lo.lnf_g, w + Lo.lnf_b, lnf_xhat, lnf_rstd, hf);

    /* Head only where the result is consumed: every row for rows_out, else
     * predecessor rows (each row is computed independently, model.cpp:520). */
    unsigned char* need = (unsigned char*)xcalloc((size_t)T, 1);
    if (rows_out) memset(need, 1, (size_t)T);
    for (int s = 0; s < S; ++s) need[sprd[s]] = 1;
    double* logits = (double*)xcalloc((size_t)T * V, sizeof(double));
    for (int t = 0; t < T; ++t)
        if (need[t]) linear(hf + (size_t)t * D, 1, D, w + Lo.head_w, w + Lo.head_b, V, logits + (size_t)t * V);
    if (rows_out)
        for (int t = 0; t < T; ++t) {
            double lse = lse_row(logits + (size_t)t * V, V);
            for (int v = 0; v < V; ++v) rows_out[(size_t)t * V + v] = logits[(size_t)t * V + v] - lse;
        }
    for (int s = 0; s < S; ++s) {
        const double* row = logits + (size_t)sprd[s] * V;
        if (logprobs_out) logprobs_out[s] = row[labels[spos[s]]] - lse_row(row, V);
        if (scored_pos_out) scored_pos_out[s] = spos[s];
    }

    if (upstream && grad_acc) { /* backward, model.cpp:587-838 */
        double* g = grad_acc;
        double* dlog = (double*)xcalloc((size_t)T * V, sizeof(double));
        double* probs = (double*)xcalloc((size_t)V, sizeof(double));
        for (int s = 0; s < S; ++s) { /* model.cpp:637-650 */
            double u = upstream[s];
            if (u == 0.0) continue;
            const double* row = logits + (size_t)sprd[s] * V;
            double lse = lse_row(row, V);
            for (int v = 0; v < V; ++v) probs[v] = exp(row[v] - lse);
            double* dr = dlog + (size_t)sprd[s] * V;
            for (int v = 0; v < V; ++v) dr[v] -= u * probs[v];
            dr[labels[spos[s]]] += u;
        }
        double* dhf = (double*)xcalloc(TD, sizeof(double));
        for (int t = 0; t < T; ++t) { /* model.cpp:654-668 */
            if (!need[t]) continue; /* rows without scored labels have dlogits == 0 */
            const double* hft = hf + (size_t)t * D;
            const double* dl = dlog + (size_t)t * V;
            for (int i = 0; i < D; ++i) {
                const double* wr = w + Lo.head_w + (size_t)i * V;
                double* gw = g + Lo.head_w + (size_t)i * V;
                double acc = 0.0;
                for (int v = 0; v < V; ++v) {
                    acc += dl[v] * wr[v];
                    gw[v] += hft[i] * dl[v];
                }
                dhf[(size_t)t * D + i] = acc;
            }
            for (int v = 0; v < V; ++v) g[Lo.head_b + v] += dl[v];
        }
        double* dx = (double*)xcalloc(TD, sizeof(double));
        layer_norm_bwd(dhf, lnf_xhat, lnf_rstd, T, D, w + Lo.lnf_g, g + Lo.lnf_g, g + Lo.lnf_b, dx);
        double* dmid = (double*)xcalloc(TD, sizeof(double));
        double* dctx = (double*)xcalloc(TD, sizeof(double));
        double* da = (double*)xcalloc(TD, sizeof(double));
        double* dq = (double*)xcalloc(TD, sizeof(double));
        double* dk = (double*)xcalloc(TD, sizeof(double));
        double* dv = (double*)xcalloc(TD, sizeof(double));
        double* dact = (double*)xcalloc(TF, sizeof(double));
        double* dbn = (double*)xcalloc(TD, sizeof(double));
        double* dwrow = (double*)xcalloc((size_t)T, sizeof(double));
        for (int l = NL - 1; l >= 0; --l) {
            lcache* C = &LC[l];
            layer_off o = layer_offsets(c, &Lo, l);
            /* FFN, model.cpp:688-727 */
            for (int t = 0; t < T; ++t) {
                const double* dxt = dx + (size_t)t * D;
                const double* ac = C->act + (size_t)t * F;
                double* dat = dact + (size_t)t * F;
                for (int f = 0; f < F; ++f) {
                    const double* w2r = w + o.w2 + (size_t)f * D;
                    double* gw2 = g + o.w2 + (size_t)f * D;
                    double acc = 0.0;
                    for (int i = 0; i < D; ++i) {
                        acc += dxt[i] * w2r[i];
                        gw2[i] += ac[f] * dxt[i];
                    }
                    dat[f] = acc;
                }
                for (int i = 0; i < D; ++i) g[o.b2 + i] += dxt[i];
            }
            for (int t = 0; t < T; ++t) {
                const double* pre = C->pre + (size_t)t * F;
                const double* bn = C->bn + (size_t)t * D;
                double* dat = dact + (size_t)t * F;
                for (int f = 0; f < F; ++f) {
                    double dp = dat[f] * gelu_grad(pre[f]);
                    dat[f] = dp;
                    g[o.b1 + f] += dp;
                }
                for (int i = 0; i < D; ++i) {
                    const double* w1r = w + o.w1 + (size_t)i * F;
                    double* gw1 = g + o.w1 + (size_t)i * F;
                    double acc = 0.0;
                    for (int f = 0; f < F; ++f) {
                        acc += dat[f] * w1r[f];
                        gw1[f] += bn[i] * dat[f];
                    }
                    dbn[(size_t)t * D + i] = acc;
                }
            }
            memcpy(dmid, dx, TD * sizeof(double)); /* model.cpp:729-730 */
            layer_norm_bwd(dbn, C->ln2_xhat, C->ln2_rstd, T, D, w + o.ln2g, g + o.ln2g, g + o.ln2b, dmid);
            /* O projection, model.cpp:733-749 */
            for (int t = 0; t < T; ++t) {
                const double* dm = dmid + (size_t)t * D;
                const double* ct = C->ctx + (size_t)t * D;
                double* dc = dctx + (size_t)t * D;
                for (int i = 0; i < D; ++i) {
                    const double* wor = w + o.wo + (size_t)i * D;
                    double* gwo = g + o.wo + (size_t)i * D;
                    double acc = 0.0;
                    for (int e = 0; e < D; ++e) {
                        acc += dm[e] * wor[e];
                        gwo[e] += ct[i] * dm[e];
                    }
                    dc[i] = acc;
                }
                for (int e = 0; e < D; ++e) g[o.bo + e] += dm[e];
            }
            /* attention, model.cpp:752-786 */
            memset(dq, 0, TD * sizeof(double));
            memset(dk, 0, TD * sizeof(double));
            memset(dv, 0, TD * sizeof(double));
            for (int h = 0; h < H; ++h) {
                const int ho = h * Dh;
                for (int i = 0; i < T; ++i) {
                    const double* pr = C->probs + ((size_t)h * T + i) * T;
                    const double* dci = dctx + (size_t)i * D + ho;
                    double dot = 0.0;
                    for (int j = 0; j <= i; ++j) {
                        if (!allowed(seg, i, j)) continue;
                        const double* vj = C->v + (size_t)j * D + ho;
                        double dw = 0.0;
                        for (int e = 0; e < Dh; ++e) dw += dci[e] * vj[e];
                        dwrow[j] = dw;
                        dot += pr[j] * dw;
                        double* dvj = dv + (size_t)j * D + ho;
                        for (int e = 0; e < Dh; ++e) dvj[e] += pr[j] * dci[e];
                    }
                    const double* qi = C->q + (size_t)i * D + ho;
                    double* dqi = dq + (size_t)i * D + ho;
                    for (int j = 0; j <= i; ++j) {
                        if (!allowed(seg, i, j)) continue;
                        double ds = pr[j] * (dwrow[j] - dot) * scale;
                        const double* kj = C->k + (size_t)j * D + ho;
                        double* dkj = dk + (size_t)j * D + ho;
                        for (int e = 0; e < Dh; ++e) {
                            dqi[e] += ds * kj[e];
                            dkj[e] += ds * qi[e];
                        }
                    }
                }
            }
            /* QKV, model.cpp:789-817 */
            for (int t = 0; t < T; ++t) {
                const double* at = C->a + (size_t)t * D;
                const double* dqt = dq + (size_t)t * D;
                const double* dkt = dk + (size_t)t * D;
                const double* dvt = dv + (size_t)t * D;
                double* dat = da + (size_t)t * D;
                for (int i = 0; i < D; ++i) {
                    const double* wqr = w + o.wq + (size_t)i * D;
                    const double* wkr = w + o.wk + (size_t)i * D;
                    const double* wvr = w + o.wv + (size_t)i * D;
                    double* gq = g + o.wq + (size_t)i * D;
                    double* gk = g + o.wk + (size_t)i * D;
                    double* gv = g + o.wv + (size_t)i * D;
                    double acc = 0.0;
                    for (int e = 0; e < D; ++e) {
                        acc += dqt[e] * wqr[e] + dkt[e] * wkr[e] + dvt[e] * wvr[e];
                        gq[e] += at[i] * dqt[e];
                        gk[e] += at[i] * dkt[e];
                        gv[e] += at[i] * dvt[e];
                    }
                    dat[i] = acc;
                }
                for (int e = 0; e < D; ++e) {
                    g[o.bq + e] += dqt[e];
                    g[o.bk + e] += dkt[e];
                    g[o.bv + e] += dvt[e];
                }
            }
            memcpy(dx, dmid, TD * sizeof(double)); /* model.cpp:820-822 */
            layer_norm_bwd(da, C->ln1_xhat, C->ln1_rstd, T, D, w + o.ln1g, g + o.ln1g, g + o.ln1b, dx);
        }
        for (int t = 0; t < T; ++t) /* embeddings, model.cpp:826-834 */
            for (int i = 0; i < D; ++i) {
                g[Lo.tok_emb + (size_t)tokens[t] * D + i] += dx[(size_t)t * D + i];
                g[Lo.pos_emb + (size_t)positions[t] * D + i] += dx[(size_t)t * D + i];
            }
        free(dlog); free(probs); free(dhf); free(dx); free(dmid); free(dctx); free(da);
        free(dq); free(dk); free(dv); free(dact); free(dbn); free(dwrow);
    }

    for (int l = 0; l < NL; ++l) {
        lcache* C = &LC[l];
        free(C->x_in); free(C->ln1_xhat); free(C->ln1_rstd); free(C->a); free(C->q); free(C->k);
        free(C->v); free(C->probs); free(C->ctx); free(C->x_mid); free(C->ln2_xhat);
        free(C->ln2_rstd); free(C->bn); free(C->pre); free(C->act);
    }
    free(LC); free(x); free(tmp); free(scores); free(lnf_xhat); free(lnf_rstd); free(hf);
    free(need); free(logits); free(seg); free(spos); free(sprd);
    return S;
}

/* ------------------------------------------------------------------------ */
/* GRPO: proj/src/grpo.cpp:24-151                                            */

int orc_group_advantages(const double* r, int G, int mean_only, double* a) {
    if (G < 2) return -ORC_E_CONFIG; /* grpo.cpp:25, 41 */
    double mean = 0.0;
    for (int i = 0; i < G; ++i) mean += r[i];
    mean /= (double)G;
    if (mean_only) { /* grpo.cpp:40-48 */
        for (int i = 0; i < G; ++i) a[i] = r[i] - mean;
        return 0;
    }
    double var = 0.0;
    for (int i = 0; i < G; ++i) var += (r[i] - mean) * (r[i] - mean);
    var /= (double)G;
    double sd = sqrt(var);
    for (int i = 0; i < G; ++i) a[i] = sd < 1e-8 ? 0.0 : (r[i] - mean) / sd;
    return 0;
}

/* eval_clip, grpo.cpp:64-80 */
static void clip_eval(double lp, double old, double A, double eps, double* val, double* grad,
                      int* clipped) {
    double r = exp(lp - old);
    double lo = 1.0 - eps, hi = 1.0 + eps;
    double cl = r < lo ? lo : (r > hi ? hi : r);
    double un = r * A, cv = cl * A;
    *clipped = (r < lo || r > hi);
    if (un <= cv) {
        *val = un;
        *grad = r * A;
    } else {
        *val = cv;
        *grad = (r > lo && r < hi) ? r * A : 0.0;
    }
}

/* eval_kl, grpo.cpp:89-93 */
static void kl_eval(double lp, double ref, double* val, double* grad) {
    double d = ref - lp;
    double e = expm1(d);
    *val = e - d;
    *grad = -e;
}

double orc_clipped_term(double lp, double old, double A, double eps) {
    double v, g;
    int c;
    clip_eval(lp, old, A, eps, &v, &g, &c);
    return v;
}

double orc_kl_term(double lp, double ref) {
    double v, g;
    kl_eval(lp, ref, &v, &g);
    return v;
}

/* per_sample_terms, grpo.cpp:111-151.  out4 = {clip_term, kl, clipped_units, total_units}. */
int orc_sample_terms(const double* lp, const double* old, const double* ref, int n, double A,
                     double eps, double beta, int granularity, double* upstream, double* out4) {
    if (n <= 0) return -ORC_E_SHAPE;
    if (!isfinite(A)) return -ORC_E_NUMERIC;
    double ct = 0.0, kl = 0.0;
    int clipped = 0, units;
    if (granularity == 0) {
        const double inv = 1.0 / (double)n;
        for (int t = 0; t < n; ++t) {
            double cv, cg, kv, kg;
            int c;
            clip_eval(lp[t], old[t], A, eps, &cv, &cg, &c);
            kl_eval(lp[t], ref[t], &kv, &kg);
            ct += inv * cv;
            kl += inv * kv;
            upstream[t] = inv * (cg - beta * kg);
            clipped += c;
        }
        units = n;
    } else {
        double sn = 0.0, so = 0.0, sr = 0.0;
        for (int t = 0; t < n; ++t) {
            sn += lp[t];
            so += old[t];
            sr += ref[t];
        }
        double cv, cg, kv, kg;
        int c;
        clip_eval(sn, so, A, eps, &cv, &cg, &c);
        kl_eval(sn, sr, &kv, &kg);
        ct = cv;
        kl = kv;
        for (int t = 0; t < n; ++t) upstream[t] = cg - beta * kg;
        clipped = c;
        units = 1;
    }
    out4[0] = ct;
    out4[1] = kl;
    out4[2] = clipped;
    out4[3] = units;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* The whole hot path: Pipeline::train_microbatch shared-prompt branch,      */
/* pipeline.cpp:97-141.  w_old == NULL selects rollout_weights mode, where   */
/* old_lp_in supplies the old log-probs (pipeline.cpp:113-119).              */
/* stats5 += {objective_sum, clip_sum, kl_sum, clipped_units, total_units}.  */
/* lp3 (optional) receives [policy | old | ref] log-probs, S each.           */

int orc_train_microbatch(const orc_cfg* c, const double* w_pol, const double* w_old,
                         const double* w_ref, const int* prompt, int P, const int* resp_flat,
                         const int* resp_lens, int G, const double* advantages,
                         const double* old_lp_in, double eps, double beta, int granularity,
                         double* grad_acc, double* stats5, double* lp3) {
    long Tl = P;
    for (int g = 0; g < G; ++g) Tl += resp_lens[g] > 0 ? resp_lens[g] : 0;
    int T = (int)Tl;
    int *tok = (int*)xcalloc((size_t)T, sizeof(int)), *lab = (int*)xcalloc((size_t)T, sizeof(int)),
        *pos = (int*)xcalloc((size_t)T, sizeof(int)), *sp = (int*)xcalloc((size_t)(G > 0 ? G : 1), sizeof(int)),
        *seg = (int*)xcalloc((size_t)T, sizeof(int)), *prd = (int*)xcalloc((size_t)T, sizeof(int));
    int rc = orc_pack(prompt, P, resp_flat, resp_lens, G, c->max_seq, tok, lab, pos, sp, seg, prd);
    if (rc < 0) goto out;
    int S = T - P;
    double* lp = (double*)xcalloc((size_t)S * 3, sizeof(double));
    double *lpp = lp, *lpo = lp + S, *lpr = lp + 2 * S;
    rc = orc_forward(c, w_pol, tok, pos, T, P, resp_lens, G, lab, lpp, NULL, NULL, NULL, NULL);
    if (rc >= 0 && w_old) rc = orc_forward(c, w_old, tok, pos, T, P, resp_lens, G, lab, lpo, NULL, NULL, NULL, NULL);
    if (rc >= 0 && !w_old) memcpy(lpo, old_lp_in, sizeof(double) * (size_t)S);
    if (rc >= 0) rc = orc_forward(c, w_ref, tok, pos, T, P, resp_lens, G, lab, lpr, NULL, NULL, NULL, NULL);
    if (rc < 0) { free(lp); goto out; }
    double* up = (double*)xcalloc((size_t)S, sizeof(double));
    int off = 0;
    for (int g = 0; g < G && rc >= 0; ++g) {
        double t4[4];
        int n = resp_lens[g];
        int r2 = orc_sample_terms(lpp + off, lpo + off, lpr + off, n, advantages[g], eps, beta,
                                  granularity, up + off, t4);
        if (r2 < 0) { rc = r2; break; }
        stats5[0] += t4[0] - beta * t4[1];
        stats5[1] += t4[0];
        stats5[2] += t4[1];
        stats5[3] += t4[2];
        stats5[4] += t4[3];
        for (int t = 0; t < n; ++t) up[off + t] = -up[off + t]; /* pipeline.cpp:138 */
        off += n;
    }
    if (rc >= 0)
        rc = orc_forward(c, w_pol, tok, pos, T, P, resp_lens, G, lab, NULL, NULL, up, grad_acc, NULL);
    if (lp3 && rc >= 0) memcpy(lp3, lp, sizeof(double) * 3 * (size_t)S);
    free(up);
    free(lp);
out:
    free(tok); free(lab); free(pos); free(sp); free(seg); free(prd);
    return rc < 0 ? rc : T;
}
