/*
 * asp_oracle.c -- the CPU ORACLE for the AsyncSpade decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2510_07486_b200/) never calls it and shares no
 * code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C99: fp64 arithmetic, fixed loop order,
 * one thread, no blocking, no fusion.  Every function follows the passage
 * of arXiv 2510.07486 (reference/PAPER.md, "P:<line>") it cites, with the
 * readings R1..R17 of SURVEY.md §8(c) (restated in DESIGN.md §3) wherever
 * the paper is silent or garbled.
 *
 * Pins (what checks this file against something other than itself) live in
 * tests/test_oracle_pins.py.  Parity is pinned for every entry point; the
 * one part no pin can reach -- whether readings R4-R6 match what the
 * authors ran -- is "parity unpinned", because the paper
 * prints no worked example.
 *
 * Condition bits returned by every call (same numeric values as the
 * product ABI by documented convention, not by shared header):
 *   1 = non-finite input/value seen, 2 = regression matrix not positive
 *   definite (passthrough used), 4 = a row shorter than top_k (padded).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_FLAG_NONFINITE 1u
#define OR_FLAG_NOT_PD 2u
#define OR_FLAG_SHORT_ROW 4u

/* predict flags (documented convention) */
#define OR_ASSEMBLY_MASK 0xFu
#define OR_ASSEMBLY_MASKED_SHARED 0u
#define OR_ASSEMBLY_SINGLE 1u
#define OR_ASSEMBLY_PER_WINDOW 2u
#define OR_SIGN_NEGATED (1u << 4)
#define OR_EPS_ABSOLUTE (1u << 5)
#define OR_NORM_NONE (1u << 6)
#define OR_DOUBLE_SOFTMAX (1u << 7)

/* bf16 bit pattern -> double: a bf16 is the top half of an IEEE fp32. */
static double bf16_to_double(uint16_t h) {
    uint32_t bits = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &bits, 4);
    return (double)f;
}

/* ------------------------------------------------------------------------
 * Linear algebra for the ridge regression (Alg. 1 Step 3).
 * ---------------------------------------------------------------------- */

/* In-place Cholesky G = L L^T of an n x n row-major SPD matrix (lower
 * triangle overwritten by L).  Returns 0, or -1 on a pivot <= 0 / non-finite
 * (non-positive pivot -> not positive definite). */
static int cholesky(double *A, int n) {
    for (int j = 0; j < n; j++) {
        double s = A[j * n + j];
        for (int k = 0; k < j; k++) s -= A[j * n + k] * A[j * n + k];
        if (!(s > 0.0) || !isfinite(s)) return -1;
        double d = sqrt(s);
        A[j * n + j] = d;
        for (int i = j + 1; i < n; i++) {
            double t = A[i * n + j];
            for (int k = 0; k < j; k++) t -= A[i * n + k] * A[j * n + k];
            A[i * n + j] = t / d;
        }
    }
    return 0;
}

/* Solve (L L^T) x = b given the Cholesky factor L (lower triangle of A). */
static void cholesky_solve(const double *A, int n, const double *b, double *x) {
    double y[64];
    for (int i = 0; i < n; i++) {
        double t = b[i];
        for (int k = 0; k < i; k++) t -= A[i * n + k] * y[k];
        y[i] = t / A[i * n + i];
    }
    for (int i = n - 1; i >= 0; i--) {
        double t = y[i];
        for (int k = i + 1; k < n; k++) t -= A[k * n + i] * x[k];
        x[i] = t / A[i * n + i];
    }
}

/* softmax(v[0..n-1]) with max-subtraction. */
static void softmax(const double *v, int n, double *out) {
    double m = v[0];
    for (int i = 1; i < n; i++)
        if (v[i] > m) m = v[i];
    double s = 0.0;
    for (int i = 0; i < n; i++) {
        out[i] = exp(v[i] - m);
        s += out[i];
    }
    for (int i = 0; i < n; i++) out[i] /= s;
}

/* Ridge weights omega = (Hist Hist^T + eps I)^{-1} Hist y over the nh rows
 * `hist` (each D long), target y.  Eq. 2 linearised as in
 * Alg. 1 Step 3.  eps is relative (eps * mean diag G0, reading
 * R7) unless `absolute`; an all-zero history gets the floor 1e-30.
 * Returns 0 or -1 (not PD). */
static int ridge_weights(const double *const *hist, int nh, const double *y, int D,
                         double eps, int absolute, double *omega) {
    double G[64 * 64], beta[64];
    for (int i = 0; i < nh; i++) {
        for (int j = 0; j < nh; j++) {
            double s = 0.0;
            for (int d = 0; d < D; d++) s += hist[i][d] * hist[j][d];
            G[i * nh + j] = s;
        }
        double s = 0.0;
        for (int d = 0; d < D; d++) s += hist[i][d] * y[d];
        beta[i] = s;
    }
    double e = eps;
    if (!absolute) {
        double tr = 0.0;
        for (int i = 0; i < nh; i++) tr += G[i * nh + i];
        e = eps * (tr / nh);
    }
    if (e == 0.0) e = 1e-30;
    for (int i = 0; i < nh; i++) G[i * nh + i] += e;
    if (cholesky(G, nh) != 0) return -1;
    cholesky_solve(G, nh, beta, omega);
    for (int i = 0; i < nh; i++)
        if (!isfinite(omega[i])) return -1;
    return 0;
}

/* ------------------------------------------------------------------------
 * a1 predict: next query q_hat_{t+1} from the window (Eq. 4-5;
 * Alg. 1 Steps 1-6).  Window layout [n_rows][W][D] fp32; logical
 * slot j (0 = oldest, W-1 = newest = Q_t) lives at physical slot
 * (ring_start + j) % W.
 * ---------------------------------------------------------------------- */
uint32_t asp_oracle_predict(int32_t n_rows, int32_t W, int32_t D, int32_t ring_start,
                            double eps, uint32_t flags, const float *q_window,
                            float *q_hat) {
    uint32_t cond = 0;
    const uint32_t mode = flags & OR_ASSEMBLY_MASK;
    const double sgn = (flags & OR_SIGN_NEGATED) ? -1.0 : 1.0;    /* reading R2 */
    const int absolute = (flags & OR_EPS_ABSOLUTE) ? 1 : 0;
    double *Q = (double *)malloc(sizeof(double) * (size_t)W * D);
    double *acc = (double *)malloc(sizeof(double) * (size_t)D);
    const double *hist[64];
    double omega[64], r[64];

    for (int32_t row = 0; row < n_rows; row++) {
        const float *win = q_window + (size_t)row * W * D;
        int finite = 1;
        /* Step 1: read the window in logical order. */
        for (int j = 0; j < W; j++) {
            const float *src = win + (size_t)((ring_start + j) % W) * D;
            for (int d = 0; d < D; d++) {
                Q[(size_t)j * D + d] = (double)src[d];
                if (!isfinite(src[d])) finite = 0;
            }
        }
        const double *newest = Q + (size_t)(W - 1) * D;
        float *out = q_hat + (size_t)row * D;
        if (!finite) cond |= OR_FLAG_NONFINITE;
        if (W == 1 || !finite) {                  /* passthrough */
            for (int d = 0; d < D; d++) out[d] = (float)newest[d];
            continue;
        }
        const int n = W - 1;                      /* reading R1 */
        for (int d = 0; d < D; d++) acc[d] = 0.0;
        int ok = 1;

        if (mode == OR_ASSEMBLY_PER_WINDOW) {
            /* Eq. 5 literal: for k = 1..n regress Q_t on the k
             * most recent older queries Q[W-1-k..W-2], apply the softmax
             * weights to the one-step-shifted suffix Q[W-k..W-1], average
             * the m = n candidates (reading R8). */
            for (int k = 1; k <= n && ok; k++) {
                for (int i = 0; i < k; i++) hist[i] = Q + (size_t)(W - 1 - k + i) * D;
                if (ridge_weights(hist, k, newest, D, eps, absolute, omega) != 0) { ok = 0; break; }
                for (int i = 0; i < k; i++) omega[i] *= sgn;
                softmax(omega, k, r);
                for (int i = 0; i < k; i++)
                    for (int d = 0; d < D; d++) acc[d] += r[i] * Q[(size_t)(W - k + i) * D + d];
            }
            if (ok)
                for (int d = 0; d < D; d++) out[d] = (float)(acc[d] / n);
        } else {
            /* Step 3: one ridge solve over the n older queries
             * Q[0..n-1] (Q_hist) regressing the newest Q[W-1] (q_prev). */
            for (int i = 0; i < n; i++) hist[i] = Q + (size_t)i * D;
            if (ridge_weights(hist, n, newest, D, eps, absolute, omega) != 0) ok = 0;
            if (ok && mode == OR_ASSEMBLY_SINGLE) {
                if (flags & OR_NORM_NONE) {
                    /* raw linear predictor (reading R17, test-only) */
                    for (int i = 0; i < n; i++) r[i] = omega[i];
                } else {
                    for (int i = 0; i < n; i++) r[i] = sgn * omega[i];
                    softmax(r, n, r);
                }
                /* Eq. 4: weight of Q_{t-i} applied to Q_{t+1-i},
                 * i.e. omega[i] (row i of Q_hist) -> Q[i+1]. */
                for (int i = 0; i < n; i++)
                    for (int d = 0; d < D; d++) acc[d] += r[i] * Q[(size_t)(i + 1) * D + d];
                for (int d = 0; d < D; d++) out[d] = (float)acc[d];
            } else if (ok) {
                /* Masked-shared assembly, Steps 4-6, readings
                 * R3-R6: row j = 1..W keeps the first n_j = min(j, n)
                 * weights, softmaxed over just those (single softmax; the
                 * literal double softmax behind OR_DOUBLE_SOFTMAX), applied
                 * to the newest n_j queries Q[W-n_j..W-1]; then the mean of
                 * the m = W candidates. */
                double p[64];
                for (int i = 0; i < n; i++) p[i] = sgn * omega[i];
                if (flags & OR_DOUBLE_SOFTMAX) softmax(p, n, p);
                for (int j = 1; j <= W; j++) {
                    const int nj = j < n ? j : n;
                    softmax(p, nj, r);
                    for (int i = 0; i < nj; i++)
                        for (int d = 0; d < D; d++)
                            acc[d] += r[i] * Q[(size_t)(W - nj + i) * D + d];
                }
                for (int d = 0; d < D; d++) out[d] = (float)(acc[d] / W);
            }
        }
        if (!ok) {                                /* not PD -> passthrough */
            cond |= OR_FLAG_NOT_PD;
            for (int d = 0; d < D; d++) out[d] = (float)newest[d];
        }
    }
    free(Q);
    free(acc);
    return cond;
}

/* ------------------------------------------------------------------------
 * a2 score: token criticality (Alg. 1 Step 7; GQA layout P:260).
 * s[b,h,n] = max over the G = Hq/Hkv query heads of group h of
 * sum_d q_hat[b, h*G+g, d] * K[b,h,n,d], for n < seq_lens[b] (reading R10;
 * sum with agg = 1).  No 1/sqrt(D) (reading R11).  Exact in fp64: bf16 x
 * fp32 products are exact in double.  Positions n >= seq_lens[b] get -inf.
 * ---------------------------------------------------------------------- */
uint32_t asp_oracle_score(int32_t B, int32_t Hq, int32_t Hkv, int32_t D, int32_t L_cap,
                          const int32_t *seq_lens, const float *q_hat,
                          const uint16_t *k_cache, int32_t agg, double *scores) {
    const int G = Hq / Hkv;
    uint32_t cond = 0;
    for (int b = 0; b < B; b++)
        for (int h = 0; h < Hkv; h++) {
            double *srow = scores + ((size_t)b * Hkv + h) * L_cap;
            for (int n = 0; n < L_cap; n++) {
                if (n >= seq_lens[b]) { srow[n] = -INFINITY; continue; }
                const uint16_t *kr = k_cache + (((size_t)b * Hkv + h) * L_cap + n) * D;
                double best = 0.0;
                for (int g = 0; g < G; g++) {
                    const float *q = q_hat + ((size_t)b * Hq + (size_t)h * G + g) * D;
                    double s = 0.0;
                    for (int d = 0; d < D; d++) s += (double)q[d] * bf16_to_double(kr[d]);
                    if (g == 0) best = s;
                    else if (agg == 1) best += s;
                    else if (s > best) best = s;
                }
                if (!isfinite(best)) cond |= OR_FLAG_NONFINITE;
                srow[n] = best;
            }
        }
    return cond;
}

/* ------------------------------------------------------------------------
 * Quest comparator: page upper bounds, SPEC
 * page_level_select, the paper's Quest baseline at page size 16
 * (P:356).  Tokens [0, len) of row (b, h) are cut into
 * consecutive pages of P (the last one may be short); for page j,
 *   maxK_d = max over its tokens of K[d],  minK_d = min over its tokens,
 *   U_g = sum_d max(q_gd * maxK_d, q_gd * minK_d),
 * reduced over the group like the token score (max, or sum with agg = 1).
 * Output bounds[b][h][j] for j < ceil(len / P), -inf beyond.
 * ---------------------------------------------------------------------- */
uint32_t asp_oracle_page_bounds(int32_t B, int32_t Hq, int32_t Hkv, int32_t D, int32_t L_cap,
                                int32_t P, const int32_t *seq_lens, const float *q,
                                const uint16_t *k_cache, int32_t agg, double *bounds) {
    const int G = Hq / Hkv;
    const int NP = (L_cap + P - 1) / P;
    uint32_t cond = 0;
    double *mx = (double *)malloc(sizeof(double) * D), *mn = (double *)malloc(sizeof(double) * D);
    for (int b = 0; b < B; b++)
        for (int h = 0; h < Hkv; h++) {
            double *brow = bounds + ((size_t)b * Hkv + h) * NP;
            for (int j = 0; j < NP; j++) {
                const int t0 = j * P;
                int t1 = t0 + P;
                if (t1 > seq_lens[b]) t1 = seq_lens[b];
                if (t0 >= t1) { brow[j] = -INFINITY; continue; }
                for (int d = 0; d < D; d++) { mx[d] = -INFINITY; mn[d] = INFINITY; }
                for (int t = t0; t < t1; t++) {
                    const uint16_t *kr = k_cache + (((size_t)b * Hkv + h) * L_cap + t) * D;
                    for (int d = 0; d < D; d++) {
                        const double v = bf16_to_double(kr[d]);
                        if (v > mx[d]) mx[d] = v;
                        if (v < mn[d]) mn[d] = v;
                    }
                }
                double best = 0.0;
                for (int g = 0; g < G; g++) {
                    const float *qg = q + ((size_t)b * Hq + (size_t)h * G + g) * D;
                    double u = 0.0;
                    for (int d = 0; d < D; d++) {
                        const double a = (double)qg[d] * mx[d], c = (double)qg[d] * mn[d];
                        u += a > c ? a : c;
                    }
                    if (g == 0) best = u;
                    else if (agg == 1) best += u;
                    else if (u > best) best = u;
                }
                if (!isfinite(best)) cond |= OR_FLAG_NONFINITE;
                brow[j] = best;
            }
        }
    free(mx);
    free(mn);
    return cond;
}

/* ------------------------------------------------------------------------
 * a3 select: per row, the k tokens with the largest score (P:191, P:267
 * item (2)).  Definition: sort the row by (score descending, index
 * ascending) -- lower index wins ties (reading R9) -- take the first k,
 * emit them in ascending index order.  NaN sorts below every
 * number (R14); -0.0 == +0.0 by C comparison.  A row shorter than k emits
 * all its tokens then -1 padding (R13).
 * ---------------------------------------------------------------------- */
static const double *g_sort_row;   /* qsort context (single-threaded oracle) */

static int by_score_desc_index_asc(const void *pa, const void *pb) {
    const int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    const double sa = g_sort_row[a], sb = g_sort_row[b];
    const int na = isnan(sa), nb = isnan(sb);
    if (na != nb) return na ? 1 : -1;
    if (!na) {
        if (sa > sb) return -1;
        if (sa < sb) return 1;
    }
    return (a < b) ? -1 : (a > b) ? 1 : 0;
}

static int by_index_asc(const void *pa, const void *pb) {
    const int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    return (a < b) ? -1 : (a > b) ? 1 : 0;
}

uint32_t asp_oracle_select(int32_t n_rows, int32_t L_cap, const int32_t *row_lens,
                           const double *scores, int32_t k, int32_t *idx) {
    uint32_t cond = 0;
    int32_t *order = (int32_t *)malloc(sizeof(int32_t) * (size_t)(L_cap > 0 ? L_cap : 1));
    for (int32_t row = 0; row < n_rows; row++) {
        const int32_t len = row_lens[row];
        const double *s = scores + (size_t)row * L_cap;
        int32_t *out = idx + (size_t)row * k;
        for (int32_t n = 0; n < len; n++) {
            order[n] = n;
            if (isnan(s[n])) cond |= OR_FLAG_NONFINITE;
        }
        g_sort_row = s;
        qsort(order, (size_t)len, sizeof(int32_t), by_score_desc_index_asc);
        const int32_t take = len < k ? len : k;
        if (len < k) cond |= OR_FLAG_SHORT_ROW;
        qsort(order, (size_t)take, sizeof(int32_t), by_index_asc);
        for (int32_t i = 0; i < k; i++) out[i] = i < take ? order[i] : -1;
    }
    free(order);
    return cond;
}

/* ------------------------------------------------------------------------
 * a4 sparse decode attention over the selected tokens ("participate
 * in the attention computation").  For query head
 * hq of KV head h = hq / G: the attended set is
 *   { idx[b,h,j] : 0 <= idx < len - n_fresh }  U  [len - n_fresh, len)
 * (reading R12: the n_fresh newest tokens are always attended, each token
 * at most once).  logits l_j = sm_scale * q . K_j, p = softmax(l),
 * out = sum_j p_j V_j; all in fp64, rounded once to fp32.  Empty set -> 0.
 * ---------------------------------------------------------------------- */
static void attend(int D, double sm_scale, const uint16_t *q, const uint16_t *kbase,
                   const uint16_t *vbase, const int32_t *tok, int ntok, float *out) {
    double *l = (double *)malloc(sizeof(double) * (size_t)(ntok > 0 ? ntok : 1));
    double m = -INFINITY;
    for (int j = 0; j < ntok; j++) {
        const uint16_t *kr = kbase + (size_t)tok[j] * D;
        double s = 0.0;
        for (int d = 0; d < D; d++) s += bf16_to_double(q[d]) * bf16_to_double(kr[d]);
        l[j] = sm_scale * s;
        if (l[j] > m) m = l[j];
    }
    double den = 0.0;
    for (int j = 0; j < ntok; j++) {
        l[j] = exp(l[j] - m);
        den += l[j];
    }
    for (int d = 0; d < D; d++) {
        double o = 0.0;
        for (int j = 0; j < ntok; j++) o += l[j] * bf16_to_double(vbase[(size_t)tok[j] * D + d]);
        out[d] = ntok > 0 ? (float)(o / den) : 0.0f;
    }
    free(l);
}

uint32_t asp_oracle_sparse_decode(int32_t B, int32_t Hq, int32_t Hkv, int32_t D,
                                  int32_t L_cap, int32_t k, int32_t n_fresh, double sm_scale,
                                  const int32_t *seq_lens, const uint16_t *q,
                                  const uint16_t *k_cache, const uint16_t *v_cache,
                                  const int32_t *idx, float *out) {
    const int G = Hq / Hkv;
    int32_t *tok = (int32_t *)malloc(sizeof(int32_t) * (size_t)(k + n_fresh + 1));
    for (int b = 0; b < B; b++)
        for (int h = 0; h < Hkv; h++) {
            const int32_t len = seq_lens[b];
            const int32_t fresh_lo = len - n_fresh > 0 ? len - n_fresh : 0;
            int ntok = 0;
            for (int j = 0; j < k; j++) {
                const int32_t t = idx[((size_t)b * Hkv + h) * k + j];
                if (t >= 0 && t < fresh_lo) tok[ntok++] = t;
            }
            for (int32_t t = fresh_lo; t < len; t++) tok[ntok++] = t;
            const size_t kv_off = ((size_t)b * Hkv + h) * L_cap * D;
            for (int g = 0; g < G; g++) {
                const size_t qo = ((size_t)b * Hq + (size_t)h * G + g) * D;
                attend(D, sm_scale, q + qo, k_cache + kv_off, v_cache + kv_off, tok, ntok,
                       out + qo);
            }
        }
    free(tok);
    return 0;
}

/* Dense attention over all len tokens: the special case
 * the sparse decode must reduce to when k = len, n_fresh = 0. */
uint32_t asp_oracle_dense_attention(int32_t B, int32_t Hq, int32_t Hkv, int32_t D,
                                    int32_t L_cap, double sm_scale, const int32_t *seq_lens,
                                    const uint16_t *q, const uint16_t *k_cache,
                                    const uint16_t *v_cache, float *out) {
    const int G = Hq / Hkv;
    int32_t *tok = (int32_t *)malloc(sizeof(int32_t) * (size_t)(L_cap + 1));
    for (int b = 0; b < B; b++)
        for (int h = 0; h < Hkv; h++) {
            for (int32_t t = 0; t < seq_lens[b]; t++) tok[t] = t;
            const size_t kv_off = ((size_t)b * Hkv + h) * L_cap * D;
            for (int g = 0; g < G; g++) {
                const size_t qo = ((size_t)b * Hq + (size_t)h * G + g) * D;
                attend(D, sm_scale, q + qo, k_cache + kv_off, v_cache + kv_off, tok,
                       seq_lens[b], out + qo);
            }
        }
    free(tok);
    return 0;
}
