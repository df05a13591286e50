/*
 * ls2_oracle.c -- TEST INFRASTRUCTURE ONLY (not the product path).
 *
 * Plain single-threaded fp64 CPU oracle of LearnedSort 2.0 (arXiv 2107.03290).
 * It follows the paper's Alg. 1 and Alg. 2 step by step,
 * in the paper's order and notation, with the model construction of SURVEY
 * §8(c) O1-O5 (the paper leaves training unspecified) and the readings
 * R1..R13 listed in DESIGN.md §3. No blocking, fusion or reordering beyond what
 * the algorithms state. Library primitives used as steps: qsort (sample sort,
 * guard fallback, reference sort), fma/floor from libm.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math (no contraction: the only
 * fused multiply-add is the explicit fma() of the leaf line, O6).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.
 */
#include "ls2_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* PMAX = 1 - 2^-52: the largest prediction, so floor(PMAX*f) < f (R10). */
static const double PMAX = 1.0 - 0x1p-52;

void lso_config_default(lso_config *cfg) {
    cfg->fanout = 1000;       /* P:328 "default fan-out parameter was 1000" */
    cfg->leaf_count = 1000;   /* P:328 "two layers and 1000 leaf models"   */
    cfg->sample_stride = 100; /* P:328 "1% sample"; strided reading R9      */
    cfg->frag_capacity = 100; /* P:328 "fragment capacities were capped at 100" */
}

/* ---------------------------------------------------------------- keys -- */

/* ord: IEEE totalOrder key for binary64 (sign-magnitude -> biased), identity
 * for u64 (R12). x precedes y iff ord(x) < ord(y). */
uint64_t lso_ord(uint64_t bits, int dtype) {
    if (dtype == LSO_U64) return bits;
    return (bits >> 63) ? ~bits : (bits | 0x8000000000000000ULL);
}

double lso_xd(uint64_t bits, int dtype) {
    if (dtype == LSO_U64) return (double)bits; /* round-to-nearest-even */
    double d;
    memcpy(&d, &bits, sizeof d);
    return d;
}

static int is_nan_bits(uint64_t bits) {
    return (bits & 0x7fffffffffffffffULL) > 0x7ff0000000000000ULL;
}

static int is_finite_key(uint64_t bits, int dtype) {
    if (dtype == LSO_U64) return 1;
    return (bits & 0x7ff0000000000000ULL) != 0x7ff0000000000000ULL;
}

/* clampd with ordered comparisons; a NaN argument maps to lo (R13). Never
 * fmin/fmax (signed-zero behaviour is implementation-defined). */
static double clampd(double v, double lo, double hi) {
    return v >= lo ? (v <= hi ? v : hi) : lo;
}

static int g_qsort_dtype; /* qsort has no context argument; the oracle is single-threaded */

static int cmp_ord(const void *a, const void *b) {
    uint64_t x = lso_ord(*(const uint64_t *)a, g_qsort_dtype);
    uint64_t y = lso_ord(*(const uint64_t *)b, g_qsort_dtype);
    return (x > y) - (x < y);
}

void lso_reference_sort(uint64_t *A, uint64_t n, int dtype) {
    g_qsort_dtype = dtype;
    qsort(A, (size_t)n, sizeof(uint64_t), cmp_ord);
}

/* --------------------------------------------------------------- model -- */

/* O3: root routing, a min-max linear map onto [0, L). */
static uint64_t route(const lso_model *m, double x) {
    double xc = clampd(x, m->xmin, m->xmax);
    double r = (xc - m->xmin) * m->root_scale;
    double last = (double)(m->leaf_count - 1);
    return (r < last) ? (uint64_t)(int64_t)r : (uint64_t)(m->leaf_count - 1);
}

/* O1-O5. The paper: "trained with a uniformly selected 1% sample"; the
 * model "takes a key (x) and returns the count of keys ... less than x". */
int lso_train(const uint64_t *keys, uint64_t n, int dtype, uint32_t stride,
              uint32_t leaf_count, lso_model *out) {
    if (n == 0 || stride == 0 || leaf_count == 0 || leaf_count > LSO_MAX_LEAVES)
        return LSO_E_INVALID;
    memset(out, 0, sizeof *out);
    out->leaf_count = leaf_count;

    /* O1: strided sample S[k] = A[k*s], k < m = ceil(n/s); sorted by ord. */
    uint64_t m = (n + stride - 1) / stride;
    uint64_t *S = (uint64_t *)malloc(m * sizeof(uint64_t));
    double *y = (double *)malloc(m * sizeof(double));
    if (!S || !y) { free(S); free(y); return LSO_E_INTERNAL; }
    for (uint64_t k = 0; k < m; k++) S[k] = keys[k * stride];
    lso_reference_sort(S, m, dtype);
    out->n_sample = m;

    /* O2: range of the finite sample entries. */
    uint64_t kf = m, kl = m;
    for (uint64_t k = 0; k < m; k++)
        if (is_finite_key(S[k], dtype)) { if (kf == m) kf = k; kl = k; }
    if (kf == m || lso_xd(S[kf], dtype) == lso_xd(S[kl], dtype)) {
        /* degenerate model: p == 0 everywhere */
        double v = (kf == m) ? 0.0 : lso_xd(S[kf], dtype);
        out->xmin = out->xmax = v;
        out->root_scale = 0.0;
        out->degenerate = 1;
        free(S); free(y);
        return LSO_OK;
    }
    out->xmin = lso_xd(S[kf], dtype);
    out->xmax = lso_xd(S[kl], dtype);
    out->root_scale = (double)leaf_count / (out->xmax - out->xmin);

    /* O4: y_k = first(k)/m, first(k) = smallest index holding a key equal to S[k]
     * (the strict-less eCDF of the sample; R8). */
    uint64_t first = 0;
    for (uint64_t k = 0; k < m; k++) {
        if (k > 0 && S[k] != S[k - 1]) first = k;
        y[k] = (double)first / (double)m;
    }

    /* O3 + O5: route the sorted sample; leaf l owns [beg_l, end_l). Chord
     * through the leaf's first sample key and the next leaf's first key. */
    uint64_t k = 0;
    for (uint32_t l = 0; l < leaf_count; l++) {
        uint64_t beg = k;
        while (k < m && route(out, lso_xd(S[k], dtype)) == l) k++;
        uint64_t end = k;
        double x1, y1;
        if (end < m) {
            x1 = clampd(lso_xd(S[end], dtype), out->xmin, out->xmax);
            y1 = y[end];
        } else {
            x1 = out->xmax;
            y1 = PMAX;
        }
        double hi = (y1 < PMAX) ? y1 : PMAX;
        lso_leaf *L = &out->leaf[l];
        if (end > beg) {
            double x0 = clampd(lso_xd(S[beg], dtype), out->xmin, out->xmax);
            double y0 = y[beg];
            L->a = (x1 > x0) ? (y1 - y0) / (x1 - x0) : 0.0;
            L->c = x0;
            L->b = y0;
            L->lo = y0;
            L->hi = hi;
        } else {
            L->a = 0.0;
            L->c = 0.0;
            L->b = hi;
            L->lo = hi;
            L->hi = hi;
        }
    }
    free(S);
    free(y);
    if (k != m) return LSO_E_INTERNAL; /* routing was not monotone */
    return LSO_OK;
}

/* O6: p = F_A(x) in [0, PMAX]. The "+ 0.0" turns -0.0 into +0.0. */
double lso_predict(const lso_model *m, uint64_t bits, int dtype) {
    double xc = clampd(lso_xd(bits, dtype), m->xmin, m->xmax);
    uint64_t l = route(m, xc);
    const lso_leaf *L = &m->leaf[l];
    double y = fma(L->a, xc - L->c, L->b);
    return clampd(y, L->lo, L->hi) + 0.0;
}

/* O7 / Alg.1: pos = F_A(x)·f^{1+p} − p·(i·f), truncated and clamped. */
uint64_t lso_bucket_l0(double p, uint32_t f) {
    int64_t b = (int64_t)(p * (double)f);
    return (uint64_t)(b < (int64_t)f - 1 ? b : (int64_t)f - 1);
}

uint64_t lso_bucket_l1(double p, uint32_t f, uint64_t parent) {
    double F2 = (double)f * (double)f;
    int64_t b = (int64_t)(p * F2) - (int64_t)parent * (int64_t)f;
    if (b < 0) b = 0;
    if (b > (int64_t)f - 1) b = (int64_t)f - 1;
    return (uint64_t)b;
}

/* Alg.2: adj = (i·f+j)/f², pos = [F_A(x) − adj]·A.size, floored and
 * clamped into the n'-slot histogram (R5). */
uint64_t lso_cs_pos(double p, uint64_t i, uint64_t j, uint32_t f, uint64_t n_total,
                    uint64_t nprime) {
    double F2 = (double)f * (double)f;
    double adj = (double)(i * (uint64_t)f + j) / F2;
    double v = floor((p - adj) * (double)n_total);
    double top = (double)(nprime - 1);
    return (uint64_t)(int64_t)clampd(v, 0.0, top);
}

static uint64_t bucket_of(const lso_model *m, uint64_t x, int dtype, int level,
                          uint64_t parent, uint32_t f) {
    double p = lso_predict(m, x, dtype);
    return level == 0 ? lso_bucket_l0(p, f) : lso_bucket_l1(p, f, parent);
}

/* ------------------------------------------------------------- Alg. 1 --- */

uint64_t lso_partition(uint64_t *A, uint64_t n, const lso_model *m, int dtype, int level,
                       uint64_t parent, uint32_t f, uint32_t c, uint64_t *S_B, lso_frag *S_F) {
    /* Frag <- f fragments of capacity c; S_B <- [0]*f; S_F <- []; w <- 0 */
    uint64_t *Frag = (uint64_t *)malloc((size_t)f * c * sizeof(uint64_t));
    uint64_t *fill = (uint64_t *)calloc(f, sizeof(uint64_t));
    if (!Frag || !fill) { free(Frag); free(fill); return (uint64_t)-1; }
    memset(S_B, 0, (size_t)f * sizeof(uint64_t));
    uint64_t nfrag = 0, w = 0;

    for (uint64_t k = 0; k < n; k++) {              /* for x in A */
        uint64_t x = A[k];
        uint64_t pos = bucket_of(m, x, dtype, level, parent, f); /* predict */
        Frag[pos * c + fill[pos]++] = x;            /* Frag[pos].append(x) */
        S_B[pos]++;                                 /* S_B[pos]++ */
        if (fill[pos] == c) {                       /* fragment is full */
            memcpy(&A[w], &Frag[pos * c], (size_t)c * sizeof(uint64_t));
            w += c;
            S_F[nfrag].bucket = pos;
            S_F[nfrag].size = c;
            nfrag++;
            fill[pos] = 0;                          /* Frag[pos].clear() */
        }
    }
    /* copy the remaining fragments that were not full; the loop
     * clears Frag[i] (P:132 typo, R2); empty fragments are not logged */
    for (uint32_t i = 0; i < f; i++) {
        uint64_t s = fill[i];
        if (s == 0) continue;
        memcpy(&A[w], &Frag[(uint64_t)i * c], (size_t)s * sizeof(uint64_t));
        S_F[nfrag].bucket = i;
        S_F[nfrag].size = s;
        nfrag++;
        w += s;
        fill[i] = 0;
    }
    free(Frag);
    free(fill);
    if (w != n) return (uint64_t)-1;
    return nfrag;
}

/* Defragment: place sibling fragments of each bucket contiguously (P:267,
 * Fig.3c), fragments of a bucket in log order (S:161 reference mode). */
int lso_defragment(uint64_t *A, uint64_t n, uint32_t f, const uint64_t *S_B,
                   const lso_frag *S_F, uint64_t nfrag, uint64_t *scratch) {
    uint64_t *cursor = (uint64_t *)malloc((size_t)f * sizeof(uint64_t));
    uint64_t *seen = (uint64_t *)calloc(f, sizeof(uint64_t));
    if (!cursor || !seen) { free(cursor); free(seen); return LSO_E_INTERNAL; }
    uint64_t start = 0;
    for (uint32_t b = 0; b < f; b++) { cursor[b] = start; start += S_B[b]; }
    int rc = LSO_OK;
    if (start != n) rc = LSO_E_INTERNAL;
    uint64_t r = 0;
    for (uint64_t q = 0; q < nfrag && rc == LSO_OK; q++) {
        uint64_t b = S_F[q].bucket, s = S_F[q].size;
        if (b >= f || r + s > n || seen[b] + s > S_B[b]) { rc = LSO_E_INTERNAL; break; }
        memcpy(&scratch[cursor[b]], &A[r], (size_t)s * sizeof(uint64_t));
        cursor[b] += s;
        seen[b] += s;
        r += s;
    }
    if (rc == LSO_OK && r != n) rc = LSO_E_INTERNAL;
    for (uint32_t b = 0; b < f && rc == LSO_OK; b++)
        if (seen[b] != S_B[b]) rc = LSO_E_INTERNAL;
    if (rc == LSO_OK) memcpy(A, scratch, (size_t)n * sizeof(uint64_t));
    free(cursor);
    free(seen);
    return rc;
}

/* Is-Homogeneous: "all the elements in the bucket are equal"; equality
 * is bit equality of ord (R11); empty and single-key ranges are homogeneous. */
int lso_is_homogeneous(const uint64_t *A, uint64_t n, int dtype) {
    for (uint64_t k = 1; k < n; k++)
        if (lso_ord(A[k], dtype) != lso_ord(A[0], dtype)) return 0;
    return 1;
}

/* ------------------------------------------------------------- Alg. 2 --- */

uint64_t lso_counting_sort(uint64_t *A, uint64_t nprime, const lso_model *m, int dtype,
                           uint64_t i, uint64_t j, uint32_t f, uint64_t n_total,
                           uint64_t *K, uint64_t *T) {
    memset(K, 0, (size_t)nprime * sizeof(uint64_t));         /* K <- [0]*n' */
    for (uint64_t k = 0; k < nprime; k++) {                   /* histogram */
        double p = lso_predict(m, A[k], dtype);
        K[lso_cs_pos(p, i, j, f, n_total, nprime)]++;
    }
    uint64_t max_group = 0;
    for (uint64_t k = 0; k < nprime; k++)
        if (K[k] > max_group) max_group = K[k];
    for (uint64_t k = 1; k < nprime; k++) K[k] += K[k - 1]; /* running totals */
    for (uint64_t k = 0; k < nprime; k++) {                   /* placement (R4) */
        double p = lso_predict(m, A[k], dtype);
        uint64_t pos = lso_cs_pos(p, i, j, f, n_total, nprime);
        K[pos]--;
        T[K[pos]] = A[k];
    }
    memcpy(A, T, (size_t)nprime * sizeof(uint64_t));        /* copy back */
    return max_group;
}

uint64_t lso_insertion_sort(uint64_t *A, uint64_t n, int dtype, uint64_t guard_limit,
                            int *guard_fired) {
    uint64_t shifts = 0;
    if (guard_fired) *guard_fired = 0;
    for (uint64_t k = 1; k < n; k++) {
        uint64_t x = A[k], o = lso_ord(x, dtype);
        uint64_t j = k;
        while (j > 0 && lso_ord(A[j - 1], dtype) > o) {
            A[j] = A[j - 1];
            j--;
            shifts++;
        }
        A[j] = x;
        if (guard_limit && shifts > guard_limit) {
            /* O11 guard (documented deviation): same result, bounded time */
            lso_reference_sort(A, n, dtype);
            if (guard_fired) *guard_fired = 1;
            return shifts;
        }
    }
    return shifts;
}

int lso_sort(uint64_t *A, uint64_t n, int dtype, const lso_config *cfg_in,
             const lso_model *inject, lso_model *model_out, lso_dumps *dumps,
             lso_stats *stats) {
    lso_config cfg;
    if (cfg_in) cfg = *cfg_in; else lso_config_default(&cfg);
    const uint32_t f = cfg.fanout, c = cfg.frag_capacity;
    if (dtype != LSO_F64 && dtype != LSO_U64) return LSO_E_INVALID;
    if (f < 2 || c < 1 || cfg.sample_stride < 1 || cfg.leaf_count < 1 ||
        cfg.leaf_count > LSO_MAX_LEAVES)
        return LSO_E_INVALID;
    lso_stats st;
    memset(&st, 0, sizeof st);

    /* O0: NaN -> error before any mutation */
    if (dtype == LSO_F64)
        for (uint64_t k = 0; k < n; k++)
            if (is_nan_bits(A[k])) return LSO_E_NAN;

    lso_model *model = (lso_model *)malloc(sizeof(lso_model));
    if (!model) return LSO_E_INTERNAL;
    int rc = LSO_OK;
    if (n <= 1) {
        memset(model, 0, sizeof *model);
        model->leaf_count = cfg.leaf_count;
        model->degenerate = 1;
        if (inject) *model = *inject;
        if (model_out) *model_out = *model;
        if (stats) *stats = st;
        if (dumps) {
            for (uint64_t k = 0; k < n; k++) {
                if (dumps->p) dumps->p[k] = lso_predict(model, A[k], dtype);
                if (dumps->b0) dumps->b0[k] = (uint32_t)lso_bucket_l0(lso_predict(model, A[k], dtype), f);
            }
        }
        free(model);
        return LSO_OK;
    }
    if (inject) *model = *inject;
    else rc = lso_train(A, n, dtype, cfg.sample_stride, cfg.leaf_count, model);
    if (rc != LSO_OK) { free(model); return rc; }
    if (model_out) *model_out = *model;

    const uint64_t ff = (uint64_t)f * f;
    /* per-key dumps in input order, before any mutation */
    const int want_raw = dumps && (dumps->pos || dumps->hist1_raw);
    uint64_t *hist1_raw = want_raw ? (uint64_t *)calloc(ff, sizeof(uint64_t)) : NULL;
    if (want_raw && !hist1_raw) { free(model); return LSO_E_INTERNAL; }
    for (uint64_t k = 0; k < n && dumps; k++) {
        double p = lso_predict(model, A[k], dtype);
        uint64_t b0 = lso_bucket_l0(p, f), b1 = lso_bucket_l1(p, f, b0);
        if (hist1_raw) hist1_raw[b0 * f + b1]++;
        if (dumps && dumps->p) dumps->p[k] = p;
        if (dumps && dumps->b0) dumps->b0[k] = (uint32_t)b0;
        if (dumps && dumps->b1) dumps->b1[k] = (uint32_t)b1;
    }
    if (dumps && dumps->pos) {
        for (uint64_t k = 0; k < n; k++) {
            double p = lso_predict(model, A[k], dtype);
            uint64_t b0 = lso_bucket_l0(p, f), b1 = lso_bucket_l1(p, f, b0);
            dumps->pos[k] = (uint32_t)lso_cs_pos(p, b0, b1, f, n, hist1_raw[b0 * f + b1]);
        }
    }
    if (dumps && dumps->hist1_raw) memcpy(dumps->hist1_raw, hist1_raw, ff * sizeof(uint64_t));
    free(hist1_raw);

    uint64_t *S_B = (uint64_t *)calloc(f, sizeof(uint64_t));
    uint64_t *S_B1 = (uint64_t *)calloc(f, sizeof(uint64_t));
    lso_frag *S_F = (lso_frag *)malloc((n / c + f + 1) * sizeof(lso_frag));
    uint64_t *scratch = (uint64_t *)malloc(n * sizeof(uint64_t));
    uint64_t *K = (uint64_t *)malloc(n * sizeof(uint64_t));
    if (!S_B || !S_B1 || !S_F || !scratch || !K) { rc = LSO_E_INTERNAL; goto done; }
    if (dumps && dumps->S_B1) memset(dumps->S_B1, 0, ff * sizeof(uint64_t));
    if (dumps && dumps->H0) memset(dumps->H0, 0, f);
    if (dumps && dumps->H1) memset(dumps->H1, 0, ff);

    /* Model-based partitioning (level 0), then Defragment */
    uint64_t nfrag = lso_partition(A, n, model, dtype, 0, 0, f, c, S_B, S_F);
    if (nfrag == (uint64_t)-1) { rc = LSO_E_INTERNAL; goto done; }
    rc = lso_defragment(A, n, f, S_B, S_F, nfrag, scratch);
    if (rc != LSO_OK) goto done;
    if (dumps && dumps->S_B) memcpy(dumps->S_B, S_B, f * sizeof(uint64_t));

    /* Re-partition each bucket in f sub-buckets */
    uint64_t r = 0; /* read head */
    for (uint32_t i = 0; i < f; i++) {
        uint64_t nb = S_B[i], s = r;
        if (lso_is_homogeneous(&A[s], nb, dtype)) {
            if (dumps && dumps->H0) dumps->H0[i] = 1;
            if (nb >= 2) { st.h0_buckets++; st.h0_keys += nb; }
            r += nb; /* skip this bucket */
            continue;
        }
        uint64_t nf1 = lso_partition(&A[s], nb, model, dtype, 1, i, f, c, S_B1, S_F);
        if (nf1 == (uint64_t)-1) { rc = LSO_E_INTERNAL; goto done; }
        rc = lso_defragment(&A[s], nb, f, S_B1, S_F, nf1, scratch);
        if (rc != LSO_OK) goto done;
        if (dumps && dumps->S_B1) memcpy(&dumps->S_B1[(uint64_t)i * f], S_B1, f * sizeof(uint64_t));
        for (uint32_t j = 0; j < f; j++) {                 /* iterate the sub-buckets */
            uint64_t np = S_B1[j], sp = r;
            if (lso_is_homogeneous(&A[sp], np, dtype)) {
                if (dumps && dumps->H1) dumps->H1[(uint64_t)i * f + j] = 1;
                if (np >= 2) { st.h1_subbuckets++; st.h1_keys += np; }
            } else {
                uint64_t g = lso_counting_sort(&A[sp], np, model, dtype, i, j, f, n, K, scratch);
                st.counting_sorts++;
                if (g > st.max_group) st.max_group = g;
                if (np > st.max_subbucket) st.max_subbucket = np;
                /* touch-up, per sub-bucket: equivalent to the global pass
                 * because p is monotone (R15); guarded (O11) */
                int fired = 0;
                st.shifts += lso_insertion_sort(&A[sp], np, dtype, 32 * np + 4096, &fired);
                st.guard_fired += (uint64_t)fired;
            }
            r += np; /* update the read head */
        }
    }
    if (r != n) { rc = LSO_E_INTERNAL; goto done; }
    /* the touch-up "guarantees that the input has been monotonically ordered" */
    for (uint64_t k = 1; k < n; k++)
        if (lso_ord(A[k - 1], dtype) > lso_ord(A[k], dtype)) { rc = LSO_E_INTERNAL; goto done; }
done:
    if (stats) *stats = st;
    free(S_B); free(S_B1); free(S_F); free(scratch); free(K); free(model);
    return rc;
}
