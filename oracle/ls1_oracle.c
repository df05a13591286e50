/*
 * ls1_oracle.c -- TEST INFRASTRUCTURE ONLY (not the product path).
 *
 * the original LearnedSort ("LearnedSort 1.0") as a CPU
 * oracle variant, so that the paper's LS 2.0 / LS 1.0 ratios (4.78x on
 * high-duplicate inputs, 1.60x elsewhere: P:27) can be put in
 * context on the same host. Context only, never a target.
 *
 * The paper describes LS 1.0 in prose only (Fig. 1 caption P:49, P:58, P:65,
 * P:76); the steps below follow that prose in its order:
 *   1. train the eCDF model on a sample -- the same model as the
 *      LS 2.0 oracle (lso_train), so the two variants
 *      differ only where the paper says they differ;
 *   2. "exception-based" duplicates: keys that repeat in the sample
 *      are "problematic"; an associative table (a hash table) counts
 *      their occurrences during the sort and they skip partitioning;
 *   3. partition into FIXED-capacity buckets by the model's prediction
 *      ("fixed-capacity buckets", "the same capacity to every
 *      bucket"); a key whose bucket is full goes to the spill bucket (P:58,
 *      P:65); one more round of the same inside every bucket ("for
 *      another round until the buckets get small");
 *   4. model-based counting sort inside every sub-bucket, then the
 *      insertion-sort clean-up;
 *   5. the spill bucket is sorted by a comparison sort (std::sort in the
 *      paper; qsort here) and merged with the partitioned keys, and the
 *      problematic keys are re-written from their counts.
 * Readings where the prose is silent (R-LS1a..d):
 *   a) capacities: level 0 cap0 = ceil(slack * n / f), level 1
 *      cap1 = ceil(slack * cap0 / f) for every bucket (fixed), slack
 *      1.1 by default; both can be given explicitly;
 *   b) a sample value is "problematic" when it occurs >= exc_min times in the
 *      sorted sample, exc_min = max(2, ceil(m / f)) by default (a value that
 *      alone is expected to fill a level-0 bucket);
 *   c) exactly two partitioning rounds with the same fan-out as LS 2.0;
 *   d) the insertion sort runs per sub-bucket (equal to one global pass
 *      because the model is monotone, R15), with the O11 guard.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this code.
 */
#include "ls2_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int g_ls1_dtype; /* qsort has no context argument; single-threaded */

static int cmp_ord1(const void *a, const void *b) {
    uint64_t x = lso_ord(*(const uint64_t *)a, g_ls1_dtype);
    uint64_t y = lso_ord(*(const uint64_t *)b, g_ls1_dtype);
    return (x > y) - (x < y);
}

void ls1o_config_default(ls1o_config *cfg) {
    cfg->fanout = 1000;      /* same f as LS 2.0, reading c */
    cfg->leaf_count = 1000;  /* same model */
    cfg->sample_stride = 100;
    cfg->slack = 1.1;        /* reading a */
    cfg->cap0 = 0;
    cfg->cap1 = 0;
    cfg->exc_min = 0;        /* reading b */
}

/* ------------------------------------------- the associative table */

typedef struct {
    uint64_t *key;   /* ord of the problematic key, valid where used[] */
    uint64_t *count; /* occurrences met during the sort */
    uint8_t *used;
    uint64_t mask;
} exc_table;

static uint64_t mix64(uint64_t z) { /* splitmix64 finaliser: the hash */
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27; z *= 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* slot of ord o (linear probing), or -1 if o is not a problematic key */
static int64_t exc_find(const exc_table *t, uint64_t o) {
    if (!t->mask) return -1;
    for (uint64_t h = mix64(o) & t->mask;; h = (h + 1) & t->mask) {
        if (!t->used[h]) return -1;
        if (t->key[h] == o) return (int64_t)h;
    }
}

static void exc_insert(exc_table *t, uint64_t o) {
    uint64_t h = mix64(o) & t->mask;
    while (t->used[h]) h = (h + 1) & t->mask;
    t->used[h] = 1;
    t->key[h] = o;
    t->count[h] = 0;
}

/* ------------------------------------------------------------- the sort -- */

int ls1o_sort(uint64_t *A, uint64_t n, int dtype, const ls1o_config *cfg_in, ls1o_stats *stats) {
    ls1o_config cfg;
    if (cfg_in) cfg = *cfg_in; else ls1o_config_default(&cfg);
    const uint32_t f = cfg.fanout;
    if (dtype != LSO_F64 && dtype != LSO_U64) return LSO_E_INVALID;
    if (f < 2 || cfg.sample_stride < 1 || cfg.leaf_count < 1 || cfg.leaf_count > LSO_MAX_LEAVES ||
        !(cfg.slack > 0.0))
        return LSO_E_INVALID;
    ls1o_stats st;
    memset(&st, 0, sizeof st);
    if (dtype == LSO_F64) /* NaN -> error before any mutation (as the LS 2.0 oracle) */
        for (uint64_t k = 0; k < n; k++)
            if ((A[k] & 0x7fffffffffffffffULL) > 0x7ff0000000000000ULL) return LSO_E_NAN;
    if (n <= 1) { if (stats) *stats = st; return LSO_OK; }

    int rc = LSO_OK;
    lso_model *model = (lso_model *)malloc(sizeof(lso_model));
    const uint64_t m = (n + cfg.sample_stride - 1) / cfg.sample_stride;
    uint64_t *smp = (uint64_t *)malloc(m * sizeof(uint64_t));
    exc_table X;
    memset(&X, 0, sizeof X);
    uint64_t *B0 = NULL, *B1 = NULL, *cnt0 = NULL, *cnt1 = NULL, *spill = NULL, *main_ = NULL;
    uint64_t *K = NULL, *T = NULL;
    if (!model || !smp) { rc = LSO_E_INTERNAL; goto done; }

    /* 1. the model */
    rc = lso_train(A, n, dtype, cfg.sample_stride, cfg.leaf_count, model);
    if (rc != LSO_OK) goto done;

    /* 2. problematic keys from the (sorted) sample (reading b) */
    for (uint64_t k = 0; k < m; k++) smp[k] = A[k * cfg.sample_stride];
    g_ls1_dtype = dtype;
    qsort(smp, (size_t)m, sizeof(uint64_t), cmp_ord1);
    {
        uint64_t emin = cfg.exc_min ? cfg.exc_min : (m + f - 1) / f;
        if (emin < 2) emin = 2;
        uint64_t nexc = 0;
        for (uint64_t k = 0; k < m;) {
            uint64_t e = k;
            while (e < m && lso_ord(smp[e], dtype) == lso_ord(smp[k], dtype)) e++;
            if (e - k >= emin) nexc++;
            k = e;
        }
        if (nexc) {
            uint64_t sz = 4;
            while (sz < 2 * nexc) sz <<= 1;
            X.mask = sz - 1;
            X.key = (uint64_t *)malloc(sz * sizeof(uint64_t));
            X.count = (uint64_t *)malloc(sz * sizeof(uint64_t));
            X.used = (uint8_t *)calloc(sz, 1);
            if (!X.key || !X.count || !X.used) { rc = LSO_E_INTERNAL; goto done; }
            for (uint64_t k = 0; k < m;) {
                uint64_t e = k;
                while (e < m && lso_ord(smp[e], dtype) == lso_ord(smp[k], dtype)) e++;
                if (e - k >= emin) exc_insert(&X, lso_ord(smp[k], dtype));
                k = e;
            }
        }
        st.exception_values = nexc;
    }

    /* 3. level 0: fixed-capacity buckets, overflow to the spill bucket */
    const uint64_t cap0 = cfg.cap0 ? cfg.cap0 : (uint64_t)ceil(cfg.slack * (double)n / f);
    const uint64_t cap1 = cfg.cap1 ? cfg.cap1 : (uint64_t)ceil(cfg.slack * (double)cap0 / f);
    B0 = (uint64_t *)malloc((size_t)f * cap0 * sizeof(uint64_t));
    cnt0 = (uint64_t *)calloc(f, sizeof(uint64_t));
    B1 = (uint64_t *)malloc((size_t)f * cap1 * sizeof(uint64_t));
    cnt1 = (uint64_t *)calloc(f, sizeof(uint64_t));
    spill = (uint64_t *)malloc(n * sizeof(uint64_t));
    main_ = (uint64_t *)malloc(n * sizeof(uint64_t));
    K = (uint64_t *)malloc(cap1 * sizeof(uint64_t));
    T = (uint64_t *)malloc(cap1 * sizeof(uint64_t));
    if (!B0 || !cnt0 || !B1 || !cnt1 || !spill || !main_ || !K || !T) { rc = LSO_E_INTERNAL; goto done; }
    uint64_t nspill = 0, nmain = 0;
    for (uint64_t k = 0; k < n; k++) {
        const int64_t h = exc_find(&X, lso_ord(A[k], dtype));
        if (h >= 0) { X.count[h]++; st.exception_keys++; continue; } /* skip partitioning */
        const uint64_t b = lso_bucket_l0(lso_predict(model, A[k], dtype), f);
        if (cnt0[b] < cap0) B0[b * cap0 + cnt0[b]++] = A[k];
        else spill[nspill++] = A[k];
    }
    st.spill_l0 = nspill;

    /* level 1 inside every bucket, then 4. counting sort + insertion sort */
    for (uint32_t i = 0; i < f; i++) {
        memset(cnt1, 0, f * sizeof(uint64_t));
        for (uint64_t k = 0; k < cnt0[i]; k++) {
            const uint64_t x = B0[i * cap0 + k];
            const uint64_t j = lso_bucket_l1(lso_predict(model, x, dtype), f, i);
            if (cnt1[j] < cap1) B1[j * cap1 + cnt1[j]++] = x;
            else spill[nspill++] = x;
        }
        for (uint32_t j = 0; j < f; j++) {
            uint64_t *S = &B1[j * cap1];
            const uint64_t np = cnt1[j];
            if (np == 0) continue;
            lso_counting_sort(S, np, model, dtype, i, j, f, n, K, T);
            int fired = 0;
            st.shifts += lso_insertion_sort(S, np, dtype, 32 * np + 4096, &fired);
            st.guard_fired += (uint64_t)fired;
            memcpy(&main_[nmain], S, np * sizeof(uint64_t));
            nmain += np;
        }
    }
    st.spill_keys = nspill;

    /* 5. sort the spill bucket (std::sort in the paper), then merge the three
     * sorted streams: partitioned keys, spill, problematic keys by count */
    g_ls1_dtype = dtype;
    qsort(spill, (size_t)nspill, sizeof(uint64_t), cmp_ord1);
    {
        /* problematic keys in order: sorted slots of the table */
        uint64_t nx = 0;
        uint64_t *xs = NULL;
        if (X.mask) {
            xs = (uint64_t *)malloc((X.mask + 1) * 2 * sizeof(uint64_t));
            if (!xs) { rc = LSO_E_INTERNAL; goto done; }
            for (uint64_t h = 0; h <= X.mask; h++)
                if (X.used[h] && X.count[h]) { xs[2 * nx] = X.key[h]; xs[2 * nx + 1] = X.count[h]; nx++; }
            /* (insertion sort by ord: the table holds few keys) */
            for (uint64_t a = 1; a < nx; a++) {
                uint64_t o = xs[2 * a], c = xs[2 * a + 1], b = a;
                while (b > 0 && xs[2 * (b - 1)] > o) { xs[2 * b] = xs[2 * (b - 1)]; xs[2 * b + 1] = xs[2 * (b - 1) + 1]; b--; }
                xs[2 * b] = o; xs[2 * b + 1] = c;
            }
        }
        uint64_t a = 0, s = 0, x = 0, w = 0;
        while (w < n) {
            const uint64_t oa = a < nmain ? lso_ord(main_[a], dtype) : UINT64_MAX;
            const uint64_t os = s < nspill ? lso_ord(spill[s], dtype) : UINT64_MAX;
            const uint64_t ox = x < nx ? xs[2 * x] : UINT64_MAX;
            if (a < nmain && oa <= os && oa <= ox) A[w++] = main_[a++];
            else if (s < nspill && os <= ox) A[w++] = spill[s++];
            else if (x < nx) {
                /* re-write the problematic key from its count */
                uint64_t bits = xs[2 * x];
                if (dtype == LSO_F64) /* ord -> bits (inverse of lso_ord) */
                    bits = (bits >> 63) ? (bits & 0x7fffffffffffffffULL) : ~bits;
                for (uint64_t c = 0; c < xs[2 * x + 1]; c++) A[w++] = bits;
                x++;
            } else { rc = LSO_E_INTERNAL; break; }
        }
        free(xs);
        if (rc == LSO_OK && (a != nmain || s != nspill || x != nx)) rc = LSO_E_INTERNAL;
    }
    for (uint64_t k = 1; rc == LSO_OK && k < n; k++)
        if (lso_ord(A[k - 1], dtype) > lso_ord(A[k], dtype)) rc = LSO_E_INTERNAL;
done:
    if (stats) *stats = st;
    free(model); free(smp); free(X.key); free(X.count); free(X.used);
    free(B0); free(cnt0); free(B1); free(cnt1); free(spill); free(main_); free(K); free(T);
    return rc;
}
