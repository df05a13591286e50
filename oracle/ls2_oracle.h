/*
 * ls2_oracle.h -- TEST INFRASTRUCTURE ONLY (not the product path).
 *
 * A plain, slow, single-threaded CPU oracle of LearnedSort 2.0
 * (Kristo, Vaidya, Kraska, "Defeating duplicates: A re-design of the
 * LearnedSort algorithm", arXiv 2107.03290). Citations: P:n = line n of
 * /root/reference/PAPER.md, S:n = line n of SPEC.md, SURVEY §8(c) Ox = the
 * step list the oracle follows, Rn = a reading listed in DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load this library. It shares no code, header,
 * constant or helper with the CUDA path (paper_2107_03290_b200/csrc, include/).
 *
 * Keys are passed as raw 64-bit patterns (uint64_t); dtype says how to read
 * them (0 = IEEE binary64, 1 = unsigned 64-bit integer).
 */
#ifndef LS2_ORACLE_H
#define LS2_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSO_F64 0
#define LSO_U64 1

#define LSO_OK 0
#define LSO_E_INVALID 1
#define LSO_E_NAN 2
#define LSO_E_INTERNAL 7

#define LSO_MAX_LEAVES 4096

/* One leaf line: p = clamp(fma(a, xc - c, b), lo, hi) */
typedef struct {
    double a, c, b, lo, hi;
} lso_leaf;

/* Two-layer model F_A: a min-max linear root plus L linear leaves. */
typedef struct {
    uint32_t leaf_count; /* L */
    uint32_t degenerate; /* 1 if the sample had < 2 distinct finite values (O2) */
    uint64_t n_sample;   /* m */
    double xmin, xmax, root_scale;
    lso_leaf leaf[LSO_MAX_LEAVES];
} lso_model;

/* Alg. 1's S_F entries, extended with the bucket id (paper gap; R3). */
typedef struct {
    uint64_t bucket, size;
} lso_frag;

typedef struct {
    uint32_t fanout;        /* f   (1000)        */
    uint32_t leaf_count;    /* L   (1000 leaves) */
    uint32_t sample_stride; /* s   (1% sample => 100) */
    uint32_t frag_capacity; /* c   (100) */
} lso_config;

/* Optional outputs. Every pointer may be NULL. Per-key arrays are indexed by
 * INPUT position (values are functions of (key, model, n, raw level-1 counts)). */
typedef struct {
    double *p;         /* [n]  F_A(x)                                   */
    uint32_t *b0;      /* [n]  level-0 bucket                            */
    uint32_t *b1;      /* [n]  level-1 sub-bucket (parent = own b0)      */
    uint32_t *pos;     /* [n]  counting-sort slot with n' = raw hist1    */
    uint64_t *S_B;     /* [f]     level-0 bucket sizes (Alg.1 output)    */
    uint64_t *S_B1;    /* [f*f]   level-1 sizes S'_B; rows of H0 buckets are 0 */
    uint64_t *hist1_raw; /* [f*f] histogram of (b0,b1) over all keys     */
    uint8_t *H0;       /* [f]     homogeneous level-0 buckets            */
    uint8_t *H1;       /* [f*f]   homogeneous sub-buckets (rows of H0 buckets are 0) */
} lso_dumps;

typedef struct {
    uint64_t h0_buckets, h0_keys;          /* homogeneous level-0 buckets with >= 2 keys */
    uint64_t h1_subbuckets, h1_keys;       /* homogeneous sub-buckets with >= 2 keys     */
    uint64_t counting_sorts;               /* Alg.2 counting-sort invocations            */
    uint64_t shifts;                       /* insertion-sort shifts                      */
    uint64_t guard_fired;                  /* O11 guard firings                          */
    uint64_t max_group;                    /* largest run of equal pos                   */
    uint64_t max_subbucket;                /* largest sub-bucket that was counting-sorted */
} lso_stats;

void lso_config_default(lso_config *cfg);

/* ord(x): the total order key (SURVEY §8(c) "Definitions"; R12). */
uint64_t lso_ord(uint64_t bits, int dtype);
/* xd(x): the key as binary64 (round-to-nearest-even for u64). */
double lso_xd(uint64_t bits, int dtype);

/* O1-O5: strided sample, sort, eCDF targets, chord fit. stride >= 1, n >= 1. */
int lso_train(const uint64_t *keys, uint64_t n, int dtype, uint32_t stride,
              uint32_t leaf_count, lso_model *out);
/* O6 */
double lso_predict(const lso_model *m, uint64_t bits, int dtype);
/* O7 (Alg.1 P:107 read as f^{1+p} and p·(i·f); R1) */
uint64_t lso_bucket_l0(double p, uint32_t f);
uint64_t lso_bucket_l1(double p, uint32_t f, uint64_t parent);
/* Alg.2 P:188-190 with the clamp reading R5 */
uint64_t lso_cs_pos(double p, uint64_t i, uint64_t j, uint32_t f, uint64_t n_total,
                    uint64_t nprime);

/* Alg. 1. Writes S_B[f] and the fragment log; returns #fragments
 * or (uint64_t)-1 on error. S_F must hold n/c + f entries. */
uint64_t lso_partition(uint64_t *A, uint64_t n, const lso_model *m, int dtype, int level,
                       uint64_t parent, uint32_t f, uint32_t c, uint64_t *S_B, lso_frag *S_F);
/* Defragment (S:161 reference mode). scratch holds n keys.
 * Returns LSO_OK or LSO_E_INTERNAL ("corrupt partition state"). */
int lso_defragment(uint64_t *A, uint64_t n, uint32_t f, const uint64_t *S_B,
                   const lso_frag *S_F, uint64_t nfrag, uint64_t *scratch);
/* Is-Homogeneous (R11) */
int lso_is_homogeneous(const uint64_t *A, uint64_t n, int dtype);
/* Model-based counting sort of one sub-bucket (Alg.2). K has
 * nprime entries, T has nprime keys. Returns the largest run of equal pos. */
uint64_t lso_counting_sort(uint64_t *A, uint64_t nprime, const lso_model *m, int dtype,
                           uint64_t i, uint64_t j, uint32_t f, uint64_t n_total,
                           uint64_t *K, uint64_t *T);
/* Insertion sort touch-up with the O11 guard; returns shifts.
 * guard_limit = 0 disables the guard. */
uint64_t lso_insertion_sort(uint64_t *A, uint64_t n, int dtype, uint64_t guard_limit,
                            int *guard_fired);

/* The whole of Alg. 2. If `inject` is non-NULL it is used as F_A,
 * otherwise the model is trained by lso_train (O1-O5). model_out, dumps and
 * stats may be NULL. */
int lso_sort(uint64_t *A, uint64_t n, int dtype, const lso_config *cfg,
             const lso_model *inject, lso_model *model_out, lso_dumps *dumps,
             lso_stats *stats);

/* The plain definition of the result: sort by ord (qsort). */
void lso_reference_sort(uint64_t *A, uint64_t n, int dtype);

/* ---- LearnedSort 1.0 as an oracle variant (ls1_oracle.c).
 * Fixed-capacity buckets + spill bucket + exception table.
 * Context only (the paper's LS 2.0 / LS 1.0 ratios); readings R-LS1a..d. */
typedef struct {
    uint32_t fanout, leaf_count, sample_stride;
    double slack;     /* capacities = ceil(slack * expected size) (R-LS1a) */
    uint64_t cap0;    /* level-0 bucket capacity; 0 = ceil(slack * n / f)     */
    uint64_t cap1;    /* level-1 capacity; 0 = ceil(slack * cap0 / f)         */
    uint64_t exc_min; /* sample count of a problematic key; 0 = max(2, ceil(m/f)) (R-LS1b) */
} ls1o_config;

typedef struct {
    uint64_t spill_l0, spill_keys;          /* keys spilled at level 0 / in total   */
    uint64_t exception_values, exception_keys; /* problematic keys: table entries / keys counted */
    uint64_t shifts, guard_fired;
} ls1o_stats;

void ls1o_config_default(ls1o_config *cfg);
/* Sorts A[0..n) in place. Returns LSO_OK, LSO_E_INVALID, LSO_E_NAN or
 * LSO_E_INTERNAL. stats may be NULL. */
int ls1o_sort(uint64_t *A, uint64_t n, int dtype, const ls1o_config *cfg, ls1o_stats *stats);

#ifdef __cplusplus
}
#endif
#endif
