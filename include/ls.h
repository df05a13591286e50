/*
 * ls.h -- C ABI of libls.so: LearnedSort 2.0's data-parallel hot path on B200
 * (sm_100a). Kristo, Vaidya, Kraska, "Defeating duplicates: A re-design of the
 * LearnedSort algorithm", arXiv 2107.03290. P:n = PAPER.md line n, S:n =
 * SPEC.md line n, Rn = reading n in DESIGN.md §3.
 *
 * Conventions for every entry point:
 *   - Plain pointers and sizes only. "d_" pointers are DEVICE memory, "h_"
 *     pointers HOST memory; the caller allocates and owns every buffer (the
 *     library performs no cudaMalloc on the sort path). The only library-owned
 *     object is ls_comm.
 *   - Keys are 8-byte values: LS_F64 (IEEE binary64) or LS_U64 (unsigned
 *     64-bit). Order is IEEE totalOrder for f64 (-0.0 before +0.0; +-inf
 *     accepted) and the natural order for u64 (R12). NaN -> LS_E_NAN before
 *     any mutation.
 *   - n must be < 2^32. n <= 1 is a no-op returning LS_OK.
 *   - All work is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream). Calls that return a status or stats synchronise
 *     that stream once at the end. No C++ exception crosses the ABI; on any
 *     error the thread-local ls_last_error() describes it.
 */
#ifndef LS_H
#define LS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { LS_F64 = 0, LS_U64 = 1 } ls_dtype;

typedef enum {
    LS_OK = 0,
    LS_E_INVALID = 1,   /* bad argument, or an injected model that is not monotone-safe */
    LS_E_NAN = 2,       /* an fp64 NaN key; the input is left untouched          */
    LS_E_WORKSPACE = 3, /* ws_bytes smaller than ls_workspace_bytes()                     */
    LS_E_CAPACITY = 4,  /* ls_sort_multi: out_cap < n_out (n_out is still reported)       */
    LS_E_CUDA = 5,      /* a CUDA runtime error                                           */
    LS_E_NCCL = 6,      /* an NCCL error                                                  */
    LS_E_INTERNAL = 7   /* an invariant was violated ("corrupt partition state")   */
} ls_status;

#define LS_MAX_FANOUT 1024
#define LS_MAX_LEAVES 1024

/* flags */
#define LS_FLAG_PHASE_TIMING 0x1ULL /* record CUDA events between phases (ls_stats.phase_ms) */
#define LS_FLAG_VALIDATE_MODEL 0x2ULL /* ls_sort_with_model: reject unsafe models (default on) */
#define LS_FLAG_PEER_SCATTER 0x8ULL /* ls_sort_multi: the destination scatter stores
                                       every run straight into the destination rank's d_out (its
                                       allocation mapped here with CUDA IPC: NVLink peer stores),
                                       at this rank's slice of it; no send buffer, no NCCL
                                       all-to-all (NCCL still carries the samples, the counts,
                                       the handles and one closing all-reduce). d_out must be
                                       device memory that CUDA IPC can export (cudaMalloc /
                                       the PyTorch caching allocator). Same output. */
#define LS_FLAG_FUSED_ROUND1 0x4ULL /* ls_sort: partition every level-0 bucket of 64K..~219K keys
                                       with one 8-CTA cluster (count and scatter of
                                       round 1 in one kernel, the bucket staged in shared memory,
                                       the histogram exchanged through DSMEM). Same output, ids
                                       and S'_B; off by default: measured slower on B200
                                        */

/* Algorithm constants (fan-out 1000, 1000 leaves, 1% sample) and the
 * free tuning knob big_threshold (R-Q22: sub-buckets above it take the exact
 * big-bucket path instead of the shared-memory counting sort). */
typedef struct {
    uint32_t fanout;        /* f, 2..LS_MAX_FANOUT, default 1000            */
    uint32_t leaf_count;    /* L, 1..LS_MAX_LEAVES, default 1000            */
    uint32_t sample_stride; /* s >= 1, default 100 (strided 1% sample, R9)  */
    uint32_t fit;           /* 0 = chord fit (R7); the only fit implemented  */
    uint32_t big_threshold; /* T_small in keys, 64..4096, default 4096       */
    uint32_t reserved;
    uint64_t flags;         /* LS_FLAG_*                                      */
} ls_config;

void ls_config_default(ls_config *cfg);

/* One leaf line of F_A: p = clamp(fma(a, xc - c, b), lo, hi)  (R7, R13). */
typedef struct {
    double a, c, b, lo, hi;
} ls_leaf;

/* The two-layer eCDF model F_A: a min-max linear root routing
 * xc = clamp(x, xmin, xmax) to leaf floor((xc - xmin) * root_scale), and
 * leaf_count linear leaves. Host POD, caller-owned (~40 KB). */
typedef struct {
    uint32_t dtype, leaf_count;
    uint64_t n_sample;   /* m, the number of sample keys it was fitted on */
    uint32_t degenerate; /* 1: fewer than 2 distinct finite sample values, p == 0 */
    uint32_t reserved;
    double xmin, xmax, root_scale;
    ls_leaf leaf[LS_MAX_LEAVES];
} ls_model;

enum {
    LS_PHASE_FIT = 0, LS_PHASE_COUNT0, LS_PHASE_SCATTER0, LS_PHASE_COUNT1, LS_PHASE_SCATTER1,
    LS_PHASE_CLASSIFY, LS_PHASE_BUCKETSORT, LS_PHASE_BIG, LS_NUM_PHASES
};

typedef struct {
    uint64_t n;
    uint64_t h0_buckets, h0_keys;       /* homogeneous level-0 buckets with >= 2 keys */
    uint64_t h1_subbuckets, h1_keys;    /* homogeneous sub-buckets with >= 2 keys     */
    uint64_t small_subbuckets, small_keys; /* counting-sorted in shared memory    */
    uint64_t big_subbuckets, big_keys;  /* non-homogeneous sub-buckets > big_threshold        */
    uint64_t max_group;                 /* largest run of equal counting-sort positions       */
    uint64_t big_passes;                /* radix passes spent on big sub-buckets              */
    uint64_t kernel_launches;           /* kernels this call launched                         */
    uint64_t fused_buckets;             /* level-0 buckets partitioned cluster-resident (f2)  */
    uint64_t round0_exact;              /* 1: round 0 took the exact count pass (a sample-
                                           estimated bucket capacity did not hold)           */
    uint64_t peer_scatter;              /* ls_sort_multi: 1 if LS_FLAG_PEER_SCATTER's fused peer
                                           scatter ran (0: the NCCL all-to-all, also the collective
                                           fallback when a buffer cannot be mapped)              */
    uint64_t remote_keys;               /* ls_sort_multi: keys this rank sent to other ranks
                                           (8 bytes each over NVLink)                           */
    float phase_ms[LS_NUM_PHASES];      /* with LS_FLAG_PHASE_TIMING                          */
} ls_stats;

/* Optional device outputs of ls_sort_with_model / ls_sort for parity checks.
 * Any pointer may be NULL. Rows of homogeneous level-0 buckets are zero in
 * S_B1 and H1, exactly as Alg. 2 never partitions them. */
typedef struct {
    uint64_t *d_S_B;  /* [f]    level-0 bucket sizes (Alg. 1 S_B)   */
    uint32_t *d_S_B1; /* [f*f]  level-1 sizes S'_B                  */
    uint8_t *d_H0;    /* [f]    homogeneous level-0 buckets          */
    uint8_t *d_H1;    /* [f*f]  homogeneous sub-buckets              */
    ls_model *h_model;/* host: the model the call fitted / used      */
} ls_dumps;

const char *ls_status_string(ls_status s);
const char *ls_last_error(void);

/* Device workspace needed by ls_sort / ls_sort_with_model / ls_train_rmi /
 * ls_bucket_ids for n keys (CUB-style size query). About 14.7n bytes + ~90 MB:
 * the scratch copy B of Alg. 2's partition rounds (n + n/4 + 4096 f keys:
 * round 0 gives every level-0 bucket a sample-estimated region),
 * the round-1 bucket ids (2 bytes per B slot), the in-bucket task and
 * big-item lists, per-unit tables. */
ls_status ls_workspace_bytes(uint64_t n, ls_dtype dtype, const ls_config *cfg, size_t *bytes);

/* Fit F_A on a sample (north_star (1); R7-R9): d_sample holds m
 * keys in any order (e.g. the strided 1% sample A[100k]); the model is the
 * chord interpolant of the sample's strict-less eCDF through the first sample
 * key of every non-empty leaf. Written to *out (host). Parameters are a pure
 * function of the sample (no reductions in floating point), so they are
 * bit-identical to any correct implementation of R7. */
ls_status ls_train_rmi(const void *d_sample, uint64_t m, ls_dtype dtype, const ls_config *cfg,
                       ls_model *out, void *d_ws, size_t ws_bytes, void *stream);

/* Sort n keys in place (Alg. 2): strided sample + fit, level-0
 * partition (one scatter pass reserving runs in per-bucket capacities taken
 * from the sample; the exact count -> decoupled-lookback -> scatter passes
 * only when a capacity does not hold), level-1 segmented partition (count,
 * then a scatter reserving runs on one cursor per sub-bucket), homogeneous-
 * bucket skip, model counting sort with collision-group touch-up, exact
 * big-bucket path. dumps/stats may be NULL.
 * d_keys must be 16-byte aligned and d_ws 256-byte aligned (cudaMalloc /
 * torch allocations are; an odd-offset slice is not): LS_E_INVALID otherwise,
 * for every entry point that takes device keys and a workspace.
 * Launch sequence: every decision inside it is taken on the device, so the
 * second call with the same (d_keys, n, dtype, cfg, d_ws, device) captures it
 * into a CUDA Graph and later calls replay it with one launch (kept in a
 * 16-entry process-wide cache; not used with dumps or ls_sort_with_model;
 * with LS_FLAG_PHASE_TIMING the phase events are event-record nodes of the
 * graph). Environment: LS_GRAPH=0 launches directly; LS_GRAPH=2
 * turns a failed capture into LS_E_CUDA instead of a direct launch. */
ls_status ls_sort(void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg, void *d_ws,
                  size_t ws_bytes, void *stream, ls_stats *stats, const ls_dumps *dumps);

/* As ls_sort but with an injected model (parity hook). The model
 * is validated (finite, a >= 0, lo <= hi, hi_l <= lo_{l+1}, hi <= 1 - 2^-52,
 * root_scale >= 0) and rejected with LS_E_INVALID otherwise. */
ls_status ls_sort_with_model(void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg,
                             const ls_model *model, void *d_ws, size_t ws_bytes, void *stream,
                             ls_stats *stats, const ls_dumps *dumps);

/* End-to-end: h_keys (host, ideally pinned) -> d_buf (n keys, device) ->
 * ls_sort -> h_keys. The copies run on `stream` inside the call. */
ls_status ls_sort_host(void *h_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg,
                       void *d_buf, void *d_ws, size_t ws_bytes, void *stream, ls_stats *stats);

/* Per-key model outputs for a given model (parity hook; Alg. 1, Alg. 2
 * P:188-190): p = F_A(x) (fp64 bits), b0, b1 (parent = own b0), the
 * counting-sort slot pos with n' = hist1[b0*f+b1] (R5), and the raw
 * histograms of b0 and of (b0,b1) over all keys. Any output may be NULL
 * except that d_pos needs the histogram (computed internally). */
ls_status ls_bucket_ids(const void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg,
                        const ls_model *model, double *d_p, uint32_t *d_b0, uint32_t *d_b1,
                        uint32_t *d_pos, uint64_t *d_hist0, uint64_t *d_hist1, void *d_ws,
                        size_t ws_bytes, void *stream);

/* ------------------------------------------------------------ multi-GPU -- */
/* Sample-based global range split: every rank samples its shard,
 * the samples are all-gathered, R-1 splitters are chosen on the lexicographic
 * key (ord(x), rank, index) so runs of equal keys may straddle ranks, every key
 * is routed to its destination rank, the shards are exchanged with an NCCL
 * all-to-all over NVLink, and each rank sorts what it received with ls_sort.
 * Rank r returns the r-th contiguous slice of the global order. */
typedef struct ls_comm ls_comm;

#define LS_UNIQUE_ID_BYTES 128
ls_status ls_comm_unique_id(uint8_t id[LS_UNIQUE_ID_BYTES]);
ls_status ls_comm_init(const uint8_t id[LS_UNIQUE_ID_BYTES], int rank, int world, ls_comm **out);
void ls_comm_destroy(ls_comm *comm);

/* Workspace for ls_sort_multi with out_cap output slots. */
ls_status ls_multi_workspace_bytes(uint64_t n_in, uint64_t out_cap, int world, ls_dtype dtype,
                                   const ls_config *cfg, size_t *bytes);

ls_status ls_sort_multi(ls_comm *comm, const void *d_in, uint64_t n_in, void *d_out,
                        uint64_t out_cap, uint64_t *n_out, ls_dtype dtype, const ls_config *cfg,
                        void *d_ws, size_t ws_bytes, void *stream, ls_stats *stats);

/* Host-side planning steps of ls_sort_multi, exported so the exchange logic can
 * be exercised without GPUs (gloo tests). Entries are (ord, rank, index)
 * triples. ls_multi_splitters: writes the R-1 entries of ranks floor(k*v/R),
 * k=1..R-1, in the lexicographic order of the v non-sentinel entries among the
 * `count` gathered sample entries (reordering h_entries). ls_multi_plan:
 * from the R x R count matrix (row = source rank) computes, for `rank`, the
 * send displacements, the receive counts/displacements and n_out. */
typedef struct {
    uint64_t ord;
    uint32_t rank;
    uint32_t pad;
    uint64_t index;
} ls_tagged;

ls_status ls_multi_splitters(ls_tagged *h_entries, uint64_t count, int world, ls_tagged *h_splitters);
ls_status ls_multi_plan(const uint64_t *h_counts, int world, int rank, uint64_t *h_send_displ,
                        uint64_t *h_recv_counts, uint64_t *h_recv_displ, uint64_t *n_out);
/* Destination rank of a key: the number of splitters strictly below
 * (ord(x), rank, index) in lexicographic order. Host reference of the device rule. */
int ls_multi_dest(const ls_tagged *h_splitters, int world, uint64_t ord, uint32_t rank,
                  uint64_t index);

/* The device steps of ls_sort_multi for ONE rank, without a communicator, so
 * the routing kernels run for world > 1 on a single GPU (tests): nothing
 * waits on another rank.
 * ls_multi_sample: step 1, the LS_MULTI_SAMPLE tagged split-sample entries of
 *   this rank's shard d_in[n_in] into d_samples (device, caller-owned; entries
 *   beyond n_in are sentinels with rank 0xffffffff).
 * ls_multi_route: steps 3 + 5 with the given R-1 splitters (host): the
 *   destination counts (h_counts[world], host) and the shard regrouped by
 *   destination into d_send[n_in] (device; destination p's keys start at
 *   sum_{q<p} h_counts[q], in no particular order inside). d_ws holds at least
 *   ls_multi_workspace_bytes(n_in, 0, world, ...) bytes. Synchronous on
 *   `stream`. Errors: LS_E_INVALID (bad sizes / world), LS_E_WORKSPACE,
 *   LS_E_NAN (NaN key; d_send untouched). */
#define LS_MULTI_SAMPLE 16384
ls_status ls_multi_sample(const void *d_in, uint64_t n_in, int rank, ls_dtype dtype,
                          ls_tagged *d_samples, void *stream);
ls_status ls_multi_route(const void *d_in, uint64_t n_in, int rank, int world,
                         const ls_tagged *h_splitters, ls_dtype dtype, void *d_send,
                         uint64_t *h_counts, void *d_ws, size_t ws_bytes, void *stream);
/* SURVEY §8(f) f1, the fused destination scatter of LS_FLAG_PEER_SCATTER for
 * ONE rank without a communicator: steps 3 + 5 with the given R-1 splitters,
 * the scatter storing destination p's keys straight into h_dst[p] (a device
 * pointer valid on this GPU: local memory, or a peer GPU's buffer mapped with
 * CUDA IPC / peer access) from element h_dst_off[p] on, h_counts[p] of them
 * (reported on the host), in no particular order inside. h_dst and h_dst_off
 * are host arrays of `world` entries (8-byte-aligned pointers; unused when
 * h_counts[p] == 0). Nothing is written before the counts are known; the
 * caller sizes and places the slices (e.g. from every rank's counts, as
 * ls_sort_multi does with ls_multi_plan). d_ws: ls_multi_workspace_bytes(n_in,
 * 0, world, ...) bytes. Synchronous on `stream`. Errors: LS_E_INVALID,
 * LS_E_WORKSPACE, LS_E_NAN (nothing written). */
ls_status ls_multi_route_peer(const void *d_in, uint64_t n_in, int rank, int world,
                              const ls_tagged *h_splitters, ls_dtype dtype, void *const *h_dst,
                              const uint64_t *h_dst_off, uint64_t *h_counts, void *d_ws,
                              size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif
