// ls_common.cuh -- device-side building blocks of libls (sm_100a).
//
// The fp64 arithmetic here is the bit-exact contract with the oracle's readings
// R7-R13: explicit round-to-nearest intrinsics so that nvcc never
// contracts a multiply-add except the leaf line's single fma (R13).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ls.h"

namespace ls {

enum { DT_F64 = 0, DT_U64 = 1 };

constexpr double PMAX = 1.0 - 0x1p-52;  // R10
constexpr uint64_t LB_FLAG_A = 1ull << 62;  // decoupled lookback: aggregate published
constexpr uint64_t LB_FLAG_P = 2ull << 62;  // decoupled lookback: inclusive prefix published
constexpr uint64_t LB_VALUE = (1ull << 62) - 1;

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// --------------------------------------------------------------- keys ------
// ord (IEEE totalOrder as an unsigned key): negative -> ~b, else b | 2^63.
// Written as one xor with a sign mask (an arithmetic shift of the high word
// and one 3-input logic op per word in SASS, no selects).
template <int DT>
__device__ __forceinline__ uint64_t to_ord(uint64_t b) {
    if (DT == DT_U64) return b;
    const uint32_t hi = (uint32_t)(b >> 32), m = (uint32_t)((int32_t)hi >> 31);
    return ((uint64_t)(hi ^ (m | 0x80000000u)) << 32) | (uint32_t)((uint32_t)b ^ m);
}
template <int DT>
__device__ __forceinline__ uint64_t from_ord(uint64_t o) {
    if (DT == DT_U64) return o;
    const uint32_t hi = (uint32_t)(o >> 32), m = ~(uint32_t)((int32_t)hi >> 31);
    return ((uint64_t)(hi ^ (m | 0x80000000u)) << 32) | (uint32_t)((uint32_t)o ^ m);
}
template <int DT>
__device__ __forceinline__ double xd(uint64_t b) {
    if (DT == DT_U64) return __ull2double_rn(b);
    return __longlong_as_double((long long)b);
}
template <int DT>
__device__ __forceinline__ bool is_finite_key(uint64_t b) {
    if (DT == DT_U64) return true;
    return (b & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
}
__device__ __forceinline__ bool is_nan_bits(uint64_t b) {
    return (b & 0x7fffffffffffffffull) > 0x7ff0000000000000ull;
}
// R13: ordered comparisons, NaN -> lo, never fmin/fmax
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
    return v >= lo ? (v <= hi ? v : hi) : lo;
}

// -------------------------------------------------------------- model ------
// b0 as a search (exact): b0 is a monotone step function of ord(x) (R15:
// a >= 0, hi_l <= lo_{l+1}), so b0(x) = #{b >= 1 : thr_b <= ord(x)} with
// thr_b = min{o : b0(o) >= b}. k_b0_thresholds finds the f-1 thresholds by
// bisection with the very predict()/bucket0() of the full path, and a uniform
// grid of B0_CELLS cells over [xmin, xmax] (cell(x) monotone in ord) records,
// per cell, the range of thresholds that fall inside it: cell = off | cnt<<10
// (cnt saturates at 63 = "search to the end"). A key then costs the root
// arithmetic, one 2-byte and ~cnt 8-byte shared-memory loads instead of five
// 8-byte leaf loads and the fp64 leaf line.
constexpr int B0_CELLS = 16384;
// Cells holding >= B0_SUBMIN thresholds (duplicate-heavy or very skewed
// inputs: config 5's Zipf head puts ~350 of 999 thresholds into one cell) get
// a refined grid of B0_SUB sub-cells (the grid at 64x the resolution: the
// fine index trunc(64 r) is exact, 64 being a power of two), up to B0_NSUB such
// cells. Cell entry count field: 0..61 exact, 62 = refined (offset field =
// sub-grid number), 63 = more than 61 thresholds, not refined.
constexpr int B0_SUB = 64;
constexpr int B0_NSUB = 64;
constexpr uint32_t B0_SUBMIN = 16;
constexpr uint32_t B0_REFINED = 62, B0_SAT = 63;
// Device copy of F_A. leaf[] holds (a, c, b, lo, hi) per leaf, 40 bytes.
struct DevModel {
    double xmin, xmax, root_scale, last;  // last = (double)(L-1)
    uint32_t L, degenerate;
    uint64_t n_sample;
    double leaf[LS_MAX_LEAVES * 5];
    // b0 search structure (k_b0_thresholds / k_b0_cells)
    double cell_scale;                        // B0_CELLS / (xmax - xmin), 0 if degenerate
    uint32_t nthr, pad_;                      // valid thresholds: thr[0 .. nthr)
    unsigned long long thr[LS_MAX_FANOUT];    // thr[b-1] = min{o : b0(o) >= b}
    alignas(16) uint16_t cell[B0_CELLS];
    alignas(16) uint16_t sub[B0_NSUB * B0_SUB];  // refined cells' sub-grids (same entry format)
    uint16_t sub_cell[B0_NSUB];               // the cell of each sub-grid
    uint32_t nsub;                            // refined cells (may exceed B0_NSUB: the rest stay B0_SAT)
};

// Root parameters held in registers (uniform across the grid).
struct Root {
    double xmin, xmax, rs, last;
    int Lm1;
};

__device__ __forceinline__ Root load_root(const DevModel *M) {
    Root r;
    r.xmin = M->xmin;
    r.xmax = M->xmax;
    r.rs = M->root_scale;
    r.last = M->last;
    r.Lm1 = (int)M->L - 1;
    return r;
}

// Root routing of O6: xc = clamp(x, xmin, xmax), leaf = trunc((xc - xmin) * rs).
template <int DT>
__device__ __forceinline__ int root_leaf(uint64_t bits, const Root &R, double &xc) {
    xc = clampd(xd<DT>(bits), R.xmin, R.xmax);
    const double r = __dmul_rn(__dsub_rn(xc, R.xmin), R.rs);
    return (r < R.last) ? __double2int_rz(r) : R.Lm1;  // (NaN r: inf * 0 -> L-1)
}

// O6: p = F_A(x). `leaf` may point to shared or global memory.
template <int DT>
__device__ __forceinline__ double predict(uint64_t bits, const Root &R, const double *leaf) {
    double xc = clampd(xd<DT>(bits), R.xmin, R.xmax);
    double r = __dmul_rn(__dsub_rn(xc, R.xmin), R.rs);
    const int l = (r < R.last) ? __double2int_rz(r) : R.Lm1;  // (NaN r: inf * 0 -> L-1)
    const double *q = leaf + 5 * l;
    double y = __fma_rn(q[0], __dsub_rn(xc, q[1]), q[2]);
    return __dadd_rn(clampd(y, q[3], q[4]), 0.0);
}

// predict() for keys known to lie in [xmin, xmax] when INNER (the root clamp
// is the identity there); plain predict() otherwise.
template <int DT, bool INNER>
__device__ __forceinline__ double predict_c(uint64_t bits, const Root &R, const double *leaf) {
    const double xc = INNER ? xd<DT>(bits) : clampd(xd<DT>(bits), R.xmin, R.xmax);
    double r = __dmul_rn(__dsub_rn(xc, R.xmin), R.rs);
    const int l = (r < R.last) ? __double2int_rz(r) : R.Lm1;
    const double *q = leaf + 5 * l;
    double y = __fma_rn(q[0], __dsub_rn(xc, q[1]), q[2]);
    return __dadd_rn(clampd(y, q[3], q[4]), 0.0);
}

// Same, reading leaf parameters through the read-only path (keys of one
// level-0 bucket share one or two leaves, so a warp's loads mostly broadcast).
template <int DT>
__device__ __forceinline__ double predict_ldg(uint64_t bits, const Root &R, const double *leaf) {
    double xc = clampd(xd<DT>(bits), R.xmin, R.xmax);
    double r = __dmul_rn(__dsub_rn(xc, R.xmin), R.rs);
    const int l = (r < R.last) ? __double2int_rz(r) : R.Lm1;  // (NaN r: inf * 0 -> L-1)
    const double *q = leaf + 5 * l;
    double y = __fma_rn(__ldg(q), __dsub_rn(xc, __ldg(q + 1)), __ldg(q + 2));
    return __dadd_rn(clampd(y, __ldg(q + 3), __ldg(q + 4)), 0.0);
}

// predict_ldg for a key known to lie in [xmin, xmax] (the root clamp is the
// identity there), and the sub-bucket g = b0 * f + b1 that the clamped keys
// (x < xmin or x > xmax) share with xmin / xmax themselves.
template <int DT>
__device__ __forceinline__ double predict_ldg_inner(uint64_t bits, const Root &R, const double *leaf) {
    const double xc = xd<DT>(bits);
    double r = __dmul_rn(__dsub_rn(xc, R.xmin), R.rs);
    const int l = (r < R.last) ? __double2int_rz(r) : R.Lm1;
    const double *q = leaf + 5 * l;
    double y = __fma_rn(__ldg(q), __dsub_rn(xc, __ldg(q + 1)), __ldg(q + 2));
    return __dadd_rn(clampd(y, __ldg(q + 3), __ldg(q + 4)), 0.0);
}

// The leaf that holds every key of sub-bucket g, + 1 (0: none). The model is
// monotone-safe (model_ok: a >= 0, lo_l <= hi_l <= lo_{l+1}), so a key of
// leaf m < l has p <= lo_l and a key of leaf m > l has p >= hi_l. A key of
// sub-bucket g has p within 1e-15 of [g/f^2, (g+1)/f^2) (p * f^2 < 2^20 is
// rounded by at most 2^-33). So if lo_l < g/f^2 - 1e-12 and (g+1)/f^2 +
// 1e-12 < hi_l, every key of g comes from leaf l and its line value y lies in
// (lo_l, hi_l): p = clamp(y) + 0 = y, with neither the routing, the clamp nor
// the -0.0 canonicalisation needed (the warp sort's fast path). Keys outside
// [xmin, xmax] (the root clamp) only reach the sub-buckets of xmin and xmax,
// which the warp sort excludes.
// One call per warp (all lanes, lane j asks for g = g0 + j): the last leaf
// with lo < P0(g0) by two ballot rounds of 32 leaves (L <= LS_MAX_LEAVES =
// 1024), then every lane walks up from it (consecutive sub-buckets: usually
// 0-1 steps).
static_assert(LS_MAX_LEAVES <= 1024, "contained_leaf_warp searches 32 x 32 leaves");
__device__ __forceinline__ uint32_t contained_leaf_warp(const double *leaf, int L, uint32_t g0, uint32_t g,
                                                        double rcpF2, int lane) {
    // (rcpF2 = RN(1/f^2): g * rcpF2 is within 2 ulps of g/f^2, far inside the margin)
    const double Q0 = __dsub_rn(__dmul_rn((double)g0, rcpF2), 1e-12);
    const int l1 = 32 * lane;
    const unsigned m1 = __ballot_sync(0xffffffffu, l1 < L && __ldg(leaf + 5 * l1 + 3) < Q0);
    if (!m1) return 0u;  // (no leaf below: the first sub-buckets take the slow path)
    const int blk = 31 - __clz(m1);
    const int l2 = 32 * blk + lane;
    const unsigned m2 = __ballot_sync(0xffffffffu, l2 < L && __ldg(leaf + 5 * l2 + 3) < Q0);
    int l = 32 * blk + (31 - __clz(m2));  // (bit 0 of m2 is set: leaf 32*blk passed round 1)
    const double P0 = __dsub_rn(__dmul_rn((double)g, rcpF2), 1e-12);
    const double P1 = __dadd_rn(__dmul_rn((double)(g + 1u), rcpF2), 1e-12);
    while (l + 1 < L && __ldg(leaf + 5 * (l + 1) + 3) < P0) l++;
    return P1 < __ldg(leaf + 5 * l + 4) ? (uint32_t)l + 1u : 0u;
}

// O7 / Alg.1 P:107 (R1)
// (p in [0, 1) and f <= 1024, so p * f^2 < 2^20: a 32-bit truncation is the
// same integer as the oracle's (int64) cast)
__device__ __forceinline__ uint32_t bucket0(double p, double F, int f) {
    const int b = __double2int_rz(__dmul_rn(p, F));
    return (uint32_t)min(b, f - 1);
}

__device__ __forceinline__ uint32_t bucket1(double p, double F2, int f, uint32_t parent) {
    const int b = __double2int_rz(__dmul_rn(p, F2)) - (int)parent * f;
    return (uint32_t)min(max(b, 0), f - 1);
}

// Sub-bucket of the prediction at the double xc (a root-clamped key).
__device__ __forceinline__ uint32_t sub_bucket_at(double xc, const Root &R, const double *leaf,
                                                  double F, double F2, int f) {
    double r = __dmul_rn(__dsub_rn(xc, R.xmin), R.rs);
    const int l = (r < R.last) ? __double2int_rz(r) : R.Lm1;
    const double *q = leaf + 5 * l;
    const double y = __fma_rn(q[0], __dsub_rn(xc, q[1]), q[2]);
    const double p = __dadd_rn(clampd(y, q[3], q[4]), 0.0);
    const uint32_t b0 = bucket0(p, F, f);
    return b0 * (uint32_t)f + bucket1(p, F2, f, b0);
}

// Grid cell of a key for the b0 search (monotone in ord).
template <int DT>
__device__ __forceinline__ int b0_cell(uint64_t bits, double xmin, double xmax, double cs) {
    // = clamp to [xmin, xmax] first, then (r < CELLS-1 ? trunc r : CELLS-1): a key
    // below xmin gets r <= 0 (cell 0), one above xmax r > (xmax - xmin) * cs,
    // which is >= CELLS-1 (cell CELLS-1); a NaN r (inf * 0, degenerate grid)
    // fails r > 0 (cell 0); the conversion saturates
    (void)xmax;
    const double r = __dmul_rn(__dsub_rn(xd<DT>(bits), xmin), cs);
    return r > 0.0 ? min(__double2int_rz(r), B0_CELLS - 1) : 0;
}

// Fine grid index (64 sub-cells per cell) of the same r: fine / 64 == b0_cell.
template <int DT>
__device__ __forceinline__ int b0_fine(uint64_t bits, double xmin, double cs) {
    const double r = __dmul_rn(__dsub_rn(xd<DT>(bits), xmin), cs);
    return r > 0.0 ? min(__double2int_rz(__dmul_rn(r, (double)B0_SUB)), B0_CELLS * B0_SUB - 1) : 0;
}

// b0 of a key from the thresholds (thr, cell in shared memory); bit-identical
// to bucket0(predict(x)) by construction (see B0_CELLS).
struct B0Search {
    double xmin, xmax, cs;
    uint32_t nthr;
    const unsigned long long *thr;
    const uint16_t *cell;
    const uint16_t *sub;
    template <int DT>
    __device__ __forceinline__ uint32_t get(uint64_t bits) const {
        const int c = b0_cell<DT>(bits, xmin, xmax, cs);
        uint32_t e = cell[c];
        uint32_t lo = e & 1023u, n = e >> 10;
        if (n == 0u) return lo;  // most keys: no threshold inside their cell
        if (n == B0_REFINED) {   // dense cell: its sub-grid
            e = sub[lo * B0_SUB + (b0_fine<DT>(bits, xmin, cs) - c * B0_SUB)];
            lo = e & 1023u;
            n = e >> 10;
            if (n == 0u) return lo;
        }
        const unsigned long long o = to_ord<DT>(bits);
        if (n == 1u) return lo + (thr[lo] <= o ? 1u : 0u);
        if (n == B0_SAT) {
            // saturated count: the thresholds of cell c end where the next
            // cell's begin (its offset, when that cell owns ords at all)
            const uint32_t en = c + 1 < B0_CELLS ? cell[c + 1] : 0u;
            const uint32_t nx = (en >> 10) == B0_REFINED ? 0u : (en & 1023u);  // (refined: a sub-grid number)
            n = (nx >= lo + 63u ? nx : nthr) - lo;
        }
        while (n > 0) {
            const uint32_t half = n >> 1;
            if (thr[lo + half] <= o) {
                lo += half + 1;
                n -= half + 1;
            } else {
                n = half;
            }
        }
        return lo;
    }
};

// Alg.2 P:188-190 (R5): pos = clamp(floor((p - adj) * n), 0, n'-1). The
// round-down conversion is floor; it saturates out-of-range values to the int
// range (and NaN to 0), so the integer clamp gives the same pos as clamping
// the double.
__device__ __forceinline__ uint32_t cs_pos(double p, double adj, double nd, int top) {
    const int v = __double2int_rd(__dmul_rn(__dsub_rn(p, adj), nd));
    return (uint32_t)min(max(v, 0), top);
}

// ------------------------------------------------------------ control -----
enum {
    ST_H0B = 0, ST_H0K, ST_H1S, ST_H1K, ST_SMALLS, ST_SMALLK, ST_BIGS, ST_BIGK, ST_MAXGRP,
    ST_BIGPASS, ST_NUM
};
enum { STATUS_NAN = 1u, STATUS_INTERNAL = 2u };
constexpr int BIG_LEVELS = 6;
constexpr uint32_t WS_MAX = 256;  // SMALL sub-buckets of WS_MIN+1..WS_MAX keys: one warp each (k_warpsort)
constexpr uint32_t WS_MIN = 32;   // tiny sub-buckets (<= WS_MIN keys) go to the block windows, many per window
constexpr uint32_t BW_MAX = 1024;  // sub-buckets up to this size fit the block windows (k_bucketsort)
constexpr uint32_t CS_S_MAX = 512;  // SMALL sub-buckets of WS_MAX+1..CS_S_MAX keys: 64-thread CTAs, 8 keys/thread
constexpr uint32_t CL_MAX = 1024;  // SMALL sub-buckets of CS_S_MAX+1..CL_MAX keys: 128-thread CTAs, 8 keys/thread
constexpr uint32_t CM_MAX = 2048;  // SMALL sub-buckets of CL_MAX+1..CM_MAX keys: 128-thread CTAs, 16 keys/thread
constexpr uint32_t CS_MAX = 4096;  // SMALL sub-buckets of WS_MAX+1..CS_MAX keys: one CTA each (k_ctasort)
// Size class of a sub-bucket of np keys (T_small = cfg.big_threshold):
//   <= 1 trivial; 2..32 block windows (many per window); 33..256 one warp;
//   257..1024 one 128-thread CTA (8 keys per thread); 1025..2048 one
//   128-thread CTA (16 per thread); 2049..T_small one 256-thread CTA;
//   > T_small the exact big path.
enum { SC_TRIVIAL = 0, SC_WINDOW, SC_WARP, SC_CTAS, SC_CTAL, SC_CTAM, SC_CTA, SC_BIG, SC_FUSED };  // (SC_FUSED: sorted by k_round1)
__host__ __device__ __forceinline__ int size_class(uint32_t np, uint32_t T_small) {
    if (np <= 1) return SC_TRIVIAL;
    if (np > T_small) return SC_BIG;
    if (np <= WS_MIN) return SC_WINDOW;
    if (np <= WS_MAX) return SC_WARP;
    if (np <= CS_S_MAX) return SC_CTAS;
    if (np <= CL_MAX) return SC_CTAL;
    if (np <= CM_MAX) return SC_CTAM;
    return SC_CTA;
}
constexpr uint32_t FR_MIN_DEFAULT = 65536;  // smallest level-0 bucket for the cluster-resident round 1
constexpr uint32_t LARGE_MIN = 262144;  // big sub-buckets above this: grid-parallel path (ls_bigpath.cu)

struct Ctl {
    uint32_t status;
    uint32_t ticket0, ticket1, U1;
    uint32_t ticket_s1;                // k_scatter1p's tile tickets
    uint32_t big_cnt[BIG_LEVELS + 1];  // items per big level list
    uint32_t big_next[BIG_LEVELS + 1]; // work counters
    uint32_t big_lv0;                  // level-0 tickets of k_big: level-0 items + the large path's level-1 items
    uint32_t big_pub1, big_done0;      // level-1 items published (in order) / first-pass tickets done
    uint32_t nchunks;                  // k_big_minmax work entries
    uint32_t nwin, wticket;            // bucket-sort windows (k_window_list) / work counter
    uint32_t ntask;                    // warp sub-bucket sorts (k_classify)
    uint32_t sticket;                  // k_warpsort's task tickets (batches of WS_BATCH)
    uint32_t nctask, nctask2, nctask3; // CTA sub-bucket sorts: SC_CTA, SC_CTAM, SC_CTAL (k_classify)
    uint32_t nctask4;                  // ... SC_CTAS
    uint32_t nlarge, npiece;           // large big items (ls_bigpath.cu) / their small pieces
    uint32_t nfill;                    // homogeneous pieces of large items (k_large_fill)
    uint32_t nfused, fticket;          // cluster-resident round 1: buckets listed / taken
    uint32_t exact0;                   // 1: round 0 by the exact count pass (reservation declined or overflowed)
    unsigned long long smin, smax;     // finite sample ord min / max
    unsigned long long stat[ST_NUM];
    unsigned long long prof[16];       // debug cycle counters (LS_DEBUG_STAGE)
};

// Big-path work item: a key range that must be sorted exactly.
struct BigItem {
    uint32_t off, size;  // global key offset, size
    uint32_t in_b;       // 1: the keys currently sit in B (else in A)
    uint32_t g;          // originating sub-bucket (for H1 dumps), or ~0u
    unsigned long long mn, mx;  // ord range (level 0: filled by k_big_minmax)
    uint32_t pad0, pad1;
    unsigned long long dif;     // OR of ord(x) ^ ord(first key): its trailing zeros are the
                                // low bits every key shares (the dense path's value stride)
};
constexpr uint32_t MM_CHUNK = 65536;
struct BigChunk {
    uint32_t item, chunk;
};

// All device pointers of one call (passed by value to kernels).
struct Args {
    uint64_t *A;  // keys (in place)
    uint64_t *B;  // scratch copy
    uint64_t n;
    int f;        // fanout
    int L;
    double F, F2, nd;
    double rcpF2;      // RN(1/f^2) for adj_of
    uint32_t S1;       // ceil(n / f^2) + 1: slot range of the in-bucket counting sort (k_warpsort)
    uint32_t C0, C1;   // level-0 / level-1 unit sizes (keys)
    uint32_t U0, U1max;
    uint32_t T_small;  // big threshold
    uint32_t T_tile;   // bucketsort window
    uint32_t ntiles;
    uint32_t big_cap;  // items per big level list
    Ctl *ctl;
    DevModel *M;
    uint64_t *S;                      // sample
    uint32_t *leaf_cnt;               // [L]
    unsigned long long *leaf_min;     // [L]
    unsigned long long *hist0;        // [f]
    unsigned long long *start0;       // [f+1]
    unsigned long long *bmin0, *bmax0;// [f] ord of bucket b's first key; != 0 iff two of its keys differ (H0)
    uint32_t *unit1_start;            // [f+1]
    unsigned long long *lb0;          // [U0*f]
    // round 0 by reservation (k_scatter0r): bucket b owns B[bsrc[b], bsrc[b] + cap0[b]),
    // tiles reserve their runs with atomicAdd on cur0[b]; shist0 = sample counts
    unsigned long long *cap0, *bsrc, *cur0;  // [f], [f+1], [f]
    uint32_t *shist0;                 // [f]
    uint64_t Bcap;                    // keys B holds (>= n)
    uint32_t force_exact0;            // host: always take the exact count pass
    uint32_t *offs0;                  // [U0*f]
    uint32_t *hist1;                  // [f*f]
    uint32_t *start1;                 // [f*f]
    uint32_t *cur1;                   // [f*f] round-1 write cursors (k_scatter1 reserves runs on them)
    uint32_t *tile_first, *tile_last; // [ntiles]
    uint4 *wlist;                     // [ntiles] non-empty windows {g0, g1, lo, hi}
    uint16_t *bid;                    // [n + 16] bucket id of each key, count -> scatter pass
    uint4 *tasks;                     // [task_cap] warp sub-bucket sorts {start, n', g, 0}
    uint4 *ctasks, *ctasks2, *ctasks3, *ctasks4;// [task_cap] CTA sub-bucket sorts {start, n', g, 0}
    uint32_t task_cap;
    // large big items (> LARGE_MIN keys): per item 1024-digit tables
    uint32_t *large;                  // [lcap] index into big[] (level 0)
    uint32_t lcap, pcap;
    uint32_t *ltot, *lstart, *lcur, *lhom;  // [lcap*1024] x3, [lcap*32]
    unsigned long long *lmin, *lmax;  // [lcap*1024]
    uint2 *pieces;                    // [pcap] small non-homogeneous pieces {off, size} (in B)
    uint4 *fills;                     // [fcap] homogeneous pieces {off, size, ord lo, ord hi}
    // cluster-resident round 1 (ls_round1.cu): level-0 buckets of fr_min..fr_cap
    // keys (fr_min = 0: off) are partitioned by one CTA cluster each
    uint32_t *fused;                  // [f] 1: bucket taken by k_round1 (k_count1/k_scatter1 skip it)
    uint32_t *flist;                  // [f] the taken buckets
    uint32_t fr_min, fr_cap;
    uint32_t fcap;
    BigItem *big;                     // [(BIG_LEVELS+1) * big_cap]
    BigChunk *chunks;                 // [chunk_cap]
    uint32_t *border;                 // [2 big_cap] k_big's first-pass items, most expensive first (k_big_order)
    uint32_t chunk_cap;
    // parity dumps (may be null)
    uint8_t *dH0, *dH1;
    uint32_t dbg;  // LS_DEBUG_STAGE (profiling ablations only; 0 in normal use)
};

// ------------------------------------------------------------ scans -------
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// In-place exclusive scan of s[0..len) by the whole block; returns the total.
// `tmp` must hold 33 uint32. All threads must call it.
__device__ __forceinline__ uint32_t block_exscan(uint32_t *s, int len, uint32_t *tmp) {
    const int per = (len + blockDim.x - 1) / blockDim.x;
    const int beg = threadIdx.x * per;
    uint32_t local = 0;
    for (int i = 0; i < per; i++)
        if (beg + i < len) local += s[beg + i];
    uint32_t incl = warp_incl_scan(local);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if (lane == 31) tmp[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < nw ? tmp[lane] : 0;
        uint32_t vi = warp_incl_scan(v);
        if (lane < nw) tmp[lane] = vi - v;
        if (lane == 31) tmp[32] = vi;  // total (nw <= 32)
    }
    __syncthreads();
    uint32_t run = tmp[w] + incl - local;
    for (int i = 0; i < per; i++) {
        if (beg + i < len) {
            uint32_t v = s[beg + i];
            s[beg + i] = run;
            run += v;
        }
    }
    uint32_t total = tmp[32];
    __syncthreads();
    return total;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_or_u64(unsigned long long v) {
    const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)v);
    const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(v >> 32));
    return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < v ? t : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
        v = t > v ? t : v;
    }
    return v;
}

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    return *(const volatile unsigned long long *)p;
}
__device__ __forceinline__ void st_volatile(unsigned long long *p, unsigned long long v) {
    *(volatile unsigned long long *)p = v;
}

}  // namespace ls

namespace ls {

// ------------------------------------------------- TMA 1-D bulk copies ----
// cp.async.bulk (the bulk-copy engine of the TMA unit; SASS UBLKCP) moves a
// contiguous global range into shared memory and signals an mbarrier with the
// byte count. Addresses 16-byte aligned, sizes multiples of 16.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(mbar)), "r"(phase)
            : "memory");
    }
}

// Stage global keys [glo, ghi) into smem so that key k lands at sdst[k - glo].
// The bulk engine needs 16-byte alignment, so the copy covers the aligned hull
// [glo & ~1, (ghi + 1) & ~1) starting at sbase; returns sbase + (glo & 1).
// Called by all threads; thread 0 issues, everyone waits.
__device__ __forceinline__ uint64_t *stage_keys(const uint64_t *g, uint32_t glo, uint32_t ghi,
                                                uint64_t *sbase, uint64_t *mbar) {
    const uint32_t alo = glo & ~1u, ahi = (ghi + 1) & ~1u;
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        const uint32_t bytes = (ahi - alo) * 8u;
        mbar_expect_tx(mbar, bytes);
        constexpr uint32_t CH = 16384;
        for (uint32_t o = 0; o < bytes; o += CH)
            bulk_g2s((char *)sbase + o, (const char *)(g + alo) + o, bytes - o < CH ? bytes - o : CH, mbar);
    }
    __syncthreads();
    mbar_wait(mbar, 0);
    return sbase + (glo - alo);
}

__device__ __forceinline__ uint32_t warp_incl_max(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = t > v ? t : v;
    }
    return v;
}

// In-place inclusive max-scan of s[0..len) (each thread: `per` consecutive).
__device__ __forceinline__ void block_incl_maxscan(uint32_t *s, int len, uint32_t *tmp) {
    const int per = (len + blockDim.x - 1) / blockDim.x;
    const int beg = threadIdx.x * per;
    uint32_t local = 0;
    for (int i = 0; i < per; i++)
        if (beg + i < len) local = s[beg + i] > local ? s[beg + i] : local;
    const uint32_t incl = warp_incl_max(local);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if (lane == 31) tmp[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t v = lane < nw ? tmp[lane] : 0;
        uint32_t vi = warp_incl_max(v);
        uint32_t ex = __shfl_up_sync(0xffffffffu, vi, 1);
        if (lane < nw) tmp[lane] = lane ? ex : 0;
    }
    __syncthreads();
    uint32_t run = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) run = 0;
    run = run > tmp[w] ? run : tmp[w];
    for (int i = 0; i < per; i++) {
        if (beg + i < len) {
            run = s[beg + i] > run ? s[beg + i] : run;
            s[beg + i] = run;
        }
    }
    __syncthreads();
}

}  // namespace ls
