// ls_partition.cu -- north_star (2): the two model-guided partition rounds.
//
// Alg. 1 as a GPU pass pair per round. The paper places keys into
// fixed-capacity fragments and defragments afterwards because a separate
// counting scan was "not insignificant" on one CPU core; on
// B200 a counting scan costs 8 B/key at HBM speed and removes the
// defragmentation pass entirely, so each round is:
//   count   : predict -> per-CTA shared-memory histogram of bucket ids ->
//             decoupled lookback across units (chained prefix, one status word
//             per (unit, bucket) carrying flag + value) -> per-unit offsets
//   scatter : predict again -> tile-local counting sort in shared memory ->
//             coalesced run stores at base[bucket] (no defragmentation: every
//             bucket is written contiguously, Fig. 3c's result directly)
// Round 0 partitions A -> B by b0 over the whole input; round 1 partitions
// each non-homogeneous level-0 bucket B -> A by b1 (a segmented round: units
// never straddle buckets). Level-0 homogeneous buckets are filled
// directly from their min key.
#include "ls_launch.h"
#include "ls_tile.cuh"
#include "ls_tilepart.cuh"

namespace ls {

// ----------------------------------------------------------------- init ----
__global__ void k_init(Ctl *ctl) {
    if (threadIdx.x == 0) {
        ctl->status = 0;
        ctl->ticket0 = ctl->ticket1 = ctl->U1 = 0;
        ctl->ticket_s1 = 0;
        ctl->nchunks = 0;
        ctl->nwin = ctl->wticket = 0;
        ctl->ntask = ctl->nctask = ctl->nctask2 = ctl->nctask3 = ctl->nctask4 = 0;
        ctl->sticket = 0;
        ctl->nfused = ctl->fticket = 0;
        ctl->exact0 = 0;
        ctl->nlarge = ctl->npiece = 0;
        ctl->nfill = 0;
        for (int i = 0; i <= BIG_LEVELS; i++) ctl->big_cnt[i] = ctl->big_next[i] = 0;
        ctl->smin = ~0ull;
        ctl->smax = 0;
        for (int i = 0; i < ST_NUM; i++) ctl->stat[i] = 0;
        for (int i = 0; i < 16; i++) ctl->prof[i] = 0;
    }
}

void launch_init(const Args &a, cudaStream_t st) { k_init<<<1, 32, 0, st>>>(a.ctl); }

// -------------------------------------------------------------- helpers ----
template <int DT, bool SMEM_MODEL>
__device__ __forceinline__ double predict_any(uint64_t b, const Root &R, const double *leaf) {
    return SMEM_MODEL ? predict<DT>(b, R, leaf) : predict_ldg<DT>(b, R, leaf);
}

// Bucket function of one partition round: level 0 -> b0, level 1 -> b1(parent).
template <int DT, int LEVEL, bool SMEM_MODEL>
struct ModelBucket {
    Root R;
    const double *leaf;
    double F, F2;
    int f;
    uint32_t parent;
    __device__ __forceinline__ uint32_t operator()(uint64_t key, uint64_t) const {
        const double p = predict_any<DT, SMEM_MODEL>(key, R, leaf);
        return LEVEL == 0 ? bucket0(p, F, f) : bucket1(p, F2, f, parent);
    }
};

// --------------------------------------------------------------- round 0 ---
// b0 search tables in shared memory (count0 / scatter0)
struct alignas(16) B0Smem {
    unsigned long long thr[LS_MAX_FANOUT];
    uint16_t cell[B0_CELLS];
    alignas(16) uint16_t sub[B0_NSUB * B0_SUB];
};

__device__ __forceinline__ B0Search load_b0_search(B0Smem &T, const DevModel *M) {
    const uint32_t V = M->nthr;
    for (uint32_t i = threadIdx.x; i < V; i += blockDim.x) T.thr[i] = M->thr[i];
    const uint4 *src = reinterpret_cast<const uint4 *>(M->cell);
    uint4 *dst = reinterpret_cast<uint4 *>(T.cell);
    for (int i = threadIdx.x; i < B0_CELLS / 8; i += blockDim.x) dst[i] = src[i];
    const uint32_t ns = min(M->nsub, (uint32_t)B0_NSUB);
    const uint4 *ssrc = reinterpret_cast<const uint4 *>(M->sub);
    uint4 *sdst = reinterpret_cast<uint4 *>(T.sub);
    for (uint32_t i = threadIdx.x; i < ns * B0_SUB / 8; i += blockDim.x) sdst[i] = ssrc[i];
    return B0Search{M->xmin, M->xmax, M->cell_scale, V, T.thr, T.cell, T.sub};
}

struct Count0Smem {
    B0Smem b0;
    uint32_t hist[LS_MAX_FANOUT];
};

template <int DT>
__global__ void __launch_bounds__(512, 3) k_count0(Args a) {
    if (!a.ctl->exact0) return;  // (round 0 went by reservation, k_scatter0r)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Count0Smem &S = *reinterpret_cast<Count0Smem *>(smem_raw);
    uint32_t *hist = S.hist;
    __shared__ uint32_t s_unit;
    __shared__ int s_nan;
    const int tid = threadIdx.x, bd = blockDim.x, f = a.f;
    if (tid == 0) s_nan = 0;
    // persistent: the b0 search tables are loaded once per CTA, then units
    // (C0 keys each) are taken in ticket order (the lookback needs that order)
    const B0Search bs = load_b0_search(S.b0, a.M);
    bool nan = false;
    auto one = [&](uint64_t b) {
        if (DT == DT_F64 && is_nan_bits(b)) nan = true;
        atomicAdd(&hist[bs.get<DT>(b)], 1u);
    };
    for (;;) {
        if (tid == 0) s_unit = atomicAdd(&a.ctl->ticket0, 1u);
        for (int b = tid; b < f; b += bd) hist[b] = 0;
        __syncthreads();
        const uint64_t u = s_unit;
        if (u >= a.U0) break;
        const uint64_t beg = u * a.C0, end = umin64(a.n, beg + a.C0);
        if ((((uintptr_t)(a.A + beg)) & 15) == 0) {
            // 4 independent 16-byte loads in flight per thread
            const ulonglong2 *A2 = (const ulonglong2 *)(a.A + beg);
            const uint64_t np = (end - beg) / 2;
            uint64_t i = tid;
            for (; i + 3 * bd < np; i += 4 * bd) {
                ulonglong2 v[4];
#pragma unroll
                for (int q = 0; q < 4; q++) v[q] = __ldcs(A2 + i + q * bd);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    one(v[q].x);
                    one(v[q].y);
                }
            }
            for (; i < np; i += bd) {
                const ulonglong2 v = __ldcs(A2 + i);
                one(v.x);
                one(v.y);
            }
            if (((end - beg) & 1) && tid == 0) one(a.A[end - 1]);
        } else {
            for (uint64_t i = beg + tid; i < end; i += bd) one(a.A[i]);
        }
        __syncthreads();
        for (int b = tid; b < f; b += bd) {
            const uint32_t c = hist[b];
            if (c) atomicAdd(&a.hist0[b], (unsigned long long)c);
            a.offs0[u * f + b] = lookback(a.lb0, u, 0, f, b, c);
        }
        __syncthreads();
    }
    if (nan) s_nan = 1;
    __syncthreads();
    if (tid == 0 && s_nan) atomicOr(&a.ctl->status, (uint32_t)STATUS_NAN);
}

// Round-1 units: a bucket of h keys is cut into nu = max(1, round(h / C1))
// units of ceil(h / nu) keys rounded up to whole scatter tiles (not C1-sized
// units plus a sliver, which would cost a whole CTA start and a partial tile).
__host__ __device__ __forceinline__ uint32_t unit1_count(uint64_t h, uint32_t C1) {
    const uint64_t nu = (h + C1 / 2) / C1;
    return h == 0 ? 0u : (uint32_t)(nu ? nu : 1);
}
__device__ __forceinline__ uint64_t unit1_size(uint64_t bbeg, uint64_t bend, uint32_t nu) {
    const uint64_t u = nu ? (bend - bbeg + nu - 1) / nu : 1;
    return (u + TP_TILE - 1) / TP_TILE * TP_TILE;
}

// S_B (Alg. 1 output), bucket starts (Alg. 2 read head) and the
// round-1 unit plan. One block.
// reserved = 1: after k_scatter0r (runs only if the reservation held: no
// bucket above its capacity; hist0 = the final cursors). reserved = 0: after
// the exact count pass (runs only if round 0 had to be exact; bsrc = start0).
__global__ void __launch_bounds__(1024) k_plan0(Args a, uint64_t *dS_B, int reserved) {
    __shared__ uint32_t s[LS_MAX_FANOUT + 1];
    __shared__ uint32_t nu[LS_MAX_FANOUT + 1];
    __shared__ uint32_t tmp[33];
    const int f = a.f, tid = threadIdx.x;
    if (reserved) {
        if (a.ctl->exact0 || a.ctl->status) return;
        bool over = false;
        for (int b = tid; b < f; b += blockDim.x) over |= a.cur0[b] > a.cap0[b];
        if (__syncthreads_or(over)) {
            if (tid == 0) a.ctl->exact0 = 1u;
            return;
        }
        for (int b = tid; b < f; b += blockDim.x) a.hist0[b] = a.cur0[b];
        __syncthreads();
    } else if (!a.ctl->exact0) {
        return;
    }
    for (int b = tid; b < f; b += blockDim.x) {
        const uint64_t h = a.hist0[b];
        s[b] = (uint32_t)h;
        nu[b] = unit1_count(h, a.C1);
        if (dS_B) dS_B[b] = h;
    }
    __syncthreads();
    const uint32_t total = block_exscan(s, f, tmp);
    const uint32_t units = block_exscan(nu, f, tmp);
    for (int b = tid; b < f; b += blockDim.x) {
        a.start0[b] = s[b];
        if (!reserved) a.bsrc[b] = s[b];
        a.unit1_start[b] = nu[b];
        // cluster-resident round 1 (ls_round1.cu) for buckets of fr_min..fr_cap keys
        const uint64_t h = a.hist0[b];
        const bool fu = a.fr_min != 0 && h >= a.fr_min && h <= a.fr_cap;
        a.fused[b] = fu ? 1u : 0u;
        if (fu) a.flist[atomicAdd(&a.ctl->nfused, 1u)] = (uint32_t)b;
    }
    if (tid == 0) {
        a.start0[f] = total;
        if (!reserved) a.bsrc[f] = total;
        a.unit1_start[f] = units;
        a.ctl->U1 = units;
        if ((uint64_t)total != a.n) atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
    }
}

// Bucket ids precomputed by the count pass (tile_partition BIDS mode).
struct NoBucket {
    __device__ __forceinline__ uint32_t operator()(uint64_t, uint64_t) const { return 0u; }
};

// Level-0 bucket through the b0 search tables (shared memory).
template <int DT>
struct B0Bucket {
    B0Search bs;
    __device__ __forceinline__ uint32_t operator()(uint64_t key, uint64_t) const {
        return bs.get<DT>(key);
    }
};

struct Scatter0Smem {
    TpSmem tp;
    uint32_t base[LS_MAX_FANOUT];
    B0Smem b0;
};

template <int DT>
__global__ void __launch_bounds__(TP_THREADS, 1) k_scatter0(Args a) {
    if (a.ctl->status || !a.ctl->exact0) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Scatter0Smem &S = *reinterpret_cast<Scatter0Smem *>(smem_raw);
    const int f = a.f, tid = threadIdx.x;
    // a contiguous run of count0 units [u0, u1) per CTA: the cursors of unit
    // u0 (count0's lookback offsets) run on into u0 + 1, ... because those
    // offsets are exclusive prefix sums over the units (one tile stream, one
    // search-table load and one pipeline start per CTA instead of per unit)
    const uint64_t u0 = (uint64_t)blockIdx.x * a.U0 / gridDim.x;
    const uint64_t u1 = (uint64_t)(blockIdx.x + 1) * a.U0 / gridDim.x;
    if (u1 <= u0) return;
    const B0Bucket<DT> bf{load_b0_search(S.b0, a.M)};
    if (tid < f) S.base[tid] = (uint32_t)a.start0[tid] + a.offs0[u0 * f + tid];
    tp_init(S.tp);
    const uint64_t beg = u0 * a.C0, end = umin64(a.n, u1 * a.C0);
    uint32_t phase = 0;
    tile_partition(S.tp, a.A, a.B, beg, end, a.n, S.base, f, bf, phase, nullptr, (TpBids *)nullptr,
                   (a.dbg & 1024u) ? a.ctl->prof : nullptr);
}

// ------------------------------------------- round 0 by reservation ------
// The paper fills fixed-capacity fragments to avoid a separate counting scan
// (P:263-267); here each level-0 bucket gets a capacity estimated from the 1 %
// sample the model was fitted on (its sample count c_b, scaled by n/m, plus
// 5 standard deviations), the scatter reserves every tile's run in its bucket
// with one atomicAdd, and the count pass (k_count0) runs only if a bucket
// overflowed or the capacities did not fit B. S_B = the final cursors (exact).
// The sample's level-0 histogram, b0 = bucket0(predict(x)) (O7) with the
// leaf lines staged in shared memory: it needs only the fitted model, not the
// b0 search tables, so it runs on the side stream while k_b0_* build them.
// 8 independent keys per thread.
struct SampHistSmem {
    double leaf[5 * LS_MAX_LEAVES];
    uint32_t h[LS_MAX_FANOUT];
};
constexpr int SH_THREADS = 512;
template <int DT>
__global__ void __launch_bounds__(SH_THREADS, 2) k_samp_hist0(Args a, uint64_t m) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SampHistSmem &S = *reinterpret_cast<SampHistSmem *>(smem_raw);
    const int f = a.f, tid = threadIdx.x;
    for (int b = tid; b < f; b += SH_THREADS) S.h[b] = 0;
    const int L = (int)a.M->L;
    for (int i = tid; i < 5 * L; i += SH_THREADS) S.leaf[i] = a.M->leaf[i];
    const Root R = load_root(a.M);
    const double F = a.F;
    __syncthreads();
    constexpr int U = 8;
    const uint64_t gs = (uint64_t)gridDim.x * SH_THREADS * U;
    for (uint64_t i = (uint64_t)blockIdx.x * SH_THREADS * U + tid; i < m; i += gs) {
        uint64_t k[U];
#pragma unroll
        for (int q = 0; q < U; q++) k[q] = i + q * SH_THREADS < m ? a.S[i + q * SH_THREADS] : 0ull;
#pragma unroll
        for (int q = 0; q < U; q++)
            if (i + q * SH_THREADS < m) atomicAdd(&S.h[bucket0(predict<DT>(k[q], R, S.leaf), F, f)], 1u);
    }
    __syncthreads();
    for (int b = tid; b < f; b += SH_THREADS)
        if (S.h[b]) atomicAdd(&a.shist0[b], S.h[b]);
}

__global__ void __launch_bounds__(1024) k_cap0(Args a, uint64_t m) {
    __shared__ unsigned long long wsum[32];
    const int f = a.f, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const double scale = (double)a.n / (double)(m ? m : 1);
    unsigned long long cap = 0;
    if (tid < f) {
        const double c = (double)a.shist0[tid];
        cap = (unsigned long long)ceil(scale * (c + 5.0 * sqrt(c) + 5.0));
        a.cap0[tid] = cap;
    }
    // exclusive scan of the capacities (64-bit)
    unsigned long long v = cap;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) wsum[w] = v;
    __syncthreads();
    if (w == 0) {
        unsigned long long x = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0ull, y = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) y += t;
        }
        wsum[lane] = y - x;
    }
    __syncthreads();
    const unsigned long long ex = wsum[w] + v - cap;
    if (tid < f) a.bsrc[tid] = ex;
    if (tid == f - 1) {
        const unsigned long long total = ex + cap;
        a.bsrc[f] = total;
        if (a.force_exact0 || total > a.Bcap || a.Bcap + (uint64_t)TP_TILE >= (1ull << 32)) a.ctl->exact0 = 1u;
    }
}

struct Scatter0rSmem {
    TpSmem tp;
    B0Smem b0;
};

template <int DT>
__global__ void __launch_bounds__(TP_THREADS, 1) k_scatter0r(Args a) {
    if (a.ctl->status || a.ctl->exact0) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Scatter0rSmem &S = *reinterpret_cast<Scatter0rSmem *>(smem_raw);
    __shared__ int s_nan;
    // a contiguous run of tiles per CTA
    const uint64_t ntiles = (a.n + TP_TILE - 1) / TP_TILE;
    const uint64_t t0 = (uint64_t)blockIdx.x * ntiles / gridDim.x;
    const uint64_t t1 = (uint64_t)(blockIdx.x + 1) * ntiles / gridDim.x;
    if (t1 <= t0) return;
    if (threadIdx.x == 0) s_nan = 0;
    const B0Search bs = load_b0_search(S.b0, a.M);
    tp_init(S.tp);
    bool nan = false;
    auto bf = [&](uint64_t key, uint64_t) -> uint32_t {
        if (DT == DT_F64) {  // NaN check on the (otherwise idle) fp64 pipe: x != x
            const double x = __longlong_as_double((long long)key);
            nan |= x != x;
        }
        return bs.get<DT>(key);
    };
    const TpReserve rs{a.cur0, a.cap0, a.bsrc, &a.ctl->exact0, (uint32_t)a.Bcap, nullptr};
    uint32_t phase = 0;
    tile_partition<false, false, false, decltype(bf), TP_THREADS, TP_KPT, TpBids, true>(
        S.tp, a.A, a.B, t0 * TP_TILE, umin64(a.n, t1 * TP_TILE), a.n, nullptr, a.f, bf, phase, nullptr,
        (TpBids *)nullptr, (a.dbg & 1024u) ? a.ctl->prof : nullptr, &rs);
    if (nan) s_nan = 1;
    __syncthreads();
    if (threadIdx.x == 0 && s_nan) atomicOr(&a.ctl->status, (uint32_t)STATUS_NAN);
}

// --------------------------------------------------------------- round 1 ---
__device__ __forceinline__ int find_bucket(const uint32_t *ustart, int f, uint32_t u) {
    int lo = 0, hi = f - 1;  // largest b with ustart[b] <= u
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (ustart[mid] <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Leaf staging of k_count1, measured per key type at 200M: fp64 keys run
// faster with only the bucket's leaf range staged (static 2.5 KB; a wide range
// reads the leaves through L1), uint64 keys (wide ranges over clustered
// values) with every leaf in dynamic shared memory.
template <int DT>
constexpr bool C1_NARROW = DT == DT_F64;
constexpr int C1_LEAVES = 64;
// p of a key of a bucket whose keys all route to one leaf (its line in
// registers): predict() without the routing and the leaf loads
template <int DT>
struct OneLeaf {
    double la, lc, lb, llo, lhi;
    __device__ __forceinline__ double operator()(uint64_t key) const {
        const double y = __fma_rn(la, __dsub_rn(xd<DT>(key), lc), lb);
        return __dadd_rn(clampd(y, llo, lhi), 0.0);
    }
};
template <int DT, bool INNER>
struct LeafTable {
    const Root &R;
    const double *leaf;
    __device__ __forceinline__ double operator()(uint64_t key) const { return predict_c<DT, INNER>(key, R, leaf); }
};

template <class PRED>
__device__ __forceinline__ void count1_range(const Args &a, int b, uint64_t beg, uint64_t end, uint64_t k0,
                                             const PRED &pred, uint32_t *hist, bool &diff) {
    const int tid = threadIdx.x, bd = blockDim.x, f = a.f;
    auto one = [&](uint64_t key) -> uint32_t {
        diff |= key != k0;
        const double p = pred(key);  // keys of one bucket: 1-2 leaves, broadcast
        const uint32_t b1 = bucket1(p, a.F2, f, (uint32_t)b);
        atomicAdd(&hist[b1], 1u);
        return b1;
    };
    {
        // 16-byte loads, 4 in flight per thread; odd head / tail keys apart.
        // b1 of every key is kept (2 bytes) for k_scatter1.
        uint64_t i0 = beg;
        if ((i0 & 1) && i0 < end) {
            if (tid == 0) a.bid[i0] = (uint16_t)one(a.B[i0]);
            i0++;
        }
        const ulonglong2 *B2 = reinterpret_cast<const ulonglong2 *>(a.B + i0);
        uint32_t *bid2 = reinterpret_cast<uint32_t *>(a.bid + i0);
        const uint64_t np = (end - i0) / 2;
        uint64_t i = tid;
        for (; i + 3 * bd < np; i += 4 * bd) {
            ulonglong2 v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = __ldcs(B2 + i + q * bd);
#pragma unroll
            for (int q = 0; q < 4; q++) bid2[i + q * bd] = one(v[q].x) | (one(v[q].y) << 16);
        }
        for (; i < np; i += bd) {
            const ulonglong2 v = __ldcs(B2 + i);
            bid2[i] = one(v.x) | (one(v.y) << 16);
        }
        if (((end - i0) & 1) && tid == 0) a.bid[end - 1] = (uint16_t)one(a.B[end - 1]);
    }
}

template <int DT>
__global__ void __launch_bounds__(512, 3) k_count1(Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];  // (!C1_NARROW: all leaves)
    __shared__ double s_leaf[C1_NARROW<DT> ? 5 * C1_LEAVES : 2];
    __shared__ uint32_t hist[LS_MAX_FANOUT];
    __shared__ uint32_t ustart[LS_MAX_FANOUT + 1];
    __shared__ uint32_t s_unit;
    const int tid = threadIdx.x, bd = blockDim.x, f = a.f;
    if (tid == 0) s_unit = atomicAdd(&a.ctl->ticket1, 1u);
    for (int b = tid; b <= f; b += bd) ustart[b] = a.unit1_start[b];
    for (int b = tid; b < f; b += bd) hist[b] = 0;
    __syncthreads();
    const uint32_t u = s_unit;
    if (u >= a.ctl->U1 || a.ctl->status) return;
    const int b = find_bucket(ustart, f, u);
    if (a.fused[b]) return;  // partitioned by k_round1
    // the leaves this bucket's keys can route to: the leaf index is monotone in
    // the key, and the bucket holds the ords [thr[b-1], thr[b]) (b0 thresholds),
    // so only leaves llo..lhi are staged (typically one or two, not all L)
    const Root R = load_root(a.M);
    const double *leaf = a.M->leaf;
    int llo, lhi;
    {
        double xc;
        llo = b > 0 ? root_leaf<DT>(from_ord<DT>(a.M->thr[b - 1]), R, xc) : 0;
        lhi = (uint32_t)b < a.M->nthr ? root_leaf<DT>(from_ord<DT>(a.M->thr[b] - 1ull), R, xc) : R.Lm1;
        if (C1_NARROW<DT>) {
            if (llo >= 0 && llo <= lhi && lhi - llo < C1_LEAVES) {
                for (int i = tid; i < 5 * (lhi - llo + 1); i += bd) s_leaf[i] = a.M->leaf[5 * llo + i];
                leaf = s_leaf - 5 * llo;
            }  // (else through L1)
        } else {
            if (!(llo >= 0 && llo <= lhi && lhi <= R.Lm1)) {  // (defensive: stage them all)
                llo = 0;
                lhi = R.Lm1;
            }
            double *sl = reinterpret_cast<double *>(smem_raw);  // leaves at their own index
            for (int i = 5 * llo + tid; i < 5 * (lhi + 1); i += bd) sl[i] = a.M->leaf[i];
            leaf = sl;
        }
        __syncthreads();
    }
    const uint32_t slice = u - ustart[b];
    // bucket b sits in B at [bsrc[b], + its size) (round 0's reserved region)
    const uint64_t bbeg = a.bsrc[b], bend = bbeg + (a.start0[b + 1] - a.start0[b]);
    const uint64_t usz = unit1_size(bbeg, bend, ustart[b + 1] - ustart[b]);
    const uint64_t beg = umin64(bend, bbeg + (uint64_t)slice * usz);  // (tile rounding can
    const uint64_t end = umin64(bend, beg + usz);                    //  leave a unit empty)
    // H0: is every key of bucket b equal to its first key?
    const uint64_t k0 = a.B[bbeg];
    bool diff = false;
    // only the buckets of xmin and xmax can hold keys outside [xmin, xmax]
    // (they are clamped onto xmin / xmax): elsewhere the root clamp is skipped
    const uint32_t b_lo = sub_bucket_at(R.xmin, R, a.M->leaf, a.F, a.F2, f) / (uint32_t)f;
    const uint32_t b_hi = sub_bucket_at(R.xmax, R, a.M->leaf, a.F, a.F2, f) / (uint32_t)f;
    if ((uint32_t)b != b_lo && (uint32_t)b != b_hi) {
        if (llo == lhi) {  // every key of the bucket routes to leaf llo
            const double *q = a.M->leaf + 5 * llo;
            const OneLeaf<DT> pred{__ldg(q), __ldg(q + 1), __ldg(q + 2), __ldg(q + 3), __ldg(q + 4)};
            count1_range(a, b, beg, end, k0, pred, hist, diff);
        } else {  // (two leaves with both lines in registers measured slower: 0.43 vs 0.40 ms)
            count1_range(a, b, beg, end, k0, LeafTable<DT, true>{R, leaf}, hist, diff);
        }
    } else {
        count1_range(a, b, beg, end, k0, LeafTable<DT, false>{R, leaf}, hist, diff);
    }
    // bmin0[b] = ord of the bucket's first key, bmax0[b] != 0 iff two keys differ
    if (__syncthreads_or(diff) && tid == 0) a.bmax0[b] = 1ull;
    if (tid == 0 && beg < end) a.bmin0[b] = to_ord<DT>(k0);
    for (int j = tid; j < f; j += bd) {
        const uint32_t c = hist[j];
        if (c) atomicAdd(&a.hist1[(uint64_t)b * f + j], c);
    }
}

constexpr uint64_t S1P_MAX_N = 128ull << 20;
template <int NT>
struct Scatter1SmemT {
    TpSmemT<NT, TP_KPT> tp;
    alignas(16) TpBidsT<NT * TP_KPT> sbid;
    uint32_t ustart[LS_MAX_FANOUT + 1];
};
typedef Scatter1SmemT<TP_THREADS> Scatter1Smem;
// (measured: two 512-thread CTAs per SM with 4K-key tiles, 1.40 ms against
// 1.03 ms for one 1024-thread CTA with 8K-key tiles at 200M Normal)

static_assert(sizeof(Scatter0Smem) <= MAX_SMEM_OPTIN, "scatter0 shared memory");
static_assert(sizeof(Scatter0rSmem) + 64 <= MAX_SMEM_OPTIN, "scatter0r shared memory");
static_assert(sizeof(Scatter1Smem) <= MAX_SMEM_OPTIN, "scatter1 shared memory");

template <int DT, int NT>
__global__ void __launch_bounds__(NT, TP_THREADS / NT) k_scatter1(Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Scatter1SmemT<NT> &S = *reinterpret_cast<Scatter1SmemT<NT> *>(smem_raw);
    const int f = a.f, tid = threadIdx.x, bd = NT;
    const uint32_t u = blockIdx.x;
    if (u >= a.ctl->U1 || a.ctl->status) return;
    for (int b = tid; b <= f; b += bd) S.ustart[b] = a.unit1_start[b];
    __syncthreads();
    const int b = find_bucket(S.ustart, f, u);
    if (a.fused[b]) return;  // partitioned by k_round1
    const uint32_t slice = u - S.ustart[b];
    // B side: the bucket's region from round 0 (bsrc); A side: start0
    const uint64_t bbeg = a.bsrc[b], bend = bbeg + (a.start0[b + 1] - a.start0[b]);
    const uint64_t usz = unit1_size(bbeg, bend, S.ustart[b + 1] - S.ustart[b]);
    const uint64_t beg = umin64(bend, bbeg + (uint64_t)slice * usz);  // (may be empty: tile rounding)
    const uint64_t end = umin64(bend, beg + usz);
    const unsigned long long mn = a.bmin0[b];
    if (bend - bbeg <= 1 || a.bmax0[b] == 0ull) {
        // homogeneous level-0 bucket: already in final position
        // after defragmentation; here it is written straight from its value.
        const uint64_t v = from_ord<DT>(mn);
        uint64_t *Ab = a.A + a.start0[b] - bbeg;
        for (uint64_t i = beg + tid; i < end; i += bd) Ab[i] = v;
        return;
    }
    // the first tiles are staged right away. Every tile reserves its run in
    // sub-bucket g with one atomicAdd on g's cursor (k_classify: cur1 = start1;
    // the counts are exact, so nothing overflows): the runs of one sub-bucket
    // are written front to back in time by whichever CTAs hold its keys, so
    // its L2 sectors fill up before they are evicted. (Per-unit regions,
    // start1 + the unit's offset, left each unit's boundary sectors partly
    // written for a whole CTA lifetime: ~0.36 GB of DRAM read-modify-write
    // per 200M keys.)
    if (tid == 0) tp_issue_first(S.tp, a.B, beg, end, a.Bcap, a.bid, &S.sbid);
    __syncthreads();
    uint32_t phase = 0;
    const NoBucket bf{};
    const TpReserve rs{nullptr, nullptr, nullptr, nullptr, (uint32_t)a.n, a.cur1 + (uint64_t)b * f};
    tile_partition<false, true, true, NoBucket, NT, TP_KPT, TpBidsT<NT * TP_KPT>, true>(
        S.tp, a.B, a.A, beg, end, a.Bcap, nullptr, f, bf, phase, a.bid, &S.sbid,
        (a.dbg & 2048u) ? a.ctl->prof + 5 : nullptr, &rs);
}

// Round-1 scatter, persistent form (LS_SCATTER1P): one CTA per SM takes the
// tiles of all level-0 buckets in bucket order from a ticket counter, the ring
// staged one tile ahead across bucket boundaries. At any time the grid works
// on ~148 consecutive tiles (about six level-0 buckets: few open sub-bucket
// write streams), no CTA waits for its first tile with an idle SM, and there is
// no last-wave tail. Same per-tile steps as tile_partition<BIDS, RESERVE> with
// the exact 32-bit cursors of the tile's bucket; homogeneous level-0 buckets
// are written from their value, tile by tile.
struct S1Desc {
    uint64_t t0;       // first staged position in B (even) / first position of a fill tile
    uint32_t th, lo;   // slot positions [lo, th) are this tile's keys
    uint32_t b, kind;  // level-0 bucket; 0: no more tiles, 1: partition tile, 2: fill tile
};
struct Scatter1pSmem {
    TpSmem tp;
    alignas(16) TpBids sbid;
    uint32_t tstart[LS_MAX_FANOUT + 1];
    uint32_t bbeg[LS_MAX_FANOUT], bsz[LS_MAX_FANOUT];  // each bucket's region in B (positions fit 32 bits: cur1)
    uint8_t bh0[LS_MAX_FANOUT];                        // 1: homogeneous (fill tiles)
    uint32_t tmp[33];
    S1Desc desc[TP_NSLOT];
};
static_assert(sizeof(Scatter1pSmem) <= MAX_SMEM_OPTIN, "scatter1p shared memory");
static_assert(TP_NSLOT == 2 && TP_THREADS >= LS_MAX_FANOUT, "k_scatter1p: two ring slots, bucket b <-> thread b");

template <int DT>
__global__ void __launch_bounds__(TP_THREADS, 1) k_scatter1p(Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Scatter1pSmem &S = *reinterpret_cast<Scatter1pSmem *>(smem_raw);
    constexpr int NT = TP_THREADS, KPT = TP_KPT, TILE = TP_TILE;
    const int f = a.f, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (a.ctl->status) return;
    // tiles per level-0 bucket (tiles start at even positions of B, as in
    // tile_partition), then their exclusive prefix: tile ticket -> bucket
    for (int b = tid; b <= f; b += NT) {
        uint32_t nt = 0;
        if (b < f) {
            const uint64_t bbeg = a.bsrc[b], h = a.fused[b] ? 0ull : a.start0[b + 1] - a.start0[b];
            const bool h0 = h <= 1 || a.bmax0[b] == 0ull;
            if (h) nt = (uint32_t)(((h0 ? h : bbeg + h - (bbeg & ~1ull)) + TILE - 1) / TILE);
            S.bbeg[b] = (uint32_t)bbeg;
            S.bsz[b] = (uint32_t)h;
            S.bh0[b] = h0;
        }
        S.tstart[b] = nt;
    }
    for (int b = tid; b < f; b += NT) S.tp.cnt[b] = 0;
    if (tid == 0) {
        for (int j = 0; j < TP_NSLOT; j++) mbar_init(&S.tp.mbar[j], 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (inits before the bulk copies)
    }
    __syncthreads();
    const uint32_t total = block_exscan(S.tstart, f + 1, S.tmp);
    // thread 0: take the next tile ticket, describe it in desc[slot] and stage it
    // (the ticket after the next is drawn one tile early: the atomic's
    // round trip is over by the time take() needs it; the bucket regions are
    // in shared memory, so take() is a bisection and one bulk-copy issue)
    uint32_t ahead = 0;
    auto take = [&](int slot) {
        const uint32_t tk = ahead;
        ahead = atomicAdd(&a.ctl->ticket_s1, 1u);
        S1Desc d{0ull, 0u, 0u, 0u, 0u};
        if (tk < total) {
            const int b = find_bucket(S.tstart, f, tk);
            const uint32_t k = tk - S.tstart[b];
            const uint64_t bbeg = S.bbeg[b], h = S.bsz[b], bend = bbeg + h;
            d.b = (uint32_t)b;
            if (S.bh0[b]) {
                d.kind = 2u;
                d.t0 = bbeg + (uint64_t)k * TILE;
                d.th = (uint32_t)umin64((uint64_t)TILE, bend - d.t0);
            } else {
                const uint64_t tbase = bbeg & ~1ull;
                d.kind = 1u;
                d.t0 = tbase + (uint64_t)k * TILE;
                d.th = (uint32_t)umin64((uint64_t)TILE, bend - d.t0);
                d.lo = k == 0 ? (uint32_t)(bbeg - tbase) : 0u;
                tp_issue<TpSmem, TpBids>(S.tp, slot, a.B, d.t0, d.t0 + d.th, a.Bcap, a.bid, &S.sbid);
            }
        }
        S.desc[slot] = d;
    };
    if (tid == 0) {
        ahead = atomicAdd(&a.ctl->ticket_s1, 1u);
        for (int j = 0; j < TP_NSLOT; j++) take(j);
    }
    __syncthreads();
    uint32_t phase = 0;
    uint64_t *const dst = a.A;
    const uint32_t lim = (uint32_t)a.n;
    for (uint32_t i = 0;; i++) {
        const int slot = (int)(i & 1u);
        const S1Desc d = S.desc[slot];
        if (d.kind == 0u) break;
        if (d.kind == 2u) {  // homogeneous level-0 bucket: written straight from its value
            const uint64_t v = from_ord<DT>(a.bmin0[d.b]);
            uint64_t *Ab = a.A + a.start0[d.b] - a.bsrc[d.b] + d.t0;
            for (uint32_t j = tid; j < d.th; j += NT) Ab[j] = v;
            __syncthreads();
            if (tid == 0 && i >= 1) take(slot ^ 1);
            __syncthreads();
            continue;
        }
        const int th = (int)d.th, lo = (int)d.lo, tn = th - lo;
        uint32_t *const cur = a.cur1 + (uint64_t)d.b * f;
        mbar_wait(&S.tp.mbar[slot], (phase >> slot) & 1u);
        const uint64_t *keys = S.tp.ring[slot];
        const uint16_t *bids = S.sbid[slot] + (d.t0 & 7);
        uint64_t key[KPT];
        uint32_t code[KPT];
#pragma unroll
        for (int k2 = 0; k2 < KPT / 2; k2++) {
            const int h = 2 * (k2 * NT + tid);
            const ulonglong2 kv = *reinterpret_cast<const ulonglong2 *>(keys + h);
            const uint32_t ip = *reinterpret_cast<const uint32_t *>(bids + h);
            key[2 * k2] = kv.x;
            key[2 * k2 + 1] = kv.y;
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int k = 2 * k2 + e;
                code[k] = 0xffffffffu;
                if (h + e >= lo && h + e < th) {
                    const uint32_t b1 = e ? ip >> 16 : ip & 0xffffu;
                    const uint32_t r = atomicAdd(&S.tp.cnt[b1], 1u);
                    code[k] = b1 | (r << 10);
                }
            }
        }
        __syncthreads();
        // every thread is past the previous tile's store phase: its ring slot
        // and descriptor are free for the tile after this one
        if (tid == 0 && i >= 1) take(slot ^ 1);
        // exclusive scan of the tile's sub-bucket counts (bucket tid <-> thread tid)
        const uint32_t c = tid < f ? S.tp.cnt[tid] : 0u;
        const uint32_t rsv = c ? atomicAdd(&cur[tid], c) : 0u;  // (first needed after the placement)
        const uint32_t incl = warp_incl_scan(c);
        if (lane == 31) S.tp.wsum[warp] = incl;
        __syncthreads();
        const uint32_t ws = lane < NT / 32 ? S.tp.wsum[lane] : 0u;
        const uint32_t wpre = __reduce_add_sync(0xffffffffu, lane < warp ? ws : 0u);
        const uint32_t ex0 = wpre + incl - c;
        if (tid < f) {
            S.tp.ex[tid] = ex0;
            S.tp.cnt[tid] = 0;
        }
        __syncthreads();
        uint64_t *sk = S.tp.ring[slot];
        uint32_t pos[KPT];
#pragma unroll
        for (int k = 0; k < KPT; k++)
            pos[k] = code[k] != 0xffffffffu ? S.tp.ex[code[k] & 1023u] + (code[k] >> 10) : 0xffffffffu;
#pragma unroll
        for (int k = 0; k < KPT; k++) {
            if (pos[k] != 0xffffffffu) {
                sk[pos[k]] = key[k];
                S.tp.sbin[pos[k]] = (uint16_t)(code[k] & 1023u);
            }
        }
        if (c) S.tp.delta[tid] = rsv - ex0;
        __syncthreads();
        {
            uint32_t bb[KPT], dd[KPT];
            uint64_t v[KPT];
#pragma unroll
            for (int k = 0; k < KPT; k++) {
                const int idx = k * NT + tid;
                bb[k] = idx < tn ? S.tp.sbin[idx] : 0u;
                v[k] = sk[idx];
            }
#pragma unroll
            for (int k = 0; k < KPT; k++) dd[k] = S.tp.delta[bb[k]];
#pragma unroll
            for (int k = 0; k < KPT; k++) {
                const int idx = k * NT + tid;
                const uint32_t q = dd[k] + (uint32_t)idx;
                if (idx < tn && q < lim) dst[q] = v[k];
            }
        }
        // (no barrier: the next tile's first barrier orders these reads of the
        // slot, sbin and delta before anything overwrites them)
        phase ^= 1u << slot;
    }
}

// ------------------------------------------------------------- classify ----
// Per level-0 bucket b (one block): H0, S'_B row, sub-bucket starts,
// H1 for n' <= 1, SMALL -> bucket-sort tiles, BIG -> big-path list.
// The per-sub-bucket part of k_classify: starts and cursors, H1 for n' <= 1
// (P:183), block windows, big-path items.
__device__ __forceinline__ void classify_rest(const Args &a, uint64_t g, uint32_t st, uint32_t c, int sc, int lane) {
    a.start1[g] = st;
    a.cur1[g] = st;
    if (sc == SC_TRIVIAL) {
        if (a.dH1) a.dH1[g] = 1;
    } else if (sc == SC_WINDOW) {  // tiny sub-buckets: block windows
        // (the first / last window sub-bucket of each tile among this
        // warp's lanes does the atomics: st and g grow with the lane)
        const uint32_t t = st / a.T_tile;
        const uint32_t wm = __activemask();
        const uint32_t below = wm & ((1u << lane) - 1u), above = wm & ~((2u << lane) - 1u);
        const uint32_t tp = __shfl_sync(wm, t, below ? 31 - __clz(below) : lane);
        const uint32_t tn = __shfl_sync(wm, t, above ? __ffs(above) - 1 : lane);
        if (!below || tp != t) atomicMin(&a.tile_first[t], (uint32_t)g);
        if (!above || tn != t) atomicMax(&a.tile_last[t], (uint32_t)g);
    } else if (sc == SC_BIG) {
        const uint32_t k = atomicAdd(&a.ctl->big_cnt[0], 1u);
        if (k < a.big_cap) {
            uint32_t lrk = 0;  // large items: grid-parallel path (ls_bigpath.cu)
            if (c > LARGE_MIN) {
                const uint32_t li = atomicAdd(&a.ctl->nlarge, 1u);
                if (li < a.lcap) {
                    a.large[li] = k;
                    lrk = li + 1u;
                } else {
                    atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
                }
            }
            a.big[k] = BigItem{st, c, 0u, (uint32_t)g, ~0ull, 0ull, lrk, 0u};
            const uint32_t nch = (c + MM_CHUNK - 1) / MM_CHUNK;
            const uint32_t base = atomicAdd(&a.ctl->nchunks, nch);
            for (uint32_t q = 0; q < nch; q++)
                if (base + q < a.chunk_cap) a.chunks[base + q] = BigChunk{k, q};
                else atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
        } else {
            atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
        }
    }
}

// 256 threads x 4 sub-buckets per thread: the block is a chain of dependent
// loads, barriers and one global atomic (latency-bound), so all f blocks are
// made resident at once (8 per SM) instead of 2 per SM in waves.
constexpr int CL_THREADS = 256;
constexpr int CL_Q = LS_MAX_FANOUT / CL_THREADS;  // sub-buckets per thread
static_assert(CL_Q * CL_THREADS == LS_MAX_FANOUT && CL_Q * (CL_THREADS / 32) == 32, "k_classify: 32 warp rows");
__global__ void __launch_bounds__(CL_THREADS, 7) k_classify(Args a) {
    __shared__ uint32_t s[LS_MAX_FANOUT];
    __shared__ uint32_t tmp[33];
    __shared__ uint32_t wcnt[5][32], wbase[5];
    const int b = blockIdx.x, f = a.f, tid = threadIdx.x;
    const int lane = tid & 31, w = tid >> 5;
    const uint64_t row = (uint64_t)b * f;
    const uint64_t bbeg = a.start0[b], nb = a.start0[b + 1] - bbeg;
    const bool h0 = nb <= 1 || a.bmax0[b] == 0ull;
    if (h0) {
        if (tid == 0) {
            if (a.dH0) a.dH0[b] = 1;
            if (nb >= 2) {
                atomicAdd(&a.ctl->stat[ST_H0B], 1ull);
                atomicAdd(&a.ctl->stat[ST_H0K], (unsigned long long)nb);
            }
        }
        for (int j = tid; j < f; j += CL_THREADS) {
            a.hist1[row + j] = 0;
            a.start1[row + j] = (uint32_t)bbeg;
        }
        return;
    }
    // sub-buckets q * CL_THREADS + tid, q < CL_Q: warp w's q-th group is the
    // 32 consecutive sub-buckets of warp row q * 8 + w
    uint32_t c[CL_Q];
#pragma unroll
    for (int q = 0; q < CL_Q; q++) {
        const int j = q * CL_THREADS + tid;
        c[q] = j < f ? a.hist1[row + j] : 0u;
        if (j < f) s[j] = c[q];
    }
    __syncthreads();
    const uint32_t total = block_exscan(s, f, tmp);
    if (tid == 0 && total != nb) atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
    // SMALL sub-buckets of <= WS_MAX keys become warp tasks, larger ones CTA
    // tasks (compacted per block: one global atomic per level-0 bucket and
    // class). A bucket of the cluster-resident round 1 has its warp-sized
    // sub-buckets sorted there already (k_round1's P5).
    uint32_t st[CL_Q], m[CL_Q][5];
    int sc[CL_Q];
    const bool fused = a.fused[b];
#pragma unroll
    for (int q = 0; q < CL_Q; q++) {
        const int j = q * CL_THREADS + tid;
        st[q] = j < f ? (uint32_t)bbeg + s[j] : 0u;
        const int sc0 = j < f ? size_class(c[q], a.T_small) : SC_TRIVIAL;
        sc[q] = (sc0 == SC_WARP && fused) ? SC_FUSED : sc0;
        m[q][0] = __ballot_sync(0xffffffffu, sc[q] == SC_WARP);
        m[q][1] = __ballot_sync(0xffffffffu, sc[q] == SC_CTA);
        m[q][2] = __ballot_sync(0xffffffffu, sc[q] == SC_CTAM);
        m[q][3] = __ballot_sync(0xffffffffu, sc[q] == SC_CTAL);
        m[q][4] = __ballot_sync(0xffffffffu, sc[q] == SC_CTAS);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 5; k++) wcnt[k][q * (CL_THREADS / 32) + w] = __popc(m[q][k]);
        }
    }
    __syncthreads();
    if (tid < 5) {
        uint32_t tot = 0;
        for (int r = 0; r < 32; r++) {
            const uint32_t t = wcnt[tid][r];
            wcnt[tid][r] = tot;
            tot += t;
        }
        uint32_t *ctr = tid == 0 ? &a.ctl->ntask : tid == 1 ? &a.ctl->nctask
                      : tid == 2 ? &a.ctl->nctask2 : tid == 3 ? &a.ctl->nctask3 : &a.ctl->nctask4;
        wbase[tid] = tot ? atomicAdd(ctr, tot) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < CL_Q; q++) {
        const int j = q * CL_THREADS + tid;
        const int wr = q * (CL_THREADS / 32) + w;
        const uint64_t g = row + (uint64_t)(j < f ? j : 0);
        const int c2 = sc[q] == SC_WARP ? 0 : sc[q] == SC_CTA ? 1 : sc[q] == SC_CTAM ? 2
                     : sc[q] == SC_CTAL ? 3 : sc[q] == SC_CTAS ? 4 : -1;
        // tasks carry the leaf that holds all their keys (+1; 0: none)
        const uint32_t wl = (m[q][0] | m[q][1] | m[q][2] | m[q][3] | m[q][4])
                                ? contained_leaf_warp(a.M->leaf, (int)a.M->L, (uint32_t)(row + (j & ~31)),
                                                      (uint32_t)g, a.rcpF2, lane)
                                : 0u;
        if (c2 >= 0) {
            const uint32_t mc = c2 == 0 ? m[q][0] : c2 == 1 ? m[q][1] : c2 == 2 ? m[q][2] : c2 == 3 ? m[q][3] : m[q][4];
            const uint32_t k = wbase[c2] + wcnt[c2][wr] + __popc(mc & ((1u << lane) - 1u));
            uint4 *list = c2 == 0 ? a.tasks : c2 == 1 ? a.ctasks : c2 == 2 ? a.ctasks2 : c2 == 3 ? a.ctasks3 : a.ctasks4;
            if (k < a.task_cap) list[k] = make_uint4(st[q], c[q], (uint32_t)g, wl);
            else atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
        }
        if (j < f) classify_rest(a, g, st[q], c[q], sc[q], lane);
    }
}

// ---------------------------------------------------------- parity hooks ---
template <int DT>
__global__ void k_bucket_ids(const uint64_t *__restrict__ keys, uint64_t n, int f,
                             const DevModel *M, double *p_out, uint32_t *b0_out, uint32_t *b1_out,
                             unsigned long long *h0, unsigned long long *h1) {
    const Root R = load_root(M);
    const double F = (double)f, F2 = (double)f * (double)f;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gs) {
        const double p = predict_ldg<DT>(keys[i], R, M->leaf);
        const uint32_t b0 = bucket0(p, F, f), b1 = bucket1(p, F2, f, b0);
        if (p_out) p_out[i] = p;
        if (b0_out) b0_out[i] = b0;
        if (b1_out) b1_out[i] = b1;
        if (h0) atomicAdd(&h0[b0], 1ull);
        if (h1) atomicAdd(&h1[(uint64_t)b0 * f + b1], 1ull);
    }
}

template <int DT>
__global__ void k_bucket_pos(const uint64_t *__restrict__ keys, uint64_t n, int f,
                             const DevModel *M, const unsigned long long *h1, uint32_t *pos) {
    const Root R = load_root(M);
    const double F = (double)f, F2 = (double)f * (double)f, nd = (double)n;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gs) {
        const double p = predict_ldg<DT>(keys[i], R, M->leaf);
        const uint32_t b0 = bucket0(p, F, f), b1 = bucket1(p, F2, f, b0);
        const uint64_t g = (uint64_t)b0 * f + b1;
        const double adj = __ddiv_rn((double)g, F2);
        pos[i] = cs_pos(p, adj, nd, (int)(h1[g] - 1));
    }
}

// -------------------------------------------------------------- launchers --
template <class K>
static void set_smem(K k, size_t bytes) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_count0(const Args &a, int dtype, cudaStream_t st) {
    const size_t sm = sizeof(Count0Smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = a.U0 < 3u * (uint32_t)sms ? a.U0 : 3u * (unsigned)sms;  // persistent, 3 per SM
    if (dtype == DT_F64) { set_smem(k_count0<DT_F64>, sm); k_count0<DT_F64><<<g, 512, sm, st>>>(a); }
    else { set_smem(k_count0<DT_U64>, sm); k_count0<DT_U64><<<g, 512, sm, st>>>(a); }
}
void launch_plan0(const Args &a, uint64_t *dS_B, int reserved, cudaStream_t st) {
    k_plan0<<<1, 1024, 0, st>>>(a, dS_B, reserved);
}
void launch_cap0(const Args &a, uint64_t m, int dtype, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t per = (uint64_t)SH_THREADS * 8;
    const unsigned g = (unsigned)umin64((m + per - 1) / per, 2ull * (uint64_t)sms);
    const size_t sm = sizeof(SampHistSmem);
    if (dtype == DT_F64) { set_smem(k_samp_hist0<DT_F64>, sm); k_samp_hist0<DT_F64><<<g ? g : 1, SH_THREADS, sm, st>>>(a, m); }
    else { set_smem(k_samp_hist0<DT_U64>, sm); k_samp_hist0<DT_U64><<<g ? g : 1, SH_THREADS, sm, st>>>(a, m); }
    k_cap0<<<1, 1024, 0, st>>>(a, m);
}
void launch_scatter0r(const Args &a, int dtype, cudaStream_t st) {
    const size_t sm = sizeof(Scatter0rSmem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t ntiles = (a.n + TP_TILE - 1) / TP_TILE;
    const unsigned g = ntiles < (uint64_t)sms ? (unsigned)ntiles : (unsigned)sms;  // one CTA per SM
    if (dtype == DT_F64) { set_smem(k_scatter0r<DT_F64>, sm); k_scatter0r<DT_F64><<<g, TP_THREADS, sm, st>>>(a); }
    else { set_smem(k_scatter0r<DT_U64>, sm); k_scatter0r<DT_U64><<<g, TP_THREADS, sm, st>>>(a); }
}
void launch_scatter0(const Args &a, int dtype, cudaStream_t st) {
    const size_t sm = sizeof(Scatter0Smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned g = a.U0 < (uint32_t)sms ? a.U0 : (unsigned)sms;  // one CTA per SM (smem-bound)
    if (dtype == DT_F64) { set_smem(k_scatter0<DT_F64>, sm); k_scatter0<DT_F64><<<g, TP_THREADS, sm, st>>>(a); }
    else { set_smem(k_scatter0<DT_U64>, sm); k_scatter0<DT_U64><<<g, TP_THREADS, sm, st>>>(a); }
}
void launch_count1(const Args &a, int dtype, cudaStream_t st) {
    const size_t sm = (size_t)5 * a.L * sizeof(double);
    if (dtype == DT_F64) k_count1<DT_F64><<<a.U1max, 512, 0, st>>>(a);
    else { set_smem(k_count1<DT_U64>, sm); k_count1<DT_U64><<<a.U1max, 512, sm, st>>>(a); }
}
// k_scatter1p below S1P_MAX_N keys, k_scatter1 above (measured at 1M / 10M /
// 100M / 200M / 1B Normal keys: 0.033 / 0.083 / 0.548 / 1.067 / 5.22 ms
// against 0.045 / 0.093 / 0.570 / 1.042 / 4.97 ms). LS_SCATTER1P=0/1 forces one.
static bool scatter1_persistent(uint64_t n) {
    static const int v = [] {
        const char *e = getenv("LS_SCATTER1P");
        return e ? atoi(e) : -1;
    }();
    return v < 0 ? n <= S1P_MAX_N : v != 0;
}
void launch_scatter1(const Args &a, int dtype, cudaStream_t st) {
    if (scatter1_persistent(a.n)) {
        const size_t sm = sizeof(Scatter1pSmem);
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (dtype == DT_F64) { set_smem(k_scatter1p<DT_F64>, sm); k_scatter1p<DT_F64><<<sms, TP_THREADS, sm, st>>>(a); }
        else { set_smem(k_scatter1p<DT_U64>, sm); k_scatter1p<DT_U64><<<sms, TP_THREADS, sm, st>>>(a); }
        return;
    }
    const size_t sm = sizeof(Scatter1Smem);
    if (dtype == DT_F64) { set_smem(k_scatter1<DT_F64, TP_THREADS>, sm); k_scatter1<DT_F64, TP_THREADS><<<a.U1max, TP_THREADS, sm, st>>>(a); }
    else { set_smem(k_scatter1<DT_U64, TP_THREADS>, sm); k_scatter1<DT_U64, TP_THREADS><<<a.U1max, TP_THREADS, sm, st>>>(a); }
}
void launch_classify(const Args &a, uint32_t *dS_B1, cudaStream_t st) {
    (void)dS_B1;
    k_classify<<<a.f, CL_THREADS, 0, st>>>(a);
}
void launch_bucket_ids(const uint64_t *keys, uint64_t n, int f, const DevModel *M, double *p,
                       uint32_t *b0, uint32_t *b1, unsigned long long *h0, unsigned long long *h1,
                       int dtype, cudaStream_t st) {
    int g = (int)umin64((n + 255) / 256, 148 * 16);
    if (g < 1) g = 1;
    if (dtype == DT_F64) k_bucket_ids<DT_F64><<<g, 256, 0, st>>>(keys, n, f, M, p, b0, b1, h0, h1);
    else k_bucket_ids<DT_U64><<<g, 256, 0, st>>>(keys, n, f, M, p, b0, b1, h0, h1);
}
void launch_bucket_pos(const uint64_t *keys, uint64_t n, int f, const DevModel *M,
                       const unsigned long long *h1, uint32_t *pos, int dtype, cudaStream_t st) {
    int g = (int)umin64((n + 255) / 256, 148 * 16);
    if (g < 1) g = 1;
    if (dtype == DT_F64) k_bucket_pos<DT_F64><<<g, 256, 0, st>>>(keys, n, f, M, h1, pos);
    else k_bucket_pos<DT_U64><<<g, 256, 0, st>>>(keys, n, f, M, h1, pos);
}

}  // namespace ls
