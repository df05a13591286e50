// ls_sortsub.cu -- north_star (3)+(4): in-bucket sort with duplicate handling.
//
// SMALL sub-buckets (2 <= n' <= T_small): Alg. 2's model-based counting sort
// in shared memory -- pos per key (R5), histogram K, exclusive
// running totals, placement (R4) -- followed by the touch-up. Because p is
// monotone (R15) the only disorder left after the counting sort is inside runs
// of equal pos ("collision groups"), so the global insertion sort of P:219 is
// replaced by ordering every collision group independently (rank within the
// group). Homogeneous sub-buckets (min == max) are skipped.
//
// BIG sub-buckets (n' > T_small, north_star (3) "high-multiplicity"): the model
// cannot separate their keys, so they take an exact path: MSD
// radix partition on ord(x) - ord(min) (12-bit digits aligned to the key
// range) into the scratch copy, then every piece is sorted in shared memory;
// pieces larger than the shared-memory sort capacity go to the next level.
#include <cooperative_groups.h>

#include "ls_launch.h"
#include "ls_warpsort.cuh"
#include "ls_wstask.cuh"

namespace cg = cooperative_groups;

namespace ls {

template <int DT>
__device__ __forceinline__ void insertion_sort(uint64_t *g, int c) {
    for (int x = 1; x < c; x++) {
        const uint64_t v = g[x];
        const uint64_t o = to_ord<DT>(v);
        int y = x;
        while (y > 0 && to_ord<DT>(g[y - 1]) > o) {
            g[y] = g[y - 1];
            y--;
        }
        g[y] = v;
    }
}

template <int DT>
__device__ __forceinline__ void cmpswap(uint64_t *g, int lo, int hi) {
    const uint64_t x = g[lo], y = g[hi];
    if (to_ord<DT>(x) > to_ord<DT>(y)) {
        g[lo] = y;
        g[hi] = x;
    }
}

// All-ascending bitonic network over next_pow2(c) slots with virtual +inf
// padding beyond c: comparators whose upper index is >= c are already ordered.
// `lanes` threads starting at `lane` cooperate; `sync` is the barrier to use.
template <int DT, bool BLOCK>
__device__ __forceinline__ void bitonic(uint64_t *g, int c, int lane, int lanes) {
    int P = 1, lg = 0;
    while (P < c) { P <<= 1; lg++; }
    const int halfP = P >> 1;
    for (int lk = 1; lk <= lg; lk++) {
        const int k = 1 << lk, lh = lk - 1;
        for (int i = lane; i < halfP; i += lanes) {
            const int blk = i >> lh, p = i & ((1 << lh) - 1);
            const int lo = blk * k + p, hi = blk * k + k - 1 - p;
            if (hi < c) cmpswap<DT>(g, lo, hi);
        }
        if (BLOCK) __syncthreads(); else __syncwarp();
        for (int lj = lk - 2; lj >= 0; lj--) {
            const int j = 1 << lj;
            for (int i = lane; i < halfP; i += lanes) {
                const int blk = i >> lj, p = i & (j - 1);
                const int lo = blk * 2 * j + p, hi = lo + j;
                if (hi < c) cmpswap<DT>(g, lo, hi);
            }
            if (BLOCK) __syncthreads(); else __syncwarp();
        }
    }
}

// Bitonic over an indexable view (same network as bitonic()).
template <class V, bool BLOCK = false>
__device__ __forceinline__ void bitonic_view(V g, int c, int lane, int lanes) {
    int P = 1, lg = 0;
    while (P < c) { P <<= 1; lg++; }
    const int halfP = P >> 1;
    auto cs = [&](int lo, int hi) {
        const uint64_t x = g[lo], y = g[hi];
        if (x > y) { g[lo] = y; g[hi] = x; }
    };
    for (int lk = 1; lk <= lg; lk++) {
        const int k = 1 << lk, lh = lk - 1;
        for (int i = lane; i < halfP; i += lanes) {
            const int blk = i >> lh, p = i & ((1 << lh) - 1);
            const int lo = blk * k + p, hi = blk * k + k - 1 - p;
            if (hi < c) cs(lo, hi);
        }
        if (BLOCK) __syncthreads(); else __syncwarp();
        for (int lj = lk - 2; lj >= 0; lj--) {
            const int j = 1 << lj;
            for (int i = lane; i < halfP; i += lanes) {
                const int blk = i >> lj, p = i & (j - 1);
                const int lo = blk * 2 * j + p, hi = lo + j;
                if (hi < c) cs(lo, hi);
            }
            if (BLOCK) __syncthreads(); else __syncwarp();
        }
    }
}

// ----------------------------------------------------------- SMALL path ----
// Windows: classify assigns every SMALL sub-bucket (2 <= n' <= T_small) to the
// window of T_tile positions its start falls in (T_tile <= T_small), so a
// window's span [lo, hi) -- its first to its last SMALL sub-bucket -- holds at
// most T_tile + T_small - 1 < BS_W keys and only SMALL or single-key
// sub-buckets. k_window_list compacts the non-empty windows.
//
// k_bucketsort is persistent (one 1024-thread CTA per SM) and pulls windows
// from a ticket counter; the next window is staged by the TMA bulk engine
// while the current one is sorted. Per window, one thread per key:
//   slot(key) = start(sub-bucket) + pos(key)   (Alg. 2, R5; adj is
//               precomputed per sub-bucket)    for keys of SMALL sub-buckets,
//   slot(key) = own position                   for single-key sub-buckets;
// K[slot]++ (the rank r comes back from the atomic), one exclusive scan over
// the span gives every sub-bucket's counting-sort placement at once (each
// sub-bucket's slots stay in its own range), keys are placed at K[slot] + r
// (R4). Touch-up (R15): only runs of equal slot
// ("collision groups") can be out of order, so the owner thread of each key
// computes its rank inside its group (groups of <= 8) and the key is written
// to its final position in shared memory; larger groups are sorted by a warp
// (register bitonic <= 32, shared-memory bitonic above; all-equal groups are
// left alone). The sorted span is stored back coalesced, skipping homogeneous
// and single-key sub-buckets, whose keys are already in place.
constexpr int BS_THREADS = 256;
constexpr int BS_KPT = 8;
constexpr int BS_W = BS_THREADS * BS_KPT;  // span capacity (4096 keys)
constexpr int BS_WORDS = BS_W / 32;
constexpr int BS_LOG_W = 11;
static_assert((1 << BS_LOG_W) == BS_W, "BS_LOG_W");
constexpr int BS_CTAS_PER_SM = 4;
constexpr int BS_MAXBIG = 256;             // collision groups > BS_RANKMAX keys per window

struct BsSmem {
    uint64_t ring[2][BS_W + BS_W / 8];      // staged spans; the current one becomes T (padded)
    alignas(16) uint32_t K[BS_W + 4];       // slot histogram -> exclusive running totals
    uint32_t gnp[BS_W];                     // at a head: g | (n' - 1) << 20; after
                                            // placement its storage is slot_of[] (u16):
                                            // the slot of T position q
    uint32_t headbits[BS_WORDS];            // sub-bucket heads (bit per position)
    uint32_t wlast[BS_WORDS];               // 1 + last head position before word w (0: none)
    uint32_t wbits[BS_WORDS];               // positions to store back (non-homogeneous SMALL sub-buckets)
    uint32_t big[BS_MAXBIG];                // slots of collision groups > 8 keys
    uint32_t wsum[33];
    uint32_t nbig, ovf;
    uint4 dq[4];                            // {g0, g1, lo, hi} of windows it .. it+3 (it & 3)
    unsigned long long st_small, st_smallk, st_h1, st_h1k, st_maxg;
    uint64_t mbar[2];
};

// head position of the sub-bucket covering span position q
__device__ __forceinline__ uint32_t head_of(const BsSmem &S, uint32_t q) {
    const uint32_t w = q >> 5;
    const uint32_t bits = S.headbits[w] & (0xffffffffu >> (31u - (q & 31u)));
    return bits ? (w << 5) + 31u - __clz(bits) : S.wlast[w] - 1u;
}

// Stage A[lo, hi) into ring slot `slot` (key k at slot[k - (lo & ~1)]); thread
// 0 only. The bulk copy covers the 16-byte-aligned hull; only if that would run
// past the end of A is the last key loaded directly.
__device__ __forceinline__ void bs_issue(BsSmem &S, int slot, const uint64_t *A, uint32_t lo,
                                         uint32_t hi, uint64_t n) {
    uint64_t *dst = S.ring[slot];
    const uint32_t a0 = lo & ~1u;
    uint32_t a1 = (hi + 1u) & ~1u;
    if (a1 > n) {
        a1 = hi & ~1u;
        dst[hi - 1 - a0] = A[hi - 1];
    }
    const uint32_t bytes = a1 > a0 ? (a1 - a0) * 8u : 0u;
    mbar_expect_tx(&S.mbar[slot], bytes);
    for (uint32_t o = 0; o < bytes; o += 32768u)
        bulk_g2s((char *)dst + o, (const char *)(A + a0) + o, bytes - o < 32768u ? bytes - o : 32768u,
                 &S.mbar[slot]);
}

// Stage window d into `slot` (thread 0); the end of the CTA's window sequence
// (d.x = ~0) is an empty transaction so the wait completes.
__device__ __forceinline__ void bs_stage(BsSmem &S, int slot, const Args &a, uint4 d) {
    if (d.x != BS_NONE) bs_issue(S, slot, a.A, d.z, d.w, a.n);
    else mbar_expect_tx(&S.mbar[slot], 0u);
}
// CTA c sorts windows c, c + G, c + 2G, ... (G = gridDim.x): no ticket on the
// critical path, and the descriptor two windows ahead is loaded early.
__device__ __forceinline__ uint4 bs_desc(const Args &a, uint32_t nwin, uint32_t it) {
    const uint32_t w = blockIdx.x + it * gridDim.x;
    return w < nwin ? a.wlist[w] : make_uint4(BS_NONE, 0u, 0u, 0u);
}

template <int DT>
__global__ void __launch_bounds__(BS_THREADS, BS_CTAS_PER_SM) k_bucketsort(Args a) {
    if (a.ctl->status) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BsSmem &S = *reinterpret_cast<BsSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nwin = min(a.ctl->nwin, a.ntiles);
    if (tid == 0) {
        mbar_init(&S.mbar[0], 1);
        mbar_init(&S.mbar[1], 1);
        S.st_small = S.st_smallk = S.st_h1 = S.st_h1k = S.st_maxg = 0;
        S.dq[0] = bs_desc(a, nwin, 0);
        S.dq[1] = bs_desc(a, nwin, 1);
        bs_stage(S, 0, a, S.dq[0]);
        bs_stage(S, 1, a, S.dq[1]);
    }
    __syncthreads();
    const double rcpF2 = a.rcpF2;
    const Root R = load_root(a.M);
    uint32_t phase = 0;
    uint32_t nx_np = 0, nx_st = 0;
    unsigned long long r_small = 0, r_smallk = 0, r_h1 = 0, r_h1k = 0;  // stats (per thread)
    // debug (LS_DEBUG_STAGE=256): cycles per phase, thread 0 of every CTA
    const bool prof = (a.dbg & 256u) && tid == 0;
    long long t_prev = clock64();
#define BS_PROF(k)                                                                  \
    do {                                                                            \
        if (prof) {                                                                 \
            const long long t_ = clock64();                                         \
            atomicAdd(&a.ctl->prof[k], (unsigned long long)(t_ - t_prev));          \
            t_prev = t_;                                                            \
        }                                                                           \
    } while (0)
    for (uint32_t it = 0;; it++) {
        const int slot = (int)(it & 1u);
        // ---- window tables (overlap with the bulk copy in flight)
        const uint4 desc = S.dq[it & 3u];
        if (desc.x == BS_NONE) break;
        const uint32_t g0 = desc.x, g1 = desc.y, lo = desc.z, hi = desc.w;
        const int span = (int)(hi - lo);
        uint4 ahead;  // descriptor of window it + 2 (thread 0), in flight meanwhile
        if (tid == 0) ahead = bs_desc(a, nwin, it + 2);
        // this window's sub-buckets g0 + tid (prefetched during the previous
        // window) and the next window's, loaded now for the next iteration
        uint32_t my_np = 0, my_st = 0;
        if (it == 0) {
            if (g0 + tid <= g1) {
                my_np = __ldg(&a.hist1[g0 + tid]);
                my_st = __ldg(&a.start1[g0 + tid]);
            }
        } else {
            my_np = nx_np;
            my_st = nx_st;
        }
        {
            const uint4 nd = S.dq[(it + 1) & 3u];
            nx_np = 0;
            nx_st = 0;
            if (nd.x != BS_NONE && nd.x + tid <= nd.y) {
                nx_np = __ldg(&a.hist1[nd.x + tid]);
                nx_st = __ldg(&a.start1[nd.x + tid]);
            }
        }
        {
            uint4 *k4 = reinterpret_cast<uint4 *>(S.K);
            const uint4 z = make_uint4(0, 0, 0, 0);
            for (int i = tid; i < (span + 4) / 4 + 1; i += BS_THREADS) k4[i] = z;
            if (tid < BS_WORDS) S.headbits[tid] = S.wbits[tid] = 0;
            if (tid == 0) S.nbig = S.ovf = 0;
        }
        __syncthreads();
        BS_PROF(0);
        for (uint32_t g = g0 + tid; g <= g1; g += BS_THREADS) {  // the window's sub-buckets
            const bool first = g == g0 + tid;
            const uint32_t np = first ? my_np : __ldg(&a.hist1[g]);
            if (np >= 1) {
                const uint32_t h = (first ? my_st : __ldg(&a.start1[g])) - lo;
                atomicOr(&S.headbits[h >> 5], 1u << (h & 31u));
                S.gnp[h] = g | ((np - 1u) << 20);
            }
        }
        __syncthreads();
        BS_PROF(1);
        if (warp == 0) {  // wlast: exclusive max-scan over the per-word last heads
            uint32_t v[BS_WORDS / 32];
            uint32_t run = 0;
            static_assert(BS_WORDS % 32 == 0, "wlast layout");
#pragma unroll
            for (int k = 0; k < BS_WORDS / 32; k++) {
                const int w = lane * (BS_WORDS / 32) + k;
                const uint32_t b = S.headbits[w];
                v[k] = b ? (uint32_t)(w << 5) + 32u - __clz(b) : 0u;
                run = v[k] > run ? v[k] : run;
            }
            uint32_t ex = __shfl_up_sync(0xffffffffu, warp_incl_max(run), 1);
            if (lane == 0) ex = 0;
#pragma unroll
            for (int k = 0; k < BS_WORDS / 32; k++) {
                S.wlast[lane * (BS_WORDS / 32) + k] = ex;
                ex = v[k] > ex ? v[k] : ex;
            }
        }
        mbar_wait(&S.mbar[slot], (phase >> slot) & 1u);
        __syncthreads();
        BS_PROF(2);
        // ---- counting-sort slots (Alg. 2)
        const uint64_t *keys = S.ring[slot] + (lo & 1u);
        uint64_t key[BS_KPT];
        uint32_t code[BS_KPT];  // slot | r << BS_LOG_W
#pragma unroll
        for (int k = 0; k < BS_KPT; k++) {
            const int i = k * BS_THREADS + tid;
            code[k] = BS_NONE;
            if (i < span) {
                const uint32_t h = head_of(S, (uint32_t)i);
                const uint32_t e = S.gnp[h];
                const uint32_t np = (e >> 20) + 1u;
                key[k] = keys[i];
                uint32_t sl = (uint32_t)i;
                // (keys of a homogeneous level-0 bucket lying inside the span
                // have no head of their own: they stay where they are)
                // (only tiny sub-buckets are sorted here; the others belong
                // to k_warpsort / k_ctasort / k_big and stay in place)
                if (size_class(np, a.T_small) == SC_WINDOW && (uint32_t)i - h < np) {
                    const double p = predict_ldg<DT>(key[k], R, a.M->leaf);
                    const double adj = adj_of(e & 0xfffffu, a.F2, rcpF2);  // (i*f + j)/f^2
                    // (the p-range spread over the n' slots, as in k_ctasort)
                    sl = h + cs_pos(p, adj, __dmul_rn(a.F2, (double)np), (int)(np - 1u));
                }
                // warp-aggregated: keys of equal slot (duplicates!) take one atomic
                const uint32_t peers = __match_any_sync(__activemask(), sl);
                const int leader = __ffs(peers) - 1;
                uint32_t r0 = 0;
                if (lane == leader) r0 = atomicAdd(&S.K[sl], (uint32_t)__popc(peers));
                r0 = __shfl_sync(peers, r0, leader);
                const uint32_t r = r0 + __popc(peers & ((1u << lane) - 1u));
                code[k] = sl | (r << BS_LOG_W);
            }
        }
        if (tid == 0) S.dq[(it + 2) & 3u] = ahead;  // read by all at the top of it + 1
        __syncthreads();
        BS_PROF(3);
        // running totals, exclusive (R4): 8 consecutive entries per
        // thread; collision groups of more than BS_RANKMAX keys are listed here
        static_assert(BS_KPT == 8, "scan layout");
        {
            uint4 *k4 = reinterpret_cast<uint4 *>(S.K) + 2 * tid;
            uint4 x0 = k4[0], x1 = k4[1];
            uint32_t v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
            uint32_t sum = 0, mg = 0;
#pragma unroll
            for (int q = 0; q < 8; q++) {
                // entries past the span hold stale totals of an earlier window
                const uint32_t t = 8 * tid + q < span ? v[q] : 0u;
                mg = t > mg ? t : mg;
                if (t > BS_RANKMAX) {
                    const uint32_t j = atomicAdd(&S.nbig, 1u);
                    if (j < BS_MAXBIG) S.big[j] = 8u * tid + q; else S.ovf = 1;
                }
                v[q] = sum;
                sum += t;
            }
            mg = __reduce_max_sync(0xffffffffu, mg);
            if (lane == 0 && mg > 1u) atomicMax(&S.st_maxg, (unsigned long long)mg);
            const uint32_t incl = warp_incl_scan(sum);
            if (lane == 31) S.wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                const uint32_t w = lane < BS_THREADS / 32 ? S.wsum[lane] : 0u;
                S.wsum[lane] = warp_incl_scan(w) - w;
            }
            __syncthreads();
            const uint32_t off = S.wsum[warp] + incl - sum;
            k4[0] = make_uint4(v[0] + off, v[1] + off, v[2] + off, v[3] + off);
            k4[1] = make_uint4(v[4] + off, v[5] + off, v[6] + off, v[7] + off);
        }
        __syncthreads();
        BS_PROF(4);
        // placement: T = the consumed slot, holding ord values;
        // slot_of[q] remembers the slot of T position q
        const PadT T{S.ring[slot], 0u};
        uint16_t *slot_of = reinterpret_cast<uint16_t *>(S.gnp);
#pragma unroll
        for (int k = 0; k < BS_KPT; k++) {
            if (code[k] != BS_NONE) {
                const uint32_t sl = code[k] & (BS_W - 1u);
                const uint32_t q = S.K[sl] + (code[k] >> BS_LOG_W);
                T[q] = to_ord<DT>(key[k]);
                slot_of[q] = (uint16_t)sl;
            }
        }
        __syncthreads();
        BS_PROF(5);
        // Touch-up per collision group (R15). T is in slot order, so a
        // group is a run of equal slot_of. Each thread owns 8 consecutive
        // positions and runs odd-even transposition rounds that only exchange
        // neighbours of equal slot (neighbouring threads via shuffles) until a
        // round pair swaps nothing in the warp; <= 8 rounds sort every group of
        // <= 8 keys inside a warp's 256 positions. Groups > 8 (listed by the
        // scan) and groups straddling two warps are sorted by a warp below.
        {
            const uint32_t q0 = 8u * tid;
            uint64_t v[8];
            uint32_t sv[8];
            {
                const uint2 s2 = reinterpret_cast<const uint2 *>(slot_of)[2 * tid];
                const uint2 s3 = reinterpret_cast<const uint2 *>(slot_of)[2 * tid + 1];
                const uint32_t sw[4] = {s2.x, s2.y, s3.x, s3.y};
                const uint64_t *row = S.ring[slot] + 9u * tid;  // = &T[q0] (padded)
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const bool in = q0 + q < (uint32_t)span;
                    v[q] = in ? row[q] : ~0ull;
                    sv[q] = in ? ((sw[q >> 1] >> (16 * (q & 1))) & 0xffffu) : 0x10000u + q;
                }
            }
            // pos is monotone in the key (R15): neighbours of different slots
            // are already in order, so the exchange needs no slot test
            auto cx = [](uint64_t &x, uint64_t &y, uint32_t, uint32_t) -> bool {
                return cx_u64(x, y, true) != 0;
            };
            for (int round = 0; round < (int)BS_RANKMAX; round += 2) {
                bool any = false;
                any |= cx(v[0], v[1], sv[0], sv[1]);
                any |= cx(v[2], v[3], sv[2], sv[3]);
                any |= cx(v[4], v[5], sv[4], sv[5]);
                any |= cx(v[6], v[7], sv[6], sv[7]);
                any |= cx(v[1], v[2], sv[1], sv[2]);
                any |= cx(v[3], v[4], sv[3], sv[4]);
                any |= cx(v[5], v[6], sv[5], sv[6]);
                const uint64_t nv = __shfl_down_sync(0xffffffffu, v[0], 1);
                const uint32_t ns = __shfl_down_sync(0xffffffffu, sv[0], 1);
                const uint64_t pv = __shfl_up_sync(0xffffffffu, v[7], 1);
                const uint32_t ps = __shfl_up_sync(0xffffffffu, sv[7], 1);
                (void)ns;
                (void)ps;
                if (lane < 31 && v[7] > nv) { v[7] = nv; any = true; }
                if (lane > 0 && pv > v[0]) { v[0] = pv; any = true; }
                if (!__any_sync(0xffffffffu, any)) break;
            }
            if (q0 < (uint32_t)span) {
                uint64_t *row = S.ring[slot] + 9u * tid;
#pragma unroll
                for (int q = 0; q < 8; q++) row[q] = v[q];
            }
            // a small group straddling two warps' ranges: list it for a warp
            if (lane == 0 && warp > 0 && q0 < (uint32_t)span && sv[0] < 0x10000u &&
                slot_of[q0 - 1] == sv[0]) {
                const uint32_t sl = sv[0], c = S.K[sl + 1] - S.K[sl];
                if (c <= BS_RANKMAX) {
                    const uint32_t j = atomicAdd(&S.nbig, 1u);
                    if (j < BS_MAXBIG) S.big[j] = sl; else S.ovf = 1;
                }
            }
        }
        __syncthreads();
        BS_PROF(6);
        // one warp per listed group: register bitonic (<= 32 / <= 64 keys) or
        // shared-memory bitonic; all-equal groups are left alone
        {
            const uint32_t nb = min(S.nbig, (uint32_t)BS_MAXBIG);
            const uint32_t extra = S.ovf ? (uint32_t)span : 0u;
            for (uint32_t k = warp; k < nb + extra; k += BS_THREADS / 32) {
                uint32_t sl;
                if (k < nb) {
                    sl = S.big[k];
                } else {  // overflow: sort every multi-key group again (rare; idempotent)
                    sl = k - nb;
                    if (S.K[sl + 1] - S.K[sl] < 2u) continue;
                }
                const uint32_t base = S.K[sl], c = S.K[sl + 1] - base;
                if ((a.dbg & 256u) && lane == 0)
                    atomicAdd(&a.ctl->prof[c <= 16 ? 10 : c <= 32 ? 11 : c <= 64 ? 12 : c <= 256 ? 13 : c <= 1024 ? 14 : 15], 1ull);
                if (c <= BS_RANKMAX) {  // a small group straddling two warps: one lane
                    if (lane == 0) {
                        for (uint32_t x = 1; x < c; x++) {
                            const uint64_t t = T[base + x];
                            uint32_t y = x;
                            while (y > 0 && T[base + y - 1] > t) {
                                T[base + y] = T[base + y - 1];
                                y--;
                            }
                            T[base + y] = t;
                        }
                    }
                    continue;
                }
                bool same = true;
                for (uint32_t q = lane; q < c; q += 32) same &= (T[base + q] == T[base]);
                if (__all_sync(0xffffffffu, same)) continue;
                if (c <= 32u) {  // register bitonic across the warp
                    uint64_t v = (uint32_t)lane < c ? T[base + lane] : ~0ull;
                    warp_sort32(v, lane);
                    if ((uint32_t)lane < c) T[base + lane] = v;
                } else if (c <= 64u) {
                    warp_sort_T<2>(T + base, c, lane);
                } else if (c <= 128u) {
                    warp_sort_T<4>(T + base, c, lane);
                } else if (c <= 256u) {
                    warp_sort_T<8>(T + base, c, lane);
                } else {
                    bitonic_view(T + base, (int)c, lane, 32);
                }
            }
        }
        __syncthreads();
        BS_PROF(7);
        // per sub-bucket classification: H1 or counting-sorted; the
        // latter are marked for the store-back
        for (uint32_t g = g0 + tid; g <= g1; g += BS_THREADS) {
            const bool first = g == g0 + tid;
            const uint32_t np = first ? my_np : __ldg(&a.hist1[g]);
            if (size_class(np, a.T_small) != SC_WINDOW) continue;  // other kernels' / single keys
            const uint32_t h = (first ? my_st : __ldg(&a.start1[g])) - lo;
            if (T[h] != T[h + np - 1u]) {  // sorted: homogeneous iff first == last
                r_small++;
                r_smallk += np;
                const uint32_t e = h + np;  // set bits [h, e)
                for (uint32_t w = h >> 5; w <= (e - 1) >> 5; w++) {
                    const uint32_t b0 = w == (h >> 5) ? (h & 31u) : 0u;
                    const uint32_t b1 = w == ((e - 1) >> 5) ? ((e - 1) & 31u) : 31u;
                    const uint32_t m = (0xffffffffu >> (31u - b1)) & (0xffffffffu << b0);
                    atomicOr(&S.wbits[w], m);
                }
            } else {
                if (a.dH1) a.dH1[g] = 1;
                r_h1++;
                r_h1k += np;
            }
        }
        __syncthreads();
        BS_PROF(8);
        // store back (coalesced), skipping keys that are already in place
        for (int q = tid; q < span; q += BS_THREADS)
            if ((S.wbits[q >> 5] >> (q & 31)) & 1u) a.A[lo + q] = from_ord<DT>(T[q]);
        __syncthreads();
        BS_PROF(9);
        phase ^= 1u << slot;
        if (tid == 0) bs_stage(S, slot, a, ahead);
    }
    if (r_small) atomicAdd(&S.st_small, r_small);
    if (r_smallk) atomicAdd(&S.st_smallk, r_smallk);
    if (r_h1) atomicAdd(&S.st_h1, r_h1);
    if (r_h1k) atomicAdd(&S.st_h1k, r_h1k);
    __syncthreads();
    if (tid == 0) {
        if (S.st_small) atomicAdd(&a.ctl->stat[ST_SMALLS], S.st_small);
        if (S.st_smallk) atomicAdd(&a.ctl->stat[ST_SMALLK], S.st_smallk);
        if (S.st_h1) atomicAdd(&a.ctl->stat[ST_H1S], S.st_h1);
        if (S.st_h1k) atomicAdd(&a.ctl->stat[ST_H1K], S.st_h1k);
        if (S.st_maxg) atomicMax(&a.ctl->stat[ST_MAXGRP], S.st_maxg);
    }
}

// ------------------------------------------------------ warp sub-bucket sort --
constexpr uint32_t WS_BATCH = 8;  // warp tasks per ticket
template <int DT>
__global__ void __launch_bounds__(WS_WARPS * 32, WS_CTAS_PER_SM) k_warpsort(Args a) {
    if (a.ctl->status) return;
    __shared__ WsSlice SL[WS_WARPS];
    __shared__ unsigned long long st_red[4];
    __shared__ uint32_t wst[WS_WARPS][4];  // per warp: small / small keys / H1 / H1 keys (off the registers)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WsSlice &W = SL[warp];
    if (threadIdx.x < 4) st_red[threadIdx.x] = 0;
    if (threadIdx.x < 4 * WS_WARPS) (&wst[0][0])[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t ntask = min(a.ctl->ntask, a.task_cap);
    if (blockIdx.x * WS_WARPS >= ntask) return;  // (no task for this block: skip the model reads)
    const Root R = load_root(a.M);
    const uint32_t g_lo = sub_bucket_at(R.xmin, R, a.M->leaf, a.F, a.F2, a.f);
    const uint32_t g_hi = sub_bucket_at(R.xmax, R, a.M->leaf, a.F, a.F2, a.f);
    uint32_t r_maxg = 0;
    bool early_h1 = false;
    // tasks taken in batches of WS_BATCH consecutive ones from a ticket
    // counter (the next batch's ticket in flight during the current one):
    // a warp that started late, or met slower sub-buckets, takes fewer, so
    // every warp finishes within about one batch of the others (the other
    // sorts of the phase run beside this kernel on a second stream)
    uint32_t t0 = 0;
    if (lane == 0) t0 = atomicAdd(&a.ctl->sticket, WS_BATCH);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    while (t0 < ntask) {
        uint32_t tn = 0;
        if (lane == 0) tn = atomicAdd(&a.ctl->sticket, WS_BATCH);
        const uint32_t t1 = min(t0 + WS_BATCH, ntask);
        uint4 nxt = a.tasks[t0];
        for (uint32_t t = t0; t < t1; t++) {
            const uint4 task = nxt;
            if (t + 1 < t1) nxt = a.tasks[t + 1];
            ws_task<DT>(a, R, g_lo, g_hi, W, wst[warp], r_maxg, early_h1, task, lane);
        }
        t0 = __shfl_sync(0xffffffffu, tn, 0);
    }
    if (lane == 0) {
        for (int q = 0; q < 4; q++)
            if (wst[warp][q]) atomicAdd(&st_red[q], (unsigned long long)wst[warp][q]);
        if (r_maxg > 1) atomicMax(&a.ctl->stat[ST_MAXGRP], (unsigned long long)r_maxg);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (st_red[0]) atomicAdd(&a.ctl->stat[ST_SMALLS], st_red[0]);
        if (st_red[1]) atomicAdd(&a.ctl->stat[ST_SMALLK], st_red[1]);
        if (st_red[2]) atomicAdd(&a.ctl->stat[ST_H1S], st_red[2]);
        if (st_red[3]) atomicAdd(&a.ctl->stat[ST_H1K], st_red[3]);
    }
}

// ------------------------------------------------------- CTA sub-bucket sort --
// One CTA per SMALL sub-bucket of WS_MAX+1..CS_MAX keys (at n ~ 10^9 the
// typical sub-bucket holds n/f^2 ~ 1000 keys). Same steps as k_warpsort with
// block barriers: coalesced loads (16 per thread), pos per key (R5),
// counting sort (K in shared memory), placement into padded T, odd-even
// touch-up on 8 consecutive positions per thread (groups straddling two warps
// and groups > 8 are sorted by warps), homogeneity = first == last, store.

template <int CAP>
struct CsSmem {
    uint64_t T[CAP + CAP / 8];
    alignas(16) uint32_t K[CAP + 8];
    uint32_t big[BS_MAXBIG];
    uint32_t wsum[33];
    uint32_t nbig, ovf, mgs;
    uint32_t huge[16], nhuge;       // listed groups of > 256 keys (<= CS_MAX / 257 of them)
    unsigned long long st[5];
};

// CS_THREADS = 256 for 2049..4096 keys (3 CTAs/SM), 128 for 257..2048 (6 CTAs/SM:
// more tasks in flight where a task is short and latency-bound).
template <int DT, int CS_THREADS, int CS_KPT, int CS_CTAS_PER_SM>
__global__ void __launch_bounds__(CS_THREADS, CS_CTAS_PER_SM) k_ctasort(Args a, const uint4 *list,
                                                                     const uint32_t *count) {
    if (a.ctl->status) return;
    constexpr int CAP = CS_THREADS * CS_KPT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CsSmem<CAP> &S = *reinterpret_cast<CsSmem<CAP> *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const PadT T{S.T, 0u};
    const uint32_t ntask = min(*count, a.task_cap);
    if (blockIdx.x >= ntask) return;  // (no task for this block: skip the model reads)
    const Root R = load_root(a.M);
    const uint32_t g_lo = sub_bucket_at(R.xmin, R, a.M->leaf, a.F, a.F2, a.f);
    const uint32_t g_hi = sub_bucket_at(R.xmax, R, a.M->leaf, a.F, a.F2, a.f);
    if (tid < 5) S.st[tid] = 0;
    bool early_h1 = false;  // (block-uniform)
    for (uint32_t t = blockIdx.x; t < ntask; t += gridDim.x) {
        const uint4 task = list[t];
        const uint32_t st = task.x, np = task.y, g = task.z;
        // every per-key loop stops (block-uniform branch) after the
        // kn = ceil(np / CS_THREADS) rows that hold keys
        const int kn = (int)((np + CS_THREADS - 1) / CS_THREADS);
        uint64_t key[CS_KPT];
        uint64_t *const gl = a.A + st + tid;  // key k * CS_THREADS + tid at gl[k * CS_THREADS]
#pragma unroll
        for (int k = 0; k < CS_KPT; k++) {
            key[k] = (uint32_t)(k * CS_THREADS + tid) < np ? gl[k * CS_THREADS] : 0ull;
        }
        // homogeneous sub-bucket (all keys equal): nothing to sort or
        // store. Tested up front only once this CTA has met one (as in the
        // warp sort: the first == last test after the sort catches every
        // case, and on inputs without such sub-buckets the up-front test is a
        // block barrier per task for nothing)
        if (early_h1) {
            const uint64_t k0 = a.A[st];
            bool diff = false;
#pragma unroll
            for (int k = 0; k < CS_KPT; k++) {
                const uint32_t i = (uint32_t)(k * CS_THREADS + tid);
                diff |= (i < np) && key[k] != k0;
            }
            if (!__syncthreads_or(diff)) {
                if (tid == 0) {
                    if (a.dH1) a.dH1[g] = 1;
                    S.st[2] += 1;
                    S.st[3] += np;
                }
                continue;
            }
        }
#pragma unroll
        for (int i = 0; i < CS_KPT / 4; i++)  // K[0..CAP): thread tid owns slots CS_KPT*tid..
            *reinterpret_cast<uint4 *>(&S.K[CS_KPT * tid + 4 * i]) = make_uint4(0, 0, 0, 0);
        if (tid == 0) S.nbig = S.ovf = S.mgs = S.nhuge = 0;
        __syncthreads();
        const double adj = adj_of(g, a.F2, a.rcpF2);  // (i*f + j)/f^2
        const int top = CAP - 1;
        // slots: the sub-bucket's p-range [adj, adj + 1/f^2) spread over the
        // CTA's CAP >= n' counters, pos = floor((p - adj) * f^2 CAP) clamped
        // to [0, CAP-1] (Alg. 2's pos spreads it over n/f^2 slots, P:188-190:
        // a sub-bucket larger than n/f^2 then fills only its first n/f^2
        // slots, and a smaller one piles every key past slot n'-1 into the
        // last slot, R5). Monotone in p, so the counting sort + touch-up give
        // R5's result (reading R-SLOT); the scan below covers CAP slots as
        // CS_KPT per thread, vector loads without bank conflicts.
        const double nsl = __dmul_rn(a.F2, (double)CAP);
        uint32_t code[CS_KPT];
        if (task.w != 0u && g != g_lo && g != g_hi) {
            // one leaf holds every key and p = its line value (k_classify's
            // contained_leaf_warp, as in the warp sort: no routing, no clamp)
            const double *q = a.M->leaf + 5 * (task.w - 1u);
            const double la = __ldg(q), lc = __ldg(q + 1), lb = __ldg(q + 2);
#pragma unroll
            for (int k = 0; k < CS_KPT; k++) {
                code[k] = BS_NONE;
                if ((uint32_t)(k * CS_THREADS + tid) < np) {
                    const double p = __fma_rn(la, __dsub_rn(xd<DT>(key[k]), lc), lb);
                    const uint32_t pos = cs_pos(p, adj, nsl, top);
                    const uint32_t r = atomicAdd(&S.K[pos], 1u);
                    code[k] = pos | (r << 12);
                }
            }
        } else if (g != g_lo && g != g_hi) {  // keys inside [xmin, xmax]: no root clamp
#pragma unroll
            for (int k = 0; k < CS_KPT; k++) {
                code[k] = BS_NONE;
                if ((uint32_t)(k * CS_THREADS + tid) < np) {
                    const double p = predict_ldg_inner<DT>(key[k], R, a.M->leaf);
                    const uint32_t pos = cs_pos(p, adj, nsl, top);
                    const uint32_t r = atomicAdd(&S.K[pos], 1u);
                    code[k] = pos | (r << 12);
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < CS_KPT; k++) {
                code[k] = BS_NONE;
                if ((uint32_t)(k * CS_THREADS + tid) < np) {
                    const double p = predict_ldg<DT>(key[k], R, a.M->leaf);
                    const uint32_t pos = cs_pos(p, adj, nsl, top);
                    const uint32_t r = atomicAdd(&S.K[pos], 1u);
                    code[k] = pos | (r << 12);
                }
            }
        }
        __syncthreads();
        // exclusive running totals over the CAP slots, CS_KPT consecutive
        // slots per thread (16-byte loads and stores); K[CAP] = n'
        {
            uint32_t c[CS_KPT];
#pragma unroll
            for (int i = 0; i < CS_KPT / 4; i++) {
                const uint4 v = *reinterpret_cast<const uint4 *>(&S.K[CS_KPT * tid + 4 * i]);
                c[4 * i] = v.x;
                c[4 * i + 1] = v.y;
                c[4 * i + 2] = v.z;
                c[4 * i + 3] = v.w;
            }
            uint32_t sum = 0, mg = 0, mgs = 0;
#pragma unroll
            for (int q = 0; q < CS_KPT; q++) {
                mg = max(mg, c[q]);
                mgs = (c[q] <= BS_RANKMAX && c[q] > mgs) ? c[q] : mgs;
                sum += c[q];
            }
            if (mg > BS_RANKMAX) {  // (duplicate-heavy inputs) list the groups > 8 keys
#pragma unroll
                for (int q = 0; q < CS_KPT; q++)
                    if (c[q] > BS_RANKMAX) {
                        const uint32_t j = atomicAdd(&S.nbig, 1u);
                        if (j < BS_MAXBIG) S.big[j] = CS_KPT * tid + q; else S.ovf = 1;
                    }
            }
            mg = __reduce_max_sync(0xffffffffu, mg);
            mgs = __reduce_max_sync(0xffffffffu, mgs);
            if (lane == 0 && mg > 1u) atomicMax(&S.st[4], (unsigned long long)mg);
            if (lane == 0 && mgs > 1u) atomicMax(&S.mgs, mgs);
            const uint32_t incl = warp_incl_scan(sum);
            if (lane == 31) S.wsum[warp] = incl;
            __syncthreads();
            if (warp == 0) {
                const uint32_t w = lane < CS_THREADS / 32 ? S.wsum[lane] : 0u;
                S.wsum[lane] = warp_incl_scan(w) - w;
            }
            __syncthreads();
            uint32_t run = S.wsum[warp] + incl - sum;
#pragma unroll
            for (int i = 0; i < CS_KPT / 4; i++) {
                uint4 v;
                v.x = run; run += c[4 * i];
                v.y = run; run += c[4 * i + 1];
                v.z = run; run += c[4 * i + 2];
                v.w = run; run += c[4 * i + 3];
                *reinterpret_cast<uint4 *>(&S.K[CS_KPT * tid + 4 * i]) = v;
            }
            if (tid == 0) S.K[CAP] = np;
        }
        __syncthreads();
        // placement
#pragma unroll
        for (int k = 0; k < CS_KPT; k++) {
            if (code[k] != BS_NONE) {
                const uint32_t pos = code[k] & 0xfffu;
                const uint32_t q = S.K[pos] + (code[k] >> 12);
                T[q] = to_ord<DT>(key[k]);
            }
        }
        __syncthreads();
        // touch-up: odd-even transposition, 16 consecutive positions per
        // thread as two rows of 8 (the second only if np > 2048). pos is
        // monotone in the key (R15), so neighbours of different slots are in
        // order already and never swap; groups of <= mgs keys need mgs rounds
        // (2 per pass), and a clean first pass ends it (duplicates).
        const int iters = (int)((S.mgs + 1u) >> 1);
        for (int half = 0; half < (CS_KPT > 8 && np > 8u * CS_THREADS ? 2 : 1); half++) {
            const uint32_t row_i = (uint32_t)(half * CS_THREADS + tid);  // row of 8 positions
            const uint32_t q0 = 8u * row_i;
            if (iters > 0) {
                uint64_t v[8];
                {
                    const uint64_t *row = S.T + 9u * row_i;
#pragma unroll
                    for (int q = 0; q < 8; q++) v[q] = q0 + q < np ? row[q] : ~0ull;
                }
                auto pass = [&](bool track) -> bool {
                    uint32_t moved = 0;
#pragma unroll
                    for (int q = 0; q < 8; q += 2) moved |= cx_u64(v[q], v[q + 1], track);
#pragma unroll
                    for (int q = 1; q < 7; q += 2) moved |= cx_u64(v[q], v[q + 1], track);
                    const uint64_t nv = __shfl_down_sync(0xffffffffu, v[0], 1);
                    const uint64_t pv = __shfl_up_sync(0xffffffffu, v[7], 1);
                    if (lane < 31 && v[7] > nv) { v[7] = nv; moved = 1; }
                    if (lane > 0 && pv > v[0]) { v[0] = pv; moved = 1; }
                    return moved != 0;
                };
                if (iters > 0) {
                    // (every pass votes: duplicate-heavy sub-buckets, the
                    // usual CTA case, mostly converge early)
                    for (int it2 = 0; it2 < iters; it2++)
                        if (!__any_sync(0xffffffffu, pass(true))) break;
                    if (q0 < np) {
                        uint64_t *row = S.T + 9u * row_i;
#pragma unroll
                        for (int q = 0; q < 8; q++) row[q] = v[q];
                    }
                }
            }
            // a small group straddling two warps' 256-position ranges: the
            // group holding position q0 (the last slot sl with K[sl] <= q0,
            // by bisection over the totals) starts before q0
            uint32_t sl = 0;
            if (lane == 0 && row_i > 0 && q0 < np) {
                uint32_t lo = 0, n = CAP;  // K[0] = 0 <= q0; K[CAP] = n' > q0
                while (n > 1) {
                    const uint32_t h = n >> 1;
                    if (S.K[lo + h] <= q0) { lo += h; n -= h; } else { n = h; }
                }
                sl = lo;
            }
            if (lane == 0 && row_i > 0 && q0 < np && S.K[sl] < q0) {
                const uint32_t c = S.K[sl + 1] - S.K[sl];
                if (c <= BS_RANKMAX) {
                    const uint32_t j = atomicAdd(&S.nbig, 1u);
                    if (j < BS_MAXBIG) S.big[j] = sl; else S.ovf = 1;
                }
            }
        }
        __syncthreads();
        // listed groups: one warp each
        {
            const uint32_t nb = min(S.nbig, (uint32_t)BS_MAXBIG);
            const uint32_t extra = S.ovf ? (uint32_t)CAP : 0u;
            for (uint32_t k = warp; k < nb + extra; k += CS_THREADS / 32) {
                uint32_t sl;
                if (k < nb) {
                    sl = S.big[k];
                } else {  // overflow: sort every multi-key group again (rare; idempotent)
                    sl = k - nb;
                    if (S.K[sl + 1] - S.K[sl] < 2u) continue;
                }
                const uint32_t base = S.K[sl], c = S.K[sl + 1] - base;
                if (c > 256u && k < nb) {  // the whole CTA sorts it below
                    if (lane == 0) S.huge[atomicAdd(&S.nhuge, 1u)] = sl;
                    continue;
                }
                if (c <= BS_RANKMAX) {
                    if (lane == 0) {
                        for (uint32_t x = 1; x < c; x++) {
                            const uint64_t tt = T[base + x];
                            uint32_t y = x;
                            while (y > 0 && T[base + y - 1] > tt) {
                                T[base + y] = T[base + y - 1];
                                y--;
                            }
                            T[base + y] = tt;
                        }
                    }
                    continue;
                }
                bool same = true;  // one value (duplicate-heavy inputs): nothing to do
                for (uint32_t q = lane; q < c; q += 32) same &= (T[base + q] == T[base]);
                if (__all_sync(0xffffffffu, same)) continue;
                if (c <= 32u) {
                    uint64_t v1 = (uint32_t)lane < c ? T[base + lane] : ~0ull;
                    warp_sort32(v1, lane);
                    if ((uint32_t)lane < c) T[base + lane] = v1;
                } else if (c <= 64u) {
                    warp_sort_T<2>(T + base, c, lane);
                } else if (c <= 128u) {
                    warp_sort_T<4>(T + base, c, lane);
                } else if (c <= 256u) {
                    warp_sort_T<8>(T + base, c, lane);
                } else {
                    bitonic_view(T + base, (int)c, lane, 32);
                }
            }
            __syncthreads();
            // listed groups of > 256 keys (duplicate-heavy inputs): shared-
            // memory bitonic by all threads, one group at a time
            const uint32_t nh = S.nhuge;
            for (uint32_t k = 0; k < nh; k++) {
                const uint32_t sl = S.huge[k];
                const uint32_t base = S.K[sl], c = S.K[sl + 1] - base;
                bool diff = false;  // one value: nothing to do
                for (uint32_t q = tid; q < c; q += CS_THREADS) diff |= (T[base + q] != T[base]);
                if (!__syncthreads_or(diff)) continue;
                bitonic_view<PadT, true>(T + base, (int)c, tid, CS_THREADS);
            }
        }
        __syncthreads();
        // homogeneous iff first == last of the sorted sub-bucket
        const bool homog = T[0] == T[np - 1u];
        early_h1 |= homog;
        if (!homog) {
            // T[k * CS_THREADS + tid] at tl[k * CS_THREADS * 9 / 8] (CS_THREADS % 8 == 0)
            const uint64_t *tl = S.T + tid + (tid >> 3);
#pragma unroll
            for (int k = 0; k < CS_KPT; k++) {
                if ((uint32_t)(k * CS_THREADS + tid) < np) gl[k * CS_THREADS] = from_ord<DT>(tl[k * CS_THREADS * 9 / 8]);
            }
        }
        if (tid == 0) {
            if (!homog) {
                S.st[0] += 1;
                S.st[1] += np;
            } else {
                if (a.dH1) a.dH1[g] = 1;
                S.st[2] += 1;
                S.st[3] += np;
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (S.st[0]) atomicAdd(&a.ctl->stat[ST_SMALLS], S.st[0]);
        if (S.st[1]) atomicAdd(&a.ctl->stat[ST_SMALLK], S.st[1]);
        if (S.st[2]) atomicAdd(&a.ctl->stat[ST_H1S], S.st[2]);
        if (S.st[3]) atomicAdd(&a.ctl->stat[ST_H1K], S.st[3]);
        if (S.st[4]) atomicMax(&a.ctl->stat[ST_MAXGRP], S.st[4]);
    }
}

// Compact the non-empty windows into wlist: {g0, g1, lo, hi}.
__global__ void k_window_list(Args a) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint4 d = make_uint4(BS_NONE, 0u, 0u, 0u);
    if (t < a.ntiles) {
        const uint32_t g0 = a.tile_first[t];
        if (g0 != BS_NONE) {
            const uint32_t g1 = a.tile_last[t];
            d = make_uint4(g0, g1, a.start1[g0], a.start1[g1] + a.hist1[g1]);
        }
    }
    const bool has = d.x != BS_NONE;
    const uint32_t m = __ballot_sync(0xffffffffu, has);
    uint32_t base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(&a.ctl->nwin, (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (has) a.wlist[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = d;
}

// ------------------------------------------------------------- BIG path ----
constexpr int BIG_THREADS = 1024;     // one CTA per SM: an item finishes twice as fast (shorter critical path)
constexpr int BIG_DIGITS = 4096;       // 12-bit MSD digits
constexpr int BIG_SORT_CAP = 8192;     // keys sorted in shared memory by one CTA
constexpr int BIG_CHUNK = BIG_SORT_CAP / 2;
constexpr int BIG_MAXWIN = 1024;       // windows classified per round
constexpr int BIG_MAXBLK = 64;         // pieces in (BIG_CHUNK, BIG_SORT_CAP] per item
constexpr int BIG_MAXWBIG = 16;        // pieces of 257..BIG_CHUNK keys per window (CTA-sorted)
constexpr int BIG_DENSE_MAX = 49152;   // slots of the counting sort by value (16-bit counters alias sk..end)
constexpr int BIG_DENSE_WIN = 4;       // windows of BIG_DENSE_MAX slots (one pass over the item each)

// The dense test of a non-homogeneous big item (mn != mx, so dif != 0):
// every key is mn + s * 2^tz with s < nsl (tz = the low bits all keys share).
__device__ __forceinline__ bool big_is_dense(uint32_t size, unsigned long long mn,
                                             unsigned long long mx, unsigned long long dif,
                                             int &tz, uint32_t &nsl) {
    tz = dif ? __ffsll((long long)dif) - 1 : 32;  // (k_big_minmax ORs 32-bit differences: 0 -> >= 32 shared bits)
    tz = min(tz, 32);
    const unsigned long long s = ((mx - mn) >> tz) + 1ull;
    nsl = (uint32_t)min(s, 0xffffffffull);
    return size > (uint32_t)BIG_SORT_CAP && s <= (unsigned long long)BIG_DENSE_MAX * BIG_DENSE_WIN;
}


// ord min/max of level-0 big items, one 64K-key chunk per work entry
// (classify wrote the chunk list), so a multi-million-key homogeneous
// sub-bucket (Zipf's top value, config 4's top level) is scanned by the whole
// GPU instead of one CTA.
template <int DT>
__global__ void __launch_bounds__(512, 3) k_big_minmax(Args a) {
    if (a.ctl->status) return;
    __shared__ unsigned long long red[64];
    __shared__ uint32_t redd[32];
    const uint32_t nch = min(a.ctl->nchunks, a.chunk_cap);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t bd = blockDim.x;
    for (uint32_t e = blockIdx.x; e < nch; e += gridDim.x) {
        const BigChunk ch = a.chunks[e];
        const BigItem item = a.big[ch.item];
        const uint32_t beg = ch.chunk * MM_CHUNK, end = min(item.size, beg + MM_CHUNK);
        const uint64_t *X = a.A + item.off;
        // dif: OR of the low 32 bits of ord ^ ord(first key): its trailing
        // zeros (32 if none) are low bits every key shares (the dense path's
        // value stride)
        const uint32_t ref = (uint32_t)to_ord<DT>(X[0]);
        uint32_t dif = 0;
        unsigned long long mn = ~0ull, mx = 0;
        uint32_t i = beg + threadIdx.x;
        for (; i + 7 * bd < end; i += 8 * bd) {  // full rounds: 8 independent loads in flight
            uint64_t v[8];
#pragma unroll
            for (int q = 0; q < 8; q++) v[q] = X[i + q * bd];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                const unsigned long long o = to_ord<DT>(v[q]);
                mn = o < mn ? o : mn;
                mx = o > mx ? o : mx;
                dif |= (uint32_t)o ^ ref;
            }
        }
        for (; i < end; i += bd) {
            const unsigned long long o = to_ord<DT>(X[i]);
            mn = o < mn ? o : mn;
            mx = o > mx ? o : mx;
            dif |= (uint32_t)o ^ ref;
        }
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        dif = __reduce_or_sync(0xffffffffu, dif);
        if ((threadIdx.x & 31) == 0) {
            red[w] = mn;
            red[32 + w] = mx;
            redd[w] = dif;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < nw; k++) {
                mn = red[k] < mn ? red[k] : mn;
                mx = red[32 + k] > mx ? red[32 + k] : mx;
                dif |= redd[k];
            }
            atomicMin(&a.big[ch.item].mn, mn);
            atomicMax(&a.big[ch.item].mx, mx);
            if (dif) atomicOr(&a.big[ch.item].dif, (unsigned long long)dif);
        }
        __syncthreads();
    }
}

// k_big's first pass takes the level-0 big items AND the level-1 items the
// large path (ls_bigpath.cu, run before k_big) has already listed, in
// decreasing estimated cost (one CTA; a counting sort on quarter-octaves of
// the cost): the CTAs then finish together instead of waiting at the grid
// barrier behind a late radix item, and the large path's ~100K-key pieces no
// longer wait for a second pass of their own (config 4: ~500 dense + ~580
// radix items of ~100K keys, 296 CTAs). Entry = level-0 index, or
// 0x80000000 | level-1 index.
static_assert(sizeof(BigItem) == 48, "BigItem is read as three 16-byte words");
constexpr int BO_CLASSES = 256;
__global__ void __launch_bounds__(1024) k_big_order(Args a) {
    if (a.ctl->status) return;
    __shared__ uint32_t h[BO_CLASSES];
    __shared__ uint32_t tmp[36];
    __shared__ unsigned long long st[5];  // H1 sub-buckets / keys, big / big keys / passes of the skipped items
    const uint32_t cnt0 = min(a.ctl->big_cnt[0], a.big_cap);
    const uint32_t pre1 = min(a.ctl->big_cnt[1], a.big_cap);
    const uint32_t cnt = cnt0 + pre1;
    for (int c = threadIdx.x; c < BO_CLASSES; c += blockDim.x) h[c] = 0;
    if (threadIdx.x < 5) st[threadIdx.x] = 0;
    __syncthreads();
    // homogeneous level-0 items (final as they are) and large ones
    // (ls_bigpath.cu) get no ticket: their statistics are counted here
    {
        uint32_t hs = 0, ls_ = 0;
        unsigned long long hk = 0, lk = 0;
        for (uint32_t i = threadIdx.x; i < cnt0; i += blockDim.x) {
            const BigItem it = a.big[i];
            if (it.mn == it.mx) {
                if (a.dH1) a.dH1[it.g] = 1;
                hs++;
                hk += it.size;
            } else if (it.pad0) {
                ls_++;
                lk += it.size;
            }
        }
        // (warp sums first: one shared-memory atomic per warp, not per item)
        hs = __reduce_add_sync(0xffffffffu, hs);
        ls_ = __reduce_add_sync(0xffffffffu, ls_);
        hk = warp_sum_u64(hk);
        lk = warp_sum_u64(lk);
        if ((threadIdx.x & 31) == 0) {
            if (hs) { atomicAdd(&st[0], (unsigned long long)hs); atomicAdd(&st[1], hk); }
            if (ls_) { atomicAdd(&st[2], (unsigned long long)ls_); atomicAdd(&st[3], lk); }
        }
    }
    auto cls = [&](uint32_t i) -> uint32_t {
        double cost;
        if (i < cnt0) {
            const BigItem it = a.big[i];
            if (it.mn == it.mx || it.pad0) return BO_CLASSES - 1;  // homogeneous / large path: no ticket
            int tz;
            uint32_t nsl;
            const uint32_t w = big_is_dense(it.size, it.mn, it.mx, it.dif, tz, nsl)
                                   ? (nsl + BIG_DENSE_MAX - 1) / BIG_DENSE_MAX  // one pass per window
                                   : it.size <= (uint32_t)BIG_SORT_CAP ? 2u : 5u;
            cost = (double)it.size * (double)w;
        } else {  // level-1 item: min/max pass + radix
            cost = (double)a.big[(size_t)a.big_cap + (i - cnt0)].size * 5.0;
        }
        const int q = (int)(__log2f((float)cost) * 4.0f);  // quarter octaves, 0..~150
        return (uint32_t)max(0, BO_CLASSES - 2 - q);
    };
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) atomicAdd(&h[cls(i)], 1u);
    __syncthreads();
    const uint32_t nskip = h[BO_CLASSES - 1];
    block_exscan(h, BO_CLASSES, tmp);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const uint32_t c = cls(i);
        if (c != BO_CLASSES - 1) a.border[atomicAdd(&h[c], 1u)] = i < cnt0 ? i : 0x80000000u | (i - cnt0);
    }
    if (threadIdx.x == 0) {
        if (st[0]) atomicAdd(&a.ctl->stat[ST_H1S], st[0]);
        if (st[1]) atomicAdd(&a.ctl->stat[ST_H1K], st[1]);
        if (st[2]) {
            atomicAdd(&a.ctl->stat[ST_BIGS], st[2]);
            atomicAdd(&a.ctl->stat[ST_BIGK], st[3]);
            atomicAdd(&a.ctl->stat[ST_BIGPASS], st[2]);
        }
        a.ctl->big_lv0 = cnt - nskip;
        a.ctl->big_next[1] = pre1;  // (consumed by the first pass's dynamic phase after them)
        a.ctl->big_pub1 = pre1;
        a.ctl->big_done0 = 0;
    }
}

template <int DT>
__device__ void big_minmax(const uint64_t *X, uint32_t size, unsigned long long &mn,
                           unsigned long long &mx, unsigned long long &dif, unsigned long long *red) {
    mn = ~0ull;
    mx = 0;
    dif = 0;
    const unsigned long long ref = to_ord<DT>(X[0]);
    for (uint32_t i = threadIdx.x; i < size; i += 4 * blockDim.x) {
        uint64_t v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = (i + q * blockDim.x < size) ? X[i + q * blockDim.x] : X[0];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const unsigned long long o = to_ord<DT>(v[q]);
            mn = o < mn ? o : mn;
            mx = o > mx ? o : mx;
            dif |= o ^ ref;
        }
    }
    mn = warp_min_u64(mn);
    mx = warp_max_u64(mx);
    dif = warp_or_u64(dif);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[w] = mn;
        red[32 + w] = mx;
        red[64 + w] = dif;
    }
    __syncthreads();
    mn = red[0];
    mx = red[32];
    dif = red[64];
    for (int i = 1; i < nw; i++) {
        mn = red[i] < mn ? red[i] : mn;
        mx = red[32 + i] > mx ? red[32 + i] : mx;
        dif |= red[64 + i];
    }
    __syncthreads();
}

static_assert(sizeof(BsSmem) * BS_CTAS_PER_SM <= 228 * 1024, "bucket sort shared memory per SM");

struct BigSmem {
    uint64_t sk[BIG_SORT_CAP + 2];          // (+2: aligned hull of a TMA-staged window)
    uint32_t start[BIG_DIGITS], end[BIG_DIGITS];  // (sk..end: the dense path's 16-bit counters)
    uint64_t mbar;
    uint32_t wlo[BIG_MAXWIN], whi[BIG_MAXWIN];
    uint32_t blk[BIG_MAXBLK];
    uint32_t wbig[BIG_MAXWBIG];             // window pieces of 257..BIG_CHUNK keys
    uint32_t tmp[36];
    uint32_t item, nblk, nwbig;
    unsigned long long red[96];
};

static_assert((BIG_SORT_CAP + 2) * 8 + 2 * BIG_DIGITS * 4 >= BIG_DENSE_MAX * 2, "dense counters fit sk..end");
static_assert(2 * BIG_MAXWIN >= BIG_DENSE_MAX / 32, "dense chunk totals fit wlo..whi");

// Counting sort by value of one big item whose keys are mn + s * 2^tz,
// s < nsl <= BIG_DENSE_MAX: 16-bit slot counters (two per 32-bit word,
// aliasing S.sk .. S.end), an exclusive scan, then every slot's value written
// count times at its place. A slot with >= 2^16 keys would wrap its counter
// and carry into (or past) its neighbour; every such wrap lowers the counter
// total, so total == size proves there was none -- otherwise nothing has been
// written and the caller sorts the item by radix (returns false). Ends with a
// block barrier.
template <int DT>
__device__ __noinline__ bool big_dense(const uint64_t *__restrict__ X, uint64_t *__restrict__ out,
                                       uint64_t *__restrict__ scratch, uint32_t size,
                                       unsigned long long mn, int tz, uint32_t nsl, BigSmem &S,
                                       unsigned long long *prof) {
    uint32_t *cw = reinterpret_cast<uint32_t *>(S.sk);
    const uint16_t *cnt = reinterpret_cast<const uint16_t *>(S.sk);
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;
    // more than one window of slots: X is read once per window, so when X is
    // `out` the runs go to the item's scratch range (which is not X) and are
    // copied to `out` at the end
    const bool multi = nsl > (uint32_t)BIG_DENSE_MAX && X == out;  // (X != out: write out directly)
    uint64_t *dst = multi ? scratch : out;
    uint32_t obase = 0;
    long long t0 = clock64();
    for (uint32_t wb = 0; wb < nsl; wb += BIG_DENSE_MAX) {
        const uint32_t wn = min((uint32_t)BIG_DENSE_MAX, nsl - wb);
        for (uint32_t w = tid; w < (wn + 1) / 2; w += bd) cw[w] = 0;
        __syncthreads();
        uint32_t inw = 0;  // keys of this window seen by this thread
        for (uint32_t i = tid; i < size; i += 8 * bd) {
            uint64_t v[8];
#pragma unroll
            for (int q = 0; q < 8; q++) v[q] = (i + q * bd < size) ? X[i + q * bd] : 0;
#pragma unroll
            for (int q = 0; q < 8; q++)
                if (i + q * bd < size) {
                    const uint32_t s = (uint32_t)((to_ord<DT>(v[q]) - mn) >> tz) - wb;
                    if (s < wn) {
                        atomicAdd(&cw[s >> 1], 1u << ((s & 1u) * 16u));
                        inw++;
                    }
                }
        }
        inw = __reduce_add_sync(0xffffffffu, inw);
        if (lane == 0) S.tmp[warp] = inw;
        __syncthreads();
        uint32_t want = 0;
        for (int w = 0; w < nwarps; w++) want += S.tmp[w];
        if (prof && tid == 0) { const long long t = clock64(); atomicAdd(&prof[6], (unsigned long long)(t - t0)); t0 = t; }
        // chunks of 32 slots, dealt round-robin to the warps (a Gaussian
        // cluster puts most keys in the middle chunks): chunk totals, their
        // exclusive scan (in S.wlo, free here), then each chunk's runs
        uint32_t *ctot = S.wlo;  // (wlo, whi: adjacent)
        const uint32_t nch = (wn + 31) / 32;
        for (uint32_t c = (uint32_t)warp; c < nch; c += (uint32_t)nwarps) {
            const uint32_t k = 32 * c + (uint32_t)lane;
            const uint32_t t = __reduce_add_sync(0xffffffffu, k < wn ? (uint32_t)cnt[k] : 0u);
            if (lane == 0) ctot[c] = t;
        }
        __syncthreads();
        const uint32_t all = block_exscan(ctot, (int)nch, S.tmp);
        __syncthreads();
        if (all != want) return false;  // a counter wrapped: radix instead (uniform decision; out untouched)
        for (uint32_t c = (uint32_t)warp; c < nch; c += (uint32_t)nwarps) {
            const uint32_t s = 32 * c, k = s + (uint32_t)lane;
            const uint32_t cc = k < wn ? cnt[k] : 0u;
            const uint32_t incl = warp_incl_scan(cc);
            const uint32_t rel = incl - cc;  // run start relative to the chunk's first key
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            const uint32_t carry = obase + ctot[c];
            // the 32 slots' runs are contiguous: output position p belongs to
            // the last slot j with rel_j <= p (an empty slot shares its start
            // with the next non-empty one, which is later) -- a 5-step search
            for (uint32_t p0 = 0; p0 < total; p0 += 128) {  // (4 independent searches in flight)
                uint32_t p[4], j[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    p[u] = p0 + 32u * u + (uint32_t)lane;
                    j[u] = 0;
                }
#pragma unroll
                for (int b = 16; b > 0; b >>= 1)
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const uint32_t r = __shfl_sync(0xffffffffu, rel, j[u] + b);
                        j[u] = r <= p[u] ? j[u] + b : j[u];
                    }
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (p[u] < total)
                        dst[carry + p[u]] = from_ord<DT>(mn + ((unsigned long long)(wb + s + j[u]) << tz));
            }
        }
        obase += want;
        __syncthreads();  // (the counters alias S.sk: the next window / item reuses it)
    }
    if (multi)
        for (uint32_t i = tid; i < size; i += bd) out[i] = dst[i];
    __syncthreads();
    if (prof && tid == 0) atomicAdd(&prof[9], (unsigned long long)(clock64() - t0));
    return true;
}

// One CTA per big item of this level: MSD radix partition X -> Y on the top
// 12 bits of ord - min, then every piece is sorted exactly in shared memory
// and written to A. Pieces <= BIG_CHUNK are gathered in windows of
// BIG_CHUNK positions (a window owns the pieces starting in it, so its span
// is <= BIG_SORT_CAP): one thread per piece of <= 16 keys (insertion sort),
// one warp per larger piece (bitonic). Pieces in (BIG_CHUNK, BIG_SORT_CAP]
// are block-sorted; larger ones become items of the next level.
template <int DT>
__device__ __forceinline__ void big_level(const Args &a, int level, BigSmem &S, uint32_t &mphase) {
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;
    const uint32_t cnt = level == 0 ? a.ctl->big_lv0 : min(*(volatile uint32_t *)&a.ctl->big_cnt[level], a.big_cap);
    const bool prof = (a.dbg & 512u) && threadIdx.x == 0;
    long long t_prev = clock64();
#define BG_PROF(k)                                                                  \
    do {                                                                            \
        if (prof) {                                                                 \
            const long long t_ = clock64();                                         \
            atomicAdd(&a.ctl->prof[k], (unsigned long long)(t_ - t_prev));          \
            t_prev = t_;                                                            \
        }                                                                           \
    } while (0)
    long long t_it = 0;
    uint32_t sz_it = 0;
    auto rec_item = [&]() {  // (profiling: the previous item's duration, packed with its size)
        if (prof && sz_it) {
            const unsigned long long dur = (unsigned long long)(clock64() - t_it);
            atomicMax(&a.ctl->prof[5], (dur << 32) | sz_it);
        }
    };
    // First pass (level 0): the first-pass tickets (k_big_order's list), then
    // the level-1 items those items create, as soon as they are published
    // (in order, big_pub1) -- no grid barrier between the two, so the pieces
    // of a multi-cluster sub-bucket do not wait for the slowest CTA. Level 1
    // is complete once every first-pass ticket is done (big_done0 == cnt).
    bool dyn = false, counted = true;
    constexpr uint32_t BI_END = 0xffffffffu, BI_DYN = 0x80000000u;
    for (;;) {
        BG_PROF(10);
        rec_item();
        if (tid == 0) {
            if (!counted) {  // the previous first-pass ticket is done (its appends are published)
                __threadfence();
                atomicAdd(&a.ctl->big_done0, 1u);
                counted = true;
            }
            uint32_t code = BI_END;
            if (level != 0) {
                const uint32_t t = atomicAdd(&a.ctl->big_next[level], 1u);
                code = t < cnt ? t : BI_END;
            } else {
                if (!dyn) {
                    const uint32_t t = atomicAdd(&a.ctl->big_next[0], 1u);
                    if (t < cnt) {
                        code = t;
                        counted = false;
                    } else {
                        dyn = true;
                    }
                }
                if (dyn) {
                    const uint32_t t = atomicAdd(&a.ctl->big_next[1], 1u);
                    for (;;) {
                        if (t < *(volatile uint32_t *)&a.ctl->big_pub1) { code = BI_DYN | t; break; }
                        if (*(volatile uint32_t *)&a.ctl->big_done0 == cnt) {
                            __threadfence();
                            code = t < *(volatile uint32_t *)&a.ctl->big_pub1 ? (BI_DYN | t) : BI_END;
                            break;
                        }
                        __nanosleep(256);
                    }
                }
            }
            S.item = code;
        }
        __syncthreads();
        const uint32_t it = S.item;
        __syncthreads();
        if (it == BI_END) break;
        int lv = level;  // the item's own level (the first pass mixes levels 0 and 1)
        uint32_t ix = it;
        if (level == 0) {
            if (it & BI_DYN) {
                lv = 1;
                ix = it & ~BI_DYN;
            } else {
                ix = a.border[it];
                lv = ix >> 31;
                ix &= 0x7fffffffu;
            }
        }
        if (lv != 0 && ix >= a.big_cap) {  // (a list overflow: status is set)
            __syncthreads();
            continue;
        }
        BigItem item;
        {  // (published by another SM during this kernel: read through L2)
            const BigItem *src = a.big + (size_t)lv * a.big_cap + ix;
            const uint4 w0 = __ldcg(reinterpret_cast<const uint4 *>(src));
            const uint4 w1 = __ldcg(reinterpret_cast<const uint4 *>(src) + 1);
            const uint4 w2 = __ldcg(reinterpret_cast<const uint4 *>(src) + 2);
            const uint4 ww[3] = {w0, w1, w2};
            memcpy(&item, ww, sizeof item);
        }
        t_it = clock64();
        sz_it = item.size;
        const uint64_t *X = (item.in_b ? a.B : a.A) + item.off;
        uint64_t *Y = (item.in_b ? a.A : a.B) + item.off;
        uint64_t *Aout = a.A + item.off;
        unsigned long long mn, mx, dif;
        if (lv == 0) {
            mn = item.mn;
            mx = item.mx;
            dif = item.dif;
        } else {
            big_minmax<DT>(X, item.size, mn, mx, dif, S.red);
        }
        if (mn == mx) {  // homogeneous: already final
            if (item.in_b)
                for (uint32_t i = tid; i < item.size; i += bd) Aout[i] = X[i];
            if (tid == 0 && lv == 0) {
                if (a.dH1) a.dH1[item.g] = 1;
                atomicAdd(&a.ctl->stat[ST_H1S], 1ull);
                atomicAdd(&a.ctl->stat[ST_H1K], (unsigned long long)item.size);
            }
            __syncthreads();
            continue;
        }
        if (tid == 0) {
            if (lv == 0) {
                atomicAdd(&a.ctl->stat[ST_BIGS], 1ull);
                atomicAdd(&a.ctl->stat[ST_BIGK], (unsigned long long)item.size);
            }
            atomicAdd(&a.ctl->stat[ST_BIGPASS], 1ull);
        }
        if (lv == 0 && item.pad0) {  // large: sorted by ls_bigpath.cu
            __syncthreads();
            continue;
        }
        // dense values: every key is mn + s * 2^tz with s < nslot (tz = the low
        // bits all keys share). A counting sort BY VALUE is then exact: count
        // the slots, scan, write every slot's value count times (16 B/key, no
        // key moves; config 4's ID clusters: ~8K values in ~100K keys)
        {
            int tz;
            uint32_t nsl;
            if (big_is_dense(item.size, mn, mx, dif, tz, nsl)) {
                BG_PROF(15);
                const bool ok = big_dense<DT>(X, Aout, a.B + item.off, item.size, mn, tz, nsl, S,
                                              prof ? a.ctl->prof : nullptr);
                BG_PROF(12);
                if (ok) {
                    if (prof) atomicAdd(&a.ctl->prof[13], 1ull);
                    continue;
                }
            }
            if (prof) atomicAdd(&a.ctl->prof[14], 1ull);
        }
        if (item.size <= BIG_SORT_CAP) {
            for (uint32_t i = tid; i < item.size; i += bd) S.sk[i] = X[i];
            __syncthreads();
            bitonic<DT, true>(S.sk, (int)item.size, tid, bd);
            for (uint32_t i = tid; i < item.size; i += bd) Aout[i] = S.sk[i];
            __syncthreads();
            continue;
        }
        BG_PROF(0);
        // MSD radix partition X -> Y on the top 12 bits of ord - mn
        const unsigned long long range = mx - mn;
        const int bits = 64 - __clzll((long long)range);
        const int shift = bits > 12 ? bits - 12 : 0;
        for (int d = tid; d < BIG_DIGITS; d += bd) S.start[d] = 0;
        if (tid == 0) S.nblk = S.nwbig = 0;
        __syncthreads();
        for (uint32_t i = tid; i < item.size; i += 4 * bd) {
            uint64_t v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = (i + q * bd < item.size) ? X[i + q * bd] : 0;
#pragma unroll
            for (int q = 0; q < 4; q++)
                if (i + q * bd < item.size)
                    atomicAdd(&S.start[(uint32_t)((to_ord<DT>(v[q]) - mn) >> shift)], 1u);
        }
        __syncthreads();
        BG_PROF(1);
        // a digit holding >= 1/16 of the item (a heavy duplicate): the scatter
        // aggregates equal digits per warp instruction (one counter update per
        // digit, and the group's keys land contiguously) instead of letting
        // up to 32 lanes serialise on one counter
        {
            uint32_t m = 0;
            for (int d = tid; d < BIG_DIGITS; d += bd) m = max(m, S.start[d]);
            m = __reduce_max_sync(0xffffffffu, m);
            if (tid == 0) S.tmp[35] = 0;
            __syncthreads();
            if (lane == 0) atomicMax(&S.tmp[35], m);
            __syncthreads();
        }
        const bool agg = S.tmp[35] * 16u >= item.size;
        block_exscan(S.start, BIG_DIGITS, S.tmp);
        for (int d = tid; d < BIG_DIGITS; d += bd) S.end[d] = S.start[d];
        __syncthreads();
        if (!agg) {
            for (uint32_t i = tid; i < item.size; i += 4 * bd) {
                uint64_t v[4];
#pragma unroll
                for (int q = 0; q < 4; q++) v[q] = (i + q * bd < item.size) ? X[i + q * bd] : 0;
#pragma unroll
                for (int q = 0; q < 4; q++)
                    if (i + q * bd < item.size) {
                        const uint32_t d = (uint32_t)((to_ord<DT>(v[q]) - mn) >> shift);
                        Y[atomicAdd(&S.end[d], 1u)] = v[q];
                    }
            }
        } else for (uint32_t i0 = (uint32_t)(tid & ~31); i0 < item.size; i0 += 4 * bd) {
            const uint32_t i = i0 + (uint32_t)lane;  // (warp-uniform bound for the match)
            uint64_t v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = (i + q * bd < item.size) ? X[i + q * bd] : 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const bool ok = i + q * bd < item.size;
                const uint32_t d = ok ? (uint32_t)((to_ord<DT>(v[q]) - mn) >> shift) : 0xffffffffu;
                const uint32_t peers = __match_any_sync(0xffffffffu, d);
                const int leader = __ffs(peers) - 1;
                uint32_t at = 0;
                if (ok && lane == leader) at = atomicAdd(&S.end[d], (uint32_t)__popc(peers));
                at = __shfl_sync(0xffffffffu, at, leader) + (uint32_t)__popc(peers & ((1u << lane) - 1u));
                if (ok) Y[at] = v[q];  // peers land contiguously
            }
        }
        __syncthreads();  // S.end[d] = end of piece d; Y holds the pieces
        BG_PROF(2);
        if (shift == 0) {  // every piece holds a single value: Y is sorted
            if (Y != Aout)
                for (uint32_t i = tid; i < item.size; i += bd) Aout[i] = Y[i];
            __syncthreads();
            continue;
        }
        const bool y_is_b = !item.in_b;
        const uint32_t nwin = (item.size + BIG_CHUNK - 1) / BIG_CHUNK;
        for (uint32_t wbase = 0; wbase < nwin; wbase += BIG_MAXWIN) {
            for (int w = tid; w < BIG_MAXWIN; w += bd) {
                S.wlo[w] = BIG_DIGITS;
                S.whi[w] = 0;
            }
            __syncthreads();
            for (int d = tid; d < BIG_DIGITS; d += bd) {  // classify the pieces in parallel
                const uint32_t ps = S.start[d], pc = S.end[d] - ps;
                if (pc == 0) continue;
                if (pc <= BIG_CHUNK) {
                    const uint32_t w = ps / BIG_CHUNK;
                    if (w >= wbase && w < wbase + BIG_MAXWIN) {
                        atomicMin(&S.wlo[w - wbase], (uint32_t)d);
                        atomicMax(&S.whi[w - wbase], (uint32_t)d);
                    }
                } else if (wbase == 0) {
                    uint32_t k = BIG_MAXBLK;
                    if (pc <= BIG_SORT_CAP) k = atomicAdd(&S.nblk, 1u);
                    if (k < BIG_MAXBLK) {
                        S.blk[k] = (uint32_t)d;
                    } else if (lv + 1 < BIG_LEVELS) {  // next level
                        const uint32_t q = atomicAdd(&a.ctl->big_cnt[lv + 1], 1u);
                        if (q < a.big_cap)
                            a.big[(size_t)(lv + 1) * a.big_cap + q] =
                                BigItem{item.off + ps, pc, y_is_b ? 1u : 0u, ~0u, ~0ull, 0ull, 0u, 0u};
                        else
                            atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
                        if (lv == 0) {  // level 1 is consumed during the first pass: publish in order
                            __threadfence();
                            while (atomicCAS(&a.ctl->big_pub1, q, q + 1u) != q) {
                            }
                        }
                    } else {
                        atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
                    }
                }
            }
            __syncthreads();
            const uint32_t wend = min(nwin - wbase, (uint32_t)BIG_MAXWIN);
            for (uint32_t w = 0; w < wend; w++) {
                const uint32_t dlo = S.wlo[w], dhi = S.whi[w];
                if (dlo > dhi) continue;  // uniform
                const uint32_t slo = S.start[dlo], shi = S.end[dhi];
                // stage Y[slo, shi) with the TMA bulk engine (aligned hull)
                const uint64_t gl = item.off + slo, gh = item.off + shi;
                if (tid == 0) {
                    const uint64_t *Yb = item.in_b ? a.A : a.B;
                    const uint64_t h0 = gl & ~1ull;
                    uint64_t h1 = (gh + 1) & ~1ull;
                    if (h1 > a.n) {
                        h1 = gh & ~1ull;
                        S.sk[gh - 1 - h0] = Yb[gh - 1];
                    }
                    const uint32_t bytes = (uint32_t)((h1 - h0) * 8);
                    mbar_expect_tx(&S.mbar, bytes);
                    for (uint32_t o = 0; o < bytes; o += 32768u)
                        bulk_g2s((char *)S.sk + o, (const char *)(Yb + h0) + o,
                                 bytes - o < 32768u ? bytes - o : 32768u, &S.mbar);
                }
                mbar_wait(&S.mbar, mphase);
                mphase ^= 1u;
                uint64_t *sk = S.sk + (gl & 1ull);
                for (uint32_t d = dlo + tid; d <= dhi; d += bd) {  // one thread per tiny piece
                    const uint32_t pc = S.end[d] - S.start[d];
                    if (pc >= 2 && pc <= 8) insertion_sort<DT>(sk + (S.start[d] - slo), (int)pc);
                }
                BG_PROF(7);
                for (uint32_t d = dlo + warp; d <= dhi; d += nwarps) {  // one warp per larger piece
                    const uint32_t pc = S.end[d] - S.start[d];
                    if (pc <= 8) continue;
                    uint64_t *g = sk + (S.start[d] - slo);
                    if (shift <= 32 && pc <= 256) {  // piece within 2^32 ords: 32-bit peeling
                        const unsigned long long pbase = mn + ((unsigned long long)d << shift);
                        if (pc <= 32) warp_sort_keys_rel<DT, 1>(g, pc, pbase, lane);
                        else if (pc <= 64) warp_sort_keys_rel<DT, 2>(g, pc, pbase, lane);
                        else if (pc <= 128) warp_sort_keys_rel<DT, 4>(g, pc, pbase, lane);
                        else warp_sort_keys_rel<DT, 8>(g, pc, pbase, lane);
                    } else if (pc <= 32) {  // registers across the warp (peel few-valued pieces)
                        warp_sort_keys<DT, 1>(g, pc, lane);
                    } else if (pc <= 64) {
                        warp_sort_keys<DT, 2>(g, pc, lane);
                    } else if (pc <= 128) {
                        warp_sort_keys<DT, 4>(g, pc, lane);
                    } else if (pc <= 256) {
                        warp_sort_keys<DT, 8>(g, pc, lane);
                    } else {  // listed for the whole CTA below (one warp would hold up the window)
                        uint32_t k = 0;
                        if (lane == 0) k = atomicAdd(&S.nwbig, 1u);
                        k = __shfl_sync(0xffffffffu, k, 0);
                        if (k < BIG_MAXWBIG) {
                            if (lane == 0) S.wbig[k] = d;
                        } else {
                            bitonic<DT, false>(g, (int)pc, lane, 32);
                        }
                    }
                }
                __syncthreads();
                // pieces of 257..BIG_CHUNK keys: shared-memory bitonic by all
                // threads, one at a time
                const uint32_t nwb = min(S.nwbig, (uint32_t)BIG_MAXWBIG);
                for (uint32_t k = 0; k < nwb; k++) {
                    const uint32_t d = S.wbig[k];
                    bitonic<DT, true>(sk + (S.start[d] - slo), (int)(S.end[d] - S.start[d]), tid, bd);
                }
                BG_PROF(8);
                if (tid == 0) S.nwbig = 0;  // for the next window (ordered by the barrier below)
                for (uint32_t i = tid; i < shi - slo; i += bd) Aout[slo + i] = sk[i];
                __syncthreads();
            }
        }
        BG_PROF(3);
        const uint32_t nblk = min(S.nblk, (uint32_t)BIG_MAXBLK);
        for (uint32_t k = 0; k < nblk; k++) {
            const uint32_t d = S.blk[k];
            const uint32_t ps = S.start[d], pc = S.end[d] - ps;
            for (uint32_t i = tid; i < pc; i += bd) S.sk[i] = Y[ps + i];
            __syncthreads();
            bitonic<DT, true>(S.sk, (int)pc, tid, bd);
            for (uint32_t i = tid; i < pc; i += bd) Aout[ps + i] = S.sk[i];
            __syncthreads();
        }
        BG_PROF(4);
    }
}

// All big-path levels in one cooperative launch: level l + 1's items are
// complete after a grid barrier; the kernel stops at the first empty level
// (for smooth inputs: at once), instead of BIG_LEVELS separate launches.
template <int DT>
__global__ void __launch_bounds__(BIG_THREADS, 1) k_big(Args a) {
    if (a.ctl->status) return;  // (set before this kernel: uniform across the grid)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BigSmem &S = *reinterpret_cast<BigSmem *>(smem_raw);
    uint32_t mphase = 0;
    if (threadIdx.x == 0) mbar_init(&S.mbar, 1);
    __syncthreads();
    cg::grid_group grid = cg::this_grid();
    for (int lv = 0; lv < BIG_LEVELS; lv++) {
        if (*(volatile uint32_t *)&a.ctl->big_cnt[lv] == 0) break;  // uniform: read after a grid barrier
        big_level<DT>(a, lv, S, mphase);
        const long long t0 = clock64();
        grid.sync();
        if ((a.dbg & 512u) && threadIdx.x == 0) {
            atomicAdd(&a.ctl->prof[11], (unsigned long long)(clock64() - t0));
        }
    }
}

// -------------------------------------------------------------- launchers --
template <int NT, int KPT, int PER_SM>
static void launch_ctasort(const Args &a, int dtype, cudaStream_t st, const uint4 *list,
                           const uint32_t *count, int sms) {
    const size_t sm = sizeof(CsSmem<NT * KPT>);
    const int g = sms * PER_SM;
    if (dtype == DT_F64) {
        cudaFuncSetAttribute(k_ctasort<DT_F64, NT, KPT, PER_SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_ctasort<DT_F64, NT, KPT, PER_SM><<<g, NT, sm, st>>>(a, list, count);
    } else {
        cudaFuncSetAttribute(k_ctasort<DT_U64, NT, KPT, PER_SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_ctasort<DT_U64, NT, KPT, PER_SM><<<g, NT, sm, st>>>(a, list, count);
    }
}

void launch_warpsort(const Args &a, int dtype, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int g = sms * WS_CTAS_PER_SM;
    if (dtype == DT_F64) k_warpsort<DT_F64><<<g, WS_WARPS * 32, 0, st>>>(a);
    else k_warpsort<DT_U64><<<g, WS_WARPS * 32, 0, st>>>(a);
}

// The other sorts of the in-bucket phase (CTA sorts, block windows): every
// one reads only its own sub-buckets, so they run beside k_warpsort.
void launch_bucketsort(const Args &a, int dtype, const cudaStream_t ss[5]) {
    {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        launch_ctasort<256, 16, 3>(a, dtype, ss[0], a.ctasks, &a.ctl->nctask, sms);
        launch_ctasort<128, 16, 6>(a, dtype, ss[1], a.ctasks2, &a.ctl->nctask2, sms);
        launch_ctasort<128, 8, 8>(a, dtype, ss[2], a.ctasks3, &a.ctl->nctask3, sms);
        launch_ctasort<64, 8, 16>(a, dtype, ss[3], a.ctasks4, &a.ctl->nctask4, sms);
    }
    const cudaStream_t st = ss[4];
    k_window_list<<<(a.ntiles + 255) / 256, 256, 0, st>>>(a);
    const size_t sm = sizeof(BsSmem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)umin64((uint64_t)sms * BS_CTAS_PER_SM, a.ntiles);
    if (dtype == DT_F64) {
        cudaFuncSetAttribute(k_bucketsort<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_bucketsort<DT_F64><<<grid, BS_THREADS, sm, st>>>(a);
    } else {
        cudaFuncSetAttribute(k_bucketsort<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_bucketsort<DT_U64><<<grid, BS_THREADS, sm, st>>>(a);
    }
}

void launch_big_minmax(const Args &a, int dtype, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dtype == DT_F64) k_big_minmax<DT_F64><<<sms * 3, 512, 0, st>>>(a);  // (3 resident per SM: one wave)
    else k_big_minmax<DT_U64><<<sms * 3, 512, 0, st>>>(a);
}

void launch_big_order(const Args &a, cudaStream_t st) { k_big_order<<<1, 1024, 0, st>>>(a); }

void launch_big(const Args &a, int dtype, cudaStream_t st) {
    const size_t sm = sizeof(BigSmem);
    int dev = 0, sms = 148, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    void *fn = dtype == DT_F64 ? (void *)k_big<DT_F64> : (void *)k_big<DT_U64>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, BIG_THREADS, sm);
    dim3 grid((unsigned)(sms * (per < 2 ? (per < 1 ? 1 : per) : 2))), block(BIG_THREADS);
    Args aa = a;
    void *args[] = {&aa};
    cudaLaunchCooperativeKernel(fn, grid, block, args, sm, st);
}

}  // namespace ls
