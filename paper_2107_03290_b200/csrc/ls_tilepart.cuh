// ls_tilepart.cuh -- the scatter half of a partition round (Alg. 1's placement
// of keys into their buckets), B200 version.
//
// One CTA of TP_THREADS threads owns a unit [beg, end) of the source and, per
// bucket b, a global write cursor base[b] (from the count pass + decoupled
// lookback). The unit is processed in tiles of TP_TILE keys:
//   * tiles are staged global -> shared by the TMA bulk-copy engine
//     (cp.async.bulk, SASS UBLKCP) into a 2-slot ring, one tile ahead, so HBM
//     reads never wait behind the compute of the current tile;
//   * every thread takes TP_KPT keys, computes their bucket and takes a rank
//     inside the tile with a shared-memory atomic;
//   * one block scan over the <= 1024 bucket counts (bucket b <-> thread b)
//     gives the tile-local bucket starts and advances the cursors;
//   * keys are placed bucket-contiguous into the (now consumed) ring slot and
//     stored by consecutive threads to consecutive addresses of each bucket
//     run -- runs of ~TP_TILE/f keys instead of one scattered key per thread.
// 1024 threads x 8 keys per tile: with f = 1000 the average run is 8 keys
// (64 B), and only one unit per SM is open at a time, which keeps the number
// of partially written L2 lines low (ncu showed ~0.95 GB of extra DRAM reads
// per 200M-key pass with 4-CTA/SM, 4K-key tiles).
#pragma once
#include "ls_common.cuh"

namespace ls {

constexpr int TP_THREADS = 1024;
constexpr int TP_KPT = 8;
constexpr int TP_TILE = TP_THREADS * TP_KPT;  // 8192 keys
constexpr int TP_NSLOT = 2;                   // ring slots (3 slots of 6K-key tiles measured slower: shorter runs)

constexpr size_t MAX_SMEM_OPTIN = 232448;  // 227 KB per block on sm_100

// Shared memory of tile_partition for NT threads x KPT keys per tile.
template <int NT, int KPT>
struct TpSmemT {
    static constexpr int TILE = NT * KPT;
    static constexpr int SLOT = TILE + 2;  // + aligned-hull slack
    uint64_t ring[TP_NSLOT][SLOT];
    uint16_t sbin[TILE];
    uint32_t cnt[LS_MAX_FANOUT];
    uint32_t ex[LS_MAX_FANOUT];
    uint32_t delta[LS_MAX_FANOUT];
    uint32_t wsum[33];
    uint32_t tot;
    uint64_t mbar[TP_NSLOT];
};
typedef TpSmemT<TP_THREADS, TP_KPT> TpSmem;
template <int TILE>
using TpBidsT = uint16_t[TP_NSLOT][TILE + 16];  // staged precomputed bucket ids (BIDS mode)
typedef TpBidsT<TP_TILE> TpBids;

// Round 0 by reservation (k_scatter0r): instead of cursors from a count pass,
// every tile reserves its run in bucket b with one atomicAdd on cur[b]; bucket
// b owns dst[bsrc[b], bsrc[b] + cap[b]). A run that would pass cap[b] is not
// written and raises *ovf (the caller then redoes the round exactly). lim =
// an index no valid run reaches (stores at or beyond it are dropped).
// cur32 != nullptr: exact 32-bit cursors (absolute destination indices,
// k_scatter1): no capacities, nothing overflows; cur, cap, bsrc, ovf unused.
struct TpReserve {
    unsigned long long *cur;
    const unsigned long long *cap, *bsrc;
    uint32_t *ovf;
    uint32_t lim;
    uint32_t *cur32;
};

constexpr uint32_t TP_SKIP = 0xffffu;  // bucket id of keys that are not moved (SKIP mode)

// Issue the bulk copy of src[t0, t1) into ring slot `slot`, so that key k lands
// at slot[k - (t0 & ~1)]. The bulk engine moves 16-byte-aligned ranges, so the
// copy covers the aligned hull [t0 & ~1, (t1 + 1) & ~1); only when that hull
// would run past the end of the array (len odd, t1 == len) is the last key
// loaded by this (single) thread directly.
template <class SM, class SB = TpBids>
__device__ __forceinline__ void tp_issue(SM &S, int slot, const uint64_t *src, uint64_t t0,
                                         uint64_t t1, uint64_t len, const uint16_t *bid = nullptr,
                                         SB *sb = nullptr) {
    uint64_t *dst = S.ring[slot];
    const uint64_t a0 = t0 & ~1ull;
    uint64_t a1 = (t1 + 1) & ~1ull;
    if (a1 > len) {
        a1 = t1 & ~1ull;
        dst[t1 - 1 - a0] = src[t1 - 1];
    }
    const uint32_t bytes = a1 > a0 ? (uint32_t)((a1 - a0) * 8) : 0u;
    // bucket ids: 16-byte-aligned hull of [t0, t1) (the id array is padded)
    const uint64_t s0 = t0 & ~7ull, s1 = (t1 + 7) & ~7ull;
    const uint32_t sbytes = bid ? (uint32_t)((s1 - s0) * 2) : 0u;
    mbar_expect_tx(&S.mbar[slot], bytes + sbytes);
    constexpr uint32_t CH = 32768;
    for (uint32_t o = 0; o < bytes; o += CH)
        bulk_g2s((char *)dst + o, (const char *)(src + a0) + o, bytes - o < CH ? bytes - o : CH,
                 &S.mbar[slot]);
    if (bid) bulk_g2s((*sb)[slot], bid + s0, sbytes, &S.mbar[slot]);
}

// Partition src[beg, end) into nb <= 1024 buckets: key -> dst[base[b]++].
// len = number of keys in the src array (bound for the aligned hull).
// base[] is in shared memory, owned by thread b. bf(key, index) -> bucket.
// All threads of the CTA call it; S.mbar must have been initialised (count 1)
// by tp_init and every phase used so far is tracked in `phase`.
// BIDS: the bucket of key i is bid[i] (precomputed by the count pass, staged
// by the bulk engine next to the keys); bf is not called.
// RESERVE: base is unused; runs are reserved through *rs (TpReserve).
// PEER: bucket b's runs go to pdst[b] + cursor (pdst: shared memory, one
// pointer per bucket -- a destination rank's receive buffer, possibly another
// GPU's memory mapped through CUDA IPC: the stores cross NVLink); dst unused.
template <bool SKIP = false, bool BIDS = false, bool ISSUED = false, class BF, int NT = TP_THREADS,
          int KPT = TP_KPT, class SB = TpBids, bool RESERVE = false, bool PEER = false>
__device__ __forceinline__ void tile_partition(TpSmemT<NT, KPT> &S, const uint64_t *__restrict__ src,
                                               uint64_t *__restrict__ dst, uint64_t beg,
                                               uint64_t end, uint64_t len, uint32_t *base,
                                               int nb, const BF &bf, uint32_t &phase,
                                               const uint16_t *bid = nullptr, SB *sb = nullptr,
                                               unsigned long long *prof = nullptr,
                                               const TpReserve *rs = nullptr,
                                               uint64_t *const *pdst = nullptr) {
    constexpr int TILE = NT * KPT;
    constexpr int BPT = (LS_MAX_FANOUT + NT - 1) / NT;  // buckets per thread in the scan
    long long tq = clock64();
    auto mark = [&](int k) {
        if (prof && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(&prof[k], (unsigned long long)(t - tq));
            tq = t;
        }
    };
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // tiles start at even key positions (tbase + i * TILE, tbase = beg rounded
    // down to even), so every staged tile is 16-byte aligned in its ring slot
    // and the rank phase reads key pairs (and id pairs) with one vector load;
    // the first tile's key at tbase < beg (when beg is odd) is not ours
    static_assert(KPT % 2 == 0, "tile_partition reads key pairs");
    const uint64_t tbase = beg & ~1ull;
    const uint64_t ntl = end > beg ? (end - tbase + TILE - 1) / TILE : 0;
    if (ntl == 0) return;
    if (!ISSUED && tid == 0)  // (ISSUED: the caller has staged the first tiles, tp_issue_first)
        for (uint64_t j = 0; j < (uint64_t)TP_NSLOT && j < ntl; j++)
            tp_issue<TpSmemT<NT, KPT>, SB>(S, (int)j, src, tbase + j * TILE, umin64(end, tbase + (j + 1) * TILE), len,
                     BIDS ? bid : nullptr, sb);
    for (int b = tid; b < nb; b += NT) S.cnt[b] = 0;
    // RESERVE: this thread's buckets' capacities and regions, once
    unsigned long long rcap[RESERVE ? BPT : 1], rsrc[RESERVE ? BPT : 1];
    if (RESERVE && !rs->cur32) {
#pragma unroll
        for (int j = 0; j < BPT; j++) {
            const int b = BPT * tid + j;
            rcap[j] = b < nb ? rs->cap[b] : 0ull;
            rsrc[j] = b < nb ? rs->bsrc[b] : 0ull;
        }
    }
    __syncthreads();
    for (uint64_t i = 0; i < ntl; i++) {
        const int slot = (int)(i % TP_NSLOT);
        const uint64_t t0 = tbase + i * TILE;                       // (even)
        const int th = (int)umin64((uint64_t)TILE, end - t0);       // slot positions [0, th) staged
        const int lo = i == 0 ? (int)(beg - tbase) : 0;             // ... of which [lo, th) are ours
        const int tn = th - lo;                                     // keys in this tile
        mbar_wait(&S.mbar[slot], (phase >> slot) & 1u);
        mark(0);
        const uint64_t *keys = S.ring[slot];                        // key t0 + h at keys[h]
        const uint16_t *bids = BIDS ? (*sb)[slot] + (t0 & 7) : nullptr;  // (t0 & 7 even: 4-byte pairs)
        uint64_t key[KPT];
        uint32_t code[KPT];
#pragma unroll
        for (int k2 = 0; k2 < KPT / 2; k2++) {
            const int h = 2 * (k2 * NT + tid);  // slot positions h, h + 1
            const ulonglong2 kv = *reinterpret_cast<const ulonglong2 *>(keys + h);
            const uint32_t ip = BIDS ? *reinterpret_cast<const uint32_t *>(bids + h) : 0u;
            key[2 * k2] = kv.x;
            key[2 * k2 + 1] = kv.y;
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int k = 2 * k2 + e;
                code[k] = 0xffffffffu;
                if (h + e >= lo && h + e < th) {
                    const uint32_t b = BIDS ? (e ? ip >> 16 : ip & 0xffffu) : bf(key[k], t0 + h + e);
                    if (!SKIP || b != TP_SKIP) {
                        const uint32_t r = atomicAdd(&S.cnt[b], 1u);
                        code[k] = b | (r << 10);
                    }
                }
            }
        }
        __syncthreads();
        mark(1);
        // every thread is past the previous tile's store phase: its ring slot
        // is free for the tile after the next one
        if (tid == 0 && i >= 1 && i - 1 + TP_NSLOT < ntl) {
            const uint64_t tp0 = tbase + (i - 1 + TP_NSLOT) * TILE;
            tp_issue<TpSmemT<NT, KPT>, SB>(S, (int)((i - 1) % TP_NSLOT), src, tp0, umin64(end, tp0 + TILE), len,
                     BIDS ? bid : nullptr, sb);
        }
        // exclusive scan of the tile's bucket counts (buckets BPT*tid ..
        // BPT*tid + BPT-1 <-> thread tid): warp scans, then every warp adds
        // the totals of the warps before it (one redux per warp instead of a
        // second barrier-separated pass)
        uint32_t cb[BPT], c = 0;
#pragma unroll
        for (int j = 0; j < BPT; j++) {
            const int b = BPT * tid + j;
            cb[j] = b < nb ? S.cnt[b] : 0u;
            c += cb[j];
        }
        // RESERVE: the runs are reserved now; the atomics' results are first
        // needed after the placement below (their latency overlaps it)
        unsigned long long rsv[RESERVE ? BPT : 1];
        if (RESERVE) {
#pragma unroll
            for (int j = 0; j < BPT; j++) {
                const int b = BPT * tid + j;
                rsv[j] = !cb[j] ? 0ull
                         : rs->cur32 ? (unsigned long long)atomicAdd(&rs->cur32[b], cb[j])
                                     : atomicAdd(&rs->cur[b], (unsigned long long)cb[j]);
            }
        }
        const uint32_t incl = warp_incl_scan(c);
        if (lane == 31) S.wsum[warp] = incl;
        __syncthreads();
        const uint32_t ws = lane < NT / 32 ? S.wsum[lane] : 0u;
        const uint32_t wpre = __reduce_add_sync(0xffffffffu, lane < warp ? ws : 0u);
        const uint32_t wtot = SKIP ? __reduce_add_sync(0xffffffffu, ws) : 0u;  // keys that move
        const uint32_t ex0 = wpre + incl - c;
        uint32_t ex = ex0;
#pragma unroll
        for (int j = 0; j < BPT; j++) {
            const int b = BPT * tid + j;
            if (b < nb) {
                S.ex[b] = ex;
                if (!RESERVE) {
                    S.delta[b] = base[b] - ex;
                    base[b] += cb[j];
                }
                S.cnt[b] = 0;
            }
            ex += cb[j];
        }
        __syncthreads();
        mark(2);
        // bucket-contiguous order inside the consumed slot (all lookups
        // first, then all stores: independent shared-memory chains)
        uint64_t *sk = S.ring[slot];
        uint32_t pos[KPT];
#pragma unroll
        for (int k = 0; k < KPT; k++)
            pos[k] = code[k] != 0xffffffffu ? S.ex[code[k] & 1023u] + (code[k] >> 10) : 0xffffffffu;
#pragma unroll
        for (int k = 0; k < KPT; k++) {
            if (pos[k] != 0xffffffffu) {
                sk[pos[k]] = key[k];
                S.sbin[pos[k]] = (uint16_t)(code[k] & 1023u);
            }
        }
        if (RESERVE) {  // run starts from the reservations (delta = start - tile offset)
            uint32_t e = ex0;
#pragma unroll
            for (int j = 0; j < BPT; j++) {
                const int b = BPT * tid + j;
                if (cb[j]) {
                    uint32_t d;
                    if (rs->cur32) {
                        d = (uint32_t)rsv[j] - e;
                    } else if (rsv[j] + cb[j] <= rcap[j]) {
                        d = (uint32_t)(rsrc[j] + rsv[j]) - e;
                    } else {  // over capacity: dropped (the round is redone exactly)
                        d = rs->lim;
                        atomicOr(rs->ovf, 1u);
                    }
                    S.delta[b] = d;
                }
                e += cb[j];
            }
        }
        __syncthreads();
        mark(3);
        {
            const int tm = SKIP ? (int)wtot : tn;
            uint32_t b[KPT], d[KPT];
            uint64_t v[KPT];
#pragma unroll
            for (int k = 0; k < KPT; k++) {
                const int idx = k * NT + tid;
                b[k] = idx < tm ? S.sbin[idx] : 0u;
                v[k] = sk[idx];
            }
#pragma unroll
            for (int k = 0; k < KPT; k++) d[k] = S.delta[b[k]];
#pragma unroll
            for (int k = 0; k < KPT; k++) {
                const int idx = k * NT + tid;
                if (RESERVE) {
                    const uint32_t q = d[k] + (uint32_t)idx;
                    if (idx < tm && q < rs->lim) dst[q] = v[k];
                } else if (PEER) {
                    if (idx < tm) pdst[b[k]][d[k] + (uint32_t)idx] = v[k];
                } else if (idx < tm) {
                    dst[d[k] + (uint32_t)idx] = v[k];
                }
            }
        }
        // (no barrier: the next tile's first barrier orders these reads of the
        // slot, sbin and delta before anything overwrites them)
        mark(4);
        phase ^= 1u << slot;
    }
    __syncthreads();  // (the caller may reuse the ring and tables right away)
}

// One thread: initialise the ring barriers and stage the first tiles of
// [beg, end) at once (before the caller's own setup), for tile_partition<..,
// ISSUED = true> after a block barrier.
template <class SM, class SB = TpBids>
__device__ __forceinline__ void tp_issue_first(SM &S, const uint64_t *src, uint64_t beg, uint64_t end,
                                              uint64_t len, const uint16_t *bid = nullptr,
                                              SB *sb = nullptr) {
    constexpr int TILE = SM::TILE;
    for (int j = 0; j < TP_NSLOT; j++) mbar_init(&S.mbar[j], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (inits before the bulk copies)
    if (end <= beg) return;
    const uint64_t base = beg & ~1ull;  // (tile_partition's tiling: even tile starts)
    for (uint64_t j = 0; j < (uint64_t)TP_NSLOT && base + j * TILE < end; j++)
        tp_issue<SM, SB>(S, (int)j, src, base + j * TILE, umin64(end, base + (j + 1) * TILE), len, bid, sb);
}

template <class SM>
__device__ __forceinline__ void tp_init(SM &S) {
    if (threadIdx.x == 0)
        for (int j = 0; j < TP_NSLOT; j++) mbar_init(&S.mbar[j], 1);
    __syncthreads();
}

}  // namespace ls
