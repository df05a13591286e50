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
constexpr int TP_SLOT = TP_TILE + 2;          // + aligned-hull slack

constexpr size_t MAX_SMEM_OPTIN = 232448;  // 227 KB per block on sm_100
typedef uint16_t TpBids[TP_NSLOT][TP_TILE + 16];  // staged precomputed bucket ids (BIDS mode)

struct TpSmem {
    uint64_t ring[TP_NSLOT][TP_SLOT];
    uint16_t sbin[TP_TILE];
    uint32_t cnt[LS_MAX_FANOUT];
    uint32_t ex[LS_MAX_FANOUT];
    uint32_t delta[LS_MAX_FANOUT];
    uint32_t wsum[33];
    uint32_t tot;
    uint64_t mbar[TP_NSLOT];
};

constexpr uint32_t TP_SKIP = 0xffffu;  // bucket id of keys that are not moved (SKIP mode)

// Issue the bulk copy of src[t0, t1) into ring slot `slot`, so that key k lands
// at slot[k - (t0 & ~1)]. The bulk engine moves 16-byte-aligned ranges, so the
// copy covers the aligned hull [t0 & ~1, (t1 + 1) & ~1); only when that hull
// would run past the end of the array (len odd, t1 == len) is the last key
// loaded by this (single) thread directly.
__device__ __forceinline__ void tp_issue(TpSmem &S, int slot, const uint64_t *src, uint64_t t0,
                                         uint64_t t1, uint64_t len, const uint16_t *bid = nullptr,
                                         TpBids *sb = nullptr) {
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
template <bool SKIP = false, bool BIDS = false, bool ISSUED = false, class BF>
__device__ __forceinline__ void tile_partition(TpSmem &S, const uint64_t *__restrict__ src,
                                               uint64_t *__restrict__ dst, uint64_t beg,
                                               uint64_t end, uint64_t len, uint32_t *base,
                                               int nb, const BF &bf, uint32_t &phase,
                                               const uint16_t *bid = nullptr, TpBids *sb = nullptr,
                                               unsigned long long *prof = nullptr) {
    long long tq = clock64();
    auto mark = [&](int k) {
        if (prof && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(&prof[k], (unsigned long long)(t - tq));
            tq = t;
        }
    };
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t ntl = (end - beg + TP_TILE - 1) / TP_TILE;
    if (ntl == 0) return;
    if (!ISSUED && tid == 0)  // (ISSUED: the caller has staged the first tiles, tp_issue_first)
        for (uint64_t j = 0; j < (uint64_t)TP_NSLOT && j < ntl; j++)
            tp_issue(S, (int)j, src, beg + j * TP_TILE, umin64(end, beg + (j + 1) * TP_TILE), len,
                     BIDS ? bid : nullptr, sb);
    if (tid < nb) S.cnt[tid] = 0;
    __syncthreads();
    for (uint64_t i = 0; i < ntl; i++) {
        const int slot = (int)(i % TP_NSLOT);
        const uint64_t t0 = beg + i * TP_TILE;
        const int tn = (int)umin64((uint64_t)TP_TILE, end - t0);
        mbar_wait(&S.mbar[slot], (phase >> slot) & 1u);
        mark(0);
        const uint64_t *keys = S.ring[slot] + (t0 & 1);
        const uint16_t *bids = BIDS ? (*sb)[slot] + (t0 & 7) : nullptr;
        uint64_t key[TP_KPT];
        uint32_t code[TP_KPT];
#pragma unroll
        for (int k = 0; k < TP_KPT; k++) {
            const int idx = k * TP_THREADS + tid;
            code[k] = 0xffffffffu;
            if (idx < tn) {
                key[k] = keys[idx];
                const uint32_t b = BIDS ? (uint32_t)bids[idx] : bf(key[k], t0 + idx);
                if (!SKIP || b != TP_SKIP) {
                    const uint32_t r = atomicAdd(&S.cnt[b], 1u);
                    code[k] = b | (r << 10);
                }
            }
        }
        __syncthreads();
        mark(1);
        // every thread is past the previous tile's store phase: its ring slot
        // is free for the tile after the next one
        if (tid == 0 && i >= 1 && i - 1 + TP_NSLOT < ntl) {
            const uint64_t tp0 = beg + (i - 1 + TP_NSLOT) * TP_TILE;
            tp_issue(S, (int)((i - 1) % TP_NSLOT), src, tp0, umin64(end, tp0 + TP_TILE), len,
                     BIDS ? bid : nullptr, sb);
        }
        // exclusive scan of the tile's bucket counts (bucket b <-> thread b):
        // warp scans, then every warp adds the totals of the warps before it
        // (one redux per warp instead of a second barrier-separated pass)
        uint32_t c = tid < nb ? S.cnt[tid] : 0u;
        const uint32_t incl = warp_incl_scan(c);
        if (lane == 31) S.wsum[warp] = incl;
        __syncthreads();
        const uint32_t ws = S.wsum[lane];
        const uint32_t wpre = __reduce_add_sync(0xffffffffu, lane < warp ? ws : 0u);
        const uint32_t wtot = SKIP ? __reduce_add_sync(0xffffffffu, ws) : 0u;  // keys that move
        if (tid < nb) {
            const uint32_t ex = wpre + incl - c;
            S.ex[tid] = ex;
            S.delta[tid] = base[tid] - ex;
            base[tid] += c;
            S.cnt[tid] = 0;
        }
        __syncthreads();
        mark(2);
        // bucket-contiguous order inside the consumed slot (all lookups
        // first, then all stores: independent shared-memory chains)
        uint64_t *sk = S.ring[slot];
        uint32_t pos[TP_KPT];
#pragma unroll
        for (int k = 0; k < TP_KPT; k++)
            pos[k] = code[k] != 0xffffffffu ? S.ex[code[k] & 1023u] + (code[k] >> 10) : 0xffffffffu;
#pragma unroll
        for (int k = 0; k < TP_KPT; k++) {
            if (pos[k] != 0xffffffffu) {
                sk[pos[k]] = key[k];
                S.sbin[pos[k]] = (uint16_t)(code[k] & 1023u);
            }
        }
        __syncthreads();
        mark(3);
        {
            const int tm = SKIP ? (int)wtot : tn;
            uint32_t b[TP_KPT], d[TP_KPT];
            uint64_t v[TP_KPT];
#pragma unroll
            for (int k = 0; k < TP_KPT; k++) {
                const int idx = k * TP_THREADS + tid;
                b[k] = idx < tm ? S.sbin[idx] : 0u;
                v[k] = sk[idx];
            }
#pragma unroll
            for (int k = 0; k < TP_KPT; k++) d[k] = S.delta[b[k]];
#pragma unroll
            for (int k = 0; k < TP_KPT; k++) {
                const int idx = k * TP_THREADS + tid;
                if (idx < tm) dst[d[k] + (uint32_t)idx] = v[k];
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
__device__ __forceinline__ void tp_issue_first(TpSmem &S, const uint64_t *src, uint64_t beg, uint64_t end,
                                               uint64_t len, const uint16_t *bid = nullptr,
                                               TpBids *sb = nullptr) {
    for (int j = 0; j < TP_NSLOT; j++) mbar_init(&S.mbar[j], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // (inits before the bulk copies)
    for (uint64_t j = 0; j < (uint64_t)TP_NSLOT && beg + j * TP_TILE < end; j++)
        tp_issue(S, (int)j, src, beg + j * TP_TILE, umin64(end, beg + (j + 1) * TP_TILE), len, bid, sb);
}

__device__ __forceinline__ void tp_init(TpSmem &S) {
    if (threadIdx.x == 0)
        for (int j = 0; j < TP_NSLOT; j++) mbar_init(&S.mbar[j], 1);
    __syncthreads();
}

}  // namespace ls
