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
#include "ls_launch.h"

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

// ----------------------------------------------------------- SMALL path ----
// One CTA per window of T_tile key positions. It owns every SMALL sub-bucket
// that starts in the window (classify recorded the first/last one), so its
// span [lo, hi) holds at most T_tile + T_small keys; the span is staged into
// shared memory by the TMA bulk engine. All sub-buckets of the span are
// processed at once, one thread per key:
//   slot(key) = start(sub-bucket) + pos   for keys of SMALL sub-buckets
//   slot(key) = own position              for everything else in the span
// so one exclusive scan over the span's slots yields the counting-sort
// placement of every sub-bucket at once (each sub-bucket's slots stay inside
// its own range, so other keys keep their places). The touch-up then gives
// every key its rank inside its collision group (run of equal slot) and
// stores it at its final position: the insertion sort's result without its
// divergent serial shifting. All-equal groups and homogeneous sub-buckets are
// detected and skipped.
constexpr int BS_THREADS = 512;
constexpr int BS_KPT = 8;          // keys per thread; span cap = 4096
constexpr int BS_SPAN = BS_THREADS * BS_KPT;
constexpr int BS_WORDS = BS_SPAN / 32;
constexpr int BS_MAXBIG = 128;     // collision groups > 8 keys per window

struct BsSmem {
    union {                        // the staged span lives in registers once the
        uint64_t keys[BS_SPAN + 2];  // slots are known, so the counting-sort target
        uint64_t T[BS_SPAN + 2];     // T (ord values) reuses its storage
    };
    alignas(16) uint32_t K[BS_SPAN + 4];    // slot histogram -> exclusive scan
    alignas(16) uint32_t gnp[BS_SPAN];      // at a head: g | n' << 20; after placement: slot of T[q]
    alignas(16) uint32_t headbits[BS_WORDS];  // sub-bucket heads (bit per position)
    alignas(16) uint32_t diffbits[BS_WORDS];  // at a head: the sub-bucket is not homogeneous
    uint32_t wlast[BS_WORDS];               // 1 + last head position before word w (0: none)
    uint32_t big[BS_MAXBIG];                // slots of collision groups > 8 keys
    uint32_t nbig, ovf;
    uint32_t tmp[36];
    unsigned long long st_small, st_smallk, st_h1, st_h1k, st_maxg;
    uint64_t mbar;
};

// head position of the sub-bucket covering span position q
__device__ __forceinline__ uint32_t head_of(const BsSmem &S, uint32_t q) {
    const uint32_t w = q >> 5;
    const uint32_t bits = S.headbits[w] & (0xffffffffu >> (31u - (q & 31u)));
    return bits ? (w << 5) + 31u - __clz(bits) : S.wlast[w] - 1u;
}
__device__ __forceinline__ bool diff_at(const BsSmem &S, uint32_t h) {
    return (S.diffbits[h >> 5] >> (h & 31u)) & 1u;
}

template <int DT>
__global__ void __launch_bounds__(BS_THREADS, 2) k_bucketsort(Args a) {
    if (a.ctl->status) return;
    const uint4 desc = a.tdesc[blockIdx.x];  // {g0, g1, lo, hi} (k_tile_desc)
    const uint32_t g0 = desc.x, g1 = desc.y, lo = desc.z, hi = desc.w;
    if (g0 == 0xffffffffu) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BsSmem &S = *reinterpret_cast<BsSmem *>(smem_raw);
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int span = (int)(hi - lo);
    // stage the span with the TMA bulk engine; zero the tables meanwhile
    const uint32_t alo = lo & ~1u, ahi = (hi + 1) & ~1u;
    if (tid == 0) {
        mbar_init(&S.mbar, 1);
        const uint32_t bytes = (ahi - alo) * 8u;
        mbar_expect_tx(&S.mbar, bytes);
        for (uint32_t o = 0; o < bytes; o += 16384)
            bulk_g2s((char *)S.keys + o, (const char *)(a.A + alo) + o, bytes - o < 16384 ? bytes - o : 16384, &S.mbar);
        S.nbig = S.ovf = 0;
        S.st_small = S.st_smallk = S.st_h1 = S.st_h1k = S.st_maxg = 0;
    }
    {
        uint4 *k4 = reinterpret_cast<uint4 *>(S.K);
        const uint4 z = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < (span + 4) / 4; i += bd) k4[i] = z;
        if (tid < BS_WORDS) S.headbits[tid] = S.diffbits[tid] = 0;
    }
    __syncthreads();
    // sub-bucket heads (P:176-183 iterate the sub-buckets of the window)
    for (uint32_t g = g0 + tid; g <= g1; g += bd) {
        const uint32_t np = __ldg(&a.hist1[g]);
        if (np >= 1) {
            const uint32_t h = __ldg(&a.start1[g]) - lo;
            atomicOr(&S.headbits[h >> 5], 1u << (h & 31u));
            S.gnp[h] = g | (np << 20);  // f*f <= 2^20, n' <= 2048
        }
    }
    __syncthreads();
    if (warp == 0) {  // wlast: exclusive max-scan over the per-word last heads
        uint32_t v[BS_WORDS / 32];
        uint32_t run = 0;
#pragma unroll
        for (int k = 0; k < BS_WORDS / 32; k++) {
            const int w = lane * (BS_WORDS / 32) + k;
            const uint32_t b = S.headbits[w];
            v[k] = b ? (uint32_t)(w << 5) + 32u - __clz(b) : 0u;  // last head + 1 in word w
            run = v[k] > run ? v[k] : run;
        }
        uint32_t incl = warp_incl_max(run);
        uint32_t ex = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) ex = 0;
#pragma unroll
        for (int k = 0; k < BS_WORDS / 32; k++) {
            S.wlast[lane * (BS_WORDS / 32) + k] = ex;
            ex = v[k] > ex ? v[k] : ex;
        }
    }
    mbar_wait(&S.mbar, 0);
    __syncthreads();
    const uint64_t *keys = S.keys + (lo - alo);
    if (a.dbg == 1) return;
    // counting-sort slots (Alg. 2)
    const Root R = load_root(a.M);
    uint32_t packed[BS_KPT];
    uint64_t kv[BS_KPT];
#pragma unroll
    for (int j = 0; j < BS_KPT; j++) {
        const int i = j * bd + tid;
        packed[j] = 0xffffffffu;
        if (i < span) {
            const uint32_t st = head_of(S, (uint32_t)i);
            const uint32_t gnp = S.gnp[st];
            const uint32_t g = gnp & 0xfffffu, np = gnp >> 20;
            const uint64_t key = keys[i];
            kv[j] = key;
            uint32_t slot = (uint32_t)i;
            if ((uint32_t)i - st < np && np >= 2) {
                const double p = predict_ldg<DT>(key, R, a.M->leaf);
                const double adj = __ddiv_rn((double)g, a.F2);  // (i*f + j)/f^2
                slot = st + cs_pos(p, adj, a.nd, (double)(np - 1));
                if (key != keys[st] && !diff_at(S, st)) atomicOr(&S.diffbits[st >> 5], 1u << (st & 31u));
            }
            const uint32_t r = atomicAdd(&S.K[slot], 1u);
            packed[j] = slot | (r << 16);
        }
    }
    __syncthreads();
    if (a.dbg == 3) return;
    block_exscan(S.K, span + 1, S.tmp);  // running totals, exclusive (R4)
    // placement. T holds ord values (plain integer compares in the
    // touch-up); gnp[q] now remembers the slot of T position q.
#pragma unroll
    for (int j = 0; j < BS_KPT; j++) {
        if (packed[j] == 0xffffffffu) continue;
        const uint32_t slot = packed[j] & 0xffffu;
        const uint32_t q = S.K[slot] + (packed[j] >> 16);
        S.T[q] = to_ord<DT>(kv[j]);
        S.gnp[q] = slot;
    }
    __syncthreads();
    if (a.dbg == 4) return;
    // Touch-up per collision group (R15), in T order: every key takes
    // its rank inside its group (keys strictly below it + equal keys placed
    // before it) and is stored at its final position -- the insertion sort's
    // result without its serial shifting. Groups of > 8 keys (typically the
    // clamped top slot of a sparse sub-bucket, R5) are ordered by a warp.
    // Only sub-buckets that are not homogeneous are written back.
    uint32_t maxg = 0;
    for (int q = tid; q < span; q += bd) {
        if (!diff_at(S, head_of(S, (uint32_t)q))) continue;  // homogeneous / not counting-sorted
        const uint32_t slot = S.gnp[q], base = S.K[slot], c = S.K[slot + 1] - base;
        const uint64_t o = S.T[q];
        uint32_t fin = (uint32_t)q;
        if (c > 1) {
            if ((uint32_t)q == base && c > maxg) maxg = c;
            if (c <= 8) {
                uint32_t rank = 0;
                for (uint32_t k = 0; k < c; k++) {
                    const uint64_t ok = S.T[base + k];
                    rank += (ok < o) || (ok == o && base + k < (uint32_t)q);
                }
                fin = base + rank;
            } else {
                if ((uint32_t)q == base) {
                    const uint32_t k = atomicAdd(&S.nbig, 1u);
                    if (k < BS_MAXBIG) S.big[k] = slot;
                    else S.ovf = 1;
                }
                continue;
            }
        }
        a.A[lo + fin] = from_ord<DT>(o);
    }
    maxg = (uint32_t)warp_max_u64(maxg);
    if (lane == 0 && maxg > 1) atomicMax(&S.st_maxg, (unsigned long long)maxg);
    __syncthreads();
    if (a.dbg == 5) return;
    // groups of > 8 keys: one warp each; all-equal groups are stored as they are
    const uint32_t nb = min(S.nbig, (uint32_t)BS_MAXBIG);
    for (uint32_t k = warp; k < nb + (S.ovf ? (uint32_t)span : 0u); k += bd >> 5) {
        uint32_t slot;
        if (k < nb) {
            slot = S.big[k];
        } else {  // overflow: scan all slots (rare)
            slot = k - nb;
            const uint32_t c = S.K[slot + 1] - S.K[slot];
            if (c <= 8 || !diff_at(S, head_of(S, S.K[slot]))) continue;
            bool listed = false;
            for (uint32_t q = 0; q < nb; q++) listed |= (S.big[q] == slot);
            if (listed) continue;
        }
        const uint32_t base = S.K[slot], c = S.K[slot + 1] - base;
        if (c <= 32) {  // register bitonic network across the warp (one key per lane)
            uint64_t v = (uint32_t)lane < c ? S.T[base + lane] : ~0ull;
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
                for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                    const uint64_t w = __shfl_xor_sync(0xffffffffu, v, jj);
                    const bool keep_min = ((lane & jj) == 0) == ((lane & kk) == 0);
                    v = keep_min ? (w < v ? w : v) : (w > v ? w : v);
                }
            }
            if ((uint32_t)lane < c) a.A[lo + base + lane] = from_ord<DT>(v);
            continue;
        }
        bool same = true;
        for (uint32_t q = lane; q < c; q += 32) same &= (S.T[base + q] == S.T[base]);
        if (!__all_sync(0xffffffffu, same)) bitonic<DT_U64, false>(S.T + base, (int)c, lane, 32);
        for (uint32_t q = lane; q < c; q += 32) a.A[lo + base + q] = from_ord<DT>(S.T[base + q]);
    }
    if (a.dbg == 6) return;
    // per sub-bucket classification: H1 or counting-sorted
    for (uint32_t g = g0 + tid; g <= g1; g += bd) {
        const uint32_t np = __ldg(&a.hist1[g]);
        if (np < 2) continue;
        if (diff_at(S, __ldg(&a.start1[g]) - lo)) {
            atomicAdd(&S.st_small, 1ull);
            atomicAdd(&S.st_smallk, (unsigned long long)np);
        } else {
            if (a.dH1) a.dH1[g] = 1;
            atomicAdd(&S.st_h1, 1ull);
            atomicAdd(&S.st_h1k, (unsigned long long)np);
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (S.st_small) atomicAdd(&a.ctl->stat[ST_SMALLS], S.st_small);
        if (S.st_smallk) atomicAdd(&a.ctl->stat[ST_SMALLK], S.st_smallk);
        if (S.st_h1) atomicAdd(&a.ctl->stat[ST_H1S], S.st_h1);
        if (S.st_h1k) atomicAdd(&a.ctl->stat[ST_H1K], S.st_h1k);
        if (S.st_maxg) atomicMax(&a.ctl->stat[ST_MAXGRP], S.st_maxg);
    }
}

// {g0, g1, lo, hi} per bucket-sort window: one dependent load per CTA instead
// of two chained ones on the critical path of every tile.
__global__ void k_tile_desc(Args a) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.ntiles) return;
    const uint32_t g0 = a.tile_first[t];
    uint4 d = make_uint4(0xffffffffu, 0u, 0u, 0u);
    if (g0 != 0xffffffffu) {
        const uint32_t g1 = a.tile_last[t];
        d = make_uint4(g0, g1, a.start1[g0], a.start1[g1] + a.hist1[g1]);
    }
    a.tdesc[t] = d;
}

// ------------------------------------------------------------- BIG path ----
constexpr int BIG_THREADS = 512;
constexpr int BIG_DIGITS = 4096;       // 12-bit MSD digits
constexpr int BIG_SORT_CAP = 8192;     // keys sorted in shared memory by one CTA
constexpr int BIG_CHUNK = BIG_SORT_CAP / 2;
constexpr int BIG_MAXWIN = 1024;       // windows classified per round
constexpr int BIG_MAXBLK = 64;         // pieces in (BIG_CHUNK, BIG_SORT_CAP] per item

// ord min/max of level-0 big items, one 64K-key chunk per work entry
// (classify wrote the chunk list), so a multi-million-key homogeneous
// sub-bucket (Zipf's top value, config 4's top level) is scanned by the whole
// GPU instead of one CTA.
template <int DT>
__global__ void __launch_bounds__(512) k_big_minmax(Args a) {
    if (a.ctl->status) return;
    __shared__ unsigned long long red[64];
    const uint32_t nch = min(a.ctl->nchunks, a.chunk_cap);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t e = blockIdx.x; e < nch; e += gridDim.x) {
        const BigChunk ch = a.chunks[e];
        const BigItem item = a.big[ch.item];
        const uint32_t beg = ch.chunk * MM_CHUNK, end = min(item.size, beg + MM_CHUNK);
        const uint64_t *X = a.A + item.off;
        unsigned long long mn = ~0ull, mx = 0;
        for (uint32_t i = beg + threadIdx.x; i < end; i += 4 * blockDim.x) {
            uint64_t v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = (i + q * blockDim.x < end) ? X[i + q * blockDim.x] : X[beg];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const unsigned long long o = to_ord<DT>(v[q]);
                mn = o < mn ? o : mn;
                mx = o > mx ? o : mx;
            }
        }
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        if ((threadIdx.x & 31) == 0) {
            red[w] = mn;
            red[32 + w] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < nw; k++) {
                mn = red[k] < mn ? red[k] : mn;
                mx = red[32 + k] > mx ? red[32 + k] : mx;
            }
            atomicMin(&a.big[ch.item].mn, mn);
            atomicMax(&a.big[ch.item].mx, mx);
        }
        __syncthreads();
    }
}

template <int DT>
__device__ void big_minmax(const uint64_t *X, uint32_t size, unsigned long long &mn,
                           unsigned long long &mx, unsigned long long *red) {
    mn = ~0ull;
    mx = 0;
    for (uint32_t i = threadIdx.x; i < size; i += 4 * blockDim.x) {
        uint64_t v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = (i + q * blockDim.x < size) ? X[i + q * blockDim.x] : X[0];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const unsigned long long o = to_ord<DT>(v[q]);
            mn = o < mn ? o : mn;
            mx = o > mx ? o : mx;
        }
    }
    mn = warp_min_u64(mn);
    mx = warp_max_u64(mx);
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[w] = mn;
        red[32 + w] = mx;
    }
    __syncthreads();
    mn = red[0];
    mx = red[32];
    for (int i = 1; i < nw; i++) {
        mn = red[i] < mn ? red[i] : mn;
        mx = red[32 + i] > mx ? red[32 + i] : mx;
    }
    __syncthreads();
}

struct BigSmem {
    uint64_t sk[BIG_SORT_CAP];
    uint32_t start[BIG_DIGITS], end[BIG_DIGITS];
    uint32_t wlo[BIG_MAXWIN], whi[BIG_MAXWIN];
    uint32_t blk[BIG_MAXBLK];
    uint32_t tmp[36];
    uint32_t item, nblk;
    unsigned long long red[64];
};

// One CTA per big item of this level: MSD radix partition X -> Y on the top
// 12 bits of ord - min, then every piece is sorted exactly in shared memory
// and written to A. Pieces <= BIG_CHUNK are gathered in windows of
// BIG_CHUNK positions (a window owns the pieces starting in it, so its span
// is <= BIG_SORT_CAP): one thread per piece of <= 16 keys (insertion sort),
// one warp per larger piece (bitonic). Pieces in (BIG_CHUNK, BIG_SORT_CAP]
// are block-sorted; larger ones become items of the next level.
template <int DT>
__global__ void __launch_bounds__(BIG_THREADS, 2) k_big(Args a, int level) {
    if (a.ctl->status) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BigSmem &S = *reinterpret_cast<BigSmem *>(smem_raw);
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;
    const uint32_t cnt = min(a.ctl->big_cnt[level], a.big_cap);
    const BigItem *list = a.big + (size_t)level * a.big_cap;
    for (;;) {
        if (tid == 0) S.item = atomicAdd(&a.ctl->big_next[level], 1u);
        __syncthreads();
        const uint32_t it = S.item;
        __syncthreads();
        if (it >= cnt) break;
        const BigItem item = list[it];
        const uint64_t *X = (item.in_b ? a.B : a.A) + item.off;
        uint64_t *Y = (item.in_b ? a.A : a.B) + item.off;
        uint64_t *Aout = a.A + item.off;
        unsigned long long mn, mx;
        if (level == 0) {
            mn = item.mn;
            mx = item.mx;
        } else {
            big_minmax<DT>(X, item.size, mn, mx, S.red);
        }
        if (mn == mx) {  // homogeneous: already final
            if (item.in_b)
                for (uint32_t i = tid; i < item.size; i += bd) Aout[i] = X[i];
            if (tid == 0 && level == 0) {
                if (a.dH1) a.dH1[item.g] = 1;
                atomicAdd(&a.ctl->stat[ST_H1S], 1ull);
                atomicAdd(&a.ctl->stat[ST_H1K], (unsigned long long)item.size);
            }
            __syncthreads();
            continue;
        }
        if (tid == 0) {
            if (level == 0) {
                atomicAdd(&a.ctl->stat[ST_BIGS], 1ull);
                atomicAdd(&a.ctl->stat[ST_BIGK], (unsigned long long)item.size);
            }
            atomicAdd(&a.ctl->stat[ST_BIGPASS], 1ull);
        }
        if (item.size <= BIG_SORT_CAP) {
            for (uint32_t i = tid; i < item.size; i += bd) S.sk[i] = X[i];
            __syncthreads();
            bitonic<DT, true>(S.sk, (int)item.size, tid, bd);
            for (uint32_t i = tid; i < item.size; i += bd) Aout[i] = S.sk[i];
            __syncthreads();
            continue;
        }
        // MSD radix partition X -> Y on the top 12 bits of ord - mn
        const unsigned long long range = mx - mn;
        const int bits = 64 - __clzll((long long)range);
        const int shift = bits > 12 ? bits - 12 : 0;
        for (int d = tid; d < BIG_DIGITS; d += bd) S.start[d] = 0;
        if (tid == 0) S.nblk = 0;
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
        block_exscan(S.start, BIG_DIGITS, S.tmp);
        for (int d = tid; d < BIG_DIGITS; d += bd) S.end[d] = S.start[d];
        __syncthreads();
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
        __syncthreads();  // S.end[d] = end of piece d; Y holds the pieces
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
                    } else if (level + 1 < BIG_LEVELS) {  // next level
                        const uint32_t q = atomicAdd(&a.ctl->big_cnt[level + 1], 1u);
                        if (q < a.big_cap)
                            a.big[(size_t)(level + 1) * a.big_cap + q] =
                                BigItem{item.off + ps, pc, y_is_b ? 1u : 0u, ~0u, ~0ull, 0ull, 0u, 0u};
                        else
                            atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
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
                for (uint32_t i = tid; i < shi - slo; i += bd) S.sk[i] = Y[slo + i];
                __syncthreads();
                for (uint32_t d = dlo + tid; d <= dhi; d += bd) {  // one thread per tiny piece
                    const uint32_t pc = S.end[d] - S.start[d];
                    if (pc >= 2 && pc <= 16) insertion_sort<DT>(S.sk + (S.start[d] - slo), (int)pc);
                }
                for (uint32_t d = dlo + warp; d <= dhi; d += nwarps) {  // one warp per larger piece
                    const uint32_t pc = S.end[d] - S.start[d];
                    if (pc > 16 && pc <= BIG_CHUNK)
                        bitonic<DT, false>(S.sk + (S.start[d] - slo), (int)pc, lane, 32);
                }
                __syncthreads();
                for (uint32_t i = tid; i < shi - slo; i += bd) Aout[slo + i] = S.sk[i];
                __syncthreads();
            }
        }
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
    }
}

// -------------------------------------------------------------- launchers --
void launch_bucketsort(const Args &a, int dtype, cudaStream_t st) {
    k_tile_desc<<<(a.ntiles + 255) / 256, 256, 0, st>>>(a);
    const size_t sm = sizeof(BsSmem);
    if (dtype == DT_F64) {
        cudaFuncSetAttribute(k_bucketsort<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_bucketsort<DT_F64><<<a.ntiles, BS_THREADS, sm, st>>>(a);
    } else {
        cudaFuncSetAttribute(k_bucketsort<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_bucketsort<DT_U64><<<a.ntiles, BS_THREADS, sm, st>>>(a);
    }
}

void launch_big_minmax(const Args &a, int dtype, cudaStream_t st) {
    if (dtype == DT_F64) k_big_minmax<DT_F64><<<148 * 4, 512, 0, st>>>(a);
    else k_big_minmax<DT_U64><<<148 * 4, 512, 0, st>>>(a);
}

void launch_big(const Args &a, int level, int dtype, cudaStream_t st) {
    const size_t sm = sizeof(BigSmem);
    const int grid = 148 * 2;
    if (dtype == DT_F64) {
        cudaFuncSetAttribute(k_big<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_big<DT_F64><<<grid, BIG_THREADS, sm, st>>>(a, level);
    } else {
        cudaFuncSetAttribute(k_big<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_big<DT_U64><<<grid, BIG_THREADS, sm, st>>>(a, level);
    }
}

}  // namespace ls
