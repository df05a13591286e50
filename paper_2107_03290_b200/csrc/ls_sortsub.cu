// ls_sortsub.cu -- north_star (3)+(4): in-bucket sort with duplicate handling.
//
// SMALL sub-buckets (2 <= n' <= T_small): Alg. 2's model-based counting sort
// in shared memory -- pos per key (R5), histogram K, exclusive
// running totals, placement (R4) -- followed by the touch-up. Because p is
// monotone (R15) the only disorder left after the counting sort is inside runs
// of equal pos ("collision groups"), so the global insertion sort of P:219 is
// replaced by sorting every collision group independently: the paper's
// insertion sort by one lane for groups <= 16 keys, a warp bitonic network for
// larger ones. Homogeneous sub-buckets (min == max) are skipped.
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
// One CTA per window of T_tile key positions; it owns every SMALL sub-bucket
// that starts in the window (classify recorded the first/last one), so its
// span is at most T_tile + T_small keys. One warp per sub-bucket.
template <int DT>
__global__ void __launch_bounds__(256) k_bucketsort(Args a) {
    if (a.ctl->status) return;
    const uint32_t t = blockIdx.x;
    const uint32_t g0 = a.tile_first[t];
    if (g0 == 0xffffffffu) return;
    const uint32_t g1 = a.tile_last[t];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int span_cap = a.T_tile + a.T_small;
    uint64_t *skeys = (uint64_t *)smem_raw;
    uint64_t *stmp = skeys + span_cap;
    uint32_t *sK = (uint32_t *)(stmp + span_cap);
    uint32_t *spr = sK + span_cap;
    __shared__ unsigned long long s_stat[5];
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;
    if (tid < 5) s_stat[tid] = 0;
    const uint32_t lo = a.start1[g0];
    const uint32_t hi = a.start1[g1] + a.hist1[g1];
    for (uint32_t i = tid; i < hi - lo; i += bd) skeys[i] = a.A[lo + i];
    __syncthreads();
    const Root R = load_root(a.M);
    const int f = a.f;
    unsigned long long st_small = 0, st_smallk = 0, st_h1 = 0, st_h1k = 0, st_maxg = 0;
    for (uint32_t g = g0 + warp; g <= g1; g += nwarps) {
        const uint32_t np = a.hist1[g];
        if (np < 2 || np > a.T_small) continue;
        const uint32_t s = a.start1[g];
        const uint32_t off = s - lo;
        uint64_t *K = skeys + off;
        uint64_t *T = stmp + off;
        uint32_t *cK = sK + off;
        uint32_t *pr = spr + off;
        // Is-Homogeneous
        unsigned long long mn = ~0ull, mx = 0;
        for (uint32_t k = lane; k < np; k += 32) {
            const unsigned long long o = to_ord<DT>(K[k]);
            mn = o < mn ? o : mn;
            mx = o > mx ? o : mx;
        }
        mn = warp_min_u64(mn);
        mx = warp_max_u64(mx);
        if (mn == mx) {
            if (lane == 0) {
                if (a.dH1) a.dH1[g] = 1;
                st_h1++;
                st_h1k += np;
            }
            continue;
        }
        // Model-based counting sort
        for (uint32_t k = lane; k < np; k += 32) cK[k] = 0;
        __syncwarp();
        const double adj = __ddiv_rn((double)g, a.F2);  // (i*f + j)/f^2
        const double top = (double)(np - 1);
        for (uint32_t k = lane; k < np; k += 32) {
            const double p = predict_ldg<DT>(K[k], R, a.M->leaf);
            const uint32_t pos = cs_pos(p, adj, a.nd, top);
            const uint32_t r = atomicAdd(&cK[pos], 1u);
            pr[k] = pos | (r << 16);
        }
        __syncwarp();
        uint32_t carry = 0;  // running totals, exclusive form (R4)
        for (uint32_t base = 0; base < np; base += 32) {
            const uint32_t k = base + lane;
            const uint32_t v = k < np ? cK[k] : 0;
            const uint32_t incl = warp_incl_scan(v);
            if (k < np) cK[k] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        __syncwarp();
        for (uint32_t k = lane; k < np; k += 32) {  // placement
            const uint32_t q = pr[k];
            T[cK[q & 0xffffu] + (q >> 16)] = K[k];
        }
        __syncwarp();
        // Touch-up per collision group (R15)
        uint32_t maxg = 0;
        for (uint32_t base = 0; base < np; base += 32) {
            const uint32_t k = base + lane;
            uint32_t c = 0, st = 0;
            if (k < np) {
                st = cK[k];
                c = (k + 1 < np ? cK[k + 1] : np) - st;
            }
            maxg = c > maxg ? c : maxg;
            if (c >= 2 && c <= 16) insertion_sort<DT>(T + st, (int)c);
            unsigned big = __ballot_sync(0xffffffffu, c > 16);
            while (big) {
                const int leader = __ffs(big) - 1;
                const uint32_t bst = __shfl_sync(0xffffffffu, st, leader);
                const uint32_t bc = __shfl_sync(0xffffffffu, c, leader);
                bitonic<DT, false>(T + bst, (int)bc, lane, 32);
                big &= big - 1;
            }
            __syncwarp();
        }
        for (uint32_t k = lane; k < np; k += 32) a.A[s + k] = T[k];
        maxg = (uint32_t)warp_max_u64(maxg);
        if (lane == 0) {
            st_small++;
            st_smallk += np;
            st_maxg = maxg > st_maxg ? maxg : st_maxg;
        }
    }
    if (lane == 0) {
        if (st_small) atomicAdd(&s_stat[0], st_small);
        if (st_smallk) atomicAdd(&s_stat[1], st_smallk);
        if (st_h1) atomicAdd(&s_stat[2], st_h1);
        if (st_h1k) atomicAdd(&s_stat[3], st_h1k);
        if (st_maxg) atomicMax(&s_stat[4], st_maxg);
    }
    __syncthreads();
    if (tid == 0) {
        if (s_stat[0]) atomicAdd(&a.ctl->stat[ST_SMALLS], s_stat[0]);
        if (s_stat[1]) atomicAdd(&a.ctl->stat[ST_SMALLK], s_stat[1]);
        if (s_stat[2]) atomicAdd(&a.ctl->stat[ST_H1S], s_stat[2]);
        if (s_stat[3]) atomicAdd(&a.ctl->stat[ST_H1K], s_stat[3]);
        if (s_stat[4]) atomicMax(&a.ctl->stat[ST_MAXGRP], s_stat[4]);
    }
}

// ------------------------------------------------------------- BIG path ----
constexpr int BIG_THREADS = 512;
constexpr int BIG_DIGITS = 4096;       // 12-bit MSD digits
constexpr int BIG_SORT_CAP = 8192;     // keys sorted in shared memory by one CTA
constexpr int BIG_CHUNK = BIG_SORT_CAP / 2;

template <int DT>
__device__ void big_minmax(const uint64_t *X, uint32_t size, unsigned long long &mn,
                           unsigned long long &mx, unsigned long long *red) {
    mn = ~0ull;
    mx = 0;
    for (uint32_t i = threadIdx.x; i < size; i += blockDim.x) {
        const unsigned long long o = to_ord<DT>(X[i]);
        mn = o < mn ? o : mn;
        mx = o > mx ? o : mx;
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

template <int DT>
__global__ void __launch_bounds__(BIG_THREADS) k_big(Args a, int level) {
    if (a.ctl->status) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint64_t *sk = (uint64_t *)smem_raw;                 // [BIG_SORT_CAP]
    uint32_t *hist = (uint32_t *)(sk + BIG_SORT_CAP);    // [BIG_DIGITS]
    uint32_t *cur = hist + BIG_DIGITS;                   // [BIG_DIGITS]
    __shared__ unsigned long long red[64];
    __shared__ uint32_t tmp[33];
    __shared__ uint32_t s_item, s_dlo, s_dhi;
    const int tid = threadIdx.x, bd = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = bd >> 5;
    const uint32_t cnt = min(a.ctl->big_cnt[level], a.big_cap);
    const BigItem *list = a.big + (size_t)level * a.big_cap;
    for (;;) {
        if (tid == 0) s_item = atomicAdd(&a.ctl->big_next[level], 1u);
        __syncthreads();
        const uint32_t it = s_item;
        __syncthreads();
        if (it >= cnt) break;
        const BigItem item = list[it];
        uint64_t *X = (item.in_b ? a.B : a.A) + item.off;
        uint64_t *Y = (item.in_b ? a.A : a.B) + item.off;
        uint64_t *Aout = a.A + item.off;
        unsigned long long mn, mx;
        big_minmax<DT>(X, item.size, mn, mx, red);
        if (mn == mx) {  // homogeneous: already final
            if (item.in_b)
                for (uint32_t i = tid; i < item.size; i += bd) Aout[i] = X[i];
            if (tid == 0 && level == 0) {
                if (a.dH1) a.dH1[item.g] = 1;
                atomicAdd(&a.ctl->stat[ST_H1S], 1ull);
                atomicAdd(&a.ctl->stat[ST_H1K], (unsigned long long)item.size);
            }
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
            for (uint32_t i = tid; i < item.size; i += bd) sk[i] = X[i];
            __syncthreads();
            bitonic<DT, true>(sk, (int)item.size, tid, bd);
            for (uint32_t i = tid; i < item.size; i += bd) Aout[i] = sk[i];
            __syncthreads();
            continue;
        }
        // MSD radix partition X -> Y on the top 12 bits of ord - mn
        const unsigned long long range = mx - mn;
        const int bits = 64 - __clzll((long long)range);
        const int shift = bits > 12 ? bits - 12 : 0;
        for (int d = tid; d < BIG_DIGITS; d += bd) hist[d] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < item.size; i += bd)
            atomicAdd(&hist[(uint32_t)((to_ord<DT>(X[i]) - mn) >> shift)], 1u);
        __syncthreads();
        for (int d = tid; d < BIG_DIGITS; d += bd) cur[d] = hist[d];
        __syncthreads();
        block_exscan(cur, BIG_DIGITS, tmp);  // cur = piece starts
        // keep starts in `hist` after the scatter: hist[d] = start, sizes from neighbours
        for (int d = tid; d < BIG_DIGITS; d += bd) {
            const uint32_t c = hist[d];
            hist[d] = cur[d];
            (void)c;
        }
        __syncthreads();
        for (uint32_t i = tid; i < item.size; i += bd) {
            const uint64_t key = X[i];
            const uint32_t d = (uint32_t)((to_ord<DT>(key) - mn) >> shift);
            Y[atomicAdd(&cur[d], 1u)] = key;
        }
        __syncthreads();
        // now hist[d] = start of piece d, cur[d] = end of piece d
        const bool y_is_b = !item.in_b;
        // (a) pieces larger than BIG_CHUNK: sort in shared memory or defer
        for (int d = 0; d < BIG_DIGITS; d++) {
            const uint32_t ps = hist[d], pc = cur[d] - hist[d];
            if (pc <= BIG_CHUNK) continue;
            if (pc <= BIG_SORT_CAP) {
                for (uint32_t i = tid; i < pc; i += bd) sk[i] = Y[ps + i];
                __syncthreads();
                bitonic<DT, true>(sk, (int)pc, tid, bd);
                for (uint32_t i = tid; i < pc; i += bd) Aout[ps + i] = sk[i];
                __syncthreads();
            } else if (tid == 0) {
                if (level + 1 < BIG_LEVELS) {
                    const uint32_t k = atomicAdd(&a.ctl->big_cnt[level + 1], 1u);
                    if (k < a.big_cap)
                        a.big[(size_t)(level + 1) * a.big_cap + k] =
                            BigItem{item.off + ps, pc, y_is_b ? 1u : 0u, ~0u};
                    else
                        atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
                } else {
                    atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
                }
            }
        }
        // (b) pieces <= BIG_CHUNK, in windows of BIG_CHUNK positions: a window
        // owns the pieces starting in it (span <= 2*BIG_CHUNK = BIG_SORT_CAP)
        const uint32_t nwin = (item.size + BIG_CHUNK - 1) / BIG_CHUNK;
        for (uint32_t w = 0; w < nwin; w++) {
            const uint32_t wlo = w * BIG_CHUNK, whi = wlo + BIG_CHUNK;
            if (tid == 0) {
                int dlo = BIG_DIGITS, dhi = -1;
                for (int d = 0; d < BIG_DIGITS; d++) {  // short scan: monotone starts
                    const uint32_t ps = hist[d], pc = cur[d] - ps;
                    if (ps >= whi) break;
                    if (ps < wlo || pc == 0 || pc > BIG_CHUNK) continue;
                    if (d < dlo) dlo = d;
                    dhi = d;
                }
                s_dlo = (uint32_t)dlo;
                s_dhi = (uint32_t)dhi;
            }
            __syncthreads();
            const int dlo = (int)s_dlo, dhi = (int)s_dhi;
            if (dhi >= dlo) {
                const uint32_t slo = hist[dlo], shi = cur[dhi];
                for (uint32_t i = tid; i < shi - slo; i += bd) sk[i] = Y[slo + i];
                __syncthreads();
                for (int d = dlo + tid; d <= dhi; d += bd) {  // tiny pieces: one lane each
                    const uint32_t pc = cur[d] - hist[d];
                    if (pc >= 2 && pc <= 16) insertion_sort<DT>(sk + (hist[d] - slo), (int)pc);
                }
                for (int d = dlo + warp; d <= dhi; d += nwarps) {  // larger: one warp each
                    const uint32_t pc = cur[d] - hist[d];
                    if (pc > 16 && pc <= BIG_CHUNK)
                        bitonic<DT, false>(sk + (hist[d] - slo), (int)pc, lane, 32);
                }
                __syncthreads();
                for (uint32_t i = tid; i < shi - slo; i += bd) Aout[slo + i] = sk[i];
            }
            __syncthreads();
        }
    }
}

// -------------------------------------------------------------- launchers --
void launch_bucketsort(const Args &a, int dtype, cudaStream_t st) {
    const size_t span = a.T_tile + a.T_small;
    const size_t sm = span * (8 + 8 + 4 + 4);
    if (dtype == DT_F64) {
        cudaFuncSetAttribute(k_bucketsort<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_bucketsort<DT_F64><<<a.ntiles, 256, sm, st>>>(a);
    } else {
        cudaFuncSetAttribute(k_bucketsort<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_bucketsort<DT_U64><<<a.ntiles, 256, sm, st>>>(a);
    }
}

void launch_big(const Args &a, int level, int dtype, cudaStream_t st) {
    const size_t sm = BIG_SORT_CAP * 8 + 2 * BIG_DIGITS * 4;
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
