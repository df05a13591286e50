// ls_tile.cuh -- the two halves of one partition round, shared by the model
// rounds (ls_partition.cu) and the multi-GPU destination split (ls_multi.cu).
#pragma once
#include "ls_common.cuh"

namespace ls {

// Decoupled lookback for one (unit, bin): publish the unit's aggregate, walk
// predecessors until an inclusive prefix is found, publish the inclusive
// prefix. Flag and value share one 64-bit word, so a single store publishes
// both. Predecessors hold lower tickets, so they are resident or finished and
// the spin terminates. `first_u` is the first unit of the segment.
__device__ __forceinline__ uint32_t lookback(unsigned long long *lb, uint64_t u, uint64_t first_u,
                                             int nb, int b, uint32_t c) {
    unsigned long long *my = lb + u * nb + b;
    if (u == first_u) {
        st_volatile(my, LB_FLAG_P | c);
        return 0;
    }
    st_volatile(my, LB_FLAG_A | c);
    uint32_t excl = 0;
    uint64_t k = u - 1;
    for (;;) {
        const unsigned long long w = ld_volatile(lb + k * nb + b);
        const unsigned long long flag = w & ~LB_VALUE;
        if (flag == 0) {
            __nanosleep(20);
            continue;
        }
        excl += (uint32_t)(w & LB_VALUE);
        if (flag == LB_FLAG_P) break;
        k--;
    }
    st_volatile(my, LB_FLAG_P | (unsigned long long)(excl + c));
    return excl;
}

// Tile-local counting sort + coalesced scatter of src[beg, end) into nb
// buckets. base[b] is the unit's global write cursor of bucket b (advanced
// here). Per tile: bucket ids and ranks via shared-memory atomics, exclusive
// scan, reorder into shared memory, then consecutive threads store
// consecutive keys of each bucket run.
template <int KPT, class BF>
__device__ __forceinline__ void tile_scatter(const uint64_t *__restrict__ src,
                                             uint64_t *__restrict__ dst, uint64_t beg,
                                             uint64_t end, uint32_t *base, uint32_t *cnt,
                                             uint32_t *tst, uint64_t *skeys, uint16_t *sbin,
                                             uint32_t *tmp, int nb, const BF &bf) {
    const int bd = blockDim.x, tid = threadIdx.x;
    const int T = KPT * bd;
    for (uint64_t t0 = beg; t0 < end; t0 += T) {
        const int tn = (int)umin64((uint64_t)T, end - t0);
        for (int b = tid; b < nb; b += bd) cnt[b] = 0;
        __syncthreads();
        uint64_t key[KPT];
        uint32_t bk[KPT], rk[KPT];
#pragma unroll
        for (int i = 0; i < KPT; i++) {
            const int idx = i * bd + tid;
            if (idx < tn) key[i] = src[t0 + idx];
        }
#pragma unroll
        for (int i = 0; i < KPT; i++) {
            const int idx = i * bd + tid;
            if (idx < tn) {
                bk[i] = bf(key[i], t0 + idx);
                rk[i] = atomicAdd(&cnt[bk[i]], 1u);
            }
        }
        __syncthreads();
        for (int b = tid; b < nb; b += bd) tst[b] = cnt[b];
        __syncthreads();
        block_exscan(tst, nb, tmp);
#pragma unroll
        for (int i = 0; i < KPT; i++) {
            const int idx = i * bd + tid;
            if (idx < tn) {
                const uint32_t pos = tst[bk[i]] + rk[i];
                skeys[pos] = key[i];
                sbin[pos] = (uint16_t)bk[i];
            }
        }
        __syncthreads();
        for (int idx = tid; idx < tn; idx += bd) {
            const uint32_t b = sbin[idx];
            dst[base[b] + (uint32_t)idx - tst[b]] = skeys[idx];
        }
        __syncthreads();
        for (int b = tid; b < nb; b += bd) base[b] += cnt[b];
    }
}

}  // namespace ls
