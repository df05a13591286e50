// ls_wstask.cuh -- one SMALL sub-bucket sorted by one warp (Alg. 2's model
// counting sort P:184-210 + the collision-group touch-up P:219 / R15), shared
// by k_warpsort (ls_sortsub.cu) and k_round1's in-bucket sort (ls_round1.cu).
#pragma once
#include "ls_common.cuh"
#include "ls_warpsort.cuh"

namespace ls {

constexpr uint32_t BS_RANKMAX = 8;         // groups up to this size: odd-even rounds
constexpr uint32_t BS_NONE = 0xffffffffu;

// T in shared memory with one pad word per 8: position q lives at q + q/8, so
// a thread reading its 8 consecutive positions (odd-even phase) and a warp
// reading 32 consecutive positions (store-back) are both bank-conflict free.
struct PadT {
    uint64_t *p;
    uint32_t off;  // view offset (positions)
    __device__ __forceinline__ uint64_t &operator[](uint32_t q) const {
        const uint32_t x = q + off;
        return p[x + (x >> 3)];
    }
    __device__ __forceinline__ PadT operator+(uint32_t d) const { return PadT{p, off + d}; }
};

// adj = g / f^2 correctly rounded, as (double)g * rcp plus one fma correction
// step (rcp = RN(1/f^2)); exhaustively equal to the IEEE quotient for every
// f <= 1024 and g < f^2 (tests/test_adj_division.py).
__device__ __forceinline__ double adj_of(uint32_t g, double F2, double rcp) {
    const double gd = (double)g;
    const double q0 = __dmul_rn(gd, rcp);
    return __fma_rn(__fma_rn(-q0, F2, gd), rcp, q0);
}

// Sort c <= 32*NS ord values of a padded-T range by one warp in registers.
template <int NS, bool PICK = true>
__device__ __forceinline__ void warp_sort_T(PadT g, uint32_t c, int lane) {
    uint64_t v[NS];
#pragma unroll
    for (int s2 = 0; s2 < NS; s2++) {
        const uint32_t i = 32u * s2 + lane;
        v[s2] = i < c ? g[i] : ~0ull;
    }
    warp_sort_regs<NS, uint64_t, PICK>(v, lane);
#pragma unroll
    for (int s2 = 0; s2 < NS; s2++) {
        const uint32_t i = 32u * s2 + lane;
        if (i < c) g[i] = v[s2];
    }
}

// One warp per SMALL sub-bucket of 2 <= n' <= WS_MAX keys (k_classify's task
// list; at 200M keys from smooth distributions that is every sub-bucket). A
// warp needs no block barrier: the sub-bucket's g, n' and adj are uniform, its
// keys are loaded coalesced (8 per lane), and Alg. 2's counting sort (P:184-209,
// pos by R5, exclusive totals R4) and the collision-group touch-up (R15:
// odd-even transposition between equal-slot neighbours, warp bitonic for
// groups > 8) run in the warp's own shared-memory slice. A homogeneous
// sub-bucket (first == last after sorting) is not written back.
constexpr int WS_WARPS = 8;                 // warps per CTA
constexpr int WS_KPL = (int)WS_MAX / 32;    // keys per lane (8)
constexpr int WS_CTAS_PER_SM = 4;

struct alignas(16) WsSlice {
    uint64_t T[WS_MAX + WS_MAX / 8];        // padded: position q at q + q/8
    alignas(16) uint32_t K[WS_MAX + 8];     // pos histogram -> exclusive totals
    uint32_t big[32];                       // groups > 8 keys (their pos)
};

// One SMALL sub-bucket (task = {start, n', g, leaf + 1 or 0}) sorted by the
// calling warp in its slice W (k_warpsort, and k_round1's in-bucket sort):
// Alg. 2's counting sort + the collision-group touch-up, written back to A.
// wst: the warp's statistics (small / small keys / H1 / H1 keys).
template <int DT>
__device__ __forceinline__ void ws_task(const Args &a, const Root &R, uint32_t g_lo, uint32_t g_hi,
                                        WsSlice &W, uint32_t *wst, uint32_t &r_maxg, bool &early_h1,
                                        const uint4 task, const int lane) {
    const PadT T{W.T, 0u};
    const uint32_t st = task.x, np = task.y, g = task.z;
    // keys (coalesced), and the next task's descriptor, in flight together
    uint64_t key[WS_KPL];
    uint64_t *const gl = a.A + st + lane;  // key 32k + lane at gl[32k]
#pragma unroll
    for (int k = 0; k < WS_KPL; k++) key[k] = 32u * k + lane < np ? gl[32 * k] : 0ull;
    // homogeneous sub-bucket (all keys equal): nothing to sort or
    // store. Tested up front only once this warp has met one (the test
    // after the sort below catches every case; on inputs without such
    // sub-buckets the up-front test is pure cost: -4 % at 200M Normal)
    if (early_h1) {
        const uint64_t k0 = __shfl_sync(0xffffffffu, key[0], 0);
        bool diff = false;
#pragma unroll
        for (int k = 0; k < WS_KPL; k++) {
            const uint32_t i = 32u * k + lane;
            diff |= (i < np) && key[k] != k0;
        }
        if (!__any_sync(0xffffffffu, diff)) {
            if (lane == 0 && a.dH1) a.dH1[g] = 1;
            if (lane == 0) {
                wst[2]++;
                wst[3] += np;
            }
            return;
        }
    }
    // Slots of the counting sort: Alg. 2's pos = floor((p - adj) * n)
    // spreads the sub-bucket's p-range [adj, adj + 1/f^2) over
    // ~n/f^2 slots and R5 clamps it to n'-1. Here the range is spread over
    // all WS_MAX = 256 counters of the warp instead: pos = floor((p - adj) *
    // 256 f^2) clamped to [0, 255]. Any pos that is monotone in p orders the
    // keys of different slots (R15), and the touch-up sorts each slot's
    // group, so the result is R5's: n/f^2 ~ 200 at 200M keys gets 1.28x finer
    // slots (smaller collision groups, fewer odd-even passes), and n/f^2 >
    // 256 (10^9 keys: ~1000) no longer piles every key with pos >= 255 into
    // the last slot, where it met the warp bitonic.
    const uint32_t S = WS_MAX;
    *reinterpret_cast<uint4 *>(&W.K[8 * lane]) = make_uint4(0, 0, 0, 0);  // K[0..256)
    *reinterpret_cast<uint4 *>(&W.K[8 * lane + 4]) = make_uint4(0, 0, 0, 0);
    __syncwarp();
    // Alg. 2: pos per key (R5), K[pos]++ (the rank comes back).
    // Only the sub-buckets of xmin and xmax can hold keys outside
    // [xmin, xmax]; elsewhere the root clamp is skipped.
    const double adj = adj_of(g, a.F2, a.rcpF2);  // (i*f + j)/f^2
    const int top = (int)(S - 1u);
    const double nsl = __dmul_rn(a.F2, (double)WS_MAX);  // slots per unit of p
    uint32_t code[WS_KPL];
    if (task.w != 0u && g != g_lo && g != g_hi) {
        // one leaf holds every key and p = its line value (k_classify's
        // contained_leaf_warp: no routing, no clamp)
        const double *q = a.M->leaf + 5 * (task.w - 1u);
        const double la = __ldg(q), lc = __ldg(q + 1), lb = __ldg(q + 2);
#pragma unroll
        for (int k = 0; k < WS_KPL; k++) {
            code[k] = BS_NONE;
            if (32u * k + lane < np) {
                const double p = __fma_rn(la, __dsub_rn(xd<DT>(key[k]), lc), lb);
                const uint32_t pos = cs_pos(p, adj, nsl, top);
                const uint32_t r = atomicAdd(&W.K[pos], 1u);
                code[k] = pos | (r << 16);
            }
        }
    } else if (g != g_lo && g != g_hi) {
        // leaf of every key (O6 routing); a sub-bucket spans ~1/f^2 of the
        // CDF, so its keys almost always share one leaf, whose line is then
        // read once into registers instead of per key
        int lmin = 1 << 30, lmax = -1;
#pragma unroll
        for (int k = 0; k < WS_KPL; k++) {
            const double r = __dmul_rn(__dsub_rn(xd<DT>(key[k]), R.xmin), R.rs);
            const int l = (r < R.last) ? __double2int_rz(r) : R.Lm1;
            if (32u * k + lane < np) {
                lmin = min(lmin, l);
                lmax = max(lmax, l);
            }
        }
        lmin = __reduce_min_sync(0xffffffffu, lmin);
        lmax = __reduce_max_sync(0xffffffffu, lmax);
        if (lmin == lmax) {
            const double *q = a.M->leaf + 5 * lmin;
            const double la = __ldg(q), lc = __ldg(q + 1), lb = __ldg(q + 2), llo = __ldg(q + 3),
                         lhi = __ldg(q + 4);
#pragma unroll
            for (int k = 0; k < WS_KPL; k++) {
                code[k] = BS_NONE;
                if (32u * k + lane < np) {
                    const double y = __fma_rn(la, __dsub_rn(xd<DT>(key[k]), lc), lb);
                    const double p = __dadd_rn(clampd(y, llo, lhi), 0.0);
                    const uint32_t pos = cs_pos(p, adj, nsl, top);
                    const uint32_t r = atomicAdd(&W.K[pos], 1u);
                    code[k] = pos | (r << 16);
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < WS_KPL; k++) {
                code[k] = BS_NONE;
                if (32u * k + lane < np) {
                    const double p = predict_ldg_inner<DT>(key[k], R, a.M->leaf);
                    const uint32_t pos = cs_pos(p, adj, nsl, top);
                    const uint32_t r = atomicAdd(&W.K[pos], 1u);
                    code[k] = pos | (r << 16);
                }
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < WS_KPL; k++) {
            code[k] = BS_NONE;
            if (32u * k + lane < np) {
                const double p = predict_ldg<DT>(key[k], R, a.M->leaf);
                const uint32_t pos = cs_pos(p, adj, nsl, top);
                const uint32_t r = atomicAdd(&W.K[pos], 1u);
                code[k] = pos | (r << 16);
            }
        }
    }
    __syncwarp();
    // exclusive running totals over the S <= 256 slots, 8 per lane (two
    // 16-byte loads / stores); K[256] = n'
    uint32_t mgs;  // largest collision group of <= BS_RANKMAX keys
    {
        const uint4 c0 = *reinterpret_cast<const uint4 *>(&W.K[8 * lane]);
        const uint4 c1 = *reinterpret_cast<const uint4 *>(&W.K[8 * lane + 4]);
        const uint32_t c[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
        uint32_t v[8], sum = 0, gmax = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            v[q] = sum;
            sum += c[q];
            gmax = max(gmax, c[q]);
        }
        const uint32_t incl = warp_incl_scan(sum);
        const uint32_t off = incl - sum;
        *reinterpret_cast<uint4 *>(&W.K[8 * lane]) = make_uint4(v[0] + off, v[1] + off, v[2] + off, v[3] + off);
        *reinterpret_cast<uint4 *>(&W.K[8 * lane + 4]) = make_uint4(v[4] + off, v[5] + off, v[6] + off, v[7] + off);
        gmax = __reduce_max_sync(0xffffffffu, gmax);
        uint32_t nbl = 0;
        if (gmax <= BS_RANKMAX) {
            mgs = gmax;
        } else {  // groups > 8 keys (duplicate-heavy inputs): list them (pos values)
            uint32_t bigm = 0;
            mgs = 0;
#pragma unroll
            for (int q = 0; q < 8; q++) {
                mgs = (c[q] <= BS_RANKMAX && c[q] > mgs) ? c[q] : mgs;
                bigm |= (c[q] > BS_RANKMAX ? 1u : 0u) << q;
            }
            mgs = __reduce_max_sync(0xffffffffu, mgs);
            const uint32_t nb = __popc(bigm);
            const uint32_t pre = warp_incl_scan(nb) - nb;
            uint32_t m = bigm, o = pre;
            while (m) {
                const int q = __ffs(m) - 1;
                m &= m - 1;
                if (o < 32) W.big[o] = 8 * lane + q;
                o++;
            }
            nbl = __shfl_sync(0xffffffffu, pre + nb, 31);  // total
        }
        r_maxg = gmax > r_maxg ? gmax : r_maxg;
        if (lane == 0) {
            W.K[WS_MAX] = np;
            W.K[WS_MAX + 7] = nbl;  // stash the count
        }
    }
    __syncwarp();
    // placement: T[K[pos] + r] = ord(key)
#pragma unroll
    for (int k = 0; k < WS_KPL; k++) {
        if (code[k] != BS_NONE) {
            const uint32_t pos = code[k] & 0xffffu;
            const uint32_t q = W.K[pos] + (code[k] >> 16);
            T[q] = to_ord<DT>(key[k]);
        }
    }
    __syncwarp();
    // touch-up: odd-even transposition on 8 consecutive positions per
    // lane. pos is monotone in the key (R15), so neighbours from different
    // slots are already in order and never swap: every compare-exchange
    // acts inside one collision group, which is sorted after as many
    // rounds as it has keys (2 rounds per iteration; none without
    // collisions; a clean pass ends it early on duplicate-heavy inputs).
    // Groups > 8 are sorted again by the warp bitonic below.
    const int iters = mgs > 1u ? (int)((mgs + 1u) >> 1) : 0;  // (no collision: nothing to do)
    const uint32_t nbl = W.K[WS_MAX + 7];
    // A first pass that moves nothing has compared every adjacent pair:
    // T is then sorted, groups > 8 included (duplicate-heavy inputs: equal
    // keys share pos, so their large groups are runs of one value)
    bool moved = false;
    if (iters > 0 || nbl > 0) {
        const uint32_t q0 = 8u * lane;
        uint64_t v[8];
        {
            const uint64_t *row = W.T + 9u * lane;
#pragma unroll
            for (int q = 0; q < 8; q++) v[q] = q0 + q < np ? row[q] : ~0ull;
        }
        // one pass = even pairs, odd pairs, the pair across lanes. Only
        // the first pass reports whether anything moved (a clean first
        // pass means every group is already in order: duplicate-heavy
        // inputs); later passes skip that bookkeeping.
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
        moved = __any_sync(0xffffffffu, pass(true));
        if (moved) {
            for (int it2 = 1; it2 < iters; it2++) pass(false);
            if (q0 < np) {
                uint64_t *row = W.T + 9u * lane;
#pragma unroll
                for (int q = 0; q < 8; q++) row[q] = v[q];
            }
        }
    }
    __syncwarp();
    // groups > 8 keys: register bitonic by the whole warp (the plain
    // select network: the single-predicate one costs the main path
    // registers here)
    if (moved) {
        for (uint32_t k = 0; k < nbl; k++) {
            uint32_t pos;
            if (nbl <= 32) {
                pos = W.big[k];
            } else {  // (more than 32 large groups: rescan the totals)
                uint32_t seen = 0;
                pos = 0;
                for (uint32_t x = 0; x < S; x++)
                    if (W.K[x + 1] - W.K[x] > BS_RANKMAX && seen++ == k) { pos = x; break; }
            }
            const uint32_t base = W.K[pos], c = W.K[pos + 1] - base;
            bool same = true;
            for (uint32_t q = lane; q < c; q += 32) same &= (T[base + q] == T[base]);
            if (__all_sync(0xffffffffu, same)) continue;  // (this group: next one)
            if (c <= 32u) {
                uint64_t v1 = (uint32_t)lane < c ? T[base + lane] : ~0ull;
                warp_sort32<false>(v1, lane);
                if ((uint32_t)lane < c) T[base + lane] = v1;
            } else if (c <= 64u) {
                warp_sort_T<2, false>(T + base, c, lane);
            } else if (c <= 128u) {
                warp_sort_T<4, false>(T + base, c, lane);
            } else {
                warp_sort_T<8, false>(T + base, c, lane);
            }
        }
    }
    __syncwarp();
    // homogeneous iff first == last of the sorted sub-bucket
    if (T[0] != T[np - 1u]) {
        const uint64_t *tl = W.T + lane + (lane >> 3);  // T[32k + lane] at tl[36k]
#pragma unroll
        for (int k = 0; k < WS_KPL; k++)
            if (32u * k + lane < np) gl[32 * k] = from_ord<DT>(tl[36 * k]);
        if (lane == 0) {
            wst[0]++;
            wst[1] += np;
        }
    } else {
        if (lane == 0 && a.dH1) a.dH1[g] = 1;
        if (lane == 0) {
            wst[2]++;
            wst[3] += np;
        }
        early_h1 = true;
    }
    __syncwarp();
}

}  // namespace ls
