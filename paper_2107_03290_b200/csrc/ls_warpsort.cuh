// ls_warpsort.cuh -- warp-wide sorting networks in registers (shuffles), used
// for collision groups (ls_sortsub.cu) and big-path pieces (ls_bigpath.cu).
#pragma once
#include "ls_common.cuh"

namespace ls {

// Compare-exchange of two u64 keys with one predicate (setp + two selp per
// half); returns 1 if they were swapped (only computed when `track`).
__device__ __forceinline__ uint32_t cx_u64(uint64_t &x, uint64_t &y, bool track) {
    uint64_t lo, hi;
    uint32_t sw = 0;
    if (track) {
        asm("{\n\t.reg .pred p;\n\t"
            "setp.gt.u64 p, %3, %4;\n\t"
            "selp.b64 %0, %4, %3, p;\n\t"
            "selp.b64 %1, %3, %4, p;\n\t"
            "selp.u32 %2, 1, 0, p;\n\t}"
            : "=l"(lo), "=l"(hi), "=r"(sw) : "l"(x), "l"(y));
    } else {
        asm("{\n\t.reg .pred p;\n\t"
            "setp.gt.u64 p, %2, %3;\n\t"
            "selp.b64 %0, %3, %2, p;\n\t"
            "selp.b64 %1, %2, %3, p;\n\t}"
            : "=l"(lo), "=l"(hi) : "l"(x), "l"(y));
    }
    x = lo;
    y = hi;
    return sw;
}

// take_min ? min(v, w) : max(v, w) for u64 with one 64-bit compare: when
// v == w either operand is right, so "take w iff (w < v) == take_min".
__device__ __forceinline__ uint64_t pick_u64(uint64_t v, uint64_t w, bool take_min) {
    uint64_t r;
    asm("{\n\t.reg .pred q, p;\n\t"
        "setp.eq.u32 q, %3, 0;\n\t"
        "setp.lt.xor.u64 p, %2, %1, q;\n\t"
        "selp.b64 %0, %2, %1, p;\n\t}"
        : "=l"(r) : "l"(v), "l"(w), "r"((uint32_t)take_min));
    return r;
}
__device__ __forceinline__ uint32_t pick_u64(uint32_t v, uint32_t w, bool take_min) {
    return take_min ? min(v, w) : max(v, w);
}
__device__ __forceinline__ uint32_t cx_u64(uint32_t &x, uint32_t &y, bool) {
    const uint32_t lo = min(x, y), hi = max(x, y);
    x = lo;
    y = hi;
    return 0;
}

// Ascending bitonic sort of 32 (one per lane) or 64 (two per lane, element
// lane + 32 s in v[s]) ord values across a warp, in registers.
// PICK: single-predicate selects (pick_u64); false: plain ternary selects.
template <bool PICK = true>
__device__ __forceinline__ void warp_sort32(uint64_t &v, int lane) {
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            const uint64_t w = __shfl_xor_sync(0xffffffffu, v, jj);
            const bool keep_min = ((lane & jj) == 0) == ((lane & kk) == 0);
            v = PICK ? pick_u64(v, w, keep_min) : (keep_min ? (w < v ? w : v) : (w > v ? w : v));
        }
    }
}
__device__ __forceinline__ void warp_sort64(uint64_t v[2], int lane) {
#pragma unroll
    for (int kk = 2; kk <= 64; kk <<= 1) {
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            if (jj == 32) {  // partner in the other register of the same lane (kk == 64: ascending)
                cx_u64(v[0], v[1], false);
            } else {
#pragma unroll
                for (int s2 = 0; s2 < 2; s2++) {
                    const int i = lane + 32 * s2;
                    const uint64_t w = __shfl_xor_sync(0xffffffffu, v[s2], jj);
                    const bool keep_min = ((i & jj) == 0) == ((i & kk) == 0);
                    v[s2] = pick_u64(v[s2], w, keep_min);
                }
            }
        }
    }
}

// Ascending bitonic sort of 32*NS ord values across a warp, in registers:
// element i = 32*s + lane lives in v[s]. Partners at distance >= 32 are in the
// same lane (register compare-exchange), closer ones are one shuffle away.
template <int NS, class U = uint64_t, bool PICK = true>
__device__ __forceinline__ void warp_sort_regs(U (&v)[NS], int lane) {
#pragma unroll
    for (int kk = 2; kk <= 32 * NS; kk <<= 1) {
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
            if (jj >= 32) {
                const int js = jj >> 5;
#pragma unroll
                for (int s2 = 0; s2 < NS; s2++) {
                    if (s2 & js) continue;
                    const int i = 32 * s2 + lane;
                    const bool asc = (i & kk) == 0;  // compile-time: kk >= 64
                    if (PICK) {
                        if (asc) cx_u64(v[s2], v[s2 | js], false);
                        else cx_u64(v[s2 | js], v[s2], false);
                    } else {
                        const U x = v[s2], y = v[s2 | js];
                        const bool sw_ = asc ? (x > y) : (x < y);
                        v[s2] = sw_ ? y : x;
                        v[s2 | js] = sw_ ? x : y;
                    }
                }
            } else {
#pragma unroll
                for (int s2 = 0; s2 < NS; s2++) {
                    const int i = 32 * s2 + lane;
                    const U w = __shfl_xor_sync(0xffffffffu, v[s2], jj);
                    const bool keep_min = ((i & jj) == 0) == ((i & kk) == 0);
                    v[s2] = PICK ? pick_u64(v[s2], w, keep_min)
                                 : (keep_min ? (w < v[s2] ? w : v[s2]) : (w > v[s2] ? w : v[s2]));
                }
            }
        }
    }
}

template <int DT, int NS>
__device__ __forceinline__ void warp_sort_piece(uint64_t *g, uint32_t pc, int lane) {
    uint64_t v[NS];
#pragma unroll
    for (int s2 = 0; s2 < NS; s2++) {
        const uint32_t i = 32u * s2 + lane;
        v[s2] = i < pc ? to_ord<DT>(g[i]) : ~0ull;
    }
    warp_sort_regs<NS>(v, lane);
#pragma unroll
    for (int s2 = 0; s2 < NS; s2++) {
        const uint32_t i = 32u * s2 + lane;
        if (i < pc) g[i] = from_ord<DT>(v[s2]);
    }
}

// Sort pc <= 32*NS keys of g (shared or global memory, key bits; DT order) by
// one warp. Pieces with few distinct values (duplicate-heavy inputs) are
// emitted by peeling: up to PEEL rounds of (warp minimum of the remaining
// keys, how many equal it, write that run); once more distinct values remain,
// or a peeled minimum had at most 2 copies (a piece of mostly distinct keys),
// the rest goes through the register bitonic network.
template <int DT, int NS, int PEEL = 4>
__device__ __forceinline__ void warp_sort_keys(uint64_t *g, uint32_t pc, int lane) {
    uint64_t v[NS];
    uint32_t live = 0;
#pragma unroll
    for (int s = 0; s < NS; s++) {
        const uint32_t i = 32u * s + lane;
        v[s] = i < pc ? to_ord<DT>(g[i]) : ~0ull;
        live |= (i < pc ? 1u : 0u) << s;
    }
    uint32_t out = 0;
    for (int r = 0; r < PEEL; r++) {
        unsigned long long m = ~0ull;
#pragma unroll
        for (int s = 0; s < NS; s++)
            if ((live >> s) & 1u) m = v[s] < m ? v[s] : m;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
            m = t < m ? t : m;
        }
        uint32_t c = 0;
#pragma unroll
        for (int s = 0; s < NS; s++) {
            const bool e = ((live >> s) & 1u) && v[s] == m;
            c += e ? 1u : 0u;
            live &= ~((e ? 1u : 0u) << s);
        }
        const uint32_t tot = __reduce_add_sync(0xffffffffu, c);
        const uint64_t key = from_ord<DT>(m);
        for (uint32_t i = out + lane; i < out + tot; i += 32) g[i] = key;
        out += tot;
        if (out >= pc) return;
        if (tot <= 2) break;  // a (nearly) unique minimum: few duplicates, the network is cheaper
    }
    __syncwarp();
    // more than PEEL distinct values: sort the remaining keys (the peeled ones
    // are the smallest and already written)
#pragma unroll
    for (int s = 0; s < NS; s++)
        if (!((live >> s) & 1u)) v[s] = ~0ull;
    warp_sort_regs<NS>(v, lane);
    const uint32_t rem = pc - out;
#pragma unroll
    for (int s = 0; s < NS; s++) {
        const uint32_t i = 32u * s + lane;
        if (i < rem) g[out + i] = from_ord<DT>(v[s]);
    }
}

// Same for a piece whose ords all lie in [base, base + 2^32): peeling works on
// 32-bit offsets with single-instruction warp reductions (REDUX), so a piece
// with up to PEEL distinct values costs PEEL short rounds (4: measured on
// config 4 against 2, 8 and 16 -- each round also writes its run).
template <int DT, int NS, int PEEL = 4>
__device__ __forceinline__ void warp_sort_keys_rel(uint64_t *g, uint32_t pc, unsigned long long base,
                                                   int lane) {
    uint32_t v[NS];
    uint32_t live = 0;
#pragma unroll
    for (int s = 0; s < NS; s++) {
        const uint32_t i = 32u * s + lane;
        v[s] = i < pc ? (uint32_t)(to_ord<DT>(g[i]) - base) : 0xffffffffu;
        live |= (i < pc ? 1u : 0u) << s;
    }
    uint32_t out = 0;
    for (int r = 0; r < PEEL; r++) {
        uint32_t m = 0xffffffffu;
#pragma unroll
        for (int s = 0; s < NS; s++)
            if ((live >> s) & 1u) m = v[s] < m ? v[s] : m;
        m = __reduce_min_sync(0xffffffffu, m);
        uint32_t c = 0;
#pragma unroll
        for (int s = 0; s < NS; s++) {
            const bool e = ((live >> s) & 1u) && v[s] == m;
            c += e ? 1u : 0u;
            live &= ~((e ? 1u : 0u) << s);
        }
        const uint32_t tot = __reduce_add_sync(0xffffffffu, c);
        const uint64_t key = from_ord<DT>(base + m);
        for (uint32_t i = out + lane; i < out + tot; i += 32) g[i] = key;
        out += tot;
        if (out >= pc) return;
        if (tot <= 2) break;  // a (nearly) unique minimum: few duplicates, the network is cheaper
    }
    __syncwarp();
    // more than PEEL distinct values: bitonic on the remaining offsets (the
    // peeled ones are gone; 0xffffffff pads sort last, and a live offset of
    // 0xffffffff is written correctly either way)
    uint32_t w[NS];
#pragma unroll
    for (int s = 0; s < NS; s++) w[s] = ((live >> s) & 1u) ? v[s] : 0xffffffffu;
    warp_sort_regs<NS, uint32_t>(w, lane);
    const uint32_t rem = pc - out;
#pragma unroll
    for (int s = 0; s < NS; s++) {
        const uint32_t i = 32u * s + lane;
        if (i < rem) g[out + i] = from_ord<DT>(base + w[s]);
    }
}

}  // namespace ls
