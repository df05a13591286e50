// ls_fit.cu -- north_star (1): strided sample + two-level linear RMI fit in fp64.
//
// The chord model (R7) only needs, per leaf l, the number
// of sample keys routed to it and its smallest key: the eCDF target of a leaf's
// first key is (#sample keys in leaves < l)/m (R8: equal keys share a leaf, so
// the strict-less rank of the leaf's first key is exactly that count). So the
// fit is a reduction + histogram + one 1000-entry scan -- no sample sort -- and
// its parameters are bit-identical to the oracle's (no floating-point
// reductions are involved).
#include "ls_launch.h"

namespace ls {

// One sample key: a single 8-byte word per 800 bytes of input, so the load
// asks L2 for a 64-byte fill (LS_SAMPLE_L2: 0 = plain streaming load)
#ifndef LS_SAMPLE_L2
#define LS_SAMPLE_L2 64
#endif
__device__ __forceinline__ uint64_t ld_sample(const uint64_t *p) {
#if LS_SAMPLE_L2 == 64
    uint64_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.b64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
#else
    return __ldcs(p);
#endif
}

template <int DT>
__global__ void __launch_bounds__(256) k_sample_minmax(const uint64_t *__restrict__ src,
                                                       uint64_t stride, uint64_t m,
                                                       uint64_t *__restrict__ S, Ctl *ctl) {
    unsigned long long mn = ~0ull, mx = 0;
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    // strided gathers (one sector per key): 8 independent loads in flight per thread
    constexpr int U = 8;
    for (uint64_t k0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < m; k0 += U * gs) {
        uint64_t b[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t k = k0 + u * gs;
            b[u] = k < m ? ld_sample(src + k * stride) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t k = k0 + u * gs;
            if (k >= m) continue;
            if (S) S[k] = b[u];
            if (is_finite_key<DT>(b[u]) && !(DT == DT_F64 && is_nan_bits(b[u]))) {
                const unsigned long long o = to_ord<DT>(b[u]);
                mn = o < mn ? o : mn;
                mx = o > mx ? o : mx;
            }
        }
    }
    mn = warp_min_u64(mn);
    mx = warp_max_u64(mx);
    if ((threadIdx.x & 31) == 0) {
        if (mn != ~0ull) atomicMin(&ctl->smin, mn);
        if (mx != 0) atomicMax(&ctl->smax, mx);
    }
}

// Root of the chord model from the finite sample range (O2).
template <int DT>
__device__ __forceinline__ bool fit_root(const Ctl *ctl, int L, Root &R, double &v) {
    unsigned long long smin = ctl->smin, smax = ctl->smax;
    if (smin > smax) {  // no finite sample key
        v = 0.0;
        return false;
    }
    R.xmin = xd<DT>(from_ord<DT>(smin));
    R.xmax = xd<DT>(from_ord<DT>(smax));
    v = R.xmin;
    if (R.xmin == R.xmax) return false;
    R.rs = __ddiv_rn((double)L, __dsub_rn(R.xmax, R.xmin));
    R.last = (double)(L - 1);
    R.Lm1 = L - 1;
    return true;
}

// O3: route every sample key to its leaf; per-leaf count and smallest ord.
template <int DT>
__global__ void __launch_bounds__(512) k_fit_hist(const uint64_t *__restrict__ S, uint64_t m, int L,
                                                  const Ctl *ctl, uint32_t *leaf_cnt,
                                                  unsigned long long *leaf_min) {
    __shared__ uint32_t cnt[LS_MAX_LEAVES];
    __shared__ unsigned long long mn[LS_MAX_LEAVES];
    Root R;
    double v;
    if (!fit_root<DT>(ctl, L, R, v)) return;  // degenerate model: nothing to fit
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        cnt[l] = 0;
        mn[l] = ~0ull;
    }
    __syncthreads();
    const uint64_t gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gs) {
        uint64_t b = S[k];
        double xc = clampd(xd<DT>(b), R.xmin, R.xmax);
        double r = __dmul_rn(__dsub_rn(xc, R.xmin), R.rs);
        int l = (r < R.last) ? (int)__double2ll_rz(r) : R.Lm1;
        atomicAdd(&cnt[l], 1u);
        atomicMin(&mn[l], (unsigned long long)to_ord<DT>(b));
    }
    __syncthreads();
    for (int l = threadIdx.x; l < L; l += blockDim.x) {
        if (cnt[l]) {
            atomicAdd(&leaf_cnt[l], cnt[l]);
            atomicMin(&leaf_min[l], mn[l]);
        }
    }
}

// O4-O5: one block of 1024 threads. beg_l = #keys in leaves < l; the next
// non-empty leaf nx(l) supplies (x1, y1); the last one runs to (xmax, PMAX).
template <int DT>
__global__ void __launch_bounds__(1024) k_fit_params(uint64_t m, int L, const Ctl *ctl,
                                                     const uint32_t *leaf_cnt,
                                                     const unsigned long long *leaf_min,
                                                     DevModel *M) {
    __shared__ uint32_t beg[LS_MAX_LEAVES];
    __shared__ int nxt[LS_MAX_LEAVES + 1];
    __shared__ uint32_t tmp[33];
    Root R;
    double v;
    const bool ok = fit_root<DT>(ctl, L, R, v);
    const int t = threadIdx.x;
    if (t == 0) {
        M->L = (uint32_t)L;
        M->n_sample = m;
        M->last = (double)(L - 1);
        M->degenerate = ok ? 0u : 1u;
        M->xmin = ok ? R.xmin : v;
        M->xmax = ok ? R.xmax : v;
        M->root_scale = ok ? R.rs : 0.0;
    }
    if (!ok) {  // degenerate model: p == 0
        for (int l = t; l < L; l += blockDim.x)
            for (int q = 0; q < 5; q++) M->leaf[5 * l + q] = 0.0;
        return;
    }
    for (int l = t; l < L; l += blockDim.x) beg[l] = leaf_cnt[l];
    __syncthreads();
    block_exscan(beg, L, tmp);
    // nxt[l] = smallest non-empty leaf index > l (or L): suffix minimum
    for (int l = t; l <= L; l += blockDim.x) nxt[l] = (l < L && leaf_cnt[l] > 0) ? l : L;
    __syncthreads();
    for (int d = 1; d <= L; d <<= 1) {
        int val[2];
        int c = 0;
        for (int l = t; l <= L && c < 2; l += blockDim.x, c++)
            val[c] = (l + d <= L) ? min(nxt[l], nxt[l + d]) : nxt[l];
        __syncthreads();
        c = 0;
        for (int l = t; l <= L && c < 2; l += blockDim.x, c++) nxt[l] = val[c];
        __syncthreads();
    }
    const double md = __ull2double_rn(m);
    for (int l = t; l < L; l += blockDim.x) {
        const int nx = nxt[l + 1];
        double x1, y1;
        if (nx < L) {
            x1 = clampd(xd<DT>(from_ord<DT>(leaf_min[nx])), R.xmin, R.xmax);
            y1 = __ddiv_rn(__ull2double_rn(beg[nx]), md);
        } else {
            x1 = R.xmax;
            y1 = PMAX;
        }
        const double hi = (y1 < PMAX) ? y1 : PMAX;
        double *q = &M->leaf[5 * l];
        if (leaf_cnt[l] > 0) {
            double x0 = clampd(xd<DT>(from_ord<DT>(leaf_min[l])), R.xmin, R.xmax);
            double y0 = __ddiv_rn(__ull2double_rn(beg[l]), md);
            q[0] = (x1 > x0) ? __ddiv_rn(__dsub_rn(y1, y0), __dsub_rn(x1, x0)) : 0.0;
            q[1] = x0;
            q[2] = y0;
            q[3] = y0;
            q[4] = hi;
        } else {
            q[0] = 0.0;
            q[1] = 0.0;
            q[2] = hi;
            q[3] = hi;
            q[4] = hi;
        }
    }
}

// ------------------------------------------------------- b0 search tables ---
// thr_b = min{o : b0(o) >= b} for b = 1..f-1 by bisection over the non-NaN ord
// domain, evaluating b0 with the same predict()/bucket0() as every other
// path; then per grid cell the range of thresholds inside its ord range.
template <int DT>
__device__ __forceinline__ uint32_t b0_at(unsigned long long o, const Root &R, const double *leaf,
                                          double F, int f) {
    return bucket0(predict_ldg<DT>(from_ord<DT>(o), R, leaf), F, f);
}
template <int DT>
__device__ __forceinline__ void ord_domain(unsigned long long &omin, unsigned long long &omax) {
    omin = DT == DT_F64 ? 0x000FFFFFFFFFFFFFull : 0ull;   // ord(-inf)
    omax = DT == DT_F64 ? 0xFFF0000000000000ull : ~0ull;  // ord(+inf)
}

// Smallest o in [lo, hi) with pred(o) true (pred monotone: false ... true),
// else hi -- the bisection "while (lo < hi) { mid; pred(mid) ? hi = mid :
// lo = mid + 1; }" run by a whole warp as a 33-ary search: each round the 32
// lanes test 32 evenly spaced points and the ballot keeps the gap holding the
// first true one (13 rounds over the 64-bit ord domain instead of 64).
template <class P>
__device__ __forceinline__ unsigned long long warp_first_true(const P &pred, unsigned long long lo,
                                                             unsigned long long hi, int lane) {
    while (hi - lo > 32) {
        const unsigned long long step = (hi - lo) / 33;  // >= 1; 32 * step < hi - lo
        const unsigned long long m = lo + step * (unsigned long long)(lane + 1);
        const uint32_t bal = __ballot_sync(0xffffffffu, pred(m));
        if (bal) {
            const int f = __ffs(bal) - 1;
            hi = lo + step * (unsigned long long)(f + 1);
            lo = f == 0 ? lo : lo + step * (unsigned long long)f + 1;
        } else {
            lo = lo + step * 32ull + 1;
        }
    }
    const unsigned long long m = lo + (unsigned long long)lane;
    const uint32_t bal = __ballot_sync(0xffffffffu, m < hi && pred(m));
    return bal ? lo + (unsigned long long)(__ffs(bal) - 1) : hi;
}

// one warp per threshold b = 1 .. f-1
template <int DT>
__global__ void __launch_bounds__(256) k_b0_thresholds(DevModel *M, int f) {
    const int lane = threadIdx.x & 31;
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) / 32 + 1;
    const Root R = load_root(M);
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        const double range = __dsub_rn(M->xmax, M->xmin);
        M->cell_scale = (M->degenerate || !(range > 0.0)) ? 0.0 : __ddiv_rn((double)B0_CELLS, range);
    }
    if (b >= f) return;
    unsigned long long lo, hi;
    ord_domain<DT>(lo, hi);
    const double F = (double)f;
    if (b0_at<DT>(hi, R, M->leaf, F, f) < (uint32_t)b) {
        if (lane == 0) M->thr[b - 1] = ~0ull;  // never reached: not counted in nthr
        return;
    }
    const unsigned long long t = warp_first_true(
        [&](unsigned long long o) { return b0_at<DT>(o, R, M->leaf, F, f) >= (uint32_t)b; }, lo, hi, lane);
    if (lane == 0) {
        M->thr[b - 1] = t;
        atomicMax(&M->nthr, (uint32_t)b);
    }
}

// Smallest o in [omin, omax] with pred(o) (pred monotone false ... true; the
// caller has checked pred(omax)), found from a guess o0 in [omin, omax]:
// gallop away from o0 to bracket the first true point, then bisect the
// bracket. The result is the plain bisection's for any guess; a guess a few
// ulps off (the grid boundaries below) needs a handful of evaluations instead
// of 64.
template <class P>
__device__ __forceinline__ unsigned long long first_true_from(const P &pred, unsigned long long omin,
                                                              unsigned long long omax, unsigned long long o0) {
    unsigned long long lo, hi;
    if (pred(o0)) {
        hi = o0;
        lo = omin;
        for (unsigned long long d = 1; hi > omin;) {
            const unsigned long long c = hi - omin > d ? hi - d : omin;
            if (!pred(c)) { lo = c + 1; break; }
            hi = c;
            if (c == omin) { lo = omin; break; }
            d = d < (1ull << 62) ? 2 * d : d;
        }
    } else {
        lo = o0 + 1;
        hi = omax;
        for (unsigned long long d = 1;;) {
            const unsigned long long c = omax - lo > d ? lo + d : omax;
            if (pred(c)) { hi = c; break; }
            lo = c + 1;  // (c < omax: pred(omax) holds)
            d = d < (1ull << 62) ? 2 * d : d;
        }
    }
    while (lo < hi) {
        const unsigned long long mid = lo + (hi - lo) / 2;
        if (pred(mid)) hi = mid; else lo = mid + 1;
    }
    return lo;
}

// The ord of the key nearest the double x, clamped into [omin, omax] (a
// starting guess only).
template <int DT>
__device__ __forceinline__ unsigned long long guess_ord(double x, unsigned long long omin, unsigned long long omax) {
    if (!(x == x) || x - x != 0.0) return omin;  // (NaN / inf: no guess)
    unsigned long long o;
    if (DT == DT_F64) o = to_ord<DT>((uint64_t)__double_as_longlong(x + 0.0));
    else o = x <= 0.0 ? 0ull : x >= 18446744073709549568.0 ? ~0ull : (unsigned long long)x;
    return o < omin ? omin : o > omax ? omax : o;
}

// #thresholds < s and <= o_hi (thr in shared memory, V of them)
__device__ __forceinline__ void thr_range(const unsigned long long *thr, uint32_t V, unsigned long long s,
                                          unsigned long long o_hi, uint32_t &off, uint32_t &end) {
    off = 0;
    end = 0;
    for (uint32_t lo = 0, n = V; n > 0;) {
        const uint32_t h = n >> 1;
        if (thr[lo + h] < s) { lo += h + 1; n -= h + 1; } else n = h;
        off = lo;
    }
    for (uint32_t lo = 0, n = V; n > 0;) {
        const uint32_t h = n >> 1;
        if (thr[lo + h] <= o_hi) { lo += h + 1; n -= h + 1; } else n = h;
        end = lo;
    }
}

// one thread per grid cell (16K cells: parallel enough for plain bisection)
template <int DT>
__global__ void __launch_bounds__(256) k_b0_cells(DevModel *M) {
    __shared__ unsigned long long thr[LS_MAX_FANOUT];
    const uint32_t V = M->nthr;
    for (uint32_t i = threadIdx.x; i < V; i += blockDim.x) thr[i] = M->thr[i];
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= B0_CELLS) return;
    const double xmin = M->xmin, xmax = M->xmax, cs = M->cell_scale;
    unsigned long long omin, omax;
    ord_domain<DT>(omin, omax);
    // first ord of grid cell >= target: bisection started at the cell's
    // nominal left edge xmin + target / cs
    auto first_ge = [&](int target, bool &none) {
        auto pred = [&](unsigned long long o) { return b0_cell<DT>(from_ord<DT>(o), xmin, xmax, cs) >= target; };
        none = !pred(omax);
        if (none) return omax;
        const double xg = cs > 0.0 ? __dadd_rn(xmin, __ddiv_rn((double)target, cs)) : xmin;
        return first_true_from(pred, omin, omax, guess_ord<DT>(xg, omin, omax));
    };
    bool none0, none1;
    const unsigned long long s = first_ge(c, none0);
    const unsigned long long e = c + 1 < B0_CELLS ? first_ge(c + 1, none1) : (none1 = true, 0ull);
    uint32_t entry = 0;
    if (!none0 && (none1 || e > s)) {  // cell c owns ords [s, o_hi]
        const unsigned long long o_hi = none1 ? omax : e - 1;
        uint32_t off, end;  // #thr < s, #thr <= o_hi
        thr_range(thr, V, s, o_hi, off, end);
        const uint32_t cnt = end - off;
        entry = off | ((cnt < B0_REFINED ? cnt : B0_SAT) << 10);
        if (cnt >= B0_SUBMIN) {  // dense cell: refined by k_b0_sub if a sub-grid is left
            const uint32_t k = atomicAdd(&M->nsub, 1u);
            if (k < (uint32_t)B0_NSUB) {
                M->sub_cell[k] = (uint16_t)c;
                entry = k | (B0_REFINED << 10);
            }
        }
    }
    M->cell[c] = (uint16_t)entry;
}

// Sub-grids of the refined cells: entry (s) of sub-grid k covers the ords whose
// fine index is 64 * sub_cell[k] + s, encoded like a cell entry (0..61 exact,
// B0_SAT above). One thread per (k, s).
template <int DT>
__global__ void __launch_bounds__(256) k_b0_sub(DevModel *M) {
    const uint32_t nsub = min(M->nsub, (uint32_t)B0_NSUB);
    if (blockIdx.x * blockDim.x / B0_SUB >= nsub) return;  // (whole block past the sub-grids)
    __shared__ unsigned long long thr[LS_MAX_FANOUT];
    const uint32_t V = M->nthr;
    for (uint32_t i = threadIdx.x; i < V; i += blockDim.x) thr[i] = M->thr[i];
    __syncthreads();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t k = (uint32_t)t / B0_SUB, sidx = (uint32_t)t % B0_SUB;
    if (k >= nsub) return;
    const int fc = (int)M->sub_cell[k] * B0_SUB + (int)sidx;  // fine index of this sub-cell
    const double xmin = M->xmin, cs = M->cell_scale;
    unsigned long long omin, omax;
    ord_domain<DT>(omin, omax);
    auto first_ge = [&](int target, bool &none) {
        auto pred = [&](unsigned long long o) { return b0_fine<DT>(from_ord<DT>(o), xmin, cs) >= target; };
        none = !pred(omax);
        if (none) return omax;
        const double xg = cs > 0.0 ? __dadd_rn(xmin, __ddiv_rn((double)target, __dmul_rn(cs, (double)B0_SUB))) : xmin;
        return first_true_from(pred, omin, omax, guess_ord<DT>(xg, omin, omax));
    };
    bool none0, none1;
    const unsigned long long s = first_ge(fc, none0);
    const unsigned long long e = fc + 1 < B0_CELLS * B0_SUB ? first_ge(fc + 1, none1) : (none1 = true, 0ull);
    uint32_t entry = 0;
    if (!none0 && (none1 || e > s)) {  // sub-cell owns ords [s, o_hi]
        const unsigned long long o_hi = none1 ? omax : e - 1;
        uint32_t off, end;  // #thr < s, #thr <= o_hi
        thr_range(thr, V, s, o_hi, off, end);
        const uint32_t cnt = end - off;
        entry = off | ((cnt < B0_REFINED ? cnt : B0_SAT) << 10);
    }
    M->sub[k * B0_SUB + sidx] = (uint16_t)entry;
}

void launch_b0_table(DevModel *M, int L, int f, int dtype, cudaStream_t st) {
    (void)L;
    cudaMemsetAsync(&M->nthr, 0, sizeof(uint32_t), st);
    cudaMemsetAsync(&M->nsub, 0, sizeof(uint32_t), st);
    const int g = (f * 32 + 255) / 256;  // k_b0_thresholds: one warp per threshold
    if (dtype == DT_F64) {
        k_b0_thresholds<DT_F64><<<g, 256, 0, st>>>(M, f);
        k_b0_cells<DT_F64><<<B0_CELLS / 256, 256, 0, st>>>(M);
        k_b0_sub<DT_F64><<<B0_NSUB * B0_SUB / 256, 256, 0, st>>>(M);
    } else {
        k_b0_thresholds<DT_U64><<<g, 256, 0, st>>>(M, f);
        k_b0_cells<DT_U64><<<B0_CELLS / 256, 256, 0, st>>>(M);
        k_b0_sub<DT_U64><<<B0_NSUB * B0_SUB / 256, 256, 0, st>>>(M);
    }
}

static int grid_for(uint64_t m, int block) {
    uint64_t g = (m + block - 1) / block;
    if (g > 148 * 8) g = 148 * 8;
    return g ? (int)g : 1;
}

void launch_sample_minmax(const uint64_t *src, uint64_t stride, uint64_t m, uint64_t *S_out,
                          Ctl *ctl, int dtype, cudaStream_t st) {
    int g = grid_for((m + 7) / 8, 256);
    if (dtype == DT_F64)
        k_sample_minmax<DT_F64><<<g, 256, 0, st>>>(src, stride, m, S_out, ctl);
    else
        k_sample_minmax<DT_U64><<<g, 256, 0, st>>>(src, stride, m, S_out, ctl);
}

void launch_fit_hist(const uint64_t *S, uint64_t m, int L, Ctl *ctl, uint32_t *leaf_cnt,
                     unsigned long long *leaf_min, int dtype, cudaStream_t st) {
    int g = grid_for(m, 512 * 8);
    if (dtype == DT_F64)
        k_fit_hist<DT_F64><<<g, 512, 0, st>>>(S, m, L, ctl, leaf_cnt, leaf_min);
    else
        k_fit_hist<DT_U64><<<g, 512, 0, st>>>(S, m, L, ctl, leaf_cnt, leaf_min);
}

void launch_fit_params(uint64_t m, int L, Ctl *ctl, const uint32_t *leaf_cnt,
                       const unsigned long long *leaf_min, DevModel *M, int dtype, cudaStream_t st) {
    if (dtype == DT_F64)
        k_fit_params<DT_F64><<<1, 1024, 0, st>>>(m, L, ctl, leaf_cnt, leaf_min, M);
    else
        k_fit_params<DT_U64><<<1, 1024, 0, st>>>(m, L, ctl, leaf_cnt, leaf_min, M);
}

}  // namespace ls
