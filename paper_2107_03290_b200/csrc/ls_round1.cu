// ls_round1.cu -- round 1 of Alg. 2 (Alg. 1 applied to every
// level-0 bucket) with the bucket resident in a CTA cluster's distributed
// shared memory.
//
// The separate path reads each level-0 bucket three times from HBM (k_count1:
// keys -> b1 histogram + each key's b1; k_scatter1: keys + b1 ids -> tile
// reorder in shared memory -> runs into A). Here one cluster of FR_CL CTAs owns
// a whole bucket of fr_min..FR_CL * (FR_Q - 2) keys:
//   P1  every CTA stages its slice of the bucket (TMA bulk copy) and computes
//       b1 of every key (predict + Alg. 1 P:107 at level 1), a b1 histogram in
//       its shared memory and the slice's ord range; b1 is kept in a.bid;
//   P2  cluster barrier; every CTA sums the FR_CL histograms through DSMEM:
//       the bucket's S'_B row (written to hist1 by rank 0), the sub-bucket
//       starts, and where its own keys of every sub-bucket go (start + the
//       lower ranks' counts). A homogeneous bucket (min == max) is
//       written straight from its value instead;
//   P3  every CTA reorders its slice by sub-bucket in its own shared memory
//       (keys and ids re-read from L2);
//   P4  one warp per sub-bucket writes the CTA's run (~n'/FR_CL keys, 8x the
//       per-tile runs of k_scatter1) to its place in A.
// HBM: 8 B/key read + 8 B/key write (+ 2 + 2 B/key of ids, mostly L2) instead
// of count1's 8 + 2 and scatter1's 16 + 2. Output, ids and S'_B are the
// separate path's (parity tests run both).
//
// Measured on B200 at 200M Normal keys (every bucket fits): 2.23 ms against
// 1.84 ms for k_count1 + k_scatter1, so it is opt-in (LS_FLAG_FUSED_ROUND1).
// The cluster shape caps the kernel at 15 co-resident 8-SM clusters (120 of
// 148 SMs), P1 alone costs what k_count1 costs on 148 SMs, and the phases of a
// bucket serialise behind two cluster barriers (per-phase clock64 counters,
// LS_DEBUG_STAGE=8192). An earlier variant that scattered every key straight
// into the owning CTA's shared memory (st.shared::cluster) took 3.0 ms:
// scattered 8-byte DSMEM stores run at ~5 B/clk per SM.
#include <cooperative_groups.h>

#include <type_traits>

#include <mutex>

#include "ls_common.cuh"
#include "ls_launch.h"
#include "ls_wstask.cuh"

namespace cg = cooperative_groups;

namespace ls {

constexpr int FR_CL = 8;            // CTAs per cluster (portable maximum)
constexpr int FR_THREADS = 1024;
constexpr uint32_t FR_Q = 27392;    // keys of the bucket held per CTA (8 B each)

struct FrSmem {
    uint64_t region[FR_Q];              // P1: this CTA's slice (TMA-staged); P3/P4: the same keys
                                        // in sub-bucket order
    uint32_t hist[LS_MAX_FANOUT];       // this CTA's b1 counts (read by the whole cluster in P2)
    uint32_t cur[LS_MAX_FANOUT];        // P3 cursors (local order by sub-bucket)
    uint32_t dst[LS_MAX_FANOUT];        // where this CTA's run of each sub-bucket goes in the bucket
    uint32_t wsum[33];
    uint32_t bucket;                    // current level-0 bucket (rank 0 writes it into every CTA)
    unsigned long long mn, mx;          // this CTA's slice: ord range
    uint64_t mbar;
};
static_assert(sizeof(FrSmem) <= 232448, "k_round1 shared memory");

template <int DT>
__global__ void __cluster_dims__(FR_CL, 1, 1) __launch_bounds__(FR_THREADS, 1) k_round1(Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FrSmem &S = *reinterpret_cast<FrSmem *>(smem_raw);
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t rank = cl.block_rank();
    const int tid = threadIdx.x, f = a.f;
    const Root R = load_root(a.M);
    const double *leaf = a.M->leaf;
    // the only level-0 buckets that can hold keys outside [xmin, xmax] (they
    // are clamped onto xmin / xmax): elsewhere the root clamp is skipped
    const uint32_t g_lo = sub_bucket_at(R.xmin, R, leaf, a.F, a.F2, f);
    const uint32_t g_hi = sub_bucket_at(R.xmax, R, leaf, a.F, a.F2, f);
    const uint32_t b_lo = g_lo / (uint32_t)f, b_hi = g_hi / (uint32_t)f;
    // P5 state: per-warp statistics and the warp sort's adaptive flags
    const int lane = tid & 31, warp = tid >> 5;
    uint32_t r_maxg = 0, wst[4] = {0u, 0u, 0u, 0u};
    bool early_h1 = false;
    if (tid == 0) mbar_init(&S.mbar, 1);
    uint32_t phase = 0;
    const bool prof = (a.dbg & 8192u) && tid == 0;
    long long t_prev = clock64();
    auto mark = [&](int k) {
        if (prof) {
            const long long t_ = clock64();
            atomicAdd(&a.ctl->prof[k], (unsigned long long)(t_ - t_prev));
            t_prev = t_;
        }
    };
    for (;;) {
        if (rank == 0 && tid == 0) {
            const uint32_t t = atomicAdd(&a.ctl->fticket, 1u);
            const uint32_t b = (t < a.ctl->nfused && a.ctl->status == 0) ? a.flist[t] : ~0u;
            for (int k = 0; k < FR_CL; k++) *cl.map_shared_rank(&S.bucket, k) = b;
        }
        mark(7);
        cl.sync();  // (A) bucket published; every CTA is done with the previous one
        mark(0);
        const uint32_t b = S.bucket;
        if (b == ~0u) break;
        const uint64_t bbeg = a.start0[b];
        const uint32_t nb = (uint32_t)(a.start0[b + 1] - bbeg);
        const uint32_t per = (nb + FR_CL - 1) / FR_CL;
        const uint64_t s0 = bbeg + min(nb, per * rank), s1 = bbeg + min(nb, per * (rank + 1));
        // stage the slice with the bulk engine (16-byte aligned hull; a last
        // odd key at the very end of B is loaded directly)
        const uint64_t h0 = s0 & ~1ull;
        if (tid == 0 && s1 > s0) {
            uint64_t h1 = (s1 + 1) & ~1ull;
            if (h1 > a.n) {
                h1 = s1 & ~1ull;
                S.region[s1 - 1 - h0] = a.B[s1 - 1];
            }
            const uint32_t bytes = (uint32_t)((h1 - h0) * 8);
            mbar_expect_tx(&S.mbar, bytes);
            for (uint32_t o = 0; o < bytes; o += 32768u)
                bulk_g2s((char *)S.region + o, (const char *)(a.B + h0) + o,
                         bytes - o < 32768u ? bytes - o : 32768u, &S.mbar);
        }
        for (int j = tid; j < f; j += FR_THREADS) S.hist[j] = 0;
        if (tid == 0) {
            S.mn = ~0ull;
            S.mx = 0ull;
        }
        __syncthreads();
        if (s1 > s0) {
            mbar_wait(&S.mbar, phase);
            phase ^= 1u;
        }
        mark(1);
        // P1: b1 per key (Alg. 1 P:107 with the parent b), histogram, ord range
        {
            const uint64_t *sk = S.region + (s0 - h0);
            const uint32_t ns = (uint32_t)(s1 - s0);
            uint16_t *bid = a.bid + s0;
            unsigned long long mn = ~0ull, mx = 0;
            auto body = [&](auto inner) {
                for (uint32_t j = tid; j < ns; j += FR_THREADS) {
                    const uint64_t key = sk[j];
                    const unsigned long long o = to_ord<DT>(key);
                    mn = o < mn ? o : mn;
                    mx = o > mx ? o : mx;
                    const double p = decltype(inner)::value ? predict_ldg_inner<DT>(key, R, leaf)
                                                            : predict_ldg<DT>(key, R, leaf);
                    const uint32_t b1 = bucket1(p, a.F2, f, b);
                    atomicAdd(&S.hist[b1], 1u);
                    bid[j] = (uint16_t)b1;
                }
            };
            if (b != b_lo && b != b_hi) body(std::true_type{});
            else body(std::false_type{});
            mn = warp_min_u64(mn);
            mx = warp_max_u64(mx);
            if ((tid & 31) == 0) {
                atomicMin(&S.mn, mn);
                atomicMax(&S.mx, mx);
            }
        }
        mark(2);
        cl.sync();  // (B) every slice's histogram and range are final; every CTA is done
                    //     reading its staged slice, so the regions become P3's destinations
        unsigned long long gmn = ~0ull, gmx = 0;
#pragma unroll
        for (int k = 0; k < FR_CL; k++) {
            const unsigned long long m0 = *cl.map_shared_rank(&S.mn, k), m1 = *cl.map_shared_rank(&S.mx, k);
            gmn = m0 < gmn ? m0 : gmn;
            gmx = m1 > gmx ? m1 : gmx;
        }
        if (rank == 0 && tid == 0) {
            a.bmin0[b] = gmn;  // (k_count1's encoding: the value, and "two keys differ")
            a.bmax0[b] = gmn != gmx ? 1ull : 0ull;
        }
        if (gmn == gmx) {
            // homogeneous level-0 bucket: final as its value
            const uint64_t v = from_ord<DT>(gmn);
            for (uint64_t i = s0 + tid; i < s1; i += FR_THREADS) a.A[i] = v;
            continue;
        }
        // P2: S'_B row, sub-bucket starts, where this CTA's keys of every
        // sub-bucket go (start + the lower ranks' counts), and the local
        // order (exclusive scan of this CTA's own counts) (f <= FR_THREADS)
        uint32_t pre = 0;
        if (tid < f) {
            uint32_t tot = 0;
#pragma unroll
            for (int k = 0; k < FR_CL; k++) {
                const uint32_t c = *cl.map_shared_rank(&S.hist[tid], k);
                pre += (uint32_t)k < rank ? c : 0u;
                tot += c;
            }
            S.cur[tid] = tot;
            if (rank == 0) a.hist1[(uint64_t)b * f + tid] = tot;
        }
        __syncthreads();
        block_exscan(S.cur, f, S.wsum);
        if (tid < f) {
            S.dst[tid] = S.cur[tid] + pre;
            S.cur[tid] = S.hist[tid];
        }
        __syncthreads();
        block_exscan(S.cur, f, S.wsum);
        mark(3);
        // P3: this CTA's slice reordered by sub-bucket in its own shared
        // memory (the staged copy is consumed); keys re-read from L2, 8 in
        // flight per thread
        {
            auto put = [&](uint64_t key, uint32_t b1) { S.region[atomicAdd(&S.cur[b1], 1u)] = key; };
            uint64_t i = s0 + tid;
            for (; i + 7 * FR_THREADS < s1; i += 8 * FR_THREADS) {
                uint64_t v[8];
                uint32_t c[8];
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    v[q] = a.B[i + q * FR_THREADS];
                    c[q] = a.bid[i + q * FR_THREADS];
                }
#pragma unroll
                for (int q = 0; q < 8; q++) put(v[q], c[q]);
            }
            for (; i < s1; i += FR_THREADS) put(a.B[i], a.bid[i]);
        }
        __syncthreads();
        mark(4);
        // P4: one run per sub-bucket (~n'/FR_CL keys) to its place in A, one
        // warp per sub-bucket (runs 8x longer than k_scatter1's per-tile runs)
        {
            uint64_t *dst = a.A + bbeg;
            for (int j = warp; j < f; j += FR_THREADS / 32) {
                const uint32_t cnt = S.hist[j], lo = S.cur[j] - cnt, d = S.dst[j];
                for (uint32_t t = lane; t < cnt; t += 32) dst[d + t] = S.region[lo + t];
            }
        }
        mark(5);
        // P5 (f2, second half): the bucket's SMALL sub-buckets of <= WS_MAX keys
        // (Alg. 2's counting sort + touch-up, ws_task) sorted by the cluster's
        // 256 warps right after the scatter, while its lines are in L2; each
        // warp's slice lives in the (consumed) region; k_classify lists no warp
        // task for a fused bucket. Starts and sizes: rank 0's P2 table (DSMEM).
        cl.sync();  // (C) every CTA's runs are in A
        {
            WsSlice *SL = reinterpret_cast<WsSlice *>(S.region);
            for (int j = (int)rank * (FR_THREADS / 32) + warp; j < f; j += FR_CL * (FR_THREADS / 32)) {
                const uint32_t s0j = *cl.map_shared_rank(&S.dst[j], 0);
                const uint32_t s1j = j + 1 < f ? *cl.map_shared_rank(&S.dst[j + 1], 0) : nb;
                const uint32_t c = s1j - s0j;
                if (size_class(c, a.T_small) != SC_WARP) continue;  // (warp-uniform)
                const uint32_t g = b * (uint32_t)f + (uint32_t)j;
                const uint32_t wl = contained_leaf_warp(leaf, R.Lm1 + 1, g, g, a.rcpF2, lane);
                ws_task<DT>(a, R, g_lo, g_hi, SL[warp], wst, r_maxg, early_h1,
                            make_uint4((uint32_t)bbeg + s0j, c, g, wl), lane);
            }
        }
        mark(6);
    }
    if (lane == 0) {
        if (wst[0]) atomicAdd(&a.ctl->stat[ST_SMALLS], (unsigned long long)wst[0]);
        if (wst[1]) atomicAdd(&a.ctl->stat[ST_SMALLK], (unsigned long long)wst[1]);
        if (wst[2]) atomicAdd(&a.ctl->stat[ST_H1S], (unsigned long long)wst[2]);
        if (wst[3]) atomicAdd(&a.ctl->stat[ST_H1K], (unsigned long long)wst[3]);
        if (r_maxg > 1) atomicMax(&a.ctl->stat[ST_MAXGRP], (unsigned long long)r_maxg);
    }
}
static_assert(sizeof(WsSlice) * (FR_THREADS / 32) <= sizeof(uint64_t) * FR_Q, "P5 warp slices fit the region");

// Active clusters of k_round1 per device (-1: not probed, 0: unavailable).
// cudaFuncSetAttribute and the cluster occupancy are per device, so the probe
// runs once per device (std::call_once per slot).
constexpr int FR_MAX_DEV = 64;
static int g_fr_clusters[FR_MAX_DEV];
static std::once_flag g_fr_once[FR_MAX_DEV];

static int fr_clusters(int dev) {
    if (dev < 0 || dev >= FR_MAX_DEV) return 0;
    std::call_once(g_fr_once[dev], [dev] {
        g_fr_clusters[dev] = 0;
        const size_t sm = sizeof(FrSmem);
        if (cudaFuncSetAttribute(k_round1<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) ==
                cudaSuccess &&
            cudaFuncSetAttribute(k_round1<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) ==
                cudaSuccess) {
            cudaLaunchConfig_t c;
            memset(&c, 0, sizeof c);
            c.gridDim = dim3(FR_CL, 1, 1);
            c.blockDim = dim3(FR_THREADS, 1, 1);
            c.dynamicSmemBytes = sm;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, (void *)k_round1<DT_F64>, &c) == cudaSuccess && n > 0)
                g_fr_clusters[dev] = n;
        }
        cudaGetLastError();  // clear a failed probe
    });
    return g_fr_clusters[dev];
}

static int current_device() {
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return d;
}

uint32_t round1_capacity() {
    return fr_clusters(current_device()) > 0 ? (uint32_t)FR_CL * (FR_Q - 2) : 0u;  // (- 2: the staged slice's hull)
}

void launch_round1(const Args &a, int dtype, cudaStream_t st) {
    const size_t sm = sizeof(FrSmem);
    const dim3 grid((unsigned)(FR_CL * fr_clusters(current_device())));
    if (dtype == DT_F64) k_round1<DT_F64><<<grid, FR_THREADS, sm, st>>>(a);
    else k_round1<DT_U64><<<grid, FR_THREADS, sm, st>>>(a);
}

}  // namespace ls
