// ls_api.cu -- C ABI of libls (include/ls.h): workspace layout, the launch
// sequence of Alg. 2 on one GPU, status/stats, and the parity hooks.
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ls.h"
#include "ls_api_internal.h"
#include "ls_launch.h"

namespace ls {

static thread_local std::string g_err;

void set_error(const char *msg) { g_err = msg ? msg : ""; }

static ls_status cuda_fail(const char *where, cudaError_t e) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    set_error(buf);
    return LS_E_CUDA;
}

#define LS_CUDA(call)                                   \
    do {                                                \
        cudaError_t e_ = (call);                        \
        if (e_ != cudaSuccess) return cuda_fail(#call, e_); \
    } while (0)

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Workspace layout. Three groups, each contiguous: arrays set to 0xFF, arrays
// set to 0, arrays written before being read.
struct Layout {
    uint64_t n, m;
    int f, L;
    uint32_t C0, C1, U0, U1max, T_small, T_tile, ntiles, big_cap;
    size_t ctl, model, leaf_cnt, leaf_min, S, hist0, start0, bmin0, bmax0, ustart, lb0, offs0,
        hist1, start1, cur1, tfirst, tlast, wlist, tasks, big, chunks, hist1_u64, B, large, ltot,
        cap0, bsrc, cur0, shist0,
        lstart, lcur, lhom, lmin, lmax, pieces, bid, fills, ctasks, ctasks2, ctasks3, ctasks4, fused, flist,
        border;
    uint32_t task_cap, lcap, pcap, fcap;
    uint32_t chunk_cap;
    uint64_t Bcap;
    size_t ff_begin, ff_end, zero_begin, zero_end, total;
};

static Layout make_layout(uint64_t n, const ls_config &cfg) {
    Layout l;
    memset(&l, 0, sizeof l);
    l.n = n;
    l.f = (int)cfg.fanout;
    l.L = (int)cfg.leaf_count;
    l.m = (n + cfg.sample_stride - 1) / cfg.sample_stride;
    l.C0 = 65536;
    l.C1 = 65536;
    l.U0 = (uint32_t)((n + l.C0 - 1) / l.C0);
    if (l.U0 == 0) l.U0 = 1;
    l.U1max = (uint32_t)((n + l.C1 - 1) / l.C1) + (uint32_t)l.f;
    l.T_small = cfg.big_threshold;
    l.T_tile = 1024;  // bucket-sort windows hold tiny sub-buckets only (span <= T_tile + WS_MIN)
    l.ntiles = (uint32_t)((n + l.T_tile - 1) / l.T_tile);
    if (l.ntiles == 0) l.ntiles = 1;
    const uint64_t ff = (uint64_t)l.f * l.f;
    // big items per level: level 0 holds the sub-buckets of > T_small keys (at most n / (T_small + 1)
    // of them); deeper levels hold pieces of > 256 keys (ls_bigpath.cu) or
    // > BIG_SORT_CAP keys (k_big): at most n / 257
    const uint64_t tb = l.T_small < 256 ? l.T_small : 256;
    l.big_cap = (uint32_t)(n / (tb + 1) + 64);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = align_up(off, 256);
        off = o + bytes;
        return o;
    };
    l.ff_begin = align_up(off, 256);
    l.leaf_min = take((size_t)l.L * 8);
    l.lcap = (uint32_t)(n / (LARGE_MIN + 1) + 1);
    l.lmin = take((size_t)l.lcap * 1024 * 8);
    l.bmin0 = take((size_t)l.f * 8);
    l.tfirst = take((size_t)l.ntiles * 4);
    l.ff_end = off;
    l.zero_begin = align_up(off, 256);
    l.leaf_cnt = take((size_t)l.L * 4);
    l.hist0 = take((size_t)l.f * 8);
    l.bmax0 = take((size_t)l.f * 8);
    l.lb0 = take((size_t)l.U0 * l.f * 8);
    l.hist1 = take(ff * 4);
    l.tlast = take((size_t)l.ntiles * 4);
    l.ltot = take((size_t)l.lcap * 1024 * 4);
    l.lmax = take((size_t)l.lcap * 1024 * 8);
    l.cur0 = take((size_t)l.f * 8);
    l.shist0 = take((size_t)l.f * 4);
    l.zero_end = off;
    l.cap0 = take((size_t)l.f * 8);
    l.bsrc = take((size_t)(l.f + 1) * 8);
    l.ctl = take(sizeof(Ctl));
    l.model = take(sizeof(DevModel));
    l.S = take((size_t)l.m * 8);
    l.start0 = take((size_t)(l.f + 1) * 8);
    l.ustart = take((size_t)(l.f + 1) * 4);
    l.offs0 = take((size_t)l.U0 * l.f * 4);
    l.start1 = take(ff * 4);
    l.cur1 = take(ff * 4);
    l.wlist = take((size_t)l.ntiles * 16);
    // B: the scratch copy of the partition rounds. Round 0 by reservation
    // leaves each level-0 bucket a sample-estimated capacity (k_cap0), so B
    // holds n + n/4 + 4096 f keys (more than the estimates in practice; when
    // they do not fit, round 0 takes the exact count pass)
    l.Bcap = n + n / 4 + (uint64_t)l.f * 4096;
    l.bid = take((size_t)(l.Bcap + 16) * 2);
    l.task_cap = (uint32_t)((n / 2 + 1) < ff ? (n / 2 + 1) : ff);
    l.tasks = take((size_t)l.task_cap * 16);
    l.ctasks = take((size_t)l.task_cap * 16);
    l.ctasks2 = take((size_t)l.task_cap * 16);
    l.ctasks3 = take((size_t)l.task_cap * 16);
    l.ctasks4 = take((size_t)l.task_cap * 16);
    l.fused = take((size_t)l.f * 4);
    l.flist = take((size_t)l.f * 4);
    l.large = take((size_t)l.lcap * 4);
    l.lstart = take((size_t)l.lcap * 1024 * 4);
    l.lcur = take((size_t)l.lcap * 1024 * 4);
    l.lhom = take((size_t)l.lcap * 32 * 4);
    l.pcap = (uint32_t)(n / 256 + 1024);  // pieces come from giant items only (<= 1024 each)
    l.pieces = take((size_t)l.pcap * 8);
    l.fcap = (uint32_t)(l.lcap * 1024 + n / 65536 + 64);
    l.fills = take((size_t)l.fcap * 16);
    l.big = take((size_t)(BIG_LEVELS + 1) * l.big_cap * sizeof(BigItem));
    l.chunk_cap = (uint32_t)(n / MM_CHUNK + l.big_cap + 1);
    l.chunks = take((size_t)l.chunk_cap * sizeof(BigChunk));
    l.border = take((size_t)l.big_cap * 8);
    l.hist1_u64 = take(ff * 8);
    l.B = take((size_t)l.Bcap * 8);
    l.total = align_up(off, 256);
    return l;
}

static Args make_args(const Layout &l, void *d_keys, void *d_ws) {
    unsigned char *w = (unsigned char *)d_ws;
    Args a;
    memset(&a, 0, sizeof a);
    a.A = (uint64_t *)d_keys;
    a.B = (uint64_t *)(w + l.B);
    a.n = l.n;
    a.f = l.f;
    a.L = l.L;
    a.F = (double)l.f;
    a.F2 = (double)l.f * (double)l.f;
    a.nd = (double)l.n;
    a.rcpF2 = 1.0 / a.F2;
    {
        const double q = (double)l.n / a.F2;
        a.S1 = q >= 1048576.0 ? 1048576u : (uint32_t)q + 2u;
    }
    a.C0 = l.C0;
    a.C1 = l.C1;
    a.U0 = l.U0;
    a.U1max = l.U1max;
    a.T_small = l.T_small;
    a.T_tile = l.T_tile;
    a.ntiles = l.ntiles;
    a.big_cap = l.big_cap;
    a.ctl = (Ctl *)(w + l.ctl);
    a.M = (DevModel *)(w + l.model);
    a.S = (uint64_t *)(w + l.S);
    a.leaf_cnt = (uint32_t *)(w + l.leaf_cnt);
    a.leaf_min = (unsigned long long *)(w + l.leaf_min);
    a.hist0 = (unsigned long long *)(w + l.hist0);
    a.start0 = (unsigned long long *)(w + l.start0);
    a.bmin0 = (unsigned long long *)(w + l.bmin0);
    a.bmax0 = (unsigned long long *)(w + l.bmax0);
    a.unit1_start = (uint32_t *)(w + l.ustart);
    a.lb0 = (unsigned long long *)(w + l.lb0);
    a.offs0 = (uint32_t *)(w + l.offs0);
    a.hist1 = (uint32_t *)(w + l.hist1);
    a.start1 = (uint32_t *)(w + l.start1);
    a.cur1 = (uint32_t *)(w + l.cur1);
    a.tile_first = (uint32_t *)(w + l.tfirst);
    a.tile_last = (uint32_t *)(w + l.tlast);
    a.wlist = (uint4 *)(w + l.wlist);
    a.bid = (uint16_t *)(w + l.bid);
    a.cap0 = (unsigned long long *)(w + l.cap0);
    a.bsrc = (unsigned long long *)(w + l.bsrc);
    a.cur0 = (unsigned long long *)(w + l.cur0);
    a.shist0 = (uint32_t *)(w + l.shist0);
    a.Bcap = l.Bcap;
    a.force_exact0 = 0;
    a.tasks = (uint4 *)(w + l.tasks);
    a.ctasks = (uint4 *)(w + l.ctasks);
    a.ctasks2 = (uint4 *)(w + l.ctasks2);
    a.ctasks3 = (uint4 *)(w + l.ctasks3);
    a.ctasks4 = (uint4 *)(w + l.ctasks4);
    a.fused = (uint32_t *)(w + l.fused);
    a.flist = (uint32_t *)(w + l.flist);
    a.large = (uint32_t *)(w + l.large);
    a.lcap = l.lcap;
    a.pcap = l.pcap;
    a.ltot = (uint32_t *)(w + l.ltot);
    a.lstart = (uint32_t *)(w + l.lstart);
    a.lcur = (uint32_t *)(w + l.lcur);
    a.lhom = (uint32_t *)(w + l.lhom);
    a.lmin = (unsigned long long *)(w + l.lmin);
    a.lmax = (unsigned long long *)(w + l.lmax);
    a.pieces = (uint2 *)(w + l.pieces);
    a.fills = (uint4 *)(w + l.fills);
    a.fcap = l.fcap;
    a.task_cap = l.task_cap;
    a.big = (BigItem *)(w + l.big);
    a.chunks = (BigChunk *)(w + l.chunks);
    a.border = (uint32_t *)(w + l.border);
    a.chunk_cap = l.chunk_cap;
    return a;
}

ls_status check_config(const ls_config &c) {
    if (c.fanout < 2 || c.fanout > LS_MAX_FANOUT) { set_error("fanout out of range [2, 1024]"); return LS_E_INVALID; }
    if (c.leaf_count < 1 || c.leaf_count > LS_MAX_LEAVES) { set_error("leaf_count out of range [1, 1024]"); return LS_E_INVALID; }
    if (c.sample_stride < 1) { set_error("sample_stride must be >= 1"); return LS_E_INVALID; }
    if (c.fit != 0) { set_error("only the chord fit (0) is implemented"); return LS_E_INVALID; }
    if (c.big_threshold < 64 || c.big_threshold > CS_MAX) { set_error("big_threshold out of range [64, 4096]"); return LS_E_INVALID; }
    return LS_OK;
}

static void to_dev_model(const ls_model &h, DevModel &d) {
    memset(&d, 0, sizeof d);
    d.xmin = h.xmin;
    d.xmax = h.xmax;
    d.root_scale = h.root_scale;
    d.L = h.leaf_count;
    d.last = (double)(h.leaf_count - 1);
    d.degenerate = h.degenerate;
    d.n_sample = h.n_sample;
    for (uint32_t l = 0; l < h.leaf_count; l++) {
        d.leaf[5 * l + 0] = h.leaf[l].a;
        d.leaf[5 * l + 1] = h.leaf[l].c;
        d.leaf[5 * l + 2] = h.leaf[l].b;
        d.leaf[5 * l + 3] = h.leaf[l].lo;
        d.leaf[5 * l + 4] = h.leaf[l].hi;
    }
}

static void from_dev_model(const DevModel &d, int dtype, ls_model &h) {
    memset(&h, 0, sizeof h);
    h.dtype = (uint32_t)dtype;
    h.leaf_count = d.L;
    h.n_sample = d.n_sample;
    h.degenerate = d.degenerate;
    h.xmin = d.xmin;
    h.xmax = d.xmax;
    h.root_scale = d.root_scale;
    for (uint32_t l = 0; l < d.L && l < LS_MAX_LEAVES; l++) {
        h.leaf[l].a = d.leaf[5 * l + 0];
        h.leaf[l].c = d.leaf[5 * l + 1];
        h.leaf[l].b = d.leaf[5 * l + 2];
        h.leaf[l].lo = d.leaf[5 * l + 3];
        h.leaf[l].hi = d.leaf[5 * l + 4];
    }
}

// The model is monotone-safe (so the touch-up only needs collision groups, R15)
static bool model_ok(const ls_model &m, const ls_config &cfg) {
    const double PM = 1.0 - 0x1p-52;
    if (m.leaf_count < 1 || m.leaf_count > LS_MAX_LEAVES) return false;
    if (!(m.xmin <= m.xmax) || !(m.root_scale >= 0.0)) return false;
    if (!isfinite(m.xmin) || !isfinite(m.xmax) || !isfinite(m.root_scale)) return false;
    for (uint32_t l = 0; l < m.leaf_count; l++) {
        const ls_leaf &q = m.leaf[l];
        if (!isfinite(q.a) || !isfinite(q.b) || !isfinite(q.c) || !isfinite(q.lo) || !isfinite(q.hi)) return false;
        if (!(q.a >= 0.0) || !(q.lo >= 0.0) || !(q.lo <= q.hi) || !(q.hi <= PM)) return false;
        if (l + 1 < m.leaf_count && !(q.hi <= m.leaf[l + 1].lo)) return false;
    }
    (void)cfg;
    return true;
}

// NVTX ranges over the host-side enqueue of each phase (a profiler's timeline
// shows which launches belong to which step of Alg. 1/2; a no-op without a
// tool attached). Under graph capture they cover the capture, not the replay.
struct NvtxPhase {
    bool open = false;
    void next(const char *name) {
        if (open) nvtxRangePop();
        nvtxRangePushA(name);
        open = true;
    }
    ~NvtxPhase() {
        if (open) nvtxRangePop();
    }
};

struct Timer {
    bool on = false;
    bool external = false;  // under stream capture: event-record nodes of the graph
    cudaEvent_t ev[LS_NUM_PHASES + 1];
    int phase_of[LS_NUM_PHASES + 1];
    int k = 0;
    cudaStream_t st;
    void start(bool enable, cudaStream_t s) {
        on = enable;
        st = s;
        if (!on) return;
        for (int i = 0; i <= LS_NUM_PHASES; i++) cudaEventCreate(&ev[i]);
        cudaEventRecord(ev[0], st);
        k = 0;
    }
    // Under capture the event-record nodes sit on a branch of their own
    // (`tst`): node k waits for the main sequence up to its mark and for node
    // k-1, and nothing on the main sequence waits for it, so the kernels run
    // back to back as they do without phase timing (in line, the 9 nodes cost
    // ~0.06 ms per 200M-key sort). join() ties the branch back before the
    // capture ends.
    cudaStream_t tst = nullptr;
    void rec_external(int i) {
        cudaEvent_t d = nullptr;
        if (tst && cudaEventCreateWithFlags(&d, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventRecord(d, st) == cudaSuccess && cudaStreamWaitEvent(tst, d, 0) == cudaSuccess) {
            cudaEventRecordWithFlags(ev[i], tst, cudaEventRecordExternal);
            branched = true;
        } else {
            cudaGetLastError();
            cudaEventRecordWithFlags(ev[i], st, cudaEventRecordExternal);
        }
        if (d) cudaEventDestroy(d);
    }
    bool branched = false;
    void join() {
        cudaEvent_t d = nullptr;
        if (!on || !branched) return;
        if (cudaEventCreateWithFlags(&d, cudaEventDisableTiming) == cudaSuccess) {
            cudaEventRecord(d, tst);
            cudaStreamWaitEvent(st, d, 0);
            cudaEventDestroy(d);
        }
    }
    void mark(int phase) {
        if (!on) return;
        phase_of[k] = phase;
        if (external) rec_external(++k);
        else cudaEventRecord(ev[++k], st);
    }
    void finish(ls_stats *s) {
        if (!on) return;
        if (s)
            for (int i = 0; i < k; i++) {
                float ms = 0;
                cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
                s->phase_ms[phase_of[i]] += ms;
            }
        for (int i = 0; i <= LS_NUM_PHASES; i++) cudaEventDestroy(ev[i]);
        on = false;
    }
};

// Side streams per device (non-blocking), for work that runs beside the
// main sequence inside one sort (forked and joined with events; captured into
// the CUDA Graph as parallel branches). nullptr if one cannot be created.
constexpr int LS_NSIDE = 5;
static cudaStream_t side_stream(int k = 0) {
    constexpr int MAXD = 64;
    static cudaStream_t s[MAXD][LS_NSIDE + 1];  // (+ the phase-timing branch of a captured sequence)
    static std::once_flag once[MAXD];
    int d = -1;
    if (k < 0 || k > LS_NSIDE || cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAXD) {
        cudaGetLastError();
        return nullptr;
    }
    std::call_once(once[d], [d] {
        for (int j = 0; j <= LS_NSIDE; j++)
            if (cudaStreamCreateWithFlags(&s[d][j], cudaStreamNonBlocking) != cudaSuccess) {
                s[d][j] = nullptr;
                cudaGetLastError();
            }
    });
    return s[d][k];
}

// The launch sequence of one sort, from the workspace initialisation to the
// big path. Every data-dependent decision is taken on the device (task lists,
// counters in Ctl), so the sequence depends only on its arguments.
static ls_status launch_sequence(Args &a, const Layout &l, const ls_config &cfg, const ls_model *inject,
                                 const ls_dumps *dumps, int dt, void *d_ws, Timer &tm, cudaStream_t st,
                                 uint64_t &launches) {
    unsigned char *w = (unsigned char *)d_ws;
    LS_CUDA(cudaMemsetAsync(w + l.ff_begin, 0xff, l.ff_end - l.ff_begin, st));
    LS_CUDA(cudaMemsetAsync(w + l.zero_begin, 0, l.zero_end - l.zero_begin, st));
    NvtxPhase nv;
    nv.next("ls_sort: sample + fit");
    launch_init(a, st);
    launches++;
    if (inject) {
        std::unique_ptr<DevModel> dm(new DevModel);
        to_dev_model(*inject, *dm);
        LS_CUDA(cudaMemcpyAsync(a.M, dm.get(), sizeof(DevModel), cudaMemcpyHostToDevice, st));
        LS_CUDA(cudaStreamSynchronize(st));  // the staging buffer dies here
    } else {
        // north_star (1): strided sample (R9) + chord fit (R7)
        launch_sample_minmax(a.A, cfg.sample_stride, l.m, a.S, a.ctl, dt, st);
        launch_fit_hist(a.S, l.m, l.L, a.ctl, a.leaf_cnt, a.leaf_min, dt, st);
        launch_fit_params(l.m, l.L, a.ctl, a.leaf_cnt, a.leaf_min, a.M, dt, st);
        launches += 3;
    }
    // round 0 by reservation: bucket capacities from the sample (k_cap0),
    // then one scatter pass; the exact count pass (k_count0 + plan +
    // k_scatter0) runs only when a capacity did not hold (kernels exit early).
    // The capacities need only the model: they are computed on the side
    // stream while the b0 search tables are built
    {
        cudaStream_t s2 = side_stream();
        cudaEvent_t ef = nullptr, ej = nullptr;
        bool fork = s2 && cudaEventCreateWithFlags(&ef, cudaEventDisableTiming) == cudaSuccess &&
                    cudaEventCreateWithFlags(&ej, cudaEventDisableTiming) == cudaSuccess;
        if (fork) LS_CUDA(cudaEventRecord(ef, st));
        if (fork && cudaStreamWaitEvent(s2, ef, 0) != cudaSuccess) fork = false;  // (then all on st)
        if (!fork) cudaGetLastError();
        launch_cap0(a, l.m, dt, fork ? s2 : st);
        launch_b0_table(a.M, l.L, l.f, dt, st);
        launches += 5;
        if (fork) {
            LS_CUDA(cudaEventRecord(ej, s2));
            LS_CUDA(cudaStreamWaitEvent(st, ej, 0));
        }
        if (ef) cudaEventDestroy(ef);
        if (ej) cudaEventDestroy(ej);
    }
    tm.mark(LS_PHASE_FIT);
    nv.next("ls_sort: round 0 (scatter0r)");
    launch_scatter0r(a, dt, st);
    launch_plan0(a, dumps ? dumps->d_S_B : nullptr, 1, st);
    launches += 2;
    tm.mark(LS_PHASE_SCATTER0);
    nv.next("ls_sort: round 0 exact redo (count0 + scatter0)");
    launch_count0(a, dt, st);
    launch_plan0(a, dumps ? dumps->d_S_B : nullptr, 0, st);
    launch_scatter0(a, dt, st);
    launches += 3;
    tm.mark(LS_PHASE_COUNT0);
    nv.next("ls_sort: round 1 count (count1)");
    if (a.fr_min) {  // buckets that fit a CTA cluster: count + scatter of round 1 in one kernel
        launch_round1(a, dt, st);
        launches++;
    }
    launch_count1(a, dt, st);
    launches++;
    tm.mark(LS_PHASE_COUNT1);
    nv.next("ls_sort: classify");
    launch_classify(a, nullptr, st);  // also turns count1's per-unit counts into offsets
    launches++;
    tm.mark(LS_PHASE_CLASSIFY);
    nv.next("ls_sort: round 1 scatter (scatter1)");
    launch_scatter1(a, dt, st);
    launches++;
    tm.mark(LS_PHASE_SCATTER1);
    nv.next("ls_sort: in-bucket sort");
    if (dumps && dumps->d_S_B1)
        LS_CUDA(cudaMemcpyAsync(dumps->d_S_B1, a.hist1, (size_t)l.f * l.f * 4, cudaMemcpyDeviceToDevice, st));
    // in-bucket sort: k_warpsort on `st`, the CTA sorts and block windows
    // beside it on the device's side stream (disjoint sub-buckets; the few
    // CTA-sized tasks of smooth inputs are latency-bound, so serialised after
    // the warp sort they cost ~60 us); joined before the big path
    {
        // one side stream per CTA-sort shape (and one for the block windows):
        // k_warpsort's 4 CTAs per SM fill the register file, so a side kernel
        // queued behind another on one stream finds no SM until the warp sort
        // retires; on separate streams they all take their slots first
        cudaStream_t ss[LS_NSIDE];
        cudaEvent_t ef = nullptr, ej[LS_NSIDE] = {};
        bool fork = cudaEventCreateWithFlags(&ef, cudaEventDisableTiming) == cudaSuccess;
        for (int j = 0; j < LS_NSIDE; j++) {
            ss[j] = side_stream(j);
            fork = fork && ss[j] && cudaEventCreateWithFlags(&ej[j], cudaEventDisableTiming) == cudaSuccess;
        }
        if (fork) LS_CUDA(cudaEventRecord(ef, st));
        for (int j = 0; fork && j < LS_NSIDE; j++)
            if (cudaStreamWaitEvent(ss[j], ef, 0) != cudaSuccess) fork = false;  // (then all on st)
        if (!fork) {
            cudaGetLastError();
            for (int j = 0; j < LS_NSIDE; j++) ss[j] = st;
        }
        // (the side streams' kernels are enqueued first: their few working
        // CTAs take SM slots before the persistent warp sort fills them, whose
        // batched task tickets let late-starting warps simply take fewer)
        launch_bucketsort(a, dt, ss);
        launch_warpsort(a, dt, st);
        launches += 7;
        tm.mark(LS_PHASE_BUCKETSORT);
        nv.next("ls_sort: big path");  // (the warp sort; the rest is in the next phase if not hidden)
        if (fork)
            for (int j = 0; j < LS_NSIDE; j++) {
                LS_CUDA(cudaEventRecord(ej[j], ss[j]));
                LS_CUDA(cudaStreamWaitEvent(st, ej[j], 0));
            }
        if (ef) cudaEventDestroy(ef);
        for (int j = 0; j < LS_NSIDE; j++)
            if (ej[j]) cudaEventDestroy(ej[j]);
    }
    launch_big_minmax(a, dt, st);
    launches++;
    launch_large(a, dt, st);
    launches += 5;
    launch_big_order(a, st);
    launches++;
    launch_big(a, dt, st);
    launches++;
    tm.mark(LS_PHASE_BIG);
    LS_CUDA(cudaGetLastError());
    return LS_OK;
}

// CUDA Graph of the launch sequence. A sort is captured the
// second time the same (keys, n, dtype, config, workspace, device) comes back
// (one-shot calls run the sequence directly) and replayed with one
// cudaGraphLaunch from then on. Off with LS_GRAPH=0; LS_GRAPH=2 turns a failed
// capture into an error (tests). Never with an injected model (host sync) or
// dumps; with LS_FLAG_PHASE_TIMING the phase events are graph nodes.
struct GraphKey {
    void *keys, *ws;
    uint64_t n;
    ls_config cfg;
    int dt, dev;
    uint32_t fr_min, dbg, fx0;
    unsigned long long ctx;  // driver context id (cuCtxGetId): a graph never outlives its context
};
struct GraphEntry {
    GraphKey k;
    cudaGraphExec_t exec;  // null: seen once
    uint64_t launches, used;
    // LS_FLAG_PHASE_TIMING: the phase events are recorded by the graph's own
    // event-record nodes (owned here, read after each replay)
    bool timed;
    cudaEvent_t ev[LS_NUM_PHASES + 1];
    int phase_of[LS_NUM_PHASES + 1];
    int nmarks;
};

static void drop_graph(GraphEntry &g) {
    if (g.exec) cudaGraphExecDestroy(g.exec);  // (freed after in-flight launches)
    if (g.timed)
        for (int i = 0; i <= LS_NUM_PHASES; i++) cudaEventDestroy(g.ev[i]);
}
static std::mutex g_graph_mu;
static std::vector<GraphEntry> g_graphs;
static uint64_t g_graph_clock = 0;
constexpr size_t GRAPH_CACHE = 16;

static bool same_key(const GraphKey &x, const GraphKey &y) {
    return x.keys == y.keys && x.ws == y.ws && x.n == y.n && x.dt == y.dt && x.dev == y.dev &&
           x.ctx == y.ctx && x.fr_min == y.fr_min && x.dbg == y.dbg && x.fx0 == y.fx0 && !memcmp(&x.cfg, &y.cfg, sizeof x.cfg);
}

static bool graphs_enabled() {
    const char *e = getenv("LS_GRAPH");
    return !(e && e[0] == '0');
}

// Id of the current driver context (unique per context, also across a
// cudaDeviceReset that re-creates the primary context at the same address).
// Resolved through the runtime's driver entry point, so libls does not link
// libcuda. 0 = unknown (graphs are then not used).
static unsigned long long current_ctx_id() {
    typedef int (*GetCur)(void **);
    typedef int (*GetId)(void *, unsigned long long *);
    static GetCur get_cur = nullptr;
    static GetId get_id = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuCtxGetCurrent", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_cur = (GetCur)f;
        f = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuCtxGetId", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_id = (GetId)f;
        cudaGetLastError();
    });
    void *ctx = nullptr;
    unsigned long long id = 0;
    if (!get_cur || !get_id || get_cur(&ctx) != 0 || !ctx || get_id(ctx, &id) != 0) return 0;
    return id;
}

// Per-thread capture streams (one per device), recreated after a failed replay.
static thread_local cudaStream_t g_cap_stream[64] = {};

// Forget every cached graph and this thread's capture streams (after a replay
// launch failed: handles from a destroyed context are not reused). Errors from
// destroying stale handles are cleared afterwards.
static void drop_all_graphs() {
    for (auto &g : g_graphs) drop_graph(g);
    g_graphs.clear();
    for (auto &c : g_cap_stream)
        if (c) {
            cudaStreamDestroy(c);
            c = nullptr;
        }
    cudaGetLastError();
}

// Run the sequence through the graph cache; false = not handled (run it directly).
static bool launch_graph(Args &a, const Layout &l, const ls_config &cfg, int dt, const GraphKey &key,
                         cudaStream_t st, uint64_t &launches, ls_status &rc, Pending *pend) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    GraphEntry *e = nullptr;
    for (auto &g : g_graphs)
        if (same_key(g.k, key)) e = &g;
    if (!e) {  // first sight: remember it, run directly
        if (g_graphs.size() >= GRAPH_CACHE) {
            size_t lru = 0;
            for (size_t i = 1; i < g_graphs.size(); i++)
                if (g_graphs[i].used < g_graphs[lru].used) lru = i;
            drop_graph(g_graphs[lru]);
            g_graphs.erase(g_graphs.begin() + lru);
        }
        GraphEntry ne;
        memset(&ne, 0, sizeof ne);
        ne.k = key;
        ne.used = ++g_graph_clock;
        g_graphs.push_back(ne);
        return false;
    }
    e->used = ++g_graph_clock;
    if (!e->exec) {  // second sight: capture on a private stream
        cudaStream_t *cs = g_cap_stream;
        if (key.dev < 0 || key.dev >= 64) return false;
        if (!cs[key.dev] && cudaStreamCreateWithFlags(&cs[key.dev], cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        Timer cap;
        cap.on = (cfg.flags & LS_FLAG_PHASE_TIMING) != 0;
        cap.st = cs[key.dev];
        cap.k = 0;
        cap.external = true;
        if (cap.on)
            for (int i = 0; i <= LS_NUM_PHASES; i++) cudaEventCreate(&cap.ev[i]);
        auto drop_events = [&] {
            if (cap.on)
                for (int i = 0; i <= LS_NUM_PHASES; i++) cudaEventDestroy(cap.ev[i]);
        };
        if (cudaStreamBeginCapture(cs[key.dev], cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            drop_events();
            return false;
        }
        cap.tst = side_stream(LS_NSIDE);  // (the timing branch; nullptr: event nodes in line)
        if (cap.on) cap.rec_external(0);
        uint64_t nl = 0;
        const ls_status r = launch_sequence(a, l, cfg, nullptr, nullptr, dt, key.ws, cap, cs[key.dev], nl);
        cap.join();
        cudaGraph_t g = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(cs[key.dev], &g);
        cudaGraphExec_t x = nullptr;
        const bool ok = r == LS_OK && ec == cudaSuccess && g &&
                        cudaGraphInstantiate(&x, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        if (!ok) {  // (not capturable here: keep running it directly, unless LS_GRAPH=2)
            cudaGetLastError();
            drop_events();
            const char *gv = getenv("LS_GRAPH");
            if (gv && gv[0] == '2') {
                set_error("LS_GRAPH=2: capture of the launch sequence failed");
                rc = LS_E_CUDA;
                return true;
            }
            return false;
        }
        e->exec = x;
        e->launches = nl;
        e->timed = cap.on;
        if (cap.on) {
            memcpy(e->ev, cap.ev, sizeof cap.ev);
            memcpy(e->phase_of, cap.phase_of, sizeof cap.phase_of);
            e->nmarks = cap.k;
        }
    }
    cudaError_t le = cudaGraphLaunch(e->exec, st);
    if (const char *f = getenv("LS_TEST_GRAPH_LAUNCH_FAIL"))  // (test hook: force the fallback below)
        if (f[0] == '1') le = cudaErrorInvalidResourceHandle;
    if (le != cudaSuccess) {  // a stale graph (e.g. after a context reset): forget every cached
        drop_all_graphs();    // graph and capture stream, then launch the sequence directly
        return false;
    }
    launches = e->launches;
    pend->timer_on = e->timed;
    pend->own_events = false;
    if (e->timed) {
        memcpy(pend->ev, e->ev, sizeof e->ev);
        memcpy(pend->phase_of, e->phase_of, sizeof e->phase_of);
        pend->nmarks = e->nmarks;
    }
    rc = LS_OK;
    return true;
}

// Enqueue the whole sort. If `sync` the stream is synchronised and the status
// and stats are collected; otherwise the caller synchronises (ls_sort_host).
ls_status enqueue_sort(void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg_in,
                       const ls_model *inject, void *d_ws, size_t ws_bytes, cudaStream_t st,
                       ls_stats *stats, const ls_dumps *dumps, Pending *pend) {
    ls_config cfg;
    if (cfg_in) cfg = *cfg_in; else ls_config_default(&cfg);
    ls_status rc = check_config(cfg);
    if (rc != LS_OK) return rc;
    if (dtype != LS_F64 && dtype != LS_U64) { set_error("bad dtype"); return LS_E_INVALID; }
    if (n >= (1ull << 32)) { set_error("n must be < 2^32"); return LS_E_INVALID; }
    if (stats) memset(stats, 0, sizeof *stats);
    if (stats) stats->n = n;
    if (n <= 1) return LS_OK;
    if (!d_keys || !d_ws) { set_error("null pointer"); return LS_E_INVALID; }
    // the bulk-copy (TMA) stages and 16-byte vector loads address keys in aligned pairs
    if (((uintptr_t)d_keys & 15) || ((uintptr_t)d_ws & 255)) {
        set_error("keys must be 16-byte aligned and the workspace 256-byte aligned");
        return LS_E_INVALID;
    }
    if (inject && !model_ok(*inject, cfg)) { set_error("injected model is not monotone-safe"); return LS_E_INVALID; }
    const Layout l = make_layout(n, cfg);
    if (ws_bytes < l.total) { set_error("workspace too small"); return LS_E_WORKSPACE; }
    Args a = make_args(l, d_keys, d_ws);
    if (const char *e = getenv("LS_DEBUG_STAGE")) a.dbg = (uint32_t)atoi(e);
    // cluster-resident round 1 with LS_FLAG_FUSED_ROUND1; LS_FR_MIN
    // overrides the smallest bucket it takes (tests)
    a.fr_cap = (cfg.flags & LS_FLAG_FUSED_ROUND1) ? round1_capacity() : 0u;
    a.fr_min = a.fr_cap ? FR_MIN_DEFAULT : 0u;
    // round 0 by the exact count pass: with the cluster-resident round 1 (it
    // reads buckets at start0), or forced (LS_EXACT0=1, tests)
    if (a.fr_cap) a.force_exact0 = 1;
    if (const char *e = getenv("LS_EXACT0")) if (e[0] == '1') a.force_exact0 = 1;
    if (const char *e = getenv("LS_FR_MIN")) a.fr_min = a.fr_cap ? (uint32_t)atoi(e) : 0u;
    const int dt = (int)dtype;
    if (dumps) {
        a.dH0 = dumps->d_H0;
        a.dH1 = dumps->d_H1;
        if (a.dH0) LS_CUDA(cudaMemsetAsync(a.dH0, 0, (size_t)l.f, st));
        if (a.dH1) LS_CUDA(cudaMemsetAsync(a.dH1, 0, (size_t)l.f * l.f, st));
    }
    uint64_t launches = 0;
    bool done = false;
    pend->timer_on = false;
    pend->own_events = true;
    if (!inject && !dumps && !a.dbg && graphs_enabled()) {
        GraphKey key;
        memset(&key, 0, sizeof key);
        key.keys = d_keys;
        key.ws = d_ws;
        key.n = n;
        key.cfg = cfg;
        key.dt = dt;
        LS_CUDA(cudaGetDevice(&key.dev));
        key.fr_min = a.fr_min;
        key.dbg = a.dbg;
        key.fx0 = a.force_exact0;
        key.ctx = current_ctx_id();
        ls_status grc = LS_OK;
        if (key.ctx) done = launch_graph(a, l, cfg, dt, key, st, launches, grc, pend);
        if (done && grc != LS_OK) return grc;
    }
    if (!done) {
        Timer tm;
        tm.start(cfg.flags & LS_FLAG_PHASE_TIMING, st);
        const ls_status lrc = launch_sequence(a, l, cfg, inject, dumps, dt, d_ws, tm, st, launches);
        if (lrc != LS_OK) return lrc;
        pend->timer_on = tm.on;
        if (tm.on) {
            memcpy(pend->ev, tm.ev, sizeof tm.ev);
            memcpy(pend->phase_of, tm.phase_of, sizeof tm.phase_of);
            pend->nmarks = tm.k;
        }
    }
    pend->ctl_dev = a.ctl;
    pend->model_dev = a.M;
    pend->launches = launches;
    pend->dtype = dt;
    LS_CUDA(cudaMemcpyAsync(&pend->ctl_host, a.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    if (dumps && dumps->h_model) {
        pend->model_host.reset(new DevModel);
        LS_CUDA(cudaMemcpyAsync(pend->model_host.get(), a.M, sizeof(DevModel), cudaMemcpyDeviceToHost, st));
        pend->model_out = dumps->h_model;
    }
    pend->active = true;
    return LS_OK;
}

ls_status finish_sort(Pending *pend, cudaStream_t st, ls_stats *stats) {
    if (!pend->active) return LS_OK;
    pend->active = false;
    LS_CUDA(cudaStreamSynchronize(st));
    const Ctl &c = pend->ctl_host;
    if (stats) {
        stats->h0_buckets = c.stat[ST_H0B];
        stats->h0_keys = c.stat[ST_H0K];
        stats->h1_subbuckets = c.stat[ST_H1S];
        stats->h1_keys = c.stat[ST_H1K];
        stats->small_subbuckets = c.stat[ST_SMALLS];
        stats->small_keys = c.stat[ST_SMALLK];
        stats->big_subbuckets = c.stat[ST_BIGS];
        stats->big_keys = c.stat[ST_BIGK];
        stats->max_group = c.stat[ST_MAXGRP];
        stats->big_passes = c.stat[ST_BIGPASS];
        stats->kernel_launches = pend->launches;
        stats->fused_buckets = c.nfused;
        stats->round0_exact = c.exact0;
    }
    if (pend->timer_on) {
        if (stats)
            for (int i = 0; i < pend->nmarks; i++) {
                float ms = 0;
                cudaEventElapsedTime(&ms, pend->ev[i], pend->ev[i + 1]);
                stats->phase_ms[pend->phase_of[i]] += ms;
            }
        if (pend->own_events)
            for (int i = 0; i <= LS_NUM_PHASES; i++) cudaEventDestroy(pend->ev[i]);
    }
    if (pend->model_out && pend->model_host) from_dev_model(*pend->model_host, pend->dtype, *pend->model_out);
    if (getenv("LS_DEBUG_STAGE")) {
        fprintf(stderr, "prof:");
        for (int i = 0; i < 16; i++) fprintf(stderr, " %llu", c.prof[i]);
        fprintf(stderr, "\ntasks: warp %u cta4096 %u cta2048 %u cta1024 %u cta512 %u windows %u large %u\n",
                c.ntask, c.nctask, c.nctask2, c.nctask3, c.nctask4, c.nwin, c.nlarge);
        fprintf(stderr, "big items per level: %u %u %u %u (first pass %u)\n", c.big_cnt[0], c.big_cnt[1],
                c.big_cnt[2], c.big_cnt[3], c.big_lv0);
        if (pend->model_dev) {
            uint32_t ns = 0;
            cudaMemcpy(&ns, &pend->model_dev->nsub, 4, cudaMemcpyDeviceToHost);
            fprintf(stderr, "b0 refined cells: %u\n", ns);
        }
    }
    if (c.status & STATUS_NAN) { set_error("NaN key in input (S:214)"); return LS_E_NAN; }
    if (c.status & STATUS_INTERNAL) { set_error("internal invariant violated (corrupt partition state)"); return LS_E_INTERNAL; }
    return LS_OK;
}

size_t workspace_bytes(uint64_t n, const ls_config &cfg) { return make_layout(n, cfg).total; }

}  // namespace ls

using namespace ls;

extern "C" {

void ls_config_default(ls_config *c) {
    memset(c, 0, sizeof *c);
    c->fanout = 1000;
    c->leaf_count = 1000;
    c->sample_stride = 100; // P:328 1% sample (R9)
    c->fit = 0;
    c->big_threshold = 4096;
    c->flags = 0;
}

const char *ls_status_string(ls_status s) {
    switch (s) {
    case LS_OK: return "LS_OK";
    case LS_E_INVALID: return "LS_E_INVALID";
    case LS_E_NAN: return "LS_E_NAN";
    case LS_E_WORKSPACE: return "LS_E_WORKSPACE";
    case LS_E_CAPACITY: return "LS_E_CAPACITY";
    case LS_E_CUDA: return "LS_E_CUDA";
    case LS_E_NCCL: return "LS_E_NCCL";
    case LS_E_INTERNAL: return "LS_E_INTERNAL";
    }
    return "LS_E_UNKNOWN";
}

const char *ls_last_error(void) { return g_err.c_str(); }

ls_status ls_workspace_bytes(uint64_t n, ls_dtype dtype, const ls_config *cfg_in, size_t *bytes) {
    ls_config cfg;
    if (cfg_in) cfg = *cfg_in; else ls_config_default(&cfg);
    ls_status rc = check_config(cfg);
    if (rc != LS_OK) return rc;
    if (dtype != LS_F64 && dtype != LS_U64) return LS_E_INVALID;
    if (!bytes) return LS_E_INVALID;
    *bytes = workspace_bytes(n, cfg);
    return LS_OK;
}

ls_status ls_sort(void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg, void *d_ws,
                  size_t ws_bytes, void *stream, ls_stats *stats, const ls_dumps *dumps) {
    Pending p;
    cudaStream_t st = (cudaStream_t)stream;
    ls_status rc = enqueue_sort(d_keys, n, dtype, cfg, nullptr, d_ws, ws_bytes, st, stats, dumps, &p);
    if (rc != LS_OK) return rc;
    return finish_sort(&p, st, stats);
}

ls_status ls_sort_with_model(void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg,
                             const ls_model *model, void *d_ws, size_t ws_bytes, void *stream,
                             ls_stats *stats, const ls_dumps *dumps) {
    if (!model) { set_error("null model"); return LS_E_INVALID; }
    Pending p;
    cudaStream_t st = (cudaStream_t)stream;
    ls_status rc = enqueue_sort(d_keys, n, dtype, cfg, model, d_ws, ws_bytes, st, stats, dumps, &p);
    if (rc != LS_OK) return rc;
    return finish_sort(&p, st, stats);
}

ls_status ls_sort_host(void *h_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg, void *d_buf,
                       void *d_ws, size_t ws_bytes, void *stream, ls_stats *stats) {
    if (stats) {
        memset(stats, 0, sizeof *stats);
        stats->n = n;
    }
    if (n <= 1) return LS_OK;  // (no copies: nothing is left in flight on return)
    if (!h_keys || !d_buf) { set_error("null pointer"); return LS_E_INVALID; }
    cudaStream_t st = (cudaStream_t)stream;
    LS_CUDA(cudaMemcpyAsync(d_buf, h_keys, n * 8, cudaMemcpyHostToDevice, st));
    Pending p;
    ls_status rc = enqueue_sort(d_buf, n, dtype, cfg, nullptr, d_ws, ws_bytes, st, stats, nullptr, &p);
    if (rc != LS_OK) return rc;
    LS_CUDA(cudaMemcpyAsync(h_keys, d_buf, n * 8, cudaMemcpyDeviceToHost, st));
    return finish_sort(&p, st, stats);
}

ls_status ls_train_rmi(const void *d_sample, uint64_t m, ls_dtype dtype, const ls_config *cfg_in,
                       ls_model *out, void *d_ws, size_t ws_bytes, void *stream) {
    ls_config cfg;
    if (cfg_in) cfg = *cfg_in; else ls_config_default(&cfg);
    ls_status rc = check_config(cfg);
    if (rc != LS_OK) return rc;
    if (!out || !d_ws || (m && !d_sample)) { set_error("null pointer"); return LS_E_INVALID; }
    if (m == 0) { set_error("empty sample (S:59)"); return LS_E_INVALID; }
    if (dtype != LS_F64 && dtype != LS_U64) return LS_E_INVALID;
    const Layout l = make_layout(m, cfg);  // (the sample buffer S of the layout is unused)
    if (ws_bytes < l.total) { set_error("workspace too small"); return LS_E_WORKSPACE; }
    Args a = make_args(l, nullptr, d_ws);
    cudaStream_t st = (cudaStream_t)stream;
    unsigned char *w = (unsigned char *)d_ws;
    LS_CUDA(cudaMemsetAsync(w + l.ff_begin, 0xff, l.ff_end - l.ff_begin, st));
    LS_CUDA(cudaMemsetAsync(w + l.zero_begin, 0, l.zero_end - l.zero_begin, st));
    launch_init(a, st);
    const uint64_t *S = (const uint64_t *)d_sample;
    launch_sample_minmax(S, 1, m, nullptr, a.ctl, (int)dtype, st);
    launch_fit_hist(S, m, l.L, a.ctl, a.leaf_cnt, a.leaf_min, (int)dtype, st);
    launch_fit_params(m, l.L, a.ctl, a.leaf_cnt, a.leaf_min, a.M, (int)dtype, st);
    LS_CUDA(cudaGetLastError());
    std::unique_ptr<DevModel> dm(new DevModel);
    LS_CUDA(cudaMemcpyAsync(dm.get(), a.M, sizeof(DevModel), cudaMemcpyDeviceToHost, st));
    LS_CUDA(cudaStreamSynchronize(st));
    from_dev_model(*dm, (int)dtype, *out);
    return LS_OK;
}

ls_status ls_bucket_ids(const void *d_keys, uint64_t n, ls_dtype dtype, const ls_config *cfg_in,
                        const ls_model *model, double *d_p, uint32_t *d_b0, uint32_t *d_b1,
                        uint32_t *d_pos, uint64_t *d_hist0, uint64_t *d_hist1, void *d_ws,
                        size_t ws_bytes, void *stream) {
    ls_config cfg;
    if (cfg_in) cfg = *cfg_in; else ls_config_default(&cfg);
    ls_status rc = check_config(cfg);
    if (rc != LS_OK) return rc;
    if (!model || !d_ws) { set_error("null pointer"); return LS_E_INVALID; }
    if (!model_ok(*model, cfg)) { set_error("model is not monotone-safe"); return LS_E_INVALID; }
    if (dtype != LS_F64 && dtype != LS_U64) return LS_E_INVALID;
    const Layout l = make_layout(n, cfg);
    if (ws_bytes < l.total) { set_error("workspace too small"); return LS_E_WORKSPACE; }
    unsigned char *w = (unsigned char *)d_ws;
    cudaStream_t st = (cudaStream_t)stream;
    DevModel *M = (DevModel *)(w + l.model);
    std::unique_ptr<DevModel> dm(new DevModel);
    to_dev_model(*model, *dm);
    LS_CUDA(cudaMemcpyAsync(M, dm.get(), sizeof(DevModel), cudaMemcpyHostToDevice, st));
    const size_t ff = (size_t)l.f * l.f;
    unsigned long long *h1 = d_hist1 ? (unsigned long long *)d_hist1 : (unsigned long long *)(w + l.hist1_u64);
    unsigned long long *h0 = (unsigned long long *)d_hist0;
    if (h0) LS_CUDA(cudaMemsetAsync(h0, 0, (size_t)l.f * 8, st));
    const bool need_h1 = d_hist1 || d_pos;
    if (need_h1) LS_CUDA(cudaMemsetAsync(h1, 0, ff * 8, st));
    if (n) {
        launch_bucket_ids((const uint64_t *)d_keys, n, l.f, M, d_p, d_b0, d_b1, h0,
                          need_h1 ? h1 : nullptr, (int)dtype, st);
        if (d_pos) launch_bucket_pos((const uint64_t *)d_keys, n, l.f, M, h1, d_pos, (int)dtype, st);
    }
    LS_CUDA(cudaGetLastError());
    LS_CUDA(cudaStreamSynchronize(st));
    return LS_OK;
}

}  // extern "C"
