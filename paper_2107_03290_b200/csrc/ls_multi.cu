// ls_multi.cu -- SURVEY §8(e): sample-based global range split across GPUs.
//
// The paper is sequential (P:414 leaves parallel execution to future work);
// this is the multi-GPU extension named by north_star: every rank samples its
// shard, the samples are all-gathered (NCCL), R-1 splitters are chosen on the
// lexicographic key (ord(x), rank, index) -- so runs of equal keys may
// straddle ranks and a heavy duplicate cannot overload one rank -- each key is
// routed to its destination rank by a count + decoupled-lookback + scatter
// pass (the same machinery as a partition round, with R buckets), the shards
// are exchanged with a grouped NCCL send/recv all-to-all over NVLink, and each
// rank sorts what it received with the single-GPU path (local model refit).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "ls.h"
#include "ls_api_internal.h"
#include "ls_launch.h"
#include "ls_tile.cuh"
#include "ls_tilepart.cuh"

struct ls_comm {
    ncclComm_t comm;
    int rank, world;
    // LS_FLAG_PEER_SCATTER: the peers' d_out as mapped here (CUDA IPC), keyed
    // by the exchanged (allocation handle, offset) so a reused buffer is
    // opened once
    struct Peer {
        cudaIpcMemHandle_t h;
        uint64_t off;
        void *base;  // cudaIpcOpenMemHandle result (nullptr: not open)
    } peer[64];
};

namespace ls {

constexpr int SPLIT_K = LS_MULTI_SAMPLE;  // sample entries per rank
constexpr uint32_t MULTI_UNIT = 65536;
constexpr int MAX_WORLD = 64;

struct Tagged {
    unsigned long long ord;
    uint32_t rank, pad;
    unsigned long long index;
};
static_assert(sizeof(Tagged) == sizeof(ls_tagged), "tagged layout");

// Destination of (o, r, i): the number of splitters strictly below it in the
// lexicographic order (ord, rank, index). Monotone, so rank p receives a
// contiguous slice of the global order.
__host__ __device__ __forceinline__ int dest_of(const Tagged *spl, int world,
                                                unsigned long long o, uint32_t r,
                                                unsigned long long i) {
    int d = 0;
    for (int k = 0; k < world - 1; k++) {
        const Tagged &s = spl[k];
        const bool below = s.ord < o || (s.ord == o && (s.rank < r || (s.rank == r && s.index < i)));
        d += below ? 1 : 0;
    }
    return d;
}

template <int DT>
__global__ void k_split_sample(const uint64_t *__restrict__ in, uint64_t n, uint32_t rank,
                               Tagged *out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= SPLIT_K) return;
    Tagged t;
    const uint64_t valid = n < (uint64_t)SPLIT_K ? n : (uint64_t)SPLIT_K;
    if ((uint64_t)k < valid) {
        const uint64_t idx = n <= (uint64_t)SPLIT_K ? (uint64_t)k : (uint64_t)k * n / SPLIT_K;
        const uint64_t b = in[idx];
        t.ord = to_ord<DT>(b);
        t.rank = rank;
        t.pad = 0;
        t.index = idx;
    } else {
        t.ord = ~0ull;
        t.rank = 0xffffffffu;
        t.pad = 0;
        t.index = ~0ull;
    }
    out[k] = t;
}

struct MultiArgs {
    const uint64_t *in;
    uint64_t *send;
    uint64_t n;
    uint32_t rank;
    int world;
    uint32_t U;
    const Tagged *spl;              // [world-1]
    unsigned long long *lb;         // [U*world]
    uint32_t *offs;                 // [U*world]
    unsigned long long *counts;     // [world] + status
    const unsigned long long *sdispl; // [world]
    uint32_t *ticket;
};

// Per destination rank: its receive buffer as seen from this GPU and where
// this rank's keys start in it.
struct PeerDst {
    uint64_t *ptr[MAX_WORLD];
    uint64_t off[MAX_WORLD];
};

template <int DT>
struct DestBucket {
    const Tagged *spl;
    int world;
    uint32_t rank;
    __device__ __forceinline__ uint32_t operator()(uint64_t key, uint64_t idx) const {
        return (uint32_t)dest_of(spl, world, to_ord<DT>(key), rank, idx);
    }
};

template <int DT>
__global__ void __launch_bounds__(512) k_dest_count(MultiArgs a) {
    __shared__ Tagged spl[MAX_WORLD];
    __shared__ uint32_t hist[MAX_WORLD];
    __shared__ uint32_t s_unit;
    __shared__ int s_nan;
    const int tid = threadIdx.x, bd = blockDim.x, R = a.world;
    if (tid == 0) {
        s_unit = atomicAdd(a.ticket, 1u);
        s_nan = 0;
    }
    if (tid < R - 1) spl[tid] = a.spl[tid];
    if (tid < R) hist[tid] = 0;
    __syncthreads();
    const uint64_t u = s_unit;
    const uint64_t beg = u * MULTI_UNIT, end = umin64(a.n, beg + MULTI_UNIT);
    bool nan = false;
    for (uint64_t i = beg + tid; i < end; i += bd) {
        const uint64_t key = a.in[i];
        if (DT == DT_F64 && is_nan_bits(key)) nan = true;
        atomicAdd(&hist[dest_of(spl, R, to_ord<DT>(key), a.rank, i)], 1u);
    }
    if (nan) s_nan = 1;
    __syncthreads();
    if (tid == 0 && s_nan) atomicOr((unsigned int *)&a.counts[R], 1u);
    for (int b = tid; b < R; b += bd) {
        const uint32_t c = hist[b];
        if (c) atomicAdd(&a.counts[b], (unsigned long long)c);
        a.offs[u * R + b] = lookback(a.lb, u, 0, R, b, c);
    }
}

// Scatter by destination rank into the send buffer: the TMA tile engine
// (ls_tilepart.cuh) with R <= 64 buckets, so runs are long and coalesced.
struct DestSmem {
    TpSmem tp;
    uint32_t base[LS_MAX_FANOUT];
    Tagged spl[MAX_WORLD];
};

template <int DT>
__global__ void __launch_bounds__(TP_THREADS, 1) k_dest_scatter(MultiArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DestSmem &S = *reinterpret_cast<DestSmem *>(smem_raw);
    const int tid = threadIdx.x, R = a.world;
    const uint64_t u = blockIdx.x;
    if (tid < R - 1) S.spl[tid] = a.spl[tid];
    if (tid < R) S.base[tid] = (uint32_t)a.sdispl[tid] + a.offs[u * R + tid];
    tp_init(S.tp);
    const uint64_t beg = u * MULTI_UNIT, end = umin64(a.n, beg + MULTI_UNIT);
    const DestBucket<DT> bf{S.spl, R, a.rank};
    uint32_t phase = 0;
    tile_partition(S.tp, a.in, a.send, beg, end, a.n, S.base, R, bf, phase);
}

// the destination scatter fused with the exchange. Bucket p
// = destination rank p; its runs are stored straight into rank p's receive
// buffer (pdst[p], another GPU's HBM mapped through CUDA IPC: NVLink peer
// stores) at this rank's slice of it, so there is no send buffer and no NCCL
// all-to-all (-16 B/key of HBM traffic on each side), and the transfer
// overlaps the partition work tile by tile.
struct PeerSmem {
    TpSmem tp;
    uint32_t base[LS_MAX_FANOUT];
    Tagged spl[MAX_WORLD];
    uint64_t *pdst[MAX_WORLD];
};

template <int DT>
__global__ void __launch_bounds__(TP_THREADS, 1) k_dest_scatter_peer(MultiArgs a, PeerDst pd) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PeerSmem &S = *reinterpret_cast<PeerSmem *>(smem_raw);
    const int tid = threadIdx.x, R = a.world;
    const uint64_t u = blockIdx.x;
    if (tid < R - 1) S.spl[tid] = a.spl[tid];
    if (tid < R) {
        S.base[tid] = (uint32_t)pd.off[tid] + a.offs[u * R + tid];
        S.pdst[tid] = pd.ptr[tid];
    }
    tp_init(S.tp);
    const uint64_t beg = u * MULTI_UNIT, end = umin64(a.n, beg + MULTI_UNIT);
    const DestBucket<DT> bf{S.spl, R, a.rank};
    uint32_t phase = 0;
    tile_partition<false, false, false, DestBucket<DT>, TP_THREADS, TP_KPT, TpBids, false, true>(
        S.tp, a.in, nullptr, beg, end, a.n, S.base, R, bf, phase, nullptr, nullptr, nullptr, nullptr, S.pdst);
}

static void launch_dest_scatter_peer(const MultiArgs &a, const PeerDst &pd, int dt, cudaStream_t st) {
    const size_t sm = sizeof(PeerSmem);
    if (dt == DT_F64) {
        cudaFuncSetAttribute(k_dest_scatter_peer<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_dest_scatter_peer<DT_F64><<<a.U, TP_THREADS, sm, st>>>(a, pd);
    } else {
        cudaFuncSetAttribute(k_dest_scatter_peer<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_dest_scatter_peer<DT_U64><<<a.U, TP_THREADS, sm, st>>>(a, pd);
    }
}

static bool tagged_lt(const ls_tagged &x, const ls_tagged &y) {
    if (x.ord != y.ord) return x.ord < y.ord;
    if (x.rank != y.rank) return x.rank < y.rank;
    return x.index < y.index;
}

static size_t al(size_t x) { return (x + 255) / 256 * 256; }

struct MultiLayout {
    size_t send, samp, gath, spl, lb, offs, counts, allcounts, sdispl, ticket, xchg, local, total;
    uint32_t U;
};

// LS_FLAG_PEER_SCATTER: what every rank publishes about its d_out
struct PeerXchg {
    cudaIpcMemHandle_t h;  // of the allocation that holds d_out
    uint64_t off;          // d_out - allocation base
    uint64_t ok;           // 1: the handle could be exported
    uint64_t pad[6];
};

static MultiLayout multi_layout(uint64_t n_in, uint64_t out_cap, int R, const ls_config &cfg) {
    MultiLayout l;
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = al(off); off = o + b; return o; };
    l.U = (uint32_t)((n_in + MULTI_UNIT - 1) / MULTI_UNIT);
    if (l.U == 0) l.U = 1;
    l.ticket = take(256);
    l.counts = take((size_t)(R + 2) * 8);
    l.lb = take((size_t)l.U * R * 8);
    const size_t zero_end = off;
    (void)zero_end;
    l.send = take((size_t)n_in * 8);
    l.samp = take((size_t)SPLIT_K * sizeof(Tagged));
    l.gath = take((size_t)SPLIT_K * R * sizeof(Tagged));
    l.spl = take((size_t)MAX_WORLD * sizeof(Tagged));
    l.offs = take((size_t)l.U * R * 4);
    l.allcounts = take((size_t)(R + 2) * R * 8);
    l.sdispl = take((size_t)R * 8);
    l.xchg = take((size_t)(R + 1) * sizeof(PeerXchg));  // (+1: the barrier word)
    l.local = al(off);
    l.total = l.local + workspace_bytes(out_cap > 1 ? out_cap : 2, cfg);
    return l;
}

// Base of the allocation that holds p (the driver's cuMemGetAddressRange,
// reached through the runtime: libls does not link libcuda).
static cudaError_t alloc_base(const void *p, uint64_t *base) {
    typedef CUresult (*RangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);
    static RangeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess || !f) return e != cudaSuccess ? e : cudaErrorNotSupported;
        fn = (RangeFn)f;
    }
    CUdeviceptr b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, (CUdeviceptr)p) != CUDA_SUCCESS) return cudaErrorInvalidValue;
    *base = (uint64_t)b;
    return cudaSuccess;
}

}  // namespace ls

using namespace ls;

#define NCCL_CHECK(call)                                                  \
    do {                                                                  \
        ncclResult_t r_ = (call);                                         \
        if (r_ != ncclSuccess) {                                          \
            set_error(ncclGetErrorString(r_));                            \
            return LS_E_NCCL;                                             \
        }                                                                 \
    } while (0)
#define CUDA_CHECK(call)                                                  \
    do {                                                                  \
        cudaError_t e_ = (call);                                          \
        if (e_ != cudaSuccess) {                                          \
            set_error(cudaGetErrorString(e_));                            \
            return LS_E_CUDA;                                             \
        }                                                                 \
    } while (0)

extern "C" {

ls_status ls_multi_splitters(ls_tagged *h_entries, uint64_t count, int world, ls_tagged *h_splitters) {
    if (world < 1 || world > MAX_WORLD || (count && !h_entries) || (world > 1 && !h_splitters)) {
        set_error("bad arguments");
        return LS_E_INVALID;
    }
    // sentinel entries (rank 0xffffffff) go last; then only the R-1 order
    // statistics are needed: successive nth_element calls, each on the part
    // right of the previous one (O(count log R) instead of a full sort)
    ls_tagged *mid = std::partition(h_entries, h_entries + count,
                                    [](const ls_tagged &e) { return e.rank != 0xffffffffu; });
    const uint64_t valid = (uint64_t)(mid - h_entries);
    {
        uint64_t from = 0;
        for (int k = 1; k < world && valid; k++) {
            const uint64_t q = (uint64_t)k * valid / (uint64_t)world;
            if (q < from) continue;  // (same rank as the previous splitter)
            std::nth_element(h_entries + from, h_entries + q, h_entries + valid, tagged_lt);
            from = q + 1;
        }
    }
    for (int k = 1; k < world; k++) {
        if (valid == 0) {
            h_splitters[k - 1].ord = ~0ull;
            h_splitters[k - 1].rank = 0xffffffffu;
            h_splitters[k - 1].pad = 0;
            h_splitters[k - 1].index = ~0ull;
        } else {
            h_splitters[k - 1] = h_entries[(uint64_t)k * valid / (uint64_t)world];
        }
    }
    return LS_OK;
}

ls_status ls_multi_plan(const uint64_t *h_counts, int world, int rank, uint64_t *h_send_displ,
                        uint64_t *h_recv_counts, uint64_t *h_recv_displ, uint64_t *n_out) {
    if (world < 1 || rank < 0 || rank >= world || !h_counts) { set_error("bad arguments"); return LS_E_INVALID; }
    uint64_t s = 0;
    for (int p = 0; p < world; p++) {
        if (h_send_displ) h_send_displ[p] = s;
        s += h_counts[(uint64_t)rank * world + p];
    }
    uint64_t r = 0;
    for (int p = 0; p < world; p++) {
        const uint64_t c = h_counts[(uint64_t)p * world + rank];
        if (h_recv_counts) h_recv_counts[p] = c;
        if (h_recv_displ) h_recv_displ[p] = r;
        r += c;
    }
    if (n_out) *n_out = r;
    return LS_OK;
}

int ls_multi_dest(const ls_tagged *h_splitters, int world, uint64_t ord, uint32_t rank, uint64_t index) {
    return dest_of((const Tagged *)h_splitters, world, ord, rank, index);
}

ls_status ls_comm_unique_id(uint8_t id[LS_UNIQUE_ID_BYTES]) {
    static_assert(sizeof(ncclUniqueId) == LS_UNIQUE_ID_BYTES, "nccl id size");
    ncclUniqueId u;
    NCCL_CHECK(ncclGetUniqueId(&u));
    memcpy(id, &u, sizeof u);
    return LS_OK;
}

ls_status ls_comm_init(const uint8_t id[LS_UNIQUE_ID_BYTES], int rank, int world, ls_comm **out) {
    if (!out || world < 1 || world > MAX_WORLD || rank < 0 || rank >= world) { set_error("bad arguments"); return LS_E_INVALID; }
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    ls_comm *c = new ls_comm();
    c->rank = rank;
    c->world = world;
    ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
    if (r != ncclSuccess) {
        set_error(ncclGetErrorString(r));
        delete c;
        return LS_E_NCCL;
    }
    *out = c;
    return LS_OK;
}

void ls_comm_destroy(ls_comm *comm) {
    if (!comm) return;
    for (int p = 0; p < MAX_WORLD; p++)
        if (comm->peer[p].base) cudaIpcCloseMemHandle(comm->peer[p].base);
    ncclCommDestroy(comm->comm);
    delete comm;
}

ls_status ls_multi_workspace_bytes(uint64_t n_in, uint64_t out_cap, int world, ls_dtype dtype,
                                   const ls_config *cfg_in, size_t *bytes) {
    ls_config cfg;
    if (cfg_in) cfg = *cfg_in; else ls_config_default(&cfg);
    if (!bytes || world < 1 || world > MAX_WORLD || (dtype != LS_F64 && dtype != LS_U64)) return LS_E_INVALID;
    if (ls_status rc = check_config(cfg)) return rc;  // (before any layout arithmetic)
    *bytes = multi_layout(n_in, out_cap, world, cfg).total;
    return LS_OK;
}

ls_status ls_sort_multi(ls_comm *comm, const void *d_in, uint64_t n_in, void *d_out,
                        uint64_t out_cap, uint64_t *n_out, ls_dtype dtype, const ls_config *cfg_in,
                        void *d_ws, size_t ws_bytes, void *stream, ls_stats *stats) {
    ls_config cfg;
    if (cfg_in) cfg = *cfg_in; else ls_config_default(&cfg);
    if (ls_status rc = check_config(cfg)) return rc;  // (before any layout work or collective)
    if (!comm || !n_out || !d_ws || (n_in && !d_in) || (out_cap && !d_out)) { set_error("null pointer"); return LS_E_INVALID; }
    if (dtype != LS_F64 && dtype != LS_U64) { set_error("bad dtype"); return LS_E_INVALID; }
    if (n_in >= (1ull << 32) || out_cap >= (1ull << 32)) { set_error("n must be < 2^32"); return LS_E_INVALID; }
    if (((uintptr_t)d_in & 15) || ((uintptr_t)d_out & 15) || ((uintptr_t)d_ws & 255)) {
        set_error("keys / output must be 16-byte aligned and the workspace 256-byte aligned");
        return LS_E_INVALID;
    }
    const int R = comm->world, me = comm->rank;
    const MultiLayout l = multi_layout(n_in, out_cap, R, cfg);
    if (ws_bytes < l.total) { set_error("workspace too small"); return LS_E_WORKSPACE; }
    cudaStream_t st = (cudaStream_t)stream;
    unsigned char *w = (unsigned char *)d_ws;
    const int dt = (int)dtype;
    // 1. split sample + all-gather
    Tagged *samp = (Tagged *)(w + l.samp), *gath = (Tagged *)(w + l.gath);
    if (dt == DT_F64) k_split_sample<DT_F64><<<(SPLIT_K + 255) / 256, 256, 0, st>>>((const uint64_t *)d_in, n_in, (uint32_t)me, samp);
    else k_split_sample<DT_U64><<<(SPLIT_K + 255) / 256, 256, 0, st>>>((const uint64_t *)d_in, n_in, (uint32_t)me, samp);
    NCCL_CHECK(ncclAllGather(samp, gath, SPLIT_K * sizeof(Tagged), ncclUint8, comm->comm, st));
    std::vector<ls_tagged> h((size_t)SPLIT_K * R);
    CUDA_CHECK(cudaMemcpyAsync(h.data(), gath, h.size() * sizeof(Tagged), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    // 2. splitters (identical on every rank: same gathered bytes, same rule)
    std::vector<ls_tagged> spl(MAX_WORLD);
    ls_status rc = ls_multi_splitters(h.data(), h.size(), R, spl.data());
    if (rc != LS_OK) return rc;
    CUDA_CHECK(cudaMemcpyAsync(w + l.spl, spl.data(), (size_t)(R > 1 ? R - 1 : 1) * sizeof(Tagged), cudaMemcpyHostToDevice, st));
    // 3. destination counts with per-unit offsets (decoupled lookback)
    CUDA_CHECK(cudaMemsetAsync(w + l.ticket, 0, l.send - l.ticket, st));
    MultiArgs a;
    a.in = (const uint64_t *)d_in;
    a.send = (uint64_t *)(w + l.send);
    a.n = n_in;
    a.rank = (uint32_t)me;
    a.world = R;
    a.U = l.U;
    a.spl = (const Tagged *)(w + l.spl);
    a.lb = (unsigned long long *)(w + l.lb);
    a.offs = (uint32_t *)(w + l.offs);
    a.counts = (unsigned long long *)(w + l.counts);
    a.sdispl = (const unsigned long long *)(w + l.sdispl);
    a.ticket = (uint32_t *)(w + l.ticket);
    if (n_in) {
        if (dt == DT_F64) k_dest_count<DT_F64><<<l.U, 512, 0, st>>>(a);
        else k_dest_count<DT_U64><<<l.U, 512, 0, st>>>(a);
    }
    // 4. all-gather [counts(R), status, out_cap] -> identical plan everywhere
    unsigned long long *row = (unsigned long long *)(w + l.counts);
    const unsigned long long cap = out_cap;
    CUDA_CHECK(cudaMemcpyAsync(row + R + 1, &cap, 8, cudaMemcpyHostToDevice, st));
    NCCL_CHECK(ncclAllGather(row, w + l.allcounts, (size_t)(R + 2), ncclUint64, comm->comm, st));
    std::vector<uint64_t> all((size_t)(R + 2) * R), mat((size_t)R * R);
    CUDA_CHECK(cudaMemcpyAsync(all.data(), w + l.allcounts, all.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    bool any_nan = false, any_cap = false;
    for (int p = 0; p < R; p++) {
        for (int q = 0; q < R; q++) mat[(size_t)p * R + q] = all[(size_t)p * (R + 2) + q];
        any_nan |= all[(size_t)p * (R + 2) + R] != 0;
    }
    std::vector<uint64_t> sd(R), rcnt(R), rd(R);
    uint64_t nout = 0;
    for (int p = 0; p < R; p++) {
        uint64_t np = 0;
        ls_multi_plan(mat.data(), R, p, nullptr, nullptr, nullptr, &np);
        if (np > all[(size_t)p * (R + 2) + R + 1]) any_cap = true;
    }
    ls_multi_plan(mat.data(), R, me, sd.data(), rcnt.data(), rd.data(), &nout);
    *n_out = nout;
    if (any_nan) { set_error("NaN key in input (S:214)"); return LS_E_NAN; }
    if (any_cap) { set_error("out_cap smaller than the received key count on some rank"); return LS_E_CAPACITY; }
    // LS_FLAG_PEER_SCATTER: every rank's d_out mapped here, or,
    // if any rank cannot export / map its buffer, the send-buffer path below
    // on every rank (the decision is collective: all-gathered flags and one
    // all-reduce of the mapping results)
    bool peer = (cfg.flags & LS_FLAG_PEER_SCATTER) != 0;
    PeerDst pd;
    memset(&pd, 0, sizeof pd);
    if (peer && R > 1) {
        PeerXchg mine;
        memset(&mine, 0, sizeof mine);
        uint64_t base = 0;
        if (alloc_base(d_out, &base) == cudaSuccess && cudaIpcGetMemHandle(&mine.h, (void *)base) == cudaSuccess) {
            mine.off = (uint64_t)(uintptr_t)d_out - base;
            mine.ok = 1;
        }
        cudaGetLastError();  // (a failed export is not an error: the collective fallback)
        unsigned char *xb = w + l.xchg;
        CUDA_CHECK(cudaMemcpyAsync(xb + (size_t)R * sizeof(PeerXchg), &mine, sizeof mine, cudaMemcpyHostToDevice, st));
        NCCL_CHECK(ncclAllGather(xb + (size_t)R * sizeof(PeerXchg), xb, sizeof(PeerXchg), ncclUint8, comm->comm, st));
        std::vector<PeerXchg> xs(R);
        CUDA_CHECK(cudaMemcpyAsync(xs.data(), xb, (size_t)R * sizeof(PeerXchg), cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        for (int p = 0; p < R; p++) peer &= xs[p].ok == 1;
        if (peer) {
            uint64_t mapped = 1;
            for (int p = 0; p < R; p++) {
                if (p == me) continue;
                ls_comm::Peer &pe = comm->peer[p];
                if (!pe.base || memcmp(&pe.h, &xs[p].h, sizeof pe.h) != 0) {
                    if (pe.base) cudaIpcCloseMemHandle(pe.base);
                    pe.base = nullptr;
                    if (cudaIpcOpenMemHandle(&pe.base, xs[p].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                        pe.base = nullptr;
                        mapped = 0;
                        cudaGetLastError();
                        continue;
                    }
                    pe.h = xs[p].h;
                }
                pe.off = xs[p].off;
                pd.ptr[p] = (uint64_t *)((unsigned char *)pe.base + pe.off);
            }
            CUDA_CHECK(cudaMemcpyAsync(xb, &mapped, 8, cudaMemcpyHostToDevice, st));
            NCCL_CHECK(ncclAllReduce(xb, xb, 1, ncclUint64, ncclMin, comm->comm, st));
            CUDA_CHECK(cudaMemcpyAsync(&mapped, xb, 8, cudaMemcpyDeviceToHost, st));
            CUDA_CHECK(cudaStreamSynchronize(st));
            peer = mapped == 1;
        }
    }
    if (peer) {
        // 5'+6'. the destination scatter stores each run straight into its
        // destination's d_out at this rank's slice (the ranks before it come
        // first: ls_multi_plan's receive order); one all-reduce then orders
        // every rank's stores before any local sort
        pd.ptr[me] = (uint64_t *)d_out;
        for (int p = 0; p < R; p++) {
            uint64_t o = 0;
            for (int q = 0; q < me; q++) o += mat[(size_t)q * R + p];
            pd.off[p] = o;
        }
        if (n_in) launch_dest_scatter_peer(a, pd, dt, st);
        CUDA_CHECK(cudaGetLastError());
        NCCL_CHECK(ncclAllReduce(w + l.xchg, w + l.xchg, 1, ncclUint64, ncclMax, comm->comm, st));
    } else {
    // 5. scatter by destination into the send buffer
    CUDA_CHECK(cudaMemcpyAsync(w + l.sdispl, sd.data(), (size_t)R * 8, cudaMemcpyHostToDevice, st));
    if (n_in) {
        const size_t sm = sizeof(DestSmem);
        if (dt == DT_F64) {
            cudaFuncSetAttribute(k_dest_scatter<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_dest_scatter<DT_F64><<<l.U, TP_THREADS, sm, st>>>(a);
        } else {
            cudaFuncSetAttribute(k_dest_scatter<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_dest_scatter<DT_U64><<<l.U, TP_THREADS, sm, st>>>(a);
        }
    }
    CUDA_CHECK(cudaGetLastError());
    // 6. all-to-all over NVLink
    const uint64_t *send = a.send;
    NCCL_CHECK(ncclGroupStart());
    for (int p = 0; p < R; p++) {
        const uint64_t sc = mat[(size_t)me * R + p];
        if (sc) NCCL_CHECK(ncclSend(send + sd[p], sc, ncclUint64, p, comm->comm, st));
        if (rcnt[p]) NCCL_CHECK(ncclRecv((uint64_t *)d_out + rd[p], rcnt[p], ncclUint64, p, comm->comm, st));
    }
    NCCL_CHECK(ncclGroupEnd());
    }
    // 7. local LearnedSort 2.0 (fresh model on the received keys)
    Pending pend;
    rc = enqueue_sort((uint64_t *)d_out, nout, dtype, &cfg, nullptr, w + l.local, ws_bytes - l.local, st, stats, nullptr, &pend);
    if (rc != LS_OK) return rc;
    rc = finish_sort(&pend, st, stats);
    {   // a collective that failed after it was enqueued (a peer died, a link
        // error) is reported by the communicator, not by the calls above
        ncclResult_t ar = ncclSuccess;
        NCCL_CHECK(ncclCommGetAsyncError(comm->comm, &ar));
        if (ar != ncclSuccess && ar != ncclInProgress) {
            set_error(ncclGetErrorString(ar));
            return LS_E_NCCL;
        }
    }
    if (stats) {
        stats->peer_scatter = peer ? 1u : 0u;
        uint64_t rk = 0;
        for (int p = 0; p < R; p++) rk += p == me ? 0 : mat[(size_t)me * R + p];
        stats->remote_keys = rk;
    }
    return rc;
}

ls_status ls_multi_sample(const void *d_in, uint64_t n_in, int rank, ls_dtype dtype,
                          ls_tagged *d_samples, void *stream) {
    if (!d_samples || (n_in && !d_in) || rank < 0 || rank >= MAX_WORLD) { set_error("bad arguments"); return LS_E_INVALID; }
    if (dtype != LS_F64 && dtype != LS_U64) { set_error("bad dtype"); return LS_E_INVALID; }
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == LS_F64) k_split_sample<DT_F64><<<(SPLIT_K + 255) / 256, 256, 0, st>>>((const uint64_t *)d_in, n_in, (uint32_t)rank, (Tagged *)d_samples);
    else k_split_sample<DT_U64><<<(SPLIT_K + 255) / 256, 256, 0, st>>>((const uint64_t *)d_in, n_in, (uint32_t)rank, (Tagged *)d_samples);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(st));
    return LS_OK;
}

ls_status ls_multi_route(const void *d_in, uint64_t n_in, int rank, int world,
                         const ls_tagged *h_splitters, ls_dtype dtype, void *d_send,
                         uint64_t *h_counts, void *d_ws, size_t ws_bytes, void *stream) {
    if (world < 1 || world > MAX_WORLD || rank < 0 || rank >= world || !h_counts || !d_ws ||
        (world > 1 && !h_splitters) || (n_in && (!d_in || !d_send))) {
        set_error("bad arguments");
        return LS_E_INVALID;
    }
    if (dtype != LS_F64 && dtype != LS_U64) { set_error("bad dtype"); return LS_E_INVALID; }
    if (n_in >= (1ull << 32)) { set_error("n must be < 2^32"); return LS_E_INVALID; }
    if (((uintptr_t)d_in & 15) || ((uintptr_t)d_send & 15) || ((uintptr_t)d_ws & 255)) {
        set_error("keys / send buffer must be 16-byte aligned and the workspace 256-byte aligned");
        return LS_E_INVALID;
    }
    ls_config cfg;
    ls_config_default(&cfg);
    const int R = world;
    const MultiLayout l = multi_layout(n_in, 0, R, cfg);
    if (ws_bytes < l.local) { set_error("workspace too small"); return LS_E_WORKSPACE; }
    cudaStream_t st = (cudaStream_t)stream;
    unsigned char *w = (unsigned char *)d_ws;
    const int dt = (int)dtype;
    if (R > 1) CUDA_CHECK(cudaMemcpyAsync(w + l.spl, h_splitters, (size_t)(R - 1) * sizeof(Tagged), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemsetAsync(w + l.ticket, 0, l.send - l.ticket, st));
    MultiArgs a;
    a.in = (const uint64_t *)d_in;
    a.send = (uint64_t *)d_send;
    a.n = n_in;
    a.rank = (uint32_t)rank;
    a.world = R;
    a.U = l.U;
    a.spl = (const Tagged *)(w + l.spl);
    a.lb = (unsigned long long *)(w + l.lb);
    a.offs = (uint32_t *)(w + l.offs);
    a.counts = (unsigned long long *)(w + l.counts);
    a.sdispl = (const unsigned long long *)(w + l.sdispl);
    a.ticket = (uint32_t *)(w + l.ticket);
    // step 3 of ls_sort_multi: destination counts, per-unit offsets
    if (n_in) {
        if (dt == DT_F64) k_dest_count<DT_F64><<<l.U, 512, 0, st>>>(a);
        else k_dest_count<DT_U64><<<l.U, 512, 0, st>>>(a);
    }
    std::vector<unsigned long long> row((size_t)R + 1);
    CUDA_CHECK(cudaMemcpyAsync(row.data(), a.counts, row.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (row[R]) { set_error("NaN key in input (S:214)"); return LS_E_NAN; }
    std::vector<uint64_t> sd(R);
    uint64_t s = 0;
    for (int p = 0; p < R; p++) {
        h_counts[p] = row[p];
        sd[p] = s;
        s += row[p];
    }
    // step 5: scatter by destination
    CUDA_CHECK(cudaMemcpyAsync(w + l.sdispl, sd.data(), (size_t)R * 8, cudaMemcpyHostToDevice, st));
    if (n_in) {
        const size_t sm = sizeof(DestSmem);
        if (dt == DT_F64) {
            cudaFuncSetAttribute(k_dest_scatter<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_dest_scatter<DT_F64><<<l.U, TP_THREADS, sm, st>>>(a);
        } else {
            cudaFuncSetAttribute(k_dest_scatter<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_dest_scatter<DT_U64><<<l.U, TP_THREADS, sm, st>>>(a);
        }
    }
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(st));
    return LS_OK;
}

ls_status ls_multi_route_peer(const void *d_in, uint64_t n_in, int rank, int world,
                              const ls_tagged *h_splitters, ls_dtype dtype, void *const *h_dst,
                              const uint64_t *h_dst_off, uint64_t *h_counts, void *d_ws,
                              size_t ws_bytes, void *stream) {
    if (world < 1 || world > MAX_WORLD || rank < 0 || rank >= world || !h_counts || !d_ws ||
        (world > 1 && !h_splitters) || (n_in && (!d_in || !h_dst || !h_dst_off))) {
        set_error("bad arguments");
        return LS_E_INVALID;
    }
    if (dtype != LS_F64 && dtype != LS_U64) { set_error("bad dtype"); return LS_E_INVALID; }
    if (n_in >= (1ull << 32)) { set_error("n must be < 2^32"); return LS_E_INVALID; }
    if (((uintptr_t)d_in & 15) || ((uintptr_t)d_ws & 255)) {
        set_error("keys must be 16-byte aligned and the workspace 256-byte aligned");
        return LS_E_INVALID;
    }
    ls_config cfg;
    ls_config_default(&cfg);
    const int R = world;
    const MultiLayout l = multi_layout(n_in, 0, R, cfg);
    if (ws_bytes < l.local) { set_error("workspace too small"); return LS_E_WORKSPACE; }
    cudaStream_t st = (cudaStream_t)stream;
    unsigned char *w = (unsigned char *)d_ws;
    const int dt = (int)dtype;
    if (R > 1) CUDA_CHECK(cudaMemcpyAsync(w + l.spl, h_splitters, (size_t)(R - 1) * sizeof(Tagged), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemsetAsync(w + l.ticket, 0, l.send - l.ticket, st));
    MultiArgs a;
    a.in = (const uint64_t *)d_in;
    a.send = nullptr;
    a.n = n_in;
    a.rank = (uint32_t)rank;
    a.world = R;
    a.U = l.U;
    a.spl = (const Tagged *)(w + l.spl);
    a.lb = (unsigned long long *)(w + l.lb);
    a.offs = (uint32_t *)(w + l.offs);
    a.counts = (unsigned long long *)(w + l.counts);
    a.sdispl = (const unsigned long long *)(w + l.sdispl);
    a.ticket = (uint32_t *)(w + l.ticket);
    if (n_in) {
        if (dt == DT_F64) k_dest_count<DT_F64><<<l.U, 512, 0, st>>>(a);
        else k_dest_count<DT_U64><<<l.U, 512, 0, st>>>(a);
    }
    std::vector<unsigned long long> row((size_t)R + 1);
    CUDA_CHECK(cudaMemcpyAsync(row.data(), a.counts, row.size() * 8, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    if (row[R]) { set_error("NaN key in input (S:214)"); return LS_E_NAN; }
    PeerDst pd;
    memset(&pd, 0, sizeof pd);
    for (int p = 0; p < R; p++) {
        h_counts[p] = row[p];
        if (n_in) {
            if (row[p] && (!h_dst[p] || ((uintptr_t)h_dst[p] & 7))) { set_error("bad destination pointer"); return LS_E_INVALID; }
            pd.ptr[p] = (uint64_t *)h_dst[p];
            pd.off[p] = h_dst_off[p];
        }
    }
    if (n_in) launch_dest_scatter_peer(a, pd, dt, st);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaStreamSynchronize(st));
    return LS_OK;
}

}  // extern "C"
