// ls_bigpath.cu -- north_star (3): the exact path for LARGE high-multiplicity
// sub-buckets (more than LARGE_MIN keys the model could not separate: SURVEY
// H5/H6 -- config 4's ID clusters, config 5's Zipf head), run grid-parallel
// instead of one CTA per sub-bucket.
//
// One MSD digit pass per large item on d = (ord(x) - min) >> shift, 10-bit
// digits aligned to the item's ord range:
//   k_large_count  : per 64K-key chunk, digit histogram + per-digit min/max
//                    (shared memory), merged into the item's tables (global)
//   k_large_scan   : per item, digit starts; a digit piece with min == max is
//                    homogeneous -- it is written by value, its keys
//                    never move; other pieces become warp sorts (<= WS_MAX keys)
//                    or per-CTA big items (k_big level 1)
//   k_large_scatter: per chunk, keys of non-homogeneous pieces only, A -> B,
//                    ranges reserved per (chunk, digit), TMA tile engine
//   k_large_fill   : per output chunk, homogeneous pieces filled from the
//                    histogram (a counting sort by value: Zipf heads cost one
//                    read and one write per key)
//   k_piece_sort   : one warp per small piece, B -> A, register bitonic
#include "ls_launch.h"
#include "ls_tilepart.cuh"
#include "ls_warpsort.cuh"

namespace ls {

constexpr int LD_BITS = 10;
constexpr int LD_DIG = 1 << LD_BITS;  // 1024 digits
constexpr int LD_WORDS = LD_DIG / 32;
constexpr uint32_t PIECE_MAX = 512;  // pieces up to this size: one warp (k_piece_sort)

__device__ __forceinline__ int large_shift(unsigned long long mn, unsigned long long mx) {
    const unsigned long long range = mx - mn;
    const int bits = range ? 64 - __clzll((long long)range) : 0;
    return bits > LD_BITS ? bits - LD_BITS : 0;
}

// ----------------------------------------------------------------- count --
template <int DT>
__global__ void __launch_bounds__(512) k_large_count(Args a) {
    if (a.ctl->status) return;
    if (a.ctl->nlarge == 0) return;  // (no large item: skip the chunk list)
    __shared__ uint32_t hist[LD_DIG];
    __shared__ unsigned long long dmn[LD_DIG], dmx[LD_DIG];
    const uint32_t nch = min(a.ctl->nchunks, a.chunk_cap);
    for (uint32_t e = blockIdx.x; e < nch; e += gridDim.x) {
        const BigChunk ch = a.chunks[e];
        const BigItem item = a.big[ch.item];
        if (item.pad0 == 0 || item.mn == item.mx) continue;  // not large / homogeneous
        const uint32_t li = item.pad0 - 1u;
        const int shift = large_shift(item.mn, item.mx);
        for (int d = threadIdx.x; d < LD_DIG; d += blockDim.x) {
            hist[d] = 0;
            dmn[d] = ~0ull;
            dmx[d] = 0;
        }
        __syncthreads();
        const uint32_t beg = ch.chunk * MM_CHUNK, end = min(item.size, beg + MM_CHUNK);
        const uint64_t *X = a.A + item.off;
        for (uint32_t i = beg + threadIdx.x; i < end; i += 4 * blockDim.x) {
            uint64_t v[4];
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = (i + q * blockDim.x < end) ? X[i + q * blockDim.x] : X[beg];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                if (i + q * blockDim.x >= end) continue;
                const unsigned long long o = to_ord<DT>(v[q]);
                const uint32_t d = (uint32_t)((o - item.mn) >> shift);
                atomicAdd(&hist[d], 1u);
                atomicMin(&dmn[d], o);
                atomicMax(&dmx[d], o);
            }
        }
        __syncthreads();
        for (int d = threadIdx.x; d < LD_DIG; d += blockDim.x) {
            if (!hist[d]) continue;
            const size_t k = (size_t)li * LD_DIG + d;
            atomicAdd(&a.ltot[k], hist[d]);
            atomicMin(&a.lmin[k], dmn[d]);
            atomicMax(&a.lmax[k], dmx[d]);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ scan --
__global__ void __launch_bounds__(LD_DIG) k_large_scan(Args a) {
    if (a.ctl->status) return;
    __shared__ uint32_t s[LD_DIG];
    __shared__ uint32_t tmp[33];
    __shared__ uint32_t hw[LD_WORDS];
    const uint32_t nl = min(a.ctl->nlarge, a.lcap);
    const int d = threadIdx.x;
    for (uint32_t li = blockIdx.x; li < nl; li += gridDim.x) {
        const uint32_t bi = a.large[li];
        const BigItem item = a.big[bi];
        if (item.mn == item.mx) continue;
        const size_t k = (size_t)li * LD_DIG + d;
        const uint32_t c = a.ltot[k];
        s[d] = c;
        if (d < LD_WORDS) hw[d] = 0;
        __syncthreads();
        block_exscan(s, LD_DIG, tmp);
        const uint32_t st = s[d];
        const bool homo = c >= 1u && a.lmin[k] == a.lmax[k];
        a.lstart[k] = st;
        a.lcur[k] = item.off + st;  // scatter cursor (k_large_scatter reserves ranges)
        if (homo) {
            atomicOr(&hw[d >> 5], 1u << (d & 31));
            const unsigned long long o = a.lmin[k];
            const uint32_t nf = (c + MM_CHUNK - 1) / MM_CHUNK;  // fill tasks of <= 64K keys
            const uint32_t q = atomicAdd(&a.ctl->nfill, nf);
            for (uint32_t x = 0; x < nf; x++) {
                if (q + x < a.fcap)
                    a.fills[q + x] = make_uint4(item.off + st + x * MM_CHUNK, min(MM_CHUNK, c - x * MM_CHUNK),
                                                (uint32_t)o, (uint32_t)(o >> 32));
                else
                    atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
            }
        }
        if (!homo && c >= 2u) {
            if (c <= PIECE_MAX) {
                const uint32_t q = atomicAdd(&a.ctl->npiece, 1u);
                if (q < a.pcap) a.pieces[q] = make_uint2(item.off + st, c);
                else atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
            } else {  // larger piece: per-CTA radix path, keys in B
                const uint32_t q = atomicAdd(&a.ctl->big_cnt[1], 1u);
                if (q < a.big_cap)
                    a.big[(size_t)a.big_cap + q] = BigItem{item.off + st, c, 1u, ~0u, ~0ull, 0ull, 0u, 0u};
                else
                    atomicOr(&a.ctl->status, (uint32_t)STATUS_INTERNAL);
            }
        }
        __syncthreads();
        if (d < LD_WORDS) a.lhom[(size_t)li * LD_WORDS + d] = hw[d];
        if (d == 0) {  // any homogeneous piece? (k_large_fill skips the item otherwise)
            uint32_t any = 0;
            for (int w = 0; w < LD_WORDS; w++) any |= hw[w];
            a.big[bi].pad1 = any ? 1u : 0u;
        }
        __syncthreads();
    }
}

// --------------------------------------------------------------- scatter --
// Keys of homogeneous pieces are skipped (TP_SKIP); the others move A -> B.
struct LargeDigit {
    unsigned long long mn;
    int shift;
    const uint32_t *hom;  // shared memory, LD_WORDS words
    template <int DT>
    __device__ __forceinline__ uint32_t get(uint64_t key) const {
        const uint32_t d = (uint32_t)((to_ord<DT>(key) - mn) >> shift);
        return ((hom[d >> 5] >> (d & 31)) & 1u) ? TP_SKIP : d;
    }
};
template <int DT>
struct LargeBucket {
    LargeDigit ld;
    __device__ __forceinline__ uint32_t operator()(uint64_t key, uint64_t) const { return ld.get<DT>(key); }
};

struct LargeSmem {
    TpSmem tp;
    uint32_t base[LD_DIG];
    uint32_t hom[LD_WORDS];
};

static_assert(sizeof(LargeSmem) <= MAX_SMEM_OPTIN, "large scatter shared memory");

template <int DT>
__global__ void __launch_bounds__(TP_THREADS, 1) k_large_scatter(Args a) {
    if (a.ctl->status) return;
    if (a.ctl->nlarge == 0) return;  // (no large item: skip the chunk list)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LargeSmem &S = *reinterpret_cast<LargeSmem *>(smem_raw);
    const int tid = threadIdx.x;
    const uint32_t nch = min(a.ctl->nchunks, a.chunk_cap);
    uint32_t phase = 0;
    tp_init(S.tp);
    for (uint32_t e = blockIdx.x; e < nch; e += gridDim.x) {
        const BigChunk ch = a.chunks[e];
        const BigItem item = a.big[ch.item];
        if (item.pad0 == 0 || item.mn == item.mx) continue;
        const uint32_t li = item.pad0 - 1u;
        if (tid < LD_WORDS) S.hom[tid] = a.lhom[(size_t)li * LD_WORDS + tid];
        S.base[tid] = 0;
        __syncthreads();
        const LargeDigit ld{item.mn, large_shift(item.mn, item.mx), S.hom};
        const uint32_t beg = ch.chunk * MM_CHUNK, end = min(item.size, beg + MM_CHUNK);
        // this chunk's count per digit, then one range reservation per digit
        for (uint32_t i = beg + tid; i < end; i += TP_THREADS) {
            const uint32_t d = ld.get<DT>(a.A[item.off + i]);
            if (d != TP_SKIP) atomicAdd(&S.base[d], 1u);
        }
        __syncthreads();
        {
            const uint32_t c = S.base[tid];
            S.base[tid] = c ? atomicAdd(&a.lcur[(size_t)li * LD_DIG + tid], c) : 0u;
        }
        __syncthreads();
        const LargeBucket<DT> bf{ld};
        tile_partition<true>(S.tp, a.A, a.B, (uint64_t)item.off + beg, (uint64_t)item.off + end, a.n,
                             S.base, LD_DIG, bf, phase);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ fill --
// Homogeneous pieces: write their value (one task per <= 64K keys).
template <int DT>
__global__ void __launch_bounds__(256) k_large_fill(Args a) {
    if (a.ctl->status) return;
    const uint32_t nf = min(a.ctl->nfill, a.fcap);
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < nf; t += nw) {
        const uint4 f = a.fills[t];
        const uint64_t v = from_ord<DT>((unsigned long long)f.z | ((unsigned long long)f.w << 32));
        uint64_t *dst = a.A + f.x;
        for (uint32_t i = lane; i < f.y; i += 32) dst[i] = v;
    }
}

// ------------------------------------------------------------ piece sort --
template <int DT>
__global__ void __launch_bounds__(256) k_piece_sort(Args a) {
    if (a.ctl->status) return;
    const int lane = threadIdx.x & 31;
    const uint32_t np_ = min(a.ctl->npiece, a.pcap);
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    for (uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < np_; t += nw) {
        const uint2 pc = a.pieces[t];
        const uint32_t off = pc.x, c = pc.y;
        const uint64_t *X = a.B + off;
        uint64_t *Y = a.A + off;
        // stage B -> A, then sort in place (peeling few-valued pieces)
        for (uint32_t i = lane; i < c; i += 32) Y[i] = X[i];
        __syncwarp();
        if (c <= 32u) warp_sort_keys<DT, 1, 16>(Y, c, lane);
        else if (c <= 64u) warp_sort_keys<DT, 2, 16>(Y, c, lane);
        else if (c <= 128u) warp_sort_keys<DT, 4, 16>(Y, c, lane);
        else if (c <= 256u) warp_sort_keys<DT, 8, 16>(Y, c, lane);
        else warp_sort_keys<DT, 16, 16>(Y, c, lane);
    }
}

// -------------------------------------------------------------- launchers --
void launch_large(const Args &a, int dtype, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t sm = sizeof(LargeSmem);
    if (dtype == DT_F64) {
        k_large_count<DT_F64><<<sms * 4, 512, 0, st>>>(a);
        k_large_scan<<<sms * 2, LD_DIG, 0, st>>>(a);
        cudaFuncSetAttribute(k_large_scatter<DT_F64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_large_scatter<DT_F64><<<sms, TP_THREADS, sm, st>>>(a);
        k_large_fill<DT_F64><<<sms * 8, 256, 0, st>>>(a);
        k_piece_sort<DT_F64><<<sms * 8, 256, 0, st>>>(a);
    } else {
        k_large_count<DT_U64><<<sms * 4, 512, 0, st>>>(a);
        k_large_scan<<<sms * 2, LD_DIG, 0, st>>>(a);
        cudaFuncSetAttribute(k_large_scatter<DT_U64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_large_scatter<DT_U64><<<sms, TP_THREADS, sm, st>>>(a);
        k_large_fill<DT_U64><<<sms * 8, 256, 0, st>>>(a);
        k_piece_sort<DT_U64><<<sms * 8, 256, 0, st>>>(a);
    }
}

}  // namespace ls
