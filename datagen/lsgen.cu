// lsgen.cu -- C-ABI around lsgen.h: host-built tables + host and device fills.
// Input generation only; no LearnedSort arithmetic lives here.
#include "lsgen.h"

#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>
#include <vector>

struct lsg_plan {
    lsg_params P;              // host view (host table pointers)
    std::vector<double> zipf_cum, level_cum, centre;
    std::vector<uint64_t> level_val;
    double *d_zipf = nullptr, *d_level_cum = nullptr, *d_centre = nullptr;
    uint64_t *d_level_val = nullptr;
    lsg_params Pd;             // device view
    bool device_ready = false;
};

static uint64_t half_bits(uint64_t n) {
    uint64_t b = 0;
    while (b < 64 && (1ULL << b) < n) b++;
    if (b < 2) b = 2;
    return (b + 1) / 2;
}

static uint64_t isqrt64(uint64_t n) {
    uint64_t r = (uint64_t)sqrt((double)n);
    while (r * r > n) r--;
    while ((r + 1) * (r + 1) <= n) r++;
    return r;
}

extern "C" {

int lsg_is_u64_dist(int dist) { return lsg_is_u64(dist); }

// zipf_s / zipf_V <= 0 select the configured defaults (0.75 / 1e6 for ZIPF_U64,
// 1.0 / 1e7 for CFG5MIX).
int lsg_create(int dist, uint64_t n, uint64_t seed, double zipf_s, uint64_t zipf_V, lsg_plan **out) {
    if (dist < 0 || dist >= LSG_NUM_DISTS || !out) return 1;
    if ((dist == LSG_TWODUPS) && n > 0xffffffffULL) return 1;
    lsg_plan *pl = new lsg_plan();
    lsg_params &P = pl->P;
    memset(&P, 0, sizeof P);
    P.dist = dist;
    P.n = n;
    P.seed = seed;
    P.feistel_bits = half_bits(n ? n : 1);
    P.isqrt_n = isqrt64(n) ? isqrt64(n) : 1;
    if (dist == LSG_MIXGAUSS) {
        for (int c = 0; c < 5; c++) {
            uint64_t w0, w1;
            lsg_words(seed, 7, (uint64_t)c, &w0, &w1);
            P.mix_mu[c] = -100.0 + 200.0 * lsg_u01(w0);
            P.mix_sigma[c] = 1.0 + 9.0 * lsg_u01(w1);
        }
    }
    if (dist == LSG_ZIPF_U64 || dist == LSG_CFG5MIX) {
        P.zipf_s = zipf_s > 0 ? zipf_s : (dist == LSG_ZIPF_U64 ? 0.75 : 1.0);
        P.zipf_V = zipf_V > 0 ? zipf_V : (dist == LSG_ZIPF_U64 ? 1000000ULL : 10000000ULL);
        pl->zipf_cum.resize(P.zipf_V);
        double acc = 0.0;
        for (uint64_t k = 0; k < P.zipf_V; k++) {
            acc += pow((double)(k + 1), -P.zipf_s);
            pl->zipf_cum[k] = acc;
        }
        P.vperm_bits = half_bits(P.zipf_V);
    }
    if (dist == LSG_TELEMETRY) {
        pl->level_cum.resize(10000);
        pl->level_val.resize(10000);
        pl->centre.resize(1000);
        double acc = 0.0;
        for (uint64_t v = 0; v < 10000; v++) {
            uint64_t w0, w1, a0, a1;
            lsg_words(seed, 11, v, &w0, &w1);
            acc += exp(2.0 * lsg_normal(w0, w1));
            pl->level_cum[v] = acc;
            lsg_words(seed, 12, v, &a0, &a1);
            pl->level_val[v] = (uint64_t)(lsg_u01(a0) * 9223372036854775808.0);
        }
        for (uint64_t j = 0; j < 1000; j++) {
            uint64_t w0, w1;
            lsg_words(seed, 13, j, &w0, &w1);
            pl->centre[j] = lsg_u01(w0) * 9223372036854775808.0;
        }
    }
    P.zipf_cum = pl->zipf_cum.empty() ? nullptr : pl->zipf_cum.data();
    P.level_cum = pl->level_cum.empty() ? nullptr : pl->level_cum.data();
    P.level_val = pl->level_val.empty() ? nullptr : pl->level_val.data();
    P.centre = pl->centre.empty() ? nullptr : pl->centre.data();
    *out = pl;
    return 0;
}

void lsg_destroy(lsg_plan *pl) {
    if (!pl) return;
    if (pl->d_zipf) cudaFree(pl->d_zipf);
    if (pl->d_level_cum) cudaFree(pl->d_level_cum);
    if (pl->d_level_val) cudaFree(pl->d_level_val);
    if (pl->d_centre) cudaFree(pl->d_centre);
    delete pl;
}

int lsg_fill_host(const lsg_plan *pl, uint64_t *out, uint64_t begin, uint64_t count) {
    for (uint64_t k = 0; k < count; k++) out[k] = lsg_value(&pl->P, begin + k);
    return 0;
}

const double *lsg_mix_params(const lsg_plan *pl) { return pl->P.mix_mu; }

}  // extern "C"

__global__ void lsg_fill_kernel(lsg_params P, uint64_t *out, uint64_t begin, uint64_t count) {
    uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
        out[k] = lsg_value(&P, begin + k);
}

template <class T>
static int upload(const std::vector<T> &h, T **d) {
    if (h.empty()) return 0;
    if (cudaMalloc(d, h.size() * sizeof(T)) != cudaSuccess) return 1;
    return cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess;
}

extern "C" int lsg_fill_device(lsg_plan *pl, void *d_out, uint64_t begin, uint64_t count,
                               void *stream) {
    if (!pl->device_ready) {
        if (upload(pl->zipf_cum, &pl->d_zipf) || upload(pl->level_cum, &pl->d_level_cum) ||
            upload(pl->level_val, &pl->d_level_val) || upload(pl->centre, &pl->d_centre))
            return 2;
        pl->Pd = pl->P;
        pl->Pd.zipf_cum = pl->d_zipf;
        pl->Pd.level_cum = pl->d_level_cum;
        pl->Pd.level_val = pl->d_level_val;
        pl->Pd.centre = pl->d_centre;
        pl->device_ready = true;
    }
    if (count == 0) return 0;
    int blocks = 148 * 8;
    lsg_fill_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(pl->Pd, (uint64_t *)d_out, begin, count);
    return cudaGetLastError() != cudaSuccess ? 3 : 0;
}
