// ls_launch.h -- host-side launchers of the libls kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include "ls_common.cuh"

namespace ls {

// fit (ls_fit.cu): strided sample + finite min/max, leaf histogram, chord params
void launch_sample_minmax(const uint64_t *src, uint64_t stride, uint64_t m, uint64_t *S_out,
                          Ctl *ctl, int dtype, cudaStream_t st);
void launch_fit_hist(const uint64_t *S, uint64_t m, int L, Ctl *ctl, uint32_t *leaf_cnt,
                     unsigned long long *leaf_min, int dtype, cudaStream_t st);
void launch_fit_params(uint64_t m, int L, Ctl *ctl, const uint32_t *leaf_cnt,
                       const unsigned long long *leaf_min, DevModel *M, int dtype, cudaStream_t st);

// b0 threshold table of the model (ls_fit.cu), after the model is final
void launch_b0_table(DevModel *M, int L, int f, int dtype, cudaStream_t st);

// partition rounds (ls_partition.cu)
void launch_init(const Args &a, cudaStream_t st);
void launch_count0(const Args &a, int dtype, cudaStream_t st);
void launch_plan0(const Args &a, uint64_t *dS_B, int reserved, cudaStream_t st);
void launch_cap0(const Args &a, uint64_t m, int dtype, cudaStream_t st);      // round 0 capacities
void launch_scatter0r(const Args &a, int dtype, cudaStream_t st);             // round 0 by reservation
void launch_scatter0(const Args &a, int dtype, cudaStream_t st);
void launch_count1(const Args &a, int dtype, cudaStream_t st);
void launch_scatter1(const Args &a, int dtype, cudaStream_t st);
void launch_classify(const Args &a, uint32_t *dS_B1, cudaStream_t st);

// cluster-resident round 1 (ls_round1.cu)
uint32_t round1_capacity();  // keys per cluster (0: clusters unavailable)
void launch_round1(const Args &a, int dtype, cudaStream_t st);

// in-bucket sort (ls_sortsub.cu)
void launch_warpsort(const Args &a, int dtype, cudaStream_t st);
void launch_bucketsort(const Args &a, int dtype, const cudaStream_t st[5]);  // the CTA sorts (st[0..3]) and block windows (st[4])
void launch_big_minmax(const Args &a, int dtype, cudaStream_t st);
void launch_big_order(const Args &a, cudaStream_t st);
void launch_big(const Args &a, int dtype, cudaStream_t st);  // all levels, one cooperative launch
void launch_large(const Args &a, int dtype, cudaStream_t st);  // ls_bigpath.cu

// parity hooks (ls_partition.cu)
void launch_bucket_ids(const uint64_t *keys, uint64_t n, int f, const DevModel *M, double *p,
                       uint32_t *b0, uint32_t *b1, unsigned long long *h0, unsigned long long *h1,
                       int dtype, cudaStream_t st);
void launch_bucket_pos(const uint64_t *keys, uint64_t n, int f, const DevModel *M,
                       const unsigned long long *h1, uint32_t *pos, int dtype, cudaStream_t st);

}  // namespace ls
