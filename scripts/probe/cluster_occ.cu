// Probe: how many clusters of size G can be co-resident (1 or 2 CTAs/SM worth of smem).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kern(int *x) { extern __shared__ int s[]; if (threadIdx.x == 0 && x) x[blockIdx.x] = s[0]; }
int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    printf("SMs %d\n", sms);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int smem : {100 * 1024, 200 * 1024}) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int thr : {512, 1024}) {
            for (int G : {1, 2, 4, 8, 16}) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(G * 64);
                cfg.blockDim = dim3(thr);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                int n = -1;
                cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
                printf("smem %dK thr %d G %2d -> max active clusters %d (CTAs %d) %s\n", smem / 1024, thr, G, n, n * G,
                       e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
