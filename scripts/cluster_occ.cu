// How many clusters of 1-CTA-per-SM kernels (200 KiB smem) can be resident on
// this B200, per cluster size: the SMs a cluster design would strand.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[threadIdx.x]; }
int main() {
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(544); cfg.dynamicSmemBytes = smem;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d of %d SMs (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
    }
    return 0;
}
