// Max active clusters on this GPU for a dummy kernel, by cluster size, block size and dynamic
// shared memory (cudaOccupancyMaxActiveClusters).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(double *p) { extern __shared__ double s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    int cs[] = {2, 4, 6, 8, 12, 16};
    int th[] = {256, 384, 512, 1024};
    int kb[] = {40, 56, 70, 74, 90, 100, 110, 150, 200};
    for (int c : cs) for (int t : th) for (int k : kb) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c * 64); cfg.blockDim = dim3(t); cfg.dynamicSmemBytes = (size_t)k * 1024;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
        printf("cs %2d threads %4d smem %3d KB -> clusters %3d (CTAs %3d)%s\n", c, t, k, n, n * c,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
