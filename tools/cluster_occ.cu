// Prints cudaOccupancyMaxActiveClusters for cluster sizes x dynamic smem sizes (B200 probe).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    int sizes[] = {1, 2, 4, 6, 8, 9, 10, 12, 14, 16};
    int smems[] = {20, 60, 100, 110, 150, 200};
    int threads[] = {160, 288};
    for (int th : threads) {
        printf("threads %d\n smem_KB:", th);
        for (int sm : smems) printf(" %6d", sm);
        printf("\n");
        for (int cs : sizes) {
            printf(" cs=%2d  :", cs);
            for (int sm : smems) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(cs * 64, 1, 1);
                cfg.blockDim = dim3(th);
                cfg.dynamicSmemBytes = sm * 1024;
                cudaLaunchAttribute a;
                a.id = cudaLaunchAttributeClusterDimension;
                a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
                cfg.attrs = &a; cfg.numAttrs = 1;
                int n = -1;
                cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
                if (e != cudaSuccess) { n = -1; cudaGetLastError(); }
                printf(" %6d", n);
            }
            printf("\n");
        }
    }
    cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
    printf("SMs %d, smem/SM %zu, smem/block optin %zu\n", pr.multiProcessorCount, pr.sharedMemPerMultiprocessor, pr.sharedMemPerBlockOptin);
    return 0;
}
