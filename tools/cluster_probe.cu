// Dev probe: which cluster launch configurations does this GPU accept?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) kprobe(int* out) {
    extern __shared__ unsigned char sm[];
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    sm[threadIdx.x] = (unsigned char)r;
    if (threadIdx.x == 0) atomicAdd(out, int(r) + 1);
}
int main() {
    int* d;
    cudaMalloc(&d, 4);
    for (int smem : {16 * 1024, 48 * 1024, 100 * 1024, 110 * 1024}) {
        for (int cy : {2}) {
            for (int gx : {1, 7}) {
                cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(gx, 4, 1);
                cfg.blockDim = dim3(256);
                cfg.dynamicSmemBytes = smem;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = 1;
                at[0].val.clusterDim.y = cy;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaError_t e = cudaLaunchKernelEx(&cfg, kprobe, d);
                cudaError_t e2 = cudaDeviceSynchronize();
                int ncl = -1;
                cudaOccupancyMaxActiveClusters(&ncl, kprobe, &cfg);
                printf("smem %d cy %d gx %d: launch %s sync %s maxActiveClusters %d\n", smem, cy, gx, cudaGetErrorString(e),
                       cudaGetErrorString(e2), ncl);
                cudaGetLastError();
            }
        }
    }
    return 0;
}
