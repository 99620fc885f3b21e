// Dev probe: cluster occupancy of a pair kernel vs its ingredients (TMEM alloc, static smem, carveout)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int kTmem>
__global__ void __launch_bounds__(256, 2) kprobe(int* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bars[24];
    __shared__ uint32_t taddr;
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    sm[threadIdx.x] = (unsigned char)r;
    if (kTmem && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&taddr)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 0) bars[0] = r;
    __syncthreads();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (kTmem && threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(256));
    if (threadIdx.x == 0) atomicAdd(out, int(r) + int(bars[0]));
}
template <int T>
void run(int smem, int carve) {
    int* d;
    cudaMalloc(&d, 4);
    cudaFuncSetAttribute(kprobe<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (carve >= 0) cudaFuncSetAttribute(kprobe<T>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(8, 64, 1);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = -1;
    cudaOccupancyMaxActiveClusters(&ncl, kprobe<T>, &cfg);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kprobe<T>, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kprobe<T>);
    printf("tmem %d smem %d carve %d: clusters %d (static %zu regs %d) launch %s %s\n", T, smem, carve, ncl,
           fa.sharedSizeBytes, fa.numRegs, cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaFree(d);
}
int main() {
    for (int smem : {100928, 90000, 60000}) {
        run<0>(smem, -1);
        run<0>(smem, 100);
        run<1>(smem, -1);
        run<1>(smem, 100);
    }
    return 0;
}
