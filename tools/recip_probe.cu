// tools/recip_probe.cu — dev probe (GPU box): clock64 timeline of ONE CTA
// reciprocal (cta_recip) and ONE CTA multiply (cta_mulr) at a given L, to see
// where the LDLT critical-path latency goes.  Tags: 0 start, 5/6 cta_mul column
// sums begin/end, 1/2 level products done, 3 level done, 4 rounding done.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o build/recip_probe tools/recip_probe.cu
//   build/recip_probe 192
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ long long g_tr[4096];
__device__ int g_tag[4096];
__device__ int g_n;
__shared__ int s_n; // event counter in shared memory: a trace point costs a few cycles
#ifdef HK_PROBE_NOTRACE
#define HK_TRACE(tag)
#else
#define HK_TRACE(tag)                                                                                         \
    do {                                                                                                      \
        if (threadIdx.x == 0) {                                                                               \
            const int k_ = s_n++;                                                                             \
            if (k_ < 4096) {                                                                                  \
                g_tr[k_] = clock64();                                                                         \
                g_tag[k_] = (tag);                                                                            \
            }                                                                                                 \
            g_n = s_n;                                                                                        \
        }                                                                                                     \
    } while (0)
#endif

#include "../paper_1810_01478_b200/csrc/mpf_ops.cuh"

using namespace hk;

__global__ void k_recip(const uint32_t* d, Meta dm, uint32_t* out, int L, int ws_words) {
    extern __shared__ __align__(16) uint32_t sm[];
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    const Meta r = cta_recip(d, dm, out, L, sm);
    if (threadIdx.x == 0) HK_TRACE(9 + 0 * r.exp);
}

__global__ void k_mul(const uint32_t* x, const uint32_t* y, uint32_t* out, int L) {
    extern __shared__ __align__(16) uint32_t sm[];
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    HK_TRACE(7);
    const Meta r = cta_mulr(x, Meta{0, 1}, y, Meta{0, 1}, out, L, ctaws_carve(sm, L));
    HK_TRACE(8 + 0 * r.exp);
}

static void dump(const char* what) {
    int n = 0;
    cudaMemcpyFromSymbol(&n, g_n, sizeof(int));
    if (n > 4096) n = 4096;
    std::vector<long long> t(n);
    std::vector<int> g(n);
    cudaMemcpyFromSymbol(t.data(), g_tr, n * sizeof(long long));
    cudaMemcpyFromSymbol(g.data(), g_tag, n * sizeof(int));
    printf("%s: %d events, total %lld cycles\n", what, n, n ? t[n - 1] - t[0] : 0);
    for (int i = 1; i < n; ++i) printf("  tag %d  +%lld\n", g[i], t[i] - t[i - 1]);
    int z = 0;
    cudaMemcpyToSymbol(g_n, &z, sizeof(int));
}

int main(int argc, char** argv) {
    const int L = argc > 1 ? atoi(argv[1]) : 192;
    std::vector<uint32_t> h(L);
    uint32_t s = 12345;
    for (auto& v : h) v = (s = s * 1664525u + 1013904223u);
    h[L - 1] |= 0x80000000u;
    uint32_t *d, *o, *y;
    cudaMalloc(&d, L * 4);
    cudaMalloc(&y, L * 4);
    cudaMalloc(&o, L * 4);
    cudaMemcpy(d, h.data(), L * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(y, h.data(), L * 4, cudaMemcpyHostToDevice);
    const int wr = ctarecipws_words(L), wc = ctaws_words(L);
    cudaFuncSetAttribute(k_recip, cudaFuncAttributeMaxDynamicSharedMemorySize, wr * 4);
    cudaFuncSetAttribute(k_mul, cudaFuncAttributeMaxDynamicSharedMemorySize, wc * 4);
    for (int rep = 0; rep < 3; ++rep) {
        int z = 0;
        cudaMemcpyToSymbol(g_n, &z, sizeof(int));
        k_recip<<<1, 256, wr * 4>>>(d, Meta{0, 1}, o, L, wr);
        cudaDeviceSynchronize();
        if (rep == 2) dump("cta_recip");
        cudaMemcpyToSymbol(g_n, &z, sizeof(int));
        k_mul<<<1, 256, wc * 4>>>(d, y, o, L);
        cudaDeviceSynchronize();
        if (rep == 2) dump("cta_mulr");
    }
    // untraced timing: 200 back-to-back single-CTA launches (CUDA events)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int pass = 0; pass < 2; ++pass) {
        cudaEventRecord(e0);
        for (int r = 0; r < 200; ++r) k_recip<<<1, 256, wr * 4>>>(d, Meta{0, 1}, o, L, wr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (pass == 1) printf("recip_us %.2f\n", ms * 1e3 / 200);
        cudaEventRecord(e0);
        for (int r = 0; r < 200; ++r) k_mul<<<1, 256, wc * 4>>>(d, y, o, L);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (pass == 1) printf("mul_us %.2f\n", ms * 1e3 / 200);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
