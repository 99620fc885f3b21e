// tools/tc_probe.cu — dev probe of the int8 tcgen05 building blocks (run on the
// GPU box): (1) one/many MMAs with A K-major, B MN-major vs a CPU GEMM;
// (2) the 1-D im2col product: D[k][t] = sum_u Yr[k][u] * X[t+u] with B read
// through an MN-major descriptor over the 16x-expanded x (cell p = x[p..p+15]).
#include "../paper_1810_01478_b200/csrc/tc_i8.cuh"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

using namespace hk::tc;

constexpr int M = 128, NN = 256, KK = 32;

// A: rows x 32 bytes per K-step, K-major interleaved: [kstep][rowgroup][chunk][8 rows][16 B]
// B: K x 256, MN-major interleaved: [kstep][nblock(16)][kgroup(4)][8 krows][16 B]
__global__ void k_gemm(const uint8_t* A, const uint8_t* B, int32_t* D, int ksteps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;                 // 128*32 = 4096 B per kstep
    uint8_t* sB = sm + 4096;          // 32*256 = 8192 B per kstep
    __shared__ uint64_t mbar;
    __shared__ uint32_t taddr_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tmem_alloc(&taddr_s, 256);
    if (tid == 0) mbar_init(&mbar, 1);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = taddr_s;
    uint32_t phase = 0;
    for (int ks = 0; ks < ksteps; ++ks) {
        // stage A (K-major): element (r, k) -> (r/8)*256 + (k/16)*128 + (r%8)*16 + k%16
        for (int i = tid; i < M * KK; i += blockDim.x) {
            const int r = i / KK, k = i % KK;
            sA[(r / 8) * 256 + (k / 16) * 128 + (r % 8) * 16 + (k % 16)] = A[(size_t)ks * M * KK + i];
        }
        // stage B (MN-major): element (k, n) -> (n/16)*512 + (k/8)*128 + (k%8)*16 + n%16
        for (int i = tid; i < KK * NN; i += blockDim.x) {
            const int k = i / NN, n = i % NN;
            sB[(n / 16) * 512 + (k / 8) * 128 + (k % 8) * 16 + (n % 16)] = B[(size_t)ks * KK * NN + i];
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            fence_after();
            const uint64_t ad = sdesc(sA, 128, 256);
            const uint64_t bd = sdesc(sB, 128, 512);
            mma_i8(tmem, ad, bd, idesc_u8(M, NN, false, true), ks > 0);
            commit(&mbar);
        }
        mbar_wait(&mbar, phase);
        phase ^= 1;
        fence_after();
    }
    // each warp reads its 32 lanes (rows), 256 columns
    for (int c0 = 0; c0 < NN; c0 += 8) {
        uint32_t v[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        tmem_ld_wait();
        const int row = warp * 32 + (tid & 31);
        for (int q = 0; q < 8; ++q) D[row * NN + c0 + q] = (int32_t)v[q];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

// im2col product: Yr [128][nb] (reversed y bytes), X [nb] bytes; output t in [t0, t0+256)
// D[k][t - t0] = sum_{u} Yr[k][u] * X[t + u]   (X zero outside [0, nb))
// B operand over the expanded array E: cell p (16 B) = X[p .. p+15], stored at
// Ebase + 16*(p - pmin).  B(k=u, n=t) = X[t+u] = byte (t+u - p) of cell p with
// p = t0 + 16*nb_blk + u  ->  nblock stride 256 B (SBO), krow stride 16 B, kgroup 128 B (LBO).
__global__ void k_im2col(const uint8_t* Yr, const uint8_t* X, int nb, int t0, int32_t* D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* sA = sm;                       // 4096 B per kstep
    uint8_t* sE = sm + 4096;                // expanded X window
    __shared__ uint64_t mbar;
    __shared__ uint32_t taddr_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int ksteps = (nb + KK - 1) / KK;
    // cells needed: p = t0 + 16*blk + u, u in [0, 32*ksteps), blk in [0,16) -> p in [t0, t0 + 256 + 32*ksteps)
    const int ncell = 256 + KK * ksteps;
    for (int c = tid; c < ncell; c += blockDim.x)
        for (int b = 0; b < 16; ++b) {
            const int idx = t0 + c + b;
            sE[c * 16 + b] = (idx >= 0 && idx < nb) ? X[idx] : 0;
        }
    if (warp == 0) tmem_alloc(&taddr_s, 256);
    if (tid == 0) mbar_init(&mbar, 1);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = taddr_s;
    uint32_t phase = 0;
    for (int ks = 0; ks < ksteps; ++ks) {
        for (int i = tid; i < M * KK; i += blockDim.x) {
            const int r = i / KK, k = i % KK, u = ks * KK + k;
            sA[(r / 8) * 256 + (k / 16) * 128 + (r % 8) * 16 + (k % 16)] = u < nb ? Yr[(size_t)r * nb + u] : 0;
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            fence_after();
            const uint64_t ad = sdesc(sA, 128, 256);
            // B rows u = ks*32 + kk: cell p = t0 + 16*blk + u -> offset 16*(16*blk + u) from sE (cell 0 = p t0)
            const uint64_t bd = sdesc(sE + 16 * (ks * KK), 128, 256);
            mma_i8(tmem, ad, bd, idesc_u8(M, NN, false, true), ks > 0);
            commit(&mbar);
        }
        mbar_wait(&mbar, phase);
        phase ^= 1;
        fence_after();
    }
    for (int c0 = 0; c0 < NN; c0 += 8) {
        uint32_t v[8];
        tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        tmem_ld_wait();
        const int row = warp * 32 + (tid & 31);
        for (int q = 0; q < 8; ++q) D[row * NN + c0 + q] = (int32_t)v[q];
    }
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 256);
}

static uint32_t rng = 12345;
static uint8_t rb() {
    rng = rng * 1664525u + 1013904223u;
    return uint8_t(rng >> 24);
}

int main() {
    int bad_total = 0;
    for (int ksteps : {1, 3}) {
        std::vector<uint8_t> A((size_t)ksteps * M * KK), B((size_t)ksteps * KK * NN);
        for (auto& a : A) a = rb();
        for (auto& b : B) b = rb();
        uint8_t *dA, *dB;
        int32_t* dD;
        cudaMalloc(&dA, A.size());
        cudaMalloc(&dB, B.size());
        cudaMalloc(&dD, M * NN * 4);
        cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
        k_gemm<<<1, 128, 4096 + 8192>>>(dA, dB, dD, ksteps);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<int32_t> D(M * NN);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < M; ++r)
            for (int n = 0; n < NN; ++n) {
                long long s = 0;
                for (int ks = 0; ks < ksteps; ++ks)
                    for (int k = 0; k < KK; ++k)
                        s += (long long)A[(size_t)ks * M * KK + r * KK + k] * B[(size_t)ks * KK * NN + k * NN + n];
                if (s != D[r * NN + n]) {
                    if (bad < 3) printf("  gemm mismatch r=%d n=%d got %d want %lld\n", r, n, D[r * NN + n], s);
                    ++bad;
                }
            }
        printf("gemm ksteps=%d: %s, %d mismatches\n", ksteps, cudaGetErrorString(e), bad);
        bad_total += bad;
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dD);
    }
    for (int nb : {64, 200}) {
        for (int t0 : {-40, 0, 100}) {
            std::vector<uint8_t> Yr((size_t)M * nb), X(nb);
            for (auto& a : Yr) a = rb();
            for (auto& b : X) b = rb();
            uint8_t *dY, *dX;
            int32_t* dD;
            cudaMalloc(&dY, Yr.size());
            cudaMalloc(&dX, X.size());
            cudaMalloc(&dD, M * NN * 4);
            cudaMemcpy(dY, Yr.data(), Yr.size(), cudaMemcpyHostToDevice);
            cudaMemcpy(dX, X.data(), X.size(), cudaMemcpyHostToDevice);
            const int ksteps = (nb + KK - 1) / KK;
            const size_t smem = 4096 + 16 * (256 + KK * ksteps);
            cudaFuncSetAttribute(k_im2col, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_im2col<<<1, 128, smem>>>(dY, dX, nb, t0, dD);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<int32_t> D(M * NN);
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int r = 0; r < M; ++r)
                for (int n = 0; n < NN; ++n) {
                    long long s = 0;
                    const int t = t0 + n;
                    for (int u = 0; u < nb; ++u) {
                        const int xi = t + u;
                        if (xi >= 0 && xi < nb) s += (long long)Yr[(size_t)r * nb + u] * X[xi];
                    }
                    if (s != D[r * NN + n]) {
                        if (bad < 3) printf("  im2col mismatch r=%d n=%d got %d want %lld\n", r, n, D[r * NN + n], s);
                        ++bad;
                    }
                }
            printf("im2col nb=%d t0=%d: %s, %d mismatches\n", nb, t0, cudaGetErrorString(e), bad);
            bad_total += bad;
            cudaFree(dY);
            cudaFree(dX);
            cudaFree(dD);
        }
    }
    printf("TOTAL_BAD %d\n", bad_total);
    return bad_total != 0;
}
