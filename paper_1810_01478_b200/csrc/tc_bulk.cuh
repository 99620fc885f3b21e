// tc_bulk.cuh — the LDLT bulk update's limb products on the 5th-gen tensor
// cores (tcgen05.mma kind::i8, u8 x u8 -> s32), for large p.
//
// For column j of step i every row k >= jfirst.. needs P_kj = x_j * y_k with
// x_j = S(j,i), y_k = B_i(k) (L-limb integers = nb = 4L bytes).  In bytes,
// P[t] = sum_u Y[u] X[t-u].  With Yr[u'] = Y[nb-1-u'] and t' = t - (nb-1):
//     D[t'] = sum_u' Yr[u'] X[t'+u']            ("1-D im2col")
// a GEMM with M = rows k (128 per tile, A = reversed y bytes, K-major), K = u'
// and N = output positions t' (256 per MMA).  B(u', t') = X[t'+u'] is read
// through an MN-major SWIZZLE_NONE descriptor over the 16x-expanded x: cell p =
// bytes X[p..p+15] at sE + 16 (p - pmin), so N-blocks are 256 B apart (SBO),
// K-rows 16 B (core matrix) and K-groups 128 B (LBO) — constant positive
// strides, no per-tile Toeplitz materialisation (validated in tools/tc_probe.cu).
//
// Only t' >= -31 is formed (the short product from limb L-8): the dropped byte
// columns are < 2^(32 (L-8) + 30) units of the product's LSB, inside the bound
// warp_round_sum's Ziv certificate uses (ubit = lsbP + 32 t0 + 46), so the
// second pass (ItemTcRound) still returns exactly RNE(c - x y) or falls back to
// the exact warp FMA.  The epilogue carries the int32 column sums into 32-bit
// limbs per row (one thread per TMEM lane) and writes them to a scratch buffer.
#pragma once

#include "hk_items.cuh"
#include "tc_i8.cuh"

namespace hk {

constexpr int kTcRows = 128;     // M per tile (TMEM lanes)
constexpr int kTcN = 256;        // N per MMA (TMEM columns)
constexpr int kTcK = 32;         // K per MMA (bytes)
constexpr int kTcGuard = 8;      // short product from limb L - 8
constexpr int kTcThreads = 128;  // 4 warps: one thread per row / TMEM lane

HK_HD int tc_nb(int L) { return 4 * L; }
HK_HD int tc_ncell(int L) { return tc_nb(L) + 352; }        // cells p in [-31, nb + 321)
HK_HD int tc_sx_words(int L) { return (tc_nb(L) + 512) / 4; }
HK_HD size_t tc_smem_bytes(int L) {
    return 4096 + 16 * (size_t)tc_ncell(L) + 4 * (size_t)tc_sx_words(L) + 64;
}
HK_HD int tc_scratch_limbs(int L) { return L + kTcGuard; }  // limbs [L-8, 2L)

struct TcBulkArgs {
    MpArr S, B;                  // S (jagged), B_i
    uint32_t* P;                 // scratch: item -> tc_scratch_limbs(L) limbs
    int N, L, i, jfirst;
    const int* err;
};

// blockIdx.x: column offset (j = jfirst + x); blockIdx.y: row tile (k0 = j + 128 y)
__global__ void __launch_bounds__(kTcThreads) k_tc_bulk(TcBulkArgs a) {
    extern __shared__ __align__(1024) uint8_t tsm[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t taddr_s;
    if (*(volatile const int*)a.err >= 0) return;
    const int N = a.N, L = a.L, nb = tc_nb(L);
    const int j = a.jfirst + int(blockIdx.x);
    const int k0 = j + kTcRows * int(blockIdx.y);
    if (j >= N || k0 >= N) return;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint8_t* sA = tsm;                                   // 4 KB: 128 rows x 32 B, K-major core matrices
    uint8_t* sE = tsm + 4096;                            // expanded x cells
    uint32_t* sX = reinterpret_cast<uint32_t*>(sE + 16 * (size_t)tc_ncell(L)); // x bytes, 32-byte zero pad
    const int pmin = -31;

    // x_j = S(j, i) bytes into sX (word 8 = byte 32 holds X[0])
    const uint32_t* xl = a.S.limbs(tri_idx(j, a.i, N), L);
    for (int w = tid; w < tc_sx_words(L); w += kTcThreads) sX[w] = (w >= 8 && w < 8 + L) ? xl[w - 8] : 0u;
    __syncthreads();
    // cells p = pmin + c: X[p .. p+15] (zero outside [0, nb))
    for (int c = tid; c < tc_ncell(L); c += kTcThreads) {
        const int off = 32 + pmin + c; // byte offset in sX (>= 1)
        const int w0 = off >> 2, sh = (off & 3) * 8;
        uint32_t W[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) W[q] = (w0 + q < tc_sx_words(L)) ? sX[w0 + q] : 0u;
        uint4 v;
        v.x = __funnelshift_r(W[0], W[1], sh);
        v.y = __funnelshift_r(W[1], W[2], sh);
        v.z = __funnelshift_r(W[2], W[3], sh);
        v.w = __funnelshift_r(W[3], W[4], sh);
        *reinterpret_cast<uint4*>(sE + 16 * (size_t)c) = v;
    }
    if (warp == 0) tc::tmem_alloc(&taddr_s, kTcN);
    if (tid == 0) tc::mbar_init(&mbar, 1);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = taddr_s;
    const uint32_t idesc = tc::idesc_u8(kTcRows, kTcN, false, true);
    uint32_t phase = 0;

    const int r = tid;            // this thread's row / TMEM lane
    const int k = k0 + r;
    const bool row_ok = k < N;
    const long long n2 = N - a.jfirst;
    const long long item = row_ok ? col_off(j - a.jfirst, int(n2)) + (k - j) : 0;
    uint32_t* Pout = a.P + item * (long long)tc_scratch_limbs(L);
    const uint32_t* yl_row = a.B.limbs(row_ok ? k : k0, L);
    uint64_t carry = 0;

    for (int tc0 = -31, ch = 0; tc0 < nb + 1; tc0 += kTcN, ++ch) {
        const int u_hi = tc0 < 0 ? nb : nb - tc0;             // u' < u_hi contribute
        const int ksteps = (u_hi + kTcK - 1) / kTcK;
        for (int ks = 0; ks < ksteps; ++ks) {
            // stage A: rows k0.., bytes u' in [32 ks, 32 ks + 32) of reversed y
            for (int q = tid; q < kTcRows * 2; q += kTcThreads) {
                const int rr = q >> 1, h = q & 1;
                const int u0 = ks * kTcK + 16 * h;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (k0 + rr < N && u0 < nb) {
                    // Yr[u0 .. u0+15] = Y[nb-1-u0 .. nb-16-u0] = reversed limbs [L-4-u0/4, L-u0/4)
                    const uint4 g = *reinterpret_cast<const uint4*>(a.B.limbs(k0 + rr, L) + (L - 4 - u0 / 4));
                    v.x = __byte_perm(g.w, 0u, 0x0123);
                    v.y = __byte_perm(g.z, 0u, 0x0123);
                    v.z = __byte_perm(g.y, 0u, 0x0123);
                    v.w = __byte_perm(g.x, 0u, 0x0123);
                }
                *reinterpret_cast<uint4*>(sA + (rr >> 3) * 256 + h * 128 + (rr & 7) * 16) = v;
            }
            tc::fence_async_smem();
            __syncthreads();
            if (tid == 0) {
                tc::fence_after();
                const uint64_t ad = tc::sdesc(sA, 128, 256);
                const uint64_t bd = tc::sdesc(sE + 16 * (size_t)(tc0 + ks * kTcK - pmin), 128, 256);
                tc::mma_i8(tmem, ad, bd, idesc, ks > 0 ? 1u : 0u);
                tc::commit(&mbar);
            }
            tc::mbar_wait(&mbar, phase);
            phase ^= 1;
            tc::fence_after();
        }
        // epilogue: this row's 256 byte-column sums -> 64 limbs (exact carries)
        for (int c8 = 0; c8 < kTcN; c8 += 8) {
            uint32_t v[8];
            tc::tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c8, v);
            tc::tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint64_t s = carry + (uint64_t)v[4 * h] + ((uint64_t)v[4 * h + 1] << 8) +
                             ((uint64_t)v[4 * h + 2] << 16) + ((uint64_t)v[4 * h + 3] << 24);
                const int lq = ch * 64 + (c8 >> 2) + h; // limb index relative to L - 8
                if (row_ok && lq < tc_scratch_limbs(L)) Pout[lq] = uint32_t(s);
                carry = s >> 32;
            }
        }
        tc::fence_before();
        __syncthreads(); // TMEM reads done before the next chunk's MMAs overwrite it
        tc::fence_after();
    }
    (void)yl_row;
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, kTcN);
}

// Second pass: S(k,j) = RNE(S(k,j) - x_j y_k) from the scratch product, with the
// Ziv certificate; exact warp FMA when it cannot certify.  Items enumerate the
// column-major triangle of columns jfirst..N-1 (as ItemTrailing / the scratch).
struct ItemTcRound {
    MpArr S, B;
    const uint32_t* P;
    int N, L, i, jfirst;
    const int* err;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int n2 = N - jfirst;
        int jj, kk;
        tri_decode(w, n2, jj, kk);
        const int j = jfirst + jj, k = jfirst + kk;
        const long long ec = tri_idx(k, j, N), ex = tri_idx(j, i, N);
        const Meta cm = S.m[ec], xm = S.m[ex], ym = B.m[k];
        uint32_t* c = S.limbs(ec, L);
        const int sp = -(xm.sign * ym.sign);
        const int t0 = L - kTcGuard;
        const int lsbP = xm.exp + ym.exp - 64 * L;
        Meta r;
        if (sp != 0) {
            const Opd X{c, L, cm.exp - 32 * L, cm.sign};
            const Opd Y{P + w * (long long)tc_scratch_limbs(L), tc_scratch_limbs(L), lsbP + 32 * t0, sp};
            bool ok = false;
            const RMeta rr = warp_round_sum(X, Y, ws, c, L, lsbP + 32 * t0 + 46, &ok);
            if (ok) r = Meta{rr.exp, rr.sign};
            else r = warp_fms(c, cm, S.limbs(ex, L), xm, B.limbs(k, L), ym, c, L, opws_carve(ws, L));
        } else {
            r = cm; // x or y zero: c unchanged (RNE(c) = c)
        }
        if (lane() == 0) S.m[ec] = r;
        wsync();
    }
};

} // namespace hk
