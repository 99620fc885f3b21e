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
constexpr int kTcKB = 4;         // MMAs (K-steps) per staged A block
constexpr int kTcABuf = 4096 * kTcKB; // bytes per A buffer (2 buffers)

HK_HD int tc_nb(int L) { return 4 * L; }
HK_HD int tc_ncell(int L) { return tc_nb(L) + 352; }        // cells p in [-31, nb + 321)
HK_HD int tc_sx_words(int L) { return (tc_nb(L) + 512) / 4; }
HK_HD size_t tc_smem_bytes(int L) {
    return 2 * (size_t)kTcABuf + 16 * (size_t)tc_ncell(L) + 4 * (size_t)tc_sx_words(L) + 64;
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
    __shared__ uint64_t mbarb[2];
    __shared__ uint32_t taddr_s;
    if (*(volatile const int*)a.err >= 0) return;
    const int N = a.N, L = a.L, nb = tc_nb(L);
    const int j = a.jfirst + int(blockIdx.x);
    const int k0 = j + kTcRows * int(blockIdx.y);
    if (j >= N || k0 >= N) return;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint8_t* sA = tsm;                                   // 2 x 16 KB: A blocks (4 K-major 128 x 32 B tiles)
    uint8_t* sE = tsm + 2 * kTcABuf;                     // expanded x cells
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
    if (tid == 0) {
        tc::mbar_init(&mbarb[0], 1);
        tc::mbar_init(&mbarb[1], 1);
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = taddr_s;
    const uint32_t idesc = tc::idesc_u8(kTcRows, kTcN, false, true);

    const int r = tid;            // this thread's row / TMEM lane
    const int k = k0 + r;
    const bool row_ok = k < N;
    const long long n2 = N - a.jfirst;
    const long long item = row_ok ? col_off(j - a.jfirst, int(n2)) + (k - j) : 0;
    uint32_t* Pout = a.P + item * (long long)tc_scratch_limbs(L);
    const uint32_t* yl_row = a.B.limbs(row_ok ? k : k0, L);
    uint64_t carry = 0;
    uint32_t bph[2] = {0u, 0u}; // per-buffer mbarrier phases

    // stage the A K-block `blk` (kTcKB MMAs = 128 rows x 128 B) into buffer `buf`
    auto stage = [&](int blk, int buf, int ksteps) {
        uint8_t* dst = sA + buf * kTcABuf;
        for (int q = tid; q < kTcRows * 2 * kTcKB; q += kTcThreads) {
            const int sub = q / (kTcRows * 2), qq = q % (kTcRows * 2);
            const int rr = qq >> 1, h = qq & 1;
            const int ks = blk * kTcKB + sub;
            const int u0 = ks * kTcK + 16 * h;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (ks < ksteps && k0 + rr < N && u0 < nb) {
                // Yr[u0 .. u0+15] = Y[nb-1-u0 .. nb-16-u0] = reversed limbs [L-4-u0/4, L-u0/4)
                const uint4 g = *reinterpret_cast<const uint4*>(a.B.limbs(k0 + rr, L) + (L - 4 - u0 / 4));
                v.x = __byte_perm(g.w, 0u, 0x0123);
                v.y = __byte_perm(g.z, 0u, 0x0123);
                v.z = __byte_perm(g.y, 0u, 0x0123);
                v.w = __byte_perm(g.x, 0u, 0x0123);
            }
            *reinterpret_cast<uint4*>(dst + sub * 4096 + (rr >> 3) * 256 + h * 128 + (rr & 7) * 16) = v;
        }
        tc::fence_async_smem();
    };

    for (int tc0 = -31, ch = 0; tc0 < nb + 1; tc0 += kTcN, ++ch) {
        const int u_hi = tc0 < 0 ? nb : nb - tc0;             // u' < u_hi contribute
        const int ksteps = (u_hi + kTcK - 1) / kTcK;
        const int nblk = (ksteps + kTcKB - 1) / kTcKB;
        // double-buffered pipeline: MMAs of block b run while block b+1 is staged
        stage(0, 0, ksteps);
        __syncthreads();
        for (int b = 0; b < nblk; ++b) {
            const int buf = b & 1;
            if (tid == 0) {
                tc::fence_after();
                for (int sub = 0; sub < kTcKB; ++sub) {
                    const int ks = b * kTcKB + sub;
                    if (ks >= ksteps) break;
                    const uint64_t ad = tc::sdesc(sA + buf * kTcABuf + sub * 4096, 128, 256);
                    const uint64_t bd = tc::sdesc(sE + 16 * (size_t)(tc0 + ks * kTcK - pmin), 128, 256);
                    tc::mma_i8(tmem, ad, bd, idesc, ks > 0 ? 1u : 0u);
                }
                tc::commit(&mbarb[buf]);
            }
            if (b + 1 < nblk) {
                if (b >= 1) { // buffer (b+1)&1 was last read by block b-1's MMAs
                    tc::mbar_wait(&mbarb[(b + 1) & 1], bph[(b + 1) & 1]);
                    bph[(b + 1) & 1] ^= 1u;
                }
                stage(b + 1, (b + 1) & 1, ksteps);
            }
            __syncthreads();
        }
        // drain: the last block's commit (and the one before, if not yet awaited)
        if (nblk >= 2) {
            tc::mbar_wait(&mbarb[(nblk - 2) & 1], bph[(nblk - 2) & 1]);
            bph[(nblk - 2) & 1] ^= 1u;
        }
        tc::mbar_wait(&mbarb[(nblk - 1) & 1], bph[(nblk - 1) & 1]);
        bph[(nblk - 1) & 1] ^= 1u;
        tc::fence_after();
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
// The window needs max(L, L+8, L) + 4 words; the rare items the certificate
// cannot settle are appended to `fb` and redone exactly by k_tc_fix (so this
// pass runs at high occupancy with a window-sized workspace).
HK_HD int tcround_words(int L) { return (L + 16 + 3) & ~3; }

struct ItemTcRound {
    MpArr S, B;
    const uint32_t* P;
    int N, L, i, jfirst;
    const int* err;
    int* fb_count;
    long long* fb;
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
        if (sp == 0) return; // x or y zero: RNE(c - 0) = c, nothing to write
        const int t0 = L - kTcGuard;
        const int lsbP = xm.exp + ym.exp - 64 * L;
        const Opd X{c, L, cm.exp - 32 * L, cm.sign};
        const Opd Y{P + w * (long long)tc_scratch_limbs(L), tc_scratch_limbs(L), lsbP + 32 * t0, sp};
        bool ok = false;
        const RMeta rr = warp_round_sum(X, Y, ws, c, L, lsbP + 32 * t0 + 46, &ok);
        if (lane() == 0) {
            if (ok) {
                S.m[ec] = Meta{rr.exp, rr.sign};
            } else {
#if defined(HK_WARP_EMU)
                fb[(*fb_count)++] = w;
#else
                fb[atomicAdd(fb_count, 1)] = w;
#endif
            }
        }
        wsync();
    }
};

#if !defined(HK_WARP_EMU)
// Exact redo of the uncertified items: S(k,j) = RNE(S(k,j) - S(j,i) B_i(k)).
__global__ void __launch_bounds__(256) k_tc_fix(MpArr S, MpArr B, int N, int L, int i, int jfirst,
                                                const int* fb_count, const long long* fb, int ws_words) {
    extern __shared__ uint32_t fsm[];
    const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    uint32_t* ws = fsm + (size_t)wib * ws_words;
    const int cnt = *fb_count;
    for (long long q = (long long)blockIdx.x * wpb + wib; q < cnt; q += (long long)gridDim.x * wpb) {
        const long long w = fb[q];
        int jj, kk;
        tri_decode(w, N - jfirst, jj, kk);
        const int j = jfirst + jj, k = jfirst + kk;
        const long long ec = tri_idx(k, j, N), ex = tri_idx(j, i, N);
        uint32_t* c = S.limbs(ec, L);
        const Meta m = warp_fms(c, S.m[ec], S.limbs(ex, L), S.m[ex], B.limbs(k, L), B.m[k], c, L, opws_carve(ws, L));
        if (lane() == 0) S.m[ec] = m;
        wsync();
    }
}
#endif

} // namespace hk
