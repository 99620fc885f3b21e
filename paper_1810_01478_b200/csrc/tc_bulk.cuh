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
#include "tc_fused.cuh"
#include "tc_i8.cuh"

namespace hk {

constexpr int kTcRows = 128;     // M per tile (TMEM lanes)
constexpr int kTcN = 256;        // N per MMA (TMEM columns per accumulator)
constexpr int kTcK = 32;         // K per MMA (bytes)
constexpr int kTcGuard = 8;      // short product from limb L - 8
constexpr int kTcThreads = 256;  // warp 0: TMA + MMA issue; warps 4-7: epilogue (TMEM lanes 32 (w % 4)..)
constexpr int kTcKB = 4;         // MMAs (K-steps) per A block
constexpr int kTcBlk = 4096 * kTcKB; // bytes per A block (one bulk copy)
constexpr int kTcStages = 4;     // A ring depth (3 with the fused rounding: its 32 KB staging)
constexpr int kTcStagesMax = 8;  // CTA pairs: one CTA per SM, a deeper ring
constexpr int kTcStagesFused = 3;
constexpr int kTcStageWords = 64 * kTcRows; // fused epilogue: one chunk's 64 limbs per row

HK_HD int tc_nb(int L) { return 4 * L; }
HK_HD int tc_ncell(int L) { return tc_nb(L) + 352; }        // cells p in [-31, nb + 321)
HK_HD int tc_sx_words(int L) { return (tc_nb(L) + 512) / 4; }
HK_HD int tc_nks(int L) { return (tc_nb(L) + kTcK - 1) / kTcK; }
HK_HD int tc_nblk(int L) { return (tc_nks(L) + kTcKB - 1) / kTcKB; }
HK_HD int tc_ntiles(int N) { return (N + kTcRows - 1) / kTcRows; }
HK_HD int tc_nchunks(int L) { return (tc_nb(L) + 32 + kTcN - 1) / kTcN; }
constexpr int kTcMaxGroups = 8; // chunk groups per product (L^-1)
constexpr int kTcEWin = 384;    // cells of x one A block's 4 K-steps read (windowed expansion)
// Full expansion: all nb + 352 cells built once per CTA.  Windowed (large p,
// where the full expansion would not fit): warps 1-3 build each block's
// 384-cell window into a ring next to the A ring, paced by the same barriers.
HK_HD int tc_stages(bool fuse, int force = 0) { return force > 0 ? force : fuse ? kTcStagesFused : kTcStages; }
HK_HD size_t tc_sx_off(int L, bool ewin, int ns) {
    const size_t e = ewin ? (size_t)ns * kTcEWin * 16 : 16 * (size_t)tc_ncell(L);
    return (size_t)ns * kTcBlk + e;
}
HK_HD size_t tc_stage_off(int L, bool ewin, int ns) {
    return (tc_sx_off(L, ewin, ns) + 4 * (size_t)tc_sx_words(L) + 127) / 128 * 128;
}
HK_HD size_t tc_smem_bytes(int L, bool ewin = false, bool fuse = false, int force_stages = 0) {
    return tc_stage_off(L, ewin, tc_stages(fuse, force_stages)) + (fuse ? 4 * (size_t)kTcStageWords : 0) + 64;
}
HK_HD bool tc_ewin(int L) { return tc_smem_bytes(L, false) > 200 * 1024; }
// The fused rounding: LDLT steps (modes 0 / 2) whose rows are whole 8-limb
// blocks, when two CTAs still fit an SM (227 KB of shared memory per SM)
HK_HD bool tc_fits2(size_t bytes) { return bytes + 1024 <= 113 * 1024; } // two CTAs per SM
HK_HD int tc_fused_stages(int L) { return tc_fits2(tc_smem_bytes(L, true, true, kTcStagesFused)) ? kTcStagesFused : 2; }
HK_HD bool tc_fusable(int L) { return L % 8 == 0 && tc_fits2(tc_smem_bytes(L, true, true, 2)); }

// A blocks (4 K-steps each) of output chunk c; chunk c covers product bytes from
// t' = -31 + 256 c, i.e. scratch limbs [64 c, 64 c + 64).
HK_HD int tc_chunk_blocks(int L, int c) {
    const int nb = tc_nb(L), tc0 = -31 + 256 * c;
    const int u_hi = tc0 < 0 ? nb : nb - tc0; // u' < u_hi contribute
    return (((u_hi + 31) / 32) + 3) / 4;
}
// First chunk of group z when the chunks are split into G groups of about
// equal MMA work (narrow L^-1 steps run G CTAs per (column, row tile)).
HK_HD int tc_group_first_chunk(int L, int G, int z) {
    if (z <= 0) return 0;
    const int nch = tc_nchunks(L);
    if (z >= G) return nch;
    long long Q = 0;
    for (int c = 0; c < nch; ++c) Q += tc_chunk_blocks(L, c);
    const long long target = Q * z / G;
    long long acc = 0;
    int c = 0;
    while (c < nch && acc < target) acc += tc_chunk_blocks(L, c++);
    return c;
}
HK_HD int tc_scratch_limbs(int L) { return L + kTcGuard; }  // limbs [L-8, 2L)
// preformatted A operand of one step: [row tile][A block][4 K-steps x 128 rows x 32 B],
// plus one all-zero tile past N (the second CTA of a pair may start there)
HK_HD size_t tc_apre_bytes(int N, int L) { return (size_t)(tc_ntiles(N) + 1) * tc_nblk(L) * kTcBlk; }

// A operand of step i in the MMA's K-major SWIZZLE_NONE layout: row k = 128 tile
// + rr, K-step ks holds reversed bytes Yr[32 ks .. 32 ks + 31] of the row operand
// (LDLT: y_k = B_i(k); L^-1: L(k, i) = S(k, i)), zero for k <= i, k >= N or past
// nb.  Tiles from tile0 = (i + 1) / 128 on.  16 B per thread, coalesced writes.
struct ItemTcPrep {
    MpArr R;   // LDLT: B_i (row k at k);  L^-1: S (row k at tri_idx(k, i)), or the panel (row k at k - i)
    uint8_t* A;
    int N, L, i, mode;
    int panel = 0;
    HK_DEV void operator()(long long u) const {
        const int nb = tc_nb(L);
        const long long per_tile = (long long)tc_nblk(L) * kTcKB * 256;
        const int tile0 = (i + 1) / kTcRows;
        u += tile0 * per_tile;
        const int tile = int(u / per_tile);
        const int rem = int(u % per_tile);
        const int ks = rem >> 8, w = rem & 255;
        const int rr = (w >> 4) * 8 + (w & 7), h = (w >> 3) & 1;
        const int k = tile * kTcRows + rr;
        const int u0 = ks * kTcK + 16 * h;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (k > i && k < N && u0 < nb) {
            const uint32_t* row = mode != 1 ? R.limbs(k, L) : R.limbs(lcol_idx(k, i, N, panel), L);
            const uint4 g = *reinterpret_cast<const uint4*>(row + (L - 4 - u0 / 4));
            v.x = __byte_perm(g.w, 0u, 0x0123);
            v.y = __byte_perm(g.z, 0u, 0x0123);
            v.z = __byte_perm(g.y, 0u, 0x0123);
            v.w = __byte_perm(g.x, 0u, 0x0123);
        }
        reinterpret_cast<uint4*>(A)[u] = v;
    }
    HK_HD long long count() const { // tiles (i + 1) / 128 .. ntiles (the last one: the zero pad tile)
        return (long long)(tc_ntiles(N) + 1 - (i + 1) / kTcRows) * tc_nblk(L) * kTcKB * 256;
    }
};

#if !defined(HK_WARP_EMU)
// griddepcontrol.wait: under programmatic dependent launch (the LDLT bulk
// stream) a grid may start before its predecessor finishes; it waits here for
// the predecessor's completion and memory before touching its outputs (no-op
// for an ordinary launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(256) k_tc_prep(ItemTcPrep f, long long n) {
    pdl_wait();
    const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) f(u);
}
#endif

// mode 0 (LDLT step i): CTA column j = jfirst + x with x operand S(j, i), rows
//   k >= j, item = (column-major triangle of columns jfirst..N-1)(k, j).
// mode 1 (L^-1 step i): CTA column c = x < b with x operand X(i, c), rows j > i,
//   item = (j - i - 1) b + c.
struct TcBulkArgs {
    MpArr S;                     // S (jagged)
    MpArr X;                     // L^-1 columns (mode 1), row-major N x m
    const uint8_t* A;            // preformatted A (ItemTcPrep)
    uint32_t* P;                 // scratch: item -> tc_scratch_limbs(L) limbs
    int N, L, i, jfirst, mode, m, b;
    const int* err;
    int nacc = 2;
    int ewin = 0;            // windowed x expansion
    int groups = 1;          // chunk groups (blockIdx.z): G > 1 only for L^-1 steps
    uint64_t* gcarry = nullptr; // [item][G - 1]: carry out of each group but the last
    // mode 2 (column-sharded LDLT, one rank's owned columns): CTA x -> local column
    // first_loc + x, global column owned[.], local entries from off[.]; x operand =
    // the broadcast panel (X) entry j - i; items = local entry index - e0
    const int* owned = nullptr;
    const long long* off = nullptr;
    long long e0 = 0;
    int first_loc = 0;
    int dev = 0; // dev what-if knobs (results wrong; tools only): 1 no window build, 2 no TMA of A, 4 no drain, 8 no P stores,
                 // 16 no fused processing, 64 issuer wait counters, 128 pair occupancy, 256 ignore the pivot flag
    // fused rounding (modes 0 / 2, groups == 1): S(k,j) = RNE(S(k,j) - x y_k) in the epilogue
    int fuse = 0;               // 1: thread-per-row stream, 2: warp-cooperative stream
    MpArr Y{};                  // y_k = B_i(k) (the row operand)
    int* fb_count = nullptr;    // items left to the exact redo
    long long* fb = nullptr;
    int force_fb = 0;           // tests: every 7th item to the exact redo (HK_TC_FORCE_FIX)
    int* viol = nullptr;        // tests: normalisation-check failures (must stay 0)
    int sleep_ns = 0;           // back-off of the epilogue / window-builder barrier polls
    int stages = 0;             // ring depth override (dev sweeps; 0 = default for the mode)
    const int* otiles = nullptr; // mode 1, sharded L^-1: this rank's row tiles (blockIdx.y -> otiles[y])
    int inv_gate = 0;            // mode 1 riding in the LDLT graph: stop once the LDLT raised a precision error
    unsigned long long* dev_cnt = nullptr; // dev (bit 64): issuer cycles waiting on empty / full / efull / accE, total
};

#if !defined(HK_WARP_EMU)
// The fused rounding (tc_fused.cuh) as the epilogue of one CTA's 128 rows:
// the thread of row k drains its product limbs chunk by chunk into its
// shared-memory row (the accumulator is released at once), then streams them
// through FusedRow into S(k,j) in place.  nacc accumulators (TMEM columns
// 256 a, chunk c in accumulator c % nacc).  accE_rank < 0: arrive on this
// CTA's accE; else on CTA accE_rank's of the cluster.
__device__ __forceinline__ void fused_epilogue(const TcBulkArgs& a, int tile, int j, int locj, const uint32_t* sX,
                                               uint32_t* sStg, uint32_t tmem, int c_lo, int nch, uint64_t* accF,
                                               uint64_t* accE, int accE_rank, int nacc = 1) {
    const int N = a.N, L = a.L;
    const int tid = threadIdx.x, warp = tid >> 5, ln = tid & 31;
    const int r = 32 * (warp & 3) + ln;
    const int k = tile * kTcRows + r;
    const bool row_ok = k >= j && k < N;
    long long item = 0, ec = 0;
    FusedRow fr;
    fr.status = 0;
    fr.wlane = ln;
    fr.wbase = reinterpret_cast<uint32_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(
                                                                         a.S.limbs(tri_idx(tile * kTcRows, j, N), L)),
                                                      0));
    if (row_ok) {
        Meta xm;
        if (a.mode == 0) {
            ec = tri_idx(k, j, N);
            item = col_off(j - a.jfirst, N - a.jfirst) + (k - j);
            xm = a.S.m[tri_idx(j, a.i, N)];
        } else {
            ec = a.off[locj] + (k - j);
            item = ec - a.e0;
            xm = a.X.m[j - a.i];
        }
        const uint64_t xt = (uint64_t(sX[8 + L - 1]) << 32) | sX[8 + L - 2];
        const uint32_t* yl = a.Y.limbs(k, L);
        const uint64_t yt = (uint64_t(yl[L - 1]) << 32) | yl[L - 2];
        fr.dev = a.dev;
        fr.setup(a.S.limbs(ec, L), a.S.m[ec], xt, xm, yt, a.Y.m[k], L);
        if (a.force_fb && item % 7 == 3 && fr.status != 0) fr.status = 2;
    }
    fr.prefetch(8 * c_lo, 16); // the first two chunks' c limbs
    uint32_t* stg = sStg + 64 * r; // 16 x 16-byte cells, XOR-swizzled by row (conflict-free)
    const int sw = r & 15;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    uint64_t carry = 0;
    const bool prof = (a.dev & 64) && a.dev_cnt && tid == 128; // one epilogue thread's time split
    unsigned long long e_wait = 0, e_drain = 0, e_proc = 0, e_t0 = clock64();
    for (int c = c_lo; c < nch; ++c) {
        const int cl = c - c_lo;
        const int ab = cl % nacc;
        const unsigned long long t0 = prof ? clock64() : 0;
        tc::mbar_wait_sleep(&accF[ab], uint32_t(cl / nacc) & 1u, a.sleep_ns);
        const unsigned long long t1 = prof ? clock64() : 0;
        tc::fence_after();
        for (int c32 = 0; c32 < kTcN; c32 += 32) {
            uint32_t v[32];
            tc::tmem_ld32(lane_base + uint32_t(ab * kTcN + c32), v);
            tc::tmem_ld_wait();
            uint32_t o[8];
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const uint64_t s = carry + (uint64_t)v[4 * h] + ((uint64_t)v[4 * h + 1] << 8) +
                                   ((uint64_t)v[4 * h + 2] << 16) + ((uint64_t)v[4 * h + 3] << 24);
                o[h] = uint32_t(s);
                carry = s >> 32;
            }
            const int q = c32 >> 4; // 16-byte cells q, q + 1: limbs 4 q .. 4 q + 7 (8 limbs per 32 columns)
            reinterpret_cast<uint4*>(stg)[q ^ sw] = make_uint4(o[0], o[1], o[2], o[3]);
            reinterpret_cast<uint4*>(stg)[(q + 1) ^ sw] = make_uint4(o[4], o[5], o[6], o[7]);
        }
        tc::fence_before();
        __syncwarp();
        if (ln == 0) { // the MMAs of chunk c + 1 may now overwrite it
            if (accE_rank < 0)
                tc::mbar_arrive(&accE[ab]);
            else
                tc::mbar_arrive_remote(&accE[ab], uint32_t(accE_rank));
        }
        fr.prefetch(8 * (c + 2), 8);              // c limbs of chunk c + 2, while c and c + 1 stream
        const unsigned long long t2 = prof ? clock64() : 0;
        for (int gg = 0; gg < 8; ++gg) {
            const int g = 8 * c + gg;
            if (!fr.wants(g) || (a.dev & 16)) continue;
            const uint4 v0 = reinterpret_cast<const uint4*>(stg)[(2 * gg) ^ sw];
            const uint4 v1 = reinterpret_cast<const uint4*>(stg)[(2 * gg + 1) ^ sw];
            const uint32_t pl[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            fr.group(g, pl);
        }
        if (prof) {
            const unsigned long long t3 = clock64();
            e_wait += t1 - t0;
            e_drain += t2 - t1;
            e_proc += t3 - t2;
        }
    }
    if (prof) {
        atomicAdd(a.dev_cnt + 8, e_wait);
        atomicAdd(a.dev_cnt + 9, e_drain);
        atomicAdd(a.dev_cnt + 10, e_proc);
        atomicAdd(a.dev_cnt + 11, clock64() - e_t0);
    }
    {
        const uint32_t zero[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        for (int g = 8 * nch; fr.wants(g); ++g) fr.group(g, zero);
    }
    if (row_ok) {
        Meta mo{0, 0};
        bool viol = false;
        const bool ok = fr.finish(&mo, &viol);
        if (viol && a.viol) atomicAdd(a.viol, 1);
        if (!ok) {
            if (!(a.dev & 512)) a.fb[atomicAdd(a.fb_count, 1)] = item;
        } else if (fr.status == 1) {
            a.S.m[ec] = mo;
        }
    }
}
#endif

#if !defined(HK_WARP_EMU)
// The fused rounding with the warp-cooperative stream (tc_fused.cuh
// warp_row_*): drain as fused_epilogue, then each epilogue warp streams its 32
// rows one at a time with coalesced c accesses (the next row's loads issued
// while the current one is computed).
__device__ __forceinline__ void fused_epilogue_warp(const TcBulkArgs& a, int tile, int j, int locj,
                                                    const uint32_t* sX, uint32_t* sStg, uint32_t tmem, int c_lo,
                                                    int nch, uint64_t* accF, uint64_t* accE, int accE_rank,
                                                    int nacc = 1) {
    const int N = a.N, L = a.L;
    const int tid = threadIdx.x, warp = tid >> 5, ln = tid & 31;
    const int r = 32 * (warp & 3) + ln, rbase = 32 * (warp & 3);
    const int k = tile * kTcRows + r;
    const bool row_ok = k >= j && k < N;
    // row r (this warp's rows rbase + 0..31) -> entry of S
    auto entry_of = [&](int rr) -> long long {
        const int kk = tile * kTcRows + rbase + rr;
        return a.mode == 0 ? tri_idx(kk, j, N) : a.off[locj] + (kk - j);
    };
    long long item = 0, ec = 0;
    FusedRow fr;
    fr.status = 0;
    if (row_ok) {
        ec = entry_of(ln);
        item = a.mode == 0 ? col_off(j - a.jfirst, N - a.jfirst) + (k - j) : ec - a.e0;
        const Meta xm = a.mode == 0 ? a.S.m[tri_idx(j, a.i, N)] : a.X.m[j - a.i];
        const uint64_t xt = (uint64_t(sX[8 + L - 1]) << 32) | sX[8 + L - 2];
        const uint32_t* yl = a.Y.limbs(k, L);
        const uint64_t yt = (uint64_t(yl[L - 1]) << 32) | yl[L - 2];
        fr.setup(a.S.limbs(ec, L), a.S.m[ec], xt, xm, yt, a.Y.m[k], L);
        if (a.force_fb && item % 7 == 3 && fr.status != 0) fr.status = 2;
    }
    WarpRowState own = warp_row_init(fr);
    fr.prefetch(8 * c_lo, 16); // the first two chunks' c limbs into L2
    uint32_t* stg = sStg + 64 * r;
    const int sw = r & 15;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    uint64_t carry = 0;
    auto row_ptr = [&](int rr) { return a.S.limbs(entry_of(rr), L); };
    // one chunk of all 32 rows; staged: product limbs from the staging rows (else zeros)
    auto stream = [&](int c, bool staged) {
        bool any = false;
        WarpRowState bn = warp_row_bcast(own, 0);
        uint32_t qn0, qn1;
        warp_row_load(bn, row_ptr(0), L, c, qn0, qn1);
        for (int rr = 0; rr < 32; ++rr) {
            WarpRowState b = bn;
            const uint32_t q0 = qn0, q1 = qn1;
            if (rr + 1 < 32) {
                bn = warp_row_bcast(own, rr + 1);
                warp_row_load(bn, row_ptr(rr + 1), L, c, qn0, qn1);
            }
            if (b.status() != 1 || 64 * c - 1 - int(b.prm & 0xffffu) >= L) continue;
            any = true;
            uint32_t p0 = 0u, p1 = 0u;
            if (staged) { // limbs 2 ln, 2 ln + 1 of staging row rbase + rr (16-byte cells, XOR-swizzled)
                const uint32_t* srow = sStg + 64 * (rbase + rr);
                const uint2 v = reinterpret_cast<const uint2*>(srow)[2 * ((ln >> 1) ^ ((rbase + rr) & 15)) + (ln & 1)];
                p0 = v.x;
                p1 = v.y;
            }
            warp_row_chunk(b, row_ptr(rr), L, c, p0, p1, q0, q1);
            if (ln == rr) own = b;
        }
        return any;
    };
    for (int c = c_lo; c < nch; ++c) {
        const int cl = c - c_lo;
        const int ab = cl % nacc;
        tc::mbar_wait_sleep(&accF[ab], uint32_t(cl / nacc) & 1u, a.sleep_ns);
        tc::fence_after();
        for (int c32 = 0; c32 < kTcN; c32 += 32) {
            uint32_t v[32];
            tc::tmem_ld32(lane_base + uint32_t(ab * kTcN + c32), v);
            tc::tmem_ld_wait();
            uint32_t o[8];
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const uint64_t s = carry + (uint64_t)v[4 * h] + ((uint64_t)v[4 * h + 1] << 8) +
                                   ((uint64_t)v[4 * h + 2] << 16) + ((uint64_t)v[4 * h + 3] << 24);
                o[h] = uint32_t(s);
                carry = s >> 32;
            }
            const int q = c32 >> 4;
            reinterpret_cast<uint4*>(stg)[q ^ sw] = make_uint4(o[0], o[1], o[2], o[3]);
            reinterpret_cast<uint4*>(stg)[(q + 1) ^ sw] = make_uint4(o[4], o[5], o[6], o[7]);
        }
        tc::fence_before();
        __syncwarp(); // the warp reads its rows' staged limbs next
        if (ln == 0) {
            if (accE_rank < 0)
                tc::mbar_arrive(&accE[ab]);
            else
                tc::mbar_arrive_remote(&accE[ab], uint32_t(accE_rank));
        }
        fr.prefetch(8 * (c + 2), 8);
        if (!(a.dev & 16)) stream(c, true);
        __syncwarp(); // staging rows rewritten by the next drain
    }
    for (int c = nch; !(a.dev & 16) && stream(c, false); ++c) {
    }
    if (row_ok) {
        Meta mo{0, 0};
        bool viol = false;
        const bool ok = warp_row_finish(own, fr, a.S.limbs(ec, L), L, &mo, &viol);
        if (viol && a.viol) atomicAdd(a.viol, 1);
        if (!ok) {
            if (!(a.dev & 512)) a.fb[atomicAdd(a.fb_count, 1)] = item;
        } else if (fr.status == 1) {
            a.S.m[ec] = mo;
        }
    }
}
#endif

#if !defined(HK_WARP_EMU)
// blockIdx.x: column offset (j = jfirst + x); blockIdx.y: row tile offset (tile = j / 128 + y).
// Rows k of the tile with j <= k < N are this CTA's items (k, j).
//
// Pipeline: thread 0 streams A blocks through a kTcStages ring with bulk copies
// (full[s]: TMA bytes landed; empty[s]: the MMAs reading slot s retired, via
// tcgen05.commit) and issues the MMAs of output chunk c into TMEM accumulator
// c & 1; warps 4-7 drain accumulator c & 1 (carry the int32 byte-column sums
// into limbs) while chunk c + 1 accumulates into the other one (accF / accE).
__global__ void __launch_bounds__(kTcThreads, 2) k_tc_bulk(TcBulkArgs a) {
    extern __shared__ __align__(1024) uint8_t tsm[];
    __shared__ uint64_t full[kTcStages], empty[kTcStages], efull[kTcStages], accF[2], accE[2];
    __shared__ uint32_t taddr_s;
    if ((a.mode != 1 || a.inv_gate) && !(a.dev & 256) && *(volatile const int*)a.err >= 0) return; // LDLT precision error raised
    const int N = a.N, L = a.L, nb = tc_nb(L);
    const int locj = a.first_loc + int(blockIdx.x);
    const int j = a.mode == 0 ? a.jfirst + int(blockIdx.x) : a.mode == 2 ? a.owned[locj] : a.i + 1; // first valid row
    const int tile = a.otiles ? a.otiles[blockIdx.y] : j / kTcRows + int(blockIdx.y);
    if (j >= N || tile * kTcRows >= N) return;
    const int tid = threadIdx.x, warp = tid >> 5, ln = tid & 31;
    const bool ewin = a.ewin != 0;
    const bool fuse = a.fuse != 0;
    const int ns = tc_stages(fuse, a.stages);              // A / window ring depth
    uint8_t* sA = tsm;                                     // ns x 16 KB A ring
    uint8_t* sE = tsm + (size_t)ns * kTcBlk;               // expanded x cells (full, or the window ring)
    uint32_t* sX = reinterpret_cast<uint32_t*>(tsm + tc_sx_off(L, ewin, ns)); // x bytes, 32 B zero pad
    uint32_t* sStg = reinterpret_cast<uint32_t*>(tsm + tc_stage_off(L, ewin, ns)); // fused: drained chunk
    const int pmin = -31;
    // cell p (byte position in X, p >= pmin) -> X[p .. p+15] from sX (zero outside [0, nb))
    auto cell = [&](int p) {
        const int off = 32 + p; // byte offset in sX (>= 1)
        const int w0 = off >> 2, sh = (off & 3) * 8;
        uint32_t W[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) W[q] = sX[w0 + q]; // w0 + 4 < (nb + 512) / 4 for every cell p < nb + 352
        uint4 v;
        v.x = __funnelshift_r(W[0], W[1], sh);
        v.y = __funnelshift_r(W[1], W[2], sh);
        v.z = __funnelshift_r(W[2], W[3], sh);
        v.w = __funnelshift_r(W[3], W[4], sh);
        return v;
    };

    // x bytes into sX (word 8 = byte 32 holds X[0]); cells p = pmin + c: X[p .. p+15]
    const uint32_t* xl = a.mode == 0   ? a.S.limbs(tri_idx(j, a.i, N), L)
                         : a.mode == 2 ? a.X.limbs(j - a.i, L)
                                       : a.X.limbs((long long)a.i * a.m + blockIdx.x, L);
    for (int w = tid; w < tc_sx_words(L); w += kTcThreads) sX[w] = (w >= 8 && w < 8 + L) ? xl[w - 8] : 0u;
    __syncthreads();
    if (!ewin) {
        for (int c = tid; c < tc_ncell(L); c += kTcThreads)
            *reinterpret_cast<uint4*>(sE + 16 * (size_t)c) = cell(pmin + c);
        tc::fence_async_smem(); // generic-proxy writes of sE -> visible to the tensor core
    }
    const int nacc = a.nacc; // TMEM accumulators (1: two CTAs per SM overlap instead)
    if (warp == 0) tc::tmem_alloc(&taddr_s, uint32_t(nacc * kTcN));
    if (tid == 0) {
        for (int s = 0; s < ns; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
            tc::mbar_init(&efull[s], 3); // one arrival per builder warp (1-3)
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&accF[b], 1);
            tc::mbar_init(&accE[b], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = taddr_s;
    // this CTA's output chunks [c_lo, nch)
    const int G = a.groups, z = int(blockIdx.z);
    const int c_lo = tc_group_first_chunk(L, G, z);
    const int nch = tc_group_first_chunk(L, G, z + 1);
    auto nblk_of = [&](int c) { return tc_chunk_blocks(L, c); };

    if (warp == 0) {
        if (ln == 0) {
            const uint32_t idesc = tc::idesc_u8(kTcRows, kTcN, false, true);
            const uint8_t* Abase = a.A + (size_t)tile * tc_nblk(L) * kTcBlk;
            int Q = 0;
            for (int c = c_lo; c < nch; ++c) Q += nblk_of(c);
            // producer cursor: block index qt -> (chunk pc, block pb)
            int qt = 0, pc = c_lo, pb = 0, pcn = nblk_of(c_lo);
            const bool prof = (a.dev & 64) && a.dev_cnt;
            unsigned long long w_empty = 0, w_full = 0, w_efull = 0, w_acc = 0, t_start = clock64();
            auto issue_tma = [&]() {
                const int s = qt % ns;
                const unsigned long long t0 = prof ? clock64() : 0;
                if (qt >= ns) tc::mbar_wait(&empty[s], uint32_t((qt / ns) - 1) & 1u);
                if (prof) w_empty += clock64() - t0;
                tc::mbar_expect_tx(&full[s], kTcBlk);
                tc::bulk_g2s(sA + (size_t)s * kTcBlk, Abase + (size_t)pb * kTcBlk, kTcBlk, &full[s]);
                ++qt;
                if (++pb == pcn && ++pc < nch) {
                    pb = 0;
                    pcn = nblk_of(pc);
                }
            };
            pdl_wait(); // the A operand comes from the preceding k_tc_prep
            while (qt < Q && qt < ns - 1 && !(a.dev & 2)) issue_tma();
            int q = 0;
            for (int c = c_lo; c < nch; ++c) {
                const int cl = c - c_lo; // local chunk index (accumulator / phase)
                const int ab = cl % nacc;
                const unsigned long long ta = prof ? clock64() : 0;
                if (cl >= nacc) tc::mbar_wait(&accE[ab], uint32_t((cl - nacc) / nacc) & 1u);
                if (prof) w_acc += clock64() - ta;
                tc::fence_after();
                const int tc0 = -31 + kTcN * c;
                const int u_hi = tc0 < 0 ? nb : nb - tc0;
                const int ksteps = (u_hi + kTcK - 1) / kTcK;
                const int nblk = nblk_of(c);
                for (int b = 0; b < nblk; ++b, ++q) {
                    const int s = q % ns;
                    const unsigned long long tf = prof ? clock64() : 0;
                    if (!(a.dev & 2)) tc::mbar_wait(&full[s], uint32_t(q / ns) & 1u);
                    const unsigned long long te = prof ? clock64() : 0;
                    if (ewin && !(a.dev & 1)) tc::mbar_wait(&efull[s], uint32_t(q / ns) & 1u);
                    if (prof) {
                        w_full += te - tf;
                        w_efull += clock64() - te;
                    }
                    tc::fence_after();
#pragma unroll
                    for (int sub = 0; sub < kTcKB; ++sub) {
                        const int ks = b * kTcKB + sub;
                        if (ks < ksteps) {
                            const uint64_t ad = tc::sdesc(sA + (size_t)s * kTcBlk + sub * 4096, 128, 256);
                            const uint64_t bd =
                                ewin ? tc::sdesc(sE + (size_t)s * kTcEWin * 16 + 16 * (size_t)(sub * kTcK), 128, 256)
                                     : tc::sdesc(sE + 16 * (size_t)(tc0 + ks * kTcK - pmin), 128, 256);
                            tc::mma_i8(tmem + uint32_t(ab * kTcN), ad, bd, idesc, ks > 0 ? 1u : 0u);
                        }
                    }
                    tc::commit(&empty[s]);
                    if (qt < Q && !(a.dev & 2)) issue_tma(); // refills the slot block q - 1 used
                }
                tc::commit(&accF[ab]);
            }
            if (prof) {
                atomicAdd(a.dev_cnt + 0, w_empty);
                atomicAdd(a.dev_cnt + 1, w_full);
                atomicAdd(a.dev_cnt + 2, w_efull);
                atomicAdd(a.dev_cnt + 3, w_acc);
                atomicAdd(a.dev_cnt + 4, clock64() - t_start);
                atomicAdd(a.dev_cnt + 5, 1ull);
            }
        }
        __syncwarp();
    } else if (warp < 4) {
        if (ewin && !(a.dev & 1)) { // warps 1-3: the x window of every block, in issue order
            const int bt = tid - 32;
            int q = 0;
            for (int c = c_lo; c < nch; ++c) {
                const int tc0 = -31 + kTcN * c, nblk = nblk_of(c);
                for (int b = 0; b < nblk; ++b, ++q) {
                    const int s = q % ns;
                    if (q >= ns) tc::mbar_wait_sleep(&empty[s], uint32_t((q / ns) - 1) & 1u, a.sleep_ns);
                    uint8_t* dst = sE + (size_t)s * kTcEWin * 16;
                    const int p0 = tc0 + b * kTcKB * kTcK;
                    for (int cc = bt; cc < kTcEWin; cc += 96) *reinterpret_cast<uint4*>(dst + 16 * cc) = cell(p0 + cc);
                    tc::fence_async_smem();
                    __syncwarp();
                    if (ln == 0) tc::mbar_arrive(&efull[s]);
                }
            }
        }
    } else if (fuse) {
        if (a.fuse == 2)
            fused_epilogue_warp(a, tile, j, locj, sX, sStg, tmem, c_lo, nch, accF, accE, -1);
        else
            fused_epilogue(a, tile, j, locj, sX, sStg, tmem, c_lo, nch, accF, accE, -1);
    } else {
        const int r = 32 * (warp & 3) + ln; // this thread's row / TMEM lane
        const int k = tile * kTcRows + r;
        const bool row_ok = k >= j && k < N;
        long long item = 0;
        if (row_ok)
            item = a.mode == 0   ? col_off(j - a.jfirst, N - a.jfirst) + (k - j)
                   : a.mode == 2 ? a.off[locj] + (k - j) - a.e0
                                 : (long long)(k - a.i - 1) * a.b + blockIdx.x;
        uint32_t* Pout = a.P + item * (long long)tc_scratch_limbs(L);
        const uint32_t lane_base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
        uint64_t carry = 0;
        for (int c = c_lo; c < nch; ++c) {
            const int cl = c - c_lo;
            const int ab = cl % nacc;
            tc::mbar_wait_sleep(&accF[ab], uint32_t(cl / nacc) & 1u, a.sleep_ns);
            tc::fence_after();
            for (int c32 = 0; c32 < kTcN && !(a.dev & 4); c32 += 32) {
                uint32_t v[32];
                tc::tmem_ld32(lane_base + uint32_t(ab * kTcN + c32), v);
                tc::tmem_ld_wait();
                uint32_t o[8];
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    const uint64_t s = carry + (uint64_t)v[4 * h] + ((uint64_t)v[4 * h + 1] << 8) +
                                       ((uint64_t)v[4 * h + 2] << 16) + ((uint64_t)v[4 * h + 3] << 24);
                    o[h] = uint32_t(s);
                    carry = s >> 32;
                }
                const int lq = c * 64 + (c32 >> 2); // limb index relative to L - 8 (multiple of 8)
                if (row_ok && !(a.dev & 8)) {
                    if (lq + 8 <= tc_scratch_limbs(L) && (L & 7) == 0) {
                        tc::st_global_v8(Pout + lq, o); // item stride (L+8) limbs: 32-byte aligned
                    } else if (lq + 8 <= tc_scratch_limbs(L)) {
                        reinterpret_cast<uint4*>(Pout + lq)[0] = make_uint4(o[0], o[1], o[2], o[3]);
                        reinterpret_cast<uint4*>(Pout + lq)[1] = make_uint4(o[4], o[5], o[6], o[7]);
                    } else {
#pragma unroll
                        for (int h = 0; h < 8; ++h)
                            if (lq + h < tc_scratch_limbs(L)) Pout[lq + h] = o[h];
                    }
                }
            }
            tc::fence_before();
            __syncwarp();
            if (ln == 0) tc::mbar_arrive(&accE[ab]);
        }
        if (G > 1 && z < G - 1 && row_ok) a.gcarry[item * (G - 1) + z] = carry; // added in the rounding pass
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0) tc::tmem_dealloc(tmem, uint32_t(nacc * kTcN));
}
#endif

// Second pass: S(k,j) = RNE(S(k,j) - x_j y_k) from the scratch product, with the
// Ziv certificate; exact warp FMA when it cannot certify.  Items enumerate the
// column-major triangle of columns jfirst..N-1 (as ItemTrailing / the scratch).
// The rounding passes first copy both operands (c: L limbs, the product: L+8
// limbs) into the warp's shared workspace with cp.async (all loads in flight at
// once), then round from shared memory; the window G needs max(L, L+8, L) + 4
// words.  The rare items the certificate cannot settle are appended to `fb`
// and redone exactly by k_tc_fix.
HK_HD int tcround_words(int L) { return align4(L) + align4(L + kTcGuard) + align4(L + 16); }

#if defined(HK_WARP_EMU)
HK_DEV void warp_stage16(uint32_t* dst, const uint32_t* src, int nwords) {
    for (int q = lane(); q < nwords; q += 32) dst[q] = src[q];
    wsync();
}
#else
// nwords % 4 == 0, both pointers 16-byte aligned
HK_DEV void warp_stage16(uint32_t* dst, const uint32_t* src, int nwords) {
    for (int q = 4 * lane(); q < nwords; q += 128)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(dst + q)), "l"(src + q)
                     : "memory");
}
#endif
HK_DEV void warp_stage_wait() {
#if !defined(HK_WARP_EMU)
    asm volatile("cp.async.wait_all;" ::: "memory");
#endif
    wsync();
}

// tests (HK_TC_FORCE_FIX): the item goes to the exact fix-up list without rounding
HK_DEV void force_to_fix(long long w, int* fb_count, long long* fb) {
    if (lane() == 0) {
#if defined(HK_WARP_EMU)
        fb[(*fb_count)++] = w;
#else
        fb[atomicAdd(fb_count, 1)] = w;
#endif
    }
    wsync();
}

// each chunk group of the product kernel started from carry 0: add the carries
// (gc[z] out of group z) back in, from the first limb of group z + 1 upwards
HK_DEV void join_group_carries(uint32_t* Ys, int L, int G, const uint64_t* gc) {
    if (lane() == 0)
        for (int z = 0; z + 1 < G; ++z) {
            uint64_t v = gc[z];
            for (int q = 64 * tc_group_first_chunk(L, G, z + 1); v != 0 && q < tc_scratch_limbs(L); ++q) {
                v += Ys[q];
                Ys[q] = uint32_t(v);
                v >>= 32;
            }
        }
    wsync();
}

struct ItemTcRound {
    MpArr S, B;
    const uint32_t* P;
    int N, L, i, jfirst;
    const int* err;
    int* fb_count;
    long long* fb;
    int force_fb = 0; // tests: every 7th certified item is sent to the exact fix-up anyway (HK_TC_FORCE_FIX)
    int direct = 0; // 1: operands read in place from global memory, only the window in shared memory
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        const int n2 = N - jfirst;
        int jj, kk;
        tri_decode(w, n2, jj, kk);
        item(w, jfirst + jj, jfirst + kk, ws);
    }
    // 2-D launch (k_cols): column offset jj, row r of that column
    HK_DEV int rows(int jj) const { return N - jfirst - jj; }
    HK_DEV void operator()(int jj, int r, uint32_t* ws) const {
        item(col_off(jj, N - jfirst) + r, jfirst + jj, jfirst + jj + r, ws);
    }
    HK_DEV void item(long long w, int j, int k, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const long long ec = tri_idx(k, j, N), ex = tri_idx(j, i, N);
        const Meta cm = S.m[ec], xm = S.m[ex], ym = B.m[k];
        uint32_t* c = S.limbs(ec, L);
        const int sp = -(xm.sign * ym.sign);
        if (sp == 0) return; // x or y zero: RNE(c - 0) = c, nothing to write
        if (force_fb && w % 7 == 3) return force_to_fix(w, fb_count, fb);
        const int t0 = L - kTcGuard;
        const int lsbP = xm.exp + ym.exp - 64 * L;
        const uint32_t* Pw = P + w * (long long)tc_scratch_limbs(L);
        const uint32_t* Xs = c;
        const uint32_t* Ys = Pw;
        uint32_t* Gw = ws;
        if (!direct) {
            uint32_t* xs = ws;
            uint32_t* ys = ws + align4(L);
            warp_stage16(xs, c, L);
            warp_stage16(ys, Pw, tc_scratch_limbs(L));
            warp_stage_wait();
            Xs = xs;
            Ys = ys;
            Gw = ys + align4(L + kTcGuard);
        }
        const Opd X{Xs, L, cm.exp - 32 * L, cm.sign, 32 * L};
        const Opd Y{Ys, tc_scratch_limbs(L), lsbP + 32 * t0, sp};
        bool ok = false;
        const RMeta rr = warp_round_sum(X, Y, Gw, c, L, lsbP + 32 * t0 + 46, &ok);
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

// L^-1 step i (mode 1): X(j,c) = RNE(X(j,c) - L(j,i) X(i,c)) for the (N-i-1) b
// product items, then (i < m) the copies X(j,i) = -L(j,i) as in ItemInvStep.
struct ItemTcRoundInv {
    MpArr S, X;
    const uint32_t* P;
    int N, L, m, i, b;
    int* fb_count;
    long long* fb;
    int force_fb = 0; // tests: every 7th certified item is sent to the exact fix-up anyway (HK_TC_FORCE_FIX)
    int G = 1;                       // chunk groups of the product kernel
    const uint64_t* gcarry = nullptr; // their carries, added here
    int panel = 0, rw = 1, rr = 0;   // sharded: L(:, i) from the panel S, this rank's rows only
    const int* err = nullptr;        // steps riding in the LDLT graph: nothing to do once a pivot failed
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (err && *(volatile const int*)err >= 0) return;
        const long long nfma = (long long)(N - i - 1) * b;
        if (w >= nfma) {
            const int j = i + 1 + int(w - nfma);
            if (!row_mine(j, rw, rr)) return;
            const long long el = lcol_idx(j, i, N, panel);
            const long long xd = (long long)j * m + i;
            copy_entry(X.limbs(xd, L), X.m + xd, S.limbs(el, L), S.m + el, L);
            if (lane() == 0) X.m[xd].sign = -X.m[xd].sign;
            wsync();
            return;
        }
        const int j = i + 1 + int(w / b), c = int(w % b);
        if (!row_mine(j, rw, rr)) return;
        const long long xc = (long long)j * m + c, xi = (long long)i * m + c, el = lcol_idx(j, i, N, panel);
        const Meta cm = X.m[xc], xm = S.m[el], ym = X.m[xi];
        const int sp = -(xm.sign * ym.sign);
        if (sp == 0) return;
        if (force_fb && w % 7 == 3) return force_to_fix(w, fb_count, fb);
        uint32_t* o = X.limbs(xc, L);
        const int t0 = L - kTcGuard;
        const int lsbP = xm.exp + ym.exp - 64 * L;
        uint32_t* Xs = ws;
        uint32_t* Ys = ws + align4(L);
        warp_stage16(Xs, o, L);
        warp_stage16(Ys, P + w * (long long)tc_scratch_limbs(L), tc_scratch_limbs(L));
        warp_stage_wait();
        if (G > 1) join_group_carries(Ys, L, G, gcarry + w * (G - 1));
        const Opd Xo{Xs, L, cm.exp - 32 * L, cm.sign, 32 * L};
        const Opd Y{Ys, tc_scratch_limbs(L), lsbP + 32 * t0, sp};
        bool ok = false;
        const RMeta rr = warp_round_sum(Xo, Y, Ys + align4(L + kTcGuard), o, L,
                                             lsbP + 32 * t0 + 46, &ok);
        if (lane() == 0) {
            if (ok) {
                X.m[xc] = Meta{rr.exp, rr.sign};
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

// Sharded LDLT step i on one rank (mode 2): local entry e = e0 + w of the owned
// columns >= i+1, S(k,j) = RNE(S(k,j) - panel(j-i) B_i(k)) (ItemDTrailing's op).
struct ItemTcRoundD {
    MpArr S, panel, B;
    const int* erow;
    const int* ecol;
    const uint32_t* P;
    int L, i;
    long long e0;
    const int* err;
    int* fb_count;
    long long* fb;
    int force_fb = 0; // tests: every 7th certified item is sent to the exact fix-up anyway (HK_TC_FORCE_FIX)
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const long long e = e0 + w;
        const int k = erow[e], j = ecol[e];
        const Meta cm = S.m[e], xm = panel.m[j - i], ym = B.m[k];
        const int sp = -(xm.sign * ym.sign);
        if (sp == 0) return;
        if (force_fb && w % 7 == 3) return force_to_fix(w, fb_count, fb);
        uint32_t* c = S.limbs(e, L);
        const int t0 = L - kTcGuard;
        const int lsbP = xm.exp + ym.exp - 64 * L;
        uint32_t* Xs = ws;
        uint32_t* Ys = ws + align4(L);
        warp_stage16(Xs, c, L);
        warp_stage16(Ys, P + w * (long long)tc_scratch_limbs(L), tc_scratch_limbs(L));
        warp_stage_wait();
        const Opd X{Xs, L, cm.exp - 32 * L, cm.sign, 32 * L};
        const Opd Y{Ys, tc_scratch_limbs(L), lsbP + 32 * t0, sp};
        bool ok = false;
        const RMeta rr = warp_round_sum(X, Y, Ys + align4(L + kTcGuard), c, L, lsbP + 32 * t0 + 46, &ok);
        if (lane() == 0) {
            if (ok) {
                S.m[e] = Meta{rr.exp, rr.sign};
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

// Exact redo of one uncertified item (full warp FMA workspace).
struct FixLdlt {
    MpArr S, B;
    int N, L, i, jfirst;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        int jj, kk;
        tri_decode(w, N - jfirst, jj, kk);
        const int j = jfirst + jj, k = jfirst + kk;
        const long long ec = tri_idx(k, j, N), ex = tri_idx(j, i, N);
        uint32_t* c = S.limbs(ec, L);
        const Meta r = warp_fms(c, S.m[ec], S.limbs(ex, L), S.m[ex], B.limbs(k, L), B.m[k], c, L, opws_carve(ws, L));
        if (lane() == 0) S.m[ec] = r;
        wsync();
    }
};
struct FixInv {
    MpArr S, X;
    int N, L, m, i, b;
    int panel = 0;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        const int j = i + 1 + int(w / b), c = int(w % b);
        const long long xc = (long long)j * m + c, xi = (long long)i * m + c, el = lcol_idx(j, i, N, panel);
        uint32_t* o = X.limbs(xc, L);
        const Meta r = warp_fms(o, X.m[xc], S.limbs(el, L), S.m[el], X.limbs(xi, L), X.m[xi], o, L, opws_carve(ws, L));
        if (lane() == 0) X.m[xc] = r;
        wsync();
    }
};

struct FixD {
    MpArr S, panel, B;
    const int* erow;
    const int* ecol;
    int L, i;
    long long e0;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        const long long e = e0 + w;
        const int k = erow[e], j = ecol[e];
        uint32_t* c = S.limbs(e, L);
        const Meta r =
            warp_fms(c, S.m[e], panel.limbs(j - i, L), panel.m[j - i], B.limbs(k, L), B.m[k], c, L, opws_carve(ws, L));
        if (lane() == 0) S.m[e] = r;
        wsync();
    }
};

#if !defined(HK_WARP_EMU)
// Column-wise launch of a per-(column, row) item (no triangle decode per item):
// blockIdx.y = column offset, warps stride over that column's rows.
template <class F>
__global__ void __launch_bounds__(256) k_cols(F f, int ws_words) {
    extern __shared__ __align__(16) uint32_t csm[];
    pdl_wait();
    const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    uint32_t* ws = csm + (size_t)wib * ws_words;
    const int jj = int(blockIdx.y), rows = f.rows(jj);
    for (int r = int(blockIdx.x) * wpb + wib; r < rows; r += int(gridDim.x) * wpb) f(jj, r, ws);
}

template <class F>
__global__ void __launch_bounds__(256) k_tc_fix(F f, const int* fb_count, const long long* fb, int ws_words,
                                                int* reset, unsigned long long* total) {
    pdl_wait();
    extern __shared__ uint32_t fsm[];
    const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    uint32_t* ws = fsm + (size_t)wib * ws_words;
    const int cnt = *fb_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *reset = 0;                                   // the counter the next step uses
        if (total) atomicAdd(total, (unsigned long long)cnt); // items redone exactly (hk_fix_count)
    }
    for (long long q = (long long)blockIdx.x * wpb + wib; q < cnt; q += (long long)gridDim.x * wpb) f(fb[q], ws);
}
#endif

} // namespace hk
