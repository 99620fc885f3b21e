// tc_pair.cuh — the LDLT bulk products with the fused rounding on CTA pairs
// (tcgen05.mma.cta_group::2): the two CTAs of a cluster on one TPC take two
// consecutive 128-row tiles of the same column j and issue one M = 256 MMA
// per K-step.  Both tiles multiply the same x = S(j,i), so the B operand (the
// Toeplitz window of x's bytes) is shared: each CTA builds and holds only its
// half of the 256 output columns (128 columns x 32 K-bytes = 4 KB per K-step
// instead of 8 KB), which halves the window build and the B-operand shared-
// memory reads per SM — the kernel's limiter with one CTA per MMA (ncu: the
// tensor core's operand reads, the TMA writes of A and the window builders
// together near the shared-memory bandwidth, tensor pipe ~50-70% busy).
//
// Roles (256 threads per CTA, as k_tc_bulk):
//   thread 0     streams its tile's A blocks through the ring (TMA); in the
//                leader (rank 0) it also issues the pair's MMAs and commits
//                them to both CTAs' barriers; in rank 1 it forwards "my A
//                block landed and my window half is built" to the leader
//   warps 1-3    build this CTA's window half of every A block
//   warps 4-7    the fused epilogue of this CTA's 128 rows (fused_epilogue),
//                releasing the accumulator on the leader's accE (8 arrivals)
// Everything else (operand formats, chunks, short product, certified
// rounding, fix-up list) is k_tc_bulk's.
#pragma once

#include "tc_bulk.cuh"

namespace hk {

constexpr int kTcEWinPair = 256; // window cells per A block and CTA (its 128 output columns + 128 K bytes)

HK_HD size_t tcp_sx_off(int ns) { return (size_t)ns * kTcBlk + (size_t)ns * kTcEWinPair * 16; }
HK_HD size_t tcp_stage_off(int L, int ns) { return (tcp_sx_off(ns) + 4 * (size_t)tc_sx_words(L) + 127) / 128 * 128; }
HK_HD size_t tcp_smem_bytes(int L, int ns) { return tcp_stage_off(L, ns) + 4 * (size_t)kTcStageWords + 64; }
// A kernel that allocates TMEM with cta_group::2 runs one CTA per SM (the
// driver's occupancy for it is one cluster per TPC, measured), so the CTA takes
// all 512 TMEM columns — two accumulators: the epilogue of chunk c overlaps the
// MMAs of chunk c + 1 — and a deep ring in up to 227 KB of shared memory
HK_HD int tcp_stages(int L) {
    for (int ns = kTcStagesMax; ns > 2; --ns)
        if (tcp_smem_bytes(L, ns) + 1024 <= 227 * 1024) return ns;
    return 2;
}
HK_HD bool tcp_ok(int L) { return L % 8 == 0 && tcp_smem_bytes(L, 2) + 1024 <= 227 * 1024; }

#if !defined(HK_WARP_EMU)
// grid (2 * pairs of row tiles, columns), cluster (2, 1, 1) — the pair along x; modes 0 / 2, fused
__global__ void __launch_bounds__(kTcThreads, 1) k_tc_pair(TcBulkArgs a) {
    extern __shared__ __align__(1024) uint8_t tsm[];
    __shared__ uint64_t full[kTcStagesMax], empty[kTcStagesMax], efull[kTcStagesMax], pready[kTcStagesMax], accF[2],
        accE[2];
    __shared__ uint32_t taddr_s;
    const uint32_t rank = tc::cluster_rank();
    const int N = a.N, L = a.L, nb = tc_nb(L);
    const int locj = a.first_loc + int(blockIdx.y);
    const int j = a.mode == 0 ? a.jfirst + int(blockIdx.y) : a.owned[locj];
    const int tile0 = j / kTcRows + (int(blockIdx.x) & ~1); // the pair's first tile: both CTAs decide alike
    if (j >= N || tile0 * kTcRows >= N) return;
    const int tile = tile0 + int(rank); // rank 1's tile may lie past N: zero A rows (padded A), no items
    const int tid = threadIdx.x, warp = tid >> 5, ln = tid & 31;
    const int ns = a.stages;
    uint8_t* sA = tsm;
    uint8_t* sE = tsm + (size_t)ns * kTcBlk;
    uint32_t* sX = reinterpret_cast<uint32_t*>(tsm + tcp_sx_off(ns));
    uint32_t* sStg = reinterpret_cast<uint32_t*>(tsm + tcp_stage_off(L, ns));
    const uint32_t* xl = a.mode == 0 ? a.S.limbs(tri_idx(j, a.i, N), L) : a.X.limbs(j - a.i, L);
    for (int w = tid; w < tc_sx_words(L); w += kTcThreads) sX[w] = (w >= 8 && w < 8 + L) ? xl[w - 8] : 0u;
    constexpr int nacc = 2;
    if (warp == 0) tc::tmem_alloc_pair(&taddr_s, uint32_t(nacc * kTcN));
    if (tid == 0) {
        for (int s = 0; s < ns; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
            tc::mbar_init(&efull[s], 3);
            tc::mbar_init(&pready[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&accF[b], 1);
            tc::mbar_init(&accE[b], 8); // the leader's: 4 epilogue warps of each CTA
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::cluster_sync(); // both CTAs' barriers initialised before any remote arrive / multicast commit
    tc::fence_after();
    const uint32_t tmem = taddr_s;
    const int nch = tc_nchunks(L);
    auto nblk_of = [&](int c) { return tc_chunk_blocks(L, c); };
    // cell p of x -> X[p .. p+15] (sX holds X at byte 32; every window cell's words lie inside sX)
    auto cell = [&](int p) {
        const int off = 32 + p;
        const int w0 = off >> 2, sh = (off & 3) * 8;
        uint32_t W[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) W[q] = sX[w0 + q];
        return make_uint4(__funnelshift_r(W[0], W[1], sh), __funnelshift_r(W[1], W[2], sh),
                          __funnelshift_r(W[2], W[3], sh), __funnelshift_r(W[3], W[4], sh));
    };

    if (warp == 0) {
        if (ln == 0) {
            const uint32_t idesc = tc::idesc_u8(2 * kTcRows, kTcN, false, true);
            const uint8_t* Abase = a.A + (size_t)tile * tc_nblk(L) * kTcBlk;
            int Q = 0;
            for (int c = 0; c < nch; ++c) Q += nblk_of(c);
            int qt = 0, pc = 0, pb = 0, pcn = nblk_of(0);
            const bool prof = (a.dev & 64) && a.dev_cnt && rank == 0;
            unsigned long long w_empty = 0, w_full = 0, w_efull = 0, w_acc = 0, w_peer = 0, t_start = clock64();
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
            asm volatile("griddepcontrol.wait;" ::: "memory"); // A comes from the preceding k_tc_prep
            while (qt < Q && qt < ns - 1) issue_tma();
            int q = 0;
            for (int c = 0; c < nch; ++c) {
                const unsigned long long ta = prof ? clock64() : 0;
                const int ab = c % nacc;
                if (rank == 0 && c >= nacc) tc::mbar_wait(&accE[ab], uint32_t((c - nacc) / nacc) & 1u);
                if (prof) w_acc += clock64() - ta;
                tc::fence_after();
                const int tc0 = -31 + kTcN * c;
                const int u_hi = tc0 < 0 ? nb : nb - tc0;
                const int ksteps = (u_hi + kTcK - 1) / kTcK;
                const int nblk = nblk_of(c);
                for (int b = 0; b < nblk; ++b, ++q) {
                    const int s = q % ns;
                    const uint32_t ph = uint32_t(q / ns) & 1u;
                    const unsigned long long t1 = prof ? clock64() : 0;
                    tc::mbar_wait(&full[s], ph);
                    const unsigned long long t2 = prof ? clock64() : 0;
                    tc::mbar_wait(&efull[s], ph);
                    if (rank == 0) {
                        const unsigned long long t3 = prof ? clock64() : 0;
                        tc::mbar_wait(&pready[s], ph); // rank 1's A block and window half
                        if (prof) {
                            w_full += t2 - t1;
                            w_efull += t3 - t2;
                            w_peer += clock64() - t3;
                        }
                        tc::fence_after();
#pragma unroll
                        for (int sub = 0; sub < kTcKB; ++sub) {
                            const int ks = b * kTcKB + sub;
                            if (ks < ksteps) {
                                const uint64_t ad = tc::sdesc(sA + (size_t)s * kTcBlk + sub * 4096, 128, 256);
                                const uint64_t bd =
                                    tc::sdesc(sE + (size_t)s * kTcEWinPair * 16 + 16 * (size_t)(sub * kTcK), 128, 256);
                                tc::mma_i8_pair(tmem + uint32_t(ab * kTcN), ad, bd, idesc, ks > 0 ? 1u : 0u);
                            }
                        }
                        tc::commit_pair(&empty[s]); // both CTAs may refill slot s
                    } else {
                        tc::mbar_arrive_remote(&pready[s], 0);
                    }
                    if (qt < Q) issue_tma();
                }
                if (rank == 0) tc::commit_pair(&accF[ab]);
            }
            if (prof) {
                atomicAdd(a.dev_cnt + 0, w_empty);
                atomicAdd(a.dev_cnt + 1, w_full);
                atomicAdd(a.dev_cnt + 2, w_efull);
                atomicAdd(a.dev_cnt + 3, w_acc);
                atomicAdd(a.dev_cnt + 4, clock64() - t_start);
                atomicAdd(a.dev_cnt + 5, 1ull);
                atomicAdd(a.dev_cnt + 6, w_peer);
            }
        }
        __syncwarp();
    } else if (warp < 4) { // this CTA's window half of every block, in issue order
        const int bt = tid - 32;
        int q = 0;
        for (int c = 0; c < nch; ++c) {
            const int tc0 = -31 + kTcN * c, nblk = nblk_of(c);
            for (int b = 0; b < nblk; ++b, ++q) {
                const int s = q % ns;
                if (q >= ns) tc::mbar_wait_sleep(&empty[s], uint32_t((q / ns) - 1) & 1u, a.sleep_ns);
                uint8_t* dst = sE + (size_t)s * kTcEWinPair * 16;
                const int p0 = tc0 + kTcRows * int(rank) + b * kTcKB * kTcK;
                for (int cc = bt; cc < kTcEWinPair; cc += 96) *reinterpret_cast<uint4*>(dst + 16 * cc) = cell(p0 + cc);
                tc::fence_async_smem();
                __syncwarp();
                if (ln == 0) tc::mbar_arrive(&efull[s]);
            }
        }
    } else {
        fused_epilogue(a, tile, j, locj, sX, sStg, tmem, 0, nch, accF, accE, 0, nacc);
    }
    tc::fence_before();
    __syncthreads();
    tc::cluster_sync(); // no remote arrive or multicast commit may target an exited CTA
    tc::fence_after();
    if (warp == 0) tc::tmem_dealloc_pair(tmem, uint32_t(nacc * kTcN));
}
#endif

} // namespace hk
