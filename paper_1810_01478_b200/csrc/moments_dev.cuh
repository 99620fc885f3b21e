// moments_dev.cuh — the exact moments on the device.
//
// mu_k = (1/beta) Gamma((k+1)/beta) = (q/2) ((k+1) q/2 - 1)!  for even q = 2/beta
// (the reference's gamma_exact factorial branch + moment, moments.cpp:83-89,
// 102-111; mpz_fac_ui there).  One CTA keeps the running factorial F as an exact
// integer in shared memory (W 32-bit limbs, thread t owns `per` consecutive
// limbs), multiplies it by the next factors (two at a time while their product
// fits a word), and after each moment's last factor writes RNE_p((q/2) F)
// straight into the context's moment array: a word-shifted copy of the top p
// bits plus one rounding increment (build_hankel's exact integer -> working
// precision conversion, moments.cpp:113-129).  No host bigint, no H2D.
//
// A multiplication by a 32-bit factor is three block phases: (1) every thread
// multiplies its segment (32-bit carry chain inside the segment, carry-out to a
// shared array); (2) it adds its lower neighbour's carry-out and reports whether
// its segment generates a carry or would propagate one; (3) the one-bit carries
// are resolved with the adder identity  carries = (A + B + cin) ^ P,  A = G | P,
// B = G  over ballots (warp level, then across the warps) and rippled in.
#pragma once

#include "mpf_ops.cuh"

namespace hk {

constexpr int kMomMaxThreads = 1024;

struct MomentsArgs {
    uint32_t* out;   // [count][L] mantissa limbs
    Meta* meta;      // [count]
    int count, L;
    unsigned q;      // 2 / beta (even)
    int per;         // limbs per thread (odd: conflict-free segment stride)
    int* inexact;    // set to 1 if any moment needed rounding
};

#if !defined(HK_WARP_EMU)

// G = F * m (G may alias F); both W = per * blockDim.x limbs.  ub: an upper
// bound of F's top nonzero limb (threads above it have nothing to multiply).
__device__ __forceinline__ void cta_mul_small(const uint32_t* F, uint32_t* G, int per, int ub, uint32_t m,
                                              uint32_t* sc, uint32_t* sw) {
    const int t = threadIdx.x, ln = t & 31, wp = t >> 5, nw = blockDim.x >> 5;
    const int base = t * per;
    uint32_t carry = 0;
    if (base <= ub + 1) {
        for (int i = 0; i < per; ++i) {
            const uint64_t pr = (uint64_t)F[base + i] * m + carry;
            G[base + i] = uint32_t(pr);
            carry = uint32_t(pr >> 32);
        }
    } else if (G != F) {
        for (int i = 0; i < per; ++i) G[base + i] = 0u;
    }
    sc[t] = carry;
    __syncthreads();
    // (2) neighbour's carry-out into this segment
    bool gen = false, prop = false;
    if (base <= ub + 2) {
        uint32_t cin = t > 0 ? sc[t - 1] : 0u;
        bool ones = true;
        for (int i = 0; i < per; ++i) {
            const uint32_t v = G[base + i];
            const uint32_t s = v + cin;
            cin = s < v ? 1u : 0u;
            if (s != v) G[base + i] = s;
            ones = ones && s == 0xffffffffu;
        }
        gen = cin != 0u;
        prop = ones;
    }
    const uint32_t gb = __ballot_sync(0xffffffffu, gen), pb = __ballot_sync(0xffffffffu, prop);
    const uint64_t A = uint64_t(gb | pb), B = uint64_t(gb);
    if (ln == 0) {
        const uint32_t g_w = uint32_t((A + B) >> 32) & 1u;
        const uint32_t p_w = (uint32_t((A + B + 1) >> 32) & 1u) & ~g_w;
        sw[wp] = g_w | (p_w << 1);
    }
    __syncthreads();
    // (3) carries into the warps, then into the lanes
    uint32_t cw = 0;
    {
        const uint32_t v = ln < nw ? sw[ln] : 0u;
        const uint32_t gw = __ballot_sync(0xffffffffu, v & 1u), pw = __ballot_sync(0xffffffffu, v & 2u);
        const uint64_t Aw = uint64_t(gw | pw), Bw = uint64_t(gw);
        const uint32_t cvec = uint32_t((Aw + Bw) ^ uint64_t(pw)); // bit w: carry into warp w
        cw = (cvec >> wp) & 1u;
    }
    const uint32_t cl = uint32_t(((A + B + cw) ^ uint64_t(pb)) >> ln) & 1u;
    if (cl) {
        for (int i = 0; i < per; ++i) {
            const uint32_t s = G[base + i] + 1u;
            G[base + i] = s;
            if (s != 0u) break;
        }
    }
    __syncthreads(); // G complete; sc / sw free for the next multiplication
}

__global__ void __launch_bounds__(kMomMaxThreads, 1) k_moments_fact(MomentsArgs a) {
    extern __shared__ __align__(16) uint32_t msm[];
    const int T = blockDim.x, t = threadIdx.x;
    const int W = a.per * T;
    uint32_t* F = msm;
    const unsigned half = a.q / 2;
    uint32_t* G = half == 1 ? F : msm + W; // (q/2) F
    const int nbuf = half == 1 ? 1 : 2;
    uint32_t* sc = msm + nbuf * W;
    uint32_t* sw = sc + T;
    for (int i = t; i < nbuf * W; i += T) msm[i] = 0u;
    __syncthreads();
    if (t == 0) F[0] = 1u;
    __syncthreads();
    int ub = 0;               // upper bound of F's top limb
    unsigned long have = 0;   // F == have!
    const int p = 32 * a.L;
    for (int k = 0; k < a.count; ++k) {
        const unsigned long arg = (unsigned long)(k + 1) * half - 1;
        while (have < arg) {
            uint32_t m;
            if (have + 2 <= arg && have + 2 < 65536) {
                m = uint32_t((have + 1) * (have + 2));
                have += 2;
            } else {
                m = uint32_t(++have);
            }
            cta_mul_small(F, F, a.per, ub, m, sc, sw);
            ub = ub + 1 < W - 1 ? ub + 1 : W - 1;
        }
        int ubg = ub;
        if (half != 1) {
            cta_mul_small(F, G, a.per, ub, uint32_t(half), sc, sw);
            ubg = ub + 1 < W - 1 ? ub + 1 : W - 1;
        }
        // top limb of G (every thread scans the same few limbs), tighten ub
        int top = ubg;
        while (top > 0 && G[top] == 0u) --top;
        ub = top;
        const int nb = 32 * top + 32 - __clz(G[top]);
        const int shift = nb - p; // out = G >> shift (negative: left shift)
        uint32_t* o = a.out + (size_t)k * a.L;
        for (int w = t; w < a.L; w += T) {
            const int b = shift + 32 * w;
            const int qd = b >> 5, r = b & 31; // floor division for negative b
            const uint32_t lo = (qd >= 0 && qd < W) ? G[qd] : 0u;
            const uint32_t hi = (qd + 1 >= 0 && qd + 1 < W) ? G[qd + 1] : 0u;
            o[w] = r ? (lo >> r) | (hi << (32 - r)) : lo;
        }
        int e = nb;
        if (shift > 0) { // RNE on the dropped bits [0, shift)
            const int rbit = shift - 1;
            const bool rb = (G[rbit >> 5] >> (rbit & 31)) & 1u;
            int st = 0;
            const int qs = rbit >> 5;
            for (int i = t; i < qs; i += T) st |= G[i] != 0u;
            if (t == 0 && (rbit & 31)) st |= (G[qs] & ((1u << (rbit & 31)) - 1u)) != 0u;
            st = __syncthreads_or(st); // also orders the stores of o
            if (t == 0) {
                if (rb || st) *a.inexact = 1;
                if (rb && (st || (o[0] & 1u))) {
                    int i = 0;
                    while (i < a.L && ++o[i] == 0u) ++i;
                    if (i == a.L) { // all ones rounded up to 2^p
                        o[a.L - 1] = 0x80000000u;
                        e = nb + 1;
                    }
                }
            }
        }
        if (t == 0) a.meta[k] = Meta{e, 1};
        __syncthreads(); // G read; the next multiplication may overwrite it
    }
}

#endif

} // namespace hk
