// mpf_warp.cuh — warp-cooperative p-bit multiprecision float primitives.
//
// Replaces the reference's GMP-backed FixScalar arithmetic
// (/root/reference/proj/src/fixedpoint.cpp:55-154, above all submul_rounded at
// :146-154) with a fixed-length binary float:
//
//     value = sign * M * 2^(e - p),  p = 32 L,  2^(p-1) <= M < 2^p   (M in L u32 limbs)
//
// Every operation returns the correctly rounded (RNE) image of its exact
// result, so results are a pure function of the inputs: GPU == host model bit
// for bit, for any thread mapping, blocking, look-ahead order or GPU count
// (oracle/mpfloat.py is the executable specification).
//
// Building blocks, all executed by one warp in lockstep:
//   warp_mul       exact integer product by column sums: lane t accumulates
//                  sum_s A[s]*B[t-s] in 96 bits (mad.lo.cc/madc.hi.cc/addc,
//                  which ptxas fuses into one IMAD.WIDE.U32 with carry-out),
//                  then carries are resolved 32 limbs at a time with a
//                  ballot-based carry-lookahead.
//   warp_round_sum RNE(X + Y) of two scaled integers with arbitrary exponents:
//                  aligned into a window anchored at the larger operand (with
//                  a sticky limb for the truncated tail of the smaller one),
//                  exact add/sub with carry-lookahead, normalise, round.
//
// The same source compiles for sm_100a and, under HK_WARP_EMU, for the host
// with warp_emu.h (lockstep emulation) so the arithmetic is unit-tested on CPU.
#pragma once

#include <cstdint>

#if defined(HK_WARP_EMU)
#include "warp_emu.h"
#include <algorithm>
#include <cmath>
#define HK_DEV inline
#define HK_HD inline
namespace hk {
HK_DEV int lane() { return hk_emu::cur_lane(); }
HK_DEV uint32_t ballot(bool p) { return hk_emu::ballot(p); }
HK_DEV uint32_t shfl(uint32_t v, int src) { return hk_emu::shfl(v, src); }
HK_DEV uint32_t shfl_up(uint32_t v, int d) { return hk_emu::shfl_up(v, d); }
HK_DEV void wsync() { hk_emu::syncwarp(); }
HK_DEV int clz32(uint32_t x) { return x ? __builtin_clz(x) : 32; }
HK_DEV uint32_t fshr(uint32_t lo, uint32_t hi, int sh) {
    return uint32_t((((uint64_t)hi << 32) | lo) >> (sh & 31));
}
HK_DEV void mac96(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t x, uint32_t y) {
    const uint64_t p = (uint64_t)x * y;
    const uint64_t lo = (uint64_t)a0 + uint32_t(p);
    a0 = uint32_t(lo);
    const uint64_t mid = (uint64_t)a1 + uint32_t(p >> 32) + (lo >> 32);
    a1 = uint32_t(mid);
    a2 += uint32_t(mid >> 32);
}
using std::max;
using std::min;
} // namespace hk
#else
#define HK_DEV __device__ __forceinline__
#define HK_HD __host__ __device__ __forceinline__
namespace hk {
HK_DEV int lane() { return int(threadIdx.x & 31); }
HK_DEV uint32_t ballot(bool p) { return __ballot_sync(0xffffffffu, p); }
HK_DEV uint32_t shfl(uint32_t v, int src) { return __shfl_sync(0xffffffffu, v, src); }
HK_DEV uint32_t shfl_up(uint32_t v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
HK_DEV void wsync() { __syncwarp(); }
HK_DEV int clz32(uint32_t x) { return __clz(x); }
HK_DEV uint32_t fshr(uint32_t lo, uint32_t hi, int sh) { return __funnelshift_r(lo, hi, sh); }
HK_DEV void mac96(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t x, uint32_t y) {
    asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
        "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
        "addc.u32 %2, %2, 0;"
        : "+r"(a0), "+r"(a1), "+r"(a2)
        : "r"(x), "r"(y));
}
} // namespace hk
#endif

namespace hk {

// A scaled integer operand: value = sign * INT(d[0..n)) * 2^lsb.
struct Opd {
    const uint32_t* d;
    int n;
    int lsb;
    int sign; // -1, 0, +1 (0 => value zero, d ignored)
};

// bits [b, b+32) of |X| where b is an absolute bit position.
HK_DEV uint32_t opd_word(const Opd& X, int b) {
    const int r = b - X.lsb;
    if (r >= 32 * X.n || r <= -32) return 0;
    const int q = r >> 5; // floor division (arithmetic shift)
    const int sh = r & 31;
    const uint32_t lo = (q >= 0 && q < X.n) ? X.d[q] : 0u;
    const uint32_t hi = (q + 1 >= 0 && q + 1 < X.n) ? X.d[q + 1] : 0u;
    return fshr(lo, hi, sh);
}

// Carry-lookahead over one 32-limb segment (one limb per lane).  `w` is the
// lane's limb after its local add, `g` whether that add overflowed; `cin` is
// the (warp-uniform) carry into lane 0.  Returns the carry out of lane 31.
HK_DEV uint32_t seg_carry(uint32_t& w, bool g, uint32_t cin) {
    const uint32_t G = ballot(g);
    const uint32_t P = ballot(w == 0xffffffffu);
    const uint32_t X = G | P;
    const uint64_t S = (uint64_t)G + X + cin;
    const uint32_t C = uint32_t(S) ^ G ^ X; // carry into each lane
    w += (C >> lane()) & 1u;
    return uint32_t(S >> 32);
}

// Same for a borrow chain: `w` = a - b (mod 2^32), `bor` = (a < b).
HK_DEV uint32_t seg_borrow(uint32_t& w, bool bor, uint32_t bin) {
    const uint32_t G = ballot(bor);
    const uint32_t P = ballot(w == 0u);
    const uint32_t X = G | P;
    const uint64_t S = (uint64_t)G + X + bin;
    const uint32_t C = uint32_t(S) ^ G ^ X;
    w -= (C >> lane()) & 1u;
    return uint32_t(S >> 32);
}

// Bit length of the integer d[0..n) (0 for zero).  Warp-uniform result.
HK_DEV int warp_bitlen(const uint32_t* d, int n) {
    for (int base = ((n - 1) >> 5) << 5; base >= 0; base -= 32) {
        const int idx = base + lane();
        const uint32_t v = idx < n ? d[idx] : 0u;
        const uint32_t m = ballot(v != 0u);
        if (m) {
            const int hl = 31 - clz32(m);
            const uint32_t top = shfl(v, hl);
            return (base + hl) * 32 + (32 - clz32(top));
        }
    }
    return 0;
}

// Is any bit of d[0..n) below relative bit position `rel` set?  Warp-uniform.
HK_DEV bool warp_any_below(const uint32_t* d, int n, int rel) {
    if (rel <= 0) return false;
    const int full = rel >> 5, part = rel & 31;
    const int lim = min(n, full + (part ? 1 : 0));
    bool any = false;
    for (int base = 0; base < lim; base += 32) {
        const int idx = base + lane();
        uint32_t v = idx < lim ? d[idx] : 0u;
        if (idx == full) v &= (part ? ((1u << part) - 1u) : 0u);
        any |= ballot(v != 0u) != 0u;
    }
    return any;
}

// Stage `n` limbs from `src` into `dst` (lane-strided copy).
HK_DEV void warp_copy(uint32_t* dst, const uint32_t* src, int n) {
    for (int i = lane(); i < n; i += 32) dst[i] = src[i];
}

// Stage B into the zero-padded layout warp_mul expects: Bp[32 + u] = B[u],
// 32 zero limbs on each side.  Bp needs n + 64 limbs.
HK_DEV void warp_stage_padded(uint32_t* Bp, const uint32_t* B, int n) {
    for (int i = lane(); i < n + 64; i += 32) Bp[i] = (i >= 32 && i < 32 + n) ? B[i - 32] : 0u;
}

// P[0 .. nA+nB) = A[0..nA) * B[0..nB) (exact).  A: plain limbs (smem), Bp: the
// padded staging of B (smem).  Column sums in 96 bits per lane, carries
// resolved per 32-limb group with a running carry / high-word state.
HK_DEV void warp_mul(const uint32_t* A, int nA, const uint32_t* Bp, int nB, uint32_t* P) {
    const int ln = lane();
    const int ntot = nA + nB;
    uint32_t cin = 0, hi_prev = 0, a1p = 0, a2p31 = 0, a2p30 = 0;
    for (int g0 = 0; g0 < ntot; g0 += 32) {
        const int t = g0 + ln;
        const int slo = max(0, g0 - (nB - 1));
        const int shi = min(g0 + 31, nA - 1);
        uint32_t a0 = 0, a1 = 0, a2 = 0;
        const uint32_t* yb = Bp + 32 + t;
#pragma unroll 4
        for (int s = slo; s <= shi; ++s) mac96(a0, a1, a2, A[s], yb[-s]);
        // limb t receives a0(t) + a1(t-1) + a2(t-2)
        uint32_t a1m1 = shfl_up(a1, 1);
        uint32_t a2m2 = shfl_up(a2, 2);
        if (ln == 0) {
            a1m1 = a1p;
            a2m2 = a2p30;
        } else if (ln == 1) {
            a2m2 = a2p31;
        }
        const uint64_t s64 = (uint64_t)a0 + a1m1 + a2m2;
        const uint32_t lo = uint32_t(s64), hi = uint32_t(s64 >> 32);
        uint32_t him1 = shfl_up(hi, 1);
        if (ln == 0) him1 = hi_prev;
        uint32_t w = lo + him1;
        const bool gen = w < lo;
        cin = seg_carry(w, gen, cin);
        if (t < ntot) P[t] = w;
        a1p = shfl(a1, 31);
        a2p31 = shfl(a2, 31);
        a2p30 = shfl(a2, 30);
        hi_prev = shfl(hi, 31);
    }
}

// Result metadata of a rounded operation.
struct RMeta {
    int exp;  // value = sign * M * 2^(exp - 32*nout)
    int sign; // -1, 0, +1
};

// out[0..nout) = RNE_{32 nout}(X + Y).  G is a smem scratch window of at least
// max(X.n, Y.n, nout) + 4 limbs that must not alias X, Y or out.  X or Y may
// alias `out` (all operand reads finish before the first write).
HK_DEV RMeta warp_round_sum(const Opd& Xin, const Opd& Yin, uint32_t* G, uint32_t* out, int nout) {
    const int ln = lane();
    const int blX = Xin.sign ? warp_bitlen(Xin.d, Xin.n) : 0;
    const int blY = Yin.sign ? warp_bitlen(Yin.d, Yin.n) : 0;
    if (blX == 0 && blY == 0) {
        for (int i = ln; i < nout; i += 32) out[i] = 0u;
        wsync();
        return RMeta{0, 0};
    }
    const int TX = Xin.lsb + blX, TY = Yin.lsb + blY;
    const bool xbig = blY == 0 || (blX != 0 && TX >= TY);
    const Opd Big = xbig ? Xin : Yin;
    const Opd Small = xbig ? Yin : Xin;
    const int blS = xbig ? blY : blX;
    const int Tbig = xbig ? TX : TY;
    const int W = max(max(Big.n, Small.n), nout) + 3; // window limbs 1..W, limb 0 = sticky
    const int base = Tbig - 32 * (W - 1);             // absolute bit of window limb 1, bit 0
    const bool small_live = blS != 0;
    const bool sticky = small_live && warp_any_below(Small.d, Small.n, base - Small.lsb);
    const bool eff_sub = small_live && (Big.sign != Small.sign);

    // G = |Big| +- |Small| over limbs 0..W (limb 0 holds the sticky unit of Small)
    uint32_t c = 0;
    for (int b0 = 0; b0 <= W; b0 += 32) {
        const int w = b0 + ln;
        uint32_t vb = 0, vs = 0;
        if (w >= 1 && w <= W) {
            const int bit = base + 32 * (w - 1);
            vb = opd_word(Big, bit);
            vs = small_live ? opd_word(Small, bit) : 0u;
        } else if (w == 0) {
            vs = sticky ? 1u : 0u;
        }
        uint32_t r;
        if (eff_sub) {
            r = vb - vs;
            c = seg_borrow(r, vb < vs, c);
        } else {
            r = vb + vs;
            c = seg_carry(r, r < vb, c);
        }
        if (w <= W) G[w] = r;
    }
    int sign = Big.sign;
    if (eff_sub && c) { // negative: two's-complement negate
        wsync();
        uint32_t cc = 1;
        for (int b0 = 0; b0 <= W; b0 += 32) {
            const int w = b0 + ln;
            uint32_t r = w <= W ? ~G[w] : 0u;
            cc = seg_carry(r, false, cc);
            if (w <= W) G[w] = r;
        }
        sign = -sign;
    }
    wsync();
    const int bl = warp_bitlen(G, W + 1);
    if (bl == 0) {
        for (int i = ln; i < nout; i += 32) out[i] = 0u;
        wsync();
        return RMeta{0, 0};
    }
    int tb = bl - 1;                 // top bit index in G
    const int lsbpos = tb - 32 * nout + 1;
    const Opd Gw{G, W + 1, 0, 1};
    bool rb = false, st = false;
    if (lsbpos - 1 >= 0) {
        rb = (G[(lsbpos - 1) >> 5] >> ((lsbpos - 1) & 31)) & 1u;
        st = warp_any_below(G, W + 1, lsbpos - 1);
    }
    const uint32_t low0 = opd_word(Gw, lsbpos);
    const bool inc = rb && (st || (low0 & 1u));
    wsync(); // every read of X / Y / G done before `out` (which may alias X or Y) is written
    // Lanes at index >= nout hold 0, so a carry out of limb nout-1 lands (and
    // stops) on lane index nout; the loop runs far enough to include it.
    uint32_t cc = inc ? 1u : 0u;
    bool ovf = false;
    for (int b0 = 0; b0 <= nout; b0 += 32) {
        const int j = b0 + ln;
        uint32_t r = j < nout ? opd_word(Gw, lsbpos + 32 * j) : 0u;
        cc = seg_carry(r, false, cc);
        if (j < nout) out[j] = r;
        ovf |= ballot(j == nout && r != 0u) != 0u;
    }
    if (ovf) { // mantissa overflowed to 2^(32 nout): renormalise
        wsync();
        for (int i = ln; i < nout; i += 32) out[i] = (i == nout - 1) ? 0x80000000u : 0u;
        ++tb;
    }
    wsync();
    return RMeta{(base - 32) + tb + 1, sign};
}

} // namespace hk
