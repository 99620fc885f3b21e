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

#ifndef HK_TRACE
#define HK_TRACE(tag) // dev probes (tools/recip_probe.cu) record timestamps here
#endif

#include <cstdint>

#if defined(HK_WARP_EMU)
#include "warp_emu.h"
#include <algorithm>
#include <cmath>
#define HK_DEV inline
#define HK_HD inline
struct uint4 {
    uint32_t x, y, z, w;
};
inline uint4 make_uint4(uint32_t x, uint32_t y, uint32_t z, uint32_t w) { return uint4{x, y, z, w}; }
namespace hk {
HK_DEV int lane() { return hk_emu::cur_lane(); }
HK_DEV uint32_t ballot(bool p) { return hk_emu::ballot(p); }
HK_DEV uint32_t shfl(uint32_t v, int src) { return hk_emu::shfl(v, src); }
HK_DEV uint32_t shfl_up(uint32_t v, int d) { return hk_emu::shfl_up(v, d); }
HK_DEV uint32_t shfl_down(uint32_t v, int d) { return hk_emu::shfl_down(v, d); }
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
HK_DEV void add96(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t b0, uint32_t b1, uint32_t b2) {
    const uint64_t lo = (uint64_t)a0 + b0;
    a0 = uint32_t(lo);
    const uint64_t mid = (uint64_t)a1 + b1 + (lo >> 32);
    a1 = uint32_t(mid);
    a2 += b2 + uint32_t(mid >> 32);
}
HK_DEV void mac64(uint64_t& acc, uint32_t& hi, uint32_t x, uint32_t y) {
    const uint64_t p = (uint64_t)x * y;
    acc += p;
    hi += acc < p;
}
HK_DEV void mac64x2(uint64_t& acc, uint32_t& hi, uint32_t x0, uint32_t y0, uint32_t x1, uint32_t y1) {
    mac64(acc, hi, x0, y0);
    mac64(acc, hi, x1, y1);
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
HK_DEV uint32_t shfl_down(uint32_t v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
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
HK_DEV void add96(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t b0, uint32_t b1, uint32_t b2) {
    asm("add.cc.u32 %0, %0, %3;\n\t"
        "addc.cc.u32 %1, %1, %4;\n\t"
        "addc.u32 %2, %2, %5;"
        : "+r"(a0), "+r"(a1), "+r"(a2)
        : "r"(b0), "r"(b1), "r"(b2));
}
// 96-bit accumulate with the low 64 bits as ONE 64-bit operand: ptxas keeps the
// accumulator in a register pair and emits IMAD.WIDE.U32 with carry-out, no moves.
HK_DEV void mac64(uint64_t& acc, uint32_t& hi, uint32_t x, uint32_t y) {
    asm("{\n\t.reg .u32 lo, h;\n\tmov.b64 {lo, h}, %0;\n\t"
        "mad.lo.cc.u32 lo, %2, %3, lo;\n\tmadc.hi.cc.u32 h, %2, %3, h;\n\taddc.u32 %1, %1, 0;\n\t"
        "mov.b64 %0, {lo, h};\n\t}"
        : "+l"(acc), "+r"(hi)
        : "r"(x), "r"(y));
}
// Two MACs into one accumulator: the two carry-outs merge into a single
// ALU-pipe IADD3.X, leaving the IMAD pipe to the IMAD.WIDEs.
HK_DEV void mac64x2(uint64_t& acc, uint32_t& hi, uint32_t x0, uint32_t y0, uint32_t x1, uint32_t y1) {
    asm("{\n\t.reg .u32 lo, h;\n\tmov.b64 {lo, h}, %0;\n\t"
        "mad.lo.cc.u32 lo, %2, %3, lo;\n\tmadc.hi.cc.u32 h, %2, %3, h;\n\taddc.u32 %1, %1, 0;\n\t"
        "mad.lo.cc.u32 lo, %4, %5, lo;\n\tmadc.hi.cc.u32 h, %4, %5, h;\n\taddc.u32 %1, %1, 0;\n\t"
        "mov.b64 %0, {lo, h};\n\t}"
        : "+l"(acc), "+r"(hi)
        : "r"(x0), "r"(y0), "r"(x1), "r"(y1));
}
} // namespace hk
#endif

namespace hk {

// A scaled integer operand: value = sign * INT(d[0..n)) * 2^lsb.
struct Opd {
    const uint32_t* d;
    int n;
    int lsb;
    int sign;    // -1, 0, +1 (0 => value zero, d ignored)
    int bl = 0;  // bit length of INT(d) when known (normalised mantissa: 32 n), else 0
};

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

// Stage `n` limbs from `src` into `dst` (lane-strided copy).
HK_DEV void warp_copy(uint32_t* dst, const uint32_t* src, int n) {
    for (int i = lane(); i < n; i += 32) dst[i] = src[i];
}

// Stage B into the zero-padded layout warp_mul expects: Bp[32 + u] = B[u],
// 32 zero limbs on each side.  Bp needs n + 64 limbs.
HK_DEV void warp_stage_padded(uint32_t* Bp, const uint32_t* B, int n) {
    for (int i = lane(); i < n + 64; i += 32) Bp[i] = (i >= 32 && i < 32 + n) ? B[i - 32] : 0u;
}

// P[tfirst .. nA+nB) = the limbs of sum_{t >= tfirst} colsum_t 2^(32 t), where
// colsum_t = sum_s A[s] B[t-s].  With tfirst = 0 this is the exact product
// A[0..nA) * B[0..nB); with tfirst > 0 it is the "short" product that drops the
// low columns and their carries (the dropped part E satisfies
// 0 <= E < min(nA,nB) 2^(32 tfirst + 32), see warp_fms).  A: plain limbs (smem),
// Bp: the padded staging of B (smem).  Column sums in 96 bits per lane, carries
// resolved per 32-limb group with a running carry / high-word state.
// 96-bit column sum of column t = g0 + lane: sum_s A[s] B[t-s] over the
// group's union s-range.  Four independent accumulator chains break the carry
// dependency (a lone warp is latency-bound otherwise).  Per 8 MACs: 2
// warp-uniform LDS.128 for x (broadcast), 8 LDS for y, 8 IMAD.WIDE.U32 + 4
// IADD3.X (SASS checked).  The prologue aligns s so the x loads are 16-byte
// vectors (A must be 16-byte aligned).
HK_DEV void colsum_group(const uint32_t* A, int nA, const uint32_t* Bp, int nB, int g0, uint32_t& a0, uint32_t& a1,
                         uint32_t& a2) {
    const int t = g0 + lane();
    const int slo = max(0, g0 - (nB - 1));
    const int shi = min(g0 + 31, nA - 1);
    uint64_t q0 = 0, q1 = 0, q2 = 0, q3 = 0;
    uint32_t h0 = 0, h1 = 0, h2 = 0, h3 = 0;
    const uint32_t* yb = Bp + 32 + t;
    int s = slo;
    for (; s <= shi && (s & 3); ++s) mac64(q0, h0, A[s], yb[-s]);
    for (; s + 7 <= shi; s += 8) {
        const uint4 xa = *reinterpret_cast<const uint4*>(A + s);
        const uint4 xb = *reinterpret_cast<const uint4*>(A + s + 4);
        mac64x2(q0, h0, xa.x, yb[-s], xb.x, yb[-s - 4]);
        mac64x2(q1, h1, xa.y, yb[-s - 1], xb.y, yb[-s - 5]);
        mac64x2(q2, h2, xa.z, yb[-s - 2], xb.z, yb[-s - 6]);
        mac64x2(q3, h3, xa.w, yb[-s - 3], xb.w, yb[-s - 7]);
    }
    for (; s <= shi; ++s) mac64(q0, h0, A[s], yb[-s]);
    a0 = uint32_t(q0);
    a1 = uint32_t(q0 >> 32);
    a2 = h0;
    add96(a0, a1, a2, uint32_t(q1), uint32_t(q1 >> 32), h1);
    add96(a0, a1, a2, uint32_t(q2), uint32_t(q2 >> 32), h2);
    add96(a0, a1, a2, uint32_t(q3), uint32_t(q3 >> 32), h3);
}

// Two column sums sharing the y operand: columns t = g0 + lane of A0*B and
// A1*B.  Each per-lane y load feeds two MACs (the bulk LDLT update pairs the
// entries (k, j) and (k, j+1), which share y = B_i(k)).
HK_DEV void colsum_group2(const uint32_t* A0, const uint32_t* A1, int nA, const uint32_t* Bp, int nB, int g0,
                          uint32_t (&r0)[3], uint32_t (&r1)[3]) {
    const int t = g0 + lane();
    const int slo = max(0, g0 - (nB - 1));
    const int shi = min(g0 + 31, nA - 1);
    uint64_t p0 = 0, p1 = 0, q0 = 0, q1 = 0;
    uint32_t hp0 = 0, hp1 = 0, hq0 = 0, hq1 = 0;
    const uint32_t* yb = Bp + 32 + t;
    int s = slo;
    for (; s <= shi && (s & 3); ++s) {
        const uint32_t y = yb[-s];
        mac64(p0, hp0, A0[s], y);
        mac64(q0, hq0, A1[s], y);
    }
    for (; s + 3 <= shi; s += 4) {
        const uint4 xa = *reinterpret_cast<const uint4*>(A0 + s);
        const uint4 xb = *reinterpret_cast<const uint4*>(A1 + s);
        const uint32_t y0 = yb[-s], y1 = yb[-s - 1], y2 = yb[-s - 2], y3 = yb[-s - 3];
        mac64x2(p0, hp0, xa.x, y0, xa.z, y2);
        mac64x2(p1, hp1, xa.y, y1, xa.w, y3);
        mac64x2(q0, hq0, xb.x, y0, xb.z, y2);
        mac64x2(q1, hq1, xb.y, y1, xb.w, y3);
    }
    for (; s <= shi; ++s) {
        const uint32_t y = yb[-s];
        mac64(p0, hp0, A0[s], y);
        mac64(q0, hq0, A1[s], y);
    }
    r0[0] = uint32_t(p0);
    r0[1] = uint32_t(p0 >> 32);
    r0[2] = hp0;
    add96(r0[0], r0[1], r0[2], uint32_t(p1), uint32_t(p1 >> 32), hp1);
    r1[0] = uint32_t(q0);
    r1[1] = uint32_t(q0 >> 32);
    r1[2] = hq0;
    add96(r1[0], r1[1], r1[2], uint32_t(q1), uint32_t(q1 >> 32), hq1);
}

// Running state of the column-sum -> limb carry resolution (warp-uniform).
struct CarryState {
    uint32_t cin = 0, hi_prev = 0, a1p = 0, a2p31 = 0, a2p30 = 0;
};

// Limb t = g0 + lane of the product from the group's column sums: limb t
// receives a0(t) + a1(t-1) + a2(t-2) + carries, resolved with the lookahead.
HK_DEV uint32_t carry_group(CarryState& cs, uint32_t a0, uint32_t a1, uint32_t a2) {
    const int ln = lane();
    uint32_t a1m1 = shfl_up(a1, 1);
    uint32_t a2m2 = shfl_up(a2, 2);
    if (ln == 0) {
        a1m1 = cs.a1p;
        a2m2 = cs.a2p30;
    } else if (ln == 1) {
        a2m2 = cs.a2p31;
    }
    const uint64_t s64 = (uint64_t)a0 + a1m1 + a2m2;
    const uint32_t lo = uint32_t(s64), hi = uint32_t(s64 >> 32);
    uint32_t him1 = shfl_up(hi, 1);
    if (ln == 0) him1 = cs.hi_prev;
    uint32_t w = lo + him1;
    const bool gen = w < lo;
    cs.cin = seg_carry(w, gen, cs.cin);
    cs.a1p = shfl(a1, 31);
    cs.a2p31 = shfl(a2, 31);
    cs.a2p30 = shfl(a2, 30);
    cs.hi_prev = shfl(hi, 31);
    return w;
}

HK_DEV void warp_mul(const uint32_t* A, int nA, const uint32_t* Bp, int nB, uint32_t* P, int tfirst = 0) {
    const int ntot = nA + nB;
    CarryState cs;
    for (int g0 = tfirst; g0 < ntot; g0 += 32) {
        uint32_t a0, a1, a2;
        colsum_group(A, nA, Bp, nB, g0, a0, a1, a2);
        const uint32_t w = carry_group(cs, a0, a1, a2);
        const int t = g0 + lane();
        if (t < ntot) P[t] = w;
    }
}

// P0 = A0*B, P1 = A1*B (from column tfirst), sharing the staged B.
HK_DEV void warp_mul2(const uint32_t* A0, const uint32_t* A1, int nA, const uint32_t* Bp, int nB, uint32_t* P0,
                      uint32_t* P1, int tfirst) {
    const int ntot = nA + nB;
    CarryState c0, c1;
    for (int g0 = tfirst; g0 < ntot; g0 += 32) {
        uint32_t r0[3], r1[3];
        colsum_group2(A0, A1, nA, Bp, nB, g0, r0, r1);
        const uint32_t w0 = carry_group(c0, r0[0], r0[1], r0[2]);
        const uint32_t w1 = carry_group(c1, r1[0], r1[1], r1[2]);
        const int t = g0 + lane();
        if (t < ntot) {
            P0[t] = w0;
            P1[t] = w1;
        }
    }
}

// ---- CTA cooperation for latency-bound single ops (the LDLT's critical path:
// reciprocal, B column, look-ahead column).  On the host emulator a "CTA" is
// one warp, so the same code is exercised with num_warps() == 1.
#if defined(HK_WARP_EMU)
HK_DEV int warp_id() { return 0; }
HK_DEV int num_warps() { return 1; }
HK_DEV void cta_sync() { wsync(); }
HK_DEV int cta_tid() { return lane(); }
HK_DEV int cta_threads() { return 32; }
#else
HK_DEV int warp_id() { return int(threadIdx.x >> 5); }
HK_DEV int num_warps() { return int(blockDim.x >> 5); }
HK_DEV void cta_sync() { __syncthreads(); }
HK_DEV int cta_tid() { return int(threadIdx.x); }
HK_DEV int cta_threads() { return int(blockDim.x); }
#endif

HK_HD int cta_cs_words(int ntot) { return 96 * ((ntot + 31) / 32); }

// Product (from column tfirst) by all warps of the CTA: warps take 32-column
// groups round-robin and park the 96-bit sums in CS, then warp 0 resolves the
// carries group by group (cheap: one lookahead per group).  A, Bp staged.
HK_DEV void cta_mul(const uint32_t* A, int nA, const uint32_t* Bp, int nB, uint32_t* P, int tfirst, uint32_t* CS) {
    const int ntot = nA + nB, ng = (ntot - tfirst + 31) / 32;
    const int w = warp_id(), nw = num_warps();
    HK_TRACE(5);
    for (int g = w; g < ng; g += nw) {
        uint32_t a0, a1, a2;
        colsum_group(A, nA, Bp, nB, tfirst + 32 * g, a0, a1, a2);
        uint32_t* c = CS + 96 * g + lane();
        c[0] = a0;
        c[32] = a1;
        c[64] = a2;
    }
    cta_sync();
    HK_TRACE(6);
    if (w == 0) {
        CarryState cs;
        for (int g = 0; g < ng; ++g) {
            const uint32_t* c = CS + 96 * g + lane();
            const uint32_t v = carry_group(cs, c[0], c[32], c[64]);
            const int t = tfirst + 32 * g + lane();
            if (t < ntot) P[t] = v;
        }
    }
    cta_sync();
}

// CTA-strided copies (all threads)
HK_DEV void cta_copy(uint32_t* dst, const uint32_t* src, int n) {
    for (int i = cta_tid(); i < n; i += cta_threads()) dst[i] = src[i];
}
HK_DEV void cta_stage_padded(uint32_t* Bp, const uint32_t* B, int n) {
    for (int i = cta_tid(); i < n + 64; i += cta_threads()) Bp[i] = (i >= 32 && i < 32 + n) ? B[i - 32] : 0u;
}

// Result metadata of a rounded operation.
struct RMeta {
    int exp;  // value = sign * M * 2^(exp - 32*nout)
    int sign; // -1, 0, +1
};

constexpr int kExact = -0x40000000; // "no uncertainty" for warp_round_sum's ubit

// ---- correctly rounded sum, four window limbs per lane (128 per warp
// iteration): each pass pays its ballot lookahead, branches and address
// arithmetic once per 128 limbs, and the carry inside a lane's four limbs is a
// plain add chain.

// The lane's four words w0..w0+3 of bits [off + 32 w, off + 32 w + 32) of INT(d[0..n)).
HK_DEV void read4(const uint32_t* d, int n, int off, int w0, uint32_t (&v)[4]) {
    const int q = (off >> 5) + w0, sh = off & 31;
    uint32_t x[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int idx = q + t;
        x[t] = (idx >= 0 && idx < n) ? d[idx] : 0u;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = fshr(x[t], x[t + 1], sh);
}

// read4 split in two: the five raw words (issued one iteration ahead by the
// streaming passes, so global-memory operands are prefetched) and the shift.
// b0: the warp's first window word this iteration (w0 = b0 + 4 lane): when the
// whole warp's range is inside [0, n) the loads go unchecked (the interior
// iterations; the bounds tests were the rounding pass's largest ALU cost).
HK_DEV void load5(const uint32_t* d, int n, int off, int b0, int w0, uint32_t (&x)[5]) {
    const int q = (off >> 5) + w0;
    const int lo = (off >> 5) + b0;
    if (lo >= 0 && lo + 128 < n) {
#pragma unroll
        for (int t = 0; t < 5; ++t) x[t] = d[q + t];
        return;
    }
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int idx = q + t;
        x[t] = (idx >= 0 && idx < n) ? d[idx] : 0u;
    }
}
HK_DEV bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
HK_DEV void shift4(const uint32_t (&x)[5], int off, uint32_t (&v)[4]) {
    const int sh = off & 31;
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = fshr(x[t], x[t + 1], sh);
}

// Carry-lookahead over lanes holding 4-limb groups: g = carry (or borrow) out
// of the lane's own chain, p = a carry (borrow) into the lane would pass through
// all four limbs.  Returns the carry into this lane; cio: carry into lane 0 in,
// carry out of lane 31 out.
HK_DEV uint32_t lane_carry_in(bool g, bool p, uint32_t& cio) {
    const uint32_t G = ballot(g), P = ballot(p);
    const uint32_t X = G | P;
    const uint64_t S = (uint64_t)G + X + cio;
    const uint32_t C = uint32_t(S) ^ G ^ X;
    cio = uint32_t(S >> 32);
    return (C >> lane()) & 1u;
}

HK_DEV void ripple_add4(uint32_t (&r)[4], uint32_t c) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const uint64_t s = (uint64_t)r[t] + c;
        r[t] = uint32_t(s);
        c = uint32_t(s >> 32);
    }
}
HK_DEV void ripple_sub4(uint32_t (&r)[4], uint32_t b) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const uint64_t s = (uint64_t)r[t] - b;
        r[t] = uint32_t(s);
        b = uint32_t(s >> 63);
    }
}

// Bit length of INT(d[0..n)) (0 for zero).  Warp-uniform.
HK_DEV int warp_bitlen(const uint32_t* d, int n) {
    for (int b0 = ((n - 1) >> 7) << 7; b0 >= 0; b0 -= 128) {
        const int w0 = b0 + 4 * lane();
        int top = -1;
        uint32_t tv = 0u;
#pragma unroll
        for (int t = 3; t >= 0; --t) {
            const int w = w0 + t;
            const uint32_t v = w < n ? d[w] : 0u;
            if (top < 0 && v != 0u) {
                top = w;
                tv = v;
            }
        }
        const uint32_t m = ballot(top >= 0);
        if (m) {
            const int hl = 31 - clz32(m);
            const int tw = int(shfl(uint32_t(top), hl));
            const uint32_t v = shfl(tv, hl);
            return tw * 32 + (32 - clz32(v));
        }
    }
    return 0;
}

// Bits [lo, hi] (0 <= lo <= hi) of INT(d[0..n)): bit0 = any set, bit1 = all set.
HK_DEV int warp_bit_range(const uint32_t* d, int n, int lo, int hi) {
    bool any = false, all = true;
    const int ql = lo >> 5, qh = hi >> 5;
    for (int b0 = ql; b0 <= qh; b0 += 128) {
        const int w0 = b0 + 4 * lane();
        bool a = false, na = false;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int w = w0 + t;
            if (w <= qh) {
                const int s = lo - 32 * w > 0 ? lo - 32 * w : 0;
                const int e = hi - 32 * w < 31 ? hi - 32 * w : 31;
                const uint32_t mask = (e == 31 ? 0xffffffffu : ((1u << (e + 1)) - 1u)) & ~((1u << s) - 1u);
                const uint32_t v = (w < n ? d[w] : 0u) & mask;
                a |= v != 0u;
                na |= v != mask;
            }
        }
        any |= ballot(a) != 0u;
        all &= ballot(na) == 0u;
    }
    return (any ? 1 : 0) | (all ? 2 : 0);
}

// out[0..nout) = RNE_{32 nout}(X + Y).  G is a smem scratch window of at least
// max(X.n, Y.n, nout) + 4 limbs that must not alias X, Y or out.  X or Y may
// alias `out` (all operand reads finish before the first write).
//
// Ziv mode (ubit != kExact): the true value is X + Y + delta with |delta| <
// 2^ubit (absolute bit position) of unknown sign.  If no rounding midpoint can
// lie within that distance, the correctly rounded result of the true value is
// RNE(X + Y): it is written and *ok = true.  Otherwise nothing is written and
// *ok = false (the caller recomputes exactly).
HK_DEV RMeta warp_round_sum(const Opd& Xin, const Opd& Yin, uint32_t* G, uint32_t* out, int nout,
                                 int ubit = kExact, bool* ok = nullptr) {
    const int ln = lane();
    if (ok) *ok = true;
    const int blX = Xin.sign ? (Xin.bl ? Xin.bl : warp_bitlen(Xin.d, Xin.n)) : 0;
    const int blY = Yin.sign ? (Yin.bl ? Yin.bl : warp_bitlen(Yin.d, Yin.n)) : 0;
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
    const int nw = W + 1;
    const bool small_live = blS != 0;
    bool sticky = false;
    if (small_live) {
        const int rel = base - Small.lsb; // Small's bits below the window
        if (rel > 0) sticky = (warp_bit_range(Small.d, Small.n, 0, min(rel, 32 * Small.n) - 1) & 1) != 0;
    }
    const bool eff_sub = small_live && (Big.sign != Small.sign);

    // G = |Big| +- |Small| over limbs 0..W (limb 0 holds the sticky unit of Small)
    const int offB = (base - 32) - Big.lsb, offS = (base - 32) - Small.lsb;
    const int nS = small_live ? Small.n : 0;
    uint32_t c = 0;
    uint32_t xb[5], xs[5];
    load5(Big.d, Big.n, offB, 0, 4 * ln, xb);
    load5(Small.d, nS, offS, 0, 4 * ln, xs);
    const bool g16 = aligned16(G);
    for (int b0 = 0; b0 < nw; b0 += 128) {
        const int w0 = b0 + 4 * ln;
        const bool edge = b0 == 0 || b0 + 128 > W; // warp-uniform: limb 0 or limbs past W in range
        uint32_t vb[4], vs[4], r[4];
        shift4(xb, offB, vb);
        shift4(xs, offS, vs);
        if (b0 + 128 < nw) { // the next iteration's words, in flight during this one
            load5(Big.d, Big.n, offB, b0 + 128, w0 + 128, xb);
            load5(Small.d, nS, offS, b0 + 128, w0 + 128, xs);
        }
        if (edge) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int w = w0 + t;
                if (w == 0) {
                    vb[t] = 0u;
                    vs[t] = sticky ? 1u : 0u;
                } else if (w > W) {
                    vb[t] = vs[t] = 0u;
                }
            }
        }
        if (eff_sub) {
            uint32_t br = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint64_t d = (uint64_t)vb[t] - vs[t] - br;
                r[t] = uint32_t(d);
                br = uint32_t(d >> 63);
            }
            const uint32_t ci = lane_carry_in(br != 0u, (r[0] | r[1] | r[2] | r[3]) == 0u, c);
            ripple_sub4(r, ci);
        } else {
            uint32_t cr = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint64_t s2 = (uint64_t)vb[t] + vs[t] + cr;
                r[t] = uint32_t(s2);
                cr = uint32_t(s2 >> 32);
            }
            const uint32_t ci = lane_carry_in(cr != 0u, (r[0] & r[1] & r[2] & r[3]) == 0xffffffffu, c);
            ripple_add4(r, ci);
        }
        if (!edge && g16) {
            *reinterpret_cast<uint4*>(G + w0) = make_uint4(r[0], r[1], r[2], r[3]);
        } else {
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (w0 + t <= W) G[w0 + t] = r[t];
        }
    }
    int sign = Big.sign;
    if (eff_sub && c) { // negative: two's-complement negate
        wsync();
        uint32_t cc = 1;
        for (int b0 = 0; b0 < nw; b0 += 128) {
            const int w0 = b0 + 4 * ln;
            uint32_t r[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) r[t] = w0 + t <= W ? ~G[w0 + t] : 0u;
            const uint32_t ci = lane_carry_in(false, (r[0] & r[1] & r[2] & r[3]) == 0xffffffffu, cc);
            ripple_add4(r, ci);
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (w0 + t <= W) G[w0 + t] = r[t];
        }
        sign = -sign;
    }
    wsync();
    const int bl = warp_bitlen(G, nw);
    if (bl == 0) {
        if (ubit != kExact) { // X + Y = 0 exactly but the true value is a tiny delta
            *ok = false;
            return RMeta{0, 0};
        }
        for (int i = ln; i < nout; i += 32) out[i] = 0u;
        wsync();
        return RMeta{0, 0};
    }
    int tb = bl - 1;                 // top bit index in G
    const int lsbpos = tb - 32 * nout + 1;
    bool rbit = false, st = false;
    if (lsbpos - 1 >= 0) rbit = (G[(lsbpos - 1) >> 5] >> ((lsbpos - 1) & 31)) & 1u;
    if (ubit != kExact) {
        // as warp_round_sum: the distance to the nearest rounding midpoint must
        // exceed the uncertainty 2^ubit (the sticky limb [0,32) is uncertain)
        const int rb_rel = lsbpos - 1;
        int u_rel = ubit - (base - 32);
        if (u_rel < 32) u_rel = 32;
        bool safe = rb_rel - u_rel >= 4;
        if (safe) {
            // fast path: the (up to) 64 bits just below the round bit almost always
            // decide it (a set bit when rbit, a clear bit otherwise); else scan all
            const int lo = rb_rel - 64 > u_rel ? rb_rel - 64 : u_rel;
            const int q = lo >> 5, sh = lo & 31, nbits = rb_rel - lo; // 4 <= nbits <= 64
            const uint32_t w0 = G[q], w1 = q + 1 < nw ? G[q + 1] : 0u, w2 = q + 2 < nw ? G[q + 2] : 0u;
            const uint64_t v = (((uint64_t)fshr(w1, w2, sh) << 32) | fshr(w0, w1, sh)) &
                               (nbits >= 64 ? ~0ull : ((1ull << nbits) - 1ull));
            const uint64_t all = nbits >= 64 ? ~0ull : ((1ull << nbits) - 1ull);
            if (rbit ? v != 0ull : v != all) {
                safe = true;
            } else {
                const int rs = warp_bit_range(G, nw, u_rel, rb_rel - 1);
                safe = rbit ? (rs & 1) != 0 : (rs & 2) == 0;
            }
        }
        if (!safe) {
            *ok = false;
            return RMeta{0, 0};
        }
        st = rbit; // safe with the round bit set: a set bit lies in [u_rel, rb_rel)
    } else if (lsbpos - 1 > 0) {
        st = (warp_bit_range(G, nw, 0, lsbpos - 2) & 1) != 0;
    }
    const bool low0 = lsbpos >= 0 && ((G[lsbpos >> 5] >> (lsbpos & 31)) & 1u);
    const bool inc = rbit && (st || low0);
    wsync(); // every read of X / Y done before `out` (which may alias X or Y) is written
    uint32_t cc = inc ? 1u : 0u;
    bool ovf = false;
    const bool o16 = aligned16(out);
    for (int b0 = 0; b0 <= nout; b0 += 128) {
        const int j0 = b0 + 4 * ln;
        const bool inner = b0 + 128 <= nout - 1; // warp-uniform: every j < nout, none == nout
        uint32_t x[5], r[4];
        load5(G, nw, lsbpos, b0, j0, x);
        shift4(x, lsbpos, r);
        if (!inner) {
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (j0 + t >= nout) r[t] = 0u;
        }
        const uint32_t ci = lane_carry_in(false, (r[0] & r[1] & r[2] & r[3]) == 0xffffffffu, cc);
        ripple_add4(r, ci);
        bool o = false;
        if (inner && o16) {
            *reinterpret_cast<uint4*>(out + j0) = make_uint4(r[0], r[1], r[2], r[3]);
        } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int j = j0 + t;
                if (j < nout) out[j] = r[t];
                if (j == nout) o = r[t] != 0u;
            }
        }
        ovf |= ballot(o) != 0u;
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
