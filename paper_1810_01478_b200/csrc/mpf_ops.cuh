// mpf_ops.cuh — correctly rounded p-bit MP-float operations (one warp each),
// built on the primitives of mpf_warp.cuh.  See oracle/mpfloat.py for the
// executable specification every op here must match bit for bit.
//
// Storage of an MP float with L limbs: `uint32_t d[L]` (little-endian) plus
// `int2 meta = {exp, sign}`:  value = sign * INT(d) * 2^(exp - 32 L).
#pragma once

#include "mpf_warp.cuh"

namespace hk {

// Test hook: the host emulator can force the reciprocal's exact midpoint test
// on every call (it is otherwise skipped unless z lies near a midpoint).
#if defined(HK_WARP_EMU)
inline bool& force_exact_recip() {
    static bool f = false;
    return f;
}
#define HK_FORCE_EXACT_RECIP (::hk::force_exact_recip())
#else
#define HK_FORCE_EXACT_RECIP false
#endif

struct Meta {
    int exp;
    int sign;
};

// Per-warp scratch for fms / mul / add at up to `nmax` limbs per operand:
//   A   [nmax]        staged left factor           ┐ reused as the rounding
//   Bp  [nmax + 64]   staged, zero-padded factor   ┘ window G (2 nmax + 64 >= 2 nmax + 4)
//   P   [2 nmax]      exact product
struct OpWs {
    uint32_t* A;
    uint32_t* Bp;
    uint32_t* P;
    uint32_t* G;
};

HK_HD int opws_words(int nmax) { return 4 * nmax + 64; }

HK_DEV OpWs opws_carve(uint32_t* base, int nmax) {
    OpWs w;
    w.A = base;
    w.Bp = base + nmax;
    w.G = base;
    w.P = base + 2 * nmax + 64;
    return w;
}

// Short product: only limb columns t >= L - kGuardLimbs of x*y are formed
// (about L^2/2 + 6L limb-MACs instead of L^2).  The dropped part E of the
// product satisfies 0 <= E < L 2^(32 t0 + 32) < 2^(32 t0 + 45) units of the
// product's LSB (L <= 4096), so the exact result lies within 2^(lsbP+32 t0+46)
// of the computed sum; warp_round_sum's Ziv test proves the rounding is still
// the correctly rounded one, else the exact full product is formed (rare: it
// needs a rounding midpoint within ~2^-70 ulp, or > ~100 bits of cancellation —
// the LDLT loses <= 12 bits per update, SURVEY C1-C3 measured).
constexpr int kGuardLimbs = 6;

HK_DEV void stage_and_mul(const uint32_t* xd, const uint32_t* yd, int L, const OpWs& ws, int t0) {
    warp_copy(ws.A, xd, L);
    warp_stage_padded(ws.Bp, yd, L);
    wsync();
    warp_mul(ws.A, L, ws.Bp, L, ws.P, t0);
    wsync();
}

// out = RNE(c + sp * |x y|) given the signed product sign sp (shared by fms / mul).
HK_DEV RMeta round_with_product(const Opd& X, const uint32_t* xd, const uint32_t* yd, int lsbP, int sp,
                                uint32_t* out, int L, const OpWs& ws) {
    const int t0 = L > kGuardLimbs ? L - kGuardLimbs : 0;
    stage_and_mul(xd, yd, L, ws, t0);
    if (t0 > 0) {
        const Opd Yh{ws.P + t0, 2 * L - t0, lsbP + 32 * t0, sp};
        bool ok = false;
        const RMeta r = warp_round_sum(X, Yh, ws.G, out, L, lsbP + 32 * t0 + 46, &ok);
        if (ok) return r;
        stage_and_mul(xd, yd, L, ws, 0); // the window overwrote A / Bp: restage, exact product
    }
    const Opd Y{ws.P, 2 * L, lsbP, sp};
    return warp_round_sum(X, Y, ws.G, out, L);
}

// out = RNE(c - x*y).  c / out may alias (in global memory).
HK_DEV Meta warp_fms(const uint32_t* cd, Meta cm, const uint32_t* xd, Meta xm, const uint32_t* yd, Meta ym,
                     uint32_t* out, int L, const OpWs& ws) {
    const int sp = -(xm.sign * ym.sign);
    const Opd X{cd, L, cm.exp - 32 * L, cm.sign, 32 * L};
    if (sp == 0) {
        const Opd Z{nullptr, 0, 0, 0};
        const RMeta r = warp_round_sum(X, Z, ws.G, out, L);
        return Meta{r.exp, r.sign};
    }
    const RMeta r = round_with_product(X, xd, yd, xm.exp + ym.exp - 64 * L, sp, out, L, ws);
    return Meta{r.exp, r.sign};
}

// out = RNE(x*y)
HK_DEV Meta warp_mulr(const uint32_t* xd, Meta xm, const uint32_t* yd, Meta ym, uint32_t* out, int L,
                      const OpWs& ws) {
    const int sp = xm.sign * ym.sign;
    const Opd Z{nullptr, 0, 0, 0};
    if (sp == 0) {
        const RMeta r = warp_round_sum(Z, Z, ws.G, out, L);
        return Meta{r.exp, r.sign};
    }
    const RMeta r = round_with_product(Z, xd, yd, xm.exp + ym.exp - 64 * L, sp, out, L, ws);
    return Meta{r.exp, r.sign};
}

// ---- paired FMA: out_q = RNE(c_q - x_q y) for q = 0, 1 with a shared y.
// Scratch (words): A0 [L] | A1 [L] | Bp [L+64] | P0 [2L] | P1 [2L]  (7L + 64);
// the rounding window reuses A0.. (>= L + 10 words needed), and a Ziv fallback
// of member 0 (single-FMA path, which clobbers [0, 4L+64)) leaves P1 intact.
HK_HD int opws2_words(int L) { return 7 * L + 64; }

HK_DEV void warp_fms2(const uint32_t* c0, Meta cm0, const uint32_t* x0, Meta xm0, const uint32_t* c1, Meta cm1,
                      const uint32_t* x1, Meta xm1, const uint32_t* yd, Meta ym, uint32_t* out0, uint32_t* out1,
                      Meta& r0, Meta& r1, int L, uint32_t* ws) {
    uint32_t* A0 = ws;
    uint32_t* A1 = ws + L;
    uint32_t* Bp = ws + 2 * L;
    uint32_t* P0 = ws + 3 * L + 64;
    uint32_t* P1 = ws + 5 * L + 64;
    const int t0 = L > kGuardLimbs ? L - kGuardLimbs : 0;
    const int sp0 = -(xm0.sign * ym.sign), sp1 = -(xm1.sign * ym.sign);
    if (t0 == 0 || sp0 == 0 || sp1 == 0 || (reinterpret_cast<uintptr_t>(A1) & 15)) { // rare / tiny: single path
        r0 = warp_fms(c0, cm0, x0, xm0, yd, ym, out0, L, opws_carve(ws, L));
        r1 = warp_fms(c1, cm1, x1, xm1, yd, ym, out1, L, opws_carve(ws, L));
        return;
    }
    warp_copy(A0, x0, L);
    warp_copy(A1, x1, L);
    warp_stage_padded(Bp, yd, L);
    wsync();
    warp_mul2(A0, A1, L, Bp, L, P0, P1, t0);
    wsync();
    const int lsb0 = xm0.exp + ym.exp - 64 * L, lsb1 = xm1.exp + ym.exp - 64 * L;
    bool ok = false;
    RMeta a = warp_round_sum(Opd{c0, L, cm0.exp - 32 * L, cm0.sign, 32 * L},
                                  Opd{P0 + t0, 2 * L - t0, lsb0 + 32 * t0, sp0}, ws, out0, L,
                                  lsb0 + 32 * t0 + 46, &ok);
    if (ok) r0 = Meta{a.exp, a.sign};
    else r0 = warp_fms(c0, cm0, x0, xm0, yd, ym, out0, L, opws_carve(ws, L));
    a = warp_round_sum(Opd{c1, L, cm1.exp - 32 * L, cm1.sign, 32 * L}, Opd{P1 + t0, 2 * L - t0, lsb1 + 32 * t0, sp1},
                            ws, out1, L, lsb1 + 32 * t0 + 46, &ok);
    if (ok) r1 = Meta{a.exp, a.sign};
    else r1 = warp_fms(c1, cm1, x1, xm1, yd, ym, out1, L, opws_carve(ws, L));
}

// out = RNE(x + y); x, y may alias out.
HK_DEV Meta warp_addr(const uint32_t* xd, Meta xm, const uint32_t* yd, Meta ym, uint32_t* out, int L,
                      const OpWs& ws) {
    const Opd X{xd, L, xm.exp - 32 * L, xm.sign, 32 * L};
    const Opd Y{yd, L, ym.exp - 32 * L, ym.sign, 32 * L};
    const RMeta r = warp_round_sum(X, Y, ws.G, out, L);
    return Meta{r.exp, r.sign};
}

// ---------------------------------------------------------------- reciprocal
//
// RNE(1/d) with d = m 2^e, m = M/2^p in [1/2, 1):
//   1. z0 = 1/m in binary64 (52+ bits);
//   2. Newton z <- z + z (1 - m z) with precision doubling up to L+2 limbs,
//      each intermediate correctly rounded at its working length;
//   3. r = RNE_p(z); one exact midpoint test sign(1 - m * mid) on the side of r
//      that z lies (z is accurate to ~2^-(p+50), so r is off by at most one ulp
//      and only when 1/m is within that distance of a midpoint);
//   4. result = r 2^-e.
// Scratch (words): Z, E, T [nmax + 1 each], A [nmax], Bp [nmax + 64],
// P [2 nmax + 2], G [2 nmax + 8], one [1], tmp [1], with nmax = L + 2.
struct RecipWs {
    uint32_t *Z, *E, *T, *A, *Bp, *P, *G, *one, *tmp;
};

HK_HD int align4(int n) { return (n + 3) & ~3; }

// Every region starts 16-byte aligned (warp_mul reads A with 128-bit loads).
HK_HD int recipws_words(int L) {
    const int nm = L + 3;
    return 3 * align4(nm + 1) + align4(nm) + align4(nm + 64) + align4(2 * nm + 2) + align4(2 * nm + 8) + 4;
}

HK_DEV RecipWs recipws_carve(uint32_t* b, int L) {
    const int nm = L + 3;
    RecipWs w;
    w.A = b;
    b += align4(nm);
    w.Z = b;
    b += align4(nm + 1);
    w.E = b;
    b += align4(nm + 1);
    w.T = b;
    b += align4(nm + 1);
    w.Bp = b;
    b += align4(nm + 64);
    w.P = b;
    b += align4(2 * nm + 2);
    w.G = b;
    b += align4(2 * nm + 8);
    w.one = b;
    w.tmp = b + 1;
    return w;
}

// sign of (X + Y), exactly (round to one limb and keep the sign).
HK_DEV int warp_sign_sum(const Opd& X, const Opd& Y, uint32_t* G, uint32_t* tmp) {
    return warp_round_sum(X, Y, G, tmp, 1).sign;
}

// P = X * Y for staged operands (copies into A / Bp first).
HK_DEV void warp_mul_staged(const uint32_t* x, int nx, const uint32_t* y, int ny, const RecipWs& w) {
    warp_copy(w.A, x, nx);
    warp_stage_padded(w.Bp, y, ny);
    wsync();
    warp_mul(w.A, nx, w.Bp, ny, w.P);
    wsync();
}

HK_DEV int recip_finish(const uint32_t* Md, int L, int nz, int zlsb, const RecipWs& w);

HK_DEV Meta warp_recip(const uint32_t* Md, Meta dm, uint32_t* out, int L, const RecipWs& w) {
    const int ln = lane();
    if (ln == 0) w.one[0] = 1u;
    // 1. binary64 seed
    const uint64_t mh = ((uint64_t)Md[L - 1] << 32) | (L >= 2 ? Md[L - 2] : 0u);
    const double md = ldexp((double)mh, -64);
    const double zd = 1.0 / md;
    int ex;
    const double fr = frexp(zd, &ex);
    const uint64_t mant = (uint64_t)ldexp(fr, 53);
    if (ln == 0) {
        w.Z[0] = uint32_t(mant);
        w.Z[1] = uint32_t(mant >> 32);
    }
    wsync();
    int nz = 2, zlsb = ex - 53;
    const Opd one{w.one, 1, 0, 1};

    // 2. Newton with precision doubling: schedule n_K = L+2, n_{k-1} = (n_k+1)/2 + 1
    int sched[32];
    int ns = 0;
    for (int n = L + 2;; n = (n + 1) / 2 + 1) {
        sched[ns++] = n;
        if (n <= 3) break;
    }
    for (int si = ns - 1; si >= 0; --si) {
        const int nk = sched[si];
        const int mn = nk >= L ? L : nk;
        const uint32_t* mdp = Md + (L - mn);
        const int mlsb = -32 * mn;
        // e = RNE_nk(1 - m z)
        warp_mul_staged(mdp, mn, w.Z, nz, w);
        const Opd mz{w.P, mn + nz, mlsb + zlsb, -1};
        const RMeta re = warp_round_sum(one, mz, w.G, w.E, nk);
        if (re.sign == 0) continue; // z already exact
        const int elsb = re.exp - 32 * nk;
        // z = RNE_nk(z + z e)
        warp_mul_staged(w.Z, nz, w.E, nk, w);
        const Opd zz{w.Z, nz, zlsb, 1};
        const Opd ze{w.P, nz + nk, zlsb + elsb, re.sign};
        const RMeta rz = warp_round_sum(zz, ze, w.G, w.Z, nk);
        nz = nk;
        zlsb = rz.exp - 32 * nk;
    }
    const int rexp = recip_finish(Md, L, nz, zlsb, w);
    for (int i = ln; i < L; i += 32) out[i] = w.T[i];
    wsync();
    return Meta{rexp - dm.exp, dm.sign};
}

// Step 3 of the reciprocal (one warp): r = RNE_L(z) into w.T, then the Ziv /
// exact midpoint test.  Returns r's exponent (r ~ 1/m in [1, 2]).
HK_DEV int recip_finish(const uint32_t* Md, int L, int nz, int zlsb, const RecipWs& w) {
    const int ln = lane();
    const Opd one{w.one, 1, 0, 1};
    const Opd zf{w.Z, nz, zlsb, 1};
    const Opd none{nullptr, 0, 0, 0};
    RMeta rr = warp_round_sum(zf, none, w.G, w.T, L);
    int rexp = rr.exp;
    // Ziv: after the last Newton step at L+2 limbs, |z - 1/m| is a few units
    // of z's last limb, so when the two discarded limbs are far from the
    // half-way pattern 0x8000..0, RNE(z) = RNE(1/m) and the exact test is
    // skipped (it runs only for the ~2^-47 fraction of near-midpoint cases).
    bool safe = false;
    if (nz == L + 2) {
        const uint64_t f = ((uint64_t)w.Z[1] << 32) | w.Z[0];
        const uint64_t half = 1ull << 63;
        safe = (f > half ? f - half : half - f) > (1ull << 16);
    }
    const Opd rneg{w.T, L, rexp - 32 * L, -1};
    const int sigma = (safe && !HK_FORCE_EXACT_RECIP) ? 0 : warp_sign_sum(zf, rneg, w.G, w.tmp);
    if (sigma != 0) {
        // is r the power of two 2^(p-1) (binade edge below)?
        bool edge = false;
        if (sigma < 0) {
            bool nz_low = false;
            for (int b0 = 0; b0 < L; b0 += 32) {
                const int j = b0 + ln;
                const uint32_t v = j < L ? w.T[j] : 0u;
                nz_low |= ballot(j < L && (j == L - 1 ? v != 0x80000000u : v != 0u)) != 0u;
            }
            edge = !nz_low;
        }
        // mid = r 2^32 +- h, h = 2^31 (or 2^30 at the binade edge), in E[0..L]
        if (sigma > 0) {
            for (int i = ln; i <= L; i += 32) w.E[i] = i == 0 ? 0x80000000u : w.T[i - 1];
        } else {
            // E = T*2^32 - h  =  (T - 1) * 2^32 + (2^32 - h)
            uint32_t bor = 1;
            for (int b0 = 0; b0 < L; b0 += 32) {
                const int j = b0 + ln;
                uint32_t v = j < L ? w.T[j] : 0u;
                bor = seg_borrow(v, false, bor);
                if (j < L) w.E[j + 1] = v;
            }
            if (ln == 0) w.E[0] = edge ? 0xC0000000u : 0x80000000u;
        }
        wsync();
        const int midlsb = rexp - 32 * L - 32;
        warp_mul_staged(Md, L, w.E, L + 1, w);
        const Opd mm{w.P, 2 * L + 1, -32 * L + midlsb, -1};
        const int tau = warp_sign_sum(one, mm, w.G, w.tmp);
        const bool odd = (w.T[0] & 1u) != 0u;
        const bool up = sigma > 0 && (tau > 0 || (tau == 0 && odd));
        const bool down = sigma < 0 && (tau < 0 || (tau == 0 && odd));
        if (up) {
            uint32_t cc = 1;
            bool ovf = false;
            for (int b0 = 0; b0 <= L; b0 += 32) {
                const int j = b0 + ln;
                uint32_t v = j < L ? w.T[j] : 0u;
                cc = seg_carry(v, false, cc);
                if (j < L) w.T[j] = v;
                ovf |= ballot(j == L && v != 0u) != 0u;
            }
            wsync();
            if (ovf) {
                for (int i = ln; i < L; i += 32) w.T[i] = i == L - 1 ? 0x80000000u : 0u;
                ++rexp;
            }
        } else if (down) {
            if (edge) {
                for (int i = ln; i < L; i += 32) w.T[i] = 0xffffffffu;
                --rexp;
            } else {
                uint32_t bor = 1;
                for (int b0 = 0; b0 < L; b0 += 32) {
                    const int j = b0 + ln;
                    uint32_t v = j < L ? w.T[j] : 0u;
                    bor = seg_borrow(v, false, bor);
                    if (j < L) w.T[j] = v;
                }
            }
        }
        wsync();
    }
    return rexp;
}

// ---------------------------------------------------------------- CTA-cooperative ops
//
// Latency matters on the LDLT's critical path (look-ahead column -> reciprocal
// -> B column, one op after the other): there one op gets a whole CTA.  All
// warps compute product column groups (cta_mul); warp 0 does the rounding and
// publishes the result metadata through shared memory.  Results are bit-identical
// to the warp versions (same correctly rounded operations).
struct CtaWs {
    OpWs op;
    uint32_t* CS;
    int* sh; // shared flags / metadata broadcast
};

HK_HD int ctaws_words(int L) { return opws_words(L) + cta_cs_words(2 * L) + 8; }

HK_DEV CtaWs ctaws_carve(uint32_t* b, int L) {
    CtaWs w;
    w.op = opws_carve(b, L);
    w.CS = b + opws_words(L);
    w.sh = reinterpret_cast<int*>(w.CS + cta_cs_words(2 * L));
    return w;
}

HK_DEV void cta_stage_and_mul(const uint32_t* xd, const uint32_t* yd, int L, const CtaWs& w, int t0) {
    cta_copy(w.op.A, xd, L);
    cta_stage_padded(w.op.Bp, yd, L);
    cta_sync();
    cta_mul(w.op.A, L, w.op.Bp, L, w.op.P, t0, w.CS);
}

HK_DEV void atomicMax_emu(int* a, int v) {
#if defined(HK_WARP_EMU)
    int cur = __atomic_load_n(a, __ATOMIC_RELAXED); // emulated lanes are host threads
    while (cur < v && !__atomic_compare_exchange_n(a, &cur, v, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
    }
#else
    atomicMax(a, v);
#endif
}

// warp 0's RMeta (and ok flag) to every thread of the CTA
HK_DEV RMeta cta_bcast_meta(const CtaWs& w, RMeta r, bool ok, bool* ok_out) {
    if (warp_id() == 0 && lane() == 0) {
        w.sh[0] = r.exp;
        w.sh[1] = r.sign;
        w.sh[2] = ok ? 1 : 0;
    }
    cta_sync();
    const RMeta o{w.sh[0], w.sh[1]};
    if (ok_out) *ok_out = w.sh[2] != 0;
    cta_sync();
    return o;
}

HK_DEV Meta cta_round_with_product(const Opd& X, const uint32_t* xd, const uint32_t* yd, int lsbP, int sp,
                                   uint32_t* out, int L, const CtaWs& w) {
    const int t0 = L > kGuardLimbs ? L - kGuardLimbs : 0;
    cta_stage_and_mul(xd, yd, L, w, t0);
    HK_TRACE(10);
    if (t0 > 0) {
        RMeta r{0, 0};
        bool ok = false;
        if (warp_id() == 0) {
            const Opd Yh{w.op.P + t0, 2 * L - t0, lsbP + 32 * t0, sp};
            r = warp_round_sum(X, Yh, w.op.G, out, L, lsbP + 32 * t0 + 46, &ok);
        }
        r = cta_bcast_meta(w, r, ok, &ok);
        HK_TRACE(11);
        if (ok) return Meta{r.exp, r.sign};
        cta_stage_and_mul(xd, yd, L, w, 0); // exact product (the window overwrote A / Bp)
    }
    RMeta r{0, 0};
    if (warp_id() == 0) {
        const Opd Y{w.op.P, 2 * L, lsbP, sp};
        r = warp_round_sum(X, Y, w.op.G, out, L);
    }
    r = cta_bcast_meta(w, r, true, nullptr);
    return Meta{r.exp, r.sign};
}

HK_DEV Meta cta_fms(const uint32_t* cd, Meta cm, const uint32_t* xd, Meta xm, const uint32_t* yd, Meta ym,
                    uint32_t* out, int L, const CtaWs& w) {
    const int sp = -(xm.sign * ym.sign);
    const Opd X{cd, L, cm.exp - 32 * L, cm.sign, 32 * L};
    if (sp == 0) {
        RMeta r{0, 0};
        if (warp_id() == 0) r = warp_round_sum(X, Opd{nullptr, 0, 0, 0}, w.op.G, out, L);
        r = cta_bcast_meta(w, r, true, nullptr);
        return Meta{r.exp, r.sign};
    }
    return cta_round_with_product(X, xd, yd, xm.exp + ym.exp - 64 * L, sp, out, L, w);
}

HK_DEV Meta cta_mulr(const uint32_t* xd, Meta xm, const uint32_t* yd, Meta ym, uint32_t* out, int L,
                     const CtaWs& w) {
    const int sp = xm.sign * ym.sign;
    const Opd Z{nullptr, 0, 0, 0};
    if (sp == 0) {
        RMeta r{0, 0};
        if (warp_id() == 0) r = warp_round_sum(Z, Z, w.op.G, out, L);
        r = cta_bcast_meta(w, r, true, nullptr);
        return Meta{r.exp, r.sign};
    }
    return cta_round_with_product(Z, xd, yd, xm.exp + ym.exp - 64 * L, sp, out, L, w);
}

// ---- CTA reciprocal, fixed-point Newton.
//
// z ~ 1/m in fixed point: Z[0..nf] (nf fraction limbs + one integer limb),
// value Z / 2^(32 nf).  One level to nk fraction limbs (all truncating):
//   T = top_mn(M) * Z                (mn = min(L, nk) limbs of m; CTA product)
//   |e|_nk = top nk fraction limbs of (T - 1)  if T >= 1   (e = 1 - m z <= 0)
//          = top nk fraction limbs of ~T       otherwise   (one's complement:
//            off by at most one unit, inside the truncation budget)
//   D = Z * |e|_nk, keep 2^-32nk and above     (CTA product)
//   Z <- (Z << 32(nk - nf)) -/+ D              (one carry pass)
// Every step truncates, so after the last level (nk = L+2) |z - 1/m| is a few
// units of 2^-32(L+2).  r = RNE_L(z) by one round; the Ziv test on the 65-66
// discarded bits certifies it, otherwise recip_finish's exact midpoint test
// runs.  Output is RNE(1/d), identical to warp_recip / oracle/mpfloat.recip.
struct FxRecipWs {
    RecipWs rw;       // A / Bp / P / Z (= z) / E (= |e|) double as the Newton buffers
    uint32_t *CS, *Z2;
    int* sh;
    uint32_t* RS;     // 160 words: warp 0's operand staging for the register levels
};

// ~64 L + 1 KB bytes: fits the 227 KB per-CTA limit up to L = 3600 (p = 115200).
HK_HD int ctarecipws_words(int L) {
    return recipws_words(L) + cta_cs_words(2 * (L + 4)) + align4(L + 4) + 8 + 160;
}

HK_DEV FxRecipWs fxrecipws_carve(uint32_t* b, int L) {
    FxRecipWs w;
    w.rw = recipws_carve(b, L);
    b += recipws_words(L);
    w.CS = b;
    b += cta_cs_words(2 * (L + 4));
    w.Z2 = b;
    b += align4(L + 4);
    w.sh = reinterpret_cast<int*>(b);
    w.RS = b + 8;
    return w;
}

// Register product for the small Newton levels: lane s holds A[s] / B[s] (a <= 32,
// b <= 32 limbs); returns C[lane] in lo and C[32 + lane] in hi.  The operands
// are parked in the warp's 160-word buffer RS (A at 0..31, B at 64.. with 32 zero
// words either side), so every column sum is a straight, unrolled run of
// broadcast / consecutive shared loads and two independent MAC chains.
HK_DEV void reg_mul(uint32_t A, int a, uint32_t B, int b, uint32_t& lo, uint32_t& hi, uint32_t* RS) {
    const int ln = lane();
    uint32_t* SA = RS;
    uint32_t* SB = RS + 32; // SB[32 + i] = B[i]
    SA[ln] = ln < a ? A : 0u;
    SB[ln] = 0u;
    SB[32 + ln] = ln < b ? B : 0u;
    SB[64 + ln] = 0u;
    SB[96 + ln] = 0u;
    wsync();
    uint32_t c0 = 0, c1 = 0, c2 = 0, d0 = 0, d1 = 0, d2 = 0;
    for (int s = 0; s < a; s += 4) { // SA is zero-padded to 32 words
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t as = SA[s + u];
            mac96(c0, c1, c2, as, SB[32 + ln - (s + u)]);
            mac96(d0, d1, d2, as, SB[64 + ln - (s + u)]);
        }
    }
    wsync(); // RS is rewritten by the next product
    CarryState cs;
    lo = carry_group(cs, c0, c1, c2);
    hi = carry_group(cs, d0, d1, d2);
}
// limb t (0 <= t < 64) of a (lo, hi) register product, for every lane's own t
HK_DEV uint32_t reg_limb(uint32_t lo, uint32_t hi, int t) {
    const uint32_t vl = shfl(lo, t & 31), vh = shfl(hi, t & 31);
    return t < 32 ? vl : vh;
}

// ---- The first Newton levels in scalar code.  A register level costs ~2200
// cycles whatever its size (two products' staging, shuffles and ballot carry
// passes: measured with tools/recip_probe.cu), and the schedule crawls through
// 3, 4, 5, 8 limbs before the sizes start to matter.  Up to 8 fraction limbs the
// same level formulas are therefore evaluated by every lane redundantly on
// compile-time-sized arrays (fully unrolled, all in registers): 2 -> 3 -> 4 ->
// 6 -> 8 limbs, each level with the two limbs of slack the schedule keeps
// (nk <= 2 nf - 2; the binary64 seed's 2 -> 3).  The result only seeds the later
// levels: the final Ziv test / exact midpoint test still decides the rounding.
template <int NA, int NB>
HK_DEV void scalar_mul(const uint32_t (&A)[NA], const uint32_t (&B)[NB], uint32_t (&P)[NA + NB]) {
    uint32_t c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
    for (int t = 0; t < NA + NB - 1; ++t) {
#pragma unroll
        for (int s = 0; s < NA; ++s)
            if (t - s >= 0 && t - s < NB) mac96(c0, c1, c2, A[s], B[t - s]);
        P[t] = c0;
        c0 = c1;
        c1 = c2;
        c2 = 0;
    }
    P[NA + NB - 1] = c0;
}

// One level nf = NF -> nk = NK fraction limbs (NK <= 8 <= L, so m_top = the top NK
// limbs Mt[8 - NK .. 8) of m): the formulas of the register / CTA levels below.
template <int NF, int NK>
HK_DEV void scalar_recip_level(const uint32_t (&Mt)[8], const uint32_t (&Zi)[NF + 1], uint32_t (&Zo)[NK + 1]) {
    uint32_t mtop[NK];
#pragma unroll
    for (int q = 0; q < NK; ++q) mtop[q] = Mt[8 - NK + q];
    uint32_t T[NK + NF + 1];
    scalar_mul<NK, NF + 1>(mtop, Zi, T); // FT = NK + NF fraction limbs
    const bool neg = T[NK + NF] != 0u;   // T >= 1  ->  e <= 0
    uint32_t E[NK];
#pragma unroll
    for (int q = 0; q < NK; ++q) E[q] = neg ? T[NF + q] : ~T[NF + q];
    uint32_t D[NF + 1 + NK];
    scalar_mul<NF + 1, NK>(Zi, E, D);
    uint32_t c = 0; // borrow / carry
#pragma unroll
    for (int q = 0; q <= NK; ++q) {
        const uint32_t zv = q >= NK - NF ? Zi[q - (NK - NF)] : 0u;
        const uint32_t dv = D[NF + q];
        const uint64_t d = neg ? (uint64_t)zv - dv - c : (uint64_t)zv + dv + c;
        Zo[q] = uint32_t(d);
        c = neg ? uint32_t(d >> 63) : uint32_t(d >> 32);
    }
}

constexpr int kScalarLevel = 8; // fraction limbs the scalar levels deliver (L >= kScalarLevel only)

// z ~ 1/m to 8 fraction limbs from the binary64 seed Z2 (2 fraction limbs + integer limb)
HK_DEV void scalar_recip8(const uint32_t (&Mt)[8], const uint32_t (&Z2)[3], uint32_t (&Z8)[9]) {
    uint32_t Z3[4], Z4[5], Z6[7];
    scalar_recip_level<2, 3>(Mt, Z2, Z3);
    scalar_recip_level<3, 4>(Mt, Z3, Z4);
    scalar_recip_level<4, 6>(Mt, Z4, Z6);
    scalar_recip_level<6, 8>(Mt, Z6, Z8);
}

// The small Newton levels (nk <= kRegLevel limbs): warp 0 alone with one limb per
// lane in registers — no shared-memory staging, no block barriers.
#ifndef HK_REG_LEVEL
#define HK_REG_LEVEL 30
#endif
#ifndef HK_SCALAR_RECIP_LEVELS
#define HK_SCALAR_RECIP_LEVELS 1
#endif
constexpr int kRegLevel = HK_REG_LEVEL;

HK_DEV Meta cta_recip(const uint32_t* Md, Meta dm, uint32_t* out, int L, uint32_t* wsb) {
    HK_TRACE(0);
    FxRecipWs w = fxrecipws_carve(wsb, L);
    const bool w0 = warp_id() == 0;
    // seed: z0 = 1/m_hi in binary64, as a fixed-point value with 2 fraction limbs
    const uint64_t mh = ((uint64_t)Md[L - 1] << 32) | (L >= 2 ? Md[L - 2] : 0u);
    const double zd = 1.0 / ldexp((double)mh, -64);
    int ex;
    const uint64_t mant = (uint64_t)ldexp(frexp(zd, &ex), 53); // zd = mant 2^(ex-53), ex in {1, 2}
    if (cta_tid() == 1) w.rw.one[0] = 1u;
    int sched[32];
    int ns = 0;
    for (int n = L + 2;; n = (n + 1) / 2 + 1) {
        sched[ns++] = n;
        if (n <= 3) break;
    }
    // levels handled in registers by warp 0 (block-uniform bookkeeping)
    int nreg = 0;
    while (nreg < ns && sched[ns - 1 - nreg] <= kRegLevel) ++nreg;
    if (w0) {
        const int ln = lane();
        // top min(L, 32) limbs of m, lane l -> Md[mbase + l]
        const int mbase = L > 32 ? L - 32 : 0;
        const uint32_t Mt = ln < L ? Md[mbase + ln] : 0u;
        uint32_t Zr; // seed: Z = mant << (64 + ex - 53), a 66-bit value with 2 fraction limbs
        {
            const int sh = ex + 11;
            const uint64_t lo = mant << sh;
            Zr = ln == 0 ? uint32_t(lo) : ln == 1 ? uint32_t(lo >> 32) : ln == 2 ? uint32_t(mant >> (64 - sh)) : 0u;
        }
        int nfr = 2;
        if (L >= kScalarLevel && HK_SCALAR_RECIP_LEVELS) { // levels up to 8 limbs in scalar code (every lane the same)
            uint32_t Mt8[8], Z2[3], Z8[9];
#pragma unroll
            for (int q = 0; q < 8; ++q) Mt8[q] = Md[L - 8 + q];
            {
                const int sh = ex + 11;
                const uint64_t lo = mant << sh;
                Z2[0] = uint32_t(lo);
                Z2[1] = uint32_t(lo >> 32);
                Z2[2] = uint32_t(mant >> (64 - sh));
            }
            scalar_recip8(Mt8, Z2, Z8);
            Zr = 0u;
#pragma unroll
            for (int q = 0; q <= 8; ++q)
                if (ln == q) Zr = Z8[q];
            nfr = kScalarLevel;
        }
        HK_TRACE(13);
        for (int r = 0; r < nreg; ++r) {
            const int nk = sched[ns - 1 - r];
            if (nk <= nfr) continue; // covered by the scalar levels
            const int mn = nk >= L ? L : nk;
            const uint32_t mv = shfl(Mt, (L - mn - mbase + ln) & 31);
            const uint32_t mtop = ln < mn ? mv : 0u;
            uint32_t tlo, thi;
            reg_mul(Zr, nfr + 1, mtop, mn, tlo, thi, w.RS); // T = m_top * z
            const int FT = mn + nfr;
            const bool neg = reg_limb(tlo, thi, FT) != 0u; // T >= 1  ->  e <= 0
            const uint32_t ev = reg_limb(tlo, thi, FT - nk + ln);
            const uint32_t E = ln < nk ? (neg ? ev : ~ev) : 0u;
            uint32_t dlo, dhi;
            reg_mul(Zr, nfr + 1, E, nk, dlo, dhi, w.RS); // D = z * |e|
            const int shl = nk - nfr;
            const uint32_t zs = shfl(Zr, (ln - shl) & 31);
            const uint32_t zv = (ln >= shl && ln - shl <= nfr) ? zs : 0u;
            const uint32_t dd = reg_limb(dlo, dhi, nfr + ln);
            const uint32_t dv = ln <= nk ? dd : 0u;
            uint32_t r2;
            if (neg) {
                r2 = zv - dv;
                seg_borrow(r2, zv < dv, 0u);
            } else {
                r2 = zv + dv;
                seg_carry(r2, r2 < zv, 0u);
            }
            Zr = ln <= nk ? r2 : 0u;
            nfr = nk;
            HK_TRACE(12);
        }
        if (ln <= nfr + 1) w.rw.Z[ln] = ln <= nfr ? Zr : 0u;
    }
    cta_sync();
    HK_TRACE(14);
    int nf = nreg ? sched[ns - nreg] : 2;
    uint32_t* Z = w.rw.Z;
    uint32_t* Zn = w.Z2;
    for (int si = ns - 1 - nreg; si >= 0; --si) {
        const int nk = sched[si];
        const int mn = nk >= L ? L : nk;
        // T = m_top * z; only limbs FT-nk .. FT are used: a short product from two
        // guard limbs below (the dropped columns perturb limb FT-nk by at most a unit,
        // inside the level's truncation budget; the final Ziv test / exact fallback
        // still decides the rounding)
        const int FT = mn + nf; // fraction limbs of T
        const int tT = FT - nk - 2 > 0 ? FT - nk - 2 : 0;
        // m_top sits in rw.T (free until the final round): staged before the first
        // CTA level, later by the warps idle during the previous level's Z update
        if (si == ns - 1 - nreg) cta_copy(w.rw.T, Md + (L - mn), mn);
        cta_stage_padded(w.rw.Bp, Z, nf + 1);
        if (cta_tid() == 0) w.sh[1] = 0;
        cta_sync();
        cta_mul(w.rw.T, mn, w.rw.Bp, nf + 1, w.rw.P, tT, w.CS);
        HK_TRACE(1);
        const bool neg = w.rw.P[FT] != 0u; // T >= 1  ->  e <= 0
        for (int q = cta_tid(); q < nk; q += cta_threads()) {
            const uint32_t v = w.rw.P[FT - nk + q];
            const uint32_t e = neg ? v : ~v;
            w.rw.E[q] = e;
            if (e != 0u) atomicMax_emu(w.sh + 1, q + 1);
        }
        cta_sync();
        // D = z * |e|: |e| < 2^(-32 (nf - 1)), so its top limbs are zero; the product
        // runs over the ne significant ones only (exact: zeros contribute nothing)
        const int ne = w.sh[1] > 0 ? w.sh[1] : 1;
        cta_copy(w.rw.A, Z, nf + 1);
        cta_stage_padded(w.rw.Bp, w.rw.E, ne);
        cta_sync();
        cta_mul(w.rw.A, nf + 1, w.rw.Bp, ne, w.rw.P, 0, w.CS);
        HK_TRACE(2);
        const int nD = nf + 1 + ne; // limbs of D
        // Z' = (Z << 32 (nk - nf)) -/+ (D >> 32 nf), over nk + 1 limbs; four limbs per
        // lane, one ballot lookahead per 128 limbs
        if (w0) {
            const int shl = nk - nf;
            uint32_t c = 0;
            for (int b0 = 0; b0 <= nk; b0 += 128) {
                const int q0 = b0 + 4 * lane();
                uint32_t r[4];
                uint32_t br = 0;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int q = q0 + t;
                    const uint32_t zv = (q <= nk && q >= shl) ? Z[q - shl] : 0u;
                    const uint32_t dv = (q <= nk && nf + q < nD) ? w.rw.P[nf + q] : 0u;
                    const uint64_t d = neg ? (uint64_t)zv - dv - br : (uint64_t)zv + dv + br;
                    r[t] = uint32_t(d);
                    br = neg ? uint32_t(d >> 63) : uint32_t(d >> 32);
                }
                if (neg) {
                    const uint32_t ci = lane_carry_in(br != 0u, (r[0] | r[1] | r[2] | r[3]) == 0u, c);
                    ripple_sub4(r, ci);
                } else {
                    const uint32_t ci = lane_carry_in(br != 0u, (r[0] & r[1] & r[2] & r[3]) == 0xffffffffu, c);
                    ripple_add4(r, ci);
                }
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (q0 + t <= nk) Zn[q0 + t] = r[t];
            }
        }
        if (si > 0 && (!w0 || num_warps() == 1)) { // stage the next level's m_top
            const int mn1 = sched[si - 1] >= L ? L : sched[si - 1];
            const int t0 = num_warps() == 1 ? cta_tid() : cta_tid() - 32;
            const int nt = num_warps() == 1 ? cta_threads() : cta_threads() - 32;
            for (int q = t0; q < mn1; q += nt) w.rw.T[q] = Md[L - mn1 + q];
        }
        cta_sync();
        HK_TRACE(3);
        uint32_t* t = Z;
        Z = Zn;
        Zn = t;
        nf = nk;
    }
    // r = RNE_L(z), Ziv test on the discarded bits, exact test if needed
    if (w0) {
        const int nz = L + 3; // nf = L + 2 fraction limbs + integer limb
        const Opd zf{Z, nz, -32 * (L + 2), 1};
        const RMeta rr = warp_round_sum(zf, Opd{nullptr, 0, 0, 0}, w.rw.G, w.rw.T, L);
        int rexp = rr.exp;
        // discarded bits: k = bitlen(Z) - 32 L (65 or 66); distance to the half
        const int kbits = (32 * (L + 2) + (Z[L + 2] >= 2u ? 2 : 1)) - 32 * L;
        const uint64_t lo64 = ((uint64_t)Z[1] << 32) | Z[0];
        const uint32_t top = Z[2] & ((1u << (kbits - 64)) - 1u); // 1 or 2 bits above the low 64
        // value f = top 2^64 + lo64, half = 2^(kbits-1)
        bool safe;
        if (kbits == 65)
            safe = top ? lo64 > (1ull << 16) : lo64 < ~0ull - (1ull << 16);
        else // kbits == 66: half = 2^65 = top 2 (binary 10) with lo64 = 0
            safe = top == 2u ? lo64 > (1ull << 16) : (top == 1u ? lo64 < ~0ull - (1ull << 16) : true);
        if (!safe || HK_FORCE_EXACT_RECIP) {
            if (Z != w.rw.Z) {
                for (int q = lane(); q < nz; q += 32) w.rw.Z[q] = Z[q];
                wsync();
            }
            rexp = recip_finish(Md, L, nz, -32 * (L + 2), w.rw);
        }
        if (lane() == 0) w.sh[0] = rexp;
    }
    cta_sync();
    HK_TRACE(4);
    const int rexp = w.sh[0];
    cta_copy(out, w.rw.T, L);
    cta_sync();
    return Meta{rexp - dm.exp, dm.sign};
}

} // namespace hk
