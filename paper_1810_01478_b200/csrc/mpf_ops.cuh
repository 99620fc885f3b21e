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
    const Opd X{cd, L, cm.exp - 32 * L, cm.sign};
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

// out = RNE(x + y); x, y may alias out.
HK_DEV Meta warp_addr(const uint32_t* xd, Meta xm, const uint32_t* yd, Meta ym, uint32_t* out, int L,
                      const OpWs& ws) {
    const Opd X{xd, L, xm.exp - 32 * L, xm.sign};
    const Opd Y{yd, L, ym.exp - 32 * L, ym.sign};
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
    const int nm = L + 2;
    return 3 * align4(nm + 1) + align4(nm) + align4(nm + 64) + align4(2 * nm + 2) + align4(2 * nm + 8) + 4;
}

HK_DEV RecipWs recipws_carve(uint32_t* b, int L) {
    const int nm = L + 2;
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
    // 3. r = RNE_L(z), then one exact midpoint test
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
    // 4. write out, exponent 1/d = (1/m) 2^-e
    for (int i = ln; i < L; i += 32) out[i] = w.T[i];
    wsync();
    return Meta{rexp - dm.exp, dm.sign};
}

} // namespace hk
