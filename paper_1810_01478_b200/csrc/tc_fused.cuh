// tc_fused.cuh — the certified rounding of the LDLT bulk update, fused into the
// tensor-core product kernel's epilogue: S(k,j) = RNE(S(k,j) - x_j y_k) is
// formed by the thread that drains row k's product from TMEM, in drain order
// (low limbs first), straight from the product limbs into c in place — no
// product scratch in HBM, no second pass (the reference's submul_rounded,
// fixedpoint.cpp:146-154: exact product, one rounding, subtract).
//
// One thread per item.  Before the first product limb arrives the thread
// predicts, from the top 64 bits of c, x and y, the sign s_R and the exponent
// E_R of R = c - x y with a rigorous error bound (192-bit arithmetic; any
// doubt -> the exact fix-up kernel).  The output LSB is then E_R - p, and the
// result is one streaming pass over absolute 32-bit words w = -8 .. L-1 of
// |R| (w < 0: the tail below the output LSB):
//     r_w = a_w + (b_w ^ m) + carry        (a, b = C, P or P, C; m = ~0 for a
//                                           difference, two's complement)
// with the P words funnel-shifted out of the drained product limbs and the C
// words out of c's limbs (a 16-limb register window, one 32-byte load per 8
// words, loaded a group ahead of the in-place stores).  When w = -1 is done,
// the Ziv certificate of warp_round_sum decides the rounding from the tail
// (the short product's dropped part and the truncation below w = -8 are the
// uncertainty); words w >= 0 then get the rounding increment and are stored
// 8 at a time, 32-byte aligned.  Items the certificate (or the prediction)
// cannot settle are left untouched and listed for the exact redo (FixLdlt /
// FixD), so every result is exactly RNE(c - x y), bit-identical to the IMAD
// path and to oracle/mpfloat.py.
#pragma once

#include "mpf_ops.cuh"

namespace hk {

HK_DEV uint64_t mulhi_u64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// 256-bit unsigned (w[0] least significant) for the exponent prediction
struct U256 {
    uint64_t w[4];
};

// (hi:lo) * 2^s, s <= 64 (negative: floor of the right shift)
HK_DEV U256 u256_shl128(uint64_t hi, uint64_t lo, int s) {
    U256 r{{0, 0, 0, 0}};
    if (s >= 0) {
        if (s == 0) {
            r.w[0] = lo;
            r.w[1] = hi;
        } else if (s >= 64) {
            r.w[1] = lo;
            r.w[2] = hi;
        } else {
            r.w[0] = lo << s;
            r.w[1] = (hi << s) | (lo >> (64 - s));
            r.w[2] = hi >> (64 - s);
        }
    } else {
        const int t = -s;
        if (t >= 128) return r;
        if (t >= 64) {
            r.w[0] = hi >> (t - 64); // t - 64 < 64
        } else {
            r.w[0] = (lo >> t) | (hi << (64 - t));
            r.w[1] = hi >> t;
        }
    }
    return r;
}

HK_DEV U256 u256_add(const U256& a, const U256& b) {
    U256 r;
    uint64_t c = 0;
    for (int i = 0; i < 4; ++i) {
        const uint64_t s = a.w[i] + b.w[i];
        const uint64_t c1 = s < a.w[i];
        r.w[i] = s + c;
        c = c1 | (r.w[i] < s);
    }
    return r;
}

HK_DEV U256 u256_sub(const U256& a, const U256& b) { // a >= b
    U256 r;
    uint64_t br = 0;
    for (int i = 0; i < 4; ++i) {
        const uint64_t d = a.w[i] - b.w[i];
        const uint64_t b1 = a.w[i] < b.w[i];
        r.w[i] = d - br;
        br = b1 | (d < br);
    }
    return r;
}

HK_DEV bool u256_ge(const U256& a, const U256& b) {
    for (int i = 3; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] > b.w[i];
    return true;
}

HK_DEV int u256_bitlen(const U256& a) {
    for (int i = 3; i >= 0; --i)
        if (a.w[i]) return 64 * i + 64 - (a.w[i] >> 32 ? clz32(uint32_t(a.w[i] >> 32)) : 32 + clz32(uint32_t(a.w[i])));
    return 0;
}

constexpr int kFuseTail = 8; // words below the output LSB carried by the stream

// One item's fused rounding.  Device code keeps every array in registers (all
// indices are compile-time after unrolling; the per-thread alignment offsets
// are applied with 3-stage select networks).
struct FusedRow {
    uint32_t* c = nullptr; // c's limbs (rewritten in place)
    int L = 0;
    int status = 0;        // 0 nothing to do (x or y zero), 1 streaming, 2 -> exact redo
    int ER = 0, sR = 0;    // exponent / sign of the result
    int Qp = 0, sig = 0;   // output word w <- product limbs w + Qp, w + Qp + 1, shifted right by sig
    int Qc = 0, tau = 0;   // ... <- c limbs w + Qc, w + Qc + 1, shifted right by tau
    int fK = 0, oc = 0;    // c window: block g + fK at group g, word offset oc in it
    int ow = 0;            // output word wg of group g sits at offset ow of its 8-word block
    int urel = 0;          // tail bits [urel, 255) decide the rounding (certificate)
    uint32_t mc = 0, mp = 0; // r = (C ^ mc) + (P ^ mp) + carry: one of them ~0 for a difference
    bool czero = false;
    bool decided = false, started = false;
    bool all1 = true, any1 = false;
    uint32_t cy1 = 0, cy2 = 0, pprev = 0, top = 0;
    uint32_t win[16], pre[8], pend[8];
    int why = 0;           // why the exact redo (tests): 1 binade, 2 sign/binade of c - x y, 3 cancellation, 4 certificate
    int dev = 0;           // what-if knobs (dev tools only, results wrong): 32 no stores, 1024 no loads,
                           // 2048 loads / stores to coalesced dummy addresses (wbase + 8 lane)
    uint32_t* wbase = nullptr;
    int wlane = 0;

    HK_DEV int nblocks() const { return L >> 3; }

    HK_DEV void load8(int b, uint32_t* v) const {
        if (czero || b < 0 || b >= nblocks() || (dev & 1024)) {
#pragma unroll
            for (int t = 0; t < 8; ++t) v[t] = 0u;
            return;
        }
        const uint32_t* p = (dev & 2048) ? wbase + 8 * wlane + 256 * (b & 3) : c + 8 * b;
#if defined(__CUDA_ARCH__)
        asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "l"(p));
#else
        for (int t = 0; t < 8; ++t) v[t] = p[t];
#endif
    }
    HK_DEV void store8(int b, const uint32_t* v) const {
        if (dev & 32) return;
        uint32_t* p = (dev & 2048) ? wbase + 8 * wlane + 256 * (b & 3) : c + 8 * b;
#if defined(__CUDA_ARCH__)
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                     "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
#else
        for (int t = 0; t < 8; ++t) p[t] = v[t];
#endif
    }

    // c: L limbs + meta; xt / yt: the top 64 bits of x's / y's mantissas
    HK_DEV void setup(uint32_t* c_, Meta cm, uint64_t xt, Meta xm, uint64_t yt, Meta ym, int L_) {
        c = c_;
        L = L_;
        const int sp = -(xm.sign * ym.sign); // R = c + sp |x y|
        if (sp == 0) {                        // RNE(c - 0) = c: nothing to write (as ItemTcRound)
            status = 0;
            return;
        }
        status = 2;
        const int p = 32 * L;
        const int TP = xm.exp + ym.exp;       // |x y| in [2^(TP-2), 2^TP)
        const uint64_t pl_lo = xt * yt, pl_hi = mulhi_u64(xt, yt);
        // |x y| / 2^(TP-128) in [pl, pl + 2^65)
        czero = cm.sign == 0;
        if (czero) {
            sR = sp;
            if (pl_hi >= (1ull << 63)) ER = TP;
            else if (pl_hi < (1ull << 63) - 4) ER = TP - 1;
            else {
                why = 1;
                return; // within 2^-61 of the binade edge
            }
        } else {
            const uint64_t ct = (uint64_t(c[L - 1]) << 32) | c[L - 2]; // |c| / 2^(ce-64) in [ct, ct + 1)
            const int ce = cm.exp;
            const int Z = ce > TP ? ce : TP;
            // both in units of 2^(Z-192); interval widths <= 2^128 + 1 and 2^129 + 1
            const U256 Cu = u256_shl128(ct, 0, 64 - (Z - ce));
            const U256 Pu = u256_shl128(pl_hi, pl_lo, 64 - (Z - TP));
            U256 A;
            if (cm.sign == sp) {
                A = u256_add(Cu, Pu);
                sR = sp;
            } else if (u256_ge(Cu, Pu)) {
                A = u256_sub(Cu, Pu);
                sR = cm.sign;
            } else {
                A = u256_sub(Pu, Cu);
                sR = sp;
            }
            // |R| in (A - 2^130, A + 2^130): the sign and the binade must not depend on the error
            const U256 E{{0, 0, 4, 0}}; // 2^130
            why = 2;
            if (!u256_ge(A, E)) return;
            const int bl = u256_bitlen(A);
            if (u256_bitlen(u256_sub(A, E)) != bl || u256_bitlen(u256_add(A, E)) != bl) return;
            why = 3;
            ER = Z - 192 + bl;
            const int dc = ER - ce; // output word w <- c bits 32 w + dc
            Qc = dc >> 5;            // floor
            tau = dc & 31;
            if (Qc < -kFuseTail) return; // cancellation > 256 bits: the in-place window would overrun
        }
        // product limb 0 (scratch) sits at absolute bit lambda = TP - p - 256
        const int delta = ER - TP + 256; // output LSB - lambda
        why = 3;
        if (delta < 224) return;         // > 32 bits cancellation against the product
        why = 0;
        Qp = delta >> 5;
        sig = delta & 31;
        urel = 302 - delta > 8 ? 302 - delta : 8; // certificate margin above the uncertainty 2^(lambda + 46)
        (void)p;
        const int coefC = czero ? 0 : sR * cm.sign, coefP = sR * sp; // |R| = coefC |c| + coefP |x y|
        mc = coefC < 0 ? 0xffffffffu : 0u; // |R| = |x y| - |c|
        mp = coefP < 0 ? 0xffffffffu : 0u; // |R| = |c| - |x y|
        cy1 = (mc | mp) & 1u;              // two's complement: + 1 at the stream's lowest word
        const int K0 = Qc - Qp - 1;
        fK = K0 >> 3;
        oc = K0 & 7;
        ow = (-1 - Qp) & 7;
        status = 1;
    }

    // the c limbs groups g0 .. g0 + ng - 1 will read, into L2 (one bulk prefetch;
    // issued a chunk ahead, so the in-order loads of the stream hit L2)
    HK_DEV void prefetch(int g0, int ng) const {
        if (status != 1 || czero) return;
        int lo = 8 * g0 + (Qc - Qp - 1), hi = 8 * (g0 + ng) + (Qc - Qp - 1) + 9; // limbs [lo, hi)
        lo = lo < 0 ? 0 : lo & ~3;
        hi = hi > L ? L : hi;
        if (hi <= lo) return;
#if defined(__CUDA_ARCH__)
        const uint32_t bytes = uint32_t((hi - lo) * 4 + 15) & ~15u;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c + lo), "r"(bytes) : "memory");
#endif
    }

    // group g: product limbs pl = scratch limbs [8 g, 8 g + 8) (zeros past the product)
    HK_DEV int group_block(int g) const { return (8 * g - 1 - Qp - ow) >> 3; }
    HK_DEV bool wants(int g) const { return status == 1 && group_block(g) < nblocks(); }

    HK_DEV void group(int g, const uint32_t (&pl)[8]) {
        const int wg = 8 * g - 1 - Qp;
        if (wg + 7 < -kFuseTail) { // every word below the stream: only the limb carry-over
            pprev = pl[7];
            return;
        }
        const int bg = g + fK;
        if (!started) {
            started = true;
            load8(bg, win);
            load8(bg + 1, win + 8);
            load8(bg + 2, pre);
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                win[t] = win[t + 8];
                win[t + 8] = pre[t];
            }
            load8(bg + 2, pre); // before this group's stores (they may overlap that block)
        }
        // c limbs a_g + u, u = 0..8 (a_g = 8 bg + oc): select network on oc
        uint32_t cq[9];
        {
            uint32_t t4[12], t2[10];
#pragma unroll
            for (int i = 0; i < 12; ++i) t4[i] = (oc & 4) ? win[i + 4] : win[i];
#pragma unroll
            for (int i = 0; i < 10; ++i) t2[i] = (oc & 2) ? t4[i + 2] : t4[i];
#pragma unroll
            for (int i = 0; i < 9; ++i) cq[i] = (oc & 1) ? t2[i + 1] : t2[i];
        }
        uint32_t o[8];
        const bool tail = wg < 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int w = wg + u;
            const uint32_t pw = fshr(u ? pl[u - 1] : pprev, pl[u], sig);
            const uint32_t cw = fshr(cq[u], cq[u + 1], tau);
            const uint64_t s = (uint64_t)(cw ^ mc) + (pw ^ mp) + cy1;
            const uint32_t r = uint32_t(s);
            if (w >= -kFuseTail && w < L) cy1 = uint32_t(s >> 32);
            if (tail && w >= -kFuseTail && w < 0) {
                const int tb = 32 * (w + kFuseTail); // tail bit of this word's bit 0
                uint32_t m = urel <= tb ? 0xffffffffu : (urel >= tb + 32 ? 0u : ~((1u << (urel - tb)) - 1u));
                if (w == -1) m &= 0x7fffffffu;
                all1 = all1 && ((r | ~m) == 0xffffffffu);
                any1 = any1 || ((r & m) != 0u);
                if (w == -1) {
                    const uint32_t rbit = r >> 31;
                    // Ziv: no rounding midpoint within the uncertainty of the tail
                    if (rbit ? !any1 : all1) {
                        status = 2;
                        why = 4;
                    }
                    decided = true;
                    cy2 = rbit; // round to nearest; a set bit below the round bit makes it no tie
                }
            }
            const uint64_t s2 = (uint64_t)r + cy2;
            o[u] = uint32_t(s2);
            if (w >= 0 && w < L) cy2 = uint32_t(s2 >> 32);
            if (w == L - 1) top = o[u];
        }
        pprev = pl[7];
        // rotate to the block grid: rot[(ow + u) & 7] = o[u]
        uint32_t r4[8], r2[8], rot[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r4[j] = (ow & 4) ? o[(j + 4) & 7] : o[j];
#pragma unroll
        for (int j = 0; j < 8; ++j) r2[j] = (ow & 2) ? r4[(j + 6) & 7] : r4[j];
#pragma unroll
        for (int j = 0; j < 8; ++j) rot[j] = (ow & 1) ? r2[(j + 7) & 7] : r2[j];
        const int bo = group_block(g);
        if (status == 1 && bo >= 0 && bo < nblocks()) {
            uint32_t blk[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) blk[j] = j < ow ? pend[j] : rot[j];
            store8(bo, blk);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) pend[j] = rot[j];
    }

    // after the last group: mantissa overflow (round-up of all ones) and the
    // result's metadata; returns false if the item needs the exact redo.
    // *viol: the normalisation check (a certified prediction cannot fail it).
    HK_DEV bool finish(Meta* out, bool* viol) {
        *viol = false;
        if (status != 1) return status == 0;
        int e = ER;
        if (cy2) { // all ones + 1
            c[L - 1] = 0x80000000u;
            ++e;
        } else if (!(top >> 31)) {
            *viol = true;
        }
        *out = Meta{e, sR};
        return true;
    }
};

// ---- the same stream, warp-cooperative: one row at a time per warp ---------
//
// The thread-per-row stream above makes every load and store of c touch 32
// rows (32 different cache lines per instruction — 4x the L1 wavefronts of the
// same bytes, coalesced; measured: the epilogue's row accesses cost ~0.7 s of
// C4's 4.1 s LDLT).  Here the warp streams one row's 64-word chunk at a time:
// lane l takes output words wb + 2l, wb + 2l + 1, reads c limbs coalesced, and
// the carries of the two chains (add/sub, rounding increment) cross the lanes
// with ballot lookahead.  Lane i keeps row i's state between chunks (packed,
// broadcast with a few shuffles).  Same arithmetic, same certificate, same
// results as FusedRow (which still does the prediction).
struct WarpRowState {
    uint32_t cy1 = 0, cy2 = 0, pprev = 0, sv0 = 0, sv1 = 0, top = 0;
    uint32_t prm = 0;   // Qp (bits 0-15) | sig (16-20) | tau (21-25) | mc (26) | mp (27) | czero (28)
    uint32_t prm2 = 0;  // Qc + 64 (bits 0-7) | urel (8-15)
    uint32_t flags = 0; // status (bits 0-1) | decided (2) | all1 (3) | any1 (4) | started (5)
    HK_DEV int status() const { return int(flags & 3u); }
};

// from FusedRow's prediction; rows it cannot stream (or with Q_c < -2: the
// warp stream keeps only two old limbs of c across chunks) go to the exact redo
HK_DEV WarpRowState warp_row_init(const FusedRow& f) {
    WarpRowState s;
    int st = f.status;
    if (st == 1 && !f.czero && f.Qc < -2) st = 2;
    if (st == 1 && (f.Qp > 0xffff || f.Qc + 64 > 255 || f.urel > 255)) st = 2;
    s.flags = uint32_t(st) | (1u << 3); // all1 = true
    if (st != 1) return s;
    s.prm = uint32_t(f.Qp) | (uint32_t(f.sig) << 16) | (uint32_t(f.tau) << 21) | ((f.mc & 1u) << 26) |
            ((f.mp & 1u) << 27) | (uint32_t(f.czero ? 1 : 0) << 28);
    s.prm2 = uint32_t(f.Qc + 64) | (uint32_t(f.urel) << 8);
    s.cy1 = f.cy1;
    return s;
}

// the c limbs lane l needs for chunk c of a row (window limbs 2l + 2, 2l + 3):
// issued a row ahead of warp_row_chunk, so the loads of the next row are in
// flight while this one is computed (coalesced across the warp)
HK_DEV void warp_row_load(const WarpRowState& st, const uint32_t* crow, int L, int c, uint32_t& q0, uint32_t& q1) {
    q0 = q1 = 0u;
    if (st.status() != 1 || ((st.prm >> 28) & 1u)) return;
    const int Qp = int(st.prm & 0xffffu), Qc = int(st.prm2 & 0xffu) - 64;
    const int wb = 64 * c - 1 - Qp;
    if (wb + 63 < -kFuseTail || wb >= L) return;
    const int i0 = wb + Qc + 2 + 2 * lane();
    if (i0 >= 0 && i0 < L) q0 = crow[i0];
    if (i0 + 1 >= 0 && i0 + 1 < L) q1 = crow[i0 + 1];
}

// Chunk c of row c_row (c limbs at crow, L limbs) by the whole warp.  st: the
// row's state (warp-uniform copy); p0, p1: this lane's staged product limbs
// 2 lane, 2 lane + 1 of the chunk (zeros past the product); q0, q1: its
// warp_row_load values.
HK_DEV void warp_row_chunk(WarpRowState& st, uint32_t* crow, int L, int c, uint32_t p0, uint32_t p1, uint32_t q0,
                           uint32_t q1) {
    const int l = lane();
    const int Qp = int(st.prm & 0xffffu), sig = int((st.prm >> 16) & 31u), tau = int((st.prm >> 21) & 31u);
    const uint32_t mc = (st.prm >> 26) & 1u ? 0xffffffffu : 0u, mp = (st.prm >> 27) & 1u ? 0xffffffffu : 0u;
    const bool czero = (st.prm >> 28) & 1u;
    const int Qc = int(st.prm2 & 0xffu) - 64, urel = int((st.prm2 >> 8) & 0xffu);
    const int wb = 64 * c - 1 - Qp; // lane l: output words wb + 2 l, wb + 2 l + 1
    uint32_t pm1 = shfl_up(p1, 1);
    if (l == 0) pm1 = st.pprev;
    const uint32_t pnext = shfl(p1, 31);
    if (wb + 63 < -kFuseTail || wb >= L) { // below the stream, or past the row's last word
        st.pprev = pnext;
        return;
    }
    const uint32_t pw0 = fshr(pm1, p0, sig), pw1 = fshr(p0, p1, sig);
    // c window v[k] = c[wb + Qc + k]; lane l: v[2l], v[2l+1] (from lane l-1) and v[2l+2], v[2l+3] (loaded)
    const int base = wb + Qc;
    auto climb = [&](int idx) -> uint32_t { return (czero || idx < 0 || idx >= L) ? 0u : crow[idx]; };
    uint32_t v0 = shfl_up(q0, 1), v1 = shfl_up(q1, 1);
    if (l == 0) {
        if (st.flags & 32u) { // the previous chunk saved them (c may be overwritten there now)
            v0 = st.sv0;
            v1 = st.sv1;
        } else {
            v0 = climb(base);
            v1 = climb(base + 1);
        }
    }
    const uint32_t nsv0 = shfl(q0, 31), nsv1 = shfl(q1, 31); // v[64], v[65]: the next chunk's first two
    const uint32_t cw0 = fshr(v0, v1, tau), cw1 = fshr(v1, q0, tau);
    const int w0 = wb + 2 * l, w1 = w0 + 1;
    // chain 1: |R| words, two's complement for a difference; words outside [-8, L) pass the carry
    const bool m0 = w0 >= -kFuseTail && w0 < L, m1 = w1 >= -kFuseTail && w1 < L;
    const uint64_t A = (uint64_t(m1 ? (cw1 ^ mc) : 0xffffffffu) << 32) | (m0 ? (cw0 ^ mc) : 0xffffffffu);
    const uint64_t B = (uint64_t(m1 ? (pw1 ^ mp) : 0u) << 32) | (m0 ? (pw0 ^ mp) : 0u);
    const uint64_t S = A + B;
    uint32_t cio = st.cy1;
    const uint64_t R = S + lane_carry_in(S < A, S == ~0ull, cio);
    st.cy1 = cio;
    const uint32_t r0 = uint32_t(R), r1 = uint32_t(R >> 32);
    if (!(st.flags & 4u)) { // the tail below the output LSB: Ziv certificate (as FusedRow::group)
        bool al = true, an = false;
        auto tailw = [&](int w, uint32_t r) {
            if (w < -kFuseTail || w >= 0) return;
            const int tb = 32 * (w + kFuseTail);
            uint32_t m = urel <= tb ? 0xffffffffu : (urel >= tb + 32 ? 0u : ~((1u << (urel - tb)) - 1u));
            if (w == -1) m &= 0x7fffffffu;
            al = al && ((r | ~m) == 0xffffffffu);
            an = an || ((r & m) != 0u);
        };
        tailw(w0, r0);
        tailw(w1, r1);
        if (ballot(!al)) st.flags &= ~8u;
        if (ballot(an)) st.flags |= 16u;
        if (wb <= -1 && -1 <= wb + 63) { // word -1 here: decide
            const int h = (-1 - wb) >> 1;
            const uint32_t rv = shfl(((-1 - wb) & 1) ? r1 : r0, h);
            const uint32_t rbit = rv >> 31;
            const bool all1 = st.flags & 8u, any1 = st.flags & 16u;
            if (rbit ? !any1 : all1) st.flags = (st.flags & ~3u) | 2u; // -> exact redo, nothing stored
            st.flags |= 4u;
            st.cy2 = rbit;
        }
    }
    if (st.flags & 4u) { // chain 2: + the rounding increment from word 0 up (words < 0 and >= L pass it)
        const bool o0 = w0 >= 0 && w0 < L, o1 = w1 >= 0 && w1 < L;
        const uint64_t U = (uint64_t(o1 ? r1 : 0xffffffffu) << 32) | (o0 ? r0 : 0xffffffffu);
        uint32_t cio2 = st.cy2;
        const uint64_t O = U + lane_carry_in(false, U == ~0ull, cio2);
        st.cy2 = cio2;
        const uint32_t x0 = uint32_t(O), x1 = uint32_t(O >> 32);
        if (wb <= L - 1 && L - 1 <= wb + 63) {
            const int h = (L - 1 - wb) >> 1;
            st.top = shfl(((L - 1 - wb) & 1) ? x1 : x0, h);
        }
        if (st.status() == 1) { // coalesced in-place stores (the next chunk reads c from wb + 64 + Qc + 2 on)
            if (o0) crow[w0] = x0;
            if (o1) crow[w1] = x1;
        }
    }
    st.pprev = pnext;
    st.sv0 = nsv0;
    st.sv1 = nsv1;
    st.flags |= 32u;
}

// shuffle a row state from lane src to the whole warp
HK_DEV WarpRowState warp_row_bcast(const WarpRowState& s, int src) {
    WarpRowState o;
    o.cy1 = shfl(s.cy1, src);
    o.cy2 = shfl(s.cy2, src);
    o.pprev = shfl(s.pprev, src);
    o.sv0 = shfl(s.sv0, src);
    o.sv1 = shfl(s.sv1, src);
    o.top = shfl(s.top, src);
    o.prm = shfl(s.prm, src);
    o.prm2 = shfl(s.prm2, src);
    o.flags = shfl(s.flags, src);
    return o;
}

// after the last chunk: overflow of an all-ones mantissa, the metadata; false
// -> exact redo; *viol: the normalisation check
HK_DEV bool warp_row_finish(const WarpRowState& s, const FusedRow& f, uint32_t* crow, int L, Meta* out, bool* viol) {
    *viol = false;
    if (f.status == 0) return true;
    if (s.status() != 1) return false;
    int e = f.ER;
    if (s.cy2) {
        crow[L - 1] = 0x80000000u;
        ++e;
    } else if (!(s.top >> 31)) {
        *viol = true;
    }
    *out = Meta{e, f.sR};
    return true;
}

} // namespace hk
