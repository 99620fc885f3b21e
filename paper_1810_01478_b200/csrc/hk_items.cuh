// hk_items.cuh — one warp-sized work item of each stage of the hot path.
//
// The CUDA kernels (kernels.cu) run these over grid-stride item ranges; the host
// emulator (tools/emu_mp.cpp) runs the very same functions on an emulated warp,
// so the index maps are tested on CPU too.
//
// HBM layout:
//   S  — the Hankel working matrix, jagged lower triangle, column-major: entry
//        (k, j), k >= j, at col_off(j) + (k - j), col_off(j) = j N - j (j-1)/2.
//        After step i, column i holds D_i at (i,i) and L(k,i) below it — the
//        in-place factor storage of ldlt.hpp:76-85 (L[j][r] = L(j+1+r, j)).
//   R  — R_i = RNE(1/D_i), N entries.  B — the quotient column B_i, N entries.
//   X  — first m columns of L^{-1}, row-major N x m (entry (r,c) valid c < min(r,m)).
//   Y  — X(l,c) R_l, N x m.  T / T2 — block-reduction tree buffers.
#pragma once

#include "mpf_ops.cuh"

namespace hk {

struct MpArr {
    uint32_t* d;
    Meta* m;
    HK_DEV uint32_t* limbs(long long e, int L) const { return d + e * (long long)L; }
};

HK_HD long long col_off(int j, int N) { return (long long)j * N - (long long)j * (j - 1) / 2; }
HK_HD long long tri_idx(int k, int j, int N) { return col_off(j, N) + (k - j); }

// Sharded L^{-1} (multi-GPU): rows are owned in 128-row blocks, block b by rank
// b % rw; the pivot column i of L arrives as a panel (rows i..N-1 at [j - i]).
constexpr int kRowBlock = 128;
HK_HD bool row_mine(int j, int rw, int rr) { return rw <= 1 || (j / kRowBlock) % rw == rr; }
HK_HD long long lcol_idx(int j, int i, int N, int panel) { return panel ? (long long)(j - i) : tri_idx(j, i, N); }

// w -> (j, k), 0 <= j <= k < n, column-major lower triangle of order n.
HK_DEV void tri_decode(long long w, int n, int& j, int& k) {
    const double b = 2.0 * n + 1.0;
    int jj = int((b - sqrt(b * b - 8.0 * double(w))) * 0.5);
    if (jj < 0) jj = 0;
    if (jj > n - 1) jj = n - 1;
    while (jj > 0 && col_off(jj, n) > w) --jj;
    while (jj + 1 < n && col_off(jj + 1, n) <= w) ++jj;
    j = jj;
    k = jj + int(w - col_off(jj, n));
}

HK_DEV void copy_entry(uint32_t* dst, Meta* dm, const uint32_t* src, const Meta* sm, int L) {
    for (int i = lane(); i < L; i += 32) dst[i] = src[i];
    if (lane() == 0) *dm = *sm;
    wsync();
}

// ---- S <- Hankel(mu): S(k,j) = mu_{k+j}
struct ItemInitS {
    MpArr S, mu;
    int N, L;
    HK_DEV void operator()(long long w, uint32_t*) const {
        int j, k;
        tri_decode(w, N, j, k);
        copy_entry(S.limbs(w, L), S.m + w, mu.limbs(k + j, L), mu.m + (k + j), L);
    }
};

// ---- R_i = RNE(1 / S_ii), pivot sign test (ldlt.cpp:111, 231-234, 280-284)
struct ItemRecip {
    MpArr S, R;
    int N, L, i;
    int* err;
    HK_DEV void operator()(long long, uint32_t* ws) const {
        if (*(volatile int*)err >= 0) return;
        const long long e = tri_idx(i, i, N);
        const Meta dm = S.m[e];
        if (dm.sign <= 0) {
            if (lane() == 0) atomicCAS_emu(err, i);
            return;
        }
        const Meta r = warp_recip(S.limbs(e, L), dm, R.limbs(i, L), L, recipws_carve(ws, L));
        if (lane() == 0) R.m[i] = r;
        wsync();
    }
    HK_DEV static void atomicCAS_emu(int* err, int i) {
#if defined(HK_WARP_EMU)
        if (*err < 0) *err = i;
#else
        atomicCAS(err, -1, i);
#endif
    }
};

// ---- B_i(k) = RNE(S(k,i) * R_i), k = i+1+t
struct ItemMulB {
    MpArr S, R, B;
    int N, L, i;
    const int* err;
    HK_DEV void operator()(long long t, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int k = i + 1 + int(t);
        const long long e = tri_idx(k, i, N);
        const Meta r = warp_mulr(S.limbs(e, L), S.m[e], R.limbs(i, L), R.m[i], B.limbs(k, L), L, opws_carve(ws, L));
        if (lane() == 0) B.m[k] = r;
        wsync();
    }
};

// ---- trailing update S(k,j) = RNE(S(k,j) - S(j,i) B_i(k)), jfirst <= j <= k < N
//      (ldlt.cpp:122-129, the hot loop; one MP-FMA per item).  Items enumerate
//      the column-major triangle of columns jfirst..N-1, so the first N-jfirst
//      items are exactly column jfirst: jfirst = i+1 with N-i-1 items is the
//      look-ahead column update (ldlt.cpp:274-277), jfirst = i+2 the bulk.
struct ItemTrailing {
    MpArr S, B;
    int N, L, i, jfirst;
    const int* err;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int n2 = N - jfirst;
        int jj, kk;
        tri_decode(w, n2, jj, kk);
        const int j = jfirst + jj, k = jfirst + kk;
        const long long ec = tri_idx(k, j, N), ex = tri_idx(j, i, N);
        uint32_t* c = S.limbs(ec, L);
        const Meta r = warp_fms(c, S.m[ec], S.limbs(ex, L), S.m[ex], B.limbs(k, L), B.m[k], c, L, opws_carve(ws, L));
        if (lane() == 0) S.m[ec] = r;
        wsync();
    }
};

// ---- the same bulk update with entries paired by row: columns j0, j0+1
//      (j0 = jfirst + 2q) share y = B_i(k) for k >= j0+1, so one warp does
//      both FMAs with one y stream (warp_fms2).  Items of pair q: index 0 is the
//      diagonal single (j0, j0), index r >= 1 the row k = j0 + r; an odd last
//      column (only row N-1) is one single item.  Same ops as ItemTrailing.
HK_HD long long pair_items(int n0, int q) { return (long long)q * n0 - (long long)q * (q - 1); }
HK_HD long long trailing2_items(int N, int jfirst) {
    const int n0 = N - jfirst;
    if (n0 <= 0) return 0;
    return pair_items(n0, n0 / 2) + (n0 & 1);
}

struct ItemTrailing2 {
    MpArr S, B;
    int N, L, i, jfirst;
    const int* err;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int n0 = N - jfirst, np = n0 / 2;
        int q = 0;
        if (w >= pair_items(n0, np)) {
            q = np; // odd last column: (N-1, N-1)
        } else {
            const double b = n0 + 1.0;
            q = int((b - sqrt(b * b - 4.0 * double(w))) * 0.5);
            if (q < 0) q = 0;
            if (q > np - 1) q = np - 1;
            while (q > 0 && pair_items(n0, q) > w) --q;
            while (q + 1 < np && pair_items(n0, q + 1) <= w) ++q;
        }
        const int j0 = jfirst + 2 * q;
        const int r = int(w - pair_items(n0, q));
        const long long ex0 = tri_idx(j0, i, N);
        if (q == np || r == 0) { // single: (j0, j0) or the odd last column
            const int k = j0;
            const long long ec = tri_idx(k, j0, N);
            uint32_t* c = S.limbs(ec, L);
            const Meta m = warp_fms(c, S.m[ec], S.limbs(ex0, L), S.m[ex0], B.limbs(k, L), B.m[k], c, L,
                                    opws_carve(ws, L));
            if (lane() == 0) S.m[ec] = m;
            wsync();
            return;
        }
        const int k = j0 + r;
        const long long ec0 = tri_idx(k, j0, N), ec1 = tri_idx(k, j0 + 1, N), ex1 = tri_idx(j0 + 1, i, N);
        uint32_t* c0 = S.limbs(ec0, L);
        uint32_t* c1 = S.limbs(ec1, L);
        Meta m0, m1;
        warp_fms2(c0, S.m[ec0], S.limbs(ex0, L), S.m[ex0], c1, S.m[ec1], S.limbs(ex1, L), S.m[ex1], B.limbs(k, L),
                  B.m[k], c0, c1, m0, m1, L, ws);
        if (lane() == 0) {
            S.m[ec0] = m0;
            S.m[ec1] = m1;
        }
        wsync();
    }
};

// ---- column i of S <- B_i (L(k,i) stored in place), k = i+1+t
struct ItemStoreL {
    MpArr S, B;
    int N, L, i;
    HK_DEV void operator()(long long t, uint32_t*) const {
        const int k = i + 1 + int(t);
        const long long e = tri_idx(k, i, N);
        copy_entry(S.limbs(e, L), S.m + e, B.limbs(k, L), B.m + k, L);
    }
};

// ---- L^{-1}: X(r,c) <- L(r,c) for c < min(r, m)   (init_work_rows, inversion.cpp:64-76)
struct ItemInvInit {
    MpArr S, X;
    int N, L, m;
    int zero = 0; // sharded: all zero (column c of X is set at step c before any use)
    HK_DEV void operator()(long long w, uint32_t*) const {
        const int r = int(w / m), c = int(w % m);
        const long long dst = (long long)r * m + c;
        if (c < r && !zero) {
            const long long e = tri_idx(r, c, N);
            copy_entry(X.limbs(dst, L), X.m + dst, S.limbs(e, L), S.m + e, L);
        } else {
            for (int q = lane(); q < L; q += 32) X.limbs(dst, L)[q] = 0u;
            if (lane() == 0) X.m[dst] = Meta{0, 0};
            wsync();
        }
    }
};

// ---- L^{-1} row elimination step i (inversion.cpp:93-102):
//      X(j,c) = RNE(X(j,c) - L(j,i) X(i,c)) for j > i, c < min(m,i);  X(j,i) = -L(j,i) if i < m
struct ItemInvStep {
    MpArr S, X;
    int N, L, m, i;
    int panel = 0, rw = 1, rr = 0; // sharded: L(:, i) from the panel S, this rank's rows only
    const int* err = nullptr;      // steps interleaved with the LDLT: nothing to do once a pivot failed
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (err && *(volatile const int*)err >= 0) return;
        const int b = i < m ? i : m;
        const long long nfma = (long long)(N - i - 1) * b;
        if (w < nfma) {
            const int j = i + 1 + int(w / b), c = int(w % b);
            if (!row_mine(j, rw, rr)) return;
            const long long el = lcol_idx(j, i, N, panel);
            const long long xc = (long long)j * m + c, xi = (long long)i * m + c;
            uint32_t* o = X.limbs(xc, L);
            const Meta r = warp_fms(o, X.m[xc], S.limbs(el, L), S.m[el], X.limbs(xi, L), X.m[xi], o, L,
                                    opws_carve(ws, L));
            if (lane() == 0) X.m[xc] = r;
            wsync();
        } else {
            const int j = i + 1 + int(w - nfma);
            if (!row_mine(j, rw, rr)) return;
            const long long el = lcol_idx(j, i, N, panel);
            const long long xd = (long long)j * m + i;
            copy_entry(X.limbs(xd, L), X.m + xd, S.limbs(el, L), S.m + el, L);
            if (lane() == 0) X.m[xd].sign = -X.m[xd].sign;
            wsync();
        }
    }
};

// ---- block: Y(l,c) = X(l,c) R_l (c < l), R_l (c == l), 0 (c > l)
struct ItemBlockY {
    MpArr X, R, Y;
    int N, L, m;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        const int l = int(w / m), c = int(w % m);
        uint32_t* o = Y.limbs(w, L);
        if (c < l) {
            const Meta r = warp_mulr(X.limbs(w, L), X.m[w], R.limbs(l, L), R.m[l], o, L, opws_carve(ws, L));
            if (lane() == 0) Y.m[w] = r;
            wsync();
        } else if (c == l) {
            copy_entry(o, Y.m + w, R.limbs(l, L), R.m + l, L);
        } else {
            for (int q = lane(); q < L; q += 32) o[q] = 0u;
            if (lane() == 0) Y.m[w] = Meta{0, 0};
            wsync();
        }
    }
};

// pair q -> (j, c), j <= c < k, row-major upper triangle
HK_DEV void pair_decode(int q, int k, int& j, int& c) {
    int jj = 0, rem = q;
    while (rem >= k - jj) {
        rem -= k - jj;
        ++jj;
    }
    j = jj;
    c = jj + rem;
}

// ---- block terms: T[q][l] = X(l,j) Y(l,c) for l in [c, N), zero elsewhere
//      (inversion.cpp:253-257: one product and one division by D_l per term)
struct ItemBlockTerms {
    MpArr X, Y, T;
    int N, L, m, k, size;
    int rw = 1, rr = 0; // sharded: this rank's rows only (the others' terms are exact zeros)
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        const int q = int(w / size), l = int(w % size);
        int j, c;
        pair_decode(q, k, j, c);
        uint32_t* o = T.limbs(w, L);
        if (l >= c && l < N && row_mine(l, rw, rr)) {
            const long long yi = (long long)l * m + c;
            if (l == j) {
                copy_entry(o, T.m + w, Y.limbs(yi, L), Y.m + yi, L);
            } else {
                const long long xi = (long long)l * m + j;
                const Meta r = warp_mulr(X.limbs(xi, L), X.m[xi], Y.limbs(yi, L), Y.m[yi], o, L, opws_carve(ws, L));
                if (lane() == 0) T.m[w] = r;
                wsync();
            }
        } else {
            for (int t = lane(); t < L; t += 32) o[t] = 0u;
            if (lane() == 0) T.m[w] = Meta{0, 0};
            wsync();
        }
    }
};

// ---- one level of the fixed pairwise tree: T2[q][t] = T[q][2t] + T[q][2t+1]
struct ItemTreeLevel {
    MpArr T, T2;
    int L, half;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        const long long q = w / half, t = w % half;
        const long long a = q * 2 * half + 2 * t, b = a + 1;
        const Meta r = warp_addr(T.limbs(a, L), T.m[a], T.limbs(b, L), T.m[b], T2.limbs(w, L), L, opws_carve(ws, L));
        if (lane() == 0) T2.m[w] = r;
        wsync();
    }
};

// ---- tree roots -> symmetric k x k block M (row-major)
struct ItemBlockOut {
    MpArr T, M;
    int L, k;
    HK_DEV void operator()(long long q, uint32_t*) const {
        int j, c;
        pair_decode(int(q), k, j, c);
        const long long a = (long long)j * k + c, b = (long long)c * k + j;
        copy_entry(M.limbs(a, L), M.m + a, T.limbs(q, L), T.m + q, L);
        if (a != b) copy_entry(M.limbs(b, L), M.m + b, T.limbs(q, L), T.m + q, L);
    }
};

// ======================================================================
// Sharded (multi-GPU) LDLT: rank r stores only the columns it owns under the
// boustrophedon map (ldlt.cpp:22-35), concatenated; entry e of the local
// storage is (row erow[e], column ecol[e]).  The pivot column i is held by
// every rank in `panel` (rows i..N-1 at panel[0..N-i)), published by its owner
// each step (ldlt.cpp:294-298 / 248 -> ncclBroadcast).

// local S <- Hankel(mu)
struct ItemDInit {
    MpArr S, mu;
    const int* erow;
    const int* ecol;
    int L;
    HK_DEV void operator()(long long e, uint32_t*) const {
        const int k = erow[e], j = ecol[e];
        copy_entry(S.limbs(e, L), S.m + e, mu.limbs(k + j, L), mu.m + (k + j), L);
    }
};

// step-i update of local entries [e0, e0 + n): S(k,j) -= panel_i(j) B_i(k)
struct ItemDTrailing {
    MpArr S, panel, B;
    const int* erow;
    const int* ecol;
    int L, i;
    long long e0;
    const int* err;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const long long e = e0 + w;
        const int k = erow[e], j = ecol[e];
        uint32_t* c = S.limbs(e, L);
        const Meta r = warp_fms(c, S.m[e], panel.limbs(j - i, L), panel.m[j - i], B.limbs(k, L), B.m[k], c, L,
                                opws_carve(ws, L));
        if (lane() == 0) S.m[e] = r;
        wsync();
    }
};

// R_i = RNE(1/panel[0]) with the pivot test
struct ItemDRecip {
    MpArr panel, R;
    int L, i;
    int* err;
    HK_DEV void operator()(long long, uint32_t* ws) const {
        if (*(volatile int*)err >= 0) return;
        const Meta dm = panel.m[0];
        if (dm.sign <= 0) {
            if (lane() == 0) ItemRecip::atomicCAS_emu(err, i);
            return;
        }
        const Meta r = warp_recip(panel.limbs(0, L), dm, R.limbs(i, L), L, recipws_carve(ws, L));
        if (lane() == 0) R.m[i] = r;
        wsync();
    }
};

// B_i(k) = RNE(panel_i(k) R_i), k = i+1+t
struct ItemDMulB {
    MpArr panel, R, B;
    int L, i;
    const int* err;
    HK_DEV void operator()(long long t, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int k = i + 1 + int(t);
        const Meta r = warp_mulr(panel.limbs(k - i, L), panel.m[k - i], R.limbs(i, L), R.m[i], B.limbs(k, L), L,
                                 opws_carve(ws, L));
        if (lane() == 0) B.m[k] = r;
        wsync();
    }
};

// contiguous entry copy dst[d0 + t] <- src[s0 + t]
struct ItemCopy {
    MpArr dst, src;
    long long d0, s0;
    int L;
    HK_DEV void operator()(long long t, uint32_t*) const {
        copy_entry(dst.limbs(d0 + t, L), dst.m + d0 + t, src.limbs(s0 + t, L), src.m + s0 + t, L);
    }
};

// ======================================================================
// CTA-cooperative items (one item per CTA) for the latency-bound critical path
// of the look-ahead: column update -> reciprocal -> B column.

HK_DEV void cta_meta_store(Meta* dst, Meta v) {
    if (cta_tid() == 0) *dst = v;
    cta_sync();
}

struct CItemRecip { // R_i = RNE(1/S_ii) with the pivot sign test
    MpArr S, R;
    int N, L, i;
    int* err;
    HK_DEV void operator()(long long, uint32_t* ws) const {
        if (*(volatile int*)err >= 0) return;
        const long long e = tri_idx(i, i, N);
        const Meta dm = S.m[e];
        if (dm.sign <= 0) {
            if (cta_tid() == 0) ItemRecip::atomicCAS_emu(err, i);
            return;
        }
        cta_meta_store(R.m + i, cta_recip(S.limbs(e, L), dm, R.limbs(i, L), L, ws));
    }
};

struct CItemMulB { // B_i(k) = RNE(S(k,i) R_i), k = i+k0+t
    MpArr S, R, B;
    int N, L, i;
    const int* err;
    int k0 = 1;
    HK_DEV void operator()(long long t, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int k = i + k0 + int(t);
        const long long e = tri_idx(k, i, N);
        cta_meta_store(B.m + k, cta_mulr(S.limbs(e, L), S.m[e], R.limbs(i, L), R.m[i], B.limbs(k, L), L,
                                         ctaws_carve(ws, L)));
    }
};

struct CItemColUpd { // look-ahead column j = i+1: S(k,j) = RNE(S(k,j) - S(j,i) B_i(k)), k = j+k0+t
    MpArr S, B;
    int N, L, i;
    const int* err;
    int k0 = 0; // 0: from the diagonal; 1: the off-diagonal part only
    HK_DEV void operator()(long long t, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int j = i + 1, k = j + k0 + int(t);
        const long long ec = tri_idx(k, j, N), ex = tri_idx(j, i, N);
        uint32_t* c = S.limbs(ec, L);
        cta_meta_store(S.m + ec, cta_fms(c, S.m[ec], S.limbs(ex, L), S.m[ex], B.limbs(k, L), B.m[k], c, L,
                                         ctaws_carve(ws, L)));
    }
};

struct CItemDRecip { // sharded: R_i from the panel
    MpArr panel, R;
    int L, i;
    int* err;
    HK_DEV void operator()(long long, uint32_t* ws) const {
        if (*(volatile int*)err >= 0) return;
        const Meta dm = panel.m[0];
        if (dm.sign <= 0) {
            if (cta_tid() == 0) ItemRecip::atomicCAS_emu(err, i);
            return;
        }
        cta_meta_store(R.m + i, cta_recip(panel.limbs(0, L), dm, R.limbs(i, L), L, ws));
    }
};

struct CItemDMulB { // sharded: B_i(k) = RNE(panel_i(k) R_i)
    MpArr panel, R, B;
    int L, i;
    const int* err;
    HK_DEV void operator()(long long t, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int k = i + 1 + int(t);
        cta_meta_store(B.m + k, cta_mulr(panel.limbs(k - i, L), panel.m[k - i], R.limbs(i, L), R.m[i], B.limbs(k, L),
                                         L, ctaws_carve(ws, L)));
    }
};

// sharded look-ahead (ldlt.cpp:274-277 on the owner of column j = i+1): the
// column's step-i update is written straight into the next panel, which is what
// gets broadcast: pnext(r) = RNE(S(j+r, j) - panel_i(1) B_i(j+r)), r = k0 + t.
// The local column keeps its step-(i-1) values until ItemDStoreL(j).
struct CItemDColUpd {
    MpArr S, panel, B, pnext;
    long long offj; // local entry of (j, j)
    int L, i;
    const int* err;
    int k0 = 0;
    HK_DEV void operator()(long long t, uint32_t* ws) const {
        if (*(volatile const int*)err >= 0) return;
        const int j = i + 1, r = k0 + int(t);
        const long long ec = offj + r;
        cta_meta_store(pnext.m + r, cta_fms(S.limbs(ec, L), S.m[ec], panel.limbs(1, L), panel.m[1], B.limbs(j + r, L),
                                            B.m[j + r], pnext.limbs(r, L), L, ctaws_carve(ws, L)));
    }
};

// sharded StoreL of owned column j: S(j,j) <- panel_j(0) = D_j, S(j+t, j) <- B_j(j+t)
struct ItemDStoreL {
    MpArr S, panel, B;
    long long offj;
    int L, j;
    HK_DEV void operator()(long long t, uint32_t*) const {
        if (t == 0)
            copy_entry(S.limbs(offj, L), S.m + offj, panel.limbs(0, L), panel.m, L);
        else
            copy_entry(S.limbs(offj + t, L), S.m + offj + t, B.limbs(j + t, L), B.m + j + t, L);
    }
};

// L^{-1} step i with one CTA per item (the step is latency-bound: N sequential
// steps of at most (N-i-1) min(m,i) independent FMAs) — same ops as ItemInvStep.
struct CItemInvStep {
    MpArr S, X;
    int N, L, m, i;
    const int* err = nullptr;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        if (err && *(volatile const int*)err >= 0) return;
        const int b = i < m ? i : m;
        const long long nfma = (long long)(N - i - 1) * b;
        if (w < nfma) {
            const int j = i + 1 + int(w / b), c = int(w % b);
            const long long el = tri_idx(j, i, N);
            const long long xc = (long long)j * m + c, xi = (long long)i * m + c;
            uint32_t* o = X.limbs(xc, L);
            cta_meta_store(X.m + xc, cta_fms(o, X.m[xc], S.limbs(el, L), S.m[el], X.limbs(xi, L), X.m[xi], o, L,
                                             ctaws_carve(ws, L)));
        } else {
            const int j = i + 1 + int(w - nfma);
            const long long el = tri_idx(j, i, N);
            const long long xd = (long long)j * m + i;
            for (int q = cta_tid(); q < L; q += cta_threads()) X.limbs(xd, L)[q] = S.limbs(el, L)[q];
            if (cta_tid() == 0) X.m[xd] = Meta{S.m[el].exp, -S.m[el].sign};
            cta_sync();
        }
    }
};

struct CItemBatch { // the CTA ops on batches (tests)
    MpArr A, B, C, O;
    int L, op;
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        Meta r;
        if (op == 0)
            r = cta_fms(C.limbs(w, L), C.m[w], A.limbs(w, L), A.m[w], B.limbs(w, L), B.m[w], O.limbs(w, L), L,
                        ctaws_carve(ws, L));
        else if (op == 1)
            r = cta_mulr(A.limbs(w, L), A.m[w], B.limbs(w, L), B.m[w], O.limbs(w, L), L, ctaws_carve(ws, L));
        else
            r = cta_recip(A.limbs(w, L), A.m[w], O.limbs(w, L), L, ws);
        cta_meta_store(O.m + w, r);
    }
};

// ---- generic batch ops (parity tests of the arithmetic itself)
struct ItemBatch {
    MpArr A, B, C, O;
    int L, op; // 0 fms: O = C - A*B; 1 mul: O = A*B; 2 add: O = A + B; 3 recip: O = 1/A
    HK_DEV void operator()(long long w, uint32_t* ws) const {
        Meta r;
        if (op == 0)
            r = warp_fms(C.limbs(w, L), C.m[w], A.limbs(w, L), A.m[w], B.limbs(w, L), B.m[w], O.limbs(w, L), L,
                         opws_carve(ws, L));
        else if (op == 1)
            r = warp_mulr(A.limbs(w, L), A.m[w], B.limbs(w, L), B.m[w], O.limbs(w, L), L, opws_carve(ws, L));
        else if (op == 2)
            r = warp_addr(A.limbs(w, L), A.m[w], B.limbs(w, L), B.m[w], O.limbs(w, L), L, opws_carve(ws, L));
        else
            r = warp_recip(A.limbs(w, L), A.m[w], O.limbs(w, L), L, recipws_carve(ws, L));
        if (lane() == 0) O.m[w] = r;
        wsync();
    }
};

} // namespace hk
