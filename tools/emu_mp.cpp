// tools/emu_mp.cpp — host lockstep-warp emulation of the device MP arithmetic
// and of the per-item stage functions (test infrastructure, CPU only).
//
// Runs the SAME source as the sm_100a kernels (csrc/mpf_warp.cuh, mpf_ops.cuh,
// hk_items.cuh compiled with -DHK_WARP_EMU) so that the carry-lookahead,
// alignment/sticky and rounding logic, and the stage index maps, are checked
// against oracle/mpfloat.py without a GPU (tests/test_emu.py).
//
// stdin protocol (all numbers decimal except limbs, which are hex):
//   op <fms|mul|add|recip> <L> <count>       then count items of 3/2/2/1 operands
//   path <L> <N> <m>                        then 2N-1 moments
//   fused <L> <count>                       then count (c, x, y) triples: the
//       tensor-core short product (byte columns from limb L-8, as k_tc_bulk
//       forms it) streamed through FusedRow (csrc/tc_fused.cuh) in drain order;
//       prints the result, or "fb" when the item goes to the exact redo
// operand line: "<sign> <exp> <limb0> ... <limb L-1>"
// Output: one operand line per result (op), or for `path`: D (N lines), the
// L^{-1} rows (N*m lines, row-major), the block (m*m lines), then "err <col>".
#define HK_WARP_EMU 1
#include "../paper_1810_01478_b200/csrc/hk_items.cuh"
#include "../paper_1810_01478_b200/csrc/tc_fused.cuh"

#include <cstdio>
#include <iostream>
#include <string>
#include <vector>

using namespace hk;

struct HostArr {
    std::vector<uint32_t> d;
    std::vector<Meta> m;
    HostArr(long long n, int L) : d(size_t(n) * L, 0u), m(size_t(n), Meta{0, 0}) {}
    MpArr view() { return MpArr{d.data(), m.data()}; }
};

static void read_opd(HostArr& a, long long e, int L) {
    int s, ex;
    std::cin >> s >> ex;
    a.m[e] = Meta{ex, s};
    for (int i = 0; i < L; ++i) {
        std::string h;
        std::cin >> h;
        a.d[size_t(e) * L + i] = uint32_t(std::stoul(h, nullptr, 16));
    }
}

static void print_opd(const HostArr& a, long long e, int L) {
    std::printf("%d %d", a.m[e].sign, a.m[e].exp);
    for (int i = 0; i < L; ++i) std::printf(" %x", a.d[size_t(e) * L + i]);
    std::printf("\n");
}

template <class F>
static void run_items(long long n, int ws_words, const F& f) {
    std::vector<uint32_t> ws(size_t(ws_words) + 64, 0xdeadbeefu);
    hk_emu::run_warp([&] {
        for (long long w = 0; w < n; ++w) f(w, ws.data());
    });
}

static int ws_words_for(int L) {
    const int a = opws_words(L), b = recipws_words(L);
    return a > b ? a : b;
}

int main() {
    std::string cmd;
    while (std::cin >> cmd) {
        if (cmd == "op") {
            std::string op;
            int L;
            long long cnt;
            std::cin >> op >> L >> cnt;
            HostArr A(cnt, L), B(cnt, L), C(cnt, L), O(cnt, L);
            // c-prefixed ops run the CTA-cooperative variants (a 1-warp CTA here)
            const bool cta = op.size() > 1 && op[0] == 'c';
            const std::string base = cta ? op.substr(1) : op;
            int code = base == "fms" ? 0 : base == "mul" ? 1 : base == "add" ? 2 : 3;
            hk::force_exact_recip() = (base == "recipx"); // recip with the exact midpoint test forced
            for (long long e = 0; e < cnt; ++e) {
                if (code == 0) {
                    read_opd(C, e, L);
                    read_opd(A, e, L);
                    read_opd(B, e, L);
                } else if (code == 3) {
                    read_opd(A, e, L);
                } else {
                    read_opd(A, e, L);
                    read_opd(B, e, L);
                }
            }
            if (cta) {
                const int ws = ctaws_words(L) > ctarecipws_words(L) ? ctaws_words(L) : ctarecipws_words(L);
                run_items(cnt, ws, CItemBatch{A.view(), B.view(), C.view(), O.view(), L, code == 3 ? 2 : code});
            } else {
                run_items(cnt, ws_words_for(L), ItemBatch{A.view(), B.view(), C.view(), O.view(), L, code});
            }
            for (long long e = 0; e < cnt; ++e) print_opd(O, e, L);
        } else if (cmd == "fused") {
            int L;
            long long cnt;
            std::cin >> L >> cnt;
            HostArr Cc(cnt, L), X(cnt, L), Y(cnt, L);
            for (long long e = 0; e < cnt; ++e) {
                read_opd(Cc, e, L);
                read_opd(X, e, L);
                read_opd(Y, e, L);
            }
            const int nb = 4 * L, T0 = 4 * L - 32, nl = L + 8;
            for (long long e = 0; e < cnt; ++e) {
                const uint8_t* xb = reinterpret_cast<const uint8_t*>(&X.d[size_t(e) * L]);
                const uint8_t* yb = reinterpret_cast<const uint8_t*>(&Y.d[size_t(e) * L]);
                // short product: column sums t >= T0, carried into limbs (the epilogue's conversion)
                std::vector<uint32_t> P(size_t(nl) + 8, 0u);
                uint64_t carry = 0;
                for (int q = 0; q < 4 * nl; q += 4) {
                    uint64_t sum = carry;
                    for (int h = 0; h < 4; ++h) {
                        const int t = T0 + q + h;
                        uint64_t col = 0;
                        for (int u = 0; u < nb; ++u)
                            if (t - u >= 0 && t - u < nb) col += uint64_t(yb[u]) * xb[t - u];
                        sum += col << (8 * h);
                    }
                    P[size_t(q / 4)] = uint32_t(sum);
                    carry = sum >> 32;
                }
                const uint32_t* xl = &X.d[size_t(e) * L];
                const uint32_t* yl = &Y.d[size_t(e) * L];
                auto top64 = [&](const uint32_t* l) { return (uint64_t(l[L - 1]) << 32) | (L > 1 ? l[L - 2] : 0u); };
                std::vector<uint32_t> cl(Cc.d.begin() + e * L, Cc.d.begin() + (e + 1) * L);
                FusedRow fr;
                fr.setup(cl.data(), Cc.m[size_t(e)], top64(xl), X.m[size_t(e)], top64(yl), Y.m[size_t(e)], L);
                int g = 0;
                for (; g < (nl + 7) / 8; ++g) {
                    uint32_t pl[8];
                    for (int t = 0; t < 8; ++t) pl[t] = P[size_t(8 * g + t)];
                    if (fr.status == 1) fr.group(g, pl);
                }
                const uint32_t zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                while (fr.wants(g)) fr.group(g++, zero);
                Meta mo{0, 0};
                bool viol = false;
                const bool ok = fr.finish(&mo, &viol);
                if (viol) std::printf("viol\n");
                else if (!ok) std::printf("fb %d\n", fr.why);
                else if (fr.status == 0) print_opd(Cc, e, L);
                else {
                    std::printf("%d %d", mo.sign, mo.exp);
                    for (int i = 0; i < L; ++i) std::printf(" %x", cl[size_t(i)]);
                    std::printf("\n");
                }
            }
        } else if (cmd == "fusedw") { // the warp-cooperative stream (csrc/tc_fused.cuh warp_row_*), 32 items per warp
            int L;
            long long cnt;
            std::cin >> L >> cnt;
            HostArr Cc(cnt, L), X(cnt, L), Y(cnt, L);
            for (long long e = 0; e < cnt; ++e) {
                read_opd(Cc, e, L);
                read_opd(X, e, L);
                read_opd(Y, e, L);
            }
            const int nb = 4 * L, T0 = 4 * L - 32, nl = L + 8, nch = (nl + 63) / 64;
            std::vector<std::string> out(static_cast<size_t>(cnt));
            for (long long w0 = 0; w0 < cnt; w0 += 32) {
                // per row: the short product as k_tc_bulk forms it, in chunks of 64 limbs
                std::vector<std::vector<uint32_t>> P(32, std::vector<uint32_t>(size_t(64) * (nch + 64), 0u));
                std::vector<std::vector<uint32_t>> crow(32, std::vector<uint32_t>(size_t(L), 0u));
                for (int r = 0; r < 32 && w0 + r < cnt; ++r) {
                    const long long e = w0 + r;
                    const uint8_t* xb = reinterpret_cast<const uint8_t*>(&X.d[size_t(e) * L]);
                    const uint8_t* yb = reinterpret_cast<const uint8_t*>(&Y.d[size_t(e) * L]);
                    uint64_t carry = 0;
                    for (int q = 0; q < 4 * nl; q += 4) {
                        uint64_t sum = carry;
                        for (int h = 0; h < 4; ++h) {
                            const int t = T0 + q + h;
                            uint64_t col = 0;
                            for (int u = 0; u < nb; ++u)
                                if (t - u >= 0 && t - u < nb) col += uint64_t(yb[u]) * xb[t - u];
                            sum += col << (8 * h);
                        }
                        P[size_t(r)][size_t(q / 4)] = uint32_t(sum);
                        carry = sum >> 32;
                    }
                    std::copy(Cc.d.begin() + e * L, Cc.d.begin() + (e + 1) * L, crow[size_t(r)].begin());
                }
                std::vector<int> stat(32, 0), why(32, 0);
                std::vector<Meta> mo(32, Meta{0, 0});
                std::vector<char> okv(32, 1), viol(32, 0); // not vector<bool>: lanes write concurrently
                hk_emu::run_warp([&] {
                    const int ln = hk::lane();
                    const long long e = w0 + ln;
                    FusedRow fr;
                    if (e < cnt) {
                        auto top64 = [&](const uint32_t* l) { return (uint64_t(l[L - 1]) << 32) | (L > 1 ? l[L - 2] : 0u); };
                        fr.setup(crow[size_t(ln)].data(), Cc.m[size_t(e)], top64(&X.d[size_t(e) * L]), X.m[size_t(e)],
                                 top64(&Y.d[size_t(e) * L]), Y.m[size_t(e)], L);
                    }
                    WarpRowState own = warp_row_init(fr);
                    for (int c = 0;; ++c) {
                        bool any = false;
                        for (int rr = 0; rr < 32; ++rr) {
                            WarpRowState b = warp_row_bcast(own, rr);
                            if (b.status() != 1) continue;
                            const int Qp = int(b.prm & 0xffffu);
                            if (64 * c - 1 - Qp >= L) continue; // row complete
                            any = true;
                            const uint32_t p0 = P[size_t(rr)][size_t(64 * c + 2 * ln)];
                            const uint32_t p1 = P[size_t(rr)][size_t(64 * c + 2 * ln + 1)];
                            uint32_t q0, q1;
                            warp_row_load(b, crow[size_t(rr)].data(), L, c, q0, q1);
                            warp_row_chunk(b, crow[size_t(rr)].data(), L, c, p0, p1, q0, q1);
                            if (ln == rr) own = b;
                        }
                        if (!any && c >= nch) break;
                    }
                    Meta m{0, 0};
                    bool v = false;
                    const bool ok = warp_row_finish(own, fr, crow[size_t(ln)].data(), L, &m, &v);
                    stat[size_t(ln)] = fr.status;
                    okv[size_t(ln)] = ok;
                    viol[size_t(ln)] = v;
                    mo[size_t(ln)] = m;
                    why[size_t(ln)] = fr.why;
                });
                for (int r = 0; r < 32 && w0 + r < cnt; ++r) {
                    const long long e = w0 + r;
                    char buf[64];
                    if (viol[size_t(r)]) out[size_t(e)] = "viol";
                    else if (!okv[size_t(r)]) {
                        std::snprintf(buf, sizeof buf, "fb %d", why[size_t(r)]);
                        out[size_t(e)] = buf;
                    } else {
                        const Meta m = stat[size_t(r)] == 0 ? Cc.m[size_t(e)] : mo[size_t(r)];
                        std::string ln = std::to_string(m.sign) + " " + std::to_string(m.exp);
                        for (int i = 0; i < L; ++i) {
                            std::snprintf(buf, sizeof buf, " %x", crow[size_t(r)][size_t(i)]);
                            ln += buf;
                        }
                        out[size_t(e)] = ln;
                    }
                }
            }
            for (auto& o : out) std::printf("%s\n", o.c_str());
        } else if (cmd == "path") {
            int L, N, m;
            std::cin >> L >> N >> m;
            HostArr mu(2 * N - 1, L);
            for (int e = 0; e < 2 * N - 1; ++e) read_opd(mu, e, L);
            const long long ntri = (long long)N * (N + 1) / 2;
            HostArr S(ntri, L), R(N, L), Bq(N, L), X((long long)N * m, L), Y((long long)N * m, L);
            int err = -1;
            const int ws = ws_words_for(L);
            run_items(ntri, ws, ItemInitS{S.view(), mu.view(), N, L});
            for (int i = 0; i < N && err < 0; ++i) {
                run_items(1, ws, ItemRecip{S.view(), R.view(), N, L, i, &err});
                if (err >= 0) break;
                const int nb = N - i - 1;
                run_items(nb, ws, ItemMulB{S.view(), R.view(), Bq.view(), N, L, i, &err});
                // paired bulk kernel (ItemTrailing2) as the device path runs it
                const int ws2 = opws2_words(L) > ws ? opws2_words(L) : ws;
                run_items(trailing2_items(N, i + 1), ws2, ItemTrailing2{S.view(), Bq.view(), N, L, i, i + 1, &err});
                run_items(nb, ws, ItemStoreL{S.view(), Bq.view(), N, L, i});
            }
            if (err < 0) {
                run_items((long long)N * m, ws, ItemInvInit{S.view(), X.view(), N, L, m});
                for (int i = 0; i < N; ++i) {
                    const int b = i < m ? i : m;
                    const long long items = (long long)(N - i - 1) * b + (i < m ? N - i - 1 : 0);
                    run_items(items, ws, ItemInvStep{S.view(), X.view(), N, L, m, i});
                }
                run_items((long long)N * m, ws, ItemBlockY{X.view(), R.view(), Y.view(), N, L, m});
                int size = 1;
                while (size < N) size *= 2;
                const int k = m, npair = k * (k + 1) / 2;
                HostArr T((long long)npair * size, L), T2((long long)npair * size, L), M((long long)k * k, L);
                run_items((long long)npair * size, ws, ItemBlockTerms{X.view(), Y.view(), T.view(), N, L, m, k, size});
                HostArr* cur = &T;
                HostArr* nxt = &T2;
                for (int half = size / 2; half >= 1; half /= 2) {
                    run_items((long long)npair * half, ws, ItemTreeLevel{cur->view(), nxt->view(), L, half});
                    std::swap(cur, nxt);
                }
                run_items(npair, ws, ItemBlockOut{cur->view(), M.view(), L, k});
                for (int i = 0; i < N; ++i) print_opd(S, tri_idx(i, i, N), L);
                for (long long e = 0; e < (long long)N * m; ++e) print_opd(X, e, L);
                for (long long e = 0; e < (long long)k * k; ++e) print_opd(M, e, L);
            }
            std::printf("err %d\n", err);
        }
        std::fflush(stdout);
    }
    return 0;
}
