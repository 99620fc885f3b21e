// host_math.cpp — host-side pieces of the path that the reference also runs on
// the host (compiled by g++, linked into libhankel_b200.so):
//
//  * exact moments (moments.cpp:80-111, the factorial path of gamma_exact):
//    a small schoolbook big integer, factorials by repeated small multiplies,
//    then the correctly rounded conversion to the p-bit float format;
//  * the small symmetric eigensolve (jacobi.cpp:27-103): cyclic Jacobi, but in
//    IEEE binary128 (113-bit significand) instead of binary64 so that lambda is
//    good to ~32 digits (the 20-digit target).
//  * assign_columns (ldlt.cpp:22-35).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <exception>
#include <thread>
#include <vector>

namespace hk_host {

using Big = std::vector<uint32_t>; // little-endian magnitude

static void big_mul_small(Big& a, uint32_t m) {
    uint64_t carry = 0;
    for (auto& w : a) {
        const uint64_t t = (uint64_t)w * m + carry;
        w = uint32_t(t);
        carry = t >> 32;
    }
    if (carry) a.push_back(uint32_t(carry));
}

static int big_bitlen(const Big& a) {
    for (int i = int(a.size()) - 1; i >= 0; --i)
        if (a[size_t(i)]) return i * 32 + (32 - __builtin_clz(a[size_t(i)]));
    return 0;
}

static bool big_bit(const Big& a, long b) {
    if (b < 0) return false;
    const size_t q = size_t(b >> 5);
    return q < a.size() && ((a[q] >> (b & 31)) & 1u);
}

// word w of (a >> shift) for any shift (negative: left shift), zero outside a
static uint32_t big_word_shr(const Big& a, long shift, long w) {
    const long b = shift + 32 * w; // bit of a that lands on bit 0 of word w
    const long q = b >= 0 ? b / 32 : -((-b + 31) / 32);
    const int r = int(b - 32 * q);
    auto word = [&](long i) -> uint64_t { return (i >= 0 && size_t(i) < a.size()) ? a[size_t(i)] : 0u; };
    const uint64_t two = word(q) | (word(q + 1) << 32);
    return uint32_t(two >> r);
}

// any bit of a below bit `b` set?
static bool big_sticky_below(const Big& a, long b) {
    if (b <= 0) return false;
    const size_t q = size_t(b >> 5);
    for (size_t i = 0; i < q && i < a.size(); ++i)
        if (a[i]) return true;
    const int r = int(b & 31);
    return r && q < a.size() && (a[q] & ((1u << r) - 1u));
}

// RNE of the positive integer `a` into `limbs` words; returns exp; sets exact.
// Word-shifted (the conversion is a shift plus one rounding increment).
static int big_to_mpf(const Big& a, int limbs, uint32_t* out, bool& exact) {
    const int p = 32 * limbs;
    const int nb = big_bitlen(a);
    std::fill(out, out + limbs, 0u);
    exact = true;
    if (nb == 0) return 0;
    const long shift = long(nb) - p; // out = a >> shift (shift may be negative)
    for (int w = 0; w < limbs; ++w) out[w] = big_word_shr(a, shift, w);
    if (shift > 0) {
        const bool rb = big_bit(a, shift - 1);
        const bool st = big_sticky_below(a, shift - 1);
        exact = !rb && !st;
        if (rb && (st || (out[0] & 1u))) {
            int i = 0;
            while (i < limbs && ++out[i] == 0u) ++i;
            if (i == limbs) { // overflow to 2^p
                out[limbs - 1] = 0x80000000u;
                return nb + 1;
            }
        }
    }
    return nb;
}

// ---- odd q = 2/beta (beta = 2, 2/3, 2/5, ...): Gamma at half-integers (moments.cpp:90-99)
//
// mu_k = (q/2) Gamma((k+1) q / 2).  For even (k+1) q the Gamma is a factorial and
// mu_k = q (n-1)! / 2 is exact.  For odd (k+1) q = 2n + 1,
//     mu_k = q (2n)! / (2 4^n n!) sqrt(pi) = A sqrt(pi) 2^(-2n-1),  A = q (n+1)(n+2)...(2n),
// which is irrational: the correctly rounded p-bit value is taken from
// S = floor(sqrt(pi) 2^P) (pi by Machin's formula, as pi_scaled, moments.cpp:36-44,
// then an integer square root) with a Ziv test on both ends of A [S - 1, S + 2],
// P raised until they round alike.  Host GMP (libgmp.so.10), as the reference.
extern "C" {
struct hk_mpz {
    int alloc, size;
    unsigned long* d;
};
void __gmpz_init(hk_mpz*);
void __gmpz_clear(hk_mpz*);
void __gmpz_set_ui(hk_mpz*, unsigned long);
void __gmpz_mul(hk_mpz*, const hk_mpz*, const hk_mpz*);
void __gmpz_mul_ui(hk_mpz*, const hk_mpz*, unsigned long);
void __gmpz_mul_2exp(hk_mpz*, const hk_mpz*, unsigned long);
void __gmpz_fdiv_q_2exp(hk_mpz*, const hk_mpz*, unsigned long);
void __gmpz_tdiv_q_ui(hk_mpz*, const hk_mpz*, unsigned long);
void __gmpz_add(hk_mpz*, const hk_mpz*, const hk_mpz*);
void __gmpz_sub(hk_mpz*, const hk_mpz*, const hk_mpz*);
void __gmpz_sqrt(hk_mpz*, const hk_mpz*);
size_t __gmpz_sizeinbase(const hk_mpz*, int);
void* __gmpz_export(void*, size_t*, int, size_t, int, size_t, const hk_mpz*);
}

namespace {
struct Z { // RAII mpz
    hk_mpz v;
    Z() { __gmpz_init(&v); }
    ~Z() { __gmpz_clear(&v); }
    Z(const Z&) = delete;
    Z& operator=(const Z&) = delete;
};

// sum_k (-1)^k 2^bits / ((2k+1) x^(2k+1)), each term truncated (error < number of terms)
void atan_recip_scaled(hk_mpz* out, unsigned long x, unsigned long bits) {
    Z term, t;
    __gmpz_set_ui(&term.v, 1);
    __gmpz_mul_2exp(&term.v, &term.v, bits);
    __gmpz_tdiv_q_ui(&term.v, &term.v, x);
    __gmpz_set_ui(out, 0);
    for (unsigned long k = 0; term.v.size != 0; ++k) {
        __gmpz_tdiv_q_ui(&t.v, &term.v, 2 * k + 1);
        if (k % 2 == 0)
            __gmpz_add(out, out, &t.v);
        else
            __gmpz_sub(out, out, &t.v);
        __gmpz_tdiv_q_ui(&term.v, &term.v, x * x);
    }
}

// floor(sqrt(pi) 2^P) to within a few units: pi 2^(2P) by Machin (64 guard bits), then isqrt
void sqrt_pi_scaled(hk_mpz* out, unsigned long P) {
    Z a, b;
    atan_recip_scaled(&a.v, 5, 2 * P + 64);
    atan_recip_scaled(&b.v, 239, 2 * P + 64);
    __gmpz_mul_ui(&a.v, &a.v, 16);
    __gmpz_mul_ui(&b.v, &b.v, 4);
    __gmpz_sub(&a.v, &a.v, &b.v);
    __gmpz_fdiv_q_2exp(&a.v, &a.v, 64);
    __gmpz_sqrt(out, &a.v);
}

Big to_big(const hk_mpz* z) {
    const size_t words = (__gmpz_sizeinbase(z, 2) + 31) / 32;
    Big out(words ? words : 1, 0u);
    size_t cnt = 0;
    __gmpz_export(out.data(), &cnt, -1, 4, 0, 0, z);
    out.resize(cnt ? cnt : 1);
    return out;
}
} // namespace

// RNE of the positive integer v to `limbs` words (big_to_mpf) — or report that v and
// v + width round differently (the Ziv test failed)
static bool round_both(const hk_mpz* lo, const hk_mpz* hi, int limbs, uint32_t* out, int* e) {
    std::vector<uint32_t> a(static_cast<size_t>(limbs)), b(static_cast<size_t>(limbs));
    bool ex = true;
    const int ea = big_to_mpf(to_big(lo), limbs, a.data(), ex);
    const int eb = big_to_mpf(to_big(hi), limbs, b.data(), ex);
    if (ea != eb || a != b) return false;
    std::copy(a.begin(), a.end(), out);
    *e = ea;
    return true;
}

static int odd_q_moments(unsigned long q, int count, int limbs, uint32_t* out_limbs, int32_t* out_exps,
                         int32_t* out_signs, int* exact, const char** why) {
    unsigned long P = 32ul * unsigned(limbs) + 96;
    Z S;
    sqrt_pi_scaled(&S.v, P);
    bool all_exact = true;
    for (int k = 0; k < count; ++k) {
        const unsigned long t2 = (unsigned long)(k + 1) * q; // 2 x the Gamma argument
        uint32_t* o = out_limbs + size_t(k) * limbs;
        out_signs[k] = 1;
        if (t2 % 2 == 0) { // mu = q (n-1)! / 2, exact
            Big f{1u};
            for (unsigned long t = 2; t + 1 <= t2 / 2; ++t) big_mul_small(f, uint32_t(t));
            big_mul_small(f, uint32_t(q));
            bool ex = true;
            out_exps[k] = big_to_mpf(f, limbs, o, ex) - 1;
            all_exact = all_exact && ex;
            continue;
        }
        const unsigned long n = (t2 - 1) / 2;
        Z A;
        __gmpz_set_ui(&A.v, q);
        for (unsigned long t = n + 1; t <= 2 * n; ++t) __gmpz_mul_ui(&A.v, &A.v, t);
        for (;;) { // value = A sqrt(pi) 2^(-2n-1), sqrt(pi) 2^P in [S - 1, S + 2]
            Z lo, hi, t;
            __gmpz_set_ui(&t.v, 1);
            __gmpz_sub(&t.v, &S.v, &t.v);
            __gmpz_mul(&lo.v, &A.v, &t.v);
            __gmpz_set_ui(&t.v, 2);
            __gmpz_add(&t.v, &S.v, &t.v);
            __gmpz_mul(&hi.v, &A.v, &t.v);
            int e = 0;
            if (round_both(&lo.v, &hi.v, limbs, o, &e)) {
                out_exps[k] = e - int(P) - int(2 * n + 1);
                break;
            }
            P += 128; // an end of the bracket rounds elsewhere: more digits of sqrt(pi)
            sqrt_pi_scaled(&S.v, P);
        }
        all_exact = false;
    }
    *exact = all_exact ? 1 : 0;
    (void)why;
    return 0;
}

} // namespace hk_host

extern "C" int hk_moments_impl(unsigned beta_num, unsigned beta_den, int count, int limbs, uint32_t* out_limbs,
                               int32_t* out_exps, int32_t* out_signs, int* exact, const char** why) {
    using namespace hk_host;
    if (beta_num == 0 || beta_den == 0 || (2ul * beta_den) % beta_num != 0) {
        *why = "unsupported beta: 2/beta must be a positive integer";
        return 3;
    }
    if (count < 1 || limbs < 1) {
        *why = "need count >= 1 and limbs >= 1";
        return 3;
    }
    const unsigned long q = 2ul * beta_den / beta_num; // doubled_inverse (moments.cpp:64-66)
    if (q % 2 != 0) return odd_q_moments(q, count, limbs, out_limbs, out_exps, out_signs, exact, why);
    // mu_k = (q/2) * ((k+1) q/2 - 1)!   (moments.cpp:83-89, 105-107)
    Big f{1u};
    unsigned long have = 0; // f == have!
    bool all_exact = true;
    for (int k = 0; k < count; ++k) {
        const unsigned long arg = (unsigned long)(k + 1) * q / 2 - 1;
        while (have < arg) { // two factors per pass while their product fits a word
            if (have + 2 <= arg && have + 2 < 65536) {
                big_mul_small(f, uint32_t((have + 1) * (have + 2)));
                have += 2;
            } else {
                big_mul_small(f, uint32_t(++have));
            }
        }
        Big scaled;
        const Big* mup = &f;
        if (q / 2 != 1) {
            scaled = f;
            big_mul_small(scaled, uint32_t(q / 2));
            mup = &scaled;
        }
        const Big& mu = *mup;
        bool ex = true;
        out_exps[k] = big_to_mpf(mu, limbs, out_limbs + size_t(k) * limbs, ex);
        out_signs[k] = 1;
        all_exact = all_exact && ex;
    }
    *exact = all_exact ? 1 : 0;
    return 0;
}

extern "C" int hk_assign_columns(int n, int workers, int32_t* owner) {
    if (n < 1 || workers < 1) return 3;
    for (int c = 0; c < n; ++c) {
        const int block = c / workers, r = c % workers;
        owner[c] = (block % 2 == 0) ? r : workers - 1 - r;
    }
    return 0;
}

// ------------------------------------------------------------ binary128 Jacobi

namespace {

using q128 = __float128;

q128 qabs(q128 x) { return x < 0 ? -x : x; }

q128 qsqrt(q128 x) {
    if (x <= 0) return 0;
    q128 s = std::sqrt((double)x);
    for (int it = 0; it < 3; ++it) s = (s + x / s) / 2;
    return s;
}

// Cyclic Jacobi, jacobi.cpp:27-72 line for line, in binary128.
std::vector<q128> jacobi_q(std::vector<q128> m, int k, double tol_factor, int max_sweeps) {
    auto at = [&](int i, int j) -> q128& { return m[size_t(i) * size_t(k) + size_t(j)]; };
    auto off = [&]() {
        q128 s = 0;
        for (int i = 0; i < k; ++i)
            for (int j = i + 1; j < k; ++j) s += 2 * at(i, j) * at(i, j);
        return qsqrt(s);
    };
    q128 fro = 0;
    for (auto v : m) fro += v * v;
    const q128 tol = q128(tol_factor) * qsqrt(fro);
    int sweep = 0;
    while (k > 1 && off() > tol) {
        if (++sweep > max_sweeps) throw std::runtime_error("jacobi_eigenvalues: no convergence after max sweeps");
        for (int p = 0; p < k - 1; ++p)
            for (int qq = p + 1; qq < k; ++qq) {
                const q128 apq = at(p, qq);
                if (apq == 0) continue;
                const q128 app = at(p, p), aqq = at(qq, qq);
                const q128 theta = (aqq - app) / (2 * apq);
                const q128 t = (theta >= 0 ? q128(1) : q128(-1)) / (qabs(theta) + qsqrt(theta * theta + 1));
                const q128 c = 1 / qsqrt(t * t + 1);
                const q128 s = t * c;
                at(p, p) = app - t * apq;
                at(qq, qq) = aqq + t * apq;
                at(p, qq) = 0;
                at(qq, p) = 0;
                for (int r = 0; r < k; ++r) {
                    if (r == p || r == qq) continue;
                    const q128 arp = at(r, p), arq = at(r, qq);
                    at(r, p) = c * arp - s * arq;
                    at(p, r) = at(r, p);
                    at(r, qq) = s * arp + c * arq;
                    at(qq, r) = at(r, qq);
                }
            }
    }
    std::vector<q128> ev(static_cast<size_t>(k));
    for (int i = 0; i < k; ++i) ev[size_t(i)] = at(i, i);
    std::sort(ev.begin(), ev.end());
    return ev;
}

// p-bit float -> binary128: top 128 bits, scaled (truncation below 2^-125 rel.)
q128 mpf_to_q(const uint32_t* d, int limbs, int exp, int sign) {
    if (sign == 0) return 0;
    unsigned __int128 top = 0;
    for (int i = 0; i < 4; ++i) {
        const int idx = limbs - 1 - i;
        top = (top << 32) | (idx >= 0 ? d[idx] : 0u);
    }
    // top = the leading 128 bits of M (zero padded): value ~= top 2^(exp - 128)
    q128 v = (q128)top;
    int e = exp - 128;
    while (e > 0) {
        const int s = std::min(e, 60);
        v *= (q128)(1ull << s);
        e -= s;
    }
    while (e < 0) {
        const int s = std::min(-e, 60);
        v /= (q128)(1ull << s);
        e += s;
    }
    return sign < 0 ? -v : v;
}

void split_dd(q128 v, double& hi, double& lo) {
    hi = (double)v;
    lo = (double)(v - (q128)hi);
}

} // namespace

// block: k*k MP floats (host SoA).  Fills s lambdas (hi/lo) and trunc errors.
extern "C" int hk_block_eigs_impl(int k, int limbs, const uint32_t* l, const int32_t* e, const int32_t* sg, int s,
                                  double* lam_hi, double* lam_lo, double* trunc, const char** why) {
    if (s < 1 || s > k) {
        *why = "smallest_eigs_of_H: need 1 <= s <= k";
        return 3;
    }
    try {
        std::vector<q128> M(size_t(k) * size_t(k));
        for (int i = 0; i < k * k; ++i) M[size_t(i)] = mpf_to_q(l + size_t(i) * limbs, limbs, e[i], sg[i]);
        const double tol = 1e-32;
        // the k and (k-1) blocks are independent solves: the second on its own thread
        // (software binary128 is slow: ~0.2 ms per 8x8 solve)
        std::vector<q128> mum;
        std::exception_ptr err2;
        std::thread t2;
        if (k > 1) {
            std::vector<q128> Mm(size_t(k - 1) * size_t(k - 1));
            for (int i = 0; i < k - 1; ++i)
                for (int j = 0; j < k - 1; ++j) Mm[size_t(i) * size_t(k - 1) + size_t(j)] = M[size_t(i) * size_t(k) + size_t(j)];
            t2 = std::thread([&, Mm = std::move(Mm)] {
                try {
                    mum = jacobi_q(Mm, k - 1, tol, 100);
                } catch (...) {
                    err2 = std::current_exception();
                }
            });
        }
        std::vector<q128> mu;
        try {
            mu = jacobi_q(M, k, tol, 100);
        } catch (...) {
            if (t2.joinable()) t2.join();
            throw;
        }
        if (t2.joinable()) t2.join();
        if (err2) std::rethrow_exception(err2);
        for (int i = 1; i <= s; ++i) {
            const q128 mi = mu[size_t(k - i)];
            if (mi <= 0) {
                *why = "smallest_eigs_of_H: non-positive block eigenvalue; the truncation is too aggressive or the "
                       "precision too small";
                return 1;
            }
            const q128 lam = 1 / mi;
            split_dd(lam, lam_hi[i - 1], lam_lo[i - 1]);
            trunc[i - 1] = i <= k - 1 ? (double)(lam - 1 / mum[size_t(k - 1 - i)]) : std::nan("");
        }
    } catch (const std::exception& ex) {
        static thread_local std::string msg;
        msg = ex.what();
        *why = msg.c_str();
        return 1;
    }
    return 0;
}

// jacobi_eigenvalues (jacobi.hpp:16-17; jacobi.cpp:27-72) on a host binary64
// block: the same cyclic sweep and stopping rule, carried in binary128, the
// ascending eigenvalues rounded to binary64.  No device.
extern "C" int hk_jacobi_eigenvalues(const double* m, int k, double tol_factor, int max_sweeps, double* out) {
    if (!m || !out || k < 1 || max_sweeps < 0) return 3;
    try {
        std::vector<q128> M(size_t(k) * size_t(k));
        for (size_t i = 0; i < M.size(); ++i) M[i] = m[i];
        const std::vector<q128> ev = jacobi_q(M, k, tol_factor, max_sweeps);
        for (int i = 0; i < k; ++i) out[i] = (double)ev[size_t(i)];
    } catch (const std::exception&) {
        return 1;
    }
    return 0;
}

// smallest_eigs_of_H (jacobi.hpp:29-30) on a host k x k MP block (no device).
extern "C" int hk_block_eigenvalues(int k, int limbs, const uint32_t* l, const int32_t* e, const int32_t* sg, int s,
                                    double* lam_hi, double* lam_lo, double* trunc) {
    if (k < 1 || limbs < 1 || !l || !e || !sg || !lam_hi || !lam_lo || !trunc) return 3;
    const char* why = "";
    return hk_block_eigs_impl(k, limbs, l, e, sg, s, lam_hi, lam_lo, trunc, &why);
}
