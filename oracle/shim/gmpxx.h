// oracle/shim/gmpxx.h — TEST INFRASTRUCTURE ONLY (oracle build of the reference).
//
// A small, self-written C++ value wrapper over the GMP C ABI declared in
// oracle/shim/gmp.h.  It exposes exactly the `mpz_class` / `mpq_class` surface
// the reference sources and tests use (SURVEY.md §8c lists it): construction
// from integers and decimal strings, + - * / % (truncating division, as the
// gmpxx documentation specifies for mpz_class), shifts, comparisons, abs / sgn /
// cmp, get_d / get_str / get_mpz_t, and the rational subset used by
// proj/tests/rational_oracle.hpp.  It is not GMP's own header and does not
// reproduce its expression-template machinery; every operation materialises a
// temporary, which is fine for an oracle.
#pragma once

#include "gmp.h"

#include <cstdlib>
#include <ostream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

class mpz_class {
public:
    mpz_class() { mpz_init(z_); }
    mpz_class(const mpz_class& o) { mpz_init_set(z_, o.z_); }
    mpz_class(mpz_class&& o) noexcept {
        mpz_init(z_);
        mpz_swap(z_, o.z_);
    }
    template <class T, std::enable_if_t<std::is_integral_v<T> && std::is_signed_v<T>, int> = 0>
    mpz_class(T v) { mpz_init_set_si(z_, long(v)); }
    template <class T, std::enable_if_t<std::is_integral_v<T> && !std::is_signed_v<T>, int> = 0>
    mpz_class(T v) { mpz_init_set_ui(z_, (unsigned long)(v)); }
    explicit mpz_class(const char* s, int base = 10) {
        if (mpz_init_set_str(z_, s, base) != 0) {
            mpz_clear(z_);
            throw std::invalid_argument("mpz_class: bad integer string");
        }
    }
    explicit mpz_class(const std::string& s, int base = 10) : mpz_class(s.c_str(), base) {}
    explicit mpz_class(mpz_srcptr p) { mpz_init_set(z_, p); }
    ~mpz_class() { mpz_clear(z_); }

    mpz_class& operator=(const mpz_class& o) {
        if (this != &o) mpz_set(z_, o.z_);
        return *this;
    }
    mpz_class& operator=(mpz_class&& o) noexcept {
        mpz_swap(z_, o.z_);
        return *this;
    }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_class& operator=(T v) {
        return *this = mpz_class(v);
    }

    mpz_ptr get_mpz_t() { return z_; }
    mpz_srcptr get_mpz_t() const { return z_; }
    double get_d() const { return mpz_get_d(z_); }
    long get_si() const { return mpz_get_si(z_); }
    std::string get_str(int base = 10) const {
        char* s = mpz_get_str(nullptr, base, z_);
        std::string out(s);
        std::free(s);
        return out;
    }

    mpz_class& operator+=(const mpz_class& o) { mpz_add(z_, z_, o.z_); return *this; }
    mpz_class& operator-=(const mpz_class& o) { mpz_sub(z_, z_, o.z_); return *this; }
    mpz_class& operator*=(const mpz_class& o) { mpz_mul(z_, z_, o.z_); return *this; }
    mpz_class& operator/=(const mpz_class& o) { mpz_tdiv_q(z_, z_, o.z_); return *this; }
    mpz_class& operator%=(const mpz_class& o) { mpz_tdiv_r(z_, z_, o.z_); return *this; }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_class& operator+=(T v) { return *this += mpz_class(v); }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_class& operator-=(T v) { return *this -= mpz_class(v); }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_class& operator*=(T v) { return *this *= mpz_class(v); }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_class& operator/=(T v) { return *this /= mpz_class(v); }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_class& operator<<=(T s) { mpz_mul_2exp(z_, z_, mp_bitcnt_t(s)); return *this; }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_class& operator>>=(T s) { mpz_fdiv_q_2exp(z_, z_, mp_bitcnt_t(s)); return *this; }
    mpz_class& operator++() { mpz_add_ui(z_, z_, 1); return *this; }
    mpz_class& operator--() { mpz_sub_ui(z_, z_, 1); return *this; }
    mpz_class operator++(int) { mpz_class t(*this); ++*this; return t; }
    mpz_class operator--(int) { mpz_class t(*this); --*this; return t; }
    mpz_class operator-() const { mpz_class t; mpz_neg(t.z_, z_); return t; }
    mpz_class operator+() const { return *this; }

private:
    mpz_t z_;
};

namespace gmpxx_shim_detail {
template <class T>
using if_int = std::enable_if_t<std::is_integral_v<T>, int>;
}

inline mpz_class operator+(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_add(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r; }
inline mpz_class operator-(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_sub(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r; }
inline mpz_class operator*(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_mul(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r; }
inline mpz_class operator/(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_tdiv_q(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r; }
inline mpz_class operator%(const mpz_class& a, const mpz_class& b) { mpz_class r; mpz_tdiv_r(r.get_mpz_t(), a.get_mpz_t(), b.get_mpz_t()); return r; }
inline int cmp(const mpz_class& a, const mpz_class& b) { return mpz_cmp(a.get_mpz_t(), b.get_mpz_t()); }
inline int sgn(const mpz_class& a) { return mpz_sgn(a.get_mpz_t()); }
inline mpz_class abs(const mpz_class& a) { mpz_class r; mpz_abs(r.get_mpz_t(), a.get_mpz_t()); return r; }

#define GMPXX_SHIM_MIXED(OP)                                                                              \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline auto operator OP(const mpz_class& a, T b) { return a OP mpz_class(b); }                         \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline auto operator OP(T a, const mpz_class& b) { return mpz_class(a) OP b; }
GMPXX_SHIM_MIXED(+)
GMPXX_SHIM_MIXED(-)
GMPXX_SHIM_MIXED(*)
GMPXX_SHIM_MIXED(/)
GMPXX_SHIM_MIXED(%)

template <class T, gmpxx_shim_detail::if_int<T> = 0>
inline mpz_class operator<<(const mpz_class& a, T s) { mpz_class r; mpz_mul_2exp(r.get_mpz_t(), a.get_mpz_t(), mp_bitcnt_t(s)); return r; }
template <class T, gmpxx_shim_detail::if_int<T> = 0>
inline mpz_class operator>>(const mpz_class& a, T s) { mpz_class r; mpz_fdiv_q_2exp(r.get_mpz_t(), a.get_mpz_t(), mp_bitcnt_t(s)); return r; }

#define GMPXX_SHIM_CMP(OP)                                                                                \
    inline bool operator OP(const mpz_class& a, const mpz_class& b) { return cmp(a, b) OP 0; }             \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline bool operator OP(const mpz_class& a, T b) { return cmp(a, mpz_class(b)) OP 0; }                 \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline bool operator OP(T a, const mpz_class& b) { return cmp(mpz_class(a), b) OP 0; }
GMPXX_SHIM_CMP(==)
GMPXX_SHIM_CMP(!=)
GMPXX_SHIM_CMP(<)
GMPXX_SHIM_CMP(<=)
GMPXX_SHIM_CMP(>)
GMPXX_SHIM_CMP(>=)

inline std::ostream& operator<<(std::ostream& os, const mpz_class& a) { return os << a.get_str(); }

// ---------------------------------------------------------------------------
class mpq_class {
public:
    mpq_class() { mpq_init(); }
    mpq_class(const mpq_class& o) { mpq_init(); __gmpq_set(q_, o.q_); }
    mpq_class(mpq_class&& o) noexcept { mpq_init(); __gmpq_swap(q_, o.q_); }
    mpq_class(const mpz_class& z) { mpq_init(); __gmpq_set_z(q_, z.get_mpz_t()); }
    template <class T, gmpxx_shim_detail::if_int<T> = 0>
    mpq_class(T v) : mpq_class(mpz_class(v)) {}
    // num/den, NOT canonicalised (gmpxx semantics); callers canonicalise.
    mpq_class(const mpz_class& n, const mpz_class& d) {
        mpq_init();
        mpz_set(&q_->_mp_num, n.get_mpz_t());
        mpz_set(&q_->_mp_den, d.get_mpz_t());
    }
    template <class A, class B, gmpxx_shim_detail::if_int<A> = 0, gmpxx_shim_detail::if_int<B> = 0>
    mpq_class(A n, B d) : mpq_class(mpz_class(n), mpz_class(d)) {}
    ~mpq_class() { __gmpq_clear(q_); }

    mpq_class& operator=(const mpq_class& o) { if (this != &o) __gmpq_set(q_, o.q_); return *this; }
    mpq_class& operator=(mpq_class&& o) noexcept { __gmpq_swap(q_, o.q_); return *this; }
    mpq_class& operator=(const mpz_class& z) { __gmpq_set_z(q_, z.get_mpz_t()); return *this; }
    template <class T, gmpxx_shim_detail::if_int<T> = 0>
    mpq_class& operator=(T v) { return *this = mpz_class(v); }

    void canonicalize() { __gmpq_canonicalize(q_); }
    mpq_ptr get_mpq_t() { return q_; }
    mpq_srcptr get_mpq_t() const { return q_; }
    double get_d() const { return __gmpq_get_d(q_); }
    std::string get_str(int base = 10) const {
        char* s = __gmpq_get_str(nullptr, base, q_);
        std::string out(s);
        std::free(s);
        return out;
    }

    mpq_class& operator+=(const mpq_class& o) { __gmpq_add(q_, q_, o.q_); return *this; }
    mpq_class& operator-=(const mpq_class& o) { __gmpq_sub(q_, q_, o.q_); return *this; }
    mpq_class& operator*=(const mpq_class& o) { __gmpq_mul(q_, q_, o.q_); return *this; }
    mpq_class& operator/=(const mpq_class& o) { __gmpq_div(q_, q_, o.q_); return *this; }
    mpq_class operator-() const { mpq_class t; __gmpq_neg(t.q_, q_); return t; }

private:
    void mpq_init() { __gmpq_init(q_); }
    mpq_t q_;
};

inline mpq_class operator+(const mpq_class& a, const mpq_class& b) { mpq_class r(a); r += b; return r; }
inline mpq_class operator-(const mpq_class& a, const mpq_class& b) { mpq_class r(a); r -= b; return r; }
inline mpq_class operator*(const mpq_class& a, const mpq_class& b) { mpq_class r(a); r *= b; return r; }
inline mpq_class operator/(const mpq_class& a, const mpq_class& b) { mpq_class r(a); r /= b; return r; }
inline int cmp(const mpq_class& a, const mpq_class& b) { return __gmpq_cmp(a.get_mpq_t(), b.get_mpq_t()); }
inline int sgn(const mpq_class& a) { return mpq_sgn(a.get_mpq_t()); }
inline mpq_class abs(const mpq_class& a) { mpq_class r; __gmpq_abs(r.get_mpq_t(), a.get_mpq_t()); return r; }

#define GMPXX_SHIM_QMIXED(OP)                                                                             \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline mpq_class operator OP(const mpq_class& a, T b) { return a OP mpq_class(b); }                    \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline mpq_class operator OP(T a, const mpq_class& b) { return mpq_class(a) OP b; }                    \
    inline mpq_class operator OP(const mpq_class& a, const mpz_class& b) { return a OP mpq_class(b); }     \
    inline mpq_class operator OP(const mpz_class& a, const mpq_class& b) { return mpq_class(a) OP b; }
GMPXX_SHIM_QMIXED(+)
GMPXX_SHIM_QMIXED(-)
GMPXX_SHIM_QMIXED(*)
GMPXX_SHIM_QMIXED(/)

#define GMPXX_SHIM_QCMP(OP)                                                                               \
    inline bool operator OP(const mpq_class& a, const mpq_class& b) { return cmp(a, b) OP 0; }             \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline bool operator OP(const mpq_class& a, T b) { return cmp(a, mpq_class(b)) OP 0; }                 \
    template <class T, gmpxx_shim_detail::if_int<T> = 0>                                                   \
    inline bool operator OP(T a, const mpq_class& b) { return cmp(mpq_class(a), b) OP 0; }
GMPXX_SHIM_QCMP(==)
GMPXX_SHIM_QCMP(!=)
GMPXX_SHIM_QCMP(<)
GMPXX_SHIM_QCMP(<=)
GMPXX_SHIM_QCMP(>)
GMPXX_SHIM_QCMP(>=)

inline std::ostream& operator<<(std::ostream& os, const mpq_class& a) { return os << a.get_str(); }
