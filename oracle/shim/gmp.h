/* oracle/shim/gmp.h — TEST INFRASTRUCTURE ONLY (oracle build of the reference).
 *
 * A minimal, self-written declaration of the subset of the GMP C ABI that the
 * reference (`/root/reference/proj/src/*.cpp`, `proj/tests/*.hpp`) calls.  The
 * container ships `libgmp.so.10` (the runtime) but no development headers, so
 * the reference cannot compile as shipped.  Only the struct
 * layout of the public ABI (x86-64: 64-bit limbs) and the exported `__gmpz_*` /
 * `__gmpq_*` entry points are declared here; the macros `mpz_sgn`,
 * `mpz_odd_p` and `mpq_sgn` are restated from the documented layout.
 *
 * GMP version: whatever `/usr/lib/x86_64-linux-gnu/libgmp.so.10` is (10.5.0 in
 * this image).  All integer operations the reference uses are exact, so the
 * results do not depend on the GMP version.
 */
#ifndef HANKEL_ORACLE_GMP_SHIM_H
#define HANKEL_ORACLE_GMP_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef unsigned long mp_bitcnt_t;
typedef long mp_exp_t;

typedef struct {
    int _mp_alloc;
    int _mp_size;
    mp_limb_t* _mp_d;
} __mpz_struct;

typedef struct {
    __mpz_struct _mp_num;
    __mpz_struct _mp_den;
} __mpq_struct;

typedef __mpz_struct mpz_t[1];
typedef __mpq_struct mpq_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;
typedef __mpq_struct* mpq_ptr;
typedef const __mpq_struct* mpq_srcptr;

/* ---- integers ---- */
void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_si(mpz_ptr, long);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
int __gmpz_init_set_str(mpz_ptr, const char*, int);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
int __gmpz_set_str(mpz_ptr, const char*, int);
void __gmpz_swap(mpz_ptr, mpz_ptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_add_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul_si(mpz_ptr, mpz_srcptr, long);
void __gmpz_mul_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_mul_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
unsigned long __gmpz_tdiv_q_ui(mpz_ptr, mpz_srcptr, unsigned long);
void __gmpz_tdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_fdiv_q_2exp(mpz_ptr, mpz_srcptr, mp_bitcnt_t);
void __gmpz_fdiv_qr(mpz_ptr, mpz_ptr, mpz_srcptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
int __gmpz_cmp_si(mpz_srcptr, long);
int __gmpz_cmp_ui(mpz_srcptr, unsigned long);
int __gmpz_tstbit(mpz_srcptr, mp_bitcnt_t);
mp_bitcnt_t __gmpz_scan1(mpz_srcptr, mp_bitcnt_t);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
char* __gmpz_get_str(char*, int, mpz_srcptr);
double __gmpz_get_d(mpz_srcptr);
double __gmpz_get_d_2exp(long*, mpz_srcptr);
long __gmpz_get_si(mpz_srcptr);
void __gmpz_fac_ui(mpz_ptr, unsigned long);
void __gmpz_sqrt(mpz_ptr, mpz_srcptr);

#define mpz_init __gmpz_init
#define mpz_init_set __gmpz_init_set
#define mpz_init_set_si __gmpz_init_set_si
#define mpz_init_set_ui __gmpz_init_set_ui
#define mpz_init_set_str __gmpz_init_set_str
#define mpz_clear __gmpz_clear
#define mpz_set __gmpz_set
#define mpz_set_si __gmpz_set_si
#define mpz_set_ui __gmpz_set_ui
#define mpz_set_str __gmpz_set_str
#define mpz_swap __gmpz_swap
#define mpz_add __gmpz_add
#define mpz_add_ui __gmpz_add_ui
#define mpz_sub __gmpz_sub
#define mpz_sub_ui __gmpz_sub_ui
#define mpz_mul __gmpz_mul
#define mpz_mul_si __gmpz_mul_si
#define mpz_mul_ui __gmpz_mul_ui
#define mpz_mul_2exp __gmpz_mul_2exp
#define mpz_neg __gmpz_neg
#define mpz_abs __gmpz_abs
#define mpz_tdiv_q __gmpz_tdiv_q
#define mpz_tdiv_r __gmpz_tdiv_r
#define mpz_tdiv_q_ui __gmpz_tdiv_q_ui
#define mpz_tdiv_q_2exp __gmpz_tdiv_q_2exp
#define mpz_fdiv_q_2exp __gmpz_fdiv_q_2exp
#define mpz_fdiv_qr __gmpz_fdiv_qr
#define mpz_cmp __gmpz_cmp
#define mpz_cmp_si __gmpz_cmp_si
#define mpz_cmp_ui __gmpz_cmp_ui
#define mpz_tstbit __gmpz_tstbit
#define mpz_scan1 __gmpz_scan1
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_get_str __gmpz_get_str
#define mpz_get_d __gmpz_get_d
#define mpz_get_d_2exp __gmpz_get_d_2exp
#define mpz_get_si __gmpz_get_si
#define mpz_fac_ui __gmpz_fac_ui
#define mpz_sqrt __gmpz_sqrt
/* documented-layout macros */
#define mpz_sgn(z) ((z)->_mp_size < 0 ? -1 : (z)->_mp_size > 0)
#define mpz_odd_p(z) ((z)->_mp_size != 0 && ((z)->_mp_d[0] & 1))

/* ---- rationals ---- */
void __gmpq_init(mpq_ptr);
void __gmpq_clear(mpq_ptr);
void __gmpq_set(mpq_ptr, mpq_srcptr);
void __gmpq_set_z(mpq_ptr, mpz_srcptr);
void __gmpq_set_si(mpq_ptr, long, unsigned long);
void __gmpq_swap(mpq_ptr, mpq_ptr);
void __gmpq_canonicalize(mpq_ptr);
void __gmpq_add(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_sub(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_mul(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_div(mpq_ptr, mpq_srcptr, mpq_srcptr);
void __gmpq_neg(mpq_ptr, mpq_srcptr);
void __gmpq_abs(mpq_ptr, mpq_srcptr);
int __gmpq_cmp(mpq_srcptr, mpq_srcptr);
int __gmpq_equal(mpq_srcptr, mpq_srcptr);
double __gmpq_get_d(mpq_srcptr);
char* __gmpq_get_str(char*, int, mpq_srcptr);

#define mpq_sgn(q) ((q)->_mp_num._mp_size < 0 ? -1 : (q)->_mp_num._mp_size > 0)

#ifdef __cplusplus
}
#endif

#endif
