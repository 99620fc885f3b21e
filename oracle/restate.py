"""oracle/restate.py — TEST INFRASTRUCTURE ONLY: a CPU restatement of the
reference algorithm (fixed point on Python integers), used as the checker.

Nothing in the product imports this module.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg may use it.

It restates, line by line, the reference's semantics (paths relative to
``/root/reference/proj``):

* ``round_shift_even``  — src/fixedpoint.cpp:10-23
* ``div_round_even``    — src/fixedpoint.cpp:25-35
* ``fix_div``           — src/fixedpoint.cpp:71-84 (FixScalar::div)
* ``fix_truncate``      — src/fixedpoint.cpp:86-92
* ``submul_rounded``    — src/fixedpoint.cpp:146-154
* ``pi_scaled`` / ``sqrt_pi_scaled`` — src/moments.cpp:17-50
* ``gamma_exact`` / ``moment`` — src/moments.cpp:80-111
* ``decompose_serial``  — src/ldlt.cpp:91-135
* ``assign_columns``    — src/ldlt.cpp:22-35
* ``invert_L_partial_serial`` — src/inversion.cpp:78-104
* ``assemble_block_fixed`` — src/inversion.cpp:232-262 WITHOUT the binary64
  cast at :258 (keeps the exact fixed-point sums)
* ``jacobi_eigenvalues`` / ``smallest_eigs_of_H`` — src/jacobi.cpp:27-103

A fixed-point value is the pair ``(mantissa, frac_bits)`` meaning
``mantissa / 2**frac_bits`` (proj/include/hankel/fixedpoint.hpp:10-27).

Pinning: tests/test_oracle.py checks this module bit-for-bit against the
reference itself (oracle/_ref/ref_driver, built from /root/reference by
oracle/Makefile) and against the reference tests' known answers.
"""
from __future__ import annotations

import math
from fractions import Fraction

# ---------------------------------------------------------------- fixedpoint


def round_shift_even(m: int, shift: int) -> int:
    """RNE of m / 2**shift, sign-magnitude (fixedpoint.cpp:10-23)."""
    if shift == 0 or m == 0:
        return m
    neg = m < 0
    a = -m if neg else m
    half_bit = (a >> (shift - 1)) & 1
    exact_half = half_bit and (a & ((1 << (shift - 1)) - 1)) == 0
    q = a >> shift
    if half_bit and (not exact_half or (q & 1)):
        q += 1
    return -q if neg else q


def div_round_even(num: int, den: int) -> int:
    """RNE of num/den (fixedpoint.cpp:25-35)."""
    if den == 0:
        raise ZeroDivisionError("fixed-point div: zero divisor")
    n, d = abs(num), abs(den)
    q, r = divmod(n, d)
    r <<= 1
    if r > d or (r == d and (q & 1)):
        q += 1
    if (num < 0) != (den < 0):
        q = -q
    return q


def fix_div(a, b, out_frac: int):
    """FixScalar::div (fixedpoint.cpp:71-84): correctly rounded quotient."""
    (ma, fa), (mb, fb) = a, b
    if mb == 0:
        raise ZeroDivisionError("fixed-point div: zero divisor")
    e = out_frac + fb - fa
    num, den = (ma << e, mb) if e >= 0 else (ma, mb << (-e))
    return (div_round_even(num, den), out_frac)


def fix_truncate(a, new_frac: int):
    """FixScalar::truncate (fixedpoint.cpp:86-92)."""
    m, f = a
    if new_frac > f or new_frac < 0:
        raise ValueError("truncate: need 0 <= new frac_bits <= current")
    return (round_shift_even(m, f - new_frac), new_frac)


def submul_rounded(acc, x, y):
    """acc -= RNE(x*y reduced to acc.frac_bits) (fixedpoint.cpp:146-154)."""
    (mc, fc), (mx, fx), (my, fy) = acc, x, y
    shift = fx + fy - fc
    if shift < 0:
        raise ValueError("submul_rounded: product carries fewer frac bits than target")
    return (mc - round_shift_even(mx * my, shift), fc)


def fix_to_fraction(a) -> Fraction:
    return Fraction(a[0], 1 << a[1])


# ---------------------------------------------------------------- moments


def _arctan_recip_scaled(x: int, frac_bits: int) -> int:
    """moments.cpp:17-31 (termwise truncation toward zero, as mpz '/')."""
    term = (1 << frac_bits) // x
    x2 = x * x
    s = 0
    k = 0
    while term != 0:
        t = term // (2 * k + 1)
        s = s + t if k % 2 == 0 else s - t
        term //= x2
        k += 1
    return s


def pi_scaled(frac_bits: int) -> int:
    """moments.cpp:35-42: Machin with 64 guard bits, then RNE."""
    guard = 64
    p = 16 * _arctan_recip_scaled(5, frac_bits + guard) - 4 * _arctan_recip_scaled(239, frac_bits + guard)
    return round_shift_even(p, guard)


def sqrt_pi_scaled(frac_bits: int) -> int:
    """moments.cpp:44-50: floor(sqrt(pi) 2^frac_bits)."""
    return math.isqrt(pi_scaled(2 * frac_bits))


def doubled_inverse(beta: tuple[int, int]) -> int:
    """WeightSpec::doubled_inverse / make (moments.cpp:64-78): q = 2/beta."""
    num, den = beta
    if num == 0 or den == 0:
        raise ValueError("beta must be positive")
    if (2 * den) % num != 0:
        raise ValueError("unsupported beta: 2/beta must be a positive integer")
    return 2 * den // num


def gamma_exact(arg_times_2: int, frac_bits: int):
    """moments.cpp:80-100."""
    if arg_times_2 == 0:
        raise ValueError("gamma argument must be positive")
    if arg_times_2 % 2 == 0:
        return (math.factorial(arg_times_2 // 2 - 1) << frac_bits, frac_bits)
    n = (arg_times_2 - 1) // 2
    guard = 64
    num = math.factorial(2 * n) * sqrt_pi_scaled(frac_bits + guard)
    den = math.factorial(n) << (2 * n + guard)
    return (div_round_even(num, den), frac_bits)


def moment(beta: tuple[int, int], k: int, frac_bits: int):
    """mu_k = (1/beta) Gamma((k+1)/beta) (moments.cpp:102-111)."""
    q = doubled_inverse(beta)
    g = gamma_exact((k + 1) * q, frac_bits)
    if q % 2 == 0:
        return (g[0] * (q // 2), frac_bits)
    return (round_shift_even(g[0] * q, 1), frac_bits)


def moment_integer(beta: tuple[int, int], k: int) -> int:
    """Exact integer mu_k when 2/beta is even (the factorial path, moments.cpp:83-89, 105-107)."""
    q = doubled_inverse(beta)
    if q % 2:
        raise ValueError("moment is not an integer for this beta")
    return math.factorial((k + 1) * q // 2 - 1) * (q // 2)


# ---------------------------------------------------------------- LDLT


def assign_columns(n: int, workers: int) -> list[int]:
    """Boustrophedon ownership (ldlt.cpp:22-35)."""
    if n < 1 or workers < 1:
        raise ValueError("assign_columns: need n >= 1 and workers >= 1")
    out = []
    for c in range(n):
        block, r = divmod(c, workers)
        out.append(r if block % 2 == 0 else workers - 1 - r)
    return out


class PrecisionError(RuntimeError):
    """hankel::precision_error (errors.hpp:10-13)."""


def decompose_serial(beta, n: int, K: int):
    """Right-looking LDLT at 2K fractional bits (ldlt.cpp:91-135).

    Returns (D, L, update_count) with D[i] and L[j][r] = L(j+1+r, j) as
    (mantissa, K) pairs (ldlt.hpp:76-85).
    """
    WK = 2 * K
    mu = [moment(beta, k, K)[0] for k in range(2 * n - 1)]
    # working_column(j, WK) (moments.cpp:122-129): align K -> 2K exactly
    A = [[(mu[i + j] << (WK - K)) for i in range(j, n)] for j in range(n)]
    D, L = [None] * n, [None] * n
    updates = 0
    for i in range(n):
        ai = A[i]
        piv = ai[0]
        if piv <= 0:
            raise PrecisionError(f"LDLT pivot <= 0 at column {i}: matrix not positive definite at K={K} "
                                 "fractional bits, increase the precision")
        B = [fix_div((ai[j - i], WK), (piv, WK), WK)[0] for j in range(i + 1, n)]
        D[i] = round_shift_even(piv, WK - K)
        L[i] = [round_shift_even(b, WK - K) for b in B]
        for j in range(i + 1, n):
            mult = ai[j - i]
            aj = A[j]
            for k in range(j, n):
                aj[k - j] -= round_shift_even(mult * B[k - i - 1], WK)
            updates += n - j
        A[i] = None
    return D, L, updates


def l_entry(L, row: int, col: int) -> int:
    return L[col][row - col - 1]


def invert_L_partial_serial(L, n: int, m: int, K: int):
    """First m columns of L^{-1} at K bits by in-place row elimination
    (inversion.cpp:78-104).  rows[r] = first min(r, m) mantissas of row r."""
    if m < 1 or m > n:
        raise ValueError("invert_L_partial: need 1 <= m <= n")
    work = [[l_entry(L, r, c) for c in range(min(r, m))] for r in range(n)]
    for i in range(n):
        bound = min(m, i)
        rowi = work[i]
        for j in range(i + 1, n):
            target = work[j]
            f = target[i] if i < m else l_entry(L, j, i)
            if i < m:
                target[i] = -f
            for k in range(bound):
                target[k] -= round_shift_even(f * rowi[k], K)  # submul_rounded at K
    return work


def assemble_block_fixed(Linv, D, n: int, k: int, K: int):
    """k x k block of H^{-1} in fixed point at 2K (inversion.cpp:244-257, no :258 cast).

    Returns the symmetric block as a flat row-major list of mantissas at 2K."""
    WK = 2 * K
    one = 1 << K
    for d in D:
        if d == 0:
            raise PrecisionError("assemble_truncated_inverse: zero pivot in D")

    def lv(l, col):
        return one if l == col else Linv[l][col]

    M = [0] * (k * k)
    for j in range(k):
        for c in range(j, k):
            acc = 0
            for l in range(max(j, c), n):
                prod = lv(l, j) * lv(l, c)  # frac 2K, exact
                acc += fix_div((prod, 2 * K), (D[l], K), WK)[0]
            M[j * k + c] = acc
            M[c * k + j] = acc
    return M


def fix_to_double(m: int, f: int) -> float:
    """FixScalar::to_double (fixedpoint.cpp:102-118)."""
    if m == 0:
        return 0.0
    neg = m < 0
    a = -m if neg else m
    bits = a.bit_length()
    exp2 = -f
    if bits > 53:
        s = bits - 53
        a = round_shift_even(a, s)
        exp2 += s
    d = math.ldexp(float(a), exp2)
    if math.isinf(d):
        raise OverflowError("fixed-point value exceeds binary64 range")
    return -d if neg else d


# ---------------------------------------------------------------- jacobi


def jacobi_eigenvalues(m: list[float], k: int, tol_factor: float = 1e-14, max_sweeps: int = 100):
    """Cyclic Jacobi in binary64 (jacobi.cpp:27-72)."""
    m = list(m)

    def at(i, j):
        return m[i * k + j]

    def off():
        return math.sqrt(sum(2 * at(i, j) * at(i, j) for i in range(k) for j in range(i + 1, k)))

    tol = tol_factor * math.sqrt(sum(v * v for v in m))
    sweep = 0
    while k > 1 and off() > tol:
        sweep += 1
        if sweep > max_sweeps:
            raise RuntimeError("jacobi_eigenvalues: no convergence after max sweeps")
        for p in range(k - 1):
            for q in range(p + 1, k):
                apq = at(p, q)
                if apq == 0.0:
                    continue
                app, aqq = at(p, p), at(q, q)
                theta = (aqq - app) / (2.0 * apq)
                t = (1.0 if theta >= 0 else -1.0) / (abs(theta) + math.sqrt(theta * theta + 1.0))
                c = 1.0 / math.sqrt(t * t + 1.0)
                s = t * c
                m[p * k + p] = app - t * apq
                m[q * k + q] = aqq + t * apq
                m[p * k + q] = 0.0
                m[q * k + p] = 0.0
                for r in range(k):
                    if r == p or r == q:
                        continue
                    arp, arq = at(r, p), at(r, q)
                    m[r * k + p] = c * arp - s * arq
                    m[p * k + r] = m[r * k + p]
                    m[r * k + q] = s * arp + c * arq
                    m[q * k + r] = m[r * k + q]
    return sorted(m[i * k + i] for i in range(k))


def smallest_eigs_of_H(M: list[float], k: int, s: int):
    """jacobi.cpp:74-103: lambda_i = 1/mu_{k+1-i}, trunc_err vs the (k-1) block."""
    mu = jacobi_eigenvalues(M, k)
    mu_minus = []
    if k > 1:
        Mm = [M[i * k + j] for i in range(k - 1) for j in range(k - 1)]
        mu_minus = jacobi_eigenvalues(Mm, k - 1)
    lam, err = [], []
    for i in range(1, s + 1):
        mi = mu[k - i]
        if mi <= 0:
            raise RuntimeError("smallest_eigs_of_H: non-positive block eigenvalue")
        lam.append(1.0 / mi)
        err.append(1.0 / mi - 1.0 / mu_minus[k - 1 - i] if i <= k - 1 else float("nan"))
    return lam, err


# ---------------------------------------------------------------- high precision eigen (oracle side)


def block_eigs_mp(block_fracs, k: int, dps: int = 60):
    """Eigenvalues (ascending) of an exact rational k x k symmetric block at `dps` digits.

    The 20-digit lambda needs the fixed-point block before the binary64 cast
    (SURVEY.md §0.3); mpmath's symmetric eigensolver at dps digits does it."""
    import mpmath

    with mpmath.workdps(dps):
        A = mpmath.matrix(k, k)
        for i in range(k):
            for j in range(k):
                fr = block_fracs[i * k + j]
                A[i, j] = mpmath.mpf(fr.numerator) / fr.denominator
        ev = mpmath.eigsy(A, eigvals_only=True)
        return sorted(ev)


def pipeline_fixed(beta, n: int, K: int, k: int):
    """Whole reference path in fixed point (pipeline.cpp:26-72 without timers)."""
    k = min(k, n)
    D, L, upd = decompose_serial(beta, n, K)
    Linv = invert_L_partial_serial(L, n, k, K)
    M = assemble_block_fixed(Linv, D, n, k, K)
    return D, L, Linv, M, upd
