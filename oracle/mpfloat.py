"""oracle/mpfloat.py — TEST INFRASTRUCTURE ONLY: the bit-exact specification of
the product's p-bit multiprecision float and of the operation sequence its GPU
kernels perform.  Written with exact Python integers; used by tests to check
the CUDA path bit for bit, and never imported by the product.

Number format (include/hankel_b200.h):

    value = sign * M * 2**(e - p),   2**(p-1) <= M < 2**p,  p = 32 * L

``sign`` in {-1, 0, +1} (0 <=> value 0, then M = 0, e = 0).  ``e`` is the
binary exponent with 2**(e-1) <= |value| < 2**e.

Every arithmetic operation is the correctly rounded (round-to-nearest,
ties-to-even) image of its exact result:

    fms(c, x, y) = RNE(c - x*y)            (the MP-FMA of the LDLT update)
    mul(x, y)    = RNE(x*y)
    add(x, y)    = RNE(x + y)
    recip(d)     = RNE(1/d)

Because every op is correctly rounded, the result of each op is a function of
its inputs only, so the GPU result is bit-identical to this model regardless
of thread mapping, blocking, look-ahead order or GPU count.

The operation sequence of the product path (restating the reference's
algorithm, /root/reference/proj/src/ldlt.cpp:91-135, inversion.cpp:78-104 and
:232-262, in float arithmetic):

    LDLT step i:   R_i = recip(S_ii);  B_i(k) = mul(S_ki, R_i)   (k > i)
                   D_i = S_ii;  L(k,i) = B_i(k)
                   S_kj = fms(S_kj, S_ji, B_i(k))               (i < j <= k)
    L^{-1}:        X(j,c) = L(j,c) for c < min(j, m); for i ascending, j > i:
                   f = L(j,i); X(j,c) = fms(X(j,c), f, X(i,c)) (c < min(m, i));
                   X(j,i) = -f (i < m)
    block:         Y(l,c) = mul(X(l,c), R_l);  t_l = mul(X(l,j), Y(l,c))
                   M(j,c) = pairwise-tree sum over l in [0, 2^ceil(log2 N))
                            of t_l (t_l = 0 for l < max(j,c) or l >= N),
                            every node add() -- a fixed tree, so identical on
                            any GPU count.
"""
from __future__ import annotations

from fractions import Fraction


class MPF:
    __slots__ = ("s", "m", "e")

    def __init__(self, s: int, m: int, e: int):
        self.s, self.m, self.e = s, m, e

    def __eq__(self, o):
        return isinstance(o, MPF) and (self.s, self.m, self.e) == (o.s, o.m, o.e)

    def __repr__(self):
        return f"MPF({self.s}, 0x{self.m:x}, {self.e})"

    def to_fraction(self, p: int) -> Fraction:
        if self.s == 0:
            return Fraction(0)
        sh = self.e - p
        v = Fraction(self.m << sh) if sh >= 0 else Fraction(self.m, 1 << (-sh))
        return v if self.s > 0 else -v

    def neg(self) -> "MPF":
        return MPF(-self.s, self.m, self.e)


ZERO = MPF(0, 0, 0)


def round_scaled(n: int, scale: int, p: int) -> MPF:
    """RNE_p of the exact value n * 2**scale (n any integer)."""
    if n == 0:
        return ZERO
    s = 1 if n > 0 else -1
    a = abs(n)
    nb = a.bit_length()
    if nb <= p:
        m = a << (p - nb)
    else:
        d = nb - p
        m = a >> d
        rem = a & ((1 << d) - 1)
        half = 1 << (d - 1)
        if rem > half or (rem == half and (m & 1)):
            m += 1
            if m == 1 << p:
                m >>= 1
                nb += 1
    return MPF(s, m, scale + nb)


def from_int(n: int, p: int) -> MPF:
    return round_scaled(n, 0, p)


def from_fraction(fr: Fraction, p: int) -> MPF:
    """Correctly rounded conversion of an exact rational."""
    if fr == 0:
        return ZERO
    s = 1 if fr > 0 else -1
    a = abs(fr)
    num, den = a.numerator, a.denominator
    # choose shift so that the quotient has at least p+2 bits
    sh = p + 2 - (num.bit_length() - den.bit_length())
    if sh >= 0:
        q, r = divmod(num << sh, den)
    else:
        q, r = divmod(num, den << (-sh))
    # q has p+2 or p+3 bits; fold the remainder into a sticky bit below
    q = (q << 1) | (1 if r else 0)
    out = round_scaled(q, -sh - 1, p)
    return MPF(s, out.m, out.e) if out.s else out


def _exact(x: MPF, p: int):
    """(integer, scale) with value = integer * 2**scale."""
    return (x.s * x.m, x.e - p)


def fms(c: MPF, x: MPF, y: MPF, p: int) -> MPF:
    """RNE(c - x*y)."""
    nc, sc = _exact(c, p)
    nx, sx = _exact(x, p)
    ny, sy = _exact(y, p)
    npr, spr = nx * ny, sx + sy
    if npr == 0:
        return c if c.s != 0 else ZERO
    if nc == 0:
        return round_scaled(-npr, spr, p)
    lo = min(sc, spr)
    return round_scaled((nc << (sc - lo)) - (npr << (spr - lo)), lo, p)


def mul(x: MPF, y: MPF, p: int) -> MPF:
    nx, sx = _exact(x, p)
    ny, sy = _exact(y, p)
    return round_scaled(nx * ny, sx + sy, p)


def add(x: MPF, y: MPF, p: int) -> MPF:
    nx, sx = _exact(x, p)
    ny, sy = _exact(y, p)
    if nx == 0:
        return y if y.s else ZERO
    if ny == 0:
        return x
    lo = min(sx, sy)
    return round_scaled((nx << (sx - lo)) + (ny << (sy - lo)), lo, p)


def recip(d: MPF, p: int) -> MPF:
    """RNE(1/d) exactly: 1/(M 2^(e-p)) = 2^(p-e) / M."""
    if d.s == 0:
        raise ZeroDivisionError("recip of zero")
    # quotient with p+2 bits: 2^(2p+1) / M has p+1 or p+2 bits
    q, r = divmod(1 << (2 * p + 1), d.m)
    q = (q << 1) | (1 if r else 0)
    out = round_scaled(q, -(2 * p + 1) - 1 - (d.e - p), p)
    return MPF(d.s, out.m, out.e)


# ------------------------------------------------------------ the path


def ldlt(mu: list[int], n: int, p: int):
    """Float LDLT in the product's exact op order.  Returns (D, L, R) with
    L[i] = [L(i+1,i), ..., L(n-1,i)] and R[i] = recip(D[i])."""
    S = [[from_int(mu[i + j], p) for i in range(j, n)] for j in range(n)]
    D, L, R = [None] * n, [None] * n, [None] * n
    for i in range(n):
        col = S[i]
        piv = col[0]
        if piv.s <= 0:
            raise ArithmeticError(f"LDLT pivot <= 0 at column {i}")
        r = recip(piv, p)
        B = [mul(col[t], r, p) for t in range(1, n - i)]
        D[i], L[i], R[i] = piv, B, r
        for j in range(i + 1, n):
            x = col[j - i]
            cj = S[j]
            for k in range(j, n):
                cj[k - j] = fms(cj[k - j], x, B[k - i - 1], p)
        S[i] = None
    return D, L, R


def invert_L_partial(L, n: int, m: int, p: int):
    """X rows: X[r] = first min(r, m) entries of row r of L^{-1}."""
    def l_entry(r, c):
        return L[c][r - c - 1]

    X = [[l_entry(r, c) for c in range(min(r, m))] for r in range(n)]
    for i in range(n):
        bound = min(m, i)
        xi = X[i]
        for j in range(i + 1, n):
            f = l_entry(j, i)
            xj = X[j]
            for c in range(bound):
                xj[c] = fms(xj[c], f, xi[c], p)
            if i < m:
                xj[i] = f.neg()
    return X


ONE_CACHE: dict[int, MPF] = {}


def one(p: int) -> MPF:
    if p not in ONE_CACHE:
        ONE_CACHE[p] = from_int(1, p)
    return ONE_CACHE[p]


def tree_sum(terms: list[MPF], p: int) -> MPF:
    """Pairwise tree over a zero-padded power-of-two list."""
    size = 1
    while size < len(terms):
        size *= 2
    cur = list(terms) + [ZERO] * (size - len(terms))
    while len(cur) > 1:
        cur = [add(cur[2 * t], cur[2 * t + 1], p) for t in range(len(cur) // 2)]
    return cur[0]


def block(X, R, n: int, k: int, p: int):
    """k x k block of H^{-1} (row-major, symmetric) in the product's op order."""
    def xv(l, c):
        if l == c:
            return one(p)
        if c > l:
            return ZERO
        return X[l][c]

    Y = [[mul(xv(l, c), R[l], p) if c <= l else ZERO for c in range(k)] for l in range(n)]
    M = [None] * (k * k)
    for j in range(k):
        for c in range(j, k):
            lo = max(j, c)
            terms = [mul(xv(l, j), Y[l][c], p) if l >= lo else ZERO for l in range(n)]
            v = tree_sum(terms, p)
            M[j * k + c] = v
            M[c * k + j] = v
    return M
