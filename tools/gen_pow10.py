"""Generate the 10^k table (k = -300 .. 324, step 8; 64-bit significand rounded
to nearest, binary exponent) that the shortest-digit double printer of the
reference's JSON writer uses (Grisu2; include/hankel_b200.hpp json_number).
Computed from exact rationals:  python tools/gen_pow10.py"""
from fractions import Fraction


def table():
    out = []
    for k in range(-300, 325, 8):
        v = Fraction(10) ** k
        e = v.numerator.bit_length() - v.denominator.bit_length() - 64
        while v / Fraction(2) ** e >= 2 ** 64:
            e += 1
        while v / Fraction(2) ** e < 2 ** 63:
            e -= 1
        q = v / Fraction(2) ** e
        f = int(q)
        if q - f >= Fraction(1, 2):
            f += 1
        if f == 2 ** 64:
            f, e = f // 2, e + 1
        out.append((f, e, k))
    return out


if __name__ == "__main__":
    rows = table()
    for i in range(0, len(rows), 2):
        print("        " + " ".join(f"{{0x{f:016X}ull, {e}, {k}}}," for f, e, k in rows[i:i + 2]))
