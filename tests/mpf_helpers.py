"""Shared helpers for the tests: conversions between oracle/mpfloat.MPF and the
ABI's SoA arrays / the emulator's text format, and random operand generators."""
import random

from oracle import mpfloat as F


def to_line(x, L):
    limbs = [(x.m >> (32 * i)) & 0xFFFFFFFF for i in range(L)]
    return f"{x.s} {x.e} " + " ".join(f"{v:x}" for v in limbs)


def from_line(s, L):
    t = s.split()
    sg, e, m = int(t[0]), int(t[1]), 0
    for i, h in enumerate(t[2:2 + L]):
        m |= int(h, 16) << (32 * i)
    return F.MPF(sg, m, e) if sg != 0 else F.ZERO


def to_arr(xs, L):
    from paper_1810_01478_b200 import api

    a = api.MPArray.empty(len(xs), L)
    for i, x in enumerate(xs):
        a.set_entry(i, x.s, x.m, x.e)
    return a


def from_arr(a):
    out = []
    for i in range(len(a)):
        s, m, e = a.entry(i)
        out.append(F.MPF(s, m, e) if s else F.ZERO)
    return out


def rnd(L, rng: random.Random, e=None):
    """Random normalised p-bit float with the edge patterns the rounding logic cares about."""
    p = 32 * L
    m = rng.getrandbits(p) | (1 << (p - 1))
    st = rng.random()
    if st < 0.1:
        m = 1 << (p - 1)  # power of two (binade edge)
    elif st < 0.2:
        m = (1 << p) - 1  # all ones (round-up overflow)
    elif st < 0.3:
        m = (1 << (p - 1)) | rng.getrandbits(5)  # long zero run
    return F.MPF(rng.choice([1, -1]), m, rng.randint(-70, 70) if e is None else e)


def fms_cases(L, rng, count):
    """(c, x, y) triples: heavy cancellation, exact cancellation, zeros, far/near exponents."""
    p = 32 * L
    out = []
    for _ in range(count):
        x, y = rnd(L, rng), rnd(L, rng)
        r = rng.random()
        if r < 0.3:
            pr = F.mul(x, y, p)
            c = pr if rng.random() < 0.4 else F.MPF(pr.s, pr.m ^ rng.getrandbits(rng.randint(1, p)), pr.e)
        elif r < 0.4:
            c = F.ZERO
        elif r < 0.5:
            c = rnd(L, rng, e=x.e + y.e + rng.randint(-3 * p, 3 * p))
        else:
            c = rnd(L, rng, e=x.e + y.e + rng.randint(-40, 40))
        if rng.random() < 0.05:
            x = F.ZERO
        out.append((c, x, y))
    return out
