"""The drop-in boundary on CPU: libhankel_b200.so loads, exports every symbol
include/hankel_b200.h declares, and its host-only entry points work; with no GPU
the device entry points fail loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

from oracle import restate as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "hankel_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hk_[A-Za-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1810_01478_b200 import api

    lib = ctypes.CDLL(api.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert api.lib().hk_version() == 100


def test_host_moments_match_reference_moments():
    from paper_1810_01478_b200 import api

    for beta, L in (((1, 2), 64), ((1, 1), 48), ((1, 3), 200)):
        n = 40
        mu, exact = api.build_hankel(beta, n, L)
        assert exact
        for j in range(2 * n - 1):
            assert mu.to_fraction(j) == R.moment_integer(beta, j)
    # precision too small -> correctly rounded, flagged inexact
    from oracle import mpfloat as F

    for beta, L, n in (((1, 2), 2, 30), ((1, 2), 1, 40), ((1, 1), 3, 60), ((1, 3), 5, 50), ((1, 1), 1, 90)):
        mu, exact = api.build_hankel(beta, n, L)
        assert not exact
        for j in range(2 * n - 1):
            s, m, e = mu.entry(j)
            assert F.MPF(s, m, e) == F.from_int(R.moment_integer(beta, j), 32 * L), (beta, L, j)
    with pytest.raises(ValueError):
        api.build_hankel((3, 1), 4, 4)  # 2/beta not an integer (moments.cpp:74-75)


def test_assign_columns_matches_reference():
    from paper_1810_01478_b200 import api

    for n in (1, 5, 6, 17, 64):
        for w in (1, 2, 3, 4, 8):
            assert api.assign_columns(n, w) == R.assign_columns(n, w)
    with pytest.raises(ValueError):
        api.assign_columns(0, 2)


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1810_01478_b200 import api

    with pytest.raises(RuntimeError):
        api.Context(4)


def test_half_integer_gamma_moments_correctly_rounded():
    """Odd 2/beta (beta = 2, 2/3, 2/5): mu_k = (q/2) Gamma((k+1) q / 2) at half-integer
    arguments (moments.cpp:90-99; sqrt(pi) via Machin + isqrt, Ziv-checked) must be
    the correctly rounded p-bit values (mpmath at p + 200 bits)."""
    import mpmath

    from paper_1810_01478_b200 import api

    for beta, L, n in (((2, 1), 4, 30), ((2, 1), 16, 40), ((2, 3), 8, 30), ((2, 5), 3, 20), ((2, 1), 96, 64)):
        mu, exact = api.build_hankel(beta, n, L)
        assert not exact
        q, p = 2 * beta[1] // beta[0], 32 * L
        mpmath.mp.prec = p + 200
        for k in range(2 * n - 1):
            v = mpmath.mpf(q) / 2 * mpmath.gamma(mpmath.mpf((k + 1) * q) / 2)
            m, e = mpmath.frexp(v)
            M, E = int(mpmath.nint(m * mpmath.mpf(2) ** p)), int(e)
            if M == 1 << p:
                M, E = M >> 1, E + 1
            assert mu.entry(k) == (1, M, E), (beta, L, k)
