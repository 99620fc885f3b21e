"""The oracle is pinned before it is trusted (CPU only).

* oracle/restate.py (CPU restatement, Python ints) is bit-identical to the
  reference itself, compiled unchanged from /root/reference by oracle/Makefile
  (oracle/_ref/ref_driver), on D, L, L^{-1} and the fixed-point block.
* The reference's own unit tests (proj/tests/test_*.cpp) run against that build;
  the only failing cases are reference-test defects documented here.
* Known answers from the reference tests, the beta=1 closed form and the
  committed golden fixtures (tests/golden/*.json, made by make_golden.py).
"""
import json
import math
import os
import subprocess
from fractions import Fraction

import mpmath
import pytest

from oracle import mpfloat as F
from oracle import restate as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")

# Reference unit-test cases that fail against the unmodified reference, with the reason.
KNOWN_REFERENCE_TEST_DEFECTS = {
    # test_moments.cpp:39 expects floor(sqrt(pi) 2^64) but gamma_exact rounds to nearest
    # (moments.cpp:99, div_round_even): sqrt(pi) 2^64 = ...953.764 -> 954.
    "gamma at half-integer arguments tracks sqrt(pi)",
    # test_ldlt.cpp:111-133 uses an absolute 2^-K/2 bound on entries of size ~mu_{2n}.
    "property: L D L^T reconstructs H",
    # test_ldlt.cpp:167-184: K=0 does not exhaust precision for beta=1, n<=16.
    "precision exhaustion raises instead of returning garbage",
    # test_jacobi.cpp:79: c = cos(a1), s = sin(a2) with two different angles (not orthogonal).
    "property: invariance under orthogonal conjugation",
    # test_pipeline.cpp:76-79: binary64 trunc_err is exactly 0 at N=12, k=8.
    "truncation error estimates are negative once k < N",
    # test_pipeline.cpp:105-114: tiny K makes smallest_eigs_of_H throw runtime_error, not precision_error.
    "auto_precision caps out with a diagnostic",
    # test_pipeline.cpp:127-134: compute() rejects bits=0 (pipeline.cpp:28), the test expects success.
    "scan produces one row per N and keeps going after failures",
}
# asymptotics.cpp needs Boost.Math (absent; out of scope) -> not run
SKIPPED_OUT_OF_SCOPE = ["report fits", "JSON serializations"]


def ref_dump(driver, beta, n, K, k, workers=2):
    out = subprocess.run([driver, "dump", "--beta", f"{beta[0]}/{beta[1]}", "--n", str(n), "--bits", str(K), "--k",
                          str(k), "--workers", str(workers)], capture_output=True, text=True, check=True).stdout
    return json.loads(out)


@pytest.mark.parametrize("beta,n,K,k", [((1, 2), 2, 64, 2), ((1, 2), 20, 256, 8), ((1, 1), 30, 128, 8),
                                        ((1, 3), 16, 512, 8), ((1, 2), 50, 512, 8), ((1, 2), 64, 2048, 8)])
def test_restatement_bit_identical_to_reference(ref_driver, beta, n, K, k):
    d = ref_dump(ref_driver, beta, n, K, k)
    D, L, Linv, M, upd = R.pipeline_fixed(beta, n, K, k)
    h = lambda v: int(v, 16)  # noqa: E731
    assert [h(x) for x in d["D"]] == D
    assert [h(x) for x in d["L_col0"]] == L[0]
    assert all([h(x) for x in d["Linv"][r]] == Linv[r] for r in range(n))
    assert [h(x) for x in d["block"]] == M
    assert d["update_count"] == upd == n * (n * n - 1) // 6  # test_ldlt.cpp:135-145
    # binary64 lambdas: the reference's jacobi restated (jacobi.cpp:27-103)
    kk = min(k, n)
    Md = [R.fix_to_double(x, 2 * K) for x in M]
    lam, _ = R.smallest_eigs_of_H(Md, kk, min(3, kk))
    assert lam == pytest.approx(d["lambda"], rel=1e-12)


def test_reference_unit_tests_against_oracle_build(ref_driver):
    exe = os.path.join(os.path.dirname(ref_driver), "ref_unit_tests")
    args = [exe] + [f"--skip={s}" for s in SKIPPED_OUT_OF_SCOPE]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    failed = {ln[7:] for ln in out.splitlines() if ln.startswith("[FAIL] ")}
    passed = {ln[7:] for ln in out.splitlines() if ln.startswith("[ ok ] ")}
    assert failed == KNOWN_REFERENCE_TEST_DEFECTS
    assert len(passed) >= 50


def test_known_answers_from_reference_tests():
    # test_ldlt.cpp:80-87
    D, L, upd = R.decompose_serial((1, 2), 2, 64)
    assert D == [2 << 64, 168 << 64] and L[0] == [6 << 64] and upd == 1
    # test_inversion.cpp:121-133: H_2^{-1} = (1/336)[[240,-12],[-12,2]]
    Dd, Ld, Linv, M, _ = R.pipeline_fixed((1, 2), 2, 128, 2)
    Mf = [Fraction(x, 1 << 256) for x in M]
    for got, want in zip(Mf, [Fraction(240, 336), Fraction(-12, 336), Fraction(-12, 336), Fraction(2, 336)]):
        assert abs(got - want) < Fraction(1, 2**120)
    # test_jacobi.cpp:103-111 / test_pipeline.cpp:41-44
    lam, err = R.smallest_eigs_of_H([240 / 336, -12 / 336, -12 / 336, 2 / 336], 2, 1)
    assert lam[0] == pytest.approx(1.39648834586837266, rel=1e-13) and err[0] < 0
    # test_moments.cpp:23-28 (pi / sqrt(pi) mantissas)
    assert R.pi_scaled(64) == 57952155664616982739
    assert R.sqrt_pi_scaled(128) == 603134791644261162232608214451700185151
    # test_moments.cpp:61-67: mu_k = 2 (2k+1)! exactly for beta = 1/2
    for k in range(41):
        assert R.moment((1, 2), k, 32) == (2 * math.factorial(2 * k + 1) << 32, 32)
    # test_ldlt.cpp:32-52
    assert R.assign_columns(6, 3) == [0, 1, 2, 2, 1, 0]
    assert R.assign_columns(5, 2) == [0, 1, 1, 0, 0]


def test_beta1_closed_form():
    """beta=1: d_n = (n!)^2, L(i,j) = C(i,j) i!/j!, exact in fixed point."""
    n, K = 14, 64
    D, L, _ = R.decompose_serial((1, 1), n, K)
    assert D == [math.factorial(i) ** 2 << K for i in range(n)]
    for j in range(n - 1):
        for r, v in enumerate(L[j]):
            i = j + 1 + r
            assert v == (math.comb(i, j) * math.factorial(i) // math.factorial(j)) << K


def test_mpfloat_model_is_correctly_rounded():
    """The float model's ops are the nearest p-bit float (ties to even) of the exact value."""
    import random

    rng = random.Random(20240517)
    for L in (1, 2, 4):
        p = 32 * L
        for _ in range(200):
            x = F.MPF(rng.choice([1, -1]), rng.getrandbits(p) | (1 << (p - 1)), rng.randint(-50, 50))
            y = F.MPF(rng.choice([1, -1]), rng.getrandbits(p) | (1 << (p - 1)), rng.randint(-50, 50))
            c = F.MPF(rng.choice([1, -1]), rng.getrandbits(p) | (1 << (p - 1)), x.e + y.e + rng.randint(-8, 8))
            exact = c.to_fraction(p) - x.to_fraction(p) * y.to_fraction(p)
            r = F.fms(c, x, y, p)
            if exact == 0:
                assert r.s == 0
                continue
            rv = r.to_fraction(p)
            ulp = Fraction(2) ** (r.e - p)
            assert abs(rv - exact) <= ulp / 2
            assert 2 ** (p - 1) <= r.m < 2 ** p
            q = F.recip(x, p).to_fraction(p)
            assert abs(q - 1 / x.to_fraction(p)) <= Fraction(2) ** (F.recip(x, p).e - p) / 2


def test_float_model_c1_meets_tolerance_vs_golden():
    """At C1 (beta=1/2, N=64, p=3072) the float model's pivots and lambda match the oracle."""
    g = json.load(open(os.path.join(GOLD, "c1.json")))
    n, p, k = g["n"], g["p"], g["k"]
    mu = [R.moment_integer((1, 2), j) for j in range(2 * n - 1)]
    D, L, Rr = F.ldlt(mu, n, p)
    X = F.invert_L_partial(L, n, k, p)
    M = F.block(X, Rr, n, k, p)
    with mpmath.workdps(60):
        for d, want in zip(D, g["pivots"]):
            fr = d.to_fraction(p)
            assert abs(mpmath.mpf(fr.numerator) / fr.denominator / mpmath.mpf(want) - 1) < mpmath.mpf("1e-40")
        ev = R.block_eigs_mp([m.to_fraction(p) for m in M], k, dps=60)
        lam = 1 / ev[-1]
        assert abs(lam / mpmath.mpf(g["lambda"][0]) - 1) < mpmath.mpf("1e-40")


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_golden_fixture_is_self_consistent(name):
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    assert g["pivot_digits_K_vs_K+1024"] >= 30
    assert min(g["lambda_digits_K_vs_K+1024"]) >= 25
    assert float(g["lambda"][0]) == pytest.approx(g["reference_lambda_binary64"][0], rel=1e-14)
    if name == "c2":
        assert g["closed_form_pivots_match_1e-30"]
