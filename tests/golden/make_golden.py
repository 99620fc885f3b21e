"""Generate the committed golden fixtures tests/golden/*.json from the oracle.

Run HERE (needs /root/reference-built oracle/_ref/ref_driver; never on the GPU
box).  For every BASELINE config that the CPU can afford it runs the unmodified
reference (oracle/_ref/ref_driver dump) at two fixed-point
budgets K and K+1024, and stores:

* the pivots d_n as 45-significant-digit decimals (exact mantissa / 2^K),
* lambda-hat_1..3 = 1 / mu_i of the FIXED-POINT k x k block (the reference's
  own assembly, inversion.cpp:244-257, without its binary64 cast) solved with
  mpmath at 80 digits, printed to 45 digits,
* how many digits the two budgets agree on (the oracle is accepted only when
  pivots agree to rel <= 1e-30 and lambda to >= 25 digits),
* the reference's own binary64 lambdas / trunc_err and its RunRecord timings.

Additionally `model` fixtures hold SHA-256 digests of the product's exact
p-bit-float results computed by oracle/mpfloat.py (bit-exact GPU checks at
sizes where the pure-Python model is too slow to run inside a test).

Usage:  python tests/golden/make_golden.py c1 c2 [c3] [model_c2]
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
from fractions import Fraction

import mpmath

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import mpfloat as F  # noqa: E402
from oracle import restate as R  # noqa: E402

DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

CONFIGS = {
    "c1": dict(beta=(1, 2), n=64, p=3072, k=8, Ks=(2048, 3072)),
    "c2": dict(beta=(1, 1), n=256, p=6144, k=8, Ks=(2048, 3072)),
    "c3": dict(beta=(1, 3), n=512, p=36864, k=12, Ks=(3072, 4096)),
    "c4": dict(beta=(1, 2), n=1024, p=49152, k=16, Ks=(4096, 5120)),
}


def run_ref(beta, n, K, k, workers=8, cache_dir="/tmp/gold"):
    os.makedirs(cache_dir, exist_ok=True)
    cache = os.path.join(cache_dir, f"b{beta[0]}_{beta[1]}_n{n}_K{K}_k{k}.json")
    if os.path.exists(cache) and os.path.getsize(cache) > 0:
        with open(cache) as f:
            return json.load(f)
    out = subprocess.run([DRIVER, "dump", "--beta", f"{beta[0]}/{beta[1]}", "--n", str(n), "--bits", str(K), "--k",
                          str(k), "--workers", str(workers)], capture_output=True, text=True, check=True).stdout
    with open(cache, "w") as f:
        f.write(out)
    return json.loads(out)


def dec(fr: Fraction, digits=45) -> str:
    with mpmath.workdps(digits + 10):
        return mpmath.nstr(mpmath.mpf(fr.numerator) / fr.denominator, digits, strip_zeros=False)


def lambdas_from_block(d, k, dps=80):
    fb = d["block_frac_bits"]
    fr = [Fraction(int(h, 16), 1 << fb) for h in d["block"]]
    ev = R.block_eigs_mp(fr, k, dps=dps)
    with mpmath.workdps(dps):
        return [1 / ev[k - i] for i in range(1, min(3, k) + 1)]


def agree_digits(a, b):
    with mpmath.workdps(1000):
        cv = lambda v: mpmath.mpf(v.numerator) / v.denominator if isinstance(v, Fraction) else mpmath.mpf(v)  # noqa
        a, b = cv(a), cv(b)
        if a == b:
            return 1000.0
        return float(-mpmath.log10(abs(a - b) / abs(b)))


def make_config(name):
    cfg = CONFIGS[name]
    beta, n, k, Ks = cfg["beta"], cfg["n"], cfg["k"], cfg["Ks"]
    runs = [run_ref(beta, n, K, k) for K in Ks]
    K0 = Ks[0]
    D = [[Fraction(int(h, 16), 1 << K) for h in r["D"]] for r, K in zip(runs, Ks)]
    worst_pivot = 0.0  # as -log10(rel diff), i.e. digits of agreement (min over n)
    digs = []
    for a, b in zip(D[0], D[1]):
        digs.append(agree_digits(a, b))
    worst_pivot = min(digs)
    lam = [lambdas_from_block(r, min(k, n)) for r in runs]
    lam_digits = [agree_digits(x, y) for x, y in zip(lam[0], lam[1])]
    out = {
        "config": name,
        "beta": list(beta),
        "n": n,
        "p": cfg["p"],
        "k": k,
        "oracle": "reference hankel-eig (oracle/_ref/ref_driver dump) at fixed-point K fractional bits",
        "K": list(Ks),
        "pivot_digits_K_vs_K+1024": worst_pivot,
        "lambda_digits_K_vs_K+1024": lam_digits,
        "pivots": [dec(x) for x in D[1]],
        "lambda": [mpmath.nstr(x, 45, strip_zeros=False) for x in lam[1]],
        "reference_lambda_binary64": runs[1]["lambda"],
        "reference_trunc_err_binary64": runs[1]["trunc_err"],
        "reference_timing": {f"K{K}": r["timing"] for K, r in zip(Ks, runs)},
        "update_count": runs[1]["update_count"],
    }
    if beta == (1, 1):  # closed form d_n = (n!)^2
        import math

        ok = all(abs(D[1][i] - math.factorial(i) ** 2) / math.factorial(i) ** 2 < Fraction(1, 10**30) for i in range(n))
        out["closed_form_pivots_match_1e-30"] = ok
    path = os.path.join(HERE, f"{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"{name}: pivots agree K vs K+1024 to {worst_pivot:.1f} digits; lambda digits {lam_digits}; wrote {path}")


def digest(vals, p):
    h = hashlib.sha256()
    for x in vals:
        h.update(f"{x.s}:{x.e}:{x.m:x};".encode())
    return h.hexdigest()


def make_model(name):
    """Bit-exact product results (oracle/mpfloat.py) as digests."""
    cfg = CONFIGS[name[len("model_"):]]
    beta, n, p, k = cfg["beta"], cfg["n"], cfg["p"], min(cfg["k"], cfg["n"])
    mu = [R.moment_integer(beta, j) for j in range(2 * n - 1)]
    D, L, Rr = F.ldlt(mu, n, p)
    X = F.invert_L_partial(L, n, k, p)
    M = F.block(X, Rr, n, k, p)
    Xflat = [X[r][c] if c < min(r, k) else F.ZERO for r in range(n) for c in range(k)]
    out = {"config": name, "n": n, "p": p, "k": k, "D_sha256": digest(D, p), "L_col0_sha256": digest(L[0], p),
           "Linv_sha256": digest(Xflat, p), "block_sha256": digest(M, p),
           "D0_hex": f"{D[0].m:x}", "D_last_exp": D[-1].e}
    path = os.path.join(HERE, f"{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"{name}: wrote {path}")


if __name__ == "__main__":
    for name in sys.argv[1:]:
        if name.startswith("model_"):
            make_model(name)
        else:
            make_config(name)
