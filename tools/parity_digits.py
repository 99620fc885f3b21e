"""Dev tool (GPU box): SURVEY §8(d)'s "correct digits vs the oracle" for C1-C4 —
the GPU path against the reference's golden outputs (tests/golden/c*.json: the
reference compiled from /root/reference, at K_oracle, lambda from its fixed-point
block at 80 digits).  Same checks as tests/test_gpu_parity.py::check_vs_golden,
reported instead of asserted.  The oracle (restate.py) is used as the checker only.

    python tools/parity_digits.py c1 c2 c3 c4 > profiles/r01_parity_digits.jsonl
"""
import json
import os
import sys

import mpmath

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import restate as R  # noqa: E402  (checker only)
from paper_1810_01478_b200 import api  # noqa: E402


def digits(rel):
    return float(-mpmath.log10(rel)) if rel > 0 else 80.0


for name in sys.argv[1:] or ["c1", "c2"]:
    g = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}.json")))
    beta, n, L, k = tuple(g["beta"]), g["n"], g["p"] // 32, g["k"]
    mu, exact = api.build_hankel(beta, n, L)
    with api.Context(L) as ctx:
        rec = ctx.compute(mu, k)
        D = ctx.D()
        blk = ctx.block()
    with mpmath.workdps(80):
        worst = mpmath.mpf(0)
        for i, want in enumerate(g["pivots"]):
            fr = D.to_fraction(i)
            worst = max(worst, abs(mpmath.mpf(fr.numerator) / fr.denominator / mpmath.mpf(want) - 1))
        ev = R.block_eigs_mp([blk.to_fraction(i) for i in range(k * k)], k, dps=80)
        lam_digits = [digits(abs((1 / ev[k - 1 - i]) / mpmath.mpf(g["lambda"][i]) - 1)) for i in range(min(3, k))]
        lam1 = mpmath.mpf(rec.lambda_hi[0]) + mpmath.mpf(rec.lambda_lo[0])
        host_digits = digits(abs(lam1 / mpmath.mpf(g["lambda"][0]) - 1))
    print(json.dumps({"config": name, "n": n, "p_bits": g["p"], "k": k, "pivots_checked": len(g["pivots"]),
                      "pivot_min_digits": digits(worst), "pivot_worst_rel": float(worst),
                      "lambda_digits_mp_block": lam_digits, "lambda1_digits_host_hi_lo": host_digits,
                      "lambda_min": repr(lam1), "tolerance": "pivots rel <= 1e-20 (20 digits), lambda >= 20 digits",
                      "golden": f"tests/golden/{name}.json"}), flush=True)
