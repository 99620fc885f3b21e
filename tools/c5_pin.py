"""Dev tool (GPU box): pin C5 (beta=1/2, N=2048, p=114688, k=16), which no CPU
oracle can run, by the acceptance rule SURVEY §8c states for
the oracle itself: the computation at p and at p + 8192 bits must agree on
every pivot d_n to >= 30 digits and on lambda_hat_1..3 to >= 25 digits (the
two precisions share nothing but the exact moments).  Also the nested-prefix
check against the C4 reference pivots (H_1024 leads H_2048) and the Table 2
bracket (tools/c5_run.py).  Writes one JSON line."""
import json
import os
import sys
import time
from decimal import Decimal, getcontext

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1810_01478_b200 import api  # noqa: E402

getcontext().prec = 80
n, k = 2048, 16
runs = {}
for p in (114688, 114688 + 8192):
    L = p // 32
    t0 = time.perf_counter()
    mu, exact = api.build_hankel((1, 2), n, L)
    assert exact
    with api.Context(L) as ctx:
        rec = ctx.compute(mu, k)
        D = ctx.D()
    piv = []
    for i in range(n):
        s, m, e = D.entry(i)
        piv.append(Decimal(s) * Decimal(m) * (Decimal(2) ** (e - 32 * L)))
    lam = [Decimal(h) + Decimal(lo) for h, lo in zip(rec.lambda_hi, rec.lambda_lo)]
    runs[p] = dict(piv=piv, lam=lam, wall_s=time.perf_counter() - t0, ldlt_s=rec.ldlt_s, invL_s=rec.invL_s)


def digits(a, b):
    rel = abs(a / b - 1)
    return float(-rel.log10()) if rel > 0 else 80.0


a, b = runs[114688], runs[114688 + 8192]
piv_d = [digits(x, y) for x, y in zip(a["piv"], b["piv"])]
lam_d = [digits(x, y) for x, y in zip(a["lam"], b["lam"])]
g4 = json.load(open(os.path.join(ROOT, "tests", "golden", "c4.json")))
pref = min(digits(x, Decimal(w)) for x, w in zip(a["piv"], g4["pivots"]))
t2 = json.load(open(os.path.join(ROOT, "tests", "golden", "table2.json")))
tl = {r["n"]: r["lam"][0] for r in t2["rows"]}
lam1 = float(a["lam"][0])
out = {
    "config": "C5 beta=1/2 N=2048 k=16 at p=114688 and p=122880",
    "min_pivot_digits_all": min(piv_d), "min_pivot_digits_1024_2047": min(piv_d[1024:]),
    "lambda_digits": lam_d, "required": {"pivots": 30, "lambda": 25},
    "pass": min(piv_d) >= 30 and min(lam_d) >= 25,
    "prefix_min_digits_vs_c4_reference": pref,
    "table2_bracket": [tl.get(2000), lam1, tl.get(2500)],
    "bracket_holds": bool(tl.get(2000, 1e9) > lam1 > tl.get(2500, -1e9)),
    "lambda_min": str(a["lam"][0]), "lambda_min_p_plus_8192": str(b["lam"][0]),
    "time_s": {str(p): {kk: v for kk, v in r.items() if kk in ("wall_s", "ldlt_s", "invL_s")} for p, r in runs.items()},
}
print(json.dumps(out))
