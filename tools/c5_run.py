"""Dev tool (GPU box): one C5 compute (beta=1/2, N=2048, p=114688) on one B200 and
the C5 parity checks that need no CPU oracle run:
  * nested prefix: H_1024 is the leading block of H_2048, so the first 1024 LDLT
    pivots must equal the C4 reference pivots (tests/golden/c4.json) to rel 1e-20;
  * Table 2 bracket: lambda(2000) > lambda_hat(2048) > lambda(2500)
    (tests/golden/table2.json, reference_data.hpp:23-33)."""
import json
import os
import sys
import time
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1810_01478_b200 import api  # noqa: E402

n, L, k = 2048, 114688 // 32, 16
t0 = time.perf_counter()
mu, exact = api.build_hankel((1, 2), n, L)
assert exact
with api.Context(L) as ctx:
    rec = ctx.compute(mu, k)
    D = ctx.D()
wall = time.perf_counter() - t0
g4 = json.load(open(os.path.join(ROOT, "tests", "golden", "c4.json")))
from decimal import Decimal, getcontext  # noqa: E402

getcontext().prec = 60
worst = Decimal(0)
for i, want in enumerate(g4["pivots"]):
    s, m, e = D.entry(i)
    got = Decimal(s) * Decimal(m) * (Decimal(2) ** (e - 32 * L))
    rel = abs(got / Decimal(want) - 1)
    worst = max(worst, rel)
t2 = json.load(open(os.path.join(ROOT, "tests", "golden", "table2.json")))
lam = {r["n"]: r["lam"][0] for r in t2["rows"]}
lam1 = rec.lambda_hi[0] + rec.lambda_lo[0]
print(json.dumps({"config": "C5 beta=1/2 N=2048 p=114688 k=16", "lambda_min": repr(lam1), "wall_s": rec.wall_s,
                  "ldlt_s": rec.ldlt_s, "invL_s": rec.invL_s, "invH_s": rec.invH_s, "host_wall_s": wall,
                  "prefix_worst_rel_vs_c4_reference": float(worst),
                  "bracket_ok": lam[2000] > lam1 > lam[2500], "bracket": [lam[2000], lam1, lam[2500]]}))
