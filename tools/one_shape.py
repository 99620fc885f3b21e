"""Dev tool: compute() of an arbitrary shape: python tools/one_shape.py bnum,bden,n,L,k [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_01478_b200 import api  # noqa: E402

bn, bd, n, L, k = (int(x) for x in sys.argv[1].split(","))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mu, _ = api.build_hankel((bn, bd), n, L)
with api.Context(L) as ctx:
    for _ in range(reps):
        t = time.perf_counter()
        rec = ctx.compute(mu, k)
        print(f"n {n} L {L} wall {1e3 * (time.perf_counter() - t):.2f} ms ldlt {rec.ldlt_s * 1e3:.3f} invL {rec.invL_s * 1e3:.3f} "
              f"lambda {rec.lambda_hi[0]!r}", flush=True)
