"""Dev tool: ONE full compute of a BASELINE config (for ncu launch lists / captures).

    python tools/one_run.py c3 [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_01478_b200 import api  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L = cfg["p"] // 32
mu, _ = api.build_hankel(cfg["beta"], cfg["n"], L)
with api.Context(L) as ctx:
    for _ in range(reps):
        t = time.perf_counter()
        try:
            rec = ctx.compute(mu, cfg["k"])
        except api.PrecisionError:  # dev what-if runs (wrong values): still report the LDLT's device time
            print(f"ldlt {ctx.timings()[1] * 1e3:.2f} ms (precision error: what-if run)", flush=True)
            continue
        print(f"fix {ctx.fix_count()} wall {1e3 * (time.perf_counter() - t):.2f} ms ldlt {rec.ldlt_s * 1e3:.2f} invL {rec.invL_s * 1e3:.2f} invH {rec.invH_s * 1e3:.2f} eig {rec.eigen_s * 1e3:.2f} "
              f"h2d {rec.h2d_s * 1e3:.2f} d2h {rec.d2h_s * 1e3:.2f} lambda {rec.lambda_hi[0]!r}", flush=True)
