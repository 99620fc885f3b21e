"""Dev tool (GPU box): LDLT time with launches dropped (HK_DEV_SKIP) to find the
stream that bounds the step time.  Results are wrong by construction."""
import os
import subprocess
import sys

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
code = f"""
import sys, time; sys.path.insert(0, '.')
from paper_1810_01478_b200 import api
from bench import CONFIGS
c = CONFIGS['{cfg}']; L = c['p'] // 32
mu, _ = api.build_hankel(c['beta'], c['n'], L)
with api.Context(L) as ctx:
    ctx.load_moments(mu)
    best = 1e9
    for r in range(4):
        try:
            ctx.decompose()
        except Exception:
            pass
        best = min(best, ctx.timings()[1] if hasattr(ctx, 'timings') else 0)
    print(f"{{best*1e3:.2f}}")
"""
for skip in ["", "recip", "mulb", "coldiag", "coloff", "recip,mulb,coldiag,coloff", "round", "prod", "round,prod,fix",
             "storel", "fix"]:
    env = dict(os.environ, HK_DEV_SKIP=skip or "none")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(f"skip={skip or '-':32s} ldlt_ms={out.stdout.strip()} {out.stderr.strip()[-200:]}", flush=True)
