import os, subprocess, sys
code = """
import sys; sys.path.insert(0, '.')
from paper_1810_01478_b200 import api
from bench import CONFIGS
c = CONFIGS['c2']; L = c['p'] // 32
mu, _ = api.build_hankel(c['beta'], c['n'], L)
with api.Context(L) as ctx:
    ctx.load_moments(mu)
    best = 1e9
    for r in range(5):
        try: ctx.decompose()
        except Exception: pass
        best = min(best, ctx.timings()[1])
    print(f"{best*1e3:.2f}")
"""
for skip in ["none", "recip,mulb,coldiag,coloff,prod,round,fix,storel", "recip,coldiag,coloff", "recip,coldiag,coloff,mulb", "prod,round,fix,storel,recip"]:
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, HK_DEV_SKIP=skip), capture_output=True, text=True)
    print(f"skip={skip:50s} ldlt_ms={out.stdout.strip()} {out.stderr.strip()[-150:]}", flush=True)
