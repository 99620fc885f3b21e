"""Dev: does the CTA-pair product kernel launch (eager / graph, with and without PDL)?"""
import os
import sys
import subprocess

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, os
sys.path.insert(0, os.environ["ROOT"])
from paper_1810_01478_b200 import api
from tests.mpf_helpers import from_arr
mu, _ = api.build_hankel((1, 1), 64, 192)
mode = sys.argv[1]
try:
    with api.Context(192) as ctx:
        ctx.load_moments(mu)
        if mode == "eager":
            ctx.profile_ldlt()
        else:
            ctx.decompose()
        D = from_arr(ctx.D())
    os.environ["HK_TC_PAIR"] = "0"
    with api.Context(192) as ctx:
        ctx.load_moments(mu)
        ctx.decompose()
        D0 = from_arr(ctx.D())
    print(mode, "ok", "identical" if D == D0 else "DIFFERENT")
except Exception as e:
    print(mode, "error", e)
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for mode, env in (("eager", {}), ("graph", {}), ("graph", {"HK_PDL": "0"})):
    e = dict(os.environ, ROOT=root, HK_TC="1", **env)
    out = subprocess.run([sys.executable, "-c", code, mode], env=e, capture_output=True, text=True)
    print(env, (out.stdout + out.stderr).strip().splitlines()[-1:])
