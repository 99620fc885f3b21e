"""Dev tool (GPU box): per-LDLT-step device time of the bulk product kernels
(graph event nodes) for one config, to see where the trailing update's time
goes along the factorisation (wide early steps vs narrow late ones).

    python tools/step_profile.py c4 > gpurun_out/steps_c4.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_01478_b200 import api  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = CONFIGS[name]
L = cfg["p"] // 32
n = cfg["n"]
mu, _ = api.build_hankel(cfg["beta"], n, L)
with api.Context(L) as ctx:
    ctx.set_kernel_timing(True)
    ctx.load_moments(mu)
    for _ in range(2):
        ctx.decompose()
    st = ctx.kernel_step_times()
    kt = ctx.kernel_times()
ms = [a for a, _ in st]
buckets = {}
for i, v in enumerate(ms):
    b = (i // 128) * 128
    buckets[b] = buckets.get(b, 0.0) + v
print(json.dumps({"config": name, "ldlt_ms": kt["ldlt_ms"], "products_ms": kt["products_ms"], "round_ms": kt["round_ms"],
                  "per_128_steps_ms": buckets, "first": ms[:4], "last": ms[-4:],
                  "steps": [round(v, 4) for v in ms]}))
