"""Dev tool (GPU box): kernel times of hk_assemble_block at one config (torch.profiler / CUPTI)."""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_1810_01478_b200 import api  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
L = cfg["p"] // 32
mu, _ = api.build_hankel(cfg["beta"], cfg["n"], L)
torch.cuda.init()
with api.Context(L) as ctx:
    ctx.load_moments(mu)
    ctx.decompose_invert(cfg["k"])
    ctx.assemble_truncated_inverse(cfg["k"])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ctx.assemble_truncated_inverse(cfg["k"])
        torch.cuda.synchronize()
tot = collections.defaultdict(float)
cnt = collections.Counter()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name[:90]] += e.time_range.end - e.time_range.start
        cnt[e.name[:90]] += 1
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{tot[k] / 1e3:9.3f} ms  x{cnt[k]:3d}  {k}")
