"""Dev tool (GPU box): kernel timeline of one LDLT via torch.profiler (CUPTI
activity tracing sees the library's graph kernels too).  Writes
gpurun_out/timeline_<cfg>.json: [{name, stream, ts_us, dur_us}] sorted by start.

    python tools/timeline.py c2
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_1810_01478_b200 import api  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = CONFIGS[cfg_name]
L = cfg["p"] // 32
mu, _ = api.build_hankel(cfg["beta"], cfg["n"], L)
torch.cuda.init()
with api.Context(L) as ctx:
    ctx.load_moments(mu)
    ctx.decompose()  # capture the graph
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ctx.decompose()
        torch.cuda.synchronize()
events = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name
        events.append({"name": name[:80], "stream": getattr(e, "device_resource_id", None) or 0,
                       "ts_us": e.time_range.start, "dur_us": e.time_range.end - e.time_range.start})
events.sort(key=lambda x: x["ts_us"])
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
out = os.path.join(ROOT, "gpurun_out", f"timeline_{cfg_name}.json")
json.dump(events, open(out, "w"))
print(len(events), "kernel events ->", out)
