"""Dev tool: LDLT time of the 1-GPU schedule vs the sharded look-ahead schedule
(virtual world W on this one GPU, and a real 1-rank NCCL communicator).  The
virtual timings are NOT multi-GPU numbers (all shards run on one device); they
show the sharded schedule's overhead over the single-GPU graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_01478_b200 import api  # noqa: E402

C = {"c1": ((1, 2), 64, 96, 8), "c2": ((1, 1), 256, 192, 8), "c3": ((1, 3), 512, 1152, 12),
     "c4": ((1, 2), 1024, 1536, 16)}
for cfg in sys.argv[1:] or ["c2"]:
    beta, n, L, k = C[cfg]
    mu, _ = api.build_hankel(beta, n, L)
    ref = None
    for name, kw in (("1gpu", {}), ("nccl1", dict(rank=0, world=1, nccl_id=api.nccl_unique_id())),
                     ("virt2", dict(world=2, virtual=True)), ("virt4", dict(world=4, virtual=True))):
        with api.Context(L, **kw) as ctx:
            ctx.load_moments(mu)
            ts = []
            for rep in range(4):
                ctx.decompose()
                ts.append(ctx.timings())
            rec = ctx.compute(mu, k)
            d = [ctx.D().entry(i) for i in range(n)]
            same = ref is None or d == ref
            ref = ref or d
            print(f"{cfg} {name}: ldlt {rec.ldlt_s*1e3:.2f} ms wall {rec.wall_s*1e3:.2f} ms launches/run "
                  f"{ctx.launch_count()} identical={same}", flush=True)
