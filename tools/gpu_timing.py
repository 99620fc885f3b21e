"""Dev tool: stage timings of one config + latency of single MP ops (run on the GPU box)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_01478_b200 import api  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
C = {"c1": ((1, 2), 64, 96, 8), "c2": ((1, 1), 256, 192, 8), "c3": ((1, 3), 512, 1152, 12),
     "c4": ((1, 2), 1024, 1536, 16)}[cfg]
beta, n, L, k = C
mu, _ = api.build_hankel(beta, n, L)
with api.Context(L) as ctx:
    for rep in range(3):
        rec = ctx.compute(mu, k)
    print(f"{cfg}: wall {rec.wall_s*1e3:.2f} ms | ldlt {rec.ldlt_s*1e3:.2f} invL {rec.invL_s*1e3:.2f} "
          f"invH {rec.invH_s*1e3:.2f} eig {rec.eigen_s*1e3:.2f} h2d {rec.h2d_s*1e3:.2f} d2h {rec.d2h_s*1e3:.2f}")
    prof, nt = ctx.profile_ldlt()
    fm = n * (n * n - 1) // 6
    print("eager LDLT kernel ms:", {k: round(v, 3) for k, v in prof.items()},
          f"-> trailing {fm*L*L/prof['trailing']/1e9:.3f} T limb-MAC/s; per-step recip "
          f"{prof['recip']/n*1e3:.1f} us, mulB {prof['mulB']/max(n-1,1)*1e3:.1f} us")
    # single-op latency (1 item per launch)
    one = api.MPArray.empty(1, L)
    one.set_entry(0, 1, (1 << (32 * L - 1)) | 12345, 7)
    for op, name in ((api.OP_RECIP, "recip"), (api.OP_MUL, "mul"), (api.OP_FMS, "fms")):
        for _ in range(2):
            t = time.perf_counter()
            ctx.mp_batch(op, one, one, one)
            dt = time.perf_counter() - t
        print(f"single {name} (incl. H2D/D2H + launch): {dt*1e6:.1f} us")
print("peak imad", api.peak_imad(0) / 1e12)
