"""Quick GPU bring-up check (dev tool): batch-op parity vs oracle/mpfloat.py,
pipeline bit-exactness at small sizes, and a first C2 timing."""
import sys, time, random, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_01478_b200 import api
from oracle import mpfloat as F, restate as R

def to_arr(xs, L):
    a = api.MPArray.empty(len(xs), L)
    for i, x in enumerate(xs): a.set_entry(i, x.s, x.m, x.e)
    return a
def from_arr(a):
    out = []
    for i in range(len(a)):
        s, m, e = a.entry(i)
        out.append(F.MPF(s, m, e) if s else F.ZERO)
    return out
def rnd(L, rng, e=None):
    p = 32 * L
    m = rng.getrandbits(p) | (1 << (p - 1))
    st = rng.random()
    if st < 0.1: m = 1 << (p - 1)
    elif st < 0.2: m = (1 << p) - 1
    return F.MPF(rng.choice([1, -1]), m, rng.randint(-70, 70) if e is None else e)

rng = random.Random(7)
bad = 0
for L in [1, 3, 8, 96, 192, 1152]:
    p = 32 * L
    cnt = 64 if L < 1000 else 16
    with api.Context(L) as ctx:
        xs = [rnd(L, rng) for _ in range(cnt)]; ys = [rnd(L, rng) for _ in range(cnt)]
        cs = []
        for x, y in zip(xs, ys):
            pr = F.mul(x, y, p)
            r = rng.random()
            cs.append(pr if r < 0.2 else F.MPF(pr.s, pr.m ^ rng.getrandbits(rng.randint(1, p)), pr.e) if r < 0.5 else rnd(L, rng, e=x.e + y.e + rng.randint(-50, 50)))
        t = time.time()
        got = from_arr(ctx.mp_batch(api.OP_FMS, to_arr(xs, L), to_arr(ys, L), to_arr(cs, L)))
        b1 = sum(g != F.fms(c, x, y, p) for g, c, x, y in zip(got, cs, xs, ys))
        got = from_arr(ctx.mp_batch(api.OP_MUL, to_arr(xs, L), to_arr(ys, L)))
        b2 = sum(g != F.mul(x, y, p) for g, x, y in zip(got, xs, ys))
        got = from_arr(ctx.mp_batch(api.OP_ADD, to_arr(xs, L), to_arr(cs, L)))
        b3 = sum(g != F.add(x, y, p) for g, x, y in zip(got, xs, cs))
        got = from_arr(ctx.mp_batch(api.OP_RECIP, to_arr(xs, L)))
        b4 = sum(g != F.recip(x, p) for g, x in zip(got, xs))
        print(f"L={L}: fms {b1} mul {b2} add {b3} recip {b4} mismatches / {cnt} ({time.time()-t:.2f}s)", flush=True)
        bad += b1 + b2 + b3 + b4

# pipeline bit-exact vs model at small sizes
for beta, N, L, k in [((1, 2), 8, 4, 4), ((1, 1), 24, 6, 8), ((1, 2), 64, 96, 8)]:
    p = 32 * L
    mu_int = [R.moment_integer(beta, j) for j in range(2 * N - 1)]
    t = time.time()
    D, Lf, Rr = F.ldlt(mu_int, N, p); X = F.invert_L_partial(Lf, N, k, p); M = F.block(X, Rr, N, k, p)
    tm = time.time() - t
    mu, exact = api.build_hankel(beta, N, L)
    with api.Context(L) as ctx:
        ctx.load_moments(mu); ctx.decompose(); gD = from_arr(ctx.D())
        ctx.invert_L_partial(k); gX = from_arr(ctx.Linv())
        ctx.assemble_truncated_inverse(k); gM = from_arr(ctx.block())
        okD = gD == D
        okX = all(gX[r * k + c] == X[r][c] for r in range(N) for c in range(min(r, k)))
        okM = gM == M
        hi, lo, te = ctx.smallest_eigs_of_H(min(3, k))
    print(f"path beta={beta} N={N} L={L} k={k}: D {okD} X {okX} M {okM} exact_moments {exact} lambda {hi[0]!r}+{lo[0]!r} model {tm:.1f}s", flush=True)
    bad += (not okD) + (not okX) + (not okM)

# C2 timing
mu, exact = api.build_hankel((1, 1), 256, 192)
with api.Context(192) as ctx:
    for rep in range(3):
        rec = ctx.compute(mu, 8)
        print(f"C2 rep{rep}: wall {rec.wall_s*1e3:.1f} ms ldlt {rec.ldlt_s*1e3:.1f} invL {rec.invL_s*1e3:.1f} invH {rec.invH_s*1e3:.1f} eig {rec.eigen_s*1e3:.2f} lambda {rec.lambda_hi} launches {ctx.launch_count()}", flush=True)
    fmas = 256 * (256**2 - 1) // 6
    print(f"C2 MP-FMA/s (ldlt) {fmas / rec.ldlt_s:.3e}; limb-MAC/s {fmas * 192**2 / rec.ldlt_s:.3e}")
print("BAD", bad)
