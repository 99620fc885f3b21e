"""The device MP arithmetic and stage index maps, run on CPU under the lockstep
warp emulator (tools/emu_mp.cpp compiles csrc/*.cuh with -DHK_WARP_EMU), must be
bit-identical to the executable spec oracle/mpfloat.py."""
import random
import subprocess

import pytest

from oracle import mpfloat as F
from oracle import restate as R
from tests.mpf_helpers import fms_cases, from_line, rnd, to_line


def run(emu_bin, lines):
    out = subprocess.run([emu_bin], input="\n".join(lines) + "\n", capture_output=True, text=True, check=True)
    return out.stdout.strip().split("\n")


@pytest.mark.parametrize("L", [1, 2, 3, 5, 8, 33])
def test_emulated_ops_match_model(emu_bin, L):
    rng = random.Random(1000 + L)
    p = 32 * L
    cases = fms_cases(L, rng, 60)
    lines = [f"op fms {L} {len(cases)}"] + [to_line(v, L) for t in cases for v in t]
    for (c, x, y), r in zip(cases, run(emu_bin, lines)):
        assert from_line(r, L) == F.fms(c, x, y, p), (c, x, y)
    for op, fn in (("mul", F.mul), ("add", F.add)):
        pairs = []
        for _ in range(40):
            x = rnd(L, rng)
            y = rnd(L, rng, e=x.e + rng.randint(-2 * p, 2 * p)) if rng.random() < 0.5 else rnd(L, rng)
            if op == "add" and rng.random() < 0.3:
                y = F.MPF(-x.s, x.m ^ rng.getrandbits(rng.randint(0, p)), x.e)
            pairs.append((x, y))
        lines = [f"op {op} {L} {len(pairs)}"] + [to_line(v, L) for t in pairs for v in t]
        for (x, y), r in zip(pairs, run(emu_bin, lines)):
            assert from_line(r, L) == fn(x, y, p)
    ds = [rnd(L, rng) for _ in range(40)]
    for op in ("recip", "recipx"):  # recipx: exact midpoint test forced on every call
        lines = [f"op {op} {L} {len(ds)}"] + [to_line(d, L) for d in ds]
        for d, r in zip(ds, run(emu_bin, lines)):
            assert from_line(r, L) == F.recip(d, p)


@pytest.mark.parametrize("beta,N,L,m", [((1, 2), 8, 4, 4), ((1, 1), 12, 3, 5), ((1, 3), 6, 8, 6), ((1, 2), 11, 8, 4),
                                        ((1, 2), 3, 4, 3), ((1, 2), 1, 2, 1)])
def test_emulated_path_matches_model(emu_bin, beta, N, L, m):
    p = 32 * L
    mu = [R.moment_integer(beta, j) for j in range(2 * N - 1)]
    lines = [f"path {L} {N} {m}"] + [to_line(F.from_int(v, p), L) for v in mu]
    out = run(emu_bin, lines)
    D, Lf, Rr = F.ldlt(mu, N, p)
    X = F.invert_L_partial(Lf, N, m, p)
    M = F.block(X, Rr, N, m, p)
    assert out[-1] == "err -1"
    assert [from_line(s, L) for s in out[:N]] == D
    gx = [from_line(s, L) for s in out[N:N + N * m]]
    assert all(gx[r * m + c] == X[r][c] for r in range(N) for c in range(min(r, m)))
    assert [from_line(s, L) for s in out[N + N * m:N + N * m + m * m]] == M


def test_emulated_path_reports_first_bad_pivot(emu_bin):
    """beta = 1 at p = 32 bits loses positive definiteness; the first non-positive
    pivot column is reported (ldlt.cpp:83-87, 111)."""
    N, L, p = 16, 1, 32
    mu = [R.moment_integer((1, 1), j) for j in range(2 * N - 1)]
    out = run(emu_bin, [f"path {L} {N} 4"] + [to_line(F.from_int(v, p), L) for v in mu])
    col = int(out[-1].split()[1])
    try:
        F.ldlt(mu, N, p)
        model_col = -1
    except ArithmeticError as e:
        model_col = int(str(e).rsplit(" ", 1)[1])
    assert col == model_col and col > 0


@pytest.mark.parametrize("L", [1, 3, 8, 33])
def test_emulated_cta_ops_match_model(emu_bin, L):
    """The CTA-cooperative critical-path ops (as a 1-warp CTA on the host)."""
    rng = random.Random(2000 + L)
    p = 32 * L
    cases = fms_cases(L, rng, 40)
    lines = [f"op cfms {L} {len(cases)}"] + [to_line(v, L) for t in cases for v in t]
    for (c, x, y), r in zip(cases, run(emu_bin, lines)):
        assert from_line(r, L) == F.fms(c, x, y, p), (c, x, y)
    pairs = [(rnd(L, rng), rnd(L, rng)) for _ in range(30)]
    lines = [f"op cmul {L} {len(pairs)}"] + [to_line(v, L) for t in pairs for v in t]
    for (x, y), r in zip(pairs, run(emu_bin, lines)):
        assert from_line(r, L) == F.mul(x, y, p)
    ds = [rnd(L, rng) for _ in range(30)]
    for op in ("crecip", "crecipx"):
        lines = [f"op {op} {L} {len(ds)}"] + [to_line(d, L) for d in ds]
        for d, r in zip(ds, run(emu_bin, lines)):
            assert from_line(r, L) == F.recip(d, p)


def _fused_run(emu_bin, cases, L, op="fused"):
    lines = [f"{op} {L} {len(cases)}"] + [to_line(v, L) for t in cases for v in t]
    return run(emu_bin, lines)


def _ldlt_like_cases(L, rng, count):
    """Operands shaped like the trailing update: |x y| within a few bits of |c|
    (Schur-complement cancellation up to ~16 bits), random signs and mantissas."""
    p = 32 * L
    out = []
    for _ in range(count):
        x, y = rnd(L, rng), rnd(L, rng)
        e = x.e + y.e + rng.randint(-16, 16)
        c = rnd(L, rng, e=e)
        out.append((c, x, y))
    return out


@pytest.mark.parametrize("op", ["fused", "fusedw"])
@pytest.mark.parametrize("L", [8, 16, 24, 40])
def test_fused_epilogue_rounding_matches_model(emu_bin, L, op):
    """The rounding fused into the tensor-core epilogue (csrc/tc_fused.cuh),
    fed the short product exactly as k_tc_bulk forms it: every item it
    certifies equals RNE(c - x y) (oracle/mpfloat.py); the rest go to the exact
    redo, and on trailing-update-shaped operands that is rare."""
    rng = random.Random(7000 + L)
    p = 32 * L
    for cases, max_fb in ((fms_cases(L, rng, 300), 0.6), (_ldlt_like_cases(L, rng, 300), 0.08)):
        out = _fused_run(emu_bin, cases, L, op)
        assert len(out) == len(cases)
        fb = 0
        for (c, x, y), r in zip(cases, out):
            assert r != "viol", (c, x, y)
            if r.startswith("fb"):
                fb += 1
                continue
            assert from_line(r, L) == F.fms(c, x, y, p), (c, x, y)
        assert fb <= max_fb * len(cases), fb


@pytest.mark.parametrize("op", ["fused", "fusedw"])
def test_fused_epilogue_edges(emu_bin, op):
    """Binade edges, round-up overflow, ties, tiny / huge products, zero c."""
    L = 16
    p = 32 * L
    rng = random.Random(99)
    cases = []
    for _ in range(200):
        x, y = rnd(L, rng), rnd(L, rng)
        pr = F.mul(x, y, p)
        kind = rng.randrange(7)
        if kind == 0:  # c = -x y rounded: exact-ish doubling
            c = F.MPF(-pr.s, pr.m, pr.e)
        elif kind == 1:  # product far below c
            c = rnd(L, rng, e=pr.e + rng.randint(p, 4 * p))
        elif kind == 2:  # product far above c
            c = rnd(L, rng, e=pr.e - rng.randint(p, 4 * p))
        elif kind == 3:  # c a power of two, product just below half an ulp
            c = F.MPF(rng.choice([1, -1]), 1 << (p - 1), pr.e + rng.randint(1, 8))
        elif kind == 4:  # all-ones c plus a product that rounds it up
            c = F.MPF(pr.s, (1 << p) - 1, pr.e + rng.randint(p - 4, p + 4))
        elif kind == 5:
            c = F.ZERO
        else:  # c = x y exactly representable -> R = 0 or tiny
            c = F.MPF(pr.s, pr.m ^ rng.getrandbits(rng.randint(1, 40)), pr.e)
        cases.append((c, x, y))
    out = _fused_run(emu_bin, cases, L, op)
    for (c, x, y), r in zip(cases, out):
        assert r != "viol", (c, x, y)
        if not r.startswith("fb"):
            assert from_line(r, L) == F.fms(c, x, y, p), (c, x, y)
