"""Host-side drivers mirroring the reference's `hankel/pipeline.hpp` on top of the
device path (`api.Context`): `compute`, `auto_precision`, `scan` and the scan-CSV
writer/reader (pipeline.cpp:26-245).

Precision: the reference works in fixed point with K fractional bits (2K inside
the LDLT, pipeline.hpp:19).  Here every value is a p-bit float; K maps to the
smallest p that holds every moment exactly AND keeps 2K fraction bits on the
largest one:

    p(K) = 32 L,  L = ceil((bits(mu_{2N-2}) + 2K) / 128) * 4

(L a multiple of 4 so the tensor-core path applies).  Relative precision makes
every smaller entry at least as precise as the reference's fixed point.  The
search, its defaults and its agreement test are the reference's
(`auto_precision`, pipeline.cpp:74-94; AutoPrecisionOptions, pipeline.hpp:52-57).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from . import api


@dataclass
class ComputeOptions:
    """pipeline.hpp:16-23 (`workers` = GPUs; `bits` = the reference's K)."""

    n: int = 1
    beta: tuple = (1, 2)
    bits: int = 1024
    k: int = 8
    workers: int = 1
    device: int = 0
    device_moments: bool = True  # even 2/beta: hk_generate_moments instead of host build_hankel + upload


@dataclass
class AutoPrecisionOptions:
    """pipeline.hpp:52-57."""

    start_bits: int = 0  # 0 -> 1024 * ceil(n / 500)
    step_bits: int = 1024
    max_bits: int = 16384
    agree_tol: float = 1e-15


@dataclass
class RunRecord:
    """pipeline.hpp:28-48, plus p (the float precision used) and the ~32-digit lambda."""

    n: int = 0
    beta: tuple = (1, 2)
    bits: int = 0
    k: int = 0
    workers: int = 0
    lambda_: list = field(default_factory=list)  # binary64, ascending (up to 3)
    trunc_err: list = field(default_factory=list)
    required_bits: int = 0
    wall_s: float = 0.0
    ldlt_s: float = 0.0
    transpose_s: float = 0.0
    invL_s: float = 0.0
    invL_arith_s: float = 0.0
    invL_comm_s: float = 0.0
    invH_s: float = 0.0
    eigen_s: float = 0.0
    p: int = 0
    lambda_hi: list = field(default_factory=list)
    lambda_lo: list = field(default_factory=list)

    def lambda1(self) -> float:
        return self.lambda_[0]


def moment_bits(beta: tuple, n: int) -> int:
    """Bit length of the largest moment mu_{2n-2} (exact, from the moment generator)."""
    num, den = beta
    j = 2 * n - 2
    est = (math.lgamma((j + 1) * den / num) + math.log(den / num)) / math.log(2)
    L = int(est // 32) + 4
    mu, exact = api.build_hankel(beta, n, L)
    if not exact and (2 * den // num) % 2 == 0:  # odd 2/beta: rounded half-integer Gamma values
        raise api.PrecisionError("moment_bits: estimate too small")
    return int(mu.exps[-1])


def precision_bits(beta: tuple, n: int, K: int) -> int:
    """p(K) (module docstring)."""
    return 128 * math.ceil((moment_bits(beta, n) + 2 * K) / 128)


def compute(opts: ComputeOptions) -> RunRecord:
    """hankel::compute (pipeline.cpp:26-72) at the p equivalent to K = opts.bits."""
    if opts.n < 1:
        raise ValueError("compute: need N >= 1")
    if opts.bits < 1:
        raise ValueError("compute: need bits >= 1")
    if opts.workers < 1:
        raise ValueError("compute: need workers >= 1")
    if opts.k < 1:
        raise ValueError("compute: need k >= 1")
    p = precision_bits(opts.beta, opts.n, opts.bits)
    L = p // 32
    even_q = (2 * opts.beta[1] // opts.beta[0]) % 2 == 0
    if opts.device_moments and even_q:  # moments.cpp:113-133 on the device
        with api.Context(L, device=opts.device) as ctx:
            r = ctx.compute_generated(opts.beta, opts.n, opts.k)
            if not ctx.moments_exact:
                raise api.PrecisionError("compute: moments not exact at p bits")
    else:
        mu, exact = api.build_hankel(opts.beta, opts.n, L)
        if not exact and even_q:
            raise api.PrecisionError("compute: moments not exact at p bits")
        with api.Context(L, device=opts.device) as ctx:
            r = ctx.compute(mu, opts.k)
    return RunRecord(n=opts.n, beta=tuple(opts.beta), bits=opts.bits, k=r.k, workers=opts.workers,
                     lambda_=[h + l for h, l in zip(r.lambda_hi, r.lambda_lo)], trunc_err=list(r.trunc_err),
                     wall_s=r.wall_s, ldlt_s=r.ldlt_s, invL_s=r.invL_s, invL_arith_s=r.invL_s, invH_s=r.invH_s,
                     eigen_s=r.eigen_s, p=p, lambda_hi=list(r.lambda_hi), lambda_lo=list(r.lambda_lo))


def auto_precision(base: ComputeOptions, opts: AutoPrecisionOptions | None = None) -> tuple[int, RunRecord]:
    """Smallest K (step multiples from the N heuristic) whose run agrees with the
    K + step run on lambda_1 within agree_tol (pipeline.cpp:74-94)."""
    opts = opts or AutoPrecisionOptions()
    step = opts.step_bits
    k0 = opts.start_bits if opts.start_bits > 0 else step * ((base.n + 499) // 500)
    run = ComputeOptions(**{**base.__dict__, "bits": k0})
    prev = compute(run)
    bits = k0
    while bits <= opts.max_bits:
        run.bits = bits + step
        nxt = compute(run)
        if abs(prev.lambda1() - nxt.lambda1()) <= opts.agree_tol:
            prev.required_bits = bits
            return bits, prev
        prev = nxt
        bits += step
    raise api.PrecisionError(f"auto_precision: no agreement up to {opts.max_bits} bits (step {step})")


def scan(n_list, base: ComputeOptions, auto_bits: bool = False,
         auto_opts: AutoPrecisionOptions | None = None) -> list[RunRecord]:
    """pipeline.cpp:96-122: one record per N; failures become NaN rows."""
    out = []
    for n in n_list:
        run = ComputeOptions(**{**base.__dict__, "n": n})
        try:
            out.append(auto_precision(run, auto_opts)[1] if auto_bits else compute(run))
        except Exception:
            nan = float("nan")
            out.append(RunRecord(n=n, beta=tuple(run.beta), bits=run.bits, k=run.k, workers=run.workers,
                                 lambda_=[nan] * 3, trunc_err=[nan] * 3))
    return out


CSV_HEADER = ("N,beta,bits,k,workers,lambda1,trunc1,lambda2,trunc2,lambda3,trunc3,"
              "required_bits,wall_s,ldlt_s,transpose_s,invL_s,invL_arith_s,invL_comm_s,invH_s,eigen_s")


def _fmt(v: float) -> str:  # std::ostream with precision(17)
    return "nan" if v != v else f"{v:.17g}"


def to_csv_row(r: RunRecord) -> str:
    """pipeline.cpp:150-160 (17 significant digits)."""
    cols = [str(r.n), f"{r.beta[0]}/{r.beta[1]}", str(r.bits), str(r.k), str(r.workers)]
    for i in range(3):
        cols.append(_fmt(r.lambda_[i] if i < len(r.lambda_) else float("nan")))
        cols.append(_fmt(r.trunc_err[i] if i < len(r.trunc_err) else float("nan")))
    cols.append(str(r.required_bits))
    cols += [_fmt(x) for x in (r.wall_s, r.ldlt_s, r.transpose_s, r.invL_s, r.invL_arith_s, r.invL_comm_s,
                               r.invH_s, r.eigen_s)]
    return ",".join(cols)


def write_scan_csv(f, records) -> None:
    f.write(CSV_HEADER + "\n")
    for r in records:
        f.write(to_csv_row(r) + "\n")


def read_scan_csv(f) -> list[tuple[float, float]]:
    """(N, lambda1) points, NaN rows skipped (pipeline.cpp:167-207; errors as schema_error)."""
    lines = f.read().splitlines()
    if not lines:
        raise ValueError("scan CSV: empty input")
    head = lines[0].replace("\r", "").split(",")
    if "N" not in head or "lambda1" not in head:
        raise ValueError("scan CSV: header must contain N and lambda1 columns")
    ni, li = head.index("N"), head.index("lambda1")
    pts = []
    for no, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        fields = line.replace("\r", "").split(",")
        if len(fields) <= max(ni, li):
            raise ValueError(f"scan CSV: short row at line {no}")
        try:
            n, lam = float(fields[ni]), float(fields[li])
        except ValueError:
            raise ValueError(f"scan CSV: unparseable number at line {no}") from None
        if lam == lam:  # NaN rows are failed scan entries
            pts.append((n, lam))
    return pts


_POW10 = None


def _pow10_table():
    """10^k, k = -300 .. 324 step 8, as (64-bit significand rounded to nearest, exponent, k)."""
    global _POW10
    if _POW10 is None:
        from fractions import Fraction

        rows = []
        for k in range(-300, 325, 8):
            v = Fraction(10) ** k
            e = v.numerator.bit_length() - v.denominator.bit_length() - 64
            while v / Fraction(2) ** e >= 2 ** 64:
                e += 1
            while v / Fraction(2) ** e < 2 ** 63:
                e -= 1
            q = v / Fraction(2) ** e
            f = int(q) + (1 if q - int(q) >= Fraction(1, 2) else 0)
            rows.append((f // 2, e + 1, k) if f == 2 ** 64 else (f, e, k))
        _POW10 = rows
    return _POW10


def _grisu2_digits(v: float):
    """Grisu2 (Loitsch 2010), as the reference's JSON writer runs it: digits and
    decimal exponent of v > 0 (round-trip; usually, not always, the shortest)."""
    import struct

    M64 = (1 << 64) - 1

    def mul(x, y):
        ul, uh, vl, vh = x[0] & 0xFFFFFFFF, x[0] >> 32, y[0] & 0xFFFFFFFF, y[0] >> 32
        p0, p1, p2, p3 = ul * vl, ul * vh, uh * vl, uh * vh
        q = (p0 >> 32) + (p1 & 0xFFFFFFFF) + (p2 & 0xFFFFFFFF) + (1 << 31)
        return ((p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32)) & M64, x[1] + y[1] + 64)

    def normalize(x):
        f, e = x
        while f >> 63 == 0:
            f, e = f << 1, e - 1
        return f, e

    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    w = (F, 1 - 1075) if E == 0 else (F + (1 << 52), E - 1075)
    mp = normalize((2 * w[0] + 1, w[1] - 1))
    mm0 = (4 * w[0] - 1, w[1] - 2) if (F == 0 and E > 1) else (2 * w[0] - 1, w[1] - 1)
    mm = (mm0[0] << (mm0[1] - mp[1]), mp[1])
    f = -60 - mp[1] - 1
    t = abs(f * 78913) >> 18
    k = (t if f >= 0 else -t) + (1 if f > 0 else 0)  # C++ truncating division
    cf, ce, ck = _pow10_table()[(300 + k + 7) // 8]
    W, Wm, Wp = mul(normalize(w), (cf, ce)), mul(mm, (cf, ce)), mul(mp, (cf, ce))
    Mm, Mp = Wm[0] + 1, Wp[0] - 1
    dexp = -ck
    delta, dist = Mp - Mm, Mp - W[0]
    ne = -Wp[1]
    one = 1 << ne
    p1, p2 = Mp >> ne, Mp & (one - 1)
    n, pow10 = 1, 1
    for d in range(10, 1, -1):
        if p1 >= 10 ** (d - 1):
            n, pow10 = d, 10 ** (d - 1)
            break
    buf = []

    def round_last(dist, delta, rest, ten_k):
        while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
            buf[-1] -= 1
            rest += ten_k

    while n > 0:
        buf.append(p1 // pow10)
        p1 %= pow10
        n -= 1
        rest = (p1 << ne) + p2
        if rest <= delta:
            round_last(dist, delta, rest, pow10 << ne)
            return "".join(map(str, buf)), dexp + n
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        buf.append(p2 >> ne)
        p2 &= one - 1
        m += 1
        delta, dist = delta * 10, dist * 10
        if p2 <= delta:
            break
    round_last(dist, delta, p2, one)
    return "".join(map(str, buf)), dexp - m


def _json_number(v: float) -> str:
    """A double as the reference's JSON writer (nlohmann::json::dump) prints it:
    Grisu2 digits, positional between 1e-4 and 1e15, else d.ddde+XX; non-finite -> null."""
    import math

    if v != v or math.isinf(v):
        return "null"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0:
        return sign + "0.0"
    digits, dexp = _grisu2_digits(abs(v))
    k = len(digits)
    n = k + dexp
    if k <= n <= 15:
        out = digits + "0" * (n - k) + ".0"
    elif 0 < n <= 15:
        out = digits[:n] + "." + digits[n:]
    elif -4 < n <= 0:
        out = "0." + "0" * (-n) + digits
    else:
        e = n - 1
        out = digits[0] + ("." + digits[1:] if k > 1 else "") + ("e-" if e < 0 else "e+") + f"{abs(e):02d}"
    return sign + out


def _json_array(v) -> str:
    if not v:
        return "[]"
    return "[\n" + ",\n".join("    " + _json_number(x) for x in v) + "\n  ]"


def to_json(r: RunRecord) -> str:
    """pipeline.cpp:213-232 byte for byte (the reference's nlohmann::json object,
    keys sorted, dump(2))."""
    parts = [f'"N": {r.n}', f'"beta": "{r.beta[0]}/{r.beta[1]}"', f'"bits": {r.bits}', f'"k": {r.k}',
             f'"lambda": {_json_array(r.lambda_)}']
    if r.required_bits > 0:
        parts.append(f'"required_bits": {r.required_bits}')
    timing = (("eigen_s", r.eigen_s), ("invH_s", r.invH_s), ("invL_arith_s", r.invL_arith_s),
              ("invL_comm_s", r.invL_comm_s), ("invL_s", r.invL_s), ("ldlt_s", r.ldlt_s),
              ("transpose_s", r.transpose_s), ("wall_s", r.wall_s))
    parts.append('"timing": {\n' + ",\n".join(f'    "{k}": {_json_number(v)}' for k, v in timing) + "\n  }")
    parts.append(f'"trunc_err": {_json_array(r.trunc_err)}')
    parts.append(f'"workers": {r.workers}')
    return "{\n" + ",\n".join("  " + x for x in parts) + "\n}"


def to_json_ext(r: RunRecord) -> str:
    """to_json plus this build's extras: p and the (hi, lo) pairs of the ~32-digit lambdas."""
    import json

    j = json.loads(to_json(r))
    j["p_bits"] = r.p
    j["lambda_hi_lo"] = [[h, lo] for h, lo in zip(r.lambda_hi, r.lambda_lo)]
    return json.dumps(j, indent=2)
