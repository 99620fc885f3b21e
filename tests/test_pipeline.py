"""Host drivers mirroring hankel/pipeline.hpp (paper_1810_01478_b200/pipeline.py):
CSV / JSON formats (pipeline.cpp:143-231), the K -> p precision map and argument
checks.  CPU only (the moment generator is host code)."""
import io
import json
import math

import pytest

from paper_1810_01478_b200 import pipeline as P


def test_csv_roundtrip_skips_nan_rows():
    recs = [P.RunRecord(n=500, bits=1024, k=8, workers=1, lambda_=[0.12, 1.1, 33.5], trunc_err=[-1e-3, -2e-3, -3e-3],
                        required_bits=1024, wall_s=1.5),
            P.RunRecord(n=600, bits=2048, k=8, workers=1, lambda_=[float("nan")] * 3, trunc_err=[float("nan")] * 3)]
    f = io.StringIO()
    P.write_scan_csv(f, recs)
    text = f.getvalue()
    assert text.splitlines()[0] == P.CSV_HEADER
    assert text.splitlines()[1].startswith("500,1/2,1024,8,1,0.12,-0.001,1.1000000000000001,")
    assert P.read_scan_csv(io.StringIO(text)) == [(500.0, 0.12)]


@pytest.mark.parametrize("bad,msg", [("", "empty"), ("N,x\n1,2\n", "header"), ("N,lambda1\n5\n", "short row"),
                                     ("N,lambda1\n5,abc\n", "unparseable")])
def test_csv_schema_errors(bad, msg):
    with pytest.raises(ValueError, match=msg):
        P.read_scan_csv(io.StringIO(bad))


def test_json_matches_reference_keys():
    r = P.RunRecord(n=64, bits=2048, k=8, workers=1, lambda_=[1.0], trunc_err=[-1.0], required_bits=2048, p=3072)
    j = json.loads(P.to_json(r))
    assert j["N"] == 64 and j["beta"] == "1/2" and j["required_bits"] == 2048
    assert set(j["timing"]) == {"wall_s", "ldlt_s", "transpose_s", "invL_s", "invL_arith_s", "invL_comm_s", "invH_s",
                                "eigen_s"}


def test_moment_bits_exact_and_precision_map():
    # mu_j = 2 (2j+1)! for beta = 1/2: bit length of mu_{2N-2} = 2 * (4N-3)!
    for n in (8, 64, 500):
        want = (2 * math.factorial(4 * n - 3)).bit_length()
        assert P.moment_bits((1, 2), n) == want
        p = P.precision_bits((1, 2), n, 1024)
        assert p % 128 == 0 and want + 2048 <= p < want + 2048 + 128


def test_compute_argument_errors():
    for kw in ({"n": 0}, {"bits": 0}, {"workers": 0}, {"k": 0}):
        with pytest.raises(ValueError):
            P.compute(P.ComputeOptions(**kw))


def _random_records(rng, count):
    import struct

    def rd():
        r = rng.random()
        if r < 0.05:
            return 0.0
        if r < 0.08:
            return -0.0
        if r < 0.12:
            return float("nan")
        if r < 0.2:  # integers and short decimals
            return float(rng.choice([1, 2, 10, 1000, 123456789012345, 10 ** 15, 10 ** 16])) * rng.choice([1, -1])
        if r < 0.3:
            return rng.choice([1e-4, 1e-5, 0.5, 0.1, 0.001234, 12.34, 1.5e15, 9.99e14]) * rng.choice([1, -1])
        bits = rng.getrandbits(64)  # any finite double
        v = struct.unpack("<d", struct.pack("<Q", bits))[0]
        while v != v or v in (float("inf"), float("-inf")):
            v = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
        return v if rng.random() < 0.5 else v * 10.0 ** rng.randint(-30, 30)

    recs = []
    for _ in range(count):
        nl, nt = rng.randint(0, 3), rng.randint(0, 3)
        rec = P.RunRecord(n=rng.randint(1, 5000), beta=rng.choice([(1, 2), (1, 1), (1, 3), (2, 3)]),
                          bits=rng.randint(64, 20000), k=rng.randint(1, 16), workers=rng.randint(1, 64),
                          lambda_=[rd() for _ in range(nl)], trunc_err=[rd() for _ in range(nt)],
                          required_bits=rng.choice([0, 0, 1024, 4096]))
        for f in ("wall_s", "ldlt_s", "transpose_s", "invL_s", "invL_arith_s", "invL_comm_s", "invH_s", "eigen_s"):
            setattr(rec, f, abs(rd()) if rng.random() < 0.9 else rd())
        recs.append(rec)
    return recs


def _record_line(r):
    vals = [r.wall_s, r.ldlt_s, r.transpose_s, r.invL_s, r.invL_arith_s, r.invL_comm_s, r.invH_s, r.eigen_s]
    h = lambda v: "nan" if v != v else float.hex(v)  # noqa: E731
    return " ".join([str(r.n), str(r.beta[0]), str(r.beta[1]), str(r.bits), str(r.k), str(r.workers),
                     str(r.required_bits), str(len(r.lambda_))] + [h(v) for v in r.lambda_] +
                    [str(len(r.trunc_err))] + [h(v) for v in r.trunc_err] + [h(v) for v in vals])


def test_run_record_writers_byte_identical_to_reference():
    """to_csv_row / to_json of the C++ facade (build/record_fmt) and of
    pipeline.py are byte-identical to the reference's own writers
    (pipeline.cpp:150-160, 213-232; oracle/_ref/ref_driver record) on random
    records: every magnitude, NaN (null / nan), signed zero, missing lambdas."""
    import random
    import subprocess

    import os

    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    fmt = os.path.join(ROOT, "build", "record_fmt")
    if not (os.path.exists(ref) and os.path.exists(fmt)):
        pytest.skip("oracle/_ref or build/record_fmt not built")
    recs = _random_records(random.Random(2024), 400)
    inp = "\n".join(_record_line(r) for r in recs) + "\n"
    want = subprocess.run([ref, "record"], input=inp, capture_output=True, text=True, check=True).stdout
    got = subprocess.run([fmt], input=inp, capture_output=True, text=True, check=True).stdout
    blocks_w, blocks_g = want.split("\n@@\n"), got.split("\n@@\n")
    assert len(blocks_w) == len(recs) + 1
    for r, bw, bg in zip(recs, blocks_w, blocks_g):
        assert bg == bw, (r, bg, bw)
        csv_row, js = bw.split("\n", 1)
        assert P.to_csv_row(r) == csv_row
        assert P.to_json(r) == js
