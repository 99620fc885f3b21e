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
