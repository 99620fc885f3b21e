"""GPU: the reference's acceptance check against the paper's Table 2
(proj/tests/acceptance.cpp:76-131; rows from reference_data.hpp:23-33, fixture
tests/golden/table2.json made by tests/golden/make_table2.py).  auto_precision
(pipeline.cpp:74-94) re-targeted to the p-bit float (pipeline.py) must land on
the published lambda_1..lambda_3 within the acceptance tolerances, with negative
truncation-error estimates."""
import json
import os

import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "table2.json")


@pytest.fixture(scope="module")
def table2():
    return json.load(open(GOLD))


def row(table2, n):
    return next(r for r in table2["rows"] if r["n"] == n)


def test_table2_n500(table2):
    from paper_1810_01478_b200 import pipeline as P

    bits, rec = P.auto_precision(P.ComputeOptions(n=500, beta=(1, 2), k=8))
    want, tol = row(table2, 500), table2["tolerances"]["n500"]
    for i in range(3):
        assert abs(rec.lambda_[i] - want["lam"][i]) <= tol[i], (i, rec.lambda_[i], want["lam"][i])
    assert all(t < 0 for t in rec.trunc_err)
    # the search settles at the reference's K (acceptance.cpp:116-122)
    assert bits == want["required_bits"]
    assert rec.required_bits == bits


def test_table2_n1000(table2):
    from paper_1810_01478_b200 import pipeline as P

    bits, rec = P.auto_precision(P.ComputeOptions(n=1000, beta=(1, 2), k=8))
    want, tol = row(table2, 1000), table2["tolerances"]["n1000"]
    assert abs(rec.lambda_[0] - want["lam"][0]) <= tol[0], (rec.lambda_[0], want["lam"][0])
    assert all(t < 0 for t in rec.trunc_err)
    assert bits == want["required_bits"]
