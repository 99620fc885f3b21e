"""Dev tool (GPU box): the paper's Table 2 rows beyond the test suite's N = 500 /
1000 — auto_precision (pipeline.cpp:74-94, re-targeted to p-bit floats by
paper_1810_01478_b200/pipeline.py) at N = 1500, 2000, compared with the
published lambda_1..3 and required bits (reference_data.hpp rows, committed in
tests/golden/table2.json).  Writes one JSON line per N.

    python tools/table2_run.py 1500 2000 > profiles/r01_table2_large.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1810_01478_b200 import pipeline as P  # noqa: E402

gold = json.load(open(os.path.join(ROOT, "tests", "golden", "table2.json")))
for n in [int(a) for a in sys.argv[1:]] or [1500]:
    want = next(r for r in gold["rows"] if r["n"] == n)
    t = time.time()
    bits, rec = P.auto_precision(P.ComputeOptions(n=n, beta=(1, 2), k=8))
    wall = time.time() - t
    out = {"n": n, "beta": "1/2", "k": 8, "required_bits": bits, "reference_required_bits": want["required_bits"],
           "p_bits": rec.p, "lambda": rec.lambda_, "reference_lambda": want["lam"],
           "abs_err": [abs(a - b) for a, b in zip(rec.lambda_, want["lam"])],
           "rel_err": [abs(a - b) / abs(b) for a, b in zip(rec.lambda_, want["lam"])],
           "trunc_err": rec.trunc_err, "lambda_hi_lo": [[h, lo] for h, lo in zip(rec.lambda_hi, rec.lambda_lo)],
           "last_compute_s": {"wall": rec.wall_s, "ldlt": rec.ldlt_s, "invL": rec.invL_s, "invH": rec.invH_s,
                              "eigen": rec.eigen_s},
           "auto_precision_wall_s": wall}
    print(json.dumps(out), flush=True)
