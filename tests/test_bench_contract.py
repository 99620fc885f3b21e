"""The bench contract that needs no GPU: `bench.py --impl reference` times the
reference's own CPU implementation (oracle/_ref/ref_driver, the unmodified
reference compiled by oracle/Makefile) and prints exactly ONE JSON line on
stdout carrying the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_driver")):
        pytest.skip("oracle/_ref/ref_driver not built")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = p.stdout.splitlines()
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["unit"] == "MP-FMA/s"
    assert d["config"]["workload"].startswith("C1:") and d["config"]["n"] == 64 and d["config"]["p_bits"] == 3072
    assert d["value"] > 0 and d["steps"] == 1 and d["ms_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and "hankel::compute" in cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the reference's own binary64 lambda_min for C1 (tests/golden/c1.json; K differs, the value does not)
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "c1.json")))
    ref64 = gold["reference_lambda_binary64"]
    ref64 = ref64[0] if isinstance(ref64, list) else ref64
    assert abs(d["lambda_min"] - float(ref64)) < 1e-12 * abs(float(ref64))
