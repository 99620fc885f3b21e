"""GPU: the bench contract of the repo's own arm — exactly one JSON line on
stdout with the keys the driver reads — on the smallest config, on one GPU and
through the NCCL column-sharded path with a world of one (every call of the
step collective; NCCL's own prints must not reach stdout)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [[], ["--sharded"]])
def test_bench_prints_one_json_line(extra):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "2", "--warmup", "3",
                        "--no-cpu-baseline"] + extra, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = p.stdout.splitlines()
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["unit"] == "MP-FMA/s" and d["higher_is_better"] is True and d["n_gpus"] == 1 and d["steps"] == 2
    assert d["config"]["workload"].startswith("C1:") and d["value"] > 0 and d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] in ("imad", "tensor", "hbm") and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["parity"]["lambda1_digits_vs_reference"] >= d["parity"]["required_digits"]
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
