"""bench.py's CPU-side legs (no GPU): the reference arm and the cpu_baseline
measurement for every BASELINE workload, at tiny sizes, plus the JSON keys
the driver reads from the reference arm."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402
from paper_1311_1753_b200 import parfit as pf  # noqa: E402
from paper_1311_1753_b200.workloads import WORKLOADS  # noqa: E402


@pytest.mark.parametrize("name", sorted(WORKLOADS))
def test_cpu_side_leg(name):
    W = WORKLOADS[name]
    obs, pdf = W.build(pf)
    if W.unit == "bins":
        cols = np.zeros((1, 300))
    else:
        cols = W.columns(3000, seed=2)
    out, _ = bench.cpu_side(W, pf, obs, pdf, cols, W.metric, fit=False, steps=1)
    assert out["value"] > 0 and out["unit"] == f"{W.unit}/s"
    assert out["kind"] in ("reference", "port") and out["cores"] >= 1
    if name == "C3":
        assert out["kind"] == "port"  # ArgusPdf: no reference code


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_reference_arm_json(name):
    if name != "C3" and not oracle.Reference.available():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", name,
                        "--events", "2000", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
