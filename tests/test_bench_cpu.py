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
    ds = W.data(pf, obs, 300 if W.unit == "bins" else 3000, seed=2)
    out, parity = bench.cpu_side(W, pf, obs, pdf, ds, W.metric, gpu_value=1.0, steps=1)
    assert out["value"] > 0 and out["unit"] == f"{W.unit}/s"
    assert out["kind"] in ("reference", "port") and out["cores"] >= 1
    assert parity["units"] == (300 if W.unit == "bins" else 3000) and np.isfinite(parity["ref_value"])
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
    assert np.isfinite(line["metric_value"])


def test_reference_arm_never_maps_the_product_library():
    """the reference arm times the reference alone: libpfb200.so must not be
    mapped into its process (the product binding is lazy)"""
    if not oracle.Reference.available():
        pytest.skip("oracle/_ref not built")
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'C2', "
            "'--events', '3000', '--steps', '1', '--warmup', '0']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT_MAPPED' if 'libpfb200' in maps else 'CLEAN', 'REF' if 'libparfit_ref' in maps else 'NOREF')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().splitlines()[-1] == "CLEAN REF", r.stdout


def test_both_arms_share_one_config_dict():
    """the driver compares `config` of the two arms byte for byte"""
    W = WORKLOADS["C2"]
    a = json.dumps(bench.workload_config(W, 10_000_000, 10_000_000, 1, None), sort_keys=True)
    b = json.dumps(bench.workload_config(W, *bench.sizes(W, bench.argparse.Namespace(events=0), 1, 0), 1, None),
                   sort_keys=True)
    assert a == b
