"""`python -m paper_1311_1753_b200 bench`: the reference's `parfit bench`
contract (proj/tools/parfit_cli.cpp:110-182, tests/cli_smoke.sh:48-61) with GPU
counts in place of thread counts."""
import os
import subprocess
import sys

import pytest

from paper_1311_1753_b200 import cli
from paper_1311_1753_b200 import parfit as pf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- arity gate and report shape (no GPU) -----------------------------------

def test_bench_rejects_fewer_than_three_repetitions():
    with pytest.raises(pf.Error, match="bad-arity"):
        cli.cmd_bench("C1", [1, 2], 2)


@pytest.mark.parametrize("counts", [[2, 4], [1], [1, 1]])
def test_bench_needs_two_counts_including_one(counts):
    with pytest.raises(pf.Error, match="bad-arity"):
        cli.cmd_bench("C1", counts, 3)


def test_bench_cli_exit_code_on_bad_arity():
    p = subprocess.run([sys.executable, "-m", "paper_1311_1753_b200", "bench", "--gpus", "2", "4"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode == 2 and "bad-arity" in p.stderr


def test_report_format_and_unit_speedup():
    rows = [{"gpus": 1, "median_s": 0.5, "metric_value": 1.0, "metric_calls": 40},
            {"gpus": 2, "median_s": 0.25, "metric_value": 1.0, "metric_calls": 40}]
    lines = cli.format_report(rows).splitlines()
    assert lines[0] == "backend gpus time_s speedup metric_calls"
    assert len(lines) == 3
    f1, f2 = lines[1].split(), lines[2].split()
    assert f1[:2] == ["gpus", "1"] and f1[3] == "1" and f1[4] == "40"
    assert f2[:2] == ["gpus", "2"] and float(f2[3]) == 2.0


# ---- on the GPU -------------------------------------------------------------

@pytest.mark.gpu
def test_bench_rows_one_gpu_deterministic():
    rows = cli.bench_rows("C1", [1], 3, n_events=20_000)
    assert len(rows) == 1 and rows[0]["gpus"] == 1
    assert rows[0]["metric_calls"] > 0 and rows[0]["median_s"] > 0
    # a second pass from the same start lands on the bitwise-identical metric
    assert cli.bench_rows("C1", [1], 3, n_events=20_000)[0]["metric_value"] == rows[0]["metric_value"]


@pytest.mark.gpu
def test_bench_full_command(tmp_path):
    import torch
    out = tmp_path / "bench.txt"
    if torch.cuda.device_count() >= 2:
        assert cli.cmd_bench("C1", [1, 2], 3, n_events=20_000, out_path=str(out)) == 0
        lines = out.read_text().splitlines()
        assert lines[0] == "backend gpus time_s speedup metric_calls" and len(lines) == 3
        assert lines[1].split()[3] == "1"
    else:  # one GPU: refused up front, before any fit, with the visible count
        with pytest.raises(pf.Error) as ei:
            cli.cmd_bench("C1", [1, 2], 3, n_events=20_000, out_path=str(out))
        assert ei.value.args[0].startswith("bad-backend") and "1 visible" in str(ei.value)


def test_bench_rejects_non_power_of_two_counts_up_front():
    """the engine shards over powers of two; the CLI says so before any work"""
    with pytest.raises(pf.Error) as ei:
        cli.cmd_bench("C1", [1, 3], 3, n_events=1000)
    assert ei.value.args[0].startswith("bad-backend") and "powers of two" in str(ei.value)


@pytest.mark.gpu
def test_bench_full_command_oversubscribed_counts(tmp_path):
    """`parfit bench --gpus 1 2 4 --oversubscribe` on however many GPUs there
    are: the multi-device shards run (round-robin placed), the bitwise
    determinism gate across counts holds, and the report has one row per count"""
    out = tmp_path / "bench.txt"
    assert cli.cmd_bench("C1", [1, 2, 4], 3, n_events=20_000, out_path=str(out), oversubscribe=True) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "backend gpus time_s speedup metric_calls" and len(lines) == 4
    assert [ln.split()[1] for ln in lines[1:]] == ["1", "2", "4"]
    assert len({ln.split()[4] for ln in lines[1:]}) == 1  # same fit, same call count, every count
