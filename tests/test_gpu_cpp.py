"""The C++ drop-in (include/parfit_b200/parfit.hpp): reference-style client
code (tests/cpp/drop_in_test.cpp) compiled by __graft_entry__.build() and run
on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1311_1753_b200", "_build", "drop_in_test")


@pytest.mark.gpu
def test_cpp_drop_in_client():
    if not os.path.exists(BIN):
        subprocess.check_call(["python", os.path.join(ROOT, "__graft_entry__.py")])
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "golden NLL 3218448.55013740" in r.stdout
    assert "PASSED" in r.stdout
