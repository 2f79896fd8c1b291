"""GPU: the C++ drop-in (libcbct_b200.so, namespace cbct) exercised by a
reference-style C++ program compiled against include/cbct/*.hpp
(tests/cpp/dropin_test.cpp, built by `make -C paper_2110_09841_b200/csrc`)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_test")


def test_reference_style_cpp_caller_runs_on_the_gpu():
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/dropin_test not built (run __graft_entry__.build())")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN PASS" in r.stdout
