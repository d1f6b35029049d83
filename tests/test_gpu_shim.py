"""The C++ drop-in (include/sgweno_gpu.hpp) against the reference, through the
reference's own public API (oracle/shim_test.cpp, built by oracle/Makefile
where the reference headers exist; the binary travels with the snapshot)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_test")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/shim_test not built")
def test_cpp_shim_bitwise_vs_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("EQUAL") == 5
