"""GPU: the C++ drop-in shim (include/kryct_b200.hpp) used from C++ with the
reference's own types, solvers and error taxonomy (tests/cpp/test_shim.cpp,
prebuilt into oracle/_ref/test_shim by `make -C oracle shim`)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_shim")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="shim test not built (make -C oracle shim)")
def test_cpp_shim_against_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL OK" in r.stdout
