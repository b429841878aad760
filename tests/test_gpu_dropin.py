"""The C++ face (include/ifgf_b200.hpp) as a drop-in: the reference's own CombinedOperator
and GpuCombinedOperator built from the same ifgf::SurfaceMesh / ifgf::SolveConfig, the GPU
operator driven by the reference's gmres_solve (tests/cpp/drop_in_test.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "drop_in_test")


def test_cpp_drop_in():
    if not os.path.exists(BIN):
        pytest.skip("drop_in_test not built (make -C oracle, needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "0 failure(s)" in p.stdout
