"""GPU: the C++ host mirror dr_b200:: (include/dr_b200/mesh_raster.hpp) runs the reference's own rasterizer
test cases (proj/tests/test_raster.cpp) and is compared bit for bit with the reference library dr:: in the
same process (tests/cpp/test_raster_cpp.cpp, built by `make cpptest`)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "test_raster_cpp")

pytestmark = pytest.mark.gpu


def test_cpp_mirror_runs_reference_tests(cuda):
    if not os.path.exists(BIN):
        pytest.skip("build/test_raster_cpp not built (needs /root/reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
