"""The C++ mirror (include/dipole_b200.hpp) used the way the reference's own
code uses DipoleTree, compiled against libdipole_b200.so (tests/cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "test_cpp_api")


def test_cpp_drop_in_api():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.dirname(BIN)], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "passed" in r.stdout
