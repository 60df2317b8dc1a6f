"""The reference's OWN hot-path tests against our drop-in dipole::DipoleTree.

oracle/Makefile (target `dropin`, run by __graft_entry__.build() where the
reference sources exist) compiles /root/reference/proj/tests/test_bhtree.cpp
and test_fields.cpp — every TEST_CASE, fp64 tolerances replaced by the fp32
bar where the GPU's arithmetic meets fp64 naive sums (substitution table in
INTEGRATION.md) — against include/dropin/dipole/bhtree.hpp, with the
reference's callers (fields.cpp, oracles.cpp, ...) compiled unmodified against
the same header and the tree itself provided by bhtree_b200.cpp over
libdipole_b200.so. The binary travels to the GPU box prebuilt."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin", "dropin_tests")


def test_reference_bhtree_and_fields_tests_on_the_drop_in_tree():
    if not os.path.exists(BIN):
        pytest.skip("drop-in test binary not built (needs the reference sources: make -C oracle dropin)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out)
    assert m, out[-3000:]
    total, passed, failed = map(int, m.groups())
    assert r.returncode == 0 and failed == 0, out[-4000:]
    assert total >= 24  # 16 test_bhtree.cpp + 8 test_fields.cpp cases
