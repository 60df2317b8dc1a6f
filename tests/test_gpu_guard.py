"""Out-of-bounds-write check of every kernel family (compute-sanitizer is
closed on the GPU pool — running it left GPUs needing a reset — so the engine
carries its own detector): with DPL_GUARD=1 every engine allocation has 4 KB
guard zones filled with a pattern, verified after each phase of
tools/sanitize_case.py (tree build, fused and list-replay forward / adjoint,
host-batch staging, gradient forward, both flushes, Adam, render with the
direct-rgb and the tcgen05 tiny-MLP heads, sampling). The detector's positive
control writes past the end of a buffer and must be caught."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code, **extra):
    env = dict(os.environ, DPL_GUARD="1", **extra)
    return subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                          timeout=600, cwd=ROOT)


def test_guard_detector_positive_control():
    r = _run("from paper_2405_16788_b200._lib import check, lib; check(lib().dpl_guard_selftest()); print('ok')")
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("extra", [{}, {"DPL_ADJOINT_TMEM": "1"}, {"DPL_FORWARD_TMEM": "1"},
                                   {"DPL_MLP_RECOMPUTE": "1"}],
                         ids=["default", "tmem-adjoint", "tmem-forward", "mlp-recompute"])
def test_no_out_of_bounds_writes_in_any_kernel_family(extra):
    """Default kernels, then the opt-in tcgen05 / TMEM adjoint and forward and the head
    backward's recompute path under the same guard zones."""
    r = _run("import runpy; runpy.run_path('tools/sanitize_case.py', run_name='__main__')", **extra)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "guard zones intact" in r.stdout, r.stdout
