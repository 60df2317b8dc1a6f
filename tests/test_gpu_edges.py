"""Edge cases of the batched GPU API against the CPU oracle: empty and ragged
query batches (the reference's per-query API has no batch size; its callers
loop, proj/src/renderer.cpp:106-231), batches that straddle a warp boundary,
zero-area points (bhtree.cpp:205 skips far sources with area 0) and queries
that coincide with points (bhtree.cpp:219,387)."""
import numpy as np
import pytest
from parity import check, scalar
from test_gpu_parity import make, random_cloud

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    import paper_2405_16788_b200 as P

    return P


@pytest.mark.parametrize("C", [3, 49])
def test_empty_batch_is_a_no_op(eng, oracle_mod, C):
    pos, nrm, area, mu = random_cloud(500, 40, C)
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t, _ = make(eng, oracle_mod, pos, nrm, area, mu, kinds)
    p = eng.KernelParams(epsilon=0.05)
    out = t.primal(np.zeros((0, 3)), p, 2.0)
    assert out.shape == (0, C)
    buf = t.make_buffer()
    t.adjoint(np.zeros((0, 3)), p, 2.0, np.zeros((0, C), np.float32), None, buf)
    g = t.flush_gradients(buf)
    assert not np.any(g.moments) and not np.any(g.normals) and g.d_epsilon == 0.0


@pytest.mark.parametrize("q", [1, 31, 33, 127, 129])
@pytest.mark.parametrize("C", [3, 49])
def test_ragged_batches(eng, oracle_mod, q, C):
    """Batch sizes around the 32-query warp and the 128-query block: the padded
    lanes of the last warp must neither read nor contribute anything."""
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(2000, 41, C)
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    rng = np.random.default_rng(42 + q)
    xs = rng.uniform(-1.3, 1.3, (q, 3))
    d_out = rng.standard_normal((q, C)).astype(np.float32)
    p, rp = eng.KernelParams(epsilon=0.05), O.Params(0.05)
    for rep in range(2):  # the second pass replays the first one's interaction lists
        got, want = t.primal(xs, p, 2.0), r.primal_mag(rp, 2.0, xs)
        check(f"ragged q={q} C={C} primal (pass {rep})", got, want["out"], want["out_abs"])
        buf = t.make_buffer()
        t.adjoint(xs, p, 2.0, d_out, None, buf)
        g = t.flush_gradients(buf)
        w = r.adjoint_mag(rp, 2.0, xs, d_out.astype(np.float64))
        check(f"ragged q={q} C={C} moments (pass {rep})", g.moments, w["moments"], w["moments_abs"])
        check(f"ragged q={q} C={C} normals (pass {rep})", g.normals, w["normals"], w["normals_abs"])
        scalar(f"ragged q={q} C={C} d_eps (pass {rep})", g.d_epsilon, w["d_eps"], w["d_eps_abs"])


def test_zero_area_points_and_coincident_queries(eng, oracle_mod):
    """A third of the points carry area 0 (their nodes' far field is skipped when
    the whole node has area 0, bhtree.cpp:205) and a third of the queries sit
    exactly on points (the singular term is skipped, :219 / :387)."""
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(3000, 43, 5)
    area = area.copy()
    area[::3] = 0.0
    area[:64] = 0.0  # whole leaves without area
    kinds = np.array([0, 1, 1, 1, 1], np.uint8)
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    rng = np.random.default_rng(44)
    xs = rng.uniform(-1.2, 1.2, (600, 3))
    xs[::3] = pos[rng.integers(0, 3000, 200)]
    d_out = rng.standard_normal((600, 5)).astype(np.float32)
    for eps in (0.05, 0.0):  # regularized and singular kernels
        p, rp = eng.KernelParams(epsilon=eps), O.Params(eps)
        got, want = t.primal(xs, p, 2.0), r.primal_mag(rp, 2.0, xs)
        check(f"zero-area / coincident primal eps={eps}", got, want["out"], want["out_abs"])
        buf = t.make_buffer()
        t.adjoint(xs, p, 2.0, d_out, None, buf)
        g = t.flush_gradients(buf)
        w = r.adjoint_mag(rp, 2.0, xs, d_out.astype(np.float64))
        check(f"zero-area / coincident moments eps={eps}", g.moments, w["moments"], w["moments_abs"])
        check(f"zero-area / coincident normals eps={eps}", g.normals, w["normals"], w["normals_abs"])
