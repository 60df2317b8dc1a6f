"""Render step with the tiny-MLP radiance head (radiance.cpp:40-180,
renderer.cpp:106-231) against the reference's own implementation (oracle/_ref,
HeadVariant::TinyMlp): colours, point gradients, d_epsilon, d_lambda,
d_background and the head-weight gradient RenderGrads::d_head_w."""
import numpy as np
import pytest

from parity import check, scalar
from test_gpu_parity import make

pytestmark = pytest.mark.gpu


def he_weights(sizes, seed):
    """Mlp::init's He initialisation (radiance.cpp:44-57) with numpy draws."""
    rng = np.random.default_rng(seed)
    w = []
    for cols, rows in zip(sizes[:-1], sizes[1:]):
        w.append(np.sqrt(2.0 / cols) * rng.standard_normal(rows * cols))
        w.append(0.05 * rng.standard_normal(rows))  # non-zero biases exercise db
    return np.concatenate(w)


@pytest.mark.parametrize("hidden", [(32,), (64, 64), (256, 256)])
def test_render_step_tiny_mlp_head(oracle_mod, hidden):
    import paper_2405_16788_b200 as eng
    from paper_2405_16788_b200 import renderer as Rn
    from paper_2405_16788_b200 import workloads as W

    O = oracle_mod
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    w = W.config3(scale=0.02)
    c = w["cloud"]
    t, _ = make(eng, O, c.positions, c.normals, c.areas, c.moments, w["kinds"])
    eps = 1.5 * O.mean_knn_spacing(c.positions)
    K = c.channels - 1
    sizes = [22 + K, *hidden, 3]
    wts = he_weights(sizes, 5)
    t.set_mlp_head(sizes, wts)
    ref = O.RefModel(O.Cloud(c.positions, c.normals, c.areas, c.moments), eps, lam=20.0, beta=2.0)
    ref.set_mlp_head(sizes, wts)

    rays = w["rays"][:192]
    S = 32
    target = w["target"][:192]
    rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=3)
    p = eng.KernelParams(epsilon=eps)
    rgb, tape = Rn.render_forward(t, p, rs, rays, S)
    # L = (1/3) sum ||rgb - target||^2 (no batch mean: O(1) gradients, so the
    # 1e-6 absolute floor does not hide them); both sides use the reference's
    # colours for the loss gradient, the GPU colours are checked on their own
    scale = 2.0 / 3.0
    ts, dlt = O.stratified_samples(rays.shape[0], S, 2.0, 6.0, 3)
    want = ref.render_step(rays, ts, dlt, target, scale)
    d_rgb = (scale * (want["rgb"] - target)).astype(np.float32)
    buf = t.make_buffer()
    dl, dbg = Rn.render_backward(t, p, rs, tape, d_rgb, buf)
    g = t.flush_gradients(buf)
    dw = t.head_grads()
    tag = f"tiny-MLP head {sizes}"
    check(f"{tag} rgb", rgb, want["rgb"])
    check(f"{tag} moments", g.moments, want["moments"])
    check(f"{tag} normals", g.normals, want["normals"])
    scalar(f"{tag} d_epsilon", g.d_epsilon, want["d_eps"])
    scalar(f"{tag} d_lambda", dl, want["d_lambda"], atol=1e-8)
    check(f"{tag} d_background", dbg, want["d_bg"], atol=1e-8)
    check(f"{tag} d_head_w (RenderGrads::d_head_w)", dw, ref.head_grads())
    # the accumulator was reset; the direct-rgb head is restored by an empty size list
    assert np.all(t.head_grads() == 0)
    t.set_mlp_head((), ())
    rgb2, _ = Rn.render_forward(t, p, rs, rays, S)
    assert not np.allclose(rgb2, rgb)


def test_recompute_path_of_the_head_backward():
    """DPL_MLP_RECOMPUTE=1 (the path taken when HBM cannot hold the forward's
    activations on the render tape): the head backward recomputes them chunk by
    chunk and passes the same reference-TinyMlp parity tests."""
    import os
    import subprocess
    import sys

    r = subprocess.run(
        [sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-x", "-m", "gpu",
         "-k", "tiny_mlp_head"],
        env=dict(os.environ, DPL_MLP_RECOMPUTE="1"), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
