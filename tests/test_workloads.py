"""Synthetic BASELINE-config generators: determinism, shapes, recorded eps."""
import numpy as np

from paper_2405_16788_b200 import workloads as W


def test_config1_shapes_and_determinism():
    a, b = W.config1(scale=0.01), W.config1(scale=0.01)
    assert np.array_equal(a["cloud"].positions, b["cloud"].positions)
    assert np.array_equal(a["xs"], b["xs"])
    c = a["cloud"]
    assert c.positions.shape == (1000, 3) and c.moments.shape == (1000, 2)
    assert np.all(c.moments[:, 0] == 1.0)
    assert np.allclose(np.linalg.norm(c.positions, axis=1), 1, atol=1e-6)
    assert np.all(np.abs(a["xs"]) <= 1.5)
    # fp32-representable inputs (promoted exactly)
    assert np.array_equal(a["xs"].astype(np.float32).astype(np.float64), a["xs"])


def test_config2_composition():
    w = W.config2(scale=0.01)
    c = w["cloud"]
    assert c.size == 10000 and c.channels == 49
    assert list(w["kinds"][:2]) == [0, 1] and w["kinds"].sum() == 48
    assert np.all(np.abs(w["xs"]) <= 2)
    d = W.upstream(16, 49, w["d_out_seed"])
    assert d.shape == (16, 49) and d.dtype == np.float32


def test_config1_epsilon_recorded(oracle_mod):
    w = W.config1()
    eps = 1.5 * oracle_mod.mean_knn_spacing(w["cloud"].positions)
    assert eps == W.EPSILON["config1"]


def test_config3_rays_unit_and_aimed():
    w = W.config3(scale=0.01)
    rays = w["rays"]
    assert rays.shape[1] == 6
    assert np.allclose(np.linalg.norm(rays[:, 3:], axis=1), 1.0)
    assert np.allclose(np.linalg.norm(rays[:, :3], axis=1), 4.0)
    # rays start on the radius-4 sphere and point inwards
    assert np.all(np.einsum("ij,ij->i", rays[:, :3], rays[:, 3:]) < 0)
