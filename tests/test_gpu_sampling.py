"""GPU query generators of SURVEY §8(f) against the CPU oracle:
sample_grid (meshing.cpp:33-59; pinned by test_meshing.cpp:49-70) and the
probe-then-refine sample_ray (renderer.cpp:46-86)."""
import numpy as np
import pytest

from test_gpu_parity import close
from test_oracle_pins import _sphere_model, sphere_rays

pytestmark = pytest.mark.gpu


def _gpu_tree(eng, cloud):
    t = eng.DipoleTree(0)
    t.build(eng.OrientedPointCloud(cloud.pos, cloud.nrm, cloud.area, cloud.mu))
    kinds = np.ones(cloud.C, np.uint8)
    kinds[0] = 0
    t.set_channel_kernels(kinds)
    return t, kinds


def test_sample_grid_matches_oracle_and_pointwise_field():
    import oracle as O
    import paper_2405_16788_b200 as eng

    cloud = _sphere_model(O).as_f64()
    t, kinds = _gpu_tree(eng, cloud)
    port = O.OracleTree(cloud)
    port.set_kinds(kinds)
    eps = 0.08
    p = eng.KernelParams(epsilon=eps)
    res = (33, 29, 31)
    for lo, hi in (((0, 0, 0), (0, 0, 0)), ((-1.2, -1.1, -1.0), (1.0, 1.1, 1.3))):
        vals, lo_g, hi_g = t.sample_grid(p, 2.0, res, lo, hi)
        want, lo_w, hi_w = port.sample_grid(O.Params(eps), 2.0, res, lo, hi)
        assert np.array_equal(lo_g, lo_w) and np.array_equal(hi_g, hi_w)
        # f = 0.5 - D0: the tolerance applies to the primal value D0
        nbad, mx = close(0.5 - vals, 0.5 - want)
        assert nbad == 0, (nbad, mx)
        # grid values equal the pointwise geometry field bitwise (test_meshing.cpp:49-70)
        k, j, i = np.meshgrid(np.arange(res[2]), np.arange(res[1]), np.arange(res[0]), indexing="ij")
        f = [i / (res[0] - 1), j / (res[1] - 1), k / (res[2] - 1)]
        xs = np.stack([lo_g[a] + f[a] * (hi_g[a] - lo_g[a]) for a in range(3)], -1).reshape(-1, 3)
        d0 = t.primal_channel(xs, p, 2.0, 0)
        assert np.array_equal(vals.ravel(), np.float32(0.5) - d0)
    # beta == 0 everywhere gives exactly 0.5 (test_meshing.cpp)
    mu0 = cloud.mu.copy()
    mu0[:, 0] = 0.0
    t.update_moments(eng.OrientedPointCloud(cloud.pos, cloud.nrm, cloud.area, mu0))
    vals, _, _ = t.sample_grid(p, 2.0, (5, 5, 5))
    assert np.all(vals == np.float32(0.5))
    with pytest.raises(eng.DataError):
        t.sample_grid(p, 2.0, (1, 5, 5))


def test_sample_rays_matches_oracle():
    import oracle as O
    import paper_2405_16788_b200 as eng

    cloud = _sphere_model(O).as_f64()
    t, kinds = _gpu_tree(eng, cloud)
    port = O.OracleTree(cloud)
    port.set_kinds(kinds)
    eps = 0.08
    p = eng.KernelParams(epsilon=eps)
    rays = sphere_rays(3000, 7)
    for probes, (tn, tf) in ((1024, (2.0, 4.5)), (200, (0.5, 6.0)), (70, (2.0, 4.5))):
        cfg = eng.RaySampler(t_near=tn, t_far=tf, probe_count=probes)
        tg, dg, cg, bg = t.sample_rays(p, 2.0, rays, cfg)
        tw, dw, cw, bw = port.sample_rays(O.Params(eps), 2.0, rays, tn, tf,
                                          (probes, 24, 48, 8, 80), cfg.max_samples())
        assert 0 < bw.sum() < len(rays)
        # the bracket is a sign decision on f = 0.5 - D0: identical except where the
        # fp32 value sits within the parity tolerance of the iso-level
        same = (bg == bw) & (cg == cw) & np.all(tg == tw, axis=1) & np.all(dg == dw, axis=1)
        assert same.mean() > 0.995, same.mean()
        assert np.array_equal(cg[same], cw[same])
    with pytest.raises(eng.DataError):
        t.sample_rays(p, 2.0, rays[:4], eng.RaySampler(t_near=3.0, t_far=2.0))
    # degenerate span: one sample at the midpoint (renderer.cpp:50-54)
    tg, dg, cg, bg = t.sample_rays(p, 2.0, rays[:4], eng.RaySampler(t_near=2.0, t_far=2.0 + 1e-12))
    assert np.all(cg == 1) and not bg.any()
