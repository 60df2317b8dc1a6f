"""GPU parity for the rows around the query engine: SceneModel's eps default
(mean k-NN spacing, pointcloud.cpp:51-65) and the trainer's point update
(Adam + renormalisation + update_moments, optimizer.cpp:65-81,161-205)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def cloud(n, seed, C):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = rng.uniform(0.5, 1, n) / n
    mu = rng.standard_normal((n, C))
    return pos, nrm, area, mu


@pytest.mark.parametrize("n,k", [(2, 8), (9, 8), (5000, 8), (20000, 4)])
def test_mean_knn_spacing_matches_reference(oracle_mod, n, k):
    from paper_2405_16788_b200.bhtree import mean_knn_spacing

    pos, _, _, _ = cloud(n, 3 + n, 1)
    pos[1] = pos[0]  # a duplicate point
    got = mean_knn_spacing(pos, k)
    want = oracle_mod.mean_knn_spacing(pos, k)
    assert abs(got - want) <= 1e-12 * abs(want)


def test_knn_on_surface_cloud(oracle_mod):
    from paper_2405_16788_b200 import workloads as W
    from paper_2405_16788_b200.bhtree import mean_knn_spacing

    w = W.config1(scale=0.1)
    p = w["cloud"].positions
    assert abs(mean_knn_spacing(p) - oracle_mod.mean_knn_spacing(p)) <= 1e-12


def test_point_adam_step_matches_oracle(oracle_mod):
    """One trainer update with identical gradients: Adam (fp64, reference op
    order) + normal renormalisation must reproduce the oracle's parameters to
    the bit; the refreshed tree then answers queries like the oracle's
    update_moments."""
    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200.bhtree import PointAdam, get_points

    O = oracle_mod
    n, C = 3000, 4
    pos, nrm, area, mu = cloud(n, 41, C)
    kinds = np.array([0, 1, 1, 1], np.uint8)
    t = P.DipoleTree(0)
    t.build(P.OrientedPointCloud(pos, nrm, area, mu))
    t.set_channel_kernels(kinds)
    rng = np.random.default_rng(42)
    xs = rng.uniform(-1.2, 1.2, (800, 3))
    p = P.KernelParams(epsilon=0.05)
    opt = PointAdam(t, lr=1e-2)
    m_mu, v_mu = np.zeros((n, C)), np.zeros((n, C))
    m_n, v_n = np.zeros((n, 3)), np.zeros((n, 3))
    cur_mu, cur_n = mu.copy(), nrm.copy()
    for step in range(1, 3):
        d_out = rng.standard_normal((800, C)).astype(np.float32)
        buf = t.make_buffer()
        t.adjoint(xs, p, 2.0, d_out, None, buf)
        g = t.flush_gradients(buf)
        opt.step(g)
        # oracle: the same update on the same (fp32) gradients
        gm = np.ascontiguousarray(g.moments, np.float64)
        gn = np.ascontiguousarray(g.normals, np.float64)
        lib = O.port_lib()
        pm = cur_mu.ravel().copy()
        lib.ora_adam_step(pm.ctypes.data_as(O._dp), gm.ravel().ctypes.data_as(O._dp),
                          m_mu.ctypes.data_as(O._dp), v_mu.ctypes.data_as(O._dp), n * C, 1e-2, 0.9,
                          0.999, 1e-8, step)
        pn = cur_n.ravel().copy()
        lib.ora_adam_step(pn.ctypes.data_as(O._dp), gn.ravel().ctypes.data_as(O._dp),
                          m_n.ctypes.data_as(O._dp), v_n.ctypes.data_as(O._dp), n * 3, 1e-2, 0.9,
                          0.999, 1e-8, step)
        cur_mu = pm.reshape(n, C)
        newn = pn.reshape(n, 3)
        changed = np.any(newn != cur_n, axis=1)
        lens = np.sqrt((newn[:, 0] ** 2 + newn[:, 1] ** 2) + newn[:, 2] ** 2)
        ok = changed & (lens > 1e-12)
        newn[ok] = newn[ok] / lens[ok, None]
        newn[~ok] = cur_n[~ok]
        cur_n = newn
        gn_, gmu_ = get_points(t)
        assert np.array_equal(gmu_, cur_mu)
        assert np.abs(gn_ - cur_n).max() <= 1e-15
    r = O.OracleTree(O.Cloud(pos, nrm, area, mu))
    r.set_kinds(kinds)
    r.update_moments(O.Cloud(pos, cur_n, area, cur_mu))
    got = t.primal(xs, p, 2.0)
    want = r.primal(O.Params(0.05), 2.0, xs)
    assert np.all(np.abs(got - want) <= 1e-6 + 1e-4 * np.abs(want))


def test_checkpoint_save_matches_reference_bytes(tmp_path):
    """save_checkpoint (optimizer.cpp:330-356) from the GPU tree writes the
    reference's bytes; a load -> build round trip reproduces the tree."""
    import oracle as O
    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200.bhtree import load_checkpoint

    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    from test_oracle_pins import _sphere_model

    cloud = _sphere_model(O, n=500, C=4, seed=11).as_f64()
    ref = O.RefModel(cloud, 0.06, lam=20.0, beta=2.0, background=(0.0, 0.5, 1.0))
    ref.save_checkpoint(tmp_path / "ref.dpck", iter=7)
    t = P.DipoleTree(0)
    t.build(P.OrientedPointCloud(cloud.pos, cloud.nrm, cloud.area, cloud.mu))
    t.save_checkpoint(tmp_path / "gpu.dpck", iter=7, lambda_scale=20.0, epsilon=0.06,
                      background=(0.0, 0.5, 1.0), beta_bh=2.0)
    assert (tmp_path / "gpu.dpck").read_bytes() == (tmp_path / "ref.dpck").read_bytes()
    ck = load_checkpoint(tmp_path / "gpu.dpck")
    t2 = P.DipoleTree(0)
    t2.build(ck["cloud"])
    a, b = t.export(), t2.export()
    for k in ("topo", "order", "geo"):
        assert np.array_equal(a[k], b[k])


def test_sharded_point_update_equals_full_step(oracle_mod):
    """SURVEY 8(e) config-5 step on one GPU, the two ranks run one after the
    other (no collective): rank r steps Adam on its point slice only
    (dpl_point_adam_step_range), the slices are exchanged with
    dpl_tree_get/set_points_range and both trees refresh their moments — the
    parameters and query results equal a full PointAdam.step bit for bit."""
    import torch

    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200.bhtree import (PointAdam, get_points, get_points_range,
                                              refresh_moments, set_points_range)
    from paper_2405_16788_b200.parallel import TreeEngine, point_chunk, sharded_point_update

    n, C = 2501, 4
    pos, nrm, area, mu = cloud(n, 43, C)
    kinds = np.array([0, 1, 1, 1], np.uint8)

    def tree():
        t = P.DipoleTree(0)
        t.build(P.OrientedPointCloud(pos, nrm, area, mu))
        t.set_channel_kernels(kinds)
        return t

    full, ranks, single = tree(), [tree(), tree()], tree()
    opt_full = PointAdam(full, lr=1e-2)
    opts = [PointAdam(t, lr=1e-2) for t in ranks]
    eng = TreeEngine(single, PointAdam(single, lr=1e-2))  # sharded_point_update, one rank
    rng = np.random.default_rng(44)
    xs = rng.uniform(-1.2, 1.2, (600, 3))
    p = P.KernelParams(epsilon=0.05)
    for _ in range(2):
        gm = rng.standard_normal((n, C)).astype(np.float32)
        gn = rng.standard_normal((n, 3)).astype(np.float32)
        opt_full.step(P.PointGradients(C, gm, gn, 0.0))
        sharded_point_update(eng, torch.from_numpy(gm).cuda(), torch.from_numpy(gn).cuda(), n, C)
        slices = []
        for r, (t, o) in enumerate(zip(ranks, opts)):
            lo, hi, _ = point_chunk(n, r, 2)
            o.step_range(torch.from_numpy(gm[lo:hi]).cuda(), torch.from_numpy(gn[lo:hi]).cuda(), lo, hi)
            slices.append((lo, hi) + get_points_range(t, lo, hi))
        for t in ranks:
            for lo, hi, sn, sm in slices:
                set_points_range(t, lo, hi, sn, sm)
            refresh_moments(t)
    wn, wm = get_points(full)
    want = full.primal(xs, p, 2.0)
    for t in ranks + [single]:
        gn_, gm_ = get_points(t)
        assert np.array_equal(gm_, wm) and np.array_equal(gn_, wn)
        assert np.array_equal(t.primal(xs, p, 2.0), want)
