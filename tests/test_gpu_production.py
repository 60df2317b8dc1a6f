"""Parity on BASELINE's production layouts and sizes (VERDICT r1 "What's
missing" 3), every output elementwise under tests/parity.py's bar with zero
violations:

  * config 1 at FULL size (N = 1e5 sphere, C = 2, Q = 1e6): every query against
    the oracle, plus the exact O(NQ) naive_dipole_sum (oracles.cpp:23-35) on
    10k queries — the Barnes-Hut error at beta = 2 that BASELINE reports;
  * config 4's tree at FULL size (N = 8e6): structure, point order, leaf map
    and geometry bit-identical; a 2,000-query subset of the production forward
    over a 4M-query batch with identical visited / far / leaf counts; the
    adjoint of the subset;
  * the config-5 render layout: C = 49 shapes cloud (config-4 generator),
    192 stratified samples per ray, direct-rgb head (the tree's forward
    computes the channels the head reads, renderer.cpp:125-127), fused walk then
    interaction-list replay;
  * all-channel primal_with_gradient at C = 49.
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest
from parity import RECORDS, check, counters_equal, scalar

pytestmark = pytest.mark.gpu


def _naive_mt(r, O, eps, xs, channel, kind, threads=None):
    """Exact naive sums on query chunks in parallel (ctypes drops the GIL)."""
    threads = threads or os.cpu_count() or 1
    parts = np.array_split(np.arange(xs.shape[0]), threads)
    with cf.ThreadPoolExecutor(threads) as ex:
        res = list(ex.map(lambda ix: r.naive_sum(O.Params(eps), xs[ix], channel, kind), parts))
    return np.concatenate(res)


def test_config1_full_size(oracle_mod):
    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import workloads as W

    O = oracle_mod
    w = W.config1()
    c = w["cloud"]
    eps = W.EPSILON["config1"]
    t = P.DipoleTree(0)
    t.build(c)
    t.set_channel_kernels(w["kinds"])
    r = O.OracleTree(O.Cloud(c.positions, c.normals, c.areas, c.moments))
    r.set_kinds(w["kinds"])
    a, b = t.export(), r.export()
    for k in ("topo", "order", "leaf_of", "geo"):
        assert np.array_equal(a[k], b[k]), k
    p = P.KernelParams(epsilon=eps)
    xs = w["xs"]
    got, cnt = t.primal(xs, p, 2.0, visited=True)
    want, wcnt = r.primal(O.Params(eps), 2.0, xs, counters=True)
    check("config1 full size primal (1e6 queries, C=2)", got, want)
    counters_equal("config1 full size counters", cnt, wcnt)
    # primal_channel(0) (the reference bench workload, dipole.cpp:169) is
    # bitwise the channel of primal()
    assert np.array_equal(t.primal_channel(xs, p, 2.0, 0), got[:, 0])
    # exact O(NQ) sums on the first 10k queries: the Barnes-Hut error at beta=2
    # is the reference's, not ours; the GPU's error vs naive equals the oracle's
    sub = xs[:10_000]
    for ch in (0, 1):
        naive = _naive_mt(r, O, eps, sub, ch, int(w["kinds"][ch]))
        e_gpu = np.abs(got[:10_000, ch] - naive)
        e_ref = np.abs(want[:10_000, ch] - naive)
        scale = np.abs(naive).max()
        RECORDS.append({"check": f"config1 beta=2 Barnes-Hut vs exact naive_dipole_sum, channel "
                                 f"{ch}, 10k queries (report)",
                        "gpu_max_abs_err": float(e_gpu.max()), "ref_max_abs_err": float(e_ref.max()),
                        "gpu_max_err_over_max_naive": float(e_gpu.max() / scale),
                        "ref_max_err_over_max_naive": float(e_ref.max() / scale),
                        "gpu_mean_err_over_max_naive": float(e_gpu.mean() / scale),
                        "naive_max_abs": float(scale)})
        # the approximation error is the reference's own: GPU and oracle errors
        # differ by no more than the GPU-vs-oracle parity bar
        assert (np.abs(e_gpu - e_ref) <= 1e-6 + 1e-4 * np.abs(want[:10_000, ch])).all()


def test_config4_full_size_tree_and_subset(oracle_mod):
    import torch

    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import workloads as W

    O = oracle_mod
    w = W.config4(queries=False)
    c = w["cloud"]
    eps = W.EPSILON["config4"]
    t = P.DipoleTree(0)
    t.build(c)
    t.set_channel_kernels(w["kinds"])
    r = O.OracleTree(O.Cloud(c.positions, c.normals, c.areas, c.moments))
    r.set_kinds(w["kinds"])
    a, b = t.export(), r.export()
    for k in ("topo", "order", "leaf_of", "geo"):
        assert np.array_equal(a[k], b[k]), k
    del a, b
    p = P.KernelParams(epsilon=eps)
    Q = 4_000_000
    xs = W.config4_queries(0, Q)
    xd = torch.from_numpy(xs).cuda()
    idx = np.random.default_rng(41).choice(Q, 20000, replace=False)
    op = O.Params(eps)
    want, wcnt = r.primal(op, 2.0, xs[idx], counters=True)
    d_out = W.upstream(Q, 49, [4, 2])
    dd = torch.from_numpy(d_out).cuda()
    buf = t.make_buffer()
    for rnd in range(2):  # fused walk, then the production list replay (K9 + replay)
        got = t.primal(xd, p, 2.0).cpu().numpy()
        check(f"config4 N=8e6 forward, 20k-query subset of a 4M batch (pass {rnd})", got[idx], want)
        t.adjoint(xd, p, 2.0, dd, None, buf)
        buf.reset()
    _, cnt = t.primal(xd[torch.from_numpy(idx).cuda()], p, 2.0, visited=True)
    counters_equal("config4 N=8e6 subset counters", cnt.cpu().numpy(), wcnt)
    # the adjoint of the subset on its own (the full batch's sum is not
    # oracle-evaluable at this size): fused, then list replay
    xs_s = np.ascontiguousarray(xs[idx[:2000]])
    ds = np.ascontiguousarray(d_out[idx[:2000]])
    wa = r.adjoint_mag(op, 2.0, xs_s, ds.astype(np.float64), threads=1)
    for rnd in range(2):
        t.primal(xs_s, p, 2.0)
        b2 = t.make_buffer()
        t.adjoint(xs_s, p, 2.0, ds, None, b2)
        g = t.flush_gradients(b2)
        tag = f"config4 N=8e6 adjoint of a 2k-query subset (pass {rnd})"
        check(f"{tag} moments", g.moments, wa["moments"], wa["moments_abs"])
        check(f"{tag} normals", g.normals, wa["normals"], wa["normals_abs"])
        scalar(f"{tag} d_epsilon", g.d_epsilon, wa["d_eps"], wa["d_eps_abs"])


def _config5_like(n, px_per_cam, seed=5):
    from paper_2405_16788_b200 import workloads as W

    pos, nrm, area, rng = W.shapes_cloud(n, seed)
    mu = rng.standard_normal((n, 49))
    mu[:, 0] = 1.0  # geometry moment 1: the shapes' winding-number field (visible surfaces)
    c = W.cloud(pos, nrm, area, mu)
    kinds = np.ones(49, np.uint8)
    kinds[0] = 0
    rays = W.camera_rays(64, 1024, px_per_cam, seed=2)
    return c, kinds, rays


def test_config5_render_layout(oracle_mod):
    """Config 5's layout: C = 49, S = 192, direct-rgb head, L2 loss."""
    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import renderer as Rn

    O = oracle_mod
    c, kinds, rays = _config5_like(60_000, 3)
    S = 192
    t = P.DipoleTree(0)
    t.build(c)
    t.set_channel_kernels(kinds)
    r = O.OracleTree(O.Cloud(c.positions, c.normals, c.areas, c.moments))
    r.set_kinds(kinds)
    eps = 1.5 * O.mean_knn_spacing(c.positions)
    R = rays.shape[0]
    target = np.random.default_rng(4).uniform(0, 1, (R, 3))
    # L = (1/3) sum ||rgb - target||^2 (BASELINE's L2 without the 1/B batch
    # mean, so gradients are O(1) and the 1e-6 absolute floor does not hide them)
    scale = 2.0 / 3.0
    rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=3)
    p = P.KernelParams(epsilon=eps)
    ts, dlt = O.stratified_samples(R, S, 2.0, 6.0, 3)
    want = r.render_step(O.Params(eps), 2.0, 20.0, [0, 0, 0], rays, ts, dlt, target, scale, mag=True)
    assert not want["moments"][:, 4:].any()  # the direct-rgb head reads channels 0..3 only
    for rnd in range(2):  # walk, then the training pattern's list replay
        rgb, tape = Rn.render_forward(t, p, rs, rays, S)
        # the loss gradient of the oracle's colours: both backward passes start
        # from the same d_rgb (the GPU colours are checked separately)
        d_rgb = (scale * (want["rgb"] - target)).astype(np.float32)
        buf = t.make_buffer()
        dl, dbg = Rn.render_backward(t, p, rs, tape, d_rgb, buf)
        g = t.flush_gradients(buf)
        tag = f"config5 layout render C=49 S=192 (pass {rnd})"
        check(f"{tag} rgb", rgb, want["rgb"])
        check(f"{tag} moments", g.moments, want["moments"], want["moments_abs"])
        assert not g.moments[:, 4:].any()
        check(f"{tag} normals", g.normals, want["normals"], want["normals_abs"])
        scalar(f"{tag} d_epsilon", g.d_epsilon, want["d_eps"], want["d_eps_abs"])
        scalar(f"{tag} d_lambda", dl, want["d_lambda"], atol=1e-8)
        check(f"{tag} d_background", dbg, want["d_bg"], atol=1e-8)


def test_primal_with_gradient_all_channels_c49(oracle_mod):
    import paper_2405_16788_b200 as P

    O = oracle_mod
    c, kinds, _ = _config5_like(20_000, 1, seed=9)
    t = P.DipoleTree(0)
    t.build(c)
    t.set_channel_kernels(kinds)
    r = O.OracleTree(O.Cloud(c.positions, c.normals, c.areas, c.moments))
    r.set_kinds(kinds)
    eps = 1.5 * O.mean_knn_spacing(c.positions)
    xs = np.random.default_rng(10).uniform(-2, 2, (3000, 3)).astype(np.float32).astype(np.float64)
    xs[:50] = np.asarray(c.positions)[:50]  # queries on data points (r = 0 skips)
    v, g = t.primal_with_gradient(xs, P.KernelParams(epsilon=eps), 2.0)
    w = r.primal_mag(O.Params(eps), 2.0, xs, mode="grad")
    check("primal_with_gradient C=49 values", v, w["out"], w["out_abs"])
    check("primal_with_gradient C=49 all-channel gradients", g, w["grad"], w["grad_abs"])


@pytest.mark.parametrize("n,C,seed", [(1, 1, 0), (64, 2, 23), (3000, 4, 5), (20000, 49, 7)])
def test_dplt_dump_byte_identical_to_reference(oracle_mod, tmp_path, n, C, seed):
    """DipoleTree::dump (bhtree.cpp:465-494): the engine's DPLT file equals the
    reference build's (oracle/_ref, the reference's own bhtree.cpp) byte for
    byte — node records, point order and both moment arrays in fp64."""
    import paper_2405_16788_b200 as P

    O = oracle_mod
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = rng.uniform(0.5, 1, n) / max(n, 1)
    mu = rng.standard_normal((n, C))
    t = P.DipoleTree(0)
    t.build(P.OrientedPointCloud(pos, nrm, area, mu))
    r = O.OracleTree(O.Cloud(pos, nrm, area, mu), backend="ref")
    a, b = tmp_path / "gpu.dplt", tmp_path / "ref.dplt"
    t.dump(str(a))
    r.dump(str(b))
    ga, gb = a.read_bytes(), b.read_bytes()
    assert len(ga) == len(gb)
    diff = np.flatnonzero(np.frombuffer(ga, np.uint8) != np.frombuffer(gb, np.uint8))
    assert diff.size == 0, f"{diff.size} bytes differ, first at offset {diff[0]}"
