"""GPU parity against the CPU oracle (oracle/dipole_oracle.c, itself pinned
bit-for-bit to the reference in tests/test_oracle_pins.py).

Bar (BASELINE.json north_star): tree structure bit-exact; values and gradients
within 1e-4 relative / 1e-6 absolute in fp32 at the same Barnes-Hut beta.
These mirror the reference's own hot-path tests (proj/tests/test_bhtree.cpp),
re-targeted at the batched GPU API with fp32 tolerances.
"""
import numpy as np
import pytest
from parity import check, counters_equal, scalar

pytestmark = pytest.mark.gpu

RTOL, ATOL = 1e-4, 1e-6


def close(got, want, rtol=RTOL, atol=ATOL):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    bad = np.abs(got - want) > atol + rtol * np.abs(want)
    return int(bad.sum()), float(np.abs(got - want).max(initial=0.0))


def rel_scale_err(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    s = max(np.abs(want).max(initial=0.0), 1e-300)
    return float(np.abs(got - want).max(initial=0.0) / s)


def random_cloud(n, seed, C, f32=True):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1, 1, (n, 3))
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = 0.5 + 0.5 * np.abs(rng.uniform(-1, 1, n))
    mu = rng.uniform(-1, 1, (n, C))
    if f32:
        pos = pos.astype(np.float32).astype(np.float64)
    return pos, nrm, area / n, mu


@pytest.fixture(scope="module")
def eng():
    import paper_2405_16788_b200 as P

    return P


def make(eng, O, pos, nrm, area, mu, kinds=None, max_leaf=8, max_depth=20):
    t = eng.DipoleTree(0)
    t.build(eng.OrientedPointCloud(pos, nrm, area, mu), max_leaf, max_depth)
    r = O.OracleTree(O.Cloud(pos, nrm, area, mu), max_leaf, max_depth)
    if kinds is not None:
        t.set_channel_kernels(kinds)
        r.set_kinds(kinds)
    return t, r


# ---------------------------------------------------------------- structure
@pytest.mark.parametrize("n,seed,max_leaf,max_depth", [
    (1, 0, 8, 20), (2, 1, 8, 20), (9, 2, 8, 20), (1000, 3, 8, 20), (20000, 4, 8, 20),
    (5000, 5, 1, 20), (5000, 6, 32, 20), (5000, 7, 8, 4), (3000, 8, 8, 0), (3000, 9, 8, 21)])
def test_tree_structure_bit_exact(eng, oracle_mod, n, seed, max_leaf, max_depth):
    pos, nrm, area, mu = random_cloud(n, seed, 2)
    t, r = make(eng, oracle_mod, pos, nrm, area, mu, max_leaf=max_leaf, max_depth=max_depth)
    a, b = t.export(), r.export()
    for k in ("topo", "order", "leaf_of", "geo"):
        assert np.array_equal(a[k], b[k]), k


def test_tree_coincident_and_clustered(eng, oracle_mod):
    # all points coincident must terminate with a leaf (test_bhtree.cpp:48-60)
    pos = np.full((100, 3), 0.5)
    nrm = np.tile([0.0, 0.0, 1.0], (100, 1))
    t, r = make(eng, oracle_mod, pos, nrm, np.ones(100), np.ones((100, 1)))
    a, b = t.export(), r.export()
    assert np.array_equal(a["topo"], b["topo"]) and np.array_equal(a["order"], b["order"])
    leaves = a["topo"][a["topo"][:, 5] == 1]
    assert int((leaves[:, 1] - leaves[:, 0]).sum()) == 100
    # tight clusters + duplicates stress deep levels
    rng = np.random.default_rng(11)
    base = rng.uniform(-1, 1, (50, 3))
    pos = np.repeat(base, 40, axis=0) + rng.normal(0, 1e-6, (2000, 3))
    pos[::7] = pos[0]
    pos = pos.astype(np.float32).astype(np.float64)
    nrm = np.tile([1.0, 0.0, 0.0], (2000, 1))
    t, r = make(eng, oracle_mod, pos, nrm, np.full(2000, 1e-3), rng.standard_normal((2000, 2)))
    a, b = t.export(), r.export()
    for k in ("topo", "order", "leaf_of", "geo"):
        assert np.array_equal(a[k], b[k]), k


# ---------------------------------------------------------------- forward
@pytest.mark.parametrize("beta", [2.0, 4.0, np.inf])
def test_primal_parity_mixed_kernels(eng, oracle_mod, beta):
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(4000, 3, 3)
    kinds = np.array([0, 1, 1], np.uint8)
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    rng = np.random.default_rng(4)
    xs = rng.uniform(-1.5, 1.5, (3000, 3)).astype(np.float32).astype(np.float64)
    xs[:5] = pos[:5]  # coincident queries
    p = eng.KernelParams(epsilon=0.05)
    got, cnt = t.primal(xs, p, beta, visited=True)
    want, wcnt = r.primal(O.Params(0.05), beta, xs, counters=True)
    check(f"primal mixed kinds beta={beta}", got, want)
    # identical opening decisions: visited / far / point counts match exactly
    counters_equal(f"primal mixed kinds beta={beta} counters", cnt, wcnt)
    # primal_channel(c) == primal()[c] (test_bhtree.cpp:140)
    for c in range(3):
        pc = t.primal_channel(xs, p, beta, c)
        assert np.array_equal(pc, got[:, c])


def test_primal_with_gradient_parity(eng, oracle_mod):
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(3000, 7, 2)
    kinds = np.array([0, 1], np.uint8)
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    xs = np.random.default_rng(8).uniform(-1.5, 1.5, (2000, 3))
    p = eng.KernelParams(epsilon=0.2)
    v, g = t.primal_with_gradient(xs, p, 2.0)
    w = r.primal_mag(O.Params(0.2), 2.0, xs, mode="grad")
    check("primal_with_gradient values C=2", v, w["out"], w["out_abs"])
    check("primal_with_gradient gradients C=2", g, w["grad"], w["grad_abs"])
    # values of primal_with_gradient equal primal (test_bhtree.cpp:215-216), fp32 tolerance
    assert close(v, t.primal(xs, p, 2.0))[0] == 0
    v0, g0 = t.primal_grad0(xs, p, 2.0)
    check("primal_grad0 values", v0, w["out"], w["out_abs"])
    check("primal_grad0 gradient of channel 0", g0, w["grad"][:, 0], w["grad_abs"][:, 0])


def test_beta_infinity_equals_naive(eng, oracle_mod):
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(500, 3, 3)
    kinds = np.array([0, 1, 1], np.uint8)
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    xs = np.random.default_rng(4).uniform(-1.5, 1.5, (200, 3))
    got = t.primal(xs, eng.KernelParams(epsilon=0.15), np.inf)
    for c in range(3):
        want = r.naive_sum(O.Params(0.15), xs, c, int(kinds[c]))
        check(f"beta=inf vs naive_dipole_sum channel {c}", got[:, c], want)


@pytest.mark.parametrize("eps,desing,delta", [(0.0, False, 0.0), (0.0, True, 0.05), (0.3, False, 0.0)])
def test_kernel_variants(eng, oracle_mod, eps, desing, delta):
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(2000, 21, 2)
    kinds = np.array([0, 1], np.uint8)
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    xs = np.random.default_rng(22).uniform(-1.2, 1.2, (1000, 3))
    p = eng.KernelParams(epsilon=eps, desingularized=desing, desing_delta=delta)
    v, g = t.primal_with_gradient(xs, p, 2.0)
    w = r.primal_mag(O.Params(eps, desing, delta), 2.0, xs, mode="grad")
    check(f"kernel variant eps={eps} desing={desing} values", v, w["out"], w["out_abs"])
    check(f"kernel variant eps={eps} desing={desing} gradients", g, w["grad"], w["grad_abs"])


def test_config1_slice(eng, oracle_mod):
    from paper_2405_16788_b200 import workloads as W

    O = oracle_mod
    w = W.config1(scale=0.05)
    c = w["cloud"]
    t, r = make(eng, O, c.positions, c.normals, c.areas, c.moments, w["kinds"])
    eps = 1.5 * O.mean_knn_spacing(c.positions)
    xs = w["xs"]
    got = t.primal(xs, eng.KernelParams(epsilon=eps), 2.0)
    want = r.primal(O.Params(eps), 2.0, xs)
    check("config-1 slice primal", got, want)


# ---------------------------------------------------------------- adjoint
@pytest.mark.parametrize("with_grad", [False, True])
def test_adjoint_flush_parity(eng, oracle_mod, with_grad):
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(3000, 12, 3)
    kinds = np.array([0, 1, 1], np.uint8)
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    rng = np.random.default_rng(13)
    q = 2000
    xs = rng.uniform(-1.5, 1.5, (q, 3))
    d_out = rng.standard_normal((q, 3)).astype(np.float32)
    d_grad = rng.standard_normal((q, 3, 3)).astype(np.float32) if with_grad else None
    p = eng.KernelParams(epsilon=0.1)
    buf = t.make_buffer()
    t.adjoint(xs, p, 2.0, d_out, d_grad, buf)
    g = t.flush_gradients(buf)
    w = r.adjoint_mag(O.Params(0.1), 2.0, xs, d_out.astype(np.float64),
                      None if d_grad is None else d_grad.astype(np.float64))
    tag = f"adjoint+flush d_grad={with_grad}"
    check(f"{tag} moments", g.moments, w["moments"], w["moments_abs"])
    check(f"{tag} normals", g.normals, w["normals"], w["normals_abs"])
    scalar(f"{tag} d_epsilon", g.d_epsilon, w["d_eps"], w["d_eps_abs"])
    # flush zeroes the buffer: a second flush is all zeros (test_bhtree.cpp:297-299)
    g2 = t.flush_gradients(buf)
    assert not np.any(g2.moments) and g2.d_epsilon == 0.0


def test_multi_buffer_flush_order_independent(eng, oracle_mod):
    pos, nrm, area, mu = random_cloud(300, 18, 1)
    t, _ = make(eng, oracle_mod, pos, nrm, area, mu)
    rng = np.random.default_rng(19)
    xs = rng.uniform(-1, 1, (12, 3))
    ds = rng.uniform(-1, 1, (12, 1)).astype(np.float32)
    p = eng.KernelParams(epsilon=0.1)
    single = t.make_buffer()
    t.adjoint(xs, p, 2.0, ds, None, single)
    ref = t.flush_gradients(single)
    bufs = [t.make_buffer() for _ in range(3)]
    for w in range(3):
        t.adjoint(xs[w::3], p, 2.0, ds[w::3], None, bufs[w])
    got = t.flush_gradients(bufs)
    # the reference asserts 1e-10 in fp64 (test_bhtree.cpp:441); here each
    # buffer's queries form other warps (other fp32 summation groupings), so
    # both are held to the oracle's result under the parity bar, and to each other
    w = oracle_mod.OracleTree(oracle_mod.Cloud(pos, nrm, area, mu))
    wa = w.adjoint_mag(oracle_mod.Params(0.1), 2.0, xs, ds.astype(np.float64))
    check("multi-buffer flush (3 buffers) moments", got.moments, wa["moments"], wa["moments_abs"])
    check("single-buffer flush moments", ref.moments, wa["moments"], wa["moments_abs"])
    check("multi-buffer vs single-buffer flush moments", got.moments, ref.moments,
          wa["moments_abs"])


def test_zero_adjoint_leaves_accumulators_untouched(eng, oracle_mod):
    pos, nrm, area, mu = random_cloud(100, 11, 2)
    t, _ = make(eng, oracle_mod, pos, nrm, area, mu)
    buf = t.make_buffer()
    t.adjoint(np.array([[0.1, 0.2, 0.3]]), eng.KernelParams(epsilon=0.2), 2.0,
              np.zeros((1, 2), np.float32), None, buf)
    g = t.flush_gradients(buf)
    assert not np.any(g.moments) and not np.any(g.normals) and g.d_epsilon == 0.0


def test_single_point_adjoint_closed_form(eng, oracle_mod):
    # test_bhtree.cpp:259-281: radius-0 leaf seen as far field
    import math

    t = eng.DipoleTree(0)
    t.build(eng.OrientedPointCloud(np.zeros((1, 3)), np.array([[0, 0, 1.0]]), np.array([0.8]),
                                   np.array([[0.6]])))
    buf = t.make_buffer()
    t.adjoint(np.array([[0, 0, -1.0]]), eng.KernelParams(epsilon=0.3), 2.0,
              np.array([[2.5]], np.float32), None, buf)
    g = t.flush_gradients(buf)
    tau = oracle_mod.port_lib().ora_tau(1 / 0.3)
    want = 0.8 * (1 / (4 * math.pi)) * tau * 2.5 * 0.8 / 0.8  # d beta = a P_eps ds
    assert abs(g.moments[0, 0] - want) <= 1e-5 * abs(want)


# ---------------------------------------------------------------- render step
def test_render_step_parity(eng, oracle_mod):
    from paper_2405_16788_b200 import renderer as Rn
    from paper_2405_16788_b200 import workloads as W

    O = oracle_mod
    w = W.config3(scale=0.02)
    c = w["cloud"]
    t, r = make(eng, O, c.positions, c.normals, c.areas, c.moments, w["kinds"])
    eps = 1.5 * O.mean_knn_spacing(c.positions)
    rays = w["rays"][:256]
    S = 32
    target = w["target"][:256]
    rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=3)
    p = eng.KernelParams(epsilon=eps)
    rgb, tape = Rn.render_forward(t, p, rs, rays, S)
    scale = 2.0 / (3.0 * rays.shape[0])
    ts, dlt = O.stratified_samples(rays.shape[0], S, 2.0, 6.0, 3)
    want = r.render_step(O.Params(eps), 2.0, 20.0, [0, 0, 0], rays, ts, dlt, target, scale,
                         mag=True)
    # the loss gradient of the oracle's colours: both backward passes start
    # from the same d_rgb (the GPU colours are checked separately)
    d_rgb = (scale * (want["rgb"] - target)).astype(np.float32)
    buf = t.make_buffer()
    dl, dbg = Rn.render_backward(t, p, rs, tape, d_rgb, buf)
    g = t.flush_gradients(buf)
    check("render C=4 S=32 rgb", rgb, want["rgb"])
    check("render C=4 S=32 moments", g.moments, want["moments"], want["moments_abs"])
    check("render C=4 S=32 normals", g.normals, want["normals"], want["normals_abs"])
    scalar("render C=4 S=32 d_epsilon", g.d_epsilon, want["d_eps"], want["d_eps_abs"])
    scalar("render C=4 S=32 d_lambda", dl, want["d_lambda"], atol=1e-8)
    check("render C=4 S=32 d_background", dbg, want["d_bg"], atol=1e-8)


def test_render_steps_switch_to_lists(eng, oracle_mod):
    """A render_backward after render_forward makes the next render step build
    and replay interaction lists (the training pattern): the colours of the
    listed step match the walked one (same entries in the same order; a lane
    within an ulp of 6.5 eps may take the tau = 1 form), its gradients agree."""
    from paper_2405_16788_b200 import renderer as Rn
    from paper_2405_16788_b200 import workloads as W

    O = oracle_mod
    w = W.config3(scale=0.02)
    c = w["cloud"]
    t, _ = make(eng, O, c.positions, c.normals, c.areas, c.moments, w["kinds"])
    eps = 1.5 * O.mean_knn_spacing(c.positions)
    rays = w["rays"][:512]
    rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=5)
    p = eng.KernelParams(epsilon=eps)
    d_rgb = np.full((rays.shape[0], 3), 1e-3, np.float32)
    res = []
    for _ in range(3):  # walk, lists, lists
        rgb, tape = Rn.render_forward(t, p, rs, rays, 48)
        buf = t.make_buffer()
        dl, _ = Rn.render_backward(t, p, rs, tape, d_rgb, buf)
        g = t.flush_gradients(buf)
        res.append((rgb, g.moments, g.normals, g.d_epsilon, dl))
    for rgb, mom, nrm, de, dl in res[1:]:
        assert np.abs(rgb - res[0][0]).max() <= 1e-6 * np.abs(res[0][0]).max()
        assert rel_scale_err(mom, res[0][1]) < 1e-6
        assert rel_scale_err(nrm, res[0][2]) < 1e-6
        assert abs(de - res[0][3]) <= 1e-6 * abs(res[0][3]) + 1e-12
        assert abs(dl - res[0][4]) <= 1e-6 * abs(res[0][4]) + 1e-12


@pytest.mark.parametrize("C", [2, 4, 5, 17, 33, 49, 65, 70])
def test_many_channel_forward_adjoint(eng, oracle_mod, C):
    """Config-2 channel layouts (1 Dipole + C-1 Radial, N(0,1) moments and
    upstream gradients): covers the two-phase kernels' column splits (<=32,
    <=48, <=64 radial) and the multi-tile fallback beyond."""
    O = oracle_mod
    rng = np.random.default_rng(C)
    pos, nrm, area, _ = random_cloud(3000, 30 + C, 1)
    mu = rng.standard_normal((3000, C))
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    q = 1500
    xs = rng.uniform(-1.5, 1.5, (q, 3)).astype(np.float32).astype(np.float64)
    p = eng.KernelParams(epsilon=0.06)
    got = t.primal(xs, p, 2.0)
    want, wcnt = r.primal(O.Params(0.06), 2.0, xs, counters=True)
    check(f"primal C={C}", got, want)
    # the production (two-phase / tensor-core) path replays the reference's
    # opening decisions exactly: identical visited / far / leaf-point counts
    _, cnt = t.primal(xs, p, 2.0, visited=True)
    counters_equal(f"primal C={C} counters", cnt, wcnt)
    d_out = rng.standard_normal((q, C)).astype(np.float32)
    w = r.adjoint_mag(O.Params(0.06), 2.0, xs, d_out.astype(np.float64))
    for rnd in range(2):  # fused walk, then (primal -> adjoint pair) list replay
        t.primal(xs, p, 2.0)
        buf = t.make_buffer()
        t.adjoint(xs, p, 2.0, d_out, None, buf)
        g = t.flush_gradients(buf)
        check(f"adjoint C={C} moments (pass {rnd})", g.moments, w["moments"], w["moments_abs"])
        check(f"adjoint C={C} normals (pass {rnd})", g.normals, w["normals"], w["normals_abs"])
        scalar(f"adjoint C={C} d_epsilon (pass {rnd})", g.d_epsilon, w["d_eps"], w["d_eps_abs"])


@pytest.mark.parametrize("eps", [1e-8, 0.06])
def test_regularized_specialisation_bounds(eng, oracle_mod, eps):
    """The regularized kernels zero a far entry's non-member lanes through their
    area with 1/r clamped at (6.5 eps)^2; they are chosen only when
    (6.5 eps)^2 >= 1e-12. eps = 1e-8 takes the generic kernels, eps = 0.06 the
    specialised ones; both batches hold queries ON data points (r = 0 for the
    lanes that are not members of those points' far entries)."""
    O = oracle_mod
    C = 49
    rng = np.random.default_rng(7)
    pos, nrm, area, _ = random_cloud(3000, 77, 1)
    mu = rng.standard_normal((3000, C))
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    xs = rng.uniform(-1.5, 1.5, (1500, 3)).astype(np.float32).astype(np.float64)
    xs[::25] = pos[rng.choice(3000, len(xs[::25]), replace=False)]
    p = eng.KernelParams(epsilon=eps)
    want = r.primal(O.Params(eps), 2.0, xs)
    d_out = rng.standard_normal((len(xs), C)).astype(np.float32)
    w = r.adjoint_mag(O.Params(eps), 2.0, xs, d_out.astype(np.float64))
    for rnd in range(2):  # the second primal -> adjoint pair replays interaction lists
        got = t.primal(xs, p, 2.0)
        check(f"regularized bounds eps={eps} primal (pass {rnd})", got, want)
        buf = t.make_buffer()
        t.adjoint(xs, p, 2.0, d_out, None, buf)
        g = t.flush_gradients(buf)
        tag = f"regularized bounds eps={eps} adjoint (pass {rnd})"
        check(f"{tag} moments", g.moments, w["moments"], w["moments_abs"])
        check(f"{tag} normals", g.normals, w["normals"], w["normals_abs"])
        scalar(f"{tag} d_epsilon", g.d_epsilon, w["d_eps"], w["d_eps_abs"])


# ---------------------------------------------------------------- errors
def test_error_behaviour(eng, oracle_mod):
    t = eng.DipoleTree(0)
    with pytest.raises(eng.DataError):
        t.build(eng.OrientedPointCloud(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0),
                                       np.zeros((0, 1))))
    pos, nrm, area, mu = random_cloud(10, 24, 2)
    t.build(eng.OrientedPointCloud(pos, nrm, area, mu))
    with pytest.raises(eng.DataError):
        t.set_channel_kernels([0])
    with pytest.raises(eng.DataError):
        t.update_moments(eng.OrientedPointCloud(pos[:-1], nrm[:-1], area[:-1], mu[:-1]))


def test_host_pointer_pipeline_matches_device_path(eng, oracle_mod):
    """Host-resident batches take the chunked H2D/compute/D2H pipeline. Chunks
    are Morton-sorted separately, so warp groupings (hence fp32 summation
    order) differ from the device-resident path: agreement to rounding."""
    import torch

    rng = np.random.default_rng(77)
    n, C, q = 20000, 49, 600_000
    pos, nrm, area, _ = random_cloud(n, 78, 1)
    mu = rng.standard_normal((n, C))
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t, _ = make(eng, oracle_mod, pos, nrm, area, mu, kinds)
    xs = rng.uniform(-1.2, 1.2, (q, 3)).astype(np.float32).astype(np.float64)
    d_out = rng.standard_normal((q, C)).astype(np.float32)
    p = eng.KernelParams(epsilon=0.02)
    host = t.primal(xs, p, 2.0)
    dev = t.primal(torch.from_numpy(xs).cuda(), p, 2.0).cpu().numpy()
    assert rel_scale_err(host, dev) < 1e-5
    assert close(host, dev, rtol=1e-4, atol=1e-6)[0] == 0
    b1, b2 = t.make_buffer(), t.make_buffer()
    t.adjoint(xs, p, 2.0, d_out, None, b1)
    t.adjoint(torch.from_numpy(xs).cuda(), p, 2.0, torch.from_numpy(d_out).cuda(), None, b2)
    g1, g2 = t.flush_gradients(b1), t.flush_gradients(b2)
    assert rel_scale_err(g1.moments, g2.moments) < 1e-6

    # host-async mode: same kernels, results complete at flush / synchronize;
    # pinned and pageable host buffers, back-to-back steps reusing the staging
    pin_x = torch.from_numpy(xs).pin_memory()
    pin_d = torch.from_numpy(d_out).pin_memory()
    pin_o = torch.empty((q, C), dtype=torch.float32).pin_memory()
    t.set_host_async(True)
    try:
        for xs_in, do_in, out_in in ((pin_x, pin_d, pin_o), (xs, d_out, None)):
            for _ in range(2):
                o = t.primal(xs_in, p, 2.0, out=out_in)
                b3 = t.make_buffer()
                t.adjoint(xs_in, p, 2.0, do_in, None, b3)
                g3 = t.flush_gradients(b3)
                t.synchronize()  # host-async: the point gradients land on the D2H stream
                o = o.numpy() if hasattr(o, "numpy") else o
                assert np.array_equal(o, host)
                assert np.array_equal(g3.moments, g1.moments)
                assert np.array_equal(g3.normals, g1.normals)
        o = t.primal(xs, p, 2.0)
        t.synchronize()
        assert np.array_equal(o, host)
    finally:
        t.set_host_async(False)


@pytest.mark.parametrize("env", ["DPL_ADJOINT_TMEM", "DPL_ADJOINT_TC", "DPL_ADJOINT_SINGLE_PHASE",
                                 "DPL_FORWARD_TMEM", "DPL_FORWARD_NO_TC", "DPL_FORWARD_SINGLE_PHASE",
                                 "DPL_NO_ILIST", "DPL_ILIST_POOL", "DPL_ILIST_ALWAYS"])
def test_alternate_kernel_paths(env):
    """The opt-in / fallback kernels (selected once per process from the
    environment) pass the same forward / adjoint / render parity tests."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run(
        [sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_parity.py"), "-q", "-x",
         "-m", "gpu", "-k",
         "(adjoint or render or many_channel or primal or interaction_list) and not alternate"],
        env=dict(os.environ, **{env: "1"}), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_interaction_list_reuse_is_keyed_on_the_batch(eng, oracle_mod):
    """The adjoint reuses the primal's interaction lists only for bit-identical
    queries (same tree, beta, count): queries edited in place in the same
    device buffer, a different beta, or a rebuilt tree all re-traverse."""
    import torch

    O = oracle_mod
    pos, nrm, area, mu = random_cloud(3000, 31, 49)
    kinds = np.ones(49, np.uint8)
    kinds[0] = 0
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    rng = np.random.default_rng(32)
    q = 4096
    xs1 = rng.uniform(-1.2, 1.2, (q, 3))
    xs2 = rng.uniform(-1.2, 1.2, (q, 3))
    d_out = rng.standard_normal((q, 49)).astype(np.float32)
    p = eng.KernelParams(epsilon=0.05)
    dev = torch.from_numpy(xs1).cuda()
    ddo = torch.from_numpy(d_out).cuda()
    b0 = t.make_buffer()
    for beta_f, beta_a in ((2.0, 2.0), (2.0, 3.0)):
        dev.copy_(torch.from_numpy(xs1))
        # a primal -> adjoint pair on this buffer makes the next primal build lists
        t.primal(dev, p, beta_f)
        t.adjoint(dev, p, beta_f, ddo, None, b0)
        b0.reset()
        t.primal(dev, p, beta_f)  # lists for xs1 at beta_f
        dev.copy_(torch.from_numpy(xs2))  # same pointer, new content
        b = t.make_buffer()
        t.adjoint(dev, p, beta_a, ddo, None, b)
        g = t.flush_gradients(b)
        w = r.adjoint_mag(O.Params(0.05), beta_a, xs2, d_out.astype(np.float64))
        tag = f"list reuse keyed on batch beta {beta_f}->{beta_a}"
        check(f"{tag} moments", g.moments, w["moments"], w["moments_abs"])
        check(f"{tag} normals", g.normals, w["normals"], w["normals_abs"])
        scalar(f"{tag} d_epsilon", g.d_epsilon, w["d_eps"], w["d_eps_abs"])
        # and a primal on the edited buffer matches the oracle too
        got = t.primal(dev, p, beta_a).cpu().numpy()
        check(f"{tag} primal", got, r.primal(O.Params(0.05), beta_a, xs2))
    # rebuilt tree (same queries): lists are rebuilt as well
    pos2 = pos + 0.01
    t.build(eng.OrientedPointCloud(pos2, nrm, area, mu))
    t.set_channel_kernels(kinds)
    r2 = O.OracleTree(O.Cloud(pos2, nrm, area, mu))
    r2.set_kinds(kinds)
    got = t.primal(dev, p, 2.0).cpu().numpy()
    assert close(got, r2.primal(O.Params(0.05), 2.0, xs2))[0] == 0


@pytest.mark.parametrize("C", [2, 49])
def test_list_replay_is_bitwise_the_tree_walk(eng, oracle_mod, C):
    """K9 records the entries in the reference's pop order (bhtree.cpp:188-234):
    a primal that replays the lists returns bit-for-bit what the primal that
    walked the tree itself returned, on a deep clustered cloud (every lane-mask
    and sibling-order case) and with partial warps."""
    import torch

    O = oracle_mod
    rng = np.random.default_rng(77)
    base = rng.uniform(-1, 1, (40, 3))
    pos = np.concatenate([base[rng.integers(0, 40, 6000)] + rng.normal(0, 0.02, (6000, 3)),
                          rng.uniform(-1, 1, (3000, 3))])
    n = pos.shape[0]
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = rng.uniform(0.5, 1.0, n) / n
    mu = rng.standard_normal((n, C))
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t, r = make(eng, O, pos, nrm, area, mu, kinds, max_leaf=4)
    q = 5000 + 13  # a partial last warp
    xs = rng.uniform(-1.3, 1.3, (q, 3))
    p = eng.KernelParams(epsilon=0.03)
    dev = torch.from_numpy(xs).cuda()
    walked = t.primal(dev, p, 2.0).cpu().numpy()  # no lists yet: the kernel walks the tree
    b = t.make_buffer()
    t.adjoint(dev, p, 2.0, torch.zeros((q, C), dtype=torch.float32, device="cuda"), None, b)
    listed = t.primal(dev, p, 2.0).cpu().numpy()   # primal -> adjoint pair seen: lists
    again = t.primal(dev, p, 2.0).cpu().numpy()
    assert np.array_equal(walked, listed)
    assert np.array_equal(listed, again)
    check(f"list replay C={C} primal", listed, r.primal(O.Params(0.03), 2.0, xs))


@pytest.mark.parametrize("C", [1, 2, 3, 17, 33, 49])
def test_primal_channel_bitwise_equals_primal(eng, oracle_mod, C):
    """primal_channel(c) == primal()[c] bitwise (test_bhtree.cpp:140) for every
    layout, including the dipole-only kernel primal_channel(0) uses."""
    O = oracle_mod
    pos, nrm, area, mu = random_cloud(3000, 40 + C, C)
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t, r = make(eng, O, pos, nrm, area, mu, kinds)
    xs = np.random.default_rng(41).uniform(-1.3, 1.3, (2500, 3))
    p = eng.KernelParams(epsilon=0.04)
    full = t.primal(xs, p, 2.0)
    for c in sorted({0, C // 2, C - 1}):
        assert np.array_equal(t.primal_channel(xs, p, 2.0, c), full[:, c]), c
    want = r.primal(O.Params(0.04), 2.0, xs)
    assert close(full, want)[0] == 0


def _branchy_cloud(depth):
    """A cloud whose octree has 8 non-empty children at EVERY level on the path
    to a cluster at p (7 decoy points at the centres of the sibling cells, built
    with the reference's cell arithmetic, bhtree.cpp:43-50,77-78,93-95), and
    more than 8 points at p so the path reaches `depth`: the traversal stack
    peaks at 1 + 7 * depth entries."""
    pts = [(-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)]  # bbox [-1, 1]^3: root centre 0
    p = np.array([0.30011, 0.20017, 0.10029])
    c = np.zeros(3)
    h = 1.0 * (1.0 + 1e-7)
    for _ in range(depth):
        inside = [p[a] >= c[a] for a in range(3)]
        for o in range(8):
            sgn = [1.0 if (o >> a) & 1 else -1.0 for a in range(3)]
            child = tuple(c[a] + (0.5 * h) * sgn[a] for a in range(3))
            if [((o >> a) & 1) == 1 for a in range(3)] == inside:
                nxt = np.array(child)
            else:
                pts.append(child)
        c = nxt
        h = 0.5 * h
    step = min(1e-13, 2.0 ** -(depth + 8))
    for k in range(12):  # > max_leaf points at p (distinct, far below the last cell)
        pts.append(tuple(p + step * k))
    return np.array(pts), p


@pytest.mark.parametrize("depth", [21, 42])
def test_deepest_tree_branchy_path_stack(eng, oracle_mod, depth):
    """max_depth = 21 (one 63-bit key word) and 42 (the deepest the GPU build
    supports: two key words) on a cloud that fills every level of the path: the
    per-warp stack reaches its worst case (1 + 7 * depth <= 304) in every kernel
    family; structure, opening decisions and results equal the oracle's."""
    O = oracle_mod
    pos, p = _branchy_cloud(depth)
    n = pos.shape[0]
    rng = np.random.default_rng(5)
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = np.full(n, 1.0 / n)
    C = 5
    mu = rng.standard_normal((n, C))
    kinds = np.array([0, 1, 1, 1, 1], np.uint8)
    t, r = make(eng, O, pos, nrm, area, mu, kinds, max_leaf=8, max_depth=depth)
    a, b = t.export(), r.export()
    for k in ("topo", "order", "leaf_of", "geo"):
        assert np.array_equal(a[k], b[k]), k
    assert int(a["topo"].shape[0]) == int(b["topo"].shape[0])
    prm = eng.KernelParams(epsilon=1e-7)
    if depth > 21:
        # queries inside the deepest cells open the whole path (stack peak
        # 1 + 7 * 42 = 295): the opening decisions are exact (fp64 fallback) and
        # must equal the oracle's. Their VALUES are not compared: 1e-13 from a
        # point the double-float distance (2^-46 |x| absolute) is not fp32-accurate.
        deep = p + rng.normal(0, 2.0 ** -(depth + 2), (256, 3))
        got_d, cnt_d = t.primal(deep, prm, 2.0, visited=True)
        _, wcnt_d = r.primal(O.Params(1e-7), 2.0, deep, counters=True)
        counters_equal("depth-42 tree counters (queries inside the deepest cells)", cnt_d, wcnt_d)
        assert np.isfinite(got_d).all()
        buf = t.make_buffer()
        t.adjoint(deep, prm, 2.0, np.zeros((256, C), np.float32), None, buf)  # walks the path
        t.flush_gradients(buf)
    # queries around p open the path down to their distance
    xs = p + rng.normal(0, 1e-9, (256, 3))
    xs = np.concatenate([xs, rng.uniform(-1, 1, (256, 3))])
    got, cnt = t.primal(xs, prm, 2.0, visited=True)
    want, wcnt = r.primal(O.Params(1e-7), 2.0, xs, counters=True)
    counters_equal("deepest tree counters", cnt, wcnt)
    # queries 1e-9 from a cluster whose terms cancel to ~1e-4 of their sum:
    # the Sum|terms|-scaled bar applies (tests/parity.py)
    wm = r.primal_mag(O.Params(1e-7), 2.0, xs)
    check(f"deepest tree (depth {depth}, 8 children per path node) primal", got, want, wm["out_abs"])
    d_out = rng.standard_normal((xs.shape[0], C)).astype(np.float32)
    w = r.adjoint_mag(O.Params(1e-7), 2.0, xs, d_out.astype(np.float64))
    for rnd in range(2):  # fused walk, then list replay
        t.primal(xs, prm, 2.0)
        buf = t.make_buffer()
        t.adjoint(xs, prm, 2.0, d_out, None, buf)
        g = t.flush_gradients(buf)
        check(f"deepest tree d{depth} adjoint moments (pass {rnd})", g.moments, w["moments"], w["moments_abs"])
        check(f"deepest tree d{depth} adjoint normals (pass {rnd})", g.normals, w["normals"], w["normals_abs"])
    with pytest.raises(eng.UsageError):
        t.build(eng.OrientedPointCloud(pos, nrm, area, mu), 8, 43)
