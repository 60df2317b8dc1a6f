"""Pin the CPU oracle (oracle/dipole_oracle.c) to the reference.

1. Golden vectors in tests/golden/ were produced by the reference itself
   (proj/src compiled unmodified, tests/golden/make_golden.py). The restatement
   must reproduce them BIT-FOR-BIT (same fp64 operation order, no FMA).
2. Known-answer closed forms from the reference's own tests
   (proj/tests/test_kernels.cpp, test_oracles.cpp, test_bhtree.cpp).
3. When oracle/_ref is built (this container), fresh random cross-checks.
CPU only.
"""
import glob
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TREES = sorted(glob.glob(os.path.join(GOLD, "*_c*.npz")))


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


def test_kernel_coeffs_bitwise(oracle_mod):
    O = oracle_mod
    g = load("kernels.npz")
    for a, (eps, ds, dl) in enumerate(g["params"]):
        for order in range(3):
            for k, r in enumerate(g["rs"]):
                want = g["coeffs"][a, order, k]
                if np.isnan(want).all():
                    continue
                got = O.kernel_coeffs(float(r), O.Params(eps, bool(ds), dl), order)
                assert np.array_equal(got, want), (eps, ds, order, r)
    lib = O.port_lib()
    assert np.array_equal([lib.ora_erf(x) for x in g["erf_x"]], g["erf"])
    assert np.array_equal([lib.ora_tau(t) for t in g["tau_t"]], g["tau"])
    assert np.array_equal([lib.ora_normal_hazard(z) for z in g["haz_z"]], g["haz"])


@pytest.mark.parametrize("path", TREES, ids=[os.path.basename(p) for p in TREES])
def test_tree_queries_adjoint_bitwise(oracle_mod, path):
    O = oracle_mod
    g = np.load(path)
    cl = O.Cloud(g["pos"], g["nrm"], g["area"], g["mu"])
    t = O.OracleTree(cl, int(g["max_leaf"]), int(g["max_depth"]))
    t.set_kinds(g["kinds"])
    e = t.export()
    assert np.array_equal(e["topo"], g["topo"])
    assert np.array_equal(e["geo"], g["geo"])
    assert np.array_equal(e["order"], g["order"])
    p = O.Params(float(g["eps"]))
    C = g["mu"].shape[1]
    for bi, beta in enumerate(g["betas"]):
        vals, cnt = t.primal(p, beta, g["xs"], counters=True, threads=1)
        assert np.array_equal(vals, g[f"primal_{bi}"])
        assert np.array_equal(cnt[:, 0], g[f"visited_{bi}"])
        v2, g2 = t.primal(p, beta, g["xs"], mode="grad", threads=1)
        assert np.array_equal(g2, g[f"grad_{bi}"])
        ch = t.primal(p, beta, g["xs"], mode="channel", channel=min(1, C - 1), threads=1)
        assert np.array_equal(ch, g[f"chan1_{bi}"])
    for tag, dg in (("nog", None), ("g", g["d_grad"])):
        m, n, de = t.adjoint(p, g["betas"][0], g["xs"], g["d_out"], dg, threads=1)
        assert np.array_equal(m, g[f"adj_{tag}_moments"])
        assert np.array_equal(n, g[f"adj_{tag}_normals"])
        assert de == float(g[f"adj_{tag}_deps"])
    assert np.array_equal(t.naive_sum(p, g["xs"][:16], 0, int(g["kinds"][0])), g["naive0"])
    if "rays" in g:
        ts, dl = O.stratified_samples(g["rays"].shape[0], g["ts"].shape[1], 1.0, 5.0, 3)
        assert np.array_equal(ts, g["ts"]) and np.array_equal(dl, g["deltas"])
        out = t.render_step(p, 2.0, 20.0, [0, 0, 0], g["rays"], g["ts"], g["deltas"], g["target"],
                            float(g["render_scale"]), threads=1)
        for k in ("rgb", "moments", "normals", "d_eps", "d_lambda", "d_bg"):
            assert np.array_equal(np.asarray(out[k]), g[f"render_{k}"]), k


def test_knn_spacing_and_adam(oracle_mod):
    O = oracle_mod
    g = load("misc.npz")
    assert O.mean_knn_spacing(g["knn_pos"], 8) == float(g["knn_mean"])
    p = g["adam_p0"].copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for s in range(3):
        gr = np.ascontiguousarray(g["adam_grads"][s])
        O.port_lib().ora_adam_step(p.ctypes.data_as(O._dp), gr.ctypes.data_as(O._dp),
                                   m.ctypes.data_as(O._dp), v.ctypes.data_as(O._dp), 64, 1e-2,
                                   0.9, 0.999, 1e-8, s + 1)
        assert np.array_equal(p, g["adam_after"][s])


# ---------------------------------------------------------------- known answers
def test_kernel_closed_forms(oracle_mod):
    """proj/tests/test_kernels.cpp:12-18, 35-48, 126-153."""
    O = oracle_mod
    lib = O.port_lib()
    for x in np.linspace(-8, 8, 321):
        assert abs(lib.ora_erf(x) - math.erf(x)) <= 1e-14
    assert lib.ora_tau(0.0) == 0.0
    assert abs(lib.ora_tau(10.0) - 1.0) <= 1e-15
    assert abs(lib.ora_tau(1.0) - (math.erf(1) - 2 / math.sqrt(math.pi) * math.exp(-1))) <= 1e-14
    eps = 0.3
    k = O.kernel_coeffs(0.0, O.Params(eps), 2)
    sp = math.sqrt(math.pi)
    assert abs(k[0] - 4 / (3 * sp * eps ** 3)) <= 1e-12 * k[0]           # W(0)
    assert abs(k[2] - (-4 / (sp * eps ** 4))) <= 1e-12 * abs(k[2])       # dW/de(0)
    assert abs(k[3] - 8 / (sp * eps ** 6)) <= 1e-12 * k[3]               # dWp_r/de(0)
    # series / closed-form join at t = 0.05 (test_kernels.cpp:126-142)
    lo = O.kernel_coeffs(0.05 * eps * (1 - 1e-9), O.Params(eps), 2)
    hi = O.kernel_coeffs(0.05 * eps * (1 + 1e-9), O.Params(eps), 2)
    assert np.all(np.abs(lo - hi) <= 1e-6 * np.abs(hi) + 1e-300)


def test_single_point_closed_forms(oracle_mod):
    """Single-point naive sum (test_oracles.cpp:13-51) and adjoint on a one-point
    tree (test_bhtree.cpp:259-281)."""
    O = oracle_mod
    cl = O.Cloud(np.zeros((1, 3)), np.array([[0, 0, 1.0]]), np.array([0.8]), np.array([[0.6]]))
    t = O.OracleTree(cl)
    e = t.export()
    assert e["topo"].shape[0] == 1 and e["topo"][0, 5] == 1 and e["geo"][0, 4] == 0.0
    tau = O.port_lib().ora_tau(1 / 0.3)
    v = t.naive_sum(O.Params(0.3), np.array([[0, 0, -1.0]]), 0, 0)
    want = 0.8 * 0.6 * tau / (4 * math.pi)
    assert abs(v[0] - want) <= 1e-14 * want
    m, n, de = t.adjoint(O.Params(0.3), 2.0, np.array([[0, 0, -1.0]]), np.array([[2.5]]))
    assert abs(m[0, 0] - 0.8 * tau / (4 * math.pi) * 2.5) <= 1e-12 * abs(m[0, 0])


def test_degenerate_trees(oracle_mod):
    """test_bhtree.cpp:28-61: 1 point, 2 points (midpoint centroid), 100 coincident."""
    O = oracle_mod
    two = O.Cloud(np.array([[1.0, 2, 3], [3.0, 2, 3]]), np.tile([0, 0, 1.0], (2, 1)),
                  np.array([0.7, 0.7]), np.ones((2, 1)))
    e = O.OracleTree(two).export()
    assert np.abs(e["geo"][0, :3] - [2, 2, 3]).max() <= 1e-15
    same = O.Cloud(np.full((100, 3), 0.5), np.tile([0, 0, 1.0], (100, 1)), np.ones(100),
                   np.ones((100, 1)))
    e = O.OracleTree(same).export()
    leaves = e["topo"][e["topo"][:, 5] == 1]
    assert int((leaves[:, 1] - leaves[:, 0]).sum()) == 100


# ---------------------------------------------------------------- live cross-check
@pytest.mark.parametrize("seed,n,C", [(101, 700, 2), (202, 2500, 5)])
def test_port_matches_reference_build(oracle_mod, seed, n, C):
    O = oracle_mod
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1, 1, (n, 3))
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    cl = O.Cloud(pos, nrm, rng.uniform(0.1, 1, n) / n, rng.standard_normal((n, C)))
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    a, b = O.OracleTree(cl), O.OracleTree(cl, backend="ref")
    a.set_kinds(kinds)
    b.set_kinds(kinds)
    ea, eb = a.export(), b.export()
    for k in ("topo", "geo", "order", "leaf_of"):
        assert np.array_equal(ea[k], eb[k])
    xs = rng.uniform(-1.5, 1.5, (300, 3))
    p = O.Params(0.07)
    assert np.array_equal(a.primal(p, 2.0, xs), b.primal(p, 2.0, xs))
    d = rng.standard_normal((300, C))
    ma, na, da = a.adjoint(p, 2.0, xs, d, threads=1)
    mb, nb, db = b.adjoint(p, 2.0, xs, d, threads=1)
    assert np.array_equal(ma, mb) and np.array_equal(na, nb) and da == db


def _sphere_model(O, n=1500, C=4, seed=5):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, 3))
    pos = v / np.linalg.norm(v, axis=1, keepdims=True)
    mu = np.concatenate([np.ones((n, 1)), rng.uniform(0, 1, (n, C - 1))], axis=1)
    return O.Cloud(pos, pos.copy(), np.full(n, 4 * np.pi / n), mu)


def sphere_rays(R, seed):
    """Rays from radius 3 toward random targets near the unit sphere (some miss)."""
    rng = np.random.default_rng(seed)
    o = rng.standard_normal((R, 3))
    o = 3.0 * o / np.linalg.norm(o, axis=1, keepdims=True)
    tgt = rng.uniform(-1.3, 1.3, (R, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.concatenate([o, d], axis=1)


def test_port_matches_reference_sample_grid_and_rays(oracle_mod):
    """sample_grid (meshing.cpp:33-59) and sample_ray (renderer.cpp:46-86): the
    C restatement equals the reference's own code bitwise."""
    O = oracle_mod
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    cloud = _sphere_model(O)
    eps = 0.08
    ref = O.RefModel(cloud, eps, beta=2.0)
    port = O.OracleTree(cloud)
    kinds = np.ones(cloud.C, np.uint8)
    kinds[0] = 0
    port.set_kinds(kinds)
    p = O.Params(eps)
    for lo, hi in (((0, 0, 0), (0, 0, 0)), ((-1.2, -1.1, -1.0), (1.0, 1.1, 1.3))):
        a = port.sample_grid(p, 2.0, (9, 7, 5), lo, hi)
        b = ref.sample_grid((9, 7, 5), lo, hi)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    rays = sphere_rays(200, 6)
    counts = (256, 24, 48, 8, 80)
    a = port.sample_rays(p, 2.0, rays, 2.0, 4.5, counts, 80)
    b = ref.sample_rays(rays, 2.0, 4.5, counts, 80)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert 0 < a[3].sum() < len(rays)  # both bracketed and missing rays


def test_checkpoint_reader_parses_reference_dpck(oracle_mod, tmp_path):
    """load_checkpoint (optimizer.cpp:358-388) on a file the reference's own
    save_checkpoint wrote; malformed files raise DataError like the reference."""
    O = oracle_mod
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    from paper_2405_16788_b200 import DataError
    from paper_2405_16788_b200.bhtree import load_checkpoint

    cloud = _sphere_model(O, n=300, C=5, seed=9)
    ref = O.RefModel(cloud, 0.07, lam=17.0, beta=2.5, background=(0.1, 0.2, 0.3))
    path = tmp_path / "ref.dpck"
    ref.save_checkpoint(path, iter=42)
    ck = load_checkpoint(path)
    c = cloud.as_f64()
    assert ck["iter"] == 42 and ck["head_variant"] == 0 and not ck["with_albedo"]
    assert np.array_equal(ck["cloud"].positions, c.pos)
    assert np.array_equal(ck["cloud"].normals, c.nrm)
    assert np.array_equal(ck["cloud"].areas, c.area)
    assert np.array_equal(ck["cloud"].moments, c.mu)
    assert np.array_equal(ck["initial_normals"], c.nrm)
    assert (ck["lambda_scale"], ck["epsilon"], ck["beta_bh"]) == (17.0, 0.07, 2.5)
    assert np.array_equal(ck["background"], [0.1, 0.2, 0.3])
    data = path.read_bytes()
    (tmp_path / "bad.dpck").write_bytes(b"XXXX" + data[4:])
    with pytest.raises(DataError):
        load_checkpoint(tmp_path / "bad.dpck")
    (tmp_path / "short.dpck").write_bytes(data[:len(data) // 2])
    with pytest.raises(DataError):
        load_checkpoint(tmp_path / "short.dpck")
