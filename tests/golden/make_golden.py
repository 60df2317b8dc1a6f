"""Generate the golden vectors in tests/golden/*.npz from the REFERENCE itself.

Runs only in the build container, where oracle/_ref/libdipole_ref.so has been
compiled from the unmodified /root/reference/proj sources (oracle/Makefile,
target `ref`). The fixtures are small, seeded and committed, so the CPU tests
can pin the C restatement (oracle/dipole_oracle.c) and the GPU tests can pin
the engine without /root/reference or the reference build present.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402


def random_cloud(n, seed, C):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1, 1, (n, 3))
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = (0.5 + 0.5 * np.abs(rng.uniform(-1, 1, n))) / n
    mu = rng.uniform(-1, 1, (n, C))
    return pos, nrm, area, mu


def sphere_cloud(m, C):
    """Fibonacci sphere as proj/tests/helpers.hpp:10-29 (moments: ch0 = 1)."""
    i = np.arange(m)
    z = 1.0 - 2.0 * (i + 0.5) / m
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = np.pi * (3.0 - np.sqrt(5.0)) * i
    n = np.stack([r * np.cos(phi), r * np.sin(phi), z], 1)
    mu = np.zeros((m, C))
    mu[:, 0] = 1.0
    if C > 1:
        mu[:, 1:] = np.random.default_rng(7).uniform(0, 1, (m, C - 1))
    return n.copy(), n.copy(), np.full(m, 4 * np.pi / m), mu


def kernels_fixture():
    rs = np.concatenate([[0.0, 1e-6, 1e-3], np.geomspace(1e-3, 20, 200)])
    params = [(0.0, 0, 0.0), (0.05, 0, 0.0), (0.3, 0, 0.0), (1.7, 0, 0.0), (0.0, 1, 0.05),
              (0.2, 1, 0.1)]
    out = np.zeros((len(params), 3, len(rs), 7))
    for a, (eps, ds, dl) in enumerate(params):
        for order in range(3):
            for k, r in enumerate(rs):
                if eps <= 0 and not ds and r == 0:
                    out[a, order, k] = np.nan  # singular at r = 0: undefined
                    continue
                out[a, order, k] = O.kernel_coeffs(r, O.Params(eps, ds, dl), order, backend="ref")
    xs = np.linspace(-8, 8, 161)
    erf = np.array([O.ref_lib().ref_erf_approx(x) for x in xs])
    ts = np.linspace(0, 10, 101)
    tau = np.array([O.ref_lib().ref_tau(t) for t in ts])
    zs = np.linspace(-12, 8, 81)
    haz = np.array([O.ref_lib().ref_normal_hazard(z) for z in zs])
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), rs=rs, params=np.array(params),
                        coeffs=out, erf_x=xs, erf=erf, tau_t=ts, tau=tau, haz_z=zs, haz=haz)


def tree_case(name, pos, nrm, area, mu, kinds, eps, betas, q, seed, max_leaf=8, max_depth=20,
              with_render=False):
    rng = np.random.default_rng(seed)
    cl = O.Cloud(pos, nrm, area, mu)
    t = O.OracleTree(cl, max_leaf, max_depth, backend="ref")
    t.set_kinds(kinds)
    e = t.export()
    xs = rng.uniform(-1.5, 1.5, (q, 3))
    xs[: min(3, q)] = pos[: min(3, q)]  # coincident queries
    p = O.Params(eps)
    C = mu.shape[1]
    res = dict(pos=pos, nrm=nrm, area=area, mu=mu, kinds=kinds, eps=eps, betas=np.array(betas),
               xs=xs, max_leaf=max_leaf, max_depth=max_depth, topo=e["topo"], geo=e["geo"],
               order=e["order"])
    for bi, beta in enumerate(betas):
        vals, vis = t.primal(p, beta, xs, counters=True, threads=1)
        v2, g2 = t.primal(p, beta, xs, mode="grad", threads=1)
        res[f"primal_{bi}"] = vals
        res[f"visited_{bi}"] = vis
        res[f"grad_{bi}"] = g2
        res[f"chan1_{bi}"] = t.primal(p, beta, xs, mode="channel", channel=min(1, C - 1), threads=1)
    d_out = rng.standard_normal((q, C))
    d_grad = rng.standard_normal((q, C, 3))
    for tag, dg in (("nog", None), ("g", d_grad)):
        m, n, de = t.adjoint(p, betas[0], xs, d_out, dg, threads=1)
        res[f"adj_{tag}_moments"], res[f"adj_{tag}_normals"], res[f"adj_{tag}_deps"] = m, n, de
    res["d_out"], res["d_grad"] = d_out, d_grad
    res["naive0"] = t.naive_sum(p, xs[:16], 0, int(kinds[0]))
    if with_render:
        model = O.RefModel(cl, epsilon=eps, lam=20.0, beta=2.0)
        R, S = 24, 16
        d = rng.standard_normal((R, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        rays = np.concatenate([-3.0 * d + 0.1 * rng.standard_normal((R, 3)), d], 1)
        ts, dl = O.stratified_samples(R, S, 1.0, 5.0, 3)
        target = rng.uniform(0, 1, (R, 3))
        out = model.render_step(rays, ts, dl, target, 2.0 / (3 * R), threads=1)
        res.update(rays=rays, ts=ts, deltas=dl, target=target, render_scale=2.0 / (3 * R),
                   **{f"render_{k}": np.asarray(v) for k, v in out.items()})
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **res)


def main():
    assert O.have_ref(), "build oracle/_ref first (make -C oracle ref)"
    kernels_fixture()
    pos, nrm, area, mu = random_cloud(300, 3, 3)
    tree_case("random300_c3", pos, nrm, area, mu, np.array([0, 1, 1], np.uint8), 0.15,
              [2.0, 4.0, np.inf], 64, 4)
    pos, nrm, area, mu = random_cloud(1200, 12, 2)
    pos[5] = pos[6]  # a coincident pair
    tree_case("random1200_c2_leaf4", pos, nrm, area, mu, np.array([0, 1], np.uint8), 0.08,
              [2.0], 48, 13, max_leaf=4)
    pos, nrm, area, mu = sphere_cloud(2000, 4)
    tree_case("sphere2000_c4", pos, nrm, area, mu, np.array([0, 1, 1, 1], np.uint8), 0.05,
              [2.0, 8.0], 48, 6, with_render=True)
    pos, nrm, area, mu = random_cloud(200, 21, 1)
    tree_case("random200_c1_singular", pos, nrm, area, mu, np.array([0], np.uint8), 0.0, [2.0],
              32, 22)
    # mean kNN spacing (pointcloud.cpp:51-65) and Adam (optimizer.cpp:65-81)
    rng = np.random.default_rng(9)
    kp = rng.uniform(-1, 1, (500, 3))
    adam = O.ref_lib().ref_adam_create()
    p = np.ascontiguousarray(rng.standard_normal(64))
    p0 = p.copy()
    grads = rng.standard_normal((3, 64))
    after = []
    for s in range(3):
        g = np.ascontiguousarray(grads[s])
        O.ref_lib().ref_adam_step(adam, p.ctypes.data_as(O._dp), g.ctypes.data_as(O._dp), 64, 1e-2)
        after.append(p.copy())
    O.ref_lib().ref_adam_free(adam)
    np.savez_compressed(os.path.join(HERE, "misc.npz"), knn_pos=kp,
                        knn_mean=O.mean_knn_spacing(kp, 8, backend="ref"), adam_p0=p0,
                        adam_grads=grads, adam_after=np.array(after))


if __name__ == "__main__":
    main()
