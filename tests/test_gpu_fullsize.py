"""Parity at BASELINE config 2's full size (N = 1e6 points, C = 49, Q = 4e6
queries), through properties that do not need the oracle to evaluate every
query:
  * the tree built on the GPU is bit-identical to the reference's build
    (oracle, the same 1e6 points);
  * the production step — Hilbert sort, K9 lists, list-replay forward and
    adjoint, flush — answers a random subset of the 4M queries like the oracle
    (the rest of the batch shares the warps, lists and accumulators);
  * forward / adjoint duality: the primal is linear in the point moments for
    fixed geometry, so <d_out, primal> = <d moments, moments> over the whole
    batch (the adjoint is the transpose of the forward), checked to fp32
    accumulation accuracy;
  * the adjoint is linear in d_out: a(d1) + a(d2) = a(d1 + d2).
"""
import numpy as np
import pytest
from parity import check, counters_equal, scalar

pytestmark = pytest.mark.gpu


def test_config2_full_size_properties(oracle_mod):
    import torch

    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import workloads as W

    O = oracle_mod
    w = W.config2()
    eps = W.epsilon_for("config2")
    c = w["cloud"]
    Q, C = w["xs"].shape[0], c.channels
    t = P.DipoleTree(0)
    t.build(c)
    t.set_channel_kernels(w["kinds"])
    r = O.OracleTree(O.Cloud(c.positions, c.normals, c.areas, c.moments))
    r.set_kinds(w["kinds"])
    a, b = t.export(), r.export()
    for k in ("topo", "order", "leaf_of", "geo"):
        assert np.array_equal(a[k], b[k]), k

    p = P.KernelParams(epsilon=eps)
    xs = torch.from_numpy(w["xs"]).cuda()
    d1 = W.upstream(Q, C, w["d_out_seed"])
    d2 = W.upstream(Q, C, [11, 12])
    grads = []
    for step in range(2):  # the second primal -> adjoint pair replays K9 lists
        out = t.primal(xs, p, 2.0).cpu().numpy()
        for d in (d1, d2, d1 + d2) if step == 1 else (d1,):
            buf = t.make_buffer()
            t.adjoint(xs, p, 2.0, torch.from_numpy(d).cuda(), None, buf)
            grads.append(t.flush_gradients(buf))
    g1, g1b, g2, g12 = grads

    # subset of the production batch against the reference's primal
    idx = np.random.default_rng(3).choice(Q, 1500, replace=False)
    want, wcnt = r.primal(O.Params(eps), 2.0, w["xs"][idx], counters=True)
    check("config2 full size forward, 1500-query subset of the 4M batch", out[idx], want)
    # and every output of the whole 4M-query batch (list replay pass)
    check("config2 full size forward, all 4M queries x 49 channels", out,
          r.primal(O.Params(eps), 2.0, w["xs"]))
    _, cnt = t.primal(xs[torch.from_numpy(idx).cuda()], p, 2.0, visited=True)
    counters_equal("config2 full size subset counters", cnt.cpu().numpy(), wcnt)

    # the whole 4M-query adjoint (fused, then list replay) against the oracle's
    wa = r.adjoint_mag(O.Params(eps), 2.0, w["xs"], d1.astype(np.float64))
    for name, g in (("fused", g1), ("list replay", g1b)):
        tag = f"config2 full size adjoint of all 4M queries ({name})"
        check(f"{tag} moments", g.moments, wa["moments"], wa["moments_abs"])
        check(f"{tag} normals", g.normals, wa["normals"], wa["normals_abs"])
        scalar(f"{tag} d_epsilon", g.d_epsilon, wa["d_eps"], wa["d_eps_abs"])

    # duality <d_out, primal> = <d moments, moments> (fp64 sums of fp32 terms)
    lhs = float(np.einsum("qc,qc->", d1.astype(np.float64), out.astype(np.float64)))
    rhs = float(np.einsum("mc,mc->", g1.moments.astype(np.float64), np.asarray(c.moments, np.float64)))
    scale = float(np.abs(d1).astype(np.float64).ravel() @ np.abs(out).astype(np.float64).ravel())
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)

    # the fused (first) and list-replay (second) adjoints agree; linearity in d_out
    s = np.abs(g1.moments).max()
    assert np.abs(g1b.moments - g1.moments).max() <= 1e-6 * s
    assert np.abs((g1b.moments + g2.moments) - g12.moments).max() <= 1e-5 * np.abs(g12.moments).max()
    assert np.abs((g1b.normals + g2.normals) - g12.normals).max() <= 1e-5 * np.abs(g12.normals).max()
