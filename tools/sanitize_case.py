#!/usr/bin/env python
"""Small workload for compute-sanitizer (one tool per run; profiles/r02_sanitizer.md):
every kernel family of the engine on a few thousand queries — tree build,
fused and list-replay forward / adjoint (a primal -> adjoint pair twice, so the
second pair builds and replays interaction lists), gradient forward, flush and
the split flush, the render step with both heads (direct-rgb and the tcgen05
tiny-MLP), sampling, kNN and Adam."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def guard():
    """DPL_GUARD=1: verify every engine buffer's guard zones now."""
    if os.environ.get("DPL_GUARD"):
        from paper_2405_16788_b200._lib import check, lib

        check(lib().dpl_guard_check(None))


def main():
    import torch

    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import bhtree as B
    from paper_2405_16788_b200 import parallel as Pl
    from paper_2405_16788_b200 import renderer as Rn
    from paper_2405_16788_b200 import workloads as W

    rng = np.random.default_rng(0)
    n, q, C = 3000, 4096, 49
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = rng.uniform(0.5, 1, n) / n
    mu = rng.standard_normal((n, C))
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t = P.DipoleTree(0)
    t.build(P.OrientedPointCloud(pos, nrm, area, mu))
    t.set_channel_kernels(kinds)
    p = P.KernelParams(epsilon=0.05)
    xs = torch.from_numpy(rng.uniform(-1.3, 1.3, (q, 3))).cuda()
    d_out = torch.from_numpy(rng.standard_normal((q, C)).astype(np.float32)).cuda()
    buf = t.make_buffer()
    for _ in range(2):  # fused walk, then list build + replay
        t.primal(xs, p, 2.0)
        t.adjoint(xs, p, 2.0, d_out, None, buf)
        t.flush_gradients(buf)
    guard()
    t.primal_with_gradient(xs[:512], p, 2.0)
    t.primal_channel(xs, p, 2.0, 0)
    xs_h = xs.cpu().numpy()
    t.primal(xs_h, p, 2.0)  # host batch: the engine's own staging / output buffers
    t.adjoint(xs_h, p, 2.0, d_out.cpu().numpy(), None, buf)
    t.flush_gradients(buf)
    t.adjoint(xs, p, 2.0, d_out, None, buf)
    Pl.flush_allreduce(t, buf, chunks=3)
    B.mean_knn_spacing(pos)
    opt = B.PointAdam(t)
    g = t.flush_gradients(buf)
    opt.step(g)
    guard()
    # render step (config-3 layout) with both heads
    w = W.config3(scale=0.01)
    c = w["cloud"]
    tr = P.DipoleTree(0)
    tr.build(c)
    tr.set_channel_kernels(w["kinds"])
    rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=3)
    rays = w["rays"][:64]
    pe = P.KernelParams(epsilon=0.03)
    for head in (False, True):
        if head:
            sizes = [22 + c.channels - 1, 32, 32, 3]
            nw = sum(a * b + b for a, b in zip(sizes[:-1], sizes[1:]))
            tr.set_mlp_head(sizes, rng.standard_normal(nw) * 0.2)
        for _ in range(2):
            rgb, tape = Rn.render_forward(tr, pe, rs, rays, 24)
            b2 = tr.make_buffer()
            Rn.render_backward(tr, pe, rs, tape, np.full((64, 3), 1e-2, np.float32), b2)
            tr.flush_gradients(b2)
    tr.sample_grid(pe, 2.0, (16, 16, 16))
    tr.sample_rays(pe, 2.0, rays, P.RaySampler(t_near=2.0, t_far=6.0))
    torch.cuda.synchronize()
    if os.environ.get("DPL_GUARD"):
        import ctypes as C

        from paper_2405_16788_b200._lib import check, lib

        live = C.c_int64()
        check(lib().dpl_guard_check(C.byref(live)))
        print(f"guard zones intact on {live.value} live engine buffers")
    print("sanitize case ok")


if __name__ == "__main__":
    main()
