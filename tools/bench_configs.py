#!/usr/bin/env python
"""Per-configuration timings with rooflines and CPU baselines (bench.py carries the
config-4 headline and plain timings of configs 1, 2, 3, 5 under "extra").

    python tools/bench_configs.py --config 1|3|4|5 [--steps K] [--scale s]

Config 1: forward primal, N=1e5 sphere, C=2, Q=1e6 (+ primal_channel).
Config 3: render step (65,536 rays x 128 samples) on the config-1 cloud, C=4:
          render_forward -> L2 d_rgb -> render_backward (adjoint) -> flush.
Config 4: N=8e6 shapes cloud, C=49, Q=6.4e7 forward + adjoint + flush.
Config 5: full differentiable step, N=4e6, 1,048,576 rays x 192 samples:
          render fwd/bwd, flush, Adam(beta, alpha, n; lr 1e-2) + update_moments.
eps = 1.5 x mean 8-NN spacing from the GPU kNN (dpl_mean_knn_spacing). Times
are CUDA-event per-phase means (dpl_profile_*) and wall clock per step, after
a warm-up step; prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_16788_b200 as P  # noqa: E402
from paper_2405_16788_b200 import bhtree as B  # noqa: E402
from paper_2405_16788_b200 import renderer as Rn  # noqa: E402
from paper_2405_16788_b200 import workloads as W  # noqa: E402


def timed(fn, steps, tree):
    for _ in range(2):  # the list policy settles after one primal -> adjoint pair
        fn()
    torch.cuda.synchronize()
    B.profile_read(tree)
    B.profile_enable(tree, True)
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps
    prof = B.profile_read(tree)
    B.profile_enable(tree, False)
    return 1e3 * wall, {k: v[0] / steps for k, v in prof.items() if v[1]}


def flops_fwd_adj(tot, Cd, Cr):
    """SURVEY §8(d) cost model v1 (bench.flops_model)."""
    sys.path.insert(0, ROOT)
    import bench

    return bench.flops_model(tot, Cd, Cr)


def flops_render(tot, Cd, Cr):
    """Render path: forward values + channel-0 gradient (radial
    gradient terms count 0), adjoint with d_grad[0]. tot = (V, Fn, Ff, Pn, Pf)."""
    V, Fn, Ff, Pn, Pf = [float(x) for x in tot]
    fwd, adj = flops_fwd_adj(tot, Cd, Cr)
    K1n, K1f = 26.0, 12.0
    fwd += Fn * (K1n + 1 + 13 * Cd) + Ff * (K1f + 1 + 13 * Cd) + Pn * (K1n + 13 + 6 * Cd) + Pf * (K1f + 13 + 6 * Cd)
    adj += Fn * (K1n + 30) + Ff * (K1f + 30) + Pn * (K1n + 30) + Pf * (K1f + 30)
    return fwd, adj


def sample_counts(tree, p, rays, S, t_near, t_far, seed, max_rays=65536):
    """Per-sample (V, Fn, Ff, Pn, Pf) means over the render step's sample
    positions (the stratified sampler's fp64 t, o + t dir) of a ray subset."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    R = min(rays.shape[0], max_rays)
    tot = np.zeros(5)
    for r0 in range(0, R, 8192):
        r1 = min(R, r0 + 8192)
        ts, _ = O.stratified_samples(r1 - r0, S, t_near, t_far, seed, ray_offset=r0)
        o, d = rays[r0:r1, :3], rays[r0:r1, 3:]
        xs = (o[:, None, :] + ts[:, :, None] * d[:, None, :]).reshape(-1, 3)
        _, cnt = tree.primal(torch.from_numpy(np.ascontiguousarray(xs)).cuda(), p, 2.0, visited=True)
        tot += cnt.sum(dim=0).cpu().numpy()
    return tot / (R * S)


def roofline(flops, ms, peak):
    ach = flops / (ms * 1e-3) / 1e12
    return {"flops_per_launch": flops, "ms": ms, "achieved_tflops": ach, "peak_tflops": peak,
            "frac": ach / peak, "peak_source": "measured FFMA microbenchmark (dpl_peak_fp32)"}


def build(cloud, kinds, dev):
    t = P.DipoleTree(0, stream=torch.cuda.current_stream())
    t0 = time.perf_counter()
    t.build(cloud)
    t.set_channel_kernels(kinds)
    torch.cuda.synchronize()
    return t, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--cpu", action="store_true", help="also time the reference CPU path (SURVEY 8(d) subsets)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    res = {"config": args.config, "scale": args.scale}
    if args.config in (1, 2, 4):
        w = {1: W.config1, 2: W.config2, 4: W.config4}[args.config](scale=args.scale)
        c = w["cloud"]
        t0 = time.perf_counter()
        eps = B.default_epsilon(c)
        res["eps"], res["knn_s"] = eps, time.perf_counter() - t0
        tree, res["build_s"] = build(c, w["kinds"], dev)
        Q, C = w["xs"].shape[0], c.channels
        # two query batches alternated call by call: no timed call can reuse the
        # interaction lists of the previous one (an adjoint reuses its own
        # step's primal lists, as in training)
        xs_b = [torch.from_numpy(w["xs"]).to(dev),
                torch.from_numpy(W.step_queries(w, 0, 1)).to(dev)]
        it = [0]

        def nxt():
            it[0] += 1
            return xs_b[it[0] % 2]

        out = torch.empty((Q, C), device=dev)
        p = P.KernelParams(epsilon=eps)
        ms, ph = timed(lambda: tree.primal(nxt(), p, 2.0, out=out), args.steps, tree)
        res.update(points=c.size, nodes=tree.node_count(), queries=Q, channels=C,
                   forward_ms=ms, forward_phases=ph, forward_qps=Q / (ms * 1e-3))
        _, cnt = tree.primal(xs_b[0], p, 2.0, visited=True)
        tot = cnt.sum(dim=0).cpu().numpy()
        del cnt
        peak = B.peak_fp32(0)
        f_fwd, f_adj = flops_fwd_adj(tot, 1, C - 1)
        res["visited_per_query"] = float(tot[0] / Q)
        res["interactions_per_query"] = float(tot[1:].sum() / Q)
        fw = ph.get("forward", ms)
        res["roofline_forward"] = roofline(f_fwd, fw, peak)
        if args.config == 1:
            ms, _ = timed(lambda: tree.primal_channel(nxt(), p, 2.0, 0), args.steps, tree)
            res["primal_channel_ms"] = ms
            if args.cpu:  # the reference's primal over the full 1M-query batch, all cores
                sys.path.insert(0, os.path.join(ROOT, "oracle"))
                import oracle as O

                rt = O.OracleTree(O.Cloud(c.positions, c.normals, c.areas, c.moments), backend="ref")
                rt.set_kinds(w["kinds"])
                cores = O.ref_lib().ref_hardware_concurrency()
                t0 = time.perf_counter()
                rt.primal(O.Params(eps), 2.0, w["xs"], threads=cores)
                dt = time.perf_counter() - t0
                res["reference_cpu"] = {"queries": Q, "s": dt, "queries_per_s": Q / dt,
                                        "cores": cores, "speedup_gpu": (Q / dt) and (dt / (fw * 1e-3))}
        else:
            g = torch.Generator(device=dev).manual_seed(7)
            d_out = torch.randn((Q, C), device=dev, generator=g)
            buf = tree.make_buffer()
            mom = torch.empty((c.size, C), device=dev)
            nrm = torch.empty((c.size, 3), device=dev)

            def step():
                x = nxt()
                tree.primal(x, p, 2.0, out=out)
                tree.adjoint(x, p, 2.0, d_out, None, buf)
                tree.flush_gradients(buf, out=(mom, nrm))

            ms, ph2 = timed(step, args.steps, tree)
            res.update(step_ms=ms, step_phases=ph2, step_qps=Q / (ms * 1e-3))
            res["roofline_adjoint"] = roofline(f_adj, ph2.get("adjoint", ms), peak)
    elif args.config in (6, 7):
        # SURVEY 8(f) rows on the config-3 scene (config-1 sphere cloud, C=4):
        # 6 = sample_ray over its 65,536 camera rays (probe_count 1024, [2, 6]),
        # 7 = sample_grid at 256^3 (the reference meshes at up to 512^3)
        w = W.config3(scale=args.scale)
        c, rays = w["cloud"], w["rays"]
        t0 = time.perf_counter()
        eps = B.default_epsilon(c)
        res["eps"], res["knn_s"] = eps, time.perf_counter() - t0
        tree, res["build_s"] = build(c, w["kinds"], dev)
        p = P.KernelParams(epsilon=eps)
        cfg = P.RaySampler(t_near=2.0, t_far=6.0)
        if args.config == 6:
            rays_d = torch.from_numpy(rays).to(dev)
            ms, ph = timed(lambda: tree.sample_rays(p, 2.0, rays_d, cfg), args.steps, tree)
            _, _, cnt, br = tree.sample_rays(p, 2.0, rays_d, cfg)
            res.update(rays=rays.shape[0], probe_count=1024, ms=ms, phases=ph,
                       rays_per_s=rays.shape[0] / (ms * 1e-3),
                       bracketed=float(br.float().mean()), outputs="device-resident")
            ref_sample = 512
        else:
            r = max(8, int(256 * args.scale ** (1 / 3)))
            ms, ph = timed(lambda: tree.sample_grid(p, 2.0, (r, r, r), device=dev), args.steps,
                           tree)
            res.update(resolution=r, ms=ms, phases=ph, nodes_per_s=r ** 3 / (ms * 1e-3))
        # the reference's own implementation on the host cores, bounded sample
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O

        if O.have_ref():
            ref = O.RefModel(O.Cloud(c.positions, c.normals, c.areas, c.moments), eps, beta=2.0)
            t0 = time.perf_counter()
            if args.config == 6:
                ref.sample_rays(rays[:ref_sample], 2.0, 6.0, (1024, 24, 48, 8, 80), 80)
                dt = time.perf_counter() - t0
                res["reference_cpu"] = {"rays": ref_sample, "s": dt, "rays_per_s": ref_sample / dt,
                                        "cores": O.ref_lib().ref_hardware_concurrency()}
            else:
                ref.sample_grid((64, 64, 64))
                dt = time.perf_counter() - t0
                res["reference_cpu"] = {"resolution": 64, "s": dt, "nodes_per_s": 64 ** 3 / dt,
                                        "cores": O.ref_lib().ref_hardware_concurrency()}
    elif args.config == 8:
        # config-3 render step with the tiny-MLP head (4 x 256 hidden,
        # the paper preset's depth and width) instead of the direct-rgb head
        w = W.config3(scale=args.scale)
        c, rays, S = w["cloud"], w["rays"], w["S"]
        t0 = time.perf_counter()
        eps = B.default_epsilon(c)
        res["eps"], res["knn_s"] = eps, time.perf_counter() - t0
        tree, res["build_s"] = build(c, w["kinds"], dev)
        K = c.channels - 1
        sizes = [22 + K, 256, 256, 256, 256, 3]
        rng = np.random.default_rng(5)
        wts = np.concatenate([np.concatenate([np.sqrt(2.0 / a) * rng.standard_normal(a * b),
                                              np.zeros(b)]) for a, b in zip(sizes[:-1], sizes[1:])])
        tree.set_mlp_head(sizes, wts)
        R = rays.shape[0]
        rays_d = torch.from_numpy(rays).to(dev)
        target = torch.rand((R, 3), device=dev, generator=torch.Generator(device=dev).manual_seed(4))
        p = P.KernelParams(epsilon=eps)
        rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=3)
        buf = tree.make_buffer()
        mom = torch.empty((c.size, c.channels), device=dev)
        nrm = torch.empty((c.size, 3), device=dev)
        tape = Rn.Tape()
        scale = 2.0 / (3.0 * R)

        def step():
            rgb, _ = Rn.render_forward(tree, p, rs, rays_d, S, tape=tape)
            d_rgb = (scale * (rgb - target)).float()
            Rn.render_backward(tree, p, rs, tape, d_rgb, buf)
            tree.flush_gradients(buf, out=(mom, nrm))

        ms, ph = timed(step, args.steps, tree)
        tree.head_grads()
        Q = R * S
        # executed GEMM passes: forward, weight gradient, input gradient (+ the forward
        # again when the backward recomputes the activations, DPL_MLP_RECOMPUTE=1)
        passes = 4 if os.environ.get("DPL_MLP_RECOMPUTE") else 3
        flops = 2 * Q * sum(a * b for a, b in zip(sizes[:-1], sizes[1:])) * passes
        res.update(points=c.size, rays=R, samples=S, queries=Q, mlp=sizes, step_ms=ms, phases=ph,
                   samples_per_s=Q / (ms * 1e-3), mlp_tflops=flops / (ph.get("render", ms) * 1e-3) / 1e12,
                   mlp_gemm_passes=passes)
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O

        if O.have_ref():  # the reference's own render step with the same head, bounded sample
            ref = O.RefModel(O.Cloud(c.positions, c.normals, c.areas, c.moments), eps, beta=2.0)
            ref.set_mlp_head(sizes, wts)
            nr = 256
            ts, dlt = O.stratified_samples(nr, S, 2.0, 6.0, 3)
            t0 = time.perf_counter()
            ref.render_step(rays[:nr], ts, dlt, np.full((nr, 3), 0.5), scale)
            dt = time.perf_counter() - t0
            res["reference_cpu"] = {"rays": nr, "s": dt, "samples_per_s": nr * S / dt,
                                    "cores": O.ref_lib().ref_hardware_concurrency()}
    elif args.config in (3, 5):
        if args.config == 3:
            w = W.config3(scale=args.scale)
            c, rays, S = w["cloud"], w["rays"], w["S"]
            kinds = w["kinds"]
        else:
            n = max(64, int(4_000_000 * args.scale))
            pos, nrm_, area, rng = W.shapes_cloud(n, 5)
            mu = rng.standard_normal((n, 49))
            mu[:, 0] = 1.0  # geometry moment 1 (winding-number field: the shapes are opaque)
            c = W.cloud(pos, nrm_, area, mu)
            kinds = np.ones(49, np.uint8)
            kinds[0] = 0
            px = max(1, int(16384 * args.scale))
            rays = W.camera_rays(64, 1024, px, seed=2)
            S = 192
        t0 = time.perf_counter()
        eps = B.default_epsilon(c)
        res["eps"], res["knn_s"] = eps, time.perf_counter() - t0
        tree, res["build_s"] = build(c, kinds, dev)
        R = rays.shape[0]
        rays_d = torch.from_numpy(rays).to(dev)
        target = torch.rand((R, 3), device=dev, generator=torch.Generator(device=dev).manual_seed(4))
        p = P.KernelParams(epsilon=eps)
        rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=3)
        buf = tree.make_buffer()
        mom = torch.empty((c.size, c.channels), device=dev)
        nrm = torch.empty((c.size, 3), device=dev)
        opt = B.PointAdam(tree, lr=1e-2) if args.config == 5 else None
        tape = Rn.Tape()
        scale = 2.0 / (3.0 * R)

        def step():
            rgb, _ = Rn.render_forward(tree, p, rs, rays_d, S, tape=tape)
            d_rgb = (scale * (rgb - target)).float()
            Rn.render_backward(tree, p, rs, tape, d_rgb, buf)
            g = tree.flush_gradients(buf, out=(mom, nrm))
            if opt is not None:
                opt.step(g)

        ms, ph = timed(step, args.steps, tree)
        Q = R * S
        res.update(points=c.size, nodes=tree.node_count(), rays=R, samples=S, queries=Q,
                   channels=c.channels, step_ms=ms, phases=ph, samples_per_s=Q / (ms * 1e-3))
        # roofline: the direct-rgb render step evaluates channels 0..3 (values)
        # and the channel-0 gradient, and adjoints channels 0..3 with d_grad[0]
        # (renderer.cpp:125-127, radiance.cpp:133-145) — the 4-channel rate
        per = sample_counts(tree, p, rays, S, 2.0, 6.0, 3)
        f_fwd, f_adj = flops_render(per * Q, 1, 3)
        peak = B.peak_fp32(0)
        res["counters_per_sample"] = per.tolist()
        res["roofline_forward"] = roofline(f_fwd, ph.get("forward", ms), peak)
        res["roofline_adjoint"] = roofline(f_adj, ph.get("adjoint", ms), peak)
        res["channels_computed"] = "0..3 of %d (the direct-rgb head's inputs; the reference evaluates all %d, the rest never reach the output)" % (c.channels, c.channels)
        if args.cpu:  # the reference's render_ray + render_ray_backward on a 4,096-ray subset
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle as O

            nr = min(R, 4096)
            t0 = time.perf_counter()
            ref = O.RefModel(O.Cloud(c.positions, c.normals, c.areas, c.moments), eps, beta=2.0)
            t_build = time.perf_counter() - t0
            ts, dlt = O.stratified_samples(nr, S, 2.0, 6.0, 3)
            tgt = np.random.default_rng(4).uniform(0, 1, (nr, 3))
            t0 = time.perf_counter()
            ref.render_step(rays[:nr], ts, dlt, tgt, 2.0 / (3.0 * nr))
            dt = time.perf_counter() - t0
            res["reference_cpu"] = {"rays": nr, "samples": nr * S, "s": dt,
                                    "samples_per_s": nr * S / dt, "tree_build_s": t_build,
                                    "cores": O.ref_lib().ref_hardware_concurrency(),
                                    "note": "render_ray + render_ray_backward per ray (all channels), one flush"}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
