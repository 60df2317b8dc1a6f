"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved; these generators stand in with
the shapes, sizes and distributions BASELINE.json states. Values are drawn in
fp32 (numpy PCG64, fixed seeds) and promoted exactly to fp64, so the GPU and
the CPU oracle consume identical arrays. Interpretation choices left open by
BASELINE.json are recorded next to each generator.

``scale`` shrinks N and Q proportionally for parity tests that must finish on
the CPU oracle in seconds.
"""
from __future__ import annotations

import math

import numpy as np

from .bhtree import OrientedPointCloud

FOUR_PI = 4.0 * math.pi


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def _unit(rng, n):
    v = rng.standard_normal((n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def sphere_points(rng, n):
    """Uniform on the unit sphere, outward normals."""
    p = _unit(rng, n)
    return p, p.copy()


def torus_points(rng, n, R=1.0, r=0.35):
    """Uniform by area on a torus (rejection on the (R + r cos phi) density)."""
    out_p, out_n = [], []
    need = n
    while need > 0:
        m = int(need * 1.6) + 16
        th = rng.uniform(0, 2 * math.pi, m)
        ph = rng.uniform(0, 2 * math.pi, m)
        keep = rng.uniform(0, 1, m) < (R + r * np.cos(ph)) / (R + r)
        th, ph = th[keep][:need], ph[keep][:need]
        ring = R + r * np.cos(ph)
        out_p.append(np.stack([ring * np.cos(th), ring * np.sin(th), r * np.sin(ph)], 1))
        out_n.append(np.stack([np.cos(ph) * np.cos(th), np.cos(ph) * np.sin(th), np.sin(ph)], 1))
        need -= len(th)
    return np.concatenate(out_p), np.concatenate(out_n)


def random_rotation(rng):
    q = rng.standard_normal(4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def cloud(pos, nrm, area, mu):
    return OrientedPointCloud(_f32(pos), _f32(nrm), _f32(area), _f32(mu))


# ---------------------------------------------------------------------------
def config1(scale=1.0, seed=0):
    """Config 1: N=100,000 uniform on the unit sphere, normal = position,
    area 4 pi / N; C=2: channel 0 Dipole with geometry moment 1 (winding-number
    field), channel 1 Radial attribute ~ U[0,1]. Q=1,000,000 queries U[-1.5,1.5]^3."""
    n = max(16, int(100_000 * scale))
    q = max(32, int(1_000_000 * scale))
    rng = np.random.default_rng(seed)
    p, nn = sphere_points(rng, n)
    mu = np.stack([np.ones(n), rng.uniform(0, 1, n)], 1)
    c = cloud(p, nn, np.full(n, FOUR_PI / n), mu)
    qrng = np.random.default_rng([seed, 1])
    xs = _f32(qrng.uniform(-1.5, 1.5, (q, 3)))
    return dict(cloud=c, xs=xs, kinds=np.array([0, 1], np.uint8), name="config1")


def config2(scale=1.0, seed=0):
    """Config 2: N=1,000,000 — 95% torus (R=1, r=0.35; position jitter
    N(0, 0.005^2), normals + N(0, 0.05^2) renormalised), 5% outliers
    U[-2,2]^3 with random unit normals. Every point gets area 4 pi^2 R r / 950,000
    (recorded choice; BASELINE leaves areas open). C=49 channels ~ N(0,1): channel
    0 Dipole, 1..48 Radial. Q=4,000,000 U[-2,2]^3 (unsorted). Adjoint upstream
    gradients N(0,1) per query per channel."""
    n = max(32, int(1_000_000 * scale))
    q = max(32, int(4_000_000 * scale))
    rng = np.random.default_rng(seed + 2)
    nt = int(round(0.95 * n))
    no = n - nt
    p, nn = torus_points(rng, nt)
    p = p + rng.normal(0, 0.005, p.shape)
    nn = nn + rng.normal(0, 0.05, nn.shape)
    nn /= np.linalg.norm(nn, axis=1, keepdims=True)
    po = rng.uniform(-2, 2, (no, 3))
    pn = _unit(rng, no)
    pos = np.concatenate([p, po])
    nrm = np.concatenate([nn, pn])
    area = np.full(n, 4 * math.pi ** 2 * 1.0 * 0.35 / nt)
    mu = rng.standard_normal((n, 49))
    c = cloud(pos, nrm, area, mu)
    qrng = np.random.default_rng([seed + 2, 1])
    xs = _f32(qrng.uniform(-2, 2, (q, 3)))
    kinds = np.ones(49, np.uint8)
    kinds[0] = 0
    return dict(cloud=c, xs=xs, kinds=kinds, name="config2",
                d_out_seed=[seed + 2, 2])


def upstream(q, C, seed):
    """N(0,1) adjoint inputs (fp32)."""
    return np.random.default_rng(seed).standard_normal((q, C), dtype=np.float32)


def shapes_cloud(n, seed, shapes=64, outlier_frac=0.03):
    """Config 4/5 generator: union of `shapes` spheres/tori (alternating), centres
    U[-1.5,1.5]^3, scale U[0.1,0.4], uniform random rotation, torus r/R = 0.35,
    points proportional to surface area; plus 3% outliers U[-2,2]^3 with random
    normals. Areas: shape area / points on that shape; outliers get the mean
    per-point shape area (recorded choice)."""
    rng = np.random.default_rng(seed)
    ns = n - int(round(outlier_frac * n))
    centres = rng.uniform(-1.5, 1.5, (shapes, 3))
    scales = rng.uniform(0.1, 0.4, shapes)
    is_torus = np.arange(shapes) % 2 == 1
    areas = np.where(is_torus, 4 * math.pi ** 2 * scales * (0.35 * scales), 4 * math.pi * scales ** 2)
    counts = np.floor(ns * areas / areas.sum()).astype(np.int64)
    counts[: ns - counts.sum()] += 1
    P, N, A = [], [], []
    for s in range(shapes):
        k = int(counts[s])
        if is_torus[s]:
            p, nn = torus_points(rng, k, R=scales[s], r=0.35 * scales[s])
        else:
            p, nn = sphere_points(rng, k)
            p = p * scales[s]
        Rm = random_rotation(rng)
        P.append(p @ Rm.T + centres[s])
        N.append(nn @ Rm.T)
        A.append(np.full(k, areas[s] / max(k, 1)))
    no = n - ns
    P.append(rng.uniform(-2, 2, (no, 3)))
    N.append(_unit(rng, no))
    A.append(np.full(no, areas.sum() / ns))
    return np.concatenate(P), np.concatenate(N), np.concatenate(A), rng


def config4(scale=1.0, seed=0, queries=True):
    """Config 4: N=8,000,000 shapes cloud, C=49 N(0,1) moments; Q=64,000,000
    Morton-unsorted uniform queries U[-2,2]^3; forward + adjoint.
    queries=False skips the 64M-query draw (see config4_queries for slices)."""
    n = max(64, int(8_000_000 * scale))
    q = max(32, int(64_000_000 * scale))
    pos, nrm, area, rng = shapes_cloud(n, seed + 4)
    mu = rng.standard_normal((n, 49))
    kinds = np.ones(49, np.uint8)
    kinds[0] = 0
    xs = config4_queries(0, q, seed=seed) if queries else None
    return dict(cloud=cloud(pos, nrm, area, mu), xs=xs, kinds=kinds, name="config4",
                d_out_seed=[seed + 4, 2], q=q)


def config4_queries(lo, hi, batch=0, seed=0):
    """Queries [lo, hi) of config-4 query batch `batch` (batch 0 is config4()'s
    xs). Each coordinate is one 64-bit PCG64 draw, so a slice is drawn by
    advancing the generator: every rank of a sharded run gets exactly its part
    of the same global batch, whatever the rank count."""
    rng = np.random.default_rng([seed + 4, 1] if batch == 0 else [seed + 4, 1, batch])
    rng.bit_generator.advance(3 * int(lo))
    return _f32(rng.uniform(-2, 2, (int(hi) - int(lo), 3)))


def fibonacci_dirs(k):
    i = np.arange(k) + 0.5
    z = 1 - 2 * i / k
    r = np.sqrt(1 - z * z)
    ph = math.pi * (3 - math.sqrt(5)) * np.arange(k)
    return np.stack([r * np.cos(ph), r * np.sin(ph), z], 1)


def camera_rays(cams, res, px_per_cam, seed, fov=60.0, radius=4.0):
    """Pinhole cameras on a radius-4 sphere (Fibonacci directions, up = +y)
    looking at the origin; `px_per_cam` pixels per camera drawn without
    replacement; rays through pixel centres (generate_ray(px+.5, py+.5))."""
    from .renderer import generate_rays, look_at

    rng = np.random.default_rng(seed)
    out = []
    for d in fibonacci_dirs(cams):
        cam = look_at(radius * d, (0, 0, 0), (0, 1, 0), fov, res, res)
        pix = rng.choice(res * res, px_per_cam, replace=False)
        out.append(generate_rays(cam, pix % res + 0.5, pix // res + 0.5))
    return np.concatenate(out)


def config3(scale=1.0, seed=0):
    """Config 3: config-1 cloud with C=4 (channel 0 Dipole geometry moment 1,
    channel 1 = config-1 attribute, channels 2,3 ~ U[0,1] seed 1, all Radial);
    65,536 rays from 16 cameras (512x512, 60 deg), 4,096 random pixels each;
    128 stratified samples on [2,6] (seed 3); L2 loss against targets U[0,1]^3
    (seed 4): d_rgb = 2 (rgb - target) / (3 B)."""
    c1 = config1(scale=scale, seed=seed)
    cl = c1["cloud"]
    n = cl.size
    extra = np.random.default_rng(1).uniform(0, 1, (n, 2))
    mu = np.concatenate([cl.moments, _f32(extra)], 1)
    c = type(cl)(cl.positions, cl.normals, cl.areas, mu)
    px = max(1, int(4096 * scale))
    rays = camera_rays(16, 512, px, seed=2)
    B = rays.shape[0]
    target = np.random.default_rng(4).uniform(0, 1, (B, 3))
    return dict(cloud=c, rays=rays, S=128, t_near=2.0, t_far=6.0, sample_seed=3, target=target,
                scale_drgb=2.0 / (3.0 * B), kinds=np.array([0, 1, 1, 1], np.uint8),
                name="config3")


# Regularisation widths eps = 1.5 x mean 8-NN spacing (SceneModel::prepare,
# fields.cpp:10-11), computed ONCE by the CPU oracle on the full-size clouds
# (bit-identical to the reference's kd-tree result; tests/test_workloads.py
# re-derives config 1) and recorded here; queries use them as KernelParams.epsilon.
EPSILON = {
    "config1": 0.018716529322515815,
    "config2": 0.016877094843460314,
    "config3": 0.018716529322515815,  # config-1 cloud
    # the reference's mean_knn_spacing(8) on the config-4 cloud (oracle/_ref,
    # 48 s on 8 cores); the GPU kNN gives 0.007361985575915615 (summation order)
    "config4": 0.0073619855759169215,
}


def epsilon_for(name, scale=1.0):
    """Recorded eps at full size; for shrunken development runs the surface
    spacing scales like N^(-1/2)."""
    return EPSILON[name] / math.sqrt(scale)


def step_queries(w, rank, k):
    """Query batch k of a rank: k = 0 is rank_queries(); k > 0 are fresh draws
    from the same distribution (benchmarks alternate batches so that no step
    can reuse the previous step's traversal)."""
    if k == 0:
        return rank_queries(w, rank)
    lo, hi = {"config1": (-1.5, 1.5), "config2": (-2, 2), "config4": (-2, 2)}[w["name"]]
    q = w["xs"].shape[0]
    return _f32(np.random.default_rng([7919, rank, k]).uniform(lo, hi, (q, 3)))


def rank_queries(w, rank, seed=0):
    """Weak scaling: rank r > 0 draws its own queries from the same distribution."""
    if rank == 0:
        return w["xs"]
    lo, hi = {"config1": (-1.5, 1.5), "config2": (-2, 2), "config4": (-2, 2)}[w["name"]]
    q = w["xs"].shape[0]
    return _f32(np.random.default_rng([seed, 1000 + rank]).uniform(lo, hi, (q, 3)))
