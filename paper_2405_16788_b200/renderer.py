"""Render step over the engine: render_ray / render_ray_backward for ray batches.

Mirrors proj/src/renderer.cpp:106-231 (no lights) with the direct-rgb head
(proj/src/radiance.cpp:133-145): the forward records a device tape, the
backward takes d_rgb per ray and emits the tree adjoint into a GradientBuffer.
Also provides look_at / generate_ray (renderer.cpp:16-38) in numpy fp64.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import KernelParams, RenderParams, check, lib
from .bhtree import DipoleTree, GradientBuffer, _in, _out_like


def look_at(position, target, up, fov_deg, width, height):
    """Camera::look_at (renderer.cpp:16-33): returns (position, R (3x3, columns
    x, y, z), fx, fy, cx, cy)."""
    position = np.asarray(position, np.float64)
    z = np.asarray(target, np.float64) - position
    z = z / np.sqrt((z[0] * z[0] + z[1] * z[1]) + z[2] * z[2])
    x = np.cross(z, np.asarray(up, np.float64))
    x = x / np.sqrt((x[0] * x[0] + x[1] * x[1]) + x[2] * x[2])
    y = np.cross(z, x)
    f = 0.5 * width / np.tan(0.5 * fov_deg * np.pi / 180.0)
    return dict(position=position, R=np.stack([x, y, z], axis=1), fx=f, fy=f, cx=0.5 * width,
                cy=0.5 * height, width=width, height=height)


def generate_rays(cam, px, py):
    """generate_ray (renderer.cpp:35-38) for arrays of pixel coordinates -> (R, 6)."""
    px = np.asarray(px, np.float64)
    py = np.asarray(py, np.float64)
    dc = np.stack([(px - cam["cx"]) / cam["fx"], (py - cam["cy"]) / cam["fy"], np.ones_like(px)], 1)
    d = dc @ cam["R"].T
    d = d / np.sqrt((d[:, 0] ** 2 + d[:, 1] ** 2) + d[:, 2] ** 2)[:, None]
    o = np.broadcast_to(cam["position"], d.shape)
    return np.ascontiguousarray(np.concatenate([o, d], axis=1))


@dataclass
class RenderSettings:
    lambda_scale: float = 20.0     # SceneModel::lambda_scale (fields.hpp:17)
    beta_bh: float = 2.0           # SceneModel::beta_bh (fields.hpp:18)
    background: tuple = (0.0, 0.0, 0.0)
    t_near: float = 2.0
    t_far: float = 6.0
    seed: int = 3

    def c(self):
        rp = RenderParams()
        rp.lambda_scale = self.lambda_scale
        rp.beta_bh = self.beta_bh
        for i in range(3):
            rp.background[i] = self.background[i]
        rp.t_near = self.t_near
        rp.t_far = self.t_far
        rp.seed = self.seed
        return rp


class Tape:
    def __init__(self):
        h = C.c_void_p()
        check(lib().dpl_tape_create(C.byref(h)))
        self._h = h.value

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().dpl_tape_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None


def render_forward(tree: DipoleTree, params: KernelParams, rs: RenderSettings, rays, S: int,
                   ts=None, deltas=None, tape: Tape | None = None):
    """render_ray for R rays; returns (rgb (R, 3) fp32, tape)."""
    R = int(rays.shape[0])
    rp, k1 = _in(rays, np.float64, (R, 6))
    tp, k2 = _in(ts, np.float64, (R, S)) if ts is not None else (None, None)
    dp, k3 = _in(deltas, np.float64, (R, S)) if deltas is not None else (None, None)
    op, rgb = _out_like(k1, (R, 3), np.float32)
    tape = tape or Tape()
    rpc = rs.c()
    check(lib().dpl_render_forward(tree._h, C.byref(params), C.byref(rpc), rp, R, int(S), tp, dp,
                                   op, tape._h))
    return rgb, tape


def render_backward(tree: DipoleTree, params: KernelParams, rs: RenderSettings, tape: Tape, d_rgb,
                    buf: GradientBuffer):
    """render_ray_backward (d_weight = 0) for the taped rays; returns
    (d_lambda, d_background)."""
    dp, k = _in(d_rgb, np.float32)
    rpc = rs.c()
    dl = C.c_double()
    dbg = (C.c_double * 3)()
    check(lib().dpl_render_backward(tree._h, C.byref(params), C.byref(rpc), tape._h, dp, buf._h,
                                    C.byref(dl), dbg))
    buf.dirty = True
    return dl.value, np.array(list(dbg))


def uniform(seed: int, counter: int) -> float:
    return float(lib().dpl_uniform(seed, counter))
