"""Python mirror of ``dipole::DipoleTree`` (proj/include/dipole/bhtree.hpp:51-130).

Same method names, argument meaning and error behaviour as the reference, with
batched queries: where the reference takes one ``Vec3 x`` per call, these take
``xs`` of shape (Q, 3) and return (Q, C) outputs. Arrays may be numpy arrays
(host) or torch tensors (host or CUDA); outputs follow the query array's
device unless ``out=`` is given. Every call runs the sm_100a kernels of
libdipole_b200.so — there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (DPL_DIPOLE, DPL_RADIAL, Counters, DataError, KernelParams, NumericalError,
                   check, lib)

try:  # torch is optional plumbing (device memory, streams)
    import torch
except Exception:  # pragma: no cover
    torch = None

Dipole, Radial = DPL_DIPOLE, DPL_RADIAL


def _is_torch(a):
    return torch is not None and isinstance(a, torch.Tensor)


def _in(a, np_dtype, shape=None):
    """(pointer, keepalive) for an input array."""
    if a is None:
        return None, None
    if _is_torch(a):
        tdt = {np.float64: torch.float64, np.float32: torch.float32, np.uint8: torch.uint8}[np_dtype]
        t = a.detach().to(tdt).contiguous()
        if shape is not None:
            t = t.reshape(shape)
        return t.data_ptr(), t
    arr = np.ascontiguousarray(a, dtype=np_dtype)
    if shape is not None:
        arr = arr.reshape(shape)
    return arr.ctypes.data, arr


def _out_like(ref, shape, np_dtype):
    """Allocate an output on the device of `ref`."""
    if _is_torch(ref) and ref.is_cuda:
        tdt = {np.float32: torch.float32, np.float64: torch.float64, np.int64: torch.int64,
               np.int32: torch.int32, np.uint8: torch.uint8}[np_dtype]
        t = torch.empty(shape, dtype=tdt, device=ref.device)
        return t.data_ptr(), t
    arr = np.empty(shape, dtype=np_dtype)
    return arr.ctypes.data, arr


@dataclass
class OrientedPointCloud:
    """OrientedPointCloud (pointcloud.hpp:19-35) in SoA form: moments[:, 0] is the
    geometry moment and moments[:, 1:] the k_appearance appearance moments."""

    positions: object
    normals: object
    areas: object
    moments: object

    @property
    def size(self):
        return int(self.positions.shape[0])

    @property
    def channels(self):
        return int(self.moments.shape[1]) if len(self.moments.shape) > 1 else 1

    @property
    def k_appearance(self):
        return self.channels - 1


@dataclass
class PointGradients:
    """PointGradients (bhtree.hpp:28-36)."""

    channels: int
    moments: object   # N x C
    normals: object   # N x 3
    d_epsilon: float = 0.0

    def moment(self, point, channel):
        return self.moments[point, channel]


class GradientBuffer:
    """GradientBuffer (bhtree.hpp:40-49): device fp64 accumulators."""

    def __init__(self, tree: "DipoleTree"):
        h = C.c_void_p()
        check(lib().dpl_gradbuf_create(tree._h, C.byref(h)))
        self._h = h.value
        self.tree = tree
        self.dirty = False

    def reset(self):
        check(lib().dpl_gradbuf_zero(self._h))
        self.dirty = False

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().dpl_gradbuf_destroy(self._h)
            except Exception:  # interpreter shutdown: the process frees the device
                pass
            self._h = None


class DipoleTree:
    kDefaultMaxLeafSize = 8
    kDefaultMaxDepth = 20

    def __init__(self, device: int = 0, stream=None):
        h = C.c_void_p()
        s = None
        if stream is not None:
            s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        check(lib().dpl_tree_create(int(device), s, C.byref(h)))
        self._h = h.value
        self.device = device
        self.stream_ptr = s  # None: the library's own (blocking) stream
        self._built = False
        self._kinds = None
        self._async = False
        self._keep = []  # host arrays in flight (host-async mode)

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().dpl_tree_destroy(self._h)
            except Exception:  # interpreter shutdown: the process frees the device
                pass
            self._h = None

    def set_stream(self, stream):
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        check(lib().dpl_tree_set_stream(self._h, s))
        self.stream_ptr = s

    def synchronize(self):
        check(lib().dpl_tree_sync(self._h))
        self._keep.clear()

    def set_host_async(self, on: bool):
        """Host-async mode (dpl_tree_set_host_async): primal / adjoint on host
        batches return once queued; results are valid after synchronize() or
        flush_gradients(). Inputs must not be modified before then."""
        check(lib().dpl_tree_set_host_async(self._h, 1 if on else 0))
        self._async = bool(on)
        if not on:
            self._keep.clear()

    def prefetch(self, xs):
        """Host-async mode: upload the NEXT primal's host batch now (dpl_tree_prefetch);
        the primal given the same array skips its own upload."""
        q = int(xs.shape[0])
        xp, keep = _in(xs, np.float64, (q, 3))
        check(lib().dpl_tree_prefetch(self._h, xp, q))
        self._hold(keep)

    def _hold(self, *objs):
        if self._async:
            self._keep.append(objs)

    # -- build / moments ---------------------------------------------------------
    def build(self, cloud: OrientedPointCloud, max_leaf_size=kDefaultMaxLeafSize,
              max_depth=kDefaultMaxDepth):
        """DipoleTree::build (bhtree.cpp:158-169)."""
        n = cloud.size
        if n == 0:
            raise DataError("DipoleTree::build: empty cloud")
        Cc = cloud.channels
        p, k1 = _in(cloud.positions, np.float64, (n, 3))
        q, k2 = _in(cloud.normals, np.float64, (n, 3))
        a, k3 = _in(cloud.areas, np.float64, (n,))
        m, k4 = _in(cloud.moments, np.float64, (n, Cc))
        check(lib().dpl_tree_build(self._h, p, q, a, m, n, Cc, int(max_leaf_size), int(max_depth)))
        self._built = True
        self._kinds = np.zeros(Cc, np.uint8)

    def update_moments(self, cloud: OrientedPointCloud):
        """DipoleTree::update_moments (bhtree.cpp:171-176)."""
        n = cloud.size
        Cc = cloud.channels
        p, k1 = _in(cloud.positions, np.float64, (n, 3))
        q, k2 = _in(cloud.normals, np.float64, (n, 3))
        a, k3 = _in(cloud.areas, np.float64, (n,))
        m, k4 = _in(cloud.moments, np.float64, (n, Cc))
        check(lib().dpl_tree_update_moments(self._h, p, q, a, m, n, Cc))

    def set_channel_kernels(self, kernels):
        """DipoleTree::set_channel_kernels (bhtree.cpp:178-182)."""
        k = np.ascontiguousarray(kernels, dtype=np.uint8)
        check(lib().dpl_tree_set_channel_kernels(self._h, k.ctypes.data, len(k)))
        self._kinds = k.copy()

    def channel_kernels(self):
        return None if self._kinds is None else self._kinds.copy()

    def channels(self) -> int:
        c = C.c_int32()
        check(lib().dpl_tree_channels(self._h, C.byref(c)))
        return c.value

    def point_count(self) -> int:
        c = C.c_int64()
        check(lib().dpl_tree_point_count(self._h, C.byref(c)))
        return c.value

    def node_count(self) -> int:
        c = C.c_int64()
        check(lib().dpl_tree_node_count(self._h, C.byref(c)))
        return c.value

    def export(self):
        """nodes() + point_order() + point_leaf as arrays (TreeNode, bhtree.hpp:15-24)."""
        nn, n = self.node_count(), self.point_count()
        geo = np.zeros((nn, 5))
        topo = np.zeros((nn, 6), np.int32)
        order = np.zeros(n, np.int32)
        leaf_of = np.zeros(n, np.int32)
        check(lib().dpl_tree_export(self._h, geo.ctypes.data, topo.ctypes.data, order.ctypes.data,
                                    leaf_of.ctypes.data))
        return dict(geo=geo, topo=topo, order=order, leaf_of=leaf_of)

    def nodes(self):
        e = self.export()
        g, t = e["geo"], e["topo"]
        return dict(centroid=g[:, :3], area=g[:, 3], radius=g[:, 4], begin=t[:, 0], end=t[:, 1],
                    child_begin=t[:, 2], child_count=t[:, 3], parent=t[:, 4],
                    leaf=t[:, 5].astype(bool))

    def point_order(self):
        return self.export()["order"]

    def export_moments(self):
        nn, Cc = self.node_count(), self.channels()
        mv = np.zeros((nn, Cc, 3), np.float32)
        ms = np.zeros((nn, Cc), np.float32)
        check(lib().dpl_tree_export_moments(self._h, mv.ctypes.data, ms.ctypes.data))
        return mv, ms

    def dump(self, path: str):
        """DipoleTree::dump "DPLT" v1 (bhtree.cpp:465-494)."""
        check(lib().dpl_tree_dump(self._h, str(path).encode()))

    # -- forward queries ----------------------------------------------------------
    def primal(self, xs, params: KernelParams, beta_bh: float, out=None, visited=False):
        """DipoleTree::primal (bhtree.cpp:188-234) for a (Q, 3) batch -> (Q, C) fp32.
        visited=True also returns the per-query counters (Q, 5): visited, far
        near/far, point near/far."""
        q = int(xs.shape[0])
        Cc = self.channels()
        xp, xk = _in(xs, np.float64, (q, 3))
        if out is None:
            op, out = _out_like(xk, (q, Cc), np.float32)
        else:
            op = out.data_ptr() if _is_torch(out) else out.ctypes.data
        cnt = None
        cp = None
        if visited:
            cp, cnt = _out_like(xk, (q, 5), np.int64)
        check(lib().dpl_primal(self._h, C.byref(params), float(beta_bh), xp, q, op, None, cp))
        self._hold(xk, out)
        return (out, cnt) if visited else out

    def primal_channel(self, xs, params: KernelParams, beta_bh: float, channel: int):
        """DipoleTree::primal_channel (bhtree.cpp:236-274) -> (Q,) fp32."""
        q = int(xs.shape[0])
        xp, xk = _in(xs, np.float64, (q, 3))
        op, out = _out_like(xk, (q,), np.float32)
        check(lib().dpl_primal_channel(self._h, C.byref(params), float(beta_bh), xp, q,
                                       int(channel), op))
        self._hold(xk, out)
        return out

    def primal_with_gradient(self, xs, params: KernelParams, beta_bh: float):
        """DipoleTree::primal_with_gradient (bhtree.cpp:276-334) -> ((Q, C), (Q, C, 3))."""
        q = int(xs.shape[0])
        Cc = self.channels()
        xp, xk = _in(xs, np.float64, (q, 3))
        op, out = _out_like(xk, (q, Cc), np.float32)
        gp, grad = _out_like(xk, (q, Cc, 3), np.float32)
        check(lib().dpl_primal(self._h, C.byref(params), float(beta_bh), xp, q, op, gp, None))
        return out, grad

    # -- tiny-MLP radiance head (radiance.cpp:40-180) ---------------------------
    def set_mlp_head(self, sizes, w):
        """Render with the tiny-MLP head: sizes [22 + K, hidden..., 3], w the
        reference's flat fp64 weights. sizes=() restores the direct-rgb head."""
        sz = np.ascontiguousarray(sizes, dtype=np.int32)
        wv = np.ascontiguousarray(w, dtype=np.float64).ravel()
        self._head_nw = int(wv.size) if sz.size else 0
        check(lib().dpl_tree_set_mlp_head(self._h, sz.ctypes.data if sz.size else None,
                                          int(sz.size), wv.ctypes.data if wv.size else None,
                                          int(wv.size)))

    def head_grads(self):
        """RenderGrads::d_head_w since the last call (fp64); resets the accumulator."""
        out = np.zeros(self._head_nw)
        check(lib().dpl_head_grads(self._h, out.ctypes.data, out.size))
        return out

    # -- DPCK checkpoints (optimizer.cpp:294-388) --------------------------------
    def save_checkpoint(self, path, iter=0, lambda_scale=20.0, epsilon=0.0, background=(0, 0, 0),
                        beta_bh=2.0, initial_normals=None, head_variant=0, with_albedo=False,
                        mlp_sizes=(), mlp_w=()):
        """save_checkpoint (optimizer.cpp:330-356) of the tree's current cloud."""
        from ._lib import CheckpointMeta

        m = CheckpointMeta(int(iter), int(head_variant), int(bool(with_albedo)), 0,
                           float(lambda_scale), float(epsilon),
                           (C.c_double * 3)(*[float(b) for b in background]), float(beta_bh))
        ip = None
        if initial_normals is not None:
            inn = np.ascontiguousarray(initial_normals, dtype=np.float64).reshape(-1, 3)
            ip = inn.ctypes.data
        sz = np.ascontiguousarray(mlp_sizes, dtype=np.int32)
        wv = np.ascontiguousarray(mlp_w, dtype=np.float64)
        check(lib().dpl_checkpoint_save(self._h, str(path).encode(), C.byref(m), ip,
                                        sz.ctypes.data if sz.size else None, int(sz.size),
                                        wv.ctypes.data if wv.size else None, int(wv.size)))

    # -- query generators ----------------------------------------
    def sample_grid(self, params: KernelParams, beta_bh: float, resolution, lo=(0, 0, 0),
                    hi=(0, 0, 0), device=None):
        """sample_grid (meshing.cpp:33-59): geometry_field = 0.5 - primal_channel(x, 0)
        on a res0 x res1 x res2 grid. Returns (values (r2, r1, r0) fp32, lo, hi);
        lo == hi selects the cloud's bounding box padded by 5%."""
        res = np.ascontiguousarray(resolution, dtype=np.int32).reshape(3)
        lo_ = np.ascontiguousarray(lo, dtype=np.float64).reshape(3)
        hi_ = np.ascontiguousarray(hi, dtype=np.float64).reshape(3)
        shape = (int(res[2]), int(res[1]), int(res[0]))
        if device is not None:  # values stay on the GPU
            vals = torch.empty(shape, dtype=torch.float32, device=device)
            vp = vals.data_ptr()
        else:
            vals = np.empty(shape, np.float32)
            vp = vals.ctypes.data
        lo_o, hi_o = np.empty(3), np.empty(3)
        check(lib().dpl_sample_grid(self._h, C.byref(params), float(beta_bh), res.ctypes.data,
                                    lo_.ctypes.data, hi_.ctypes.data, vp,
                                    lo_o.ctypes.data, hi_o.ctypes.data))
        return vals, lo_o, hi_o

    def sample_rays(self, params: KernelParams, beta_bh: float, rays, sampler=None):
        """sample_ray (renderer.cpp:46-86) for a (R, 6) batch of rays (origin, dir).
        Returns (t (R, M), delta (R, M), count (R,), bracketed (R,)); row r holds
        count[r] ascending samples."""
        from ._lib import RaySampler

        cfg = sampler or RaySampler()
        rp, rk = _in(rays, np.float64)
        R = int(rays.shape[0])
        M = cfg.max_samples()
        # outputs live where the rays live (CUDA tensors in, CUDA tensors out)
        tp, t = _out_like(rk, (R, M), np.float64)
        dp, d = _out_like(rk, (R, M), np.float64)
        cp, cnt = _out_like(rk, (R,), np.int32)
        bp, br = _out_like(rk, (R,), np.uint8)
        check(lib().dpl_sample_rays(self._h, C.byref(params), float(beta_bh), rp, R, C.byref(cfg),
                                    M, tp, dp, cp, bp))
        return t, d, cnt, (br != 0)

    def primal_grad0(self, xs, params: KernelParams, beta_bh: float):
        """Values of all channels and the gradient of channel 0 only (render path)."""
        q = int(xs.shape[0])
        Cc = self.channels()
        xp, xk = _in(xs, np.float64, (q, 3))
        op, out = _out_like(xk, (q, Cc), np.float32)
        gp, grad = _out_like(xk, (q, 3), np.float32)
        check(lib().dpl_primal_grad0(self._h, C.byref(params), float(beta_bh), xp, q, op, gp))
        return out, grad

    # -- adjoint ------------------------------------------------------------------
    def make_buffer(self) -> GradientBuffer:
        return GradientBuffer(self)

    def adjoint(self, xs, params: KernelParams, beta_bh: float, d_out, d_grad, buf: GradientBuffer):
        """DipoleTree::adjoint (bhtree.cpp:345-417) for a (Q, 3) batch; d_out (Q, C),
        d_grad None or (Q, C, 3). xs=None reuses the batch of the immediately
        preceding primal() (its device copy: a host batch is uploaded once)."""
        q = int(xs.shape[0]) if xs is not None else int(d_out.shape[0])
        Cc = self.channels()
        xp, k1 = _in(xs, np.float64, (q, 3)) if xs is not None else (None, None)
        dp, k2 = _in(d_out, np.float32, (q, Cc))
        gp, k3 = _in(d_grad, np.float32, (q, Cc, 3)) if d_grad is not None else (None, None)
        check(lib().dpl_adjoint(self._h, C.byref(params), float(beta_bh), xp, q, dp, gp, buf._h))
        self._hold(k1, k2, k3)
        buf.dirty = True

    def flush_gradients(self, buffers, device_out=None, out=None) -> PointGradients:
        """DipoleTree::flush_gradients (bhtree.cpp:419-463); zeroes the buffers.
        device_out: a torch device to receive the outputs (else numpy);
        out: preallocated (moments N x C, normals N x 3) fp32 arrays/tensors."""
        if isinstance(buffers, GradientBuffer):
            buffers = [buffers]
        n, Cc = self.point_count(), self.channels()
        arr = (C.c_void_p * len(buffers))(*[b._h for b in buffers])
        if out is not None:
            mom, nrm = out
            mp = mom.data_ptr() if _is_torch(mom) else mom.ctypes.data
            np_ = nrm.data_ptr() if _is_torch(nrm) else nrm.ctypes.data
        elif device_out is not None:
            mom = torch.empty((n, Cc), dtype=torch.float32, device=device_out)
            nrm = torch.empty((n, 3), dtype=torch.float32, device=device_out)
            mp, np_ = mom.data_ptr(), nrm.data_ptr()
        else:
            mom = np.empty((n, Cc), np.float32)
            nrm = np.empty((n, 3), np.float32)
            mp, np_ = mom.ctypes.data, nrm.ctypes.data
        de = C.c_double()
        check(lib().dpl_flush(self._h, arr, len(buffers), mp, np_, C.byref(de)))
        if self._async:  # host outputs complete after synchronize()
            self._hold(mom, nrm)
        else:
            self._keep.clear()  # dpl_flush synchronizes every stream of the handle
        for b in buffers:
            b.dirty = False
        return PointGradients(Cc, mom, nrm, de.value)


    # -- flush split for the cross-rank sum (parallel.flush_allreduce) ------------
    def flush_begin(self, buffers) -> float:
        """Sum the buffers, node push-down; returns this rank's d_epsilon."""
        if isinstance(buffers, GradientBuffer):
            buffers = [buffers]
        arr = (C.c_void_p * len(buffers))(*[b._h for b in buffers])
        de = C.c_double()
        check(lib().dpl_flush_begin(self._h, arr, len(buffers), C.byref(de)))
        return de.value

    def flush_rows(self, buffer: GradientBuffer, lo: int, hi: int, rows):
        """Gradient rows [d moments | d normal] (C + 3 wide, fp32 CUDA tensor) of the
        sorted points [lo, hi), stream-ordered on the tree's stream."""
        check(lib().dpl_flush_rows(self._h, buffer._h, int(lo), int(hi), rows.data_ptr()))

    def flush_end(self, buffers, rows, out=None, device_out=None) -> tuple:
        """Rows N x (C + 3) in tree order -> (moments N x C, normals N x 3) in the
        original order; zeroes the buffers."""
        if isinstance(buffers, GradientBuffer):
            buffers = [buffers]
        n, Cc = self.point_count(), self.channels()
        arr = (C.c_void_p * len(buffers))(*[b._h for b in buffers])
        if out is not None:
            mom, nrm = out
            mp = mom.data_ptr() if _is_torch(mom) else mom.ctypes.data
            np_ = nrm.data_ptr() if _is_torch(nrm) else nrm.ctypes.data
        else:
            dev = device_out if device_out is not None else rows.device
            mom = torch.empty((n, Cc), dtype=torch.float32, device=dev)
            nrm = torch.empty((n, 3), dtype=torch.float32, device=dev)
            mp, np_ = mom.data_ptr(), nrm.data_ptr()
        check(lib().dpl_flush_end(self._h, arr, len(buffers), rows.data_ptr(), mp, np_))
        self._keep.clear()
        for b in buffers:
            b.dirty = False
        return mom, nrm


def launch_count() -> int:
    """Kernel launches issued through the engine in this process."""
    return int(lib().dpl_launch_count())


def mean_knn_spacing(positions, k: int = 8, device: int = 0) -> float:
    """OrientedPointCloud::mean_knn_spacing (pointcloud.cpp:51-65) on the GPU."""
    n = int(positions.shape[0])
    p, keep = _in(positions, np.float64, (n, 3))
    out = C.c_double()
    check(lib().dpl_mean_knn_spacing(int(device), p, n, int(k), C.byref(out)))
    return out.value


def default_epsilon(cloud: OrientedPointCloud, device: int = 0) -> float:
    """SceneModel::prepare's eps when unset: 1.5 x mean 8-NN spacing (fields.cpp:10-11)."""
    return 1.5 * mean_knn_spacing(cloud.positions, 8, device)


class PointAdam:
    """Trainer::step's point-parameter update (optimizer.cpp:161-205): Adam on
    geometry moments, appearance moments and normals, then update_moments."""

    def __init__(self, tree: DipoleTree, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8):
        h = C.c_void_p()
        check(lib().dpl_point_adam_create(tree._h, C.byref(h)))
        self._h = h.value
        self.tree = tree
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().dpl_point_adam_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def step(self, grads: PointGradients, lr=None):
        n, Cc = self.tree.point_count(), self.tree.channels()
        gm, k1 = _in(grads.moments, np.float32, (n, Cc))
        gn, k2 = _in(grads.normals, np.float32, (n, 3))
        check(lib().dpl_point_adam_step(self.tree._h, self._h, gm, gn,
                                        float(self.lr if lr is None else lr), self.beta1,
                                        self.beta2, self.eps))


    def step_range(self, g_moments, g_normals, lo: int, hi: int, lr=None):
        """Sharded update: Adam on points [lo, hi) with that slice's
        summed gradients ((hi - lo) x C, (hi - lo) x 3); no update_moments —
        exchange the slices (get_points_range / set_points_range), then
        refresh_moments. One Adam step per call."""
        k = hi - lo
        Cc = self.tree.channels()
        gm, k1 = _in(g_moments, np.float32, (k, Cc)) if k > 0 else (None, None)
        gn, k2 = _in(g_normals, np.float32, (k, 3)) if k > 0 else (None, None)
        check(lib().dpl_point_adam_step_range(self.tree._h, self._h, gm, gn, int(lo), int(hi),
                                              float(self.lr if lr is None else lr), self.beta1,
                                              self.beta2, self.eps))


def get_points_range(tree: DipoleTree, lo: int, hi: int, normals=None, moments=None):
    """Parameters of points [lo, hi) (original order, fp64) into the given arrays
    (host numpy or torch, any device) or new numpy arrays."""
    k, Cc = hi - lo, tree.channels()
    if normals is None:
        normals = np.zeros((k, 3))
    if moments is None:
        moments = np.zeros((k, Cc))
    pn = normals.data_ptr() if _is_torch(normals) else normals.ctypes.data
    pm = moments.data_ptr() if _is_torch(moments) else moments.ctypes.data
    check(lib().dpl_tree_get_points_range(tree._h, int(lo), int(hi), pn, pm))
    return normals, moments


def set_points_range(tree: DipoleTree, lo: int, hi: int, normals, moments):
    """Overwrite the parameters of points [lo, hi) (fp64, original order)."""
    k, Cc = hi - lo, tree.channels()
    pn, k1 = _in(normals, np.float64, (k, 3))
    pm, k2 = _in(moments, np.float64, (k, Cc))
    check(lib().dpl_tree_set_points_range(tree._h, int(lo), int(hi), pn, pm))


def refresh_moments(tree: DipoleTree):
    """update_moments (bhtree.cpp:171-176) from the tree's current parameters."""
    check(lib().dpl_tree_refresh_moments(tree._h))


def get_points(tree: DipoleTree):
    """(normals N x 3, moments N x C) fp64 of the tree's current cloud."""
    n, Cc = tree.point_count(), tree.channels()
    nrm = np.zeros((n, 3))
    mu = np.zeros((n, Cc))
    check(lib().dpl_tree_get_points(tree._h, nrm.ctypes.data, mu.ctypes.data))
    return nrm, mu


PHASES = ("sort", "forward", "adjoint", "flush", "render", "moments")


def profile_enable(tree: DipoleTree, on=True):
    check(lib().dpl_profile_enable(tree._h, int(on)))


def profile_read(tree: DipoleTree):
    """{phase: (total_ms, launches)} since the previous read (CUDA events)."""
    ms = (C.c_double * 6)()
    cnt = (C.c_int64 * 6)()
    check(lib().dpl_profile_read(tree._h, ms, cnt))
    return {p: (ms[i], cnt[i]) for i, p in enumerate(PHASES)}


def peak_fp32(device=0) -> float:
    v = C.c_double()
    check(lib().dpl_peak_fp32(int(device), C.byref(v)))
    return v.value


def peak_fp64(device=0) -> float:
    v = C.c_double()
    check(lib().dpl_peak_fp64(int(device), C.byref(v)))
    return v.value


def load_checkpoint(path):
    """load_checkpoint (optimizer.cpp:358-388): host arrays + scalars of a DPCK file."""
    from ._lib import CheckpointMeta

    m = CheckpointMeta()
    n, K, ns, nw = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int64()
    p = str(path).encode()
    check(lib().dpl_checkpoint_read(p, C.byref(m), C.byref(n), C.byref(K), C.byref(ns),
                                    C.byref(nw), None, None, None, None, None, None, None))
    N, Cc = n.value, K.value + 1
    pos, nrm, inn = (np.empty((N, 3)) for _ in range(3))
    area, mu = np.empty(N), np.empty((N, Cc))
    sizes, w = np.empty(ns.value, np.int32), np.empty(nw.value)
    check(lib().dpl_checkpoint_read(p, C.byref(m), C.byref(n), C.byref(K), C.byref(ns),
                                    C.byref(nw), pos.ctypes.data, nrm.ctypes.data,
                                    area.ctypes.data, mu.ctypes.data, inn.ctypes.data,
                                    sizes.ctypes.data, w.ctypes.data))
    return dict(iter=m.iter, cloud=OrientedPointCloud(pos, nrm, area, mu), initial_normals=inn,
                head_variant=m.head_variant, with_albedo=bool(m.with_albedo), mlp_sizes=sizes,
                mlp_w=w, lambda_scale=m.lambda_scale, epsilon=m.epsilon,
                background=np.array(m.background[:]), beta_bh=m.beta_bh)
