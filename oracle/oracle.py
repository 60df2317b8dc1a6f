"""ctypes bindings for the CPU oracle — TEST INFRASTRUCTURE ONLY.

Two back-ends with one Python surface:
  * ``port``: ``oracle/liboracle.so``, the plain-C restatement
    (``oracle/dipole_oracle.c``) of the reference hot path;
  * ``ref``:  ``oracle/_ref/libdipole_ref.so``, the reference's own sources
    (/root/reference/proj/src) compiled unmodified plus ``ref_driver.cpp``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this module, and only as the checker / the timed CPU baseline. The
product library never calls it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libdipole_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_up = C.POINTER(C.c_uint8)


class Params(C.Structure):
    """KernelParams (kernels.hpp:24-29) / dpl_kernel_params."""

    _fields_ = [
        ("epsilon", C.c_double),
        ("desingularized", C.c_int32),
        ("reserved", C.c_int32),
        ("desing_delta", C.c_double),
        ("coincident_value", C.c_double),
    ]

    def __init__(self, epsilon=0.0, desingularized=False, desing_delta=0.0, coincident_value=0.0):
        super().__init__(float(epsilon), int(bool(desingularized)), 0, float(desing_delta),
                         float(coincident_value))


class Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("visited", "far_near", "far_far", "pt_near", "pt_far")]


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


_port = None
_ref = None


def have_port():
    return os.path.exists(PORT_PATH)


def have_ref():
    return os.path.exists(REF_PATH)


def port_lib():
    global _port
    if _port is None:
        lib = C.CDLL(PORT_PATH)
        lib.ora_tree_build.restype = C.c_void_p
        lib.ora_tree_build.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_int32, C.c_int32, C.c_int32]
        lib.ora_tree_free.argtypes = [C.c_void_p]
        lib.ora_tree_update_moments.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, C.c_int64, C.c_int32]
        lib.ora_tree_set_kinds.argtypes = [C.c_void_p, _up, C.c_int32]
        lib.ora_tree_node_count.restype = C.c_int64
        lib.ora_tree_node_count.argtypes = [C.c_void_p]
        lib.ora_tree_export.argtypes = [C.c_void_p, _dp, _ip, _ip, _ip]
        lib.ora_tree_export_moments.argtypes = [C.c_void_p, _dp, _dp]
        lib.ora_primal.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, _dp, C.c_int64,
                                   C.c_int, C.c_int, _dp, _dp, C.POINTER(Counters), C.c_int]
        lib.ora_adjoint.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, _dp, C.c_int64,
                                    _dp, _dp, C.c_int, _dp, _dp, _dp]
        lib.ora_primal_ex.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, _dp, C.c_int64,
                                      C.c_int, C.c_int, _dp, _dp, C.c_void_p, C.c_int, _dp, _dp]
        lib.ora_adjoint_ex.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, _dp, C.c_int64,
                                       _dp, _dp, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.ora_render_step_ex.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, C.c_double,
                                           _dp, _dp, C.c_int64, C.c_int32, _dp, _dp, _dp,
                                           C.c_double, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp,
                                           _dp, _dp, _dp]
        lib.ora_naive_sum.argtypes = [C.c_void_p, C.POINTER(Params), _dp, C.c_int64, C.c_int,
                                      C.c_int, _dp, _dp]
        lib.ora_naive_adjoint.argtypes = [C.c_void_p, C.POINTER(Params), _dp, C.c_int64, _dp, _dp,
                                          _dp, _dp, _dp]
        lib.ora_kernel_coeffs.argtypes = [C.c_double, C.POINTER(Params), C.c_int, _dp]
        lib.ora_erf.restype = C.c_double
        lib.ora_erf.argtypes = [C.c_double]
        lib.ora_tau.restype = C.c_double
        lib.ora_tau.argtypes = [C.c_double]
        lib.ora_normal_hazard.restype = C.c_double
        lib.ora_normal_hazard.argtypes = [C.c_double]
        lib.ora_uniform.restype = C.c_double
        lib.ora_uniform.argtypes = [C.c_uint64, C.c_uint64]
        lib.ora_stratified_samples.argtypes = [C.c_int64, C.c_int32, C.c_double, C.c_double,
                                               C.c_uint64, C.c_int64, _dp, _dp]
        lib.ora_render_step.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, C.c_double, _dp,
                                        _dp, C.c_int64, C.c_int32, _dp, _dp, _dp, C.c_double,
                                        C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.ora_mean_knn_spacing.restype = C.c_double
        lib.ora_mean_knn_spacing.argtypes = [_dp, C.c_int64, C.c_int]
        lib.ora_adam_step.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_double, C.c_double,
                                      C.c_double, C.c_double, C.c_int64]
        lib.ora_sample_grid.restype = C.c_int
        lib.ora_sample_grid.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, _ip, _dp, _dp,
                                        _dp, C.c_int64, C.c_int, _dp, _dp, _dp]
        lib.ora_sample_rays.argtypes = [C.c_void_p, C.POINTER(Params), C.c_double, _dp, C.c_int64,
                                        C.c_double, C.c_double, _ip, C.c_int32, C.c_int, _dp, _dp,
                                        _ip, _up]
        _port = lib
    return _port


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_PATH)
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_hardware_concurrency.restype = C.c_int
        lib.ref_kernel_coeffs.argtypes = [C.c_double, C.POINTER(Params), C.c_int, _dp]
        lib.ref_tau.restype = C.c_double
        lib.ref_tau.argtypes = [C.c_double]
        lib.ref_erf_approx.restype = C.c_double
        lib.ref_erf_approx.argtypes = [C.c_double]
        lib.ref_normal_hazard.restype = C.c_double
        lib.ref_normal_hazard.argtypes = [C.c_double]
        lib.ref_model_save_checkpoint.argtypes = [vp, C.c_int32, C.c_char_p]
        lib.ref_model_set_mlp_head.argtypes = [vp, _ip, C.c_int32, _dp, C.c_int64]
        lib.ref_model_head_grads.argtypes = [vp, _dp]
        lib.ref_sample_grid.argtypes = [vp, _ip, _dp, _dp, C.c_int, _dp, _dp, _dp]
        lib.ref_sample_rays.argtypes = [vp, _dp, C.c_int64, C.c_double, C.c_double, _ip, C.c_int32,
                                        _dp, _dp, _ip, _up]
        lib.ref_mean_knn_spacing.restype = C.c_double
        lib.ref_mean_knn_spacing.argtypes = [_dp, C.c_int64, C.c_int]
        lib.ref_tree_build.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_int32, C.c_int32,
                                       C.c_int32, C.POINTER(vp)]
        lib.ref_tree_free.argtypes = [vp]
        lib.ref_tree_set_kinds.argtypes = [vp, _up, C.c_int32]
        lib.ref_tree_update_moments.argtypes = [vp, _dp, _dp, _dp, _dp, C.c_int64, C.c_int32]
        lib.ref_tree_node_count.restype = C.c_int64
        lib.ref_tree_node_count.argtypes = [vp]
        lib.ref_tree_export.argtypes = [vp, _dp, _ip, _ip]
        lib.ref_tree_dump.argtypes = [vp, C.c_char_p]
        lib.ref_primal.argtypes = [vp, C.POINTER(Params), C.c_double, _dp, C.c_int64, C.c_int,
                                   C.c_int, _dp, _dp, _lp, C.c_int]
        lib.ref_adjoint.argtypes = [vp, C.POINTER(Params), C.c_double, _dp, C.c_int64, _dp, _dp,
                                    C.c_int, _dp, _dp, _dp]
        lib.ref_bufs_create.argtypes = [vp, C.c_int, C.POINTER(vp)]
        lib.ref_bufs_free.argtypes = [vp]
        lib.ref_adjoint_into.argtypes = [vp, C.POINTER(Params), C.c_double, _dp, C.c_int64, _dp,
                                         vp]
        lib.ref_bufs_flush.argtypes = [vp, vp, _dp, _dp, _dp]
        lib.ref_naive_sum.argtypes = [vp, C.POINTER(Params), _dp, C.c_int64, C.c_int, C.c_int,
                                      C.c_int, _dp, _dp, C.c_int]
        lib.ref_naive_adjoint.argtypes = [vp, C.POINTER(Params), _dp, C.c_int64, _dp, _dp, _up,
                                          _dp, _dp, _dp]
        lib.ref_model_create.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.c_int32, C.c_double,
                                         C.c_double, C.c_double, _dp, C.POINTER(vp)]
        lib.ref_model_free.argtypes = [vp]
        lib.ref_model_epsilon.restype = C.c_double
        lib.ref_model_epsilon.argtypes = [vp]
        lib.ref_render_step.argtypes = [vp, _dp, _dp, _dp, C.c_int64, C.c_int32, _dp, C.c_double,
                                        C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.ref_adam_create.restype = vp
        lib.ref_adam_free.argtypes = [vp]
        lib.ref_adam_step.argtypes = [vp, _dp, _dp, C.c_int64, C.c_double]
        _ref = lib
    return _ref


def _check_ref(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {ref_lib().ref_last_error().decode()}")


@dataclass
class Cloud:
    pos: np.ndarray   # N x 3 f64
    nrm: np.ndarray   # N x 3 f64
    area: np.ndarray  # N f64
    mu: np.ndarray    # N x C f64

    @property
    def n(self):
        return self.pos.shape[0]

    @property
    def C(self):
        return self.mu.shape[1]

    def as_f64(self):
        return Cloud(_d(self.pos).reshape(-1, 3), _d(self.nrm).reshape(-1, 3), _d(self.area).ravel(),
                     _d(self.mu).reshape(self.pos.shape[0], -1))


class OracleTree:
    """DipoleTree (bhtree.hpp:51-130) evaluated on the CPU by `backend`."""

    def __init__(self, cloud: Cloud, max_leaf=8, max_depth=20, backend="port"):
        self.backend = backend
        c = cloud.as_f64()
        self.cloud = c
        self.C = c.C
        self.n = c.n
        if backend == "port":
            self._lib = port_lib()
            self._h = self._lib.ora_tree_build(_ptr(c.pos), _ptr(c.nrm), _ptr(c.area), _ptr(c.mu),
                                               c.n, c.C, max_leaf, max_depth)
            if not self._h:
                raise ValueError("DataError: empty cloud")
        else:
            self._lib = ref_lib()
            h = C.c_void_p()
            _check_ref(self._lib.ref_tree_build(_ptr(c.pos), _ptr(c.nrm), _ptr(c.area), _ptr(c.mu),
                                                c.n, c.C, max_leaf, max_depth, C.byref(h)))
            self._h = h.value
        self.kinds = np.zeros(self.C, np.uint8)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            (self._lib.ora_tree_free if self.backend == "port" else self._lib.ref_tree_free)(h)
            self._h = None

    # -- structure -----------------------------------------------------------
    def set_kinds(self, kinds):
        k = np.ascontiguousarray(kinds, dtype=np.uint8)
        self.kinds = k.copy()
        f = self._lib.ora_tree_set_kinds if self.backend == "port" else self._lib.ref_tree_set_kinds
        rc = f(self._h, _ptr(k, _up), len(k))
        if rc:
            raise ValueError("DataError: channel count mismatch")

    def update_moments(self, cloud: Cloud):
        c = cloud.as_f64()
        f = (self._lib.ora_tree_update_moments if self.backend == "port"
             else self._lib.ref_tree_update_moments)
        rc = f(self._h, _ptr(c.pos), _ptr(c.nrm), _ptr(c.area), _ptr(c.mu), c.n, c.C)
        if rc:
            raise ValueError("DataError: cloud/tree size mismatch")
        self.cloud = c

    def sample_grid(self, params, beta, res, lo=(0, 0, 0), hi=(0, 0, 0), threads=0):
        """sample_grid (meshing.cpp:33-59), port backend: (values r2 x r1 x r0, lo, hi)."""
        assert self.backend == "port"
        res = np.ascontiguousarray(res, dtype=np.int32)
        vals = np.zeros((int(res[2]), int(res[1]), int(res[0])))
        lo_o, hi_o = np.zeros(3), np.zeros(3)
        rc = self._lib.ora_sample_grid(self._h, C.byref(params), beta, _ptr(res, _ip),
                                       _ptr(_d(lo)), _ptr(_d(hi)), _ptr(self.cloud.pos), self.n,
                                       threads, _ptr(vals), _ptr(lo_o), _ptr(hi_o))
        if rc:
            raise ValueError("DataError: sample_grid resolution")
        return vals, lo_o, hi_o

    def sample_rays(self, params, beta, rays, t_near, t_far, counts5, max_s, threads=0):
        """sample_ray (renderer.cpp:46-86), port backend."""
        assert self.backend == "port"
        rays = _d(rays).reshape(-1, 6)
        R = rays.shape[0]
        k = np.ascontiguousarray(counts5, dtype=np.int32)
        t, d = np.zeros((R, max_s)), np.zeros((R, max_s))
        cnt, br = np.zeros(R, np.int32), np.zeros(R, np.uint8)
        self._lib.ora_sample_rays(self._h, C.byref(params), beta, _ptr(rays), R, t_near, t_far,
                                  _ptr(k, _ip), max_s, threads, _ptr(t), _ptr(d), _ptr(cnt, _ip),
                                  _ptr(br, _up))
        return t, d, cnt, br.astype(bool)

    def node_count(self):
        f = self._lib.ora_tree_node_count if self.backend == "port" else self._lib.ref_tree_node_count
        return int(f(self._h))

    def export(self):
        nn = self.node_count()
        geo = np.zeros((nn, 5))
        topo = np.zeros((nn, 6), np.int32)
        order = np.zeros(self.n, np.int32)
        if self.backend == "port":
            leaf_of = np.zeros(self.n, np.int32)
            self._lib.ora_tree_export(self._h, _ptr(geo), _ptr(topo, _ip), _ptr(order, _ip),
                                      _ptr(leaf_of, _ip))
        else:
            self._lib.ref_tree_export(self._h, _ptr(geo), _ptr(topo, _ip), _ptr(order, _ip))
            leaf_of = np.full(self.n, -1, np.int32)
            for i in np.nonzero(topo[:, 5])[0]:
                leaf_of[order[topo[i, 0]:topo[i, 1]]] = i
        return dict(geo=geo, topo=topo, order=order, leaf_of=leaf_of)

    def export_moments(self):
        assert self.backend == "port"
        nn = self.node_count()
        mv = np.zeros((nn, self.C, 3))
        ms = np.zeros((nn, self.C))
        self._lib.ora_tree_export_moments(self._h, _ptr(mv), _ptr(ms))
        return mv, ms

    def dump(self, path):
        assert self.backend == "ref"
        _check_ref(self._lib.ref_tree_dump(self._h, path.encode()))

    # -- queries -------------------------------------------------------------
    def primal(self, params: Params, beta, xs, mode="values", channel=0, counters=False,
               threads=None):
        xs = _d(xs).reshape(-1, 3)
        q = xs.shape[0]
        threads = threads or os.cpu_count() or 1
        m = {"values": 0, "grad": 1, "channel": 2}[mode]
        out = np.zeros(q if m == 2 else (q, self.C))
        grad = np.zeros((q, self.C, 3)) if m == 1 else None
        if self.backend == "port":
            cnt = (Counters * q)() if counters else None
            self._lib.ora_primal(self._h, C.byref(params), beta, _ptr(xs), q, m, channel,
                                 _ptr(out), _ptr(grad), cnt, threads)
            cres = (np.frombuffer(cnt, dtype=np.int64).reshape(q, 5).copy() if counters else None)
        else:
            vis = np.zeros(q, np.int64) if counters else None
            _check_ref(self._lib.ref_primal(self._h, C.byref(params), beta, _ptr(xs), q, m,
                                            channel, _ptr(out), _ptr(grad), _ptr(vis, _lp), threads))
            cres = vis
        res = [out]
        if m == 1:
            res.append(grad)
        if counters:
            res.append(cres)
        return res[0] if len(res) == 1 else tuple(res)

    def adjoint(self, params: Params, beta, xs, d_out, d_grad=None, threads=None):
        xs = _d(xs).reshape(-1, 3)
        q = xs.shape[0]
        threads = threads or os.cpu_count() or 1
        d_out = _d(d_out).reshape(q, self.C)
        d_grad = None if d_grad is None else _d(d_grad).reshape(q, self.C, 3)
        mom = np.zeros((self.n, self.C))
        nrm = np.zeros((self.n, 3))
        de = C.c_double()
        if self.backend == "port":
            self._lib.ora_adjoint(self._h, C.byref(params), beta, _ptr(xs), q, _ptr(d_out),
                                  _ptr(d_grad), threads, _ptr(mom), _ptr(nrm), C.byref(de))
        else:
            _check_ref(self._lib.ref_adjoint(self._h, C.byref(params), beta, _ptr(xs), q,
                                             _ptr(d_out), _ptr(d_grad), threads, _ptr(mom),
                                             _ptr(nrm), C.byref(de)))
        return mom, nrm, de.value

    def primal_mag(self, params: Params, beta, xs, mode="values", channel=0, threads=None):
        """Port only: primal() plus the sum of |terms| of every output (dict:
        out, out_abs, and grad / grad_abs for mode "grad")."""
        assert self.backend == "port"
        xs = _d(xs).reshape(-1, 3)
        q = xs.shape[0]
        threads = threads or os.cpu_count() or 1
        m = {"values": 0, "grad": 1, "channel": 2}[mode]
        shape = q if m == 2 else (q, self.C)
        out, out_a = np.zeros(shape), np.zeros(shape)
        grad = np.zeros((q, self.C, 3)) if m == 1 else None
        grad_a = np.zeros((q, self.C, 3)) if m == 1 else None
        self._lib.ora_primal_ex(self._h, C.byref(params), beta, _ptr(xs), q, m, channel, _ptr(out),
                                _ptr(grad), None, threads, _ptr(out_a), _ptr(grad_a))
        res = dict(out=out, out_abs=out_a)
        if m == 1:
            res.update(grad=grad, grad_abs=grad_a)
        return res

    def adjoint_mag(self, params: Params, beta, xs, d_out, d_grad=None, threads=None):
        """Port only: adjoint() plus, per flushed output, a bound on the sum of
        |terms| it accumulated (dict: moments, normals, d_eps and *_abs)."""
        assert self.backend == "port"
        xs = _d(xs).reshape(-1, 3)
        q = xs.shape[0]
        threads = threads or os.cpu_count() or 1
        d_out = _d(d_out).reshape(q, self.C)
        d_grad = None if d_grad is None else _d(d_grad).reshape(q, self.C, 3)
        mom, mom_a = np.zeros((self.n, self.C)), np.zeros((self.n, self.C))
        nrm, nrm_a = np.zeros((self.n, 3)), np.zeros((self.n, 3))
        de, de_a = C.c_double(), C.c_double()
        self._lib.ora_adjoint_ex(self._h, C.byref(params), beta, _ptr(xs), q, _ptr(d_out),
                                 _ptr(d_grad), threads, _ptr(mom), _ptr(nrm), C.byref(de),
                                 _ptr(mom_a), _ptr(nrm_a), C.byref(de_a))
        return dict(moments=mom, normals=nrm, d_eps=de.value, moments_abs=mom_a,
                    normals_abs=nrm_a, d_eps_abs=de_a.value)

    def gradient_buffers(self, workers):
        """Reference backend only: `workers` caller-held GradientBuffers
        (make_buffer), filled by RefBuffers.adjoint and flushed by RefBuffers.flush."""
        assert self.backend == "ref"
        return RefBuffers(self, workers)

    def naive_sum(self, params: Params, xs, channel, kind, with_grad=False):
        xs = _d(xs).reshape(-1, 3)
        q = xs.shape[0]
        out = np.zeros(q)
        grad = np.zeros((q, 3)) if with_grad else None
        if self.backend == "port":
            self._lib.ora_naive_sum(self._h, C.byref(params), _ptr(xs), q, channel, kind,
                                    _ptr(out), _ptr(grad))
        else:
            _check_ref(self._lib.ref_naive_sum(self._h, C.byref(params), _ptr(xs), q, channel,
                                               kind, int(with_grad), _ptr(out), _ptr(grad), 0))
        return (out, grad) if with_grad else out

    def naive_adjoint(self, params: Params, xs, d_out, d_grad=None):
        xs = _d(xs).reshape(-1, 3)
        q = xs.shape[0]
        d_out = _d(d_out).reshape(q, self.C)
        d_grad = None if d_grad is None else _d(d_grad).reshape(q, self.C, 3)
        mom = np.zeros((self.n, self.C))
        nrm = np.zeros((self.n, 3))
        de = C.c_double()
        if self.backend == "port":
            self._lib.ora_naive_adjoint(self._h, C.byref(params), _ptr(xs), q, _ptr(d_out),
                                        _ptr(d_grad), _ptr(mom), _ptr(nrm), C.byref(de))
        else:
            _check_ref(self._lib.ref_naive_adjoint(self._h, C.byref(params), _ptr(xs), q,
                                                   _ptr(d_out), _ptr(d_grad), _ptr(self.kinds, _up),
                                                   _ptr(mom), _ptr(nrm), C.byref(de)))
        return mom, nrm, de.value

    def render_step(self, params: Params, beta, lam, background, rays, ts, deltas, target, scale,
                    threads=None, mag=False):
        """render_ray + render_ray_backward (renderer.cpp:106-231), direct-rgb head,
        channel 0 Dipole / 1..C-1 Radial (SceneModel::prepare)."""
        assert self.backend == "port", "use RefModel for the reference render step"
        rays = _d(rays).reshape(-1, 6)
        R = rays.shape[0]
        S = ts.shape[1]
        threads = threads or os.cpu_count() or 1
        rgb = np.zeros((R, 3))
        mom = np.zeros((self.n, self.C))
        nrm = np.zeros((self.n, 3))
        de, dl = C.c_double(), C.c_double()
        dbg = np.zeros(3)
        bg = _d(background)
        mom_a = np.zeros((self.n, self.C)) if mag else None
        nrm_a = np.zeros((self.n, 3)) if mag else None
        de_a = C.c_double()
        self._lib.ora_render_step_ex(self._h, C.byref(params), beta, lam, _ptr(bg), _ptr(rays), R,
                                     S, _ptr(_d(ts)), _ptr(_d(deltas)), _ptr(_d(target)), scale,
                                     threads, _ptr(rgb), _ptr(mom), _ptr(nrm), C.byref(de),
                                     C.byref(dl), _ptr(dbg), _ptr(mom_a), _ptr(nrm_a),
                                     C.byref(de_a) if mag else None)
        res = dict(rgb=rgb, moments=mom, normals=nrm, d_eps=de.value, d_lambda=dl.value, d_bg=dbg)
        if mag:
            res.update(moments_abs=mom_a, normals_abs=nrm_a, d_eps_abs=de_a.value)
        return res


class RefBuffers:
    """One GradientBuffer per worker on a reference tree (bhtree.hpp:38-40)."""

    def __init__(self, tree: "OracleTree", workers):
        self.tree = tree
        self.workers = int(workers)
        h = C.c_void_p()
        _check_ref(tree._lib.ref_bufs_create(tree._h, self.workers, C.byref(h)))
        self._h = h.value

    def __del__(self):
        if getattr(self, "_h", None):
            self.tree._lib.ref_bufs_free(self._h)
            self._h = None

    def adjoint(self, params: Params, beta, xs, d_out):
        xs = _d(xs).reshape(-1, 3)
        q = xs.shape[0]
        d_out = _d(d_out).reshape(q, self.tree.C)
        _check_ref(self.tree._lib.ref_adjoint_into(self.tree._h, C.byref(params), beta, _ptr(xs), q,
                                                   _ptr(d_out), self._h))

    def flush(self, want=True):
        mom = np.zeros((self.tree.n, self.tree.C)) if want else None
        nrm = np.zeros((self.tree.n, 3)) if want else None
        de = C.c_double()
        _check_ref(self.tree._lib.ref_bufs_flush(self.tree._h, self._h, _ptr(mom), _ptr(nrm),
                                                 C.byref(de)))
        return mom, nrm, de.value


class RefModel:
    """SceneModel prepared by the reference (fields.cpp:7-18) for the render step."""

    def __init__(self, cloud: Cloud, epsilon, lam=20.0, beta=2.0, background=(0, 0, 0)):
        c = cloud.as_f64()
        self.n, self.C = c.n, c.C
        self._lib = ref_lib()
        h = C.c_void_p()
        _check_ref(self._lib.ref_model_create(_ptr(c.pos), _ptr(c.nrm), _ptr(c.area), _ptr(c.mu),
                                              c.n, c.C, epsilon, lam, beta,
                                              _ptr(_d(background)), C.byref(h)))
        self._h = h.value

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.ref_model_free(self._h)
            self._h = None

    def set_mlp_head(self, sizes, w):
        """Tiny-MLP radiance head (radiance.cpp:40-180) with the given weights."""
        sz = np.ascontiguousarray(sizes, dtype=np.int32)
        self._w = _d(w).ravel()
        _check_ref(self._lib.ref_model_set_mlp_head(self._h, _ptr(sz, _ip), len(sz),
                                                    _ptr(self._w), len(self._w)))

    def head_grads(self):
        """d_head_w accumulated by the last render_step (RenderGrads::d_head_w)."""
        out = np.zeros(len(self._w))
        _check_ref(self._lib.ref_model_head_grads(self._h, _ptr(out)))
        return out

    def save_checkpoint(self, path, iter=0):
        """The reference's own save_checkpoint (optimizer.cpp:330-356)."""
        _check_ref(self._lib.ref_model_save_checkpoint(self._h, iter, str(path).encode()))

    def sample_grid(self, res, lo=(0, 0, 0), hi=(0, 0, 0), threads=0):
        """The reference's own sample_grid (meshing.cpp:33-59) on this model."""
        res = np.ascontiguousarray(res, dtype=np.int32)
        vals = np.zeros((int(res[2]), int(res[1]), int(res[0])))
        lo_o, hi_o = np.zeros(3), np.zeros(3)
        _check_ref(self._lib.ref_sample_grid(self._h, _ptr(res, _ip), _ptr(_d(lo)), _ptr(_d(hi)),
                                             threads, _ptr(vals), _ptr(lo_o), _ptr(hi_o)))
        return vals, lo_o, hi_o

    def sample_rays(self, rays, t_near, t_far, counts5, max_s):
        """The reference's own sample_ray (renderer.cpp:46-86) per ray."""
        rays = _d(rays).reshape(-1, 6)
        R = rays.shape[0]
        k = np.ascontiguousarray(counts5, dtype=np.int32)
        t, d = np.zeros((R, max_s)), np.zeros((R, max_s))
        cnt, br = np.zeros(R, np.int32), np.zeros(R, np.uint8)
        _check_ref(self._lib.ref_sample_rays(self._h, _ptr(rays), R, t_near, t_far, _ptr(k, _ip),
                                             max_s, _ptr(t), _ptr(d), _ptr(cnt, _ip),
                                             _ptr(br, _up)))
        return t, d, cnt, br.astype(bool)

    def render_step(self, rays, ts, deltas, target, scale, threads=None):
        rays = _d(rays).reshape(-1, 6)
        R = rays.shape[0]
        S = ts.shape[1]
        rgb = np.zeros((R, 3))
        mom = np.zeros((self.n, self.C))
        nrm = np.zeros((self.n, 3))
        de, dl = C.c_double(), C.c_double()
        dbg = np.zeros(3)
        _check_ref(self._lib.ref_render_step(self._h, _ptr(rays), _ptr(_d(ts)), _ptr(_d(deltas)),
                                             R, S, _ptr(_d(target)), scale, threads or 0,
                                             _ptr(rgb), _ptr(mom), _ptr(nrm), C.byref(de),
                                             C.byref(dl), _ptr(dbg)))
        return dict(rgb=rgb, moments=mom, normals=nrm, d_eps=de.value, d_lambda=dl.value, d_bg=dbg)


def stratified_samples(R, S, t_near, t_far, seed, ray_offset=0):
    ts = np.zeros((R, S))
    dl = np.zeros((R, S))
    port_lib().ora_stratified_samples(R, S, t_near, t_far, seed, ray_offset, _ptr(ts), _ptr(dl))
    return ts, dl


def mean_knn_spacing(pos, k=8, backend="port"):
    p = _d(pos).reshape(-1, 3)
    if backend == "port":
        return port_lib().ora_mean_knn_spacing(_ptr(p), p.shape[0], k)
    return ref_lib().ref_mean_knn_spacing(_ptr(p), p.shape[0], k)


def kernel_coeffs(r, params: Params, order=2, backend="port"):
    out = np.zeros(7)
    if backend == "port":
        port_lib().ora_kernel_coeffs(r, C.byref(params), order, _ptr(out))
    else:
        _check_ref(ref_lib().ref_kernel_coeffs(r, C.byref(params), order, _ptr(out)))
    return out
