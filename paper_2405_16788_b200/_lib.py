"""ctypes binding of libdipole_b200.so (include/dipole_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``. There is no
fallback: if it is missing, importing the engine raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdipole_b200.so")

DPL_OK, DPL_ERR_USAGE, DPL_ERR_DATA, DPL_ERR_NUMERICAL, DPL_ERR_CUDA = range(5)
DPL_DIPOLE, DPL_RADIAL = 0, 1


class DataError(RuntimeError):
    """dipole::DataError (util.hpp:35): bad input — empty cloud, size mismatch."""


class NumericalError(RuntimeError):
    """dipole::NumericalError (util.hpp:38)."""


class UsageError(ValueError):
    pass


class CudaError(RuntimeError):
    pass


class KernelParams(C.Structure):
    """KernelParams (kernels.hpp:24-29) == dpl_kernel_params."""

    _fields_ = [("epsilon", C.c_double), ("desingularized", C.c_int32), ("reserved", C.c_int32),
                ("desing_delta", C.c_double), ("coincident_value", C.c_double)]

    def __init__(self, epsilon=0.0, desingularized=False, desing_delta=0.0, coincident_value=0.0):
        super().__init__(float(epsilon), int(bool(desingularized)), 0, float(desing_delta),
                         float(coincident_value))


class Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("visited", "far_near", "far_far", "pt_near", "pt_far")]


class RenderParams(C.Structure):
    _fields_ = [("lambda_scale", C.c_double), ("beta_bh", C.c_double),
                ("background", C.c_double * 3), ("t_near", C.c_double), ("t_far", C.c_double),
                ("seed", C.c_uint64)]


class RaySampler(C.Structure):
    """RenderConfig sampler fields (renderer.hpp:33-41) == dpl_ray_sampler."""

    _fields_ = [("t_near", C.c_double), ("t_far", C.c_double), ("probe_count", C.c_int32),
                ("sparse_before", C.c_int32), ("dense_at", C.c_int32),
                ("sparse_after", C.c_int32), ("uniform_count", C.c_int32),
                ("reserved", C.c_int32)]

    def __init__(self, t_near=0.05, t_far=6.0, probe_count=1024, sparse_before=24, dense_at=48,
                 sparse_after=8, uniform_count=80):
        super().__init__(float(t_near), float(t_far), int(probe_count), int(sparse_before),
                         int(dense_at), int(sparse_after), int(uniform_count), 0)

    def max_samples(self):
        return max(max(1, self.uniform_count),
                   self.sparse_before + max(1, self.dense_at) + self.sparse_after)


class CheckpointMeta(C.Structure):
    """dpl_checkpoint_meta: DPCK scalars (optimizer.cpp:330-356)."""

    _fields_ = [("iter", C.c_int32), ("head_variant", C.c_int32), ("with_albedo", C.c_int32),
                ("reserved", C.c_int32), ("lambda_scale", C.c_double), ("epsilon", C.c_double),
                ("background", C.c_double * 3), ("beta_bh", C.c_double)]


_lib = None

_vp = C.c_void_p
_sig = {
    "dpl_last_error": (C.c_char_p, []),
    "dpl_version": (C.c_int, []),
    "dpl_launch_count": (C.c_int64, []),
    "dpl_tree_create": (C.c_int, [C.c_int, _vp, C.POINTER(_vp)]),
    "dpl_tree_destroy": (C.c_int, [_vp]),
    "dpl_tree_set_stream": (C.c_int, [_vp, _vp]),
    "dpl_tree_sync": (C.c_int, [_vp]),
    "dpl_tree_set_host_async": (C.c_int, [_vp, C.c_int]),
    "dpl_tree_build": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32,
                                 C.c_int32]),
    "dpl_tree_update_moments": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int64, C.c_int32]),
    "dpl_tree_set_channel_kernels": (C.c_int, [_vp, _vp, C.c_int32]),
    "dpl_tree_channels": (C.c_int, [_vp, C.POINTER(C.c_int32)]),
    "dpl_tree_point_count": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "dpl_tree_node_count": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "dpl_tree_export": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "dpl_tree_export_moments": (C.c_int, [_vp, _vp, _vp]),
    "dpl_tree_dump": (C.c_int, [_vp, C.c_char_p]),
    "dpl_primal": (C.c_int, [_vp, C.POINTER(KernelParams), C.c_double, _vp, C.c_int64, _vp, _vp,
                             _vp]),
    "dpl_primal_channel": (C.c_int, [_vp, C.POINTER(KernelParams), C.c_double, _vp, C.c_int64,
                                     C.c_int32, _vp]),
    "dpl_primal_grad0": (C.c_int, [_vp, C.POINTER(KernelParams), C.c_double, _vp, C.c_int64,
                                   _vp, _vp]),
    "dpl_sample_grid": (C.c_int, [_vp, C.POINTER(KernelParams), C.c_double, _vp, _vp, _vp, _vp,
                                  _vp, _vp]),
    "dpl_sample_rays": (C.c_int, [_vp, C.POINTER(KernelParams), C.c_double, _vp, C.c_int64,
                                  C.POINTER(RaySampler), C.c_int32, _vp, _vp, _vp, _vp]),
    "dpl_checkpoint_save": (C.c_int, [_vp, C.c_char_p, C.POINTER(CheckpointMeta), _vp, _vp,
                                      C.c_int32, _vp, C.c_int64]),
    "dpl_checkpoint_read": (C.c_int, [C.c_char_p, C.POINTER(CheckpointMeta), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int64), _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dpl_tree_set_mlp_head": (C.c_int, [_vp, _vp, C.c_int32, _vp, C.c_int64]),
    "dpl_head_grads": (C.c_int, [_vp, _vp, C.c_int64]),
    "dpl_gradbuf_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "dpl_gradbuf_destroy": (C.c_int, [_vp]),
    "dpl_gradbuf_zero": (C.c_int, [_vp]),
    "dpl_gradbuf_export": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "dpl_adjoint": (C.c_int, [_vp, C.POINTER(KernelParams), C.c_double, _vp, C.c_int64, _vp, _vp,
                              _vp]),
    "dpl_flush": (C.c_int, [_vp, C.POINTER(_vp), C.c_int32, _vp, _vp, C.POINTER(C.c_double)]),
    "dpl_tree_prefetch": (C.c_int, [_vp, _vp, C.c_int64]),
    "dpl_flush_begin": (C.c_int, [_vp, C.POINTER(_vp), C.c_int32, C.POINTER(C.c_double)]),
    "dpl_flush_rows": (C.c_int, [_vp, _vp, C.c_int64, C.c_int64, _vp]),
    "dpl_flush_end": (C.c_int, [_vp, C.POINTER(_vp), C.c_int32, _vp, _vp, _vp]),
    "dpl_tape_create": (C.c_int, [C.POINTER(_vp)]),
    "dpl_tape_destroy": (C.c_int, [_vp]),
    "dpl_render_forward": (C.c_int, [_vp, C.POINTER(KernelParams), C.POINTER(RenderParams), _vp,
                                     C.c_int64, C.c_int32, _vp, _vp, _vp, _vp]),
    "dpl_render_backward": (C.c_int, [_vp, C.POINTER(KernelParams), C.POINTER(RenderParams), _vp,
                                      _vp, _vp, C.POINTER(C.c_double), _vp]),
    "dpl_uniform": (C.c_double, [C.c_uint64, C.c_uint64]),
    "dpl_gemm_f32": (C.c_int, [C.c_int, _vp, C.c_int32, C.c_int32, C.c_int32, _vp, C.c_int64,
                               C.c_int32, _vp, C.c_int64, C.c_int32, _vp, C.c_int64, C.c_int32]),
    "dpl_guard_check": (C.c_int, [C.POINTER(C.c_int64)]),
    "dpl_guard_selftest": (C.c_int, []),
    "dpl_profile_enable": (C.c_int, [_vp, C.c_int]),
    "dpl_profile_read": (C.c_int, [_vp, _vp, _vp]),
    "dpl_peak_fp32": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "dpl_peak_fp64": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "dpl_mean_knn_spacing": (C.c_int, [C.c_int, _vp, C.c_int64, C.c_int32,
                                       C.POINTER(C.c_double)]),
    "dpl_point_adam_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "dpl_point_adam_destroy": (C.c_int, [_vp]),
    "dpl_point_adam_step": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, C.c_double, C.c_double,
                                      C.c_double]),
    "dpl_tree_get_points": (C.c_int, [_vp, _vp, _vp]),
    "dpl_point_adam_step_range": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_int64, C.c_double,
                                            C.c_double, C.c_double, C.c_double]),
    "dpl_tree_get_points_range": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, _vp]),
    "dpl_tree_set_points_range": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, _vp]),
    "dpl_tree_refresh_moments": (C.c_int, [_vp]),
    "dpl_adam_step": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_int64, C.c_double, C.c_double,
                                C.c_double, C.c_double, C.c_int64]),
}

EXPORTED_SYMBOLS = tuple(_sig)


def lib():
    """Load the CUDA engine; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a engine with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
        lb = C.CDLL(LIB_PATH)
        for name, (res, args) in _sig.items():
            f = getattr(lb, name)
            f.restype = res
            f.argtypes = args
        _lib = lb
    return _lib


def check(rc):
    if rc == DPL_OK:
        return
    msg = lib().dpl_last_error().decode(errors="replace")
    if rc == DPL_ERR_DATA:
        raise DataError(msg)
    if rc == DPL_ERR_NUMERICAL:
        raise NumericalError(msg)
    if rc == DPL_ERR_CUDA:
        raise CudaError(msg)
    raise UsageError(msg)
