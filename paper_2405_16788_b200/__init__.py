"""B200-native Barnes-Hut regularized dipole sums (arXiv 2405.16788 hot path).

The engine is libdipole_b200.so (sm_100a CUDA + C-ABI, include/dipole_b200.h);
this package is its host-side mirror of the reference API:
  * bhtree.DipoleTree      — dipole::DipoleTree (bhtree.hpp:51-130), batched
  * renderer.render_*      — render_ray / render_ray_backward (renderer.cpp:106-231)
  * workloads              — seeded synthetic inputs for BASELINE.json configs
"""
from ._lib import (DataError, KernelParams, NumericalError, UsageError, CudaError,  # noqa: F401
                   DPL_DIPOLE, DPL_RADIAL, RaySampler)
from .bhtree import (DipoleTree, GradientBuffer, OrientedPointCloud, PointGradients,  # noqa: F401
                     launch_count)

__all__ = ["DipoleTree", "GradientBuffer", "OrientedPointCloud", "PointGradients", "KernelParams",
           "DataError", "NumericalError", "UsageError", "CudaError", "launch_count", "RaySampler"]
