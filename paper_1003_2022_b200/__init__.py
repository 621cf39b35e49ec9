"""B200-native drop-in for the reference's space-variant filtering path.

The reference (arxiv/paper_1003_2022, Python package ``rubs``) filters an
image with a per-pixel four-direction box-spline kernel in O(1) per pixel:
four directional running sums, then a 16-vertex finite difference read
through a 7-tap Zwart-Powell interpolant.  This package keeps that API
(pkg/src/rubs/__init__.py:46-53) and runs the path in hand-written sm_100a
kernels (csrc/) behind a C ABI (include/rubs_b200.h).

There is no CPU fallback: without the native library (or without a CUDA
device) every filtering call raises.
"""

from .engine import (
    SCALE_FLOOR,
    DeviceLut,
    FdMesh,
    IntegratedImage,
    ScaleField,
    device_lut,
    fd_mesh,
    filter_space_invariant,
    filter_space_variant,
    filter_space_variant_params,
    filter_space_variant_params_batch,
    filter_space_variant3,
    filter_space_variant3_params,
    interpolate,
    scales3_many,
    lookup_many,
    preintegrate,
    thread_cap,
)
from .geometry import (
    MIN_ELONGATION_BOUND,
    as_scale_vector,
    covariance_from_params,
    covariance_general,
    covariance_of,
    direction_vectors,
    elongation_bound,
    elongation_bound3,
    scales3_from_params,
    sigma_to_size,
)
from ._native import PrecisionWarning
from .solver import Infeasible, OutOfGrid, ScaleLut, build_lut, default_lut, optimize_scale_vector
from .tensor import AnisotropyMaps, adaptive_smooth, anisotropy_from_tensor, structure_tensor

__version__ = "0.1.0"

__all__ = [
    "AnisotropyMaps",
    "adaptive_smooth",
    "anisotropy_from_tensor",
    "structure_tensor",
    "SCALE_FLOOR",
    "DeviceLut",
    "FdMesh",
    "IntegratedImage",
    "ScaleField",
    "ScaleLut",
    "Infeasible",
    "OutOfGrid",
    "PrecisionWarning",
    "MIN_ELONGATION_BOUND",
    "as_scale_vector",
    "build_lut",
    "covariance_from_params",
    "covariance_of",
    "default_lut",
    "device_lut",
    "elongation_bound",
    "fd_mesh",
    "filter_space_invariant",
    "filter_space_variant",
    "filter_space_variant_params",
    "filter_space_variant_params_batch",
    "filter_space_variant3",
    "filter_space_variant3_params",
    "scales3_many",
    "scales3_from_params",
    "covariance_general",
    "direction_vectors",
    "elongation_bound3",
    "interpolate",
    "lookup_many",
    "optimize_scale_vector",
    "preintegrate",
    "sigma_to_size",
    "thread_cap",
    "__version__",
]
