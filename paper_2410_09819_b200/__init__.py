"""B200-native mixed-precision out-of-core left-looking tile Cholesky
(arxiv 2410.09819) -- thin Python binding over the C ABI in
``include/mxp_chol.h`` (libmxpchol.so, built in-tree for sm_100a).

The binding only marshals arguments: every step of the factorization runs in
the library's CUDA kernels.  There is no CPU fallback -- if the shared
library is missing or fails to load, every entry point raises.

Matrix layout: column-major with a leading dimension, lower triangle
referenced (LAPACK ``dpotrf('L')``).  For a torch tensor that means a
Fortran-strided view: ``A.stride(0) == 1`` and ``lda = A.stride(1)``.  For a
symmetric row-major tensor ``S``, ``S.T`` is such a view of the same matrix;
after the call ``S.T`` holds L in its lower triangle.
"""
from __future__ import annotations

import ctypes
import os

from .binding import (  # noqa: F401
    FP8,
    FP16,
    FP32,
    FP64,
    MxpError,
    Plan,
    abi_version,
    generate_kms_device,
    generate_matern_device,
    generate_plgsy_device,
    host_alloc,
    host_free,
    lib,
    lib_path,
    ooc_variant_volume,
    precision_map_from_matrix,
    precision_map_from_matrix_device,
    precision_map_matern_device,
)

__all__ = [
    "FP64", "FP32", "FP16", "FP8", "MxpError", "Plan", "abi_version", "lib", "lib_path", "ooc_variant_volume",
    "precision_map_from_matrix", "precision_map_from_matrix_device", "generate_plgsy_device", "generate_kms_device",
    "generate_matern_device", "precision_map_matern_device",
    "host_alloc", "host_free",
]
