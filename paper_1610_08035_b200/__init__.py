"""B200-native SpInGP sparse-precision inference path (arXiv:1610.08035).

The product is the C-ABI shared library ``libspingp_b200.so`` (include/spingp_c.h)
built from ``csrc/`` for sm_100a.  This module is a thin ctypes mirror of that ABI
for Python callers (tests, bench.py): the same entry points, argument meaning and
error behaviour as the reference's C++ API (proj/include/spingp/*.hpp, SPEC.md
btd_core / spingp_engine), with the reference's exception types re-raised.

There is no CPU fallback: if the library is missing this import fails loudly, and
without a CUDA device every computing call raises DeviceError.
"""
from ._capi import (  # noqa: F401
    MATERN12, MATERN32, MATERN52, EQ, QP, LEAF_NPARAMS,
    WANT_GRAD, WANT_MEAN, WANT_VAR, INCLUDE_NOISE,
    SpingpError, NotPositiveDefinite, SingularProcessNoise, DuplicateTimestamp, DeviceError,
    NegativeVariance, Unsupported,
    Context, MultiContext, BTDFactor, lib, lib_path, kernel_dims, state_space, n_theta, seg_sizes,
)

__all__ = [
    "MATERN12", "MATERN32", "MATERN52", "EQ", "QP", "LEAF_NPARAMS",
    "WANT_GRAD", "WANT_MEAN", "WANT_VAR", "INCLUDE_NOISE",
    "SpingpError", "NotPositiveDefinite", "SingularProcessNoise", "DuplicateTimestamp", "DeviceError",
    "NegativeVariance", "Unsupported", "Context", "MultiContext", "BTDFactor", "lib", "lib_path", "kernel_dims", "state_space", "n_theta",
    "seg_sizes",
]
