"""B200-native (sm_100a) rank-k symmetric eigen-update — the hot path of
arXiv 1706.00773 behind the reference's own entry points.

The compute path is the CUDA library lib/libeigmod_b200.so (C ABI in
include/eigmod_b200.h); this package is its Python host side. See DESIGN.md.
"""
from .capi import (  # noqa: F401
    Context,
    DeflatedProblem,
    DeviceError,
    EigenvalueUpdate,
    NumericalError,
    UpdateResult,
    default_context,
    default_tolerance,
    deflate_problem,
    gemm_nt_device,
    apply_update,
    locate,
    locate_from_u,
    ortho_error,
    reconstruct,
    padded_rank,
    record_width,
    secular_weights,
    transform_update,
    update_decomposition,
    update_decomposition_device,
    update_eigenvalues,
    update_eigenvalues_full,
)
from .instances import CONFIGS, make_instance, make_instance_torch  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
