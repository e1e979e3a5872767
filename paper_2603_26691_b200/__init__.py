"""B200-native SCALE-TRACK hot path (arXiv 2603.26691): the two-way-coupled
Lagrangian particle step as sm_100a CUDA kernels behind a C ABI
(include/scaletrack.h).  This package is the thin Python binding; see DESIGN.md.
"""
from ._native import (BC_PERIODIC, BC_REFLECT, DECOMP_SHARDED, DECOMP_SLAB, DRAG_SCHILLER_NAUMANN, DRAG_STOKES,
                      INT_EXPONENTIAL,
                      INT_SEMI_IMPLICIT, ONE_WAY, TWO_WAY, StError)
from .api import (Config, Extrapolator, MicroConfig, ScaleTrack, hilbert_index, micro_advance, nccl_unique_id, plan_hilbert,
                  plan_layout, plan_partition)

__all__ = [
    "Config", "Extrapolator", "MicroConfig", "ScaleTrack", "micro_advance", "StError", "nccl_unique_id", "plan_layout", "plan_partition",
    "hilbert_index", "plan_hilbert",
    "BC_PERIODIC", "BC_REFLECT", "DRAG_STOKES", "DRAG_SCHILLER_NAUMANN",
    "INT_EXPONENTIAL", "INT_SEMI_IMPLICIT", "ONE_WAY", "TWO_WAY", "DECOMP_SLAB", "DECOMP_SHARDED",
]
