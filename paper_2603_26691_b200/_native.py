"""ctypes declarations of include/scaletrack.h (argument marshalling only).

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
into ``paper_2603_26691_b200/lib/libscaletrack.so``.  There is no fallback: if
the library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libscaletrack.so")

ST_ABI_VERSION = 3

ST_OK = 0
STATUS_NAMES = {
    0: "ST_OK", 1: "ST_ERR_INVALID_ARG", 2: "ST_ERR_STATE", 3: "ST_ERR_CAPACITY",
    4: "ST_ERR_OUT_OF_DOMAIN", 5: "ST_ERR_CFL", 6: "ST_ERR_CUDA", 7: "ST_ERR_NCCL",
    8: "ST_ERR_OOM", 9: "ST_ERR_UNSUPPORTED",
}
BC_PERIODIC, BC_REFLECT = 0, 1
DECOMP_SLAB, DECOMP_SHARDED = 0, 1
DRAG_STOKES, DRAG_SCHILLER_NAUMANN = 0, 1
INT_EXPONENTIAL, INT_SEMI_IMPLICIT = 0, 1
ONE_WAY, TWO_WAY = 0, 1


class StConfig(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("dims", ctypes.c_int32 * 3),
        ("origin", ctypes.c_double * 3),
        ("cell_size", ctypes.c_double * 3),
        ("chunk_cells", ctypes.c_int32),
        ("bc", ctypes.c_int32 * 3),
        ("rho_f", ctypes.c_double),
        ("nu_f", ctypes.c_double),
        ("rho_p", ctypes.c_double),
        ("gravity", ctypes.c_double * 3),
        ("drag_law", ctypes.c_int32),
        ("integrator", ctypes.c_int32),
        ("coupling", ctypes.c_int32),
        ("rebin_interval", ctypes.c_int32),
        ("capacity", ctypes.c_int64),
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("nccl_unique_id", ctypes.c_void_p),
        ("decomposition", ctypes.c_int32),
        ("slab_planes", ctypes.POINTER(ctypes.c_int32)),
    ]


class StLayout(ctypes.Structure):
    _fields_ = [
        ("z0", ctypes.c_int32), ("z1", ctypes.c_int32),
        ("kz0", ctypes.c_int32), ("kz1", ctypes.c_int32),
        ("n_chunks_global", ctypes.c_int32),
        ("nchunk", ctypes.c_int32 * 3),
        ("local_cells", ctypes.c_int64),
        ("halo_cells", ctypes.c_int32),
    ]


class StStats(ctypes.Structure):
    _fields_ = [
        ("n_particles", ctypes.c_int64), ("calls", ctypes.c_int64), ("rebins", ctypes.c_int64),
        ("last_movers", ctypes.c_int64), ("last_sent_total", ctypes.c_int64),
        ("last_recv_total", ctypes.c_int64), ("fused_rebins", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64), ("general_rebins", ctypes.c_int64),
        ("last_far", ctypes.c_int64),
    ]


# every symbol include/scaletrack.h declares: name -> (restype, argtypes)
_vp, _i32, _i64, _f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
EC_ZERO, EC_CONSTANT, EC_LINEAR = 0, 1, 2


class StEcConfig(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("max_backlog", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
    ]


class StMicroConfig(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("dims", ctypes.c_int32 * 3),
        ("origin", ctypes.c_double * 3),
        ("cell_size", ctypes.c_double * 3),
        ("bc", ctypes.c_int32 * 3),
        ("rho_f", ctypes.c_double), ("nu_f", ctypes.c_double), ("rho_p", ctypes.c_double),
        ("gravity", ctypes.c_double * 3),
        ("drag_law", ctypes.c_int32),
        ("D_v", ctypes.c_double), ("kappa_f", ctypes.c_double), ("cp_p", ctypes.c_double),
        ("latent", ctypes.c_double), ("nusselt", ctypes.c_double), ("s_vp", ctypes.c_double),
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("arithmetic", ctypes.c_int32),
    ]


ARITH_FP64 = 0
ARITH_FP32 = 1

SIGNATURES = {
    "st_config_default": (None, [ctypes.POINTER(StConfig)]),
    "st_init": (_i32, [ctypes.POINTER(StConfig), ctypes.POINTER(_vp)]),
    "st_destroy": (_i32, [_vp]),
    "st_set_fluid_field": (_i32, [_vp, _vp]),
    "st_inject": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "st_advance": (_i32, [_vp, _f64, _i32]),
    "st_get_sources": (_i32, [_vp, _vp, ctypes.POINTER(_f64)]),
    "st_request_sources": (_i32, [_vp]),
    "st_wait_sources": (_i32, [_vp, _vp, ctypes.POINTER(_f64)]),
    "st_get_count": (_i32, [_vp, ctypes.POINTER(_i64)]),
    "st_get_particles": (_i32, [_vp, _i64, ctypes.POINTER(_i64), _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "st_locate": (_i32, [_vp, _i64, _vp, _vp, _vp]),
    "st_get_migration_counts": (_i32, [_vp, _vp]),
    "st_get_layout": (_i32, [_vp, ctypes.POINTER(StLayout)]),
    "st_plan_layout": (_i32, [ctypes.POINTER(StConfig), ctypes.POINTER(StLayout)]),
    "st_plan_partition": (_i32, [ctypes.POINTER(StConfig), _vp, _vp]),
    "st_hilbert_index": (_i32, [ctypes.c_int32, ctypes.c_int64, _vp, _vp]),
    "st_plan_hilbert": (_i32, [ctypes.POINTER(StConfig), _vp, _vp]),
    "st_rebalance": (_i32, [_vp, ctypes.c_double, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "st_get_stats": (_i32, [_vp, ctypes.POINTER(StStats)]),
    "st_sync": (_i32, [_vp]),
    "st_last_timings": (_i32, [_vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]),
    "st_trace": (_i32, [_vp, ctypes.c_int64, _vp]),
    "st_last_error": (ctypes.c_char_p, [_vp]),
    "st_abi_version": (_i32, []),
    "st_nccl_unique_id": (_i32, [_vp]),
    "st_ec_init": (_i32, [ctypes.POINTER(StEcConfig), ctypes.POINTER(_vp)]),
    "st_ec_destroy": (_i32, [_vp]),
    "st_ec_step": (_i32, [_vp, _i32, _vp, _f64, _vp]),
    "st_ec_ledger": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "st_ec_backlog": (_i32, [_vp, ctypes.POINTER(_i32)]),
    "st_ec_last_error": (ctypes.c_char_p, [_vp]),
    "st_micro_config_default": (None, [ctypes.POINTER(StMicroConfig)]),
    "st_micro_advance": (_i32, [ctypes.POINTER(StMicroConfig), _i64, _vp, _vp, _vp, _vp, _vp, _vp, _f64, _i32,
                                _vp, ctypes.POINTER(_i64)]),
}

_lib = None


def load():
    """Load libscaletrack.so and declare every exported symbol.  Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `make` or __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.st_abi_version() != ST_ABI_VERSION:
        raise ImportError("libscaletrack.so ABI version mismatch")
    _lib = lib
    return lib


class StError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
