"""ctypes binding of libtfg (include/tfg.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``).  There is no fallback: if the
library is missing, importing the package's compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtfg.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)

TFG_OK, TFG_EINVAL, TFG_ERUNTIME, TFG_ECUDA = 0, 1, 2, 3
TFG_F32, TFG_F64 = 0, 1


class TfgConfig(C.Structure):
    """tfg_config == tilefuse::SchedulerConfig (scheduler.hpp:15-24)."""

    _fields_ = [
        ("ct_size", C.c_int32),
        ("num_workers", C.c_int32),
        ("cache_size_words", C.c_uint64),
        ("b_cols", C.c_int32),
        ("c_cols", C.c_int32),
        ("index_to_scalar_ratio", C.c_double),
        ("b_is_dense", C.c_int32),
        ("whole_b_cost", C.c_int32),
    ]


PLAN_REFERENCE_BITS = 1  # tfg.h TFG_PLAN_REFERENCE_BITS


class TfgProblem(C.Structure):
    """tfg_problem == FusedProblem<T> (kernels.hpp:16-43) as pointers."""

    _fields_ = [
        ("dtype", C.c_int32),
        ("n", C.c_int32),
        ("b_is_dense", C.c_int32),
        ("b_rows", C.c_int32),
        ("b_cols", C.c_int32),
        ("c_rows", C.c_int32),
        ("c_cols", C.c_int32),
        ("a_nnz", C.c_int64),
        ("b_nnz", C.c_int64),
        ("d_a_row_ptr", C.c_void_p),
        ("d_a_col_idx", C.c_void_p),
        ("d_a_val", C.c_void_p),
        ("d_b_row_ptr", C.c_void_p),
        ("d_b_col_idx", C.c_void_p),
        ("d_b_val", C.c_void_p),
        ("d_b_dense", C.c_void_p),
        ("d_c", C.c_void_p),
    ]


# (name, restype, argtypes) for every symbol include/tfg.h declares.
SIGNATURES = [
    ("tfg_last_error", C.c_char_p, []),
    ("tfg_config_default", None, [C.POINTER(TfgConfig)]),
    ("tfg_device_info", C.c_int, [i32p, i32p]),
    ("tfg_choose_tile_size", C.c_int, [C.c_int32, C.c_int32, C.c_int32, i32p]),
    ("tfg_build_schedule", C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.POINTER(TfgConfig), C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tfg_build_schedule_host", C.c_int, [C.c_int32, C.c_int32, i32p, i32p, C.POINTER(TfgConfig),
                                          C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tfg_schedule_info", C.c_int, [C.c_void_p, i32p, i32p, i64p, i64p, f64p]),
    ("tfg_schedule_export", C.c_int, [C.c_void_p, C.c_int, i32p, i32p, f64p, i64p, i32p]),
    ("tfg_schedule_import", C.c_int, [C.c_int32, C.c_int32, i64p, C.POINTER(i32p), C.POINTER(i32p),
                                      C.POINTER(f64p), C.POINTER(i64p), C.POINTER(i32p),
                                      C.POINTER(C.c_void_p)]),
    ("tfg_schedule_destroy", None, [C.c_void_p]),
    ("tfg_fused_ratio", C.c_double, [C.c_void_p]),
    ("tfg_validate_schedule", C.c_int, [C.c_int32, C.c_int32, i32p, i32p, C.c_void_p,
                                        C.POINTER(TfgConfig), i32p, i64p, i64p, C.c_char_p,
                                        C.c_size_t]),
    ("tfg_validate_messages", C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("tfg_tile_cost", C.c_int, [C.c_int32, i32p, i32p, C.c_int32, C.c_int32, i32p, C.c_int64,
                                C.POINTER(TfgConfig), C.POINTER(C.c_double)]),
    ("tfg_split_tile", C.c_int, [C.c_int32, i32p, i32p, C.c_int32, C.c_int32, i32p, C.c_int64,
                                 C.POINTER(TfgConfig), i64p, i32p, i32p, C.POINTER(C.c_double),
                                 i64p, i32p, i64p, i32p]),
    ("tfg_balance", C.c_int, [C.c_int64, i64p, C.c_int64, i64p]),
    ("tfg_nccl_unique_id", C.c_int, [C.c_void_p, C.c_size_t]),
    ("tfg_nccl_comm_init", C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("tfg_nccl_comm_destroy", C.c_int, [C.c_void_p]),
    ("tfg_partition_bounds", C.c_int, [C.c_void_p, i32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_int32, i32p]),
    ("tfg_halo_create", C.c_int, [C.c_void_p, C.c_void_p, i32p, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tfg_halo_info", C.c_int, [C.c_void_p, i32p, i64p, i64p, C.POINTER(C.c_double),
                                C.POINTER(C.c_double)]),
    ("tfg_halo_destroy", None, [C.c_void_p]),
    ("tfg_plan_execute_dist", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tfg_plan_execute_dist_emulated", C.c_int, [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                                 C.c_int32, C.POINTER(C.c_void_p), C.c_void_p]),
    ("tfg_plan_create", C.c_int, [C.POINTER(TfgProblem), C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_void_p)]),
    ("tfg_plan_create_ex", C.c_int, [C.POINTER(TfgProblem), C.c_void_p, C.c_uint32, C.c_int32,
                                     C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tfg_plan_create_partition", C.c_int, [C.POINTER(TfgProblem), C.c_void_p, C.c_int32,
                                            C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tfg_plan_d1", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    ("tfg_plan_execute_stage", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("tfg_plan_execute", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("tfg_plan_stats", C.c_int, [C.c_void_p, i64p, i64p, i64p]),
    ("tfg_plan_info", C.c_int, [C.c_void_p, i64p, i64p, i32p, i64p]),
    ("tfg_plan_kernels", C.c_int, [C.c_void_p, C.c_char_p, C.c_int32]),
    ("tfg_plan_profile", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, f64p, i64p]),
    ("tfg_plan_destroy", None, [C.c_void_p]),
    ("tfg_run_host", C.c_int, [C.POINTER(TfgProblem), C.c_void_p, C.c_void_p]),
    ("tfg_gemm_rows_host", C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                     C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    ("tfg_spmm_rows_host", C.c_int, [C.c_int32, C.c_int32, C.c_int32, i32p, i32p, C.c_void_p,
                                     C.c_void_p, C.c_int32, C.c_int32, i32p, C.c_int64, C.c_void_p]),
    ("tfg_gather_rows", C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64,
                                  C.c_void_p, C.c_void_p]),
    ("tfg_scatter_rows", C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int64,
                                   C.c_void_p, C.c_void_p]),

]

_lib = None


class TfgError(RuntimeError):
    pass


def lib():
    """Load libtfg.so (once).  Fails loudly when the CUDA build is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libtfg.so not found at {LIB_PATH}: the sm_100a CUDA library must be built "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int):
    """Map tfg_status to the reference's exception types
    (invalid_argument -> ValueError, runtime_error -> RuntimeError)."""
    if rc == TFG_OK:
        return
    msg = lib().tfg_last_error().decode(errors="replace")
    if rc == TFG_EINVAL:
        raise ValueError(msg)
    raise TfgError(msg)
