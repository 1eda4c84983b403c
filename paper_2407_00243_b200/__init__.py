"""B200-native tile fusion for D = A(BC) (arXiv 2407.00243).

Drop-in for the reference ``tilefuse`` operator API: the inspector
(``build_schedule``) and executors (``fused_gemm_spmm`` / ``fused_spmm_spmm``
/ ``unfused_*``) run as hand-written sm_100a kernels in ``libtfg.so`` behind
the C-ABI in ``include/tfg.h``.  No CPU fallback exists.
"""
from .tilefuse import (  # noqa: F401
    Csr,
    DeviceCsr,
    DeviceProblem,
    Plan,
    Schedule,
    SchedulerConfig,
    build_schedule,
    checked_schedule,
    choose_tile_size,
    device_info,
    fused_gemm_spmm,
    fused_ratio,
    fused_spmm_spmm,
    gen_banded,
    gen_random_sparse,
    gemm,
    spmm,
    import_schedule,
    run,
    schedule_from_json,
    schedule_json,
    schedule_to_json,
    unfused_gemm_spmm,
    unfused_spmm_spmm,
    validate_schedule,
)
from ._lib import LIB_PATH, lib  # noqa: F401
