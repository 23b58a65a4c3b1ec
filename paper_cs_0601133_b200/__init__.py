"""B200-native fgemm: exact C <- (alpha op(A) op(B) + beta C) mod p on sm_100a tensor cores.

The product is the CUDA library ``lib/libffgemm.so`` (C ABI: include/ffgemm.h);
this package is its thin binding (``ffgemm``) plus the multi-GPU row-panel
driver (``sharded``).  Importing it without the built library raises.
"""
from .ffgemm import (EXPORTED, FFError, fgemm, ff_device_check, ff_encode, ff_fill_uniform,  # noqa: F401
                     ff_gemm, ff_gemm_ex, ff_gemm_host, ff_gemm_limbs, ff_gemm_workspace_size,
                     ff_opts, ff_plan_query, ff_strerror, ff_version, LIB_PATH,
                     ff_trsm, ff_trsm_ex, ff_trsm_workspace_size, ftrsm, lqup, rank_det,
                     ff_prof_start, ff_prof_stop, ff_mma_ceiling,
                     ff_gemm_winograd_levels)

__all__ = ["fgemm", "ff_gemm", "ff_gemm_ex", "ff_gemm_host", "ff_gemm_limbs", "ff_encode",
           "ff_fill_uniform", "ff_plan_query", "ff_gemm_workspace_size", "ff_strerror",
           "ff_version", "ff_device_check", "ff_opts", "FFError", "EXPORTED", "LIB_PATH",
           "ff_trsm", "ff_trsm_ex", "ff_trsm_workspace_size", "ftrsm", "lqup", "rank_det",
           "ff_prof_start", "ff_prof_stop", "ff_mma_ceiling",
           "ff_gemm_winograd_levels"]
