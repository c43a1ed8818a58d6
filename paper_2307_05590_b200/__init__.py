"""B200-native (sm_100a, FP64) on-line stage of projected POD for MPT spectral signatures (arXiv 2307.05590).

The product is libpodp.so (C ABI, include/podp.h) built from ``csrc/``; ``podp`` is its thin ctypes binding.
"""
from .podp import (  # noqa: F401
    Evaluator, PodpError, load_library, LIB_PATH, EXPORTED, FLAG_DEFAULT, FLAG_OUT_R, FLAG_OUT_P, FLAG_NO_PIVOT, FLAG_PENCIL,
    FLAG_LU_LL, FLAG_LU_BLK, FLAG_LU_DYN, FLAG_LU_GENERIC, FLAG_MPT_GEMM, FLAG_MPT_PAIR,
    R_MAX, STATUS_NAMES, profile_enable, profile_read, invariants, coil_voltage, scale_signature, release_workspace,
)
