"""Loader for the in-tree sm_100a library libb2p.so (the C-ABI of include/b2p.h).

There is no CPU fallback: if the library is missing the import of the
compute API fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libb2p.so")

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp, i32, dbl, u64, i64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_longlong
    E = C.POINTER(_abi.ErrorC)
    CFG = C.POINTER(_abi.PcgConfigC)
    REP = C.POINTER(_abi.SolveReportC)
    KKT = C.POINTER(_abi.KktC)
    sig = {
        "b2p_abi_version": ([], i32),
        "b2p_device_count": ([], i32),
        "b2p_ctx_create": ([i32, C.POINTER(vp), E], i32),
        "b2p_ctx_destroy": ([vp], None),
        "b2p_ctx_set_stream": ([vp, vp], i32),
        "b2p_ctx_stream": ([vp], vp),
        "b2p_ctx_kernel_launches": ([vp], i64),
        "b2p_ctx_last_path": ([vp], i32),
        "b2p_ctx_phase_stamps": ([vp, vp, i32], i32),
        "b2p_ctx_last_solve_ms": ([vp, C.POINTER(C.c_float)], i32),
        "b2p_ctx_last_h2d_bytes": ([vp, C.POINTER(C.c_ulonglong)], i32),
        "b2p_ctx_last_phase_ms": ([vp, C.POINTER(C.c_float), i32], i32),
        "b2p_ctx_phase_accounting": ([vp, i32], i32),
        "b2p_ctx_phase_totals": ([vp, C.POINTER(C.c_float), i32, C.POINTER(i32)], i32),
        "b2p_blocktri_matvec": ([vp, i32, i32, i32, vp, vp, i32, vp, E], i32),
        "b2p_blocktri_cholesky_solve": ([vp, i32, i32, i32, vp, vp, i32, vp, E], i32),
        "b2p_blocktri_check": ([vp, i32, i32, i32, vp, C.POINTER(dbl), C.POINTER(dbl), E], i32),
        "b2p_build_schur": ([vp, i32, KKT, vp, vp, vp, E], i32),
        "b2p_stair_matrix": ([vp, i32, i32, i32, vp, vp, E], i32),
        "b2p_build_preconditioner": ([vp, i32, i32, i32, i32, i32, vp, vp, vp, E], i32),
        "b2p_apply_preconditioner": ([vp, i32, i32, i32, i32, i32, vp, vp, vp, i32, vp, E], i32),
        "b2p_pcg_solve": ([vp, i32, i32, i32, vp, i32, i32, i32, i32, vp, vp, i32, vp, i32, CFG,
                           vp, REP, vp, E], i32),
        "b2p_solve": ([vp, i32, KKT, i32, i32, CFG, vp, vp, REP, vp, E], i32),
        "b2p_solve_batched": ([vp, i32, i32, KKT, i32, i32, CFG, vp, vp, REP, E], i32),
        "b2p_solve_batched_device": ([vp, i32, i32, KKT, i32, i32, CFG, vp, vp, REP, vp, E],
                                     i32),
        "b2p_solve_batched_multi": ([C.POINTER(i32), i32, i32, i32, KKT, i32, i32, CFG, vp, vp,
                                     REP, E], i32),
        "b2p_reconstruct_primal": ([vp, i32, KKT, vp, i32, vp, E], i32),
        "b2p_sqp_step": ([vp, i32, KKT, i32, i32, CFG, vp, vp, vp, REP, vp, E], i32),
        "b2p_direct_solve_batched_device": ([vp, i32, i32, KKT, vp, vp, E], i32),
        "b2p_reconstruct_primal_batched_device": ([vp, i32, i32, KKT, vp, vp, E], i32),
        "b2p_random_kkt": ([i32, u64, i32, i32, i32, dbl, dbl, C.POINTER(_abi.KktOutC), E], i32),
        "b2p_random_kkt_batch": ([i32, u64, i32, i32, i32, i32, dbl, dbl, i32,
                                  C.POINTER(_abi.KktOutC), E], i32),
        "b2p_uniform_draws": ([u64, i32, dbl, dbl, vp, E], i32),
        "b2p_host_alloc": ([C.c_size_t], vp),
        "b2p_host_free": ([vp], None),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    if L.b2p_abi_version() != _abi.B2P_ABI_VERSION:
        raise ImportError("libb2p.so ABI version mismatch; rebuild")
    _lib = L
    return L


EXPORTED = [
    "b2p_abi_version", "b2p_device_count", "b2p_ctx_create", "b2p_ctx_destroy",
    "b2p_ctx_set_stream", "b2p_ctx_stream", "b2p_ctx_kernel_launches", "b2p_ctx_last_path",
    "b2p_ctx_phase_stamps",
    "b2p_ctx_last_solve_ms",
    "b2p_ctx_last_h2d_bytes",
    "b2p_ctx_last_phase_ms", "b2p_ctx_phase_accounting", "b2p_ctx_phase_totals",
    "b2p_blocktri_matvec", "b2p_blocktri_cholesky_solve", "b2p_blocktri_check",
    "b2p_build_schur", "b2p_stair_matrix", "b2p_build_preconditioner",
    "b2p_apply_preconditioner", "b2p_pcg_solve", "b2p_solve", "b2p_solve_batched",
    "b2p_solve_batched_device", "b2p_solve_batched_multi", "b2p_reconstruct_primal",
    "b2p_reconstruct_primal_batched_device", "b2p_sqp_step", "b2p_direct_solve_batched_device", "b2p_random_kkt",
    "b2p_random_kkt_batch", "b2p_uniform_draws", "b2p_host_alloc", "b2p_host_free",
]
