"""ctypes mirror of include/b2p.h (the C-ABI boundary).

Plain structs and enums only; no torch types cross the boundary.
"""
from __future__ import annotations

import ctypes as C

B2P_ABI_VERSION = 1

# b2p_status
OK, INVALID_ARGUMENT, RUNTIME_ERROR, BREAKDOWN, CUDA_ERROR = 0, 1, 2, 3, 4
# b2p_dtype
F64, F32 = 0, 1
# b2p_precond_kind — trajopt::PrecondKind (schur.hpp:26)
IDENTITY, BLOCK_JACOBI, STAIR, SYMMETRIC_STAIR, POLY_SPLIT = 0, 1, 2, 3, 4
# b2p_pcg_variant — trajopt::PcgVariant (pcg.hpp:12)
SEQUENTIAL, BLOCK_PARALLEL = 0, 1


class PcgConfigC(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("max_iter", C.c_int32),
        ("deterministic_reductions", C.c_int32),
        ("variant", C.c_int32),
        ("collect_trace", C.c_int32),
        ("check_residual_drift", C.c_int32),
        ("_reserved", C.c_int32),
    ]


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("exit_eta", C.c_double),
        ("wall_time", C.c_double),
        ("max_residual_drift", C.c_double),
        ("trace_len", C.c_int32),
        ("status", C.c_int32),
    ]


class ErrorC(C.Structure):
    _fields_ = [
        ("code", C.c_int32),
        ("knot", C.c_int32),
        ("iteration", C.c_int32),
        ("system", C.c_int32),
        ("message", C.c_char * 256),
    ]


class KktC(C.Structure):
    _fields_ = [
        ("N", C.c_int32),
        ("n", C.c_int32),
        ("m", C.c_int32),
        ("_pad", C.c_int32),
        ("Q", C.c_void_p),
        ("q", C.c_void_p),
        ("R", C.c_void_p),
        ("r", C.c_void_p),
        ("A", C.c_void_p),
        ("B", C.c_void_p),
        ("e", C.c_void_p),
        ("x_s", C.c_void_p),
        ("x0", C.c_void_p),
    ]


class KktOutC(C.Structure):
    _fields_ = [
        ("N", C.c_int32),
        ("n", C.c_int32),
        ("m", C.c_int32),
        ("_pad", C.c_int32),
        ("Q", C.c_void_p),
        ("q", C.c_void_p),
        ("R", C.c_void_p),
        ("r", C.c_void_p),
        ("A", C.c_void_p),
        ("B", C.c_void_p),
        ("e", C.c_void_p),
        ("x_s", C.c_void_p),
        ("x0", C.c_void_p),
    ]


KKT_FIELDS = ("Q", "q", "R", "r", "A", "B", "e", "x_s", "x0")


def kkt_shapes(N: int, n: int, m: int) -> dict:
    """Per-system array shapes of the b2p_kkt SoA layout (b2p.h)."""
    return {
        "Q": (N + 1, n, n),
        "q": (N + 1, n),
        "R": (N, m, m),
        "r": (N, m),
        "A": (N, n, n),
        "B": (N, n, m),
        "e": (N, n),
        "x_s": (n,),
        "x0": (n,),
    }
