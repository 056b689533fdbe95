"""B200-native symmetric-stair PCG hot path of arXiv 2309.08079 (MPCGPU).

Host value types mirror proj/include/trajopt; compute entry points live in
`paper_2309_08079_b200.api` and call the sm_100a library libb2p.so through the
C-ABI in include/b2p.h. There is no CPU fallback.
"""
from .types import (B2PCudaError, BlockTriMatrix, KKTSystem, PcgBreakdown, PcgConfig, PcgResult,
                    PcgVariant, Preconditioner, PrecondKind, SchurSystem, SolveReport,
                    parse_precond, precond_name)

__all__ = [
    "B2PCudaError", "BlockTriMatrix", "KKTSystem", "PcgBreakdown", "PcgConfig", "PcgResult",
    "PcgVariant", "Preconditioner", "PrecondKind", "SchurSystem", "SolveReport", "parse_precond",
    "precond_name",
]
