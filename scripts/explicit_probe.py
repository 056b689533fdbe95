"""Latency of the explicit-Phi API path (build_schur -> build_preconditioner -> pcg_solve,
three C-ABI calls, device time of the PCG kernel) at small n and c1."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2309_08079_b200.api as api  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402

for (N, n, m) in [(32, 2, 1), (32, 4, 1), (128, 4, 1), (31, 14, 7)]:
    kkt = api.random_kkt(3, N, n, m)
    sch = api.build_schur(kkt)
    P = api.build_preconditioner(sch, PrecondKind.symmetric_stair)
    ts = []
    for i in range(23):
        r = api.pcg_solve_auto(sch.S, P, sch.gamma, sch.gamma * 0, PcgConfig(epsilon=1e-8))
        if i >= 3:
            ts.append(r.report.wall_time * 1e6)
    print((N, n, m), "pcg_solve device us", round(statistics.median(ts), 1), "iters",
          r.report.iterations, "per-iter", round(statistics.median(ts) / (r.report.iterations + 1), 2))
