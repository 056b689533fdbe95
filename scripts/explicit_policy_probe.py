"""Explicit-Phi pcg_solve at c1 / c2 / NMPC shapes under the K3 configurations
(1 CTA unstaged, 1 CTA staged, clusters of 2/4/8, grid): device time per solve."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2309_08079_b200.api as api  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402

variants = {"auto": {}, "G1_unstaged": {"B2P_PCG_G": "1", "B2P_PCG_STAGE": "0"},
            "G2": {"B2P_PCG_G": "2"}, "G4": {"B2P_PCG_G": "4"}, "G8": {"B2P_PCG_G": "8"},
            "G16": {"B2P_PCG_G": "16"}}
for (N, n, m) in [(31, 14, 7), (127, 14, 7), (32, 2, 1), (128, 4, 1), (63, 14, 7), (255, 12, 4)]:
    kkt = api.random_kkt(3, N, n, m)
    sch = api.build_schur(kkt)
    P = api.build_preconditioner(sch, PrecondKind.symmetric_stair)
    row = [(N, n, m)]
    for name, env in variants.items():
        saved = dict(os.environ)
        os.environ.update(env)
        ts = []
        for i in range(13):
            r = api.pcg_solve_auto(sch.S, P, sch.gamma, sch.gamma * 0, PcgConfig(epsilon=1e-8))
            if i >= 3:
                ts.append(r.report.wall_time * 1e6)
        os.environ.clear()
        os.environ.update(saved)
        row.append(f"{name} {statistics.median(ts):.0f}")
    print(*row, "iters", r.report.iterations)
