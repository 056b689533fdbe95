"""One single solve of a BASELINE config (for ncu captures): python scripts/one_solve.py c5"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind
cases = {"c1": (1, 31, 14, 7, np.float64, 1e-8), "c2": (2, 127, 14, 7, np.float64, 1e-8),
         "c3": (3, 255, 12, 4, np.float32, 1e-4), "c5": (5, 511, 28, 14, np.float64, 1e-8)}
seed, N, n, m, dt, eps = cases[sys.argv[1] if len(sys.argv) > 1 else "c5"]
kkt = api.random_kkt(seed, N, n, m)
for _ in range(int(os.environ.get("REPS", "2"))):
    r = api.solve(kkt, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=eps), dtype=dt)
print(r.report.iterations, r.report.wall_time * 1e6)
