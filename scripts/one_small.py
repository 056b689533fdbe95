"""A few NMPC-shape single solves (double integrator, N = 32) for ncu captures of
the small-block kernel: python scripts/one_small.py [N n m]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2309_08079_b200.api as api  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402

N, n, m = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 2, 1)
kkt = api.random_kkt(11, N, n, m)
for _ in range(3):
    r = api.solve(kkt, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
print(N, n, m, r.report.iterations, api.context().last_path(), r.report.wall_time * 1e6)
