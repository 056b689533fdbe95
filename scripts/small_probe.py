"""Device latency of single solves at NMPC-sized shapes (n = 2, 4) vs c1, with
the formation + one iteration split out (max_iter = 1) and the PCG team variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import latency_sweep as ls  # noqa: E402
from latency_sweep import orc, timed  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402
import paper_2309_08079_b200.api as api  # noqa: E402
import numpy as np  # noqa: E402
import statistics  # noqa: E402


def t_cap(k, cap, env=None):
    saved = {kk: os.environ.get(kk) for kk in (env or {})}
    os.environ.update(env or {})
    ts = []
    for i in range(20):
        r = api.solve(k, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-30, max_iter=cap))
        if i >= 3:
            ts.append(r.report.wall_time * 1e6)
    for kk, vv in saved.items():
        if vv is None:
            os.environ.pop(kk, None)
        else:
            os.environ[kk] = vv
    return statistics.median(ts)


for (N, n, m) in [(32, 2, 1), (32, 4, 1), (128, 4, 1), (31, 14, 7)]:
    k = orc.random_kkt(3, N, n, m)
    v = timed(k, PrecondKind.symmetric_stair, 1e-8)
    row = [(N, n, m), round(v["us_median"], 1), v["path"], v["iterations"], v["iterations_equal"]]
    for env in ({},):
        t1, t11 = t_cap(k, 1, env), t_cap(k, 11, env)
        row += [env.get("B2P_SMALL_WARP", "cta"), "1it", round(t1, 1), "per-it",
                round((t11 - t1) / 10, 2)]
    print(*row)
