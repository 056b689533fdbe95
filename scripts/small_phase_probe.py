"""Per-phase time of the small-block kernel (B2P_PHASE_TIMING=1 globaltimer stamps):
staging, F1, F2, PCG for single NMPC-shape solves."""
import json
import os
import sys
os.environ["B2P_PHASE_TIMING"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2309_08079_b200.api as api  # noqa: E402
from paper_2309_08079_b200._lib import load  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402

for (N, n, m) in [(32, 2, 1), (32, 4, 1), (128, 4, 1)]:
    kkt = api.random_kkt(3, N, n, m)
    rows = []
    for _ in range(10):
        r = api.solve(kkt, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
        buf = np.zeros((1, 16), dtype=np.uint64)
        load().b2p_ctx_phase_stamps(api.context().handle, buf.ctypes.data, 1)
        rows.append(np.diff(buf[0, :5].astype(np.int64)) / 1e3)
    d = np.median(np.array(rows[3:]), axis=0)
    print(json.dumps({"shape": [N, n, m], "iters": r.report.iterations, "stage_us": d[0],
                      "F1_us": d[1], "F2_us": d[2], "PCG_us": d[3],
                      "pcg_us_per_iter": d[3] / (r.report.iterations + 1),
                      "event_us": r.report.wall_time * 1e6}))
