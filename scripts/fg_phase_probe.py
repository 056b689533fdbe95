"""Per-phase time of the fused grid kernel for one c5 solve (B2P_PHASE_TIMING=1 stamps of CTA 0)."""
import json, os, sys
os.environ["B2P_PHASE_TIMING"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200._lib import load
from paper_2309_08079_b200.types import PcgConfig, PrecondKind
cases = {"c5": (5, 511, 28, 14, np.float64, 1e-8), "c3": (3, 255, 12, 4, np.float32, 1e-4),
         "c2": (2, 127, 14, 7, np.float64, 1e-8)}
for name, (seed, N, n, m, dt, eps) in cases.items():
    if name != "c5":
        os.environ["B2P_FG"] = "1"
    kkt = api.random_kkt(seed, N, n, m)
    for _ in range(3):
        r = api.solve(kkt, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=eps), dtype=dt)
    buf = np.zeros((1, 16), dtype=np.uint64)
    load().b2p_ctx_phase_stamps(api.context().handle, buf.ctypes.data, 1)
    t = buf[0].astype(np.int64)
    it = r.report.iterations
    out = {"case": name, "iters": it, "device_us": r.report.wall_time * 1e6,
           "stage_us": (t[1] - t[0]) / 1e3, "F1_us": (t[2] - t[1]) / 1e3,
           "F2_err_us": (t[3] - t[2]) / 1e3, "init_us": (t[4] - t[3]) / 1e3,
           "per_iter_Srow_ups_us": t[5] / 1e3 / max(1, it), "per_iter_precond_us": t[6] / 1e3 / max(1, it),
           "per_iter_eta_p_us": t[7] / 1e3 / max(1, it)}
    print(json.dumps(out))
