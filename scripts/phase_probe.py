"""Per-phase time of the one-CTA fused kernel (B2P_PHASE_TIMING=1 globaltimer stamps)."""
import ctypes as C, json, os, sys
os.environ["B2P_PHASE_TIMING"] = "1"
os.environ.setdefault("B2P_FC", "0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200._lib import load
from paper_2309_08079_b200.types import PcgConfig, PrecondKind
B = int(os.environ.get("PB", "1184"))
KN = int(os.environ.get("PK", "64"))
kb = api.random_kkt_batch(2309, B, KN - 1, 14, 7)
for _ in range(3):
    lam, reps = api.solve_batched(kb, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
ctx = api.context()
buf = np.zeros((B, 8), dtype=np.uint64)
n = load().b2p_ctx_phase_stamps(ctx.handle, buf.ctypes.data, B)
d = np.diff(buf[:n, :5].astype(np.int64), axis=1) / 1e3  # us per system per phase
names = ["F1_knots", "F2_rows", "stage", "PCG"]
out = {nm: float(np.mean(d[:, i])) for i, nm in enumerate(names)}
out["total_per_system_us"] = float(np.mean(d.sum(axis=1)))
out["iters_mean"] = float(np.mean([r.iterations for r in reps]))
out["pcg_us_per_iter"] = out["PCG"] / (out["iters_mean"] + 1)
print(json.dumps(out))
