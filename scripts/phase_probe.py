"""Per-phase time of the one-CTA fused kernel (B2P_PHASE_TIMING=1 globaltimer
stamps) on ONE device-resident launch of PB systems (default: the c4 batch),
so every CTA runs its systems back to back as in the bench.
Prints the per-system phase split (us), the PCG per-iteration segment split
(SM clocks of thread 0) and the F1 split."""
import json, os, sys
os.environ["B2P_PHASE_TIMING"] = "1"
os.environ.setdefault("B2P_FC", "0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200._lib import load
from paper_2309_08079_b200.types import PcgConfig, PrecondKind, KKTSystem
B = int(os.environ.get("PB", "4096"))
KN = int(os.environ.get("PK", "64"))
n, m = int(os.environ.get("PN", "14")), int(os.environ.get("PM", "7"))
kb = api.random_kkt_batch(2309, B, KN - 1, n, m)
kd = KKTSystem(**{f: torch.from_numpy(np.ascontiguousarray(getattr(kb, f))).cuda()
                  for f in ("Q", "q", "R", "r", "A", "B", "e", "x_s", "x0")}, N=kb.N, n=kb.n, m=kb.m)
lam = torch.empty((B, KN * n), dtype=torch.float64, device="cuda")
ctx = api.context()
for _ in range(3):
    reps = api.solve_batched_device(kd, lam.data_ptr(), B, PrecondKind.symmetric_stair, 1,
                                    PcgConfig(epsilon=1e-8), ctx=ctx, want_reports=True)
buf = np.zeros((B, 16), dtype=np.uint64)
cnt = load().b2p_ctx_phase_stamps(ctx.handle, buf.ctypes.data, B)
b = buf[:cnt].astype(np.int64)
G = 148
steady = b[G:]  # systems after the first wave (prefetched Q, warm code)
d = np.diff(steady[:, :5], axis=1) / 1e3
names = ["F1_knots", "F2_rows", "stage", "PCG"]
out = {nm: float(np.mean(d[:, i])) for i, nm in enumerate(names)}
out["total_per_system_us"] = float(np.mean(d.sum(axis=1)))
its = np.array([max(r.iterations, 1) for r in reps][G:cnt], dtype=np.float64)
out["iters_mean"] = float(np.mean(its))
out["pcg_us_per_iter"] = out["PCG"] / (out["iters_mean"] + 1)
print(json.dumps(out))
seg = steady[:, 5:8].astype(np.uint64)
cyc = np.stack([seg[:, 0] & 0xffffffff, seg[:, 0] >> 32, seg[:, 1] & 0xffffffff, seg[:, 1] >> 32,
                seg[:, 2] & 0xffffffff], axis=1).astype(np.float64)
segn = ["Srows", "ups_reduce", "update_precond", "eta_reduce", "beta_p_barrier"]
print(json.dumps({"pcg_cycles_per_iter": {nm: round(float(np.mean(cyc[:, i] / its)), 1)
                                          for i, nm in enumerate(segn)}}))
print(json.dumps({"F1_split_us": {
    "q_wait": float(np.mean(steady[:, 11] - steady[:, 0]) / 1e3),
    "Q_inv": float(np.mean(steady[:, 8] - steady[:, 11]) / 1e3),
    "R_inv": float(np.mean(steady[:, 9] - steady[:, 8]) / 1e3),
    "barrier": float(np.mean(steady[:, 1] - steady[:, 9]) / 1e3)}}))
print(json.dumps({"F2_split_us": {"products": float(np.mean(steady[:, 10] - steady[:, 1]) / 1e3),
                                  "theta_inv": float(np.mean(steady[:, 12] - steady[:, 10]) / 1e3),
                                  "theta_inv_load": float(np.mean(steady[:, 13] - steady[:, 10]) / 1e3),
                                  "theta_inv_routine": float(np.mean(steady[:, 14] - steady[:, 13]) / 1e3),
                                  "fence": float(np.mean(steady[:, 2] - steady[:, 12]) / 1e3)}}))
first = np.diff(b[:G, :5], axis=1) / 1e3
print(json.dumps({"first_wave_us": {nm: float(np.mean(first[:, i])) for i, nm in enumerate(names)}}))
