"""Standalone reconstruct_primal on the c4 bench batch (device-resident):
CUDA-event time per batch and the HBM fraction (profiling helper)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import KKTSystem, PcgConfig, PrecondKind
B, N, n, m = int(os.environ.get("PB", "4096")), 63, 14, 7
kb = api.random_kkt_batch(2309, B, N, n, m)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
api.context().set_stream(stream.cuda_stream)  # the events below see the launches
kd = KKTSystem(N, n, m, *[torch.from_numpy(x).cuda() for x in kb.arrays()])
lam = torch.empty((B, (N + 1) * n), dtype=torch.float64, device="cuda")
api.solve_batched_device(kd, lam.data_ptr(), B, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
P = (N + 1) * n + N * m
dz = torch.empty((B, P), dtype=torch.float64, device="cuda")
for _ in range(3):
    api.reconstruct_primal_batched_device(kd, lam.data_ptr(), dz.data_ptr(), B)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = int(os.environ.get("PREPS", "20"))
e0.record()
for _ in range(reps):
    api.reconstruct_primal_batched_device(kd, lam.data_ptr(), dz.data_ptr(), B)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
pbytes = 8 * ((N + 1) * (n * n + n) + N * (m * m + m + n * n + n * m) + (N + 1) * n + P)
gbs = B * pbytes / (ms * 1e-3) / 1e9
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
i = 5
want = api.reconstruct_primal(kb.system(i), lam[i].cpu().numpy())
err = float(np.abs(dz[i].cpu().numpy() - want).max())
print(json.dumps({"ms": ms, "GBs": gbs, "frac": gbs / peak, "max_abs_diff_vs_single": err}))
