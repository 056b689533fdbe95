"""Direct (block-Thomas) baseline on the c4 batch: b2p_direct_solve_batched_device
with the half-warp block-Thomas kernel vs the round-1 one-warp kernel
(B2P_DIRECT_WARP=1), and the formation alone; CUDA events."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import KKTSystem, PcgConfig, PrecondKind
B, N, n, m = 4096, 63, 14, 7
kb = api.random_kkt_batch(2309, B, N, n, m)
kd = KKTSystem(N, n, m, *[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in kb.arrays()])
D = (N + 1) * n
lam = torch.empty((B, D), dtype=torch.float64, device="cuda")
st = torch.empty((B,), dtype=torch.int32, device="cuda")
ctx = api.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)
out = {}
for name, env in (("half_warp_thomas", "0"), ("warp_round1", "1")):
    if env == "1":
        os.environ["B2P_DIRECT_WARP"] = "1"
    else:
        os.environ.pop("B2P_DIRECT_WARP", None)
    api.direct_solve_batched_device(kd, lam.data_ptr(), st.data_ptr(), B, ctx=ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        api.direct_solve_batched_device(kd, lam.data_ptr(), st.data_ptr(), B, ctx=ctx)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out[name] = {"ms_per_batch": ms, "systems_per_s": B / (ms * 1e-3),
                 "all_ok": bool((st == -1).all().item()), "lam": lam[:8].cpu().numpy()}
d = np.abs(out["half_warp_thomas"]["lam"] - out["warp_round1"]["lam"]).max()
for v in out.values():
    v.pop("lam")
out["max_abs_diff_between"] = float(d)
# the PCG path on the same batch
lamp = torch.empty((B, D), dtype=torch.float64, device="cuda")
reps = api.solve_batched_device(kd, lamp.data_ptr(), B, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8), ctx=ctx)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(3):
    api.solve_batched_device(kd, lamp.data_ptr(), B, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8), ctx=ctx)
e1.record(stream)
torch.cuda.synchronize()
out["pcg_ms_per_batch"] = e0.elapsed_time(e1) / 3
print(json.dumps(out))
