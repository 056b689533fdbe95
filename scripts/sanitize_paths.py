"""One small solve on every kernel path, for compute-sanitizer (memcheck / racecheck /
synccheck) runs: python scripts/sanitize_paths.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2309_08079_b200.api as api  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind  # noqa: E402

cfg = PcgConfig(epsilon=1e-8)
cases = [
    ("one-CTA fused (c1)", {}, (31, 14, 7), np.float64),
    ("fused grid (c2-like)", {"B2P_FG": "1"}, (63, 14, 7), np.float64),
    ("fused cluster (c3-like)", {"B2P_FC": "1"}, (63, 12, 4), np.float32),
    ("small-block", {}, (32, 2, 1), np.float64),
    ("small-block n4", {}, (40, 4, 2), np.float64),
    ("split", {"B2P_FUSED": "0"}, (20, 3, 2), np.float64),
]
for name, env, (N, n, m), dt in cases:
    saved = dict(os.environ)
    os.environ.update(env)
    kkt = api.random_kkt(7, N, n, m)
    for kind in (PrecondKind.symmetric_stair, PrecondKind.stair, PrecondKind.block_jacobi):
        r = api.solve(kkt, kind, 1, cfg, dtype=dt)
    res, dz = api.sqp_step(kkt, cfg=cfg) if dt == np.float64 else (r, None)
    print(name, api.context().last_path(), r.report.iterations, flush=True)
    os.environ.clear()
    os.environ.update(saved)
kb = api.random_kkt_batch(9, 3, 31, 14, 7)
lam, reps = api.solve_batched(kb, cfg=cfg)
print("batched one-CTA", api.context().last_path(), [x.iterations for x in reps])
kb = api.random_kkt_batch(10, 5, 32, 2, 1)  # the small kernel's throughput build
lam, reps = api.solve_batched(kb, cfg=cfg)
print("batched small-block", api.context().last_path(), [x.iterations for x in reps])
for (N, n, m) in [(20, 3, 2), (31, 14, 7)]:  # build_schur (small formation-only / fused) +
    k = api.random_kkt(12, N, n, m)          # build_preconditioner + explicit-Phi pcg_solve
    sch = api.build_schur(k)
    P = api.build_preconditioner(sch, PrecondKind.symmetric_stair)
    r = api.pcg_solve_auto(sch.S, P, sch.gamma, sch.gamma * 0, cfg)
    print("explicit api", (N, n, m), r.report.iterations)
import torch  # noqa: E402
from paper_2309_08079_b200.types import KKTSystem  # noqa: E402
kb = api.random_kkt_batch(13, 2, 15, 14, 7)
kd = KKTSystem(15, 14, 7, *[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in kb.arrays()])
lam = torch.empty((2, 16 * 14), dtype=torch.float64, device="cuda")
st = torch.empty((2,), dtype=torch.int32, device="cuda")
api.direct_solve_batched_device(kd, lam.data_ptr(), st.data_ptr(), 2)
torch.cuda.synchronize()
print("direct baseline", st.cpu().tolist())
# round 2: several systems per CTA on the c4 kernel (next-system prefetch vs the
# formation / theta^-1 tiles, D kept in place), the odd-n padded path and the
# streaming reconstruct_primal kernel (CTAs straddling system boundaries)
SAN_B = int(os.environ.get("SAN_B", "300"))
kb = api.random_kkt_batch(14, SAN_B, 63, 14, 7)
lam, reps = api.solve_batched(kb, cfg=cfg)
print("batched one-CTA K64", SAN_B, api.context().last_path(), int(reps.iterations.sum()))
kb = api.random_kkt_batch(15, 4, 20, 13, 5)
lam, reps = api.solve_batched(kb, cfg=cfg)
print("odd-n padded", api.context().last_path(), [x.iterations for x in reps])
kb = api.random_kkt_batch(16, 7, 20, 14, 7)
kd = KKTSystem(20, 14, 7, *[torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in kb.arrays()])
lamd = torch.zeros((7, 21 * 14), dtype=torch.float64, device="cuda")
dz = torch.empty((7, kb.primal_dim()), dtype=torch.float64, device="cuda")
api.reconstruct_primal_batched_device(kd, lamd.data_ptr(), dz.data_ptr(), 7)
torch.cuda.synchronize()
print("streaming reconstruct_primal", float(dz.abs().sum()))
# n = 7, 8 on the one-CTA kernel (NB = 8 instantiation; n = 7 through the pad)
kb = api.random_kkt_batch(17, 6, 39, 8, 4)
lam, reps = api.solve_batched(kb, cfg=cfg)
print("batched one-CTA n8", api.context().last_path(), [x.iterations for x in reps])
kb = api.random_kkt_batch(18, 6, 39, 7, 2)
lam, reps = api.solve_batched(kb, cfg=cfg)
print("batched one-CTA n7 padded", api.context().last_path(), [x.iterations for x in reps])
k8 = api.random_kkt(19, 39, 8, 4)
res, dz8 = api.sqp_step(k8, cfg=cfg)
print("one-CTA n8 sqp_step", api.context().last_path(), res.report.iterations)
# padded grid / cluster shapes and the packed host batch upload
kp = api.random_kkt(20, 99, 20, 10)
r = api.solve(kp, cfg=cfg)
print("padded grid (20, 10)", api.context().last_path(), r.report.iterations)
kb = api.random_kkt_batch(21, 9, 79, 12, 4)
lam, reps = api.solve_batched(kb, cfg=cfg)
print("padded cluster (12, 4) K 80", api.context().last_path(), [x.iterations for x in reps])
os.environ["B2P_BATCH_CHUNK"] = "5"
kb = api.random_kkt_batch(22, 12, 31, 14, 7)
lam, reps = api.solve_batched(kb, cfg=cfg)
print("packed upload, chunks of 5", api.context().last_path(), [x.iterations for x in reps])
