"""Randomised shapes through the rest of the public API against the oracle:
build_schur (S, gamma, theta^-1), build_preconditioner + apply_preconditioner,
the explicit-Phi pcg_solve_auto, reconstruct_primal, sqp_step, and the
device-resident batch solve. python scripts/api_fuzz.py [count] [seed]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import pyoracle as orc
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind

count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
kinds = [PrecondKind.identity, PrecondKind.block_jacobi, PrecondKind.stair,
         PrecondKind.symmetric_stair]


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max())) if b.size else 0.0


bad = []
for t in range(count):
    N = int(rng.choice([0, 1, 2, 7, 31, 32, 33, 63, 64, 100]))
    n = int(rng.integers(1, 33))
    m = int(rng.integers(1, 17))
    kind = kinds[int(rng.integers(1, 4))]
    kkt = orc.random_kkt(int(rng.integers(1, 1 << 30)), N, n, m)
    row = {"N": N, "n": n, "m": m, "kind": int(kind)}
    try:
        g, o = api.build_schur(kkt), orc.build_schur(kkt)
        row["S"] = rel(g.S.data, o.S.data)
        row["gamma"] = rel(g.gamma, o.gamma)
        row["theta_inv"] = rel(np.asarray(g.theta_inv), np.asarray(o.theta_inv))
        P, Po = api.build_preconditioner(o, kind), orc.build_preconditioner(o, kind)
        r = rng.standard_normal(o.gamma.shape[0])
        row["apply"] = rel(api.apply_preconditioner(P, r), orc.apply_preconditioner(Po, r))
        cfg = PcgConfig(epsilon=1e-8)
        res = api.pcg_solve_auto(o.S, P, o.gamma, np.zeros_like(o.gamma), cfg)
        ores = orc.pcg_solve_auto(o.S, Po, o.gamma, np.zeros_like(o.gamma), cfg)
        row["pcg_iters_equal"] = res.report.iterations == ores.report.iterations
        row["pcg_lambda"] = rel(res.lambda_, ores.lambda_)
        lam = ores.lambda_
        row["dz"] = rel(api.reconstruct_primal(kkt, lam), orc.reconstruct_primal(kkt, lam))
        sres, sdz = api.sqp_step(kkt, kind, cfg=cfg)
        want = orc.solve(kkt, kind, cfg=cfg)
        row["sqp_iters_equal"] = sres.report.iterations == want.report.iterations
        row["sqp_dz"] = rel(sdz, orc.reconstruct_primal(kkt, want.lambda_))
        ok = (row["S"] <= 1e-12 and row["gamma"] <= 1e-12 and row["theta_inv"] <= 1e-10 and
              row["apply"] <= 1e-10 and row["pcg_iters_equal"] and row["pcg_lambda"] <= 1e-10 and
              row["dz"] <= 1e-10 and row["sqp_iters_equal"] and row["sqp_dz"] <= 1e-8)
    except Exception as e:  # noqa: BLE001
        ok, row["error"] = False, str(e)[:160]
    row["ok"] = ok
    if not ok:
        bad.append(row)
    print(json.dumps(row), flush=True)
print(json.dumps({"cases": count, "failed": len(bad), "bad": bad}))
