"""Unpreconditioned-CG iteration mismatches, explained system by system
(test infrastructure: the oracle is the checker). For every system of the
identity-preconditioned c1 / c4 sweeps whose B200 iteration count differs from
the oracle's sequential variant, record:

  * the exit counts of the B200 kernel, the oracle's sequential pcg_solve and
    its block-parallel variant (deterministic tree reductions), and of an
    extended-precision (x87 80-bit long double) CG on the same S and gamma;
  * eta'/eps of each implementation at the deciding iterations;
  * the first iteration at which the eta' traces of (B200, oracle) and of
    (oracle sequential, oracle block-parallel) differ by > 1e-3 relative;
  * the count of the oracle's PCG run on the B200-formed S (isolates the
    formation's rounding from the PCG's) and of the B200's explicit-S K3 run on
    the oracle-formed S.

  python scripts/identity_mismatch.py [out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import pyoracle as orc  # noqa: E402
import paper_2309_08079_b200.api as api  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PrecondKind, PcgVariant  # noqa: E402

orc.build()
api.require_device()
EPS = 1e-8
ID = PrecondKind.identity


def cg_longdouble(S, gamma, eps, max_iter):
    """Textbook CG (pcg.cpp:55-129 with Phi = I) in 80-bit extended precision."""
    A = S.to_dense().astype(np.longdouble)
    g = np.asarray(gamma, dtype=np.longdouble)
    lam = np.zeros_like(g)
    r = g.copy()
    p = r.copy()
    eta = r @ r
    trace = []
    for i in range(1, max_iter + 1):
        sp = A @ p
        alpha = eta / (p @ sp)
        r = r - alpha * sp
        lam = lam + alpha * p
        eta_p = r @ r
        trace.append(float(eta_p))
        if eta_p < eps:
            return i, trace
        p = r + (eta_p / eta) * p
        eta = eta_p
    return max_iter, trace


def first_divergence(a, b, tol=1e-3):
    for i, (x, y) in enumerate(zip(a, b)):
        if abs(x / y - 1.0) > tol:
            return i + 1
    return None


def explain(kkt, idx, it_batch):
    cfg = PcgConfig(epsilon=EPS, collect_trace=True)
    g = api.solve(kkt, ID, cfg=cfg)
    s = orc.solve(kkt, ID, cfg=cfg)
    sch = orc.build_schur(kkt)
    z = np.zeros(sch.S.dim())
    p = orc.pcg_solve_block_parallel(sch.S, orc.build_identity(), sch.gamma, z, PcgConfig(
        epsilon=EPS, collect_trace=True, variant=PcgVariant.block_parallel,
        deterministic_reductions=True))
    ld_it, ld_tr = cg_longdouble(sch.S, sch.gamma, EPS, sch.S.dim())
    gs = api.build_schur(kkt)  # B200-formed S, gamma
    o_on_g = orc.pcg_solve(gs.S, orc.build_identity(), gs.gamma, z, PcgConfig(epsilon=EPS))
    g_on_o = api.pcg_solve(sch.S, api.build_identity(), sch.gamma, z, PcgConfig(epsilon=EPS))
    tg, ts, tp = g.report.trace, s.report.trace, p.report.trace
    dec = sorted({g.report.iterations, s.report.iterations, p.report.iterations})

    def at(tr, i):
        return tr[i - 1] / EPS if 0 < i <= len(tr) else None

    def true_res(lam):
        return float(np.linalg.norm(sch.gamma - orc.matvec(sch.S, lam)))

    return {
        "system": int(idx),
        "iterations": {"b200_batch": int(it_batch), "b200_single": g.report.iterations,
                       "oracle_sequential": s.report.iterations,
                       "oracle_block_parallel": p.report.iterations,
                       "longdouble_cg": int(ld_it),
                       "oracle_pcg_on_b200_S": o_on_g.report.iterations,
                       "b200_pcg_on_oracle_S": g_on_o.report.iterations},
        "eta_over_eps_at": {str(i): {"b200": at(tg, i), "oracle_sequential": at(ts, i),
                                     "oracle_block_parallel": at(tp, i),
                                     "longdouble": at(ld_tr, i)} for i in dec},
        "first_trace_divergence_1e-3": {
            "b200_vs_oracle_sequential": first_divergence(tg, ts),
            "oracle_sequential_vs_block_parallel": first_divergence(ts, tp),
            "oracle_sequential_vs_longdouble": first_divergence(ts, ld_tr)},
        "true_residual_norm": {"b200": true_res(g.lambda_), "oracle_sequential": true_res(s.lambda_),
                               "oracle_block_parallel": true_res(p.lambda_)},
    }


def main():
    out = {"what": __doc__.strip().splitlines()[0], "epsilon": EPS, "sweeps": []}
    for name, seed0, B, N in (("c1", 800, 256, 31), ("c4", 900, 256, 63)):
        kb = api.random_kkt_batch(seed0, B, N, 14, 7)
        _, reps = api.solve_batched(kb, ID, 1, PcgConfig(epsilon=EPS))
        _, _, rs = orc.solve_batch(kb, ID, 1, PcgConfig(epsilon=EPS))
        _, _, rp = orc.solve_batch(kb, ID, 1, PcgConfig(epsilon=EPS, variant=1,
                                                        deterministic_reductions=True))
        it_g = np.array([r.iterations for r in reps])
        it_s = np.array([r.iterations for r in rs])
        it_p = np.array([r.iterations for r in rp])
        rows = [explain(kb.system(int(i)), i, it_g[i]) for i in np.nonzero(it_g != it_s)[0]]
        sw = {"config": name, "seed0": seed0, "systems": B, "knots": N + 1,
              "b200_equal_sequential": int((it_g == it_s).sum()),
              "b200_equal_block_parallel": int((it_g == it_p).sum()),
              "sequential_equal_block_parallel": int((it_s == it_p).sum()),
              "b200_within_one_of_either": int((np.minimum(abs(it_g - it_s), abs(it_g - it_p)) <= 1).sum()),
              "mismatches": rows}
        print(json.dumps({k: v for k, v in sw.items() if k != "mismatches"}), flush=True)
        for r in rows:
            print(json.dumps(r), flush=True)
        out["sweeps"].append(sw)
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/identity_mismatches.json"
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
