"""the CPU reference beside the GPU numbers — per-solve latency of the
oracle restatement on the box's host cores, PCG-only (sequential pcg_solve on 1 core and
pcg_solve_block_parallel on every core) and full scope (build_schur + build_preconditioner
+ pcg_solve on 1 core), median of repeated runs. Test infrastructure (the oracle)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as orc  # noqa: E402
from paper_2309_08079_b200.types import PcgConfig, PcgVariant, PrecondKind  # noqa: E402

orc.build()
cores = os.cpu_count() or 1


def med(f, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t0) * 1e6)
    return statistics.median(ts)


out = {"what": __doc__.strip().splitlines()[0], "host_threads": cores}
for name, (seed, N, n, m, eps, reps) in {"c1": (1, 31, 14, 7, 1e-8, 21),
                                          "c2": (2, 127, 14, 7, 1e-8, 11),
                                          "c3": (3, 255, 12, 4, 1e-4, 7),
                                          "c5": (5, 511, 28, 14, 1e-8, 3)}.items():
    kkt = orc.random_kkt(seed, N, n, m)
    sch = orc.build_schur(kkt)
    P = orc.build_preconditioner(sch, PrecondKind.symmetric_stair)
    seq = PcgConfig(epsilon=eps)
    par = PcgConfig(epsilon=eps, variant=PcgVariant.block_parallel, deterministic_reductions=True)
    z = sch.gamma * 0
    orc.set_threads(1)
    full = med(lambda: orc.solve(kkt, PrecondKind.symmetric_stair, 1, seq), reps)
    pcg1 = med(lambda: orc.pcg_solve_auto(sch.S, P, sch.gamma, z, seq), reps)
    orc.set_threads(0)
    pcgp = med(lambda: orc.pcg_solve_auto(sch.S, P, sch.gamma, z, par), reps)
    it = orc.pcg_solve_auto(sch.S, P, sch.gamma, z, seq).report.iterations
    out[name] = {"knots": N + 1, "nx": n, "nu": m, "epsilon": eps, "iterations": it,
                 "full_scope_1core_us": full, "pcg_sequential_1core_us": pcg1,
                 "pcg_block_parallel_all_cores_us": pcgp,
                 "note": "c3 on the fp64 oracle (the reference is fp64-only)"
                 if name == "c3" else ""}
    print(name, json.dumps(out[name]), flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cpu_ref_latency.json", "w"),
          indent=1)
