"""Randomised shape sweep over every kernel path: (N, n, m, B, kind, dtype)
drawn from ranges that straddle each path's bounds; every system's iteration
count and lambda against the oracle. python scripts/shape_fuzz.py [count] [seed]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import pyoracle as orc
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind

count = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
kinds = [PrecondKind.symmetric_stair, PrecondKind.stair, PrecondKind.block_jacobi]
bad = []
paths = {}
for t in range(count):
    N = int(rng.choice([0, 1, 2, 7, 15, 31, 32, 33, 63, 64, 65, 100, 127, 200]))
    n = int(rng.integers(1, 33))
    m = int(rng.integers(1, 17))
    B = int(rng.choice([1, 1, 2, 5, 9, 40]))
    dt = np.float64 if rng.random() < 0.85 else np.float32
    kind = kinds[int(rng.integers(0, 3))]
    if B * (N + 1) * n * n > 6e6:
        B = 1
    kb = api.random_kkt_batch(int(rng.integers(1, 1 << 30)), B, N, n, m)
    cfg = PcgConfig(epsilon=1e-8 if dt == np.float64 else 1e-4)
    try:
        lam, reps = api.solve_batched(kb, kind, 1, cfg, dtype=dt)
        path = api.context().last_path()
        _, lo, ro = orc.solve_batch(kb, kind, 1, cfg)
        it_o = np.array([r.iterations for r in ro])
        scale = np.maximum(1.0, np.abs(lo).max(axis=1))
        err = float((np.abs(lam - lo).max(axis=1) / scale).max())
        tol = 1e-10 if dt == np.float64 else 2e-3
        ok_it = np.array_equal(reps.iterations, it_o) if dt == np.float64 else \
            bool((np.abs(reps.iterations - it_o) <= 1).all())
        ok = ok_it and err <= tol
    except Exception as e:  # noqa: BLE001
        path, ok, err = -1, False, str(e)[:100]
    paths[path] = paths.get(path, 0) + 1
    row = {"N": N, "n": n, "m": m, "B": B, "dtype": np.dtype(dt).name, "kind": int(kind),
           "path": path, "ok": ok, "err": err}
    if not ok:
        bad.append(row)
    print(json.dumps(row), flush=True)
print(json.dumps({"cases": count, "failed": len(bad), "paths": paths, "bad": bad}))
