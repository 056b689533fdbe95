"""c5 (K=512, n=28) split-path probe: K1/K3 device time for launch variants."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as orc
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind
k5 = orc.random_kkt(5, 511, 28, 14)
out = {}
for G, thr in [(128, 256), (128, 512), (64, 256), (64, 512), (32, 512), (16, 512)]:
    os.environ["B2P_PCG_G"] = str(G); os.environ["B2P_PCG_THREADS"] = str(thr)
    res = []
    for i in range(6):
        r = api.solve(k5, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
        res.append(api.context().last_phase_ms())
    out[f"G{G}_t{thr}"] = {"K1_ms": res[-1][0], "K3_ms": res[-1][1], "it": r.report.iterations}
print(json.dumps(out))
