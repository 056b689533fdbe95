"""c1 single-solve device latency per kernel path (policy check):
one-CTA fused, fused cluster (G = 2, 4), fused grid, split. CUDA-event device
time of api.solve (median of 30); iterations checked against the oracle."""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as orc
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind
K = int(sys.argv[1]) if len(sys.argv) > 1 else 32
kkt = api.random_kkt(1, K - 1, 14, 7)
cfg = PcgConfig(epsilon=1e-8)
want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg).report.iterations
out = {}
for name, env in [("default", {}), ("one_cta", {"B2P_FC": "0", "B2P_FG": "0"}),
                  ("fc2", {"B2P_FC": "1", "B2P_FC_G": "2", "B2P_FG": "0"}),
                  ("fc4", {"B2P_FC": "1", "B2P_FC_G": "4", "B2P_FG": "0"}),
                  ("fg", {"B2P_FG": "1"}), ("split", {"B2P_FUSED": "0"})]:
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ts = []
        for i in range(35):
            r = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
            if i >= 5:
                ts.append(r.report.wall_time * 1e6)
        out[name] = {"us_device_median": statistics.median(ts), "path": api.context().last_path(),
                     "iterations_equal": r.report.iterations == want}
    except Exception as e:
        out[name] = {"error": str(e)[:120]}
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
print(json.dumps({"K": K, "rows": out}))
