"""Single-solve device latency of shapes the fused grid kernel runs through
its compiled (16, 8) / (32, 16) instantiations (identity / zero pads) against
the path they took before (B2P_FG_PAD=0: cluster / split); iterations checked
against the oracle. python scripts/fg_pad_probe.py [out.json]"""
import json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as orc
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind

cfg = PcgConfig(epsilon=1e-8)
rows = {}
for K, n, m in [(128, 12, 4), (256, 12, 4), (100, 20, 10), (256, 20, 10), (96, 32, 16),
                (200, 9, 3), (129, 4, 12)]:
    kkt = api.random_kkt(7, K - 1, n, m)
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg).report.iterations
    row = {}
    for name, pad in (("padded_grid", "1"), ("before", "0")):
        os.environ["B2P_FG_PAD"] = pad
        ts = []
        for i in range(25):
            r = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
            if i >= 5:
                ts.append(r.report.wall_time * 1e6)
        row[name] = {"us_device_median": round(statistics.median(ts), 1),
                     "path": api.context().last_path(), "iterations_equal": r.report.iterations == want}
    rows[f"K{K}_n{n}_m{m}"] = row
    print(f"K{K}_n{n}_m{m}", json.dumps(row), flush=True)
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fg_pad_probe.json"
json.dump({"what": __doc__.strip().splitlines()[0], "rows": rows}, open(out, "w"), indent=1)
