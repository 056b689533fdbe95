"""c1 single-solve latency across the fused variants (one CTA, cluster G, grid rp)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from latency_sweep import orc, timed  # noqa: E402
from paper_2309_08079_b200.types import PrecondKind  # noqa: E402

k1 = orc.random_kkt(1, 31, 14, 7)
out = {"onecta": timed(k1, PrecondKind.symmetric_stair, 1e-8, env={"B2P_FC": "0"})}
for g in (1, 2, 4, 8):
    out[f"cluster{g}"] = timed(k1, PrecondKind.symmetric_stair, 1e-8,
                               env={"B2P_FC": "1", "B2P_FC_G": str(g)})
for k, v in out.items():
    print(k, round(v["us_median"], 1), v["path"], v["iterations"], v["iterations_equal"])
json.dump(out, open("gpurun_out/c1_probe.json", "w"), indent=1)
