import os, sys, statistics, json
sys.path.insert(0, os.getcwd())
import paper_2309_08079_b200.api as api
from paper_2309_08079_b200.types import PcgConfig, PrecondKind
K = int(sys.argv[1])
kkt = api.random_kkt(1, K - 1, 14, 7)
out = {}
for rp in (1, 2, 3, 4, 6, 8):
    os.environ["B2P_FG"] = "1"; os.environ["B2P_FG_RP"] = str(rp)
    try:
        ts = []
        for i in range(35):
            r = api.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-8))
            if i >= 5: ts.append(r.report.wall_time * 1e6)
        out[rp] = (round(statistics.median(ts), 1), api.context().last_path(), r.report.iterations)
    except Exception as e:
        out[rp] = str(e)[:60]
print(K, json.dumps(out))
