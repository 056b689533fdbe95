"""Batched throughput (device-resident, 4096 systems unless noted) of shapes the
fused cluster kernel runs through its compiled (16, 8) instantiation (identity /
zero pads) against the split path they took before (B2P_FC_PAD=0).
python scripts/fc_pad_probe.py [out.json]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2309_08079_b200.api as api

rows = {}
for B, K, n, m in [(4096, 128, 12, 4), (4096, 100, 9, 3), (2048, 256, 16, 8), (4096, 65, 14, 5)]:
    row = {}
    for name, pad in (("padded_cluster", "1"), ("before", "0")):
        os.environ["B2P_FC_PAD"] = pad
        r = bench.nmpc_batch_throughput(api, torch, 0, B=B, N=K - 1, n=n, m=m, reps=3, seed=21)
        row[name] = {"systems_per_s": round(r["systems_per_s"]), "kernel": r["kernel"],
                     "iters_mean": r["iters_mean"]}
    rows[f"B{B}_K{K}_n{n}_m{m}"] = row
    print(f"B{B}_K{K}_n{n}_m{m}", json.dumps(row), flush=True)
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fc_pad_probe.json"
json.dump({"what": __doc__.strip().splitlines()[0], "rows": rows}, open(out, "w"), indent=1)
