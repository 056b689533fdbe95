"""Small-block kernel vs the one-CTA kernel (n padded to 8) for n <= 8 shapes:
4096-system device-resident batches (K = 64) and single solves, with parity
against the oracle; B2P_ONECTA_MIN_N selects the route (10: small-block, 7:
one-CTA for n in {7, 8})."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2309_08079_b200.api as api

out = {}
for n, m in ((7, 2), (8, 4), (8, 8), (7, 7)):
    for floor in ("10", "7"):
        os.environ["B2P_ONECTA_MIN_N"] = floor
        r = bench.shape_batch(api, torch, 0, 4096, 63, n, m, reps=5, check=64)
        key = f"n{n}_m{m}_K64_{'small' if floor == '10' else 'onecta'}"
        out[key] = {k: r[k] for k in ("systems_per_s", "ms_per_batch", "kernel", "iters_mean", "parity")}
        # single solve (device latency through the batched path with B = 1)
        r1 = bench.nmpc_batch_throughput(api, torch, 0, B=1, N=63, n=n, m=m, reps=20, seed=5)
        out[key]["single_us"] = r1["ms_per_batch"] * 1e3
        print(key, json.dumps(out[key]), flush=True)
print(json.dumps(out))
