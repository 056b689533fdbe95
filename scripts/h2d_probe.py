"""Raw pinned H2D bandwidth on the box vs the e2e batched path at several chunk sizes."""
import json, os, subprocess, sys, time
import torch
x = torch.empty(1192755200 // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty_like(x, device="cuda")
for _ in range(2):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"raw_h2d_GBs": x.numel() * 8 / ms / 1e6, "ms": ms}))
# 9 separate chunks (like upload_kkt)
parts = torch.chunk(x, 36)
dp = torch.chunk(d, 36)
e0.record()
for a, b in zip(parts, dp):
    b.copy_(a, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"chunked36_h2d_GBs": x.numel() * 8 / e0.elapsed_time(e1) / 1e6}))
del d, x
for ch in (256, 512, 1024, 2048):
    env = dict(os.environ, B2P_BATCH_CHUNK=str(ch))
    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-latency"],
                         env=env, capture_output=True, text=True).stdout.strip().splitlines()[-1]
    dd = json.loads(out)
    print(json.dumps({"chunk": ch, "e2e": dd["e2e"]["value"], "value": dd["value"]}))
