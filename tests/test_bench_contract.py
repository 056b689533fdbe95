"""bench.py keeps the driver's JSON-line contract (both arms): one line, the
required keys, consistent units, launches counted, roofline and CPU baseline
present. Small batches so the checks run in seconds."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"]


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--batch", "32"])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_b200_arm_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--batch", "296", "--cpu-seconds", "1"])
    for k in REQUIRED + ["e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks", "latency"]:
        assert k in d, k
    assert d["unit"] == "solves/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["gpu_launches"] >= d["steps"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1 and r["peak"] > 0
    assert r["fp64"]["unit"] == "TFLOP/s" and 0 < r["fp64"]["frac"] < 1
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] <= d["value"] * 1.05
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    for c in ("c1", "c2", "c3", "c5"):
        assert d["latency"][c]["us_median"] > 0
    # the reference's other bench rows and callers: direct baseline, SQP step, NMPC batch
    assert d["dense_baseline"]["all_ok"] and d["dense_baseline"]["max_rel_diff_vs_pcg"] < 1e-3
    assert d["latency"]["sqp_step_n2"]["kernel"] == "fused small"
    assert d["latency"]["nmpc_batch_n2"]["systems_per_s"] > 0
    assert d["roofline"]["onchip"]["l1tex_throughput_pct_of_peak"] > 0
