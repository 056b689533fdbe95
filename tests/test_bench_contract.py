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
    # the binding roof: FP64 FMA work; the HBM view beside it
    assert r["bound"] == "fp64" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1 and r["peak"] > 0
    assert r["hbm"]["unit"] == "GB/s" and 0 < r["hbm"]["frac"] < 1
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] <= d["value"] * 1.05
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    assert d["clocks"]["samples"] > 0 and d["clocks"]["sm_mhz"] > 0
    p = d["parity"]
    assert p["systems"] >= 256 and p["iterations_equal"] == p["systems"]
    assert p["lambda_rel_err_max"] <= 1e-10
    rows = d["baseline_configs"]
    assert rows["c1"]["symstair_1e-08"]["iterations_equal"]
    for kind in ("jacobi", "stair", "symstair"):
        for eps in ("1e-08", "0.0001"):
            c2 = rows["c2"][f"{kind}_{eps}"]
            assert c2["iterations_equal"] and c2["cpu"]["us_full_scope_1core"] > 0
    assert len(rows["c5"]["kappa_sweep"]) == 12
    assert all(r5["iterations_equal"] for r5 in rows["c5"]["kappa_sweep"])
    assert d["c4_eps_1e-4"]["value"] > d["value"]
    # the reference's other bench rows and callers: direct baseline, SQP step, NMPC batch
    assert d["dense_baseline"]["all_ok"] and d["dense_baseline"]["max_rel_diff_vs_pcg"] < 1e-3
    assert d["latency"]["sqp_step_n2"]["kernel"] == "fused small"
    assert d["latency"]["nmpc_batch_n2"]["systems_per_s"] > 0
    assert d["roofline"]["onchip"]["l1tex_throughput_pct_of_peak"] > 0


def test_reference_arm_multi_rank_launcher():
    """`bench.py --impl reference --gpus 2` without torchrun in the environment
    re-launches itself under torch.distributed.run with two ranks (the path the
    driver's scaling run takes); rank 0 alone prints the one JSON line."""
    d = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
              "--batch", "16", "--ref-budget", "1"], timeout=300)
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
