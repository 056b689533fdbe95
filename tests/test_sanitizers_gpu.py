"""compute-sanitizer over one small solve on every kernel path (race
detection). racecheck: no shared-memory hazards (the edge rows' discarded
neighbour products used to read the next array while other warps wrote it);
memcheck: no out-of-bounds or misaligned accesses, no leaks of device errors."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["racecheck", "memcheck"])
def test_every_kernel_path_is_sanitizer_clean(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    out = subprocess.run([cs, "--tool", tool, "--print-limit", "20", sys.executable,
                          os.path.join(ROOT, "scripts", "sanitize_paths.py")],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    text = out.stdout + out.stderr
    if "closed on this pool" in text:
        # the GPU pool's compute-sanitizer wrapper refuses every run (runs under it
        # left GPUs needing a reset); the logs of the last permitted runs over
        # these paths are profiles/r02_sanitizer_{racecheck,memcheck,synccheck}.log
        pytest.skip("compute-sanitizer closed on this GPU pool; see profiles/r02_sanitizer_*.log")
    assert out.returncode == 0, text[-3000:]
    for path in ("one-CTA fused", "fused grid", "fused cluster", "small-block", "split",
                 "batched one-CTA"):
        assert path in text
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards" in text, text[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in text, text[-3000:]
