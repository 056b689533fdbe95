"""The reference's SQP / NMPC / model / KKT-assembly suites (proj/tests/test_sqp.cpp,
test_nmpc.cpp, test_models.cpp, test_kkt.cpp:30-79,144-157) written in C++ against
include/trajopt_b200_sqp.hpp (the hot path's real caller).

CPU: every case with the oracle supplying the linear step (host logic: models,
linearisation, merit line search, warm starts, NMPC loop).
GPU: every case on b2p_sqp_step, plus GPU-vs-oracle parity of whole SQP and
NMPC runs (same PCG iteration count and step length at every SQP iteration)."""
import subprocess

import pytest

from paper_2309_08079_b200 import build as b


def _run(mode):
    exe = b.build_sqp_test()
    out = subprocess.run([exe, mode], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stderr[-4000:]
    assert "checks passed" in out.stdout
    return out.stdout


def test_sqp_nmpc_host_logic_with_oracle_linear_step():
    _run("cpu")


@pytest.mark.gpu
def test_sqp_nmpc_on_gpu_and_parity_with_oracle():
    s = _run("gpu")
    assert s.count("parity ") >= 6
