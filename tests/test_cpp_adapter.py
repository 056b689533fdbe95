"""The C++ adapter (include/trajopt_b200.hpp) builds against libb2p.so and, on a
B200, passes the reference's own test cases written in C++."""
import os
import subprocess

import pytest

from paper_2309_08079_b200 import build as b


def test_adapter_compiles_and_links():
    exe = b.build_adapter_test(force=True)
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_adapter_reference_cases_on_gpu():
    exe = b.build_adapter_test()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert "all checks passed" in out.stdout
