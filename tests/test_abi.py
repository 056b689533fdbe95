"""CPU-side checks of the C-ABI boundary: the library loads, exports every
entry point include/b2p.h declares, and its host-side generator reproduces
the oracle's (random_problem.cpp) draws bit for bit. No compute calls."""
import os
import re

import numpy as np
import pytest

from paper_2309_08079_b200 import _abi, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "b2p.h")).read()
    return sorted(set(re.findall(r"\b(b2p_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_header_symbol():
    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert L.b2p_abi_version() == _abi.B2P_ABI_VERSION


def test_struct_layouts_match_header():
    import ctypes as C
    assert C.sizeof(_abi.PcgConfigC) == 32
    assert C.sizeof(_abi.SolveReportC) == 40
    assert C.sizeof(_abi.ErrorC) == 16 + 256
    assert C.sizeof(_abi.KktC) == 16 + 9 * 8


@pytest.mark.parametrize("family", [0, 1, 2])
def test_product_generator_matches_oracle_bitwise(orc, family):
    import paper_2309_08079_b200.api as api
    for seed, N, n, m in [(42, 8, 3, 2), (7, 31, 14, 7), (9, 3, 12, 4)]:
        if family == 0:
            a, b = api.random_kkt(seed, N, n, m), orc.random_kkt(seed, N, n, m)
        elif family == 1:
            a = api.random_kkt_scaled(seed, N, n, m, 0.01, 2.0)
            b = orc.random_kkt_scaled(seed, N, n, m, 0.01, 2.0)
        else:
            a, b = api.random_trajectory_kkt(seed, N, n, m), orc.random_trajectory_kkt(seed, N, n, m)
        for x, y in zip(a.arrays(), b.arrays()):
            assert np.array_equal(x, y)


def test_batch_generator_uses_seed0_plus_i(orc):
    import paper_2309_08079_b200.api as api
    kb = api.random_kkt_batch(1000, 5, 7, 4, 2, threads=3)
    for i in range(5):
        one = orc.random_kkt(1000 + i, 7, 4, 2)
        for x, y in zip(kb.system(i).arrays(), one.arrays()):
            assert np.array_equal(x, y)


def test_no_device_means_loud_failure():
    import paper_2309_08079_b200.api as api
    if api.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError):
        api.require_device()
    with pytest.raises(Exception):
        api.context()


def test_argument_validation_before_any_device_work():
    """Entry points added for the SQP caller and the direct baseline reject bad
    arguments with INVALID_ARGUMENT and the message, before touching a device."""
    import ctypes as C
    L = _lib.load()
    err = _abi.ErrorC()
    assert L.b2p_direct_solve_batched_device(None, 0, 1, None, None, None, C.byref(err)) == 1
    assert b"kkt" in err.message
    assert L.b2p_uniform_draws(1, -1, 0.0, 1.0, None, C.byref(err)) == 1
    assert b"uniform_draws" in err.message
    out = np.zeros(4)
    assert L.b2p_uniform_draws(7, 4, -1.0, 1.0, out.ctypes.data, C.byref(err)) == 0
    assert np.all(np.abs(out) <= 1.0) and len(set(out.tolist())) == 4
