"""Single long-horizon solves (and batches of <= 8) of shapes the fused grid
kernel is not compiled for: fp64 n <= 32, m <= 16 run on the compiled (16, 8)
or (32, 16) kernel through an identity-padded Q / R and zero pads elsewhere
(every pad entry of S, gamma, theta^-1 and the PCG vectors stays exactly 0).
Per-system parity with the oracle: identical iteration counts, lambda within
1e-10. The reference forms and solves any (n, m) (schur.cpp:38-82)."""
import os

import numpy as np
import pytest

from paper_2309_08079_b200.types import PcgConfig, PrecondKind
from util import rel_inf_error

pytestmark = pytest.mark.gpu
TOL64 = 1e-10


@pytest.fixture(scope="module")
def api():
    import paper_2309_08079_b200.api as a
    a.require_device()
    return a


@pytest.fixture
def env():
    saved = dict(os.environ)
    yield os.environ
    os.environ.clear()
    os.environ.update(saved)


SHAPES = [(128, 12, 4), (100, 20, 10), (200, 9, 3), (96, 32, 16), (65, 16, 8), (150, 24, 5),
          (90, 16, 12)]


@pytest.mark.parametrize("K,n,m", SHAPES)
def test_padded_grid_single_solve_matches_oracle(api, orc, K, n, m):
    kkt = orc.random_kkt(9100 + K + n + m, K - 1, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    for kind in (PrecondKind.symmetric_stair, PrecondKind.stair, PrecondKind.block_jacobi):
        got = api.solve(kkt, kind, cfg=cfg)
        assert api.context().last_path() == 3  # the fused grid kernel
        want = orc.solve(kkt, kind, cfg=cfg)
        assert got.report.iterations == want.report.iterations, kind
        assert got.report.converged == want.report.converged
        assert rel_inf_error(got.lambda_, want.lambda_) <= TOL64


def test_padded_grid_warm_start_cap_trace_and_errors(api, orc):
    kkt = orc.random_kkt(9201, 119, 20, 10)
    cfg = PcgConfig(epsilon=1e-8)
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    warm = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    ow = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    assert api.context().last_path() == 3
    assert warm.report.iterations == ow.report.iterations
    assert rel_inf_error(warm.lambda_, ow.lambda_) <= TOL64
    cap = PcgConfig(epsilon=1e-14, max_iter=4)
    capped = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cap)
    oc = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cap)
    assert not capped.report.converged and capped.report.iterations == 4
    assert rel_inf_error(capped.lambda_, oc.lambda_) <= TOL64
    bad = orc.random_kkt(9202, 119, 20, 10)
    bad.R[33] = -np.eye(10)
    with pytest.raises(RuntimeError, match="build_schur: R at knot 33 is not positive definite"):
        api.solve(bad, PrecondKind.symmetric_stair, cfg=cfg)


def test_padded_grid_small_batch(api, orc, env):
    env["B2P_FC"] = "0"
    kb = api.random_kkt_batch(9301, 4, 79, 24, 12)
    cfg = PcgConfig(epsilon=1e-8)
    lam, reps = api.solve_batched(kb, PrecondKind.symmetric_stair, 1, cfg)
    assert api.context().last_path() == 3
    _, lo, ro = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, cfg)
    assert np.array_equal(reps.iterations, np.array([r.iterations for r in ro]))
    scale = np.maximum(1.0, np.abs(lo).max(axis=1))
    assert (np.abs(lam - lo).max(axis=1) / scale).max() <= TOL64


def test_padding_policy_keeps_tiny_states_off_the_wide_kernel(api, orc):
    """n = 4, m = 12 would pad to (32, 16) (8x the state): measured slower than
    the split path, so it stays there; the result still matches the oracle."""
    kkt = orc.random_kkt(9401, 128, 4, 12)
    cfg = PcgConfig(epsilon=1e-8)
    got = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert api.context().last_path() != 3
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert got.report.iterations == want.report.iterations
    assert rel_inf_error(got.lambda_, want.lambda_) <= TOL64


@pytest.mark.parametrize("N,n,m", [(20, 4, 12), (20, 6, 10), (40, 3, 9), (16, 2, 7)])
def test_split_path_control_wider_than_state(api, orc, env, N, n, m):
    """m > n on the split K1: the R_k factorisation scratch must hold an m x m
    tile (it overflowed into the gamma vectors: S and theta^-1 were right,
    gamma and lambda were not); build_schur and the solve against the oracle."""
    env["B2P_FUSED"] = "0"
    kkt = orc.random_kkt(9500 + N + n + m, N, n, m)
    gs, os_ = api.build_schur(kkt), orc.build_schur(kkt)
    assert np.abs(gs.S.data - os_.S.data).max() <= 1e-12 * max(1.0, np.abs(os_.S.data).max())
    assert np.abs(gs.gamma - os_.gamma).max() <= 1e-12 * max(1.0, np.abs(os_.gamma).max())
    cfg = PcgConfig(epsilon=1e-8)
    got = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert got.report.iterations == want.report.iterations
    assert rel_inf_error(got.lambda_, want.lambda_) <= TOL64


@pytest.mark.parametrize("K,n,m,B", [(128, 12, 4, 24), (100, 11, 3, 16), (256, 16, 8, 12),
                                     (65, 14, 5, 20), (80, 15, 8, 9)])
def test_padded_cluster_batches_match_oracle(api, orc, K, n, m, B):
    """Batches of n in [11, 16], m <= 8 at horizons the one-CTA kernel cannot
    hold (K > 64): the cluster kernel compiled at (16, 8) through the same
    identity / zero pads; per-system iteration counts and lambda."""
    kb = api.random_kkt_batch(9600 + K + n + m, B, K - 1, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    for kind in (PrecondKind.symmetric_stair, PrecondKind.block_jacobi):
        lam, reps = api.solve_batched(kb, kind, 1, cfg)
        assert api.context().last_path() == 2  # the fused cluster kernel
        _, lo, ro = orc.solve_batch(kb, kind, 1, cfg)
        assert np.array_equal(reps.iterations, np.array([r.iterations for r in ro]))
        scale = np.maximum(1.0, np.abs(lo).max(axis=1))
        assert (np.abs(lam - lo).max(axis=1) / scale).max() <= TOL64


def test_split_path_large_blocks_long_horizon_batch_and_error_isolation(api, orc):
    """B = 9 systems of K 201, n 27, m 16 (beyond every fused kernel): the split
    PCG's vector slices exceed one CTA's shared memory unstaged too, so it runs
    on a cluster; then an unrelated fp32 solve on the same context (a failed
    launch must never surface in the next call)."""
    kb = api.random_kkt_batch(9701, 9, 200, 27, 16)
    cfg = PcgConfig(epsilon=1e-8)
    lam, reps = api.solve_batched(kb, PrecondKind.symmetric_stair, 1, cfg)
    _, lo, ro = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, cfg)
    assert np.array_equal(reps.iterations, np.array([r.iterations for r in ro]))
    scale = np.maximum(1.0, np.abs(lo).max(axis=1))
    assert (np.abs(lam - lo).max(axis=1) / scale).max() <= TOL64
    k32 = orc.random_kkt(9702, 63, 11, 4)
    got = api.solve(k32, PrecondKind.stair, cfg=PcgConfig(epsilon=1e-4), dtype=np.float32)
    want = orc.solve(k32, PrecondKind.stair, cfg=PcgConfig(epsilon=1e-4))
    assert abs(got.report.iterations - want.report.iterations) <= 1


def test_randomised_shapes_every_path(api, orc):
    """scripts/shape_fuzz.py's sweep, bounded: (N, n, m, B, kind, dtype) drawn
    across every kernel path's bounds; each system against the oracle."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "shape_fuzz.py"), "60", "11"],
                         capture_output=True, text=True, timeout=900)
    import json
    last = json.loads(out.stdout.strip().splitlines()[-1])
    assert last["failed"] == 0, last["bad"]
    assert len(last["paths"]) >= 4, last["paths"]  # the sweep reached most kernel paths


def test_randomised_shapes_rest_of_the_api(api, orc):
    """scripts/api_fuzz.py, bounded: build_schur, build / apply_preconditioner,
    the explicit-Phi pcg_solve_auto, reconstruct_primal and sqp_step over
    random (N, n <= 32, m <= 16) against the oracle."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "scripts", "api_fuzz.py"), "30", "12"],
                         capture_output=True, text=True, timeout=900)
    last = json.loads(out.stdout.strip().splitlines()[-1])
    assert last["failed"] == 0, last["bad"]
