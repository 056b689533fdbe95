"""Off-BASELINE shapes on the fused one-CTA kernel (k_fused_cta templated over
even n in [8, 16] and m <= 8, the control dimension padded to 4 / 8 with
identity R and zero B, r pads): per-system parity with the oracle (identical
PCG iteration counts, lambda within 1e-10), every preconditioner kind, ragged
horizons, warm start / cap / non-PD messages, build_schur's formation-only
mode and the fused PPCG finish. The reference forms and solves any (n, m) at
runtime (schur.cpp:38-82)."""
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


SHAPES = [(64, 12, 4), (33, 12, 4), (40, 10, 3), (32, 16, 8), (64, 14, 4), (48, 12, 8),
          (20, 16, 2), (64, 10, 6), (17, 14, 8)]


@pytest.mark.parametrize("K,n,m", SHAPES)
def test_batched_one_cta_matches_oracle_per_system(api, orc, env, K, n, m):
    env["B2P_FC"] = "0"
    B = 24
    kb = api.random_kkt_batch(8100 + 31 * n + m + K, B, K - 1, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    lam, reps = api.solve_batched(kb, PrecondKind.symmetric_stair, 1, cfg)
    assert api.context().last_path() == 1  # the one-CTA fused kernel
    _, lo, ro = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, cfg)
    assert np.array_equal(reps.iterations, np.array([r.iterations for r in ro]))
    assert reps.converged.all()
    scale = np.maximum(1.0, np.abs(lo).max(axis=1))
    assert (np.abs(lam - lo).max(axis=1) / scale).max() <= TOL64


@pytest.mark.parametrize("kind", [PrecondKind.block_jacobi, PrecondKind.stair,
                                  PrecondKind.symmetric_stair])
@pytest.mark.parametrize("K,n,m", [(64, 12, 4), (29, 16, 5)])
def test_every_stair_family_kind(api, orc, env, kind, K, n, m):
    env["B2P_FC"] = "0"
    B = 12
    kb = api.random_kkt_batch(8300 + K + n, B, K - 1, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    lam, reps = api.solve_batched(kb, kind, 1, cfg)
    assert api.context().last_path() == 1
    for i in (0, 7, 11):
        want = orc.solve(kb.system(i), kind, cfg=cfg)
        assert reps[i].iterations == want.report.iterations
        assert rel_inf_error(lam[i], want.lambda_) <= TOL64


def test_single_solve_warm_start_cap_errors_and_finish(api, orc):
    """B = 1 at (K 64, n 12, m 4): the single-solve policy picks the one-CTA
    kernel; warm start, iteration cap (best iterate), the non-PD R message with
    the padded control block, build_schur's formation-only output and the
    fused sqp_step finish (one launch) against the oracle."""
    kkt = orc.random_kkt(8401, 63, 12, 4)
    cfg = PcgConfig(epsilon=1e-8)
    got = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert api.context().last_path() == 1
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert got.report.iterations == want.report.iterations
    assert rel_inf_error(got.lambda_, want.lambda_) <= TOL64
    warm = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    ow = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    assert warm.report.iterations == ow.report.iterations
    capped = api.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-14, max_iter=3))
    oc = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-14, max_iter=3))
    assert not capped.report.converged and capped.report.iterations == 3
    assert rel_inf_error(capped.lambda_, oc.lambda_) <= TOL64
    # build_schur (formation-only mode of the same kernel)
    gs, os_ = api.build_schur(kkt), orc.build_schur(kkt)
    assert np.abs(gs.S.data - os_.S.data).max() <= 1e-12 * max(1.0, np.abs(os_.S.data).max())
    assert np.abs(gs.gamma - os_.gamma).max() <= 1e-12 * max(1.0, np.abs(os_.gamma).max())
    # fused PPCG finish: one launch, dz against the oracle's reconstruct_primal
    ctx = api.context()
    before = ctx.kernel_launches()
    res, dz = api.sqp_step(kkt, cfg=cfg)
    assert ctx.kernel_launches() - before == 1
    odz = orc.reconstruct_primal(kkt, want.lambda_)
    assert np.abs(dz - odz).max() / max(1.0, np.abs(odz).max()) <= 1e-9
    bad = orc.random_kkt(8402, 63, 12, 4)
    bad.R[40] = -np.eye(4)
    with pytest.raises(RuntimeError, match="build_schur: R at knot 40 is not positive definite"):
        api.solve(bad)


ODD = [(64, 13, 7), (40, 11, 3), (33, 9, 2), (21, 15, 8), (2, 13, 4)]


@pytest.mark.parametrize("K,n,m", ODD)
def test_odd_n_padded_one_cta_matches_oracle(api, orc, env, K, n, m):
    """Odd n in [9, 15]: the one-CTA kernel on n + 1 with an identity-padded
    state (pad rows of S, theta^-1 and every PCG vector stay exactly zero);
    per-system iteration counts and lambda against the oracle."""
    env["B2P_FC"] = "0"
    B = 20
    kb = api.random_kkt_batch(8600 + 7 * n + K, B, K - 1, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    for kind in (PrecondKind.symmetric_stair, PrecondKind.stair, PrecondKind.block_jacobi):
        lam, reps = api.solve_batched(kb, kind, 1, cfg)
        assert api.context().last_path() == 1
        _, lo, ro = orc.solve_batch(kb, kind, 1, cfg)
        assert np.array_equal(reps.iterations, np.array([r.iterations for r in ro]))
        assert np.array_equal(reps.converged, np.array([bool(r.converged) for r in ro]))
        scale = np.maximum(1.0, np.abs(lo).max(axis=1))
        assert (np.abs(lam - lo).max(axis=1) / scale).max() <= TOL64


def test_odd_n_padded_single_warm_start_cap_and_errors(api, orc):
    kkt = orc.random_kkt(8701, 47, 13, 5)
    cfg = PcgConfig(epsilon=1e-8)
    got = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert got.report.iterations == want.report.iterations
    assert rel_inf_error(got.lambda_, want.lambda_) <= TOL64
    warm = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    ow = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    assert warm.report.iterations == ow.report.iterations
    assert rel_inf_error(warm.lambda_, ow.lambda_) <= TOL64
    capped = api.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-14, max_iter=3))
    oc = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-14, max_iter=3))
    assert not capped.report.converged and capped.report.iterations == 3
    assert rel_inf_error(capped.lambda_, oc.lambda_) <= TOL64
    # non-PD Q at knot 5: the reference's message, knot index unchanged by the pad
    bad = orc.random_kkt(8702, 47, 13, 5)
    bad.Q[5] = -np.eye(13)
    with pytest.raises(RuntimeError, match="build_schur: Q at knot 5 is not positive definite"):
        api.solve(bad, PrecondKind.symmetric_stair, cfg=cfg)


SMALL_N = [(64, 8, 4), (64, 7, 2), (64, 8, 8), (48, 7, 7), (33, 8, 1)]


@pytest.mark.parametrize("K,n,m", SMALL_N)
def test_small_n_long_horizon_batches_on_one_cta(api, orc, env, K, n, m):
    """n = 7, 8 at horizons K > 24: the one-CTA kernel (n = 7 through the
    identity pad to 8) instead of the small-block kernel; every stair-family
    kind against the oracle per system."""
    env["B2P_FC"] = "0"
    B = 20
    kb = api.random_kkt_batch(8800 + 5 * n + m + K, B, K - 1, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    for kind in (PrecondKind.symmetric_stair, PrecondKind.stair, PrecondKind.block_jacobi):
        lam, reps = api.solve_batched(kb, kind, 1, cfg)
        assert api.context().last_path() == 1  # the one-CTA fused kernel
        _, lo, ro = orc.solve_batch(kb, kind, 1, cfg)
        assert np.array_equal(reps.iterations, np.array([r.iterations for r in ro]))
        assert np.array_equal(reps.converged, np.array([bool(r.converged) for r in ro]))
        scale = np.maximum(1.0, np.abs(lo).max(axis=1))
        assert (np.abs(lam - lo).max(axis=1) / scale).max() <= TOL64


def test_small_n_policy_and_n8_single_solve_finish(api, orc, env):
    """Short horizons stay on the small-block kernel; n = 8 single solves at
    K 64 take the one-CTA kernel, with warm start, cap, the fused sqp_step
    finish and the non-PD message; B2P_ONECTA_MIN_N overrides the policy."""
    env["B2P_FC"] = "0"
    kb = api.random_kkt_batch(8901, 8, 16, 8, 4)  # K 17
    api.solve_batched(kb, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
    assert api.context().last_path() != 1
    env["B2P_ONECTA_MIN_N"] = "7"
    lam, reps = api.solve_batched(kb, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
    assert api.context().last_path() == 1
    _, lo, ro = orc.solve_batch(kb, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
    assert np.array_equal(reps.iterations, np.array([r.iterations for r in ro]))
    del env["B2P_ONECTA_MIN_N"]
    kkt = orc.random_kkt(8902, 63, 8, 4)
    cfg = PcgConfig(epsilon=1e-8)
    got = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert api.context().last_path() == 1
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert got.report.iterations == want.report.iterations
    assert rel_inf_error(got.lambda_, want.lambda_) <= TOL64
    warm = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    ow = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=0.5 * want.lambda_)
    assert warm.report.iterations == ow.report.iterations
    capped = api.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-14, max_iter=3))
    oc = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-14, max_iter=3))
    assert not capped.report.converged and capped.report.iterations == 3
    assert rel_inf_error(capped.lambda_, oc.lambda_) <= TOL64
    res, dz = api.sqp_step(kkt, cfg=cfg)
    odz = orc.reconstruct_primal(kkt, want.lambda_)
    assert np.abs(dz - odz).max() / max(1.0, np.abs(odz).max()) <= 1e-9
    bad = orc.random_kkt(8903, 63, 8, 4)
    bad.Q[9] = -np.eye(8)
    with pytest.raises(RuntimeError, match="build_schur: Q at knot 9 is not positive definite"):
        api.solve(bad, PrecondKind.symmetric_stair, cfg=cfg)
