"""The small-block fused kernel (csrc/small_kernels.cu: n, m <= 8 padded to
{1, 2, 4, 8}, one CTA per system, all in shared memory) against the oracle:
every preconditioner, padded and exact block sizes, ragged horizons down to
K = 1, warm starts, the iteration cap, traces, batches and every build_schur /
PCG error path. These are the shapes of the reference's SQP / NMPC callers."""
import numpy as np
import pytest

from paper_2309_08079_b200.types import PcgConfig, PcgVariant, PrecondKind
from test_parity_gpu import TOL64, _cmp, api, env  # noqa: F401
from util import rel_inf_error

pytestmark = pytest.mark.gpu

KINDS = [PrecondKind.identity, PrecondKind.block_jacobi, PrecondKind.stair,
         PrecondKind.symmetric_stair]


def _check(api, orc, kkt, kind, cfg, lambda0=None):
    got = api.solve(kkt, kind, cfg=cfg, lambda0=lambda0)
    assert api.context().last_path() == 4
    want = orc.solve(kkt, kind, cfg=cfg, lambda0=lambda0)
    if kind in (PrecondKind.identity, PrecondKind.block_jacobi) and want.report.iterations > 20:
        # documented +-1 policy for long unpreconditioned CG runs
        par = orc.solve(kkt, kind, cfg=PcgConfig(epsilon=cfg.epsilon, max_iter=cfg.max_iter,
                                                 variant=PcgVariant.block_parallel,
                                                 deterministic_reductions=True),
                        lambda0=lambda0)
        refs = (want.report.iterations, par.report.iterations)
        assert min(abs(got.report.iterations - r) for r in refs) <= 1, (got.report.iterations, refs)
        sch = orc.build_schur(kkt)
        res = lambda x: float(np.linalg.norm(sch.gamma - sch.S.to_dense() @ x))  # noqa: E731
        assert res(got.lambda_) <= 10.0 * max(res(want.lambda_), np.sqrt(cfg.epsilon))
    else:
        _cmp(got, want, TOL64, cfg.epsilon)
    return got, want


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("shape", [(32, 2, 1), (32, 4, 1), (128, 4, 1), (16, 3, 2),
                                   (20, 5, 3), (12, 8, 8), (9, 1, 1), (40, 2, 4), (7, 6, 5)])
def test_small_kernel_matches_oracle(api, orc, kind, shape):
    N, n, m = shape
    kkt = orc.random_kkt(1000 + 31 * N + 7 * n + m, N, n, m)
    _check(api, orc, kkt, kind, PcgConfig(epsilon=1e-8))


@pytest.mark.parametrize("shape", [(999, 2, 1), (2047, 1, 1), (400, 8, 4)])
def test_small_kernel_long_horizons(api, orc, shape):
    """Long horizons: more rows than threads (strided rows), unstaged knot data, or
    beyond the shared-memory bound (then the split path takes over, still exact)."""
    N, n, m = shape
    kkt = orc.random_trajectory_kkt(5 + N, N, n, m)
    cfg = PcgConfig(epsilon=1e-10)
    got = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    _cmp(got, want, TOL64, cfg.epsilon)


@pytest.mark.parametrize("N", [0, 1, 2, 31, 32, 33, 64, 200])
def test_small_kernel_ragged_horizons(api, orc, N):
    """K = N + 1 around the 32-group trip boundaries, down to the single knot."""
    kkt = orc.random_trajectory_kkt(77 + N, N, 4, 2)
    _check(api, orc, kkt, PrecondKind.symmetric_stair, PcgConfig(epsilon=1e-10))


def test_small_kernel_warm_start_cap_trace(api, orc):
    kkt = orc.random_kkt(5, 40, 4, 1)
    cfg = PcgConfig(epsilon=1e-10, collect_trace=True)
    base = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    l0 = 0.9 * base.lambda_
    got, want = _check(api, orc, kkt, PrecondKind.symmetric_stair, cfg, lambda0=l0)
    np.testing.assert_allclose(got.report.trace, want.report.trace, rtol=1e-6)
    # converged warm start: 0 iterations, lambda returned unchanged
    got0 = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg, lambda0=base.lambda_)
    assert got0.report.iterations == 0 and got0.report.converged
    assert np.array_equal(got0.lambda_, base.lambda_)
    # cap: unconverged -> best iterate, iterations == cap
    cap = PcgConfig(epsilon=1e-30, max_iter=3)
    gc = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cap)
    wc = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=cap)
    assert gc.report.iterations == 3 and not gc.report.converged
    assert rel_inf_error(gc.lambda_, wc.lambda_) <= TOL64


def test_small_kernel_batched_persistent(api, orc):
    """More systems than resident CTAs: the persistent loop over the batch."""
    B, N, n, m = 700, 32, 2, 1
    kb = api.random_kkt_batch(4000, B, N, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    lam, reps = api.solve_batched(kb, PrecondKind.symmetric_stair, cfg=cfg)
    assert api.context().last_path() == 4
    for i in (0, 1, 347, 699):
        want = orc.solve(kb.system(i), PrecondKind.symmetric_stair, cfg=cfg)
        assert reps[i].iterations == want.report.iterations
        assert rel_inf_error(lam[i], want.lambda_) <= TOL64


def test_small_kernel_error_paths(api, orc):
    def fresh():  # astype() does not copy arrays that are already f64 + contiguous
        return orc.random_kkt(9, 20, 4, 2)
    bad = fresh()
    bad.Q[0] = -np.eye(4)
    with pytest.raises(RuntimeError, match="build_schur: Q at knot 0 is not positive definite"):
        api.solve(bad)
    bad = fresh()
    bad.Q[7] = -np.eye(4)  # first used in row 7 as Q_{k+1}
    with pytest.raises(RuntimeError, match="build_schur: Q at knot 7 is not positive definite"):
        api.solve(bad)
    bad = fresh()
    bad.R[12] = -np.eye(2)
    with pytest.raises(RuntimeError, match="build_schur: R at knot 12 is not positive definite"):
        api.solve(bad)
    bad = fresh()
    bad.A[5] *= 1e3  # theta_6 = A Q^-1 A' + ... stays SPD; break it through Q_6 instead
    bad.Q[6] = np.diag([1.0, 1.0, 1.0, -1e-3])
    with pytest.raises(RuntimeError, match="build_schur: Q at knot 6 is not positive definite"):
        api.solve(bad)
    bad = fresh()
    bad.q[3, 1] = np.nan
    with pytest.raises(RuntimeError, match="non-finite"):
        api.solve(bad)


def test_small_kernel_agrees_with_split_path(api, orc, env):
    kkt = orc.random_kkt(21, 64, 4, 1)
    cfg = PcgConfig(epsilon=1e-10)
    small = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert api.context().last_path() == 4
    env["B2P_SMALL"] = "0"
    split = api.solve(kkt, PrecondKind.symmetric_stair, cfg=cfg)
    assert api.context().last_path() == 0
    assert small.report.iterations == split.report.iterations
    assert rel_inf_error(small.lambda_, split.lambda_) <= TOL64
