"""Port of proj/tests/test_pcg.cpp (PCG contracts)."""
import numpy as np
import pytest

from backends import B  # noqa: F401
from paper_2309_08079_b200.types import (BlockTriMatrix, PcgBreakdown, PcgConfig, PcgVariant,
                                         PrecondKind, precond_name)
from util import identity_system, kat


def test_identity_system_one_iteration(B, orc):  # test_pcg.cpp:32-45
    g = kat("pcg_identity_one_iteration")
    S = identity_system(3, 2)
    gamma = orc.UniformRng(g["rng_seed"]).vector(6, *g["gamma_range"])
    for variant in PcgVariant:
        res = B.pcg_solve_auto(S, B.build_identity(), gamma, np.zeros(6),
                               PcgConfig(epsilon=g["epsilon"], variant=variant))
        assert res.report.iterations == g["iterations"]
        assert res.report.converged
        assert np.abs(res.lambda_ - gamma).max() <= g["tol"]


def test_scalar_2x2_within_two_iterations(B):  # :47-60
    g = kat("pcg_scalar_2x2")
    S = BlockTriMatrix(2, 1)
    S.set_diag(0, 2.0 * np.eye(1))
    S.set_diag(1, 2.0 * np.eye(1))
    S.set_right(0, np.eye(1))
    S.set_left(1, np.eye(1))
    res = B.pcg_solve(S, B.build_identity(), np.array(g["gamma"], float), np.zeros(2),
                      PcgConfig(epsilon=g["epsilon"]))
    assert res.report.converged
    assert res.report.iterations <= g["max_iterations"]
    assert np.abs(res.lambda_ - np.array(g["lambda"])).max() <= g["tol"]


@pytest.mark.parametrize("kind", list(PrecondKind), ids=lambda k: precond_name(k, 1))
def test_every_preconditioner_reproduces_dense_solution(B, orc, kind):  # :62-78
    s = B.build_schur(orc.random_trajectory_kkt(101, 8, 3, 2))
    dense = np.linalg.solve(s.S.to_dense(), s.gamma)
    cfg = PcgConfig(epsilon=1e-10, max_iter=10 * s.S.dim())
    P = B.build_preconditioner(s, kind, 1)
    res = B.pcg_solve(s.S, P, s.gamma, np.zeros(s.S.dim()), cfg)
    assert res.report.converged
    assert np.abs(res.lambda_ - dense).max() <= 1e-6


@pytest.mark.parametrize("seed", [201, 202, 203])
def test_block_parallel_trace_matches_sequential(B, orc, seed):  # :80-102
    s = B.build_schur(orc.random_kkt(seed, 8, 3, 2))
    P = B.build_symmetric_stair(s)
    cfg = PcgConfig(epsilon=1e-10, max_iter=4 * s.S.dim(), collect_trace=True,
                    deterministic_reductions=True)
    seq = B.pcg_solve(s.S, P, s.gamma, np.zeros(s.S.dim()), cfg)
    par = B.pcg_solve_block_parallel(s.S, P, s.gamma, np.zeros(s.S.dim()), cfg)
    assert seq.report.iterations == par.report.iterations
    assert seq.report.converged == par.report.converged
    assert len(seq.report.trace) == len(par.report.trace) == seq.report.iterations
    for a, b in zip(seq.report.trace, par.report.trace):
        assert abs(a - b) <= 1e-10 * max(1.0, abs(a), abs(b))


def test_identity_cg_terminates_within_dim_plus_5(B, orc):  # :104-123
    seed, tested = 300, 0
    for _ in range(12):
        s = B.build_schur(orc.random_kkt_scaled(seed, 6, 2, 1, 1.0, 0.5))
        seed += 1
        ev = np.linalg.eigvalsh(s.S.to_dense())
        if ev.max() / ev.min() > 1e3:
            continue
        tested += 1
        cfg = PcgConfig(epsilon=1e-8, max_iter=s.S.dim() + 5)
        res = B.pcg_solve(s.S, B.build_identity(), s.gamma, np.zeros(s.S.dim()), cfg)
        assert res.report.converged
        assert res.report.iterations <= s.S.dim() + 5
    assert tested >= 8


def test_recurrence_residual_tracks_true_residual(B, orc):  # :125-136
    s = B.build_schur(orc.random_kkt(310, 12, 3, 1))
    cfg = PcgConfig(epsilon=1e-8, max_iter=4 * s.S.dim(), check_residual_drift=True)
    res = B.pcg_solve(s.S, B.build_symmetric_stair(s), s.gamma, np.zeros(s.S.dim()), cfg)
    assert res.report.converged
    assert res.report.max_residual_drift <= 1e-6


def test_converged_implies_exit_eta_below_epsilon(B, orc):  # :138-148
    s = B.build_schur(orc.random_kkt(320, 8, 2, 1))
    cfg = PcgConfig(epsilon=1e-6)
    res = B.pcg_solve(s.S, B.build_block_jacobi(s), s.gamma, np.zeros(s.S.dim()), cfg)
    if res.report.converged:
        assert res.report.exit_eta < cfg.epsilon


def test_iteration_cap_returns_best_unconverged(B, orc):  # :150-160
    s = B.build_schur(orc.random_kkt(330, 16, 3, 2))
    res = B.pcg_solve(s.S, B.build_identity(), s.gamma, np.zeros(s.S.dim()),
                      PcgConfig(epsilon=1e-14, max_iter=3))
    assert not res.report.converged
    assert res.report.iterations == 3


def test_indefinite_matrix_breakdown(B):  # :162-171
    S = BlockTriMatrix(2, 1)
    S.set_diag(0, -np.eye(1))
    S.set_diag(1, -np.eye(1))
    with pytest.raises(PcgBreakdown):
        B.pcg_solve(S, B.build_identity(), np.ones(2), np.zeros(2), PcgConfig(epsilon=1e-10))


def test_dimension_mismatch_message(B):  # :173-178
    S = identity_system(3, 2)
    with pytest.raises(ValueError, match="length 6"):
        B.pcg_solve(S, B.build_identity(), np.zeros(5), np.zeros(6), PcgConfig())


def test_warm_start_at_solution_exits_without_iterating(B, orc):  # :180-189
    s = B.build_schur(orc.random_kkt(340, 6, 2, 1))
    exact = np.linalg.solve(s.S.to_dense(), s.gamma)
    res = B.pcg_solve(s.S, B.build_symmetric_stair(s), s.gamma, exact, PcgConfig(epsilon=1e-8))
    assert res.report.converged
    assert res.report.iterations == 0


def test_property_median_iteration_ordering(B, orc):  # :191-217
    it = {k: [] for k in ("identity", "jacobi", "symstair")}
    for trial in range(100):
        s = B.build_schur(orc.random_kkt(1000 + trial, 16, 2, 1))
        cfg = PcgConfig(epsilon=1e-8, max_iter=10 * s.S.dim())
        z = np.zeros(s.S.dim())
        it["identity"].append(B.pcg_solve(s.S, B.build_identity(), s.gamma, z, cfg)
                              .report.iterations)
        it["jacobi"].append(B.pcg_solve(s.S, B.build_block_jacobi(s), s.gamma, z, cfg)
                            .report.iterations)
        it["symstair"].append(B.pcg_solve(s.S, B.build_symmetric_stair(s), s.gamma, z, cfg)
                              .report.iterations)
    med = {k: float(np.median(v)) for k, v in it.items()}
    assert med["symstair"] <= med["jacobi"] <= med["identity"]
    assert med["symstair"] < med["identity"]


def test_property_deeper_splitting_series(B, orc):  # :219-238
    by_order = [[], [], []]
    for trial in range(40):
        s = B.build_schur(orc.random_kkt(2000 + trial, 12, 2, 1))
        cfg = PcgConfig(epsilon=1e-8, max_iter=10 * s.S.dim())
        z = np.zeros(s.S.dim())
        by_order[0].append(B.pcg_solve(s.S, B.build_stair(s), s.gamma, z, cfg).report.iterations)
        for order in (1, 2):
            by_order[order].append(
                B.pcg_solve(s.S, B.build_poly_split(s, order), s.gamma, z, cfg).report.iterations)
    assert np.median(by_order[1]) <= np.median(by_order[0]) + 1
    assert np.median(by_order[2]) <= np.median(by_order[1]) + 1
