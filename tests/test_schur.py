"""Port of proj/tests/test_schur.cpp (Schur formation, preconditioner family)."""
import numpy as np
import pytest

from backends import B  # noqa: F401
from paper_2309_08079_b200.types import BlockTriMatrix, KKTSystem, PrecondKind
from util import (dense_schur_matrix, dense_schur_rhs, kat, scalar_spd_2block, standard_batch,
                  wrap)


def test_build_schur_scalar_blocks_by_hand(B):  # test_schur.cpp:41-66
    g = kat("schur_scalar_by_hand")
    one = np.ones((1, 1, 1))
    z = np.zeros((1, 1))
    kkt = KKTSystem(1, 1, 1, Q=np.ones((2, 1, 1)), q=np.zeros((2, 1)), R=one.copy(),
                    r=z.copy(), A=one.copy(), B=one.copy(), e=z.copy(), x_s=np.zeros(1),
                    x0=np.zeros(1))
    s = B.build_schur(kkt)
    assert s.S.diag(1)[0, 0] == pytest.approx(g["theta"])
    assert s.S.left(1)[0, 0] == pytest.approx(g["phi"])
    assert s.S.right(0)[0, 0] == pytest.approx(g["phi"])
    assert np.abs(s.gamma).max() == g["gamma_inf"]


def test_build_schur_matches_dense_formula(B, orc):  # :68-75
    kkt = orc.random_kkt(42, 8, 3, 2)
    s = B.build_schur(kkt)
    assert np.abs(s.S.to_dense() - dense_schur_matrix(kkt)).max() <= 1e-10
    assert np.abs(s.gamma - dense_schur_rhs(kkt)).max() <= 1e-10


def test_assembled_S_is_spd_and_structurally_symmetric(B, orc):  # :77-85
    for seed, N, n, m in standard_batch(12):
        s = B.build_schur(orc.random_kkt(seed, N, n, m))
        assert s.S.max_asymmetry() <= 1e-12
        assert np.linalg.eigvalsh(s.S.to_dense()).min() > 0.0


class TestBlockJacobi:  # :87-111
    def test_identity_blocks_invert_to_identity(self, B):
        S = BlockTriMatrix(3, 2)
        for i in range(3):
            S.set_diag(i, np.eye(2))
        P = B.build_block_jacobi(wrap(S))
        assert np.abs(P.phi_inv.to_dense() - np.eye(6)).max() == 0.0

    def test_scalar_diag(self, B):
        g = kat("jacobi_scalar")
        S = BlockTriMatrix(2, 1)
        S.set_diag(0, g["diag"][0] * np.eye(1))
        S.set_diag(1, g["diag"][1] * np.eye(1))
        P = B.build_block_jacobi(wrap(S))
        assert P.phi_inv.diag(0)[0, 0] == pytest.approx(g["phi_inv_diag"][0])
        assert P.phi_inv.diag(1)[0, 0] == pytest.approx(g["phi_inv_diag"][1])

    def test_multiply_back(self, B, orc):
        s = B.build_schur(orc.random_kkt(51, 6, 3, 2))
        P = B.build_block_jacobi(s)
        for row in range(s.S.block_rows()):
            prod = P.phi_inv.diag(row) @ s.S.diag(row)
            assert np.abs(prod - np.eye(3)).max() <= 1e-12


class TestStair:  # :113-145
    def test_2block_scalar_by_hand(self, B):
        g = kat("stair_2x2")
        schur = wrap(scalar_spd_2block())
        psi = B.stair_matrix(schur.S)
        assert np.abs(psi.to_dense() - np.array(g["psi"], float)).max() == 0.0
        P = B.build_stair(schur)
        assert np.abs(P.phi_inv.to_dense() - np.array(g["phi_inv"], float)).max() <= g["tol"]

    def test_block_diagonal_degenerates_to_jacobi(self, B, orc):
        S = BlockTriMatrix(4, 2)
        rng = orc.UniformRng(8)
        for i in range(4):
            L = rng.matrix(2, 2, -1.0, 1.0)
            S.set_diag(i, L @ L.T + 0.5 * np.eye(2))
        schur = wrap(S)
        st, jac = B.build_stair(schur), B.build_block_jacobi(schur)
        assert np.abs(st.phi_inv.to_dense() - jac.phi_inv.to_dense()).max() == 0.0

    def test_analytic_inverse_matches_dense_inverse(self, B, orc):
        s = B.build_schur(orc.random_kkt(61, 8, 2, 1))
        P = B.build_stair(s)
        psi = B.stair_matrix(s.S).to_dense()
        assert np.abs(np.linalg.inv(psi) - P.phi_inv.to_dense()).max() <= 1e-9


class TestSymmetricStair:  # :147-171
    def test_2block_scalar_mirrors_stair(self, B):
        g = kat("symstair_2x2")
        P = B.build_symmetric_stair(wrap(scalar_spd_2block()))
        assert np.abs(P.phi_inv.to_dense() - np.array(g["phi_inv"], float)).max() <= g["tol"]

    def test_block_diagonal_gives_jacobi(self, B):
        S = BlockTriMatrix(5, 1)
        for i in range(5):
            S.set_diag(i, (i + 1.0) * np.eye(1))
        schur = wrap(S)
        sym, jac = B.build_symmetric_stair(schur), B.build_block_jacobi(schur)
        assert np.abs(sym.phi_inv.to_dense() - jac.phi_inv.to_dense()).max() == 0.0

    def test_symmetric_on_assembled_systems(self, B, orc):
        s = B.build_schur(orc.random_kkt(62, 10, 3, 2))
        P = B.build_symmetric_stair(s)
        assert P.phi_inv.max_asymmetry() <= 1e-12
        d = P.phi_inv.to_dense()
        assert np.abs(d - d.T).max() <= 1e-12


class TestApplyPreconditioner:  # :173-207
    def test_identity_returns_input(self, B, orc):
        r = orc.UniformRng(9).vector(7, -1.0, 1.0)
        assert np.abs(B.apply_preconditioner(B.build_identity(), r) - r).max() == 0.0

    def test_block_jacobi_scalar(self, B):
        g = kat("apply_jacobi_scalar")
        S = BlockTriMatrix(2, 1)
        S.set_diag(0, 2.0 * np.eye(1))
        S.set_diag(1, 4.0 * np.eye(1))
        P = B.build_block_jacobi(wrap(S))
        out = B.apply_preconditioner(P, np.array(g["r"], float))
        assert out[0] == pytest.approx(g["out"][0]) and out[1] == pytest.approx(g["out"][1])

    def test_poly_order1_equals_dense_expansion(self, B, orc):
        s = B.build_schur(orc.random_kkt(63, 6, 2, 1))
        P = B.build_poly_split(s, 1)
        W = B.build_stair(s).phi_inv.to_dense()
        E = B.stair_matrix(s.S).to_dense() - s.S.to_dense()
        r = orc.UniformRng(64).vector(s.S.dim(), -1.0, 1.0)
        want = (np.eye(W.shape[0]) + W @ E) @ (W @ r)
        assert np.abs(B.apply_preconditioner(P, r) - want).max() <= 1e-10

    def test_order_must_be_at_least_one(self, B, orc):
        s = B.build_schur(orc.random_kkt(65, 3, 2, 1))
        with pytest.raises(ValueError):
            B.build_poly_split(s, 0)


def test_property_preconditioner_application_is_linear(B, orc):  # :209-223
    s = B.build_schur(orc.random_kkt(71, 7, 3, 2))
    rng = orc.UniformRng(72)
    x = rng.vector(s.S.dim(), -1.0, 1.0)
    y = rng.vector(s.S.dim(), -1.0, 1.0)
    a, b = 1.3, -0.7
    for kind in PrecondKind:
        P = B.build_preconditioner(s, kind, 2)
        lhs = B.apply_preconditioner(P, a * x + b * y)
        rhs = a * B.apply_preconditioner(P, x) + b * B.apply_preconditioner(P, y)
        assert np.abs(lhs - rhs).max() <= 1e-10


def test_property_stair_inverse_exact_across_sizes(B, orc):  # :225-236
    seed = 80
    for N in (1, 2, 4, 9, 16, 32):
        for n in (1, 2, 3, 4):
            s = B.build_schur(orc.random_kkt(seed, N, n, 1))
            seed += 1
            P = B.build_stair(s)
            prod = B.stair_matrix(s.S).to_dense() @ P.phi_inv.to_dense()
            assert np.abs(prod - np.eye(prod.shape[0])).max() <= 1e-9
