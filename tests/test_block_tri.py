"""Port of proj/tests/test_block_tri.cpp (BlockTriMatrix storage, matvec, checks)."""
import numpy as np
import pytest

from backends import B  # noqa: F401  (fixture)
from paper_2309_08079_b200.types import BlockTriMatrix
from util import kat, random_block_tri, rel_inf_error


def test_matvec_identity_case(B):  # test_block_tri.cpp:13-22
    g = kat("matvec_identity")
    M = BlockTriMatrix(3, 1)
    for i in range(3):
        M.set_diag(i, np.eye(1))
    y = B.matvec(M, np.array(g["x"], dtype=float))
    assert list(y) == g["y"]


def test_matvec_scalar_tridiagonal_by_hand(B):  # :24-34
    g = kat("matvec_scalar_tridiagonal")
    M = BlockTriMatrix(2, 1)
    M.set_diag(0, 2.0 * np.eye(1))
    M.set_diag(1, 2.0 * np.eye(1))
    M.set_right(0, np.eye(1))
    M.set_left(1, np.eye(1))
    y = B.matvec(M, np.ones(2))
    assert np.allclose(y, g["y"], rtol=0, atol=g["tol"])


def test_matvec_agrees_with_dense(B, orc):  # :36-43
    M = random_block_tri(orc.UniformRng(7), 8, 3)
    x = orc.UniformRng(99).vector(M.dim(), -1.0, 1.0)
    assert np.abs(B.matvec(M, x) - M.to_dense() @ x).max() <= 1e-12


def test_matvec_dimension_mismatch_message(B, orc):  # :45-50
    M = random_block_tri(orc.UniformRng(3), 4, 2)
    with pytest.raises(ValueError, match="expected vector of length 8"):
        B.matvec(M, np.zeros(5))


def test_to_dense_trivial_cases():  # :52-68
    M = BlockTriMatrix(1, 2)
    M.set_diag(0, np.eye(2))
    assert np.array_equal(M.to_dense(), np.eye(2))
    M = BlockTriMatrix(2, 1)
    M.set_diag(0, 2.0 * np.eye(1))
    M.set_diag(1, 2.0 * np.eye(1))
    M.set_right(0, np.eye(1))
    M.set_left(1, np.eye(1))
    assert np.array_equal(M.to_dense(), np.array(kat("to_dense_scalar_2block")["dense"], float))


def test_from_dense_round_trip_is_exact(orc):  # :70-75
    M = random_block_tri(orc.UniformRng(21), 6, 3)
    dense = M.to_dense()
    assert np.array_equal(BlockTriMatrix.from_dense(dense, 3).to_dense(), dense)


def test_symmetry_check(B, orc):  # :77-89
    M = random_block_tri(orc.UniformRng(4), 4, 2, symmetric=True)
    assert B.max_asymmetry(M) == 0.0
    M = BlockTriMatrix(2, 1)
    M.set_diag(0, np.eye(1))
    M.set_diag(1, np.eye(1))
    M.set_right(0, np.eye(1))
    assert B.max_asymmetry(M) == pytest.approx(kat("asymmetry_gap")["value"])


def test_boundary_padding_rejects_mutation():  # :91-95
    M = BlockTriMatrix(3, 2)
    with pytest.raises(ValueError):
        M.set_left(0, np.eye(2))
    with pytest.raises(ValueError):
        M.set_right(2, np.eye(2))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_block_cholesky_matches_dense(B, orc, seed):  # :97-106
    kkt = orc.random_kkt(seed, 9, 3, 2)
    s = orc.build_schur(kkt)
    x = B.cholesky_solve(s.S, s.gamma)
    want = np.linalg.solve(s.S.to_dense(), s.gamma)
    assert rel_inf_error(x, want) <= 1e-10


def test_block_cholesky_rejects_indefinite(B):  # :108-113
    M = BlockTriMatrix(2, 1)
    M.set_diag(0, -np.eye(1))
    M.set_diag(1, np.eye(1))
    with pytest.raises(RuntimeError):
        B.cholesky_solve(M, np.ones(2))


def test_property_matvec_matches_dense_across_sizes(B, orc):  # :115-127
    seed = 500
    for rows in (1, 2, 3, 5, 9, 17, 32):
        for nb in (1, 2, 3, 6):
            M = random_block_tri(orc.UniformRng(seed), rows, nb)
            seed += 1
            x = orc.UniformRng(seed * 31 + 1).vector(M.dim(), -1.0, 1.0)
            assert rel_inf_error(B.matvec(M, x), M.to_dense() @ x) <= 1e-12


@pytest.mark.gpu
def test_direct_solve_batched_device_matches_cholesky_and_pcg(orc):
    """b2p_direct_solve_batched_device (the bench's dense_baseline row): per system
    the same lambda as the single-system cholesky_solve and a tight PCG solve."""
    import torch
    import paper_2309_08079_b200.api as api
    from paper_2309_08079_b200.types import KKTSystem, PcgConfig
    api.require_device()
    for (Bn, N, n, m) in [(5, 31, 14, 7), (3, 20, 4, 2)]:
        kb = api.random_kkt_batch(321 + n, Bn, N, n, m)
        dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in kb.arrays()]
        kd = KKTSystem(N, n, m, *dev)
        D = (N + 1) * n
        lam = torch.empty((Bn, D), dtype=torch.float64, device="cuda")
        st = torch.empty((Bn,), dtype=torch.int32, device="cuda")
        api.direct_solve_batched_device(kd, lam.data_ptr(), st.data_ptr(), Bn)
        torch.cuda.synchronize()
        assert (st.cpu().numpy() == -1).all()
        got = lam.cpu().numpy()
        for i in range(Bn):
            sch = orc.build_schur(kb.system(i))
            want = orc.cholesky_solve(sch.S, sch.gamma)
            assert np.abs(got[i] - want).max() / max(1.0, np.abs(want).max()) <= 1e-10
            tight = orc.solve(kb.system(i), cfg=PcgConfig(epsilon=1e-20, max_iter=2000))
            assert np.abs(got[i] - tight.lambda_).max() / max(1.0, np.abs(want).max()) <= 1e-6
