"""Port of the reconstruct_primal cases of proj/tests/test_kkt.cpp (SURVEY §8f
rank 1: the "Trajopt PPCG finish", kkt.cpp:153-181). Every case runs on the
oracle and, marked gpu, on the B200 kernel through the C-ABI."""
import numpy as np
import pytest

from backends import B  # noqa: F401
from paper_2309_08079_b200.types import KKTSystem
from util import dense_C, dense_G, dense_g, dense_schur_matrix, dense_schur_rhs, standard_batch


def kkt_residual(kkt, dz, lam):  # test_kkt.cpp:17-26
    G, C, g, c = dense_G(kkt), dense_C(kkt), dense_g(kkt), kkt.constraint_rhs()
    stationarity = np.abs(G @ dz + g + C.T @ lam).max()
    primal = np.abs(C @ dz - c).max()
    scale = max(1.0, np.abs(g).max(), np.abs(c).max())
    return max(stationarity, primal) / scale


def dense_kkt_solve(kkt):  # kkt.cpp:129-151
    G, C = dense_G(kkt), dense_C(kkt)
    npd, nd = G.shape[0], C.shape[0]
    K = np.zeros((npd + nd, npd + nd))
    K[:npd, :npd] = G
    K[:npd, npd:] = C.T
    K[npd:, :npd] = C
    sol = np.linalg.solve(K, np.concatenate([-dense_g(kkt), kkt.constraint_rhs()]))
    return sol[:npd], sol[npd:]


def test_zero_multipliers_identity_G_give_minus_g(B, orc):  # test_kkt.cpp:101-109
    kkt = orc.random_kkt(31, 3, 2, 1)
    kkt.Q[:] = np.eye(2)
    kkt.R[:] = np.eye(1)
    dz = B.reconstruct_primal(kkt, np.zeros(kkt.dual_dim()))
    assert np.abs(dz + dense_g(kkt)).max() <= 1e-14


def test_matches_dense_oracle_primal(B, orc):  # :110-115
    kkt = orc.random_kkt(32, 4, 3, 2)
    dz_ref, lam = dense_kkt_solve(kkt)
    dz = B.reconstruct_primal(kkt, lam)
    assert np.abs(dz - dz_ref).max() <= 1e-8


def test_degenerate_single_knot_horizon(B):  # :116-128
    kkt = KKTSystem(0, 3, 0, Q=np.eye(3)[None].copy(), q=np.ones((1, 3)),
                    R=np.zeros((0, 0, 0)), r=np.zeros((0, 0)), A=np.zeros((0, 3, 3)),
                    B=np.zeros((0, 3, 0)), e=np.zeros((0, 3)), x_s=np.zeros(3), x0=np.zeros(3))
    dz = B.reconstruct_primal(kkt, np.zeros(3))
    assert np.abs(dz + np.ones(3)).max() == 0.0


def test_exact_dual_solve_closes_both_kkt_rows(B, orc):  # :131-142
    for seed, N, n, m in standard_batch(10):
        kkt = orc.random_kkt(seed, N, n, m)
        lam = np.linalg.solve(dense_schur_matrix(kkt), dense_schur_rhs(kkt))
        dz = B.reconstruct_primal(kkt, lam)
        assert kkt_residual(kkt, dz, lam) <= 1e-8
        assert np.abs(dense_C(kkt) @ dz - kkt.constraint_rhs()).max() <= 1e-8


def test_lambda_length_message(B, orc):  # kkt.cpp:154-158
    kkt = orc.random_kkt(33, 3, 2, 1)
    with pytest.raises(ValueError, match="reconstruct_primal: expected lambda of length 8, got 5"):
        B.reconstruct_primal(kkt, np.zeros(5))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(63, 14, 7), (511, 28, 14), (255, 12, 4)])
def test_b200_matches_oracle_at_baseline_shapes(orc, shape):
    import paper_2309_08079_b200.api as api
    api.require_device()
    N, n, m = shape
    kkt = orc.random_kkt(7 + N, N, n, m)
    lam = orc.solve(kkt).lambda_
    want = orc.reconstruct_primal(kkt, lam)
    got = api.reconstruct_primal(kkt, lam)
    scale = max(1.0, np.abs(want).max())
    assert np.abs(got - want).max() / scale <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("Bn,N", [(6, 31), (7, 20), (3, 0), (5, 1), (41, 9)])
def test_b200_batched_device_matches_single(orc, Bn, N):
    # ragged horizons: the streaming kernel's 16-task CTAs straddle system
    # boundaries (K = 21, 10) and the terminal knot (N = 0, 1)
    import torch
    import paper_2309_08079_b200.api as api
    api.require_device()
    n, m = 14, 7
    kb = api.random_kkt_batch(500, Bn, N, n, m)
    lam = np.stack([orc.solve(kb.system(i)).lambda_ for i in range(Bn)])
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in kb.arrays()]
    kd = KKTSystem(N, n, m, *dev)
    lam_d = torch.from_numpy(lam).cuda()
    dz_d = torch.empty((Bn, kb.primal_dim()), dtype=torch.float64, device="cuda")
    api.reconstruct_primal_batched_device(kd, lam_d.data_ptr(), dz_d.data_ptr(), Bn)
    torch.cuda.synchronize()
    got = dz_d.cpu().numpy()
    for i in range(Bn):
        want = orc.reconstruct_primal(kb.system(i), lam[i])
        assert np.abs(got[i] - want).max() / max(1.0, np.abs(want).max()) <= 1e-12


def test_sqp_step_null_dz_is_invalid_argument():  # b2p.h b2p_sqp_step (checked before any device work)
    import ctypes as C
    from paper_2309_08079_b200 import _abi, _lib
    L = _lib.load()
    err = _abi.ErrorC()
    rc = L.b2p_sqp_step(None, 0, None, 3, 1, None, None, None, None, None, None, C.byref(err))
    assert rc == 1 and b"null dz" in err.message


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(31, 14, 7), (8, 3, 2), (127, 14, 7)])
def test_sqp_step_equals_solve_then_reconstruct(orc, shape):
    """b2p_sqp_step (one upload, fused solve + primal kernel) returns exactly
    what b2p_solve followed by b2p_reconstruct_primal return, and agrees with
    the oracle's linear step, warm start included."""
    import paper_2309_08079_b200.api as api
    from paper_2309_08079_b200.types import PcgConfig
    api.require_device()
    N, n, m = shape
    kkt = orc.random_kkt(900 + N, N, n, m)
    cfg = PcgConfig(epsilon=1e-8)
    lam0 = 0.01 * orc.UniformRng(5).vector(kkt.dual_dim(), -1.0, 1.0)
    ctx = api.context()
    for l0 in (None, lam0):
        before = ctx.kernel_launches()
        res, dz = api.sqp_step(kkt, cfg=cfg, lambda0=l0)
        launched = ctx.kernel_launches() - before
        # one-CTA (n14 m7, K <= 64) and small-block (n, m <= 8) kernels run the
        # PPCG finish in their epilogue: the whole linear step is ONE launch
        fused = ctx.last_path() in (1, 4)
        assert launched == (1 if fused else 2), (launched, ctx.last_path())
        ref = api.solve(kkt, cfg=cfg, lambda0=l0)
        assert res.report.iterations == ref.report.iterations
        assert np.array_equal(res.lambda_, ref.lambda_)
        sep = api.reconstruct_primal(kkt, ref.lambda_)  # the standalone LDL' kernel
        if fused:  # explicit Q_k^-1 / R_k^-1 from the formation vs the LDL' solve
            assert np.abs(dz - sep).max() / max(1.0, np.abs(sep).max()) <= 1e-12
        else:
            assert np.array_equal(dz, sep)
        o = orc.solve(kkt, cfg=cfg, lambda0=l0)
        assert res.report.iterations == o.report.iterations
        want = orc.reconstruct_primal(kkt, o.lambda_)
        assert np.abs(dz - want).max() / max(1.0, np.abs(want).max()) <= 1e-9
