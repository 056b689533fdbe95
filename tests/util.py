"""Test helpers mirroring proj/tests/test_util.hpp (dense oracles, seeded batches)."""
import numpy as np

from paper_2309_08079_b200.types import BlockTriMatrix, KKTSystem


def dense_G(k: KKTSystem) -> np.ndarray:  # kkt.cpp:41-52
    N, n, m = k.N, k.n, k.m
    G = np.zeros((k.primal_dim(), k.primal_dim()))
    off = 0
    for i in range(N + 1):
        G[off:off + n, off:off + n] = k.Q[i]
        off += n
        if i < N:
            G[off:off + m, off:off + m] = k.R[i]
            off += m
    return G


def dense_g(k: KKTSystem) -> np.ndarray:  # kkt.cpp:54-66
    parts = []
    for i in range(k.N + 1):
        parts.append(k.q[i])
        if i < k.N:
            parts.append(k.r[i])
    return np.concatenate(parts)


def dense_C(k: KKTSystem) -> np.ndarray:  # kkt.cpp:68-81
    N, n, m = k.N, k.n, k.m
    C = np.zeros((k.dual_dim(), k.primal_dim()))
    C[:n, :n] = np.eye(n)
    stride = n + m
    for i in range(N):
        row, col = (i + 1) * n, i * stride
        C[row:row + n, col:col + n] = -k.A[i]
        C[row:row + n, col + n:col + n + m] = -k.B[i]
        C[row:row + n, col + stride:col + stride + n] = np.eye(n)
    return C


def dense_schur_matrix(k):  # test_util.hpp:16-20
    G, C = dense_G(k), dense_C(k)
    return C @ np.linalg.solve(G, C.T)


def dense_schur_rhs(k):  # test_util.hpp:22-26
    G, C = dense_G(k), dense_C(k)
    return -(k.constraint_rhs() + C @ np.linalg.solve(G, dense_g(k)))


def random_block_tri(rng, rows, nb, symmetric=False) -> BlockTriMatrix:  # test_util.hpp:30-46
    M = BlockTriMatrix(rows, nb)
    for i in range(rows):
        D = rng.matrix(nb, nb, -1.0, 1.0)
        if symmetric:
            D = 0.5 * (D + D.T)
        M.set_diag(i, D)
        if i + 1 < rows:
            R = rng.matrix(nb, nb, -1.0, 1.0)
            M.set_right(i, R)
            M.set_left(i + 1, R.T.copy() if symmetric else rng.matrix(nb, nb, -1.0, 1.0))
    return M


def standard_batch(count=50, seed0=1000):  # test_util.hpp:57-68
    Ns, ns, ms = (3, 8, 32), (2, 4), (1, 2)
    return [(seed0 + i, Ns[i % 3], ns[(i // 3) % 2], ms[(i // 6) % 2]) for i in range(count)]


def rel_inf_error(got, want):  # test_util.hpp:70-78
    want = np.asarray(want)
    scale = max(1.0, float(np.abs(want).max()))
    return float(np.abs(np.asarray(got) - want).max()) / scale


def wrap(S: BlockTriMatrix):
    """test_schur.cpp:18-28 — SchurSystem around a hand-built S."""
    from paper_2309_08079_b200.types import SchurSystem
    ti = []
    for row in range(S.block_rows()):
        inv = np.linalg.inv(S.diag(row))
        ti.append(0.5 * (inv + inv.T))
    return SchurSystem(S, np.zeros(S.dim()), np.array(ti), S.block_dim())


def scalar_spd_2block() -> BlockTriMatrix:  # test_schur.cpp:30-37
    S = BlockTriMatrix(2, 1)
    S.set_diag(0, 2.0 * np.eye(1))
    S.set_diag(1, 2.0 * np.eye(1))
    S.set_right(0, np.eye(1))
    S.set_left(1, np.eye(1))
    return S


def identity_system(blocks, nb) -> BlockTriMatrix:  # test_pcg.cpp:18-22
    S = BlockTriMatrix(blocks, nb)
    for i in range(blocks):
        S.set_diag(i, np.eye(nb))
    return S


def kat(name):
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "reference_kats.json")
    return json.load(open(path))[name]


def cg_longdouble(S, gamma, eps, max_iter):
    """Textbook CG (pcg.cpp:55-129 with Phi = I) on the dense S in x87 80-bit
    extended precision: the rounding-light reference for unpreconditioned-CG
    exit counts (scripts/identity_mismatch.py). Returns (iterations, trace)."""
    import numpy as np
    A = S.to_dense().astype(np.longdouble)
    g = np.asarray(gamma, dtype=np.longdouble)
    r = g.copy()
    p = r.copy()
    eta = r @ r
    trace = []
    for i in range(1, max_iter + 1):
        sp = A @ p
        alpha = eta / (p @ sp)
        r = r - alpha * sp
        eta_p = r @ r
        trace.append(float(eta_p))
        if eta_p < eps:
            return i, trace
        p = r + (eta_p / eta) * p
        eta = eta_p
    return max_iter, trace
