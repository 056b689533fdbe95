"""Host-side value types mirroring the reference's C++ API.

Names, field order, defaults and exception classes follow
proj/include/trajopt/{block_tri,kkt,schur,pcg}.hpp so that code written
against the reference reads the same here. Storage is numpy, row-major,
in the b2p.h layouts; the compute happens behind the C-ABI.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi


# ---------------------------------------------------------------- exceptions
class PcgBreakdown(RuntimeError):
    """p'Sp <= 0 during CG (pcg.hpp:47-50)."""


class B2PCudaError(RuntimeError):
    """Device / driver failure (no reference analog)."""


def raise_for(code: int, message: str, knot: int = -1, iteration: int = -1):
    """Map a b2p_status to the reference's exception class."""
    if code == _abi.OK:
        return
    if code == _abi.INVALID_ARGUMENT:
        raise ValueError(message)  # std::invalid_argument
    if code == _abi.BREAKDOWN:
        raise PcgBreakdown(message)
    if code == _abi.CUDA_ERROR:
        raise B2PCudaError(message)
    raise RuntimeError(message)  # std::runtime_error


# ---------------------------------------------------------------- enums
class PrecondKind(enum.IntEnum):  # schur.hpp:26
    identity = _abi.IDENTITY
    block_jacobi = _abi.BLOCK_JACOBI
    stair = _abi.STAIR
    symmetric_stair = _abi.SYMMETRIC_STAIR
    poly_split = _abi.POLY_SPLIT


class PcgVariant(enum.IntEnum):  # pcg.hpp:12
    sequential = _abi.SEQUENTIAL
    block_parallel = _abi.BLOCK_PARALLEL


def precond_name(kind: PrecondKind, order: int = 0) -> str:
    """schur.cpp:27-36 — canonical CSV names."""
    kind = PrecondKind(kind)
    return {
        PrecondKind.identity: "identity",
        PrecondKind.block_jacobi: "jacobi",
        PrecondKind.stair: "stair",
        PrecondKind.symmetric_stair: "symstair",
    }.get(kind, f"poly:{order}")


def parse_precond(name: str) -> tuple[PrecondKind, int]:
    """trajopt_cli.cpp:41-53."""
    if name == "identity":
        return PrecondKind.identity, 0
    if name == "jacobi":
        return PrecondKind.block_jacobi, 0
    if name == "stair":
        return PrecondKind.stair, 0
    if name == "symstair":
        return PrecondKind.symmetric_stair, 0
    if name.startswith("poly:"):
        order = int(name[5:])
        if order < 1:
            raise ValueError("poly preconditioner order must be >= 1: " + name)
        return PrecondKind.poly_split, order
    raise ValueError(
        f'unknown preconditioner "{name}" (expected identity|jacobi|stair|symstair|poly:<order>)')


# ---------------------------------------------------------------- config / report
@dataclass
class PcgConfig:  # pcg.hpp:14-29 (field order preserved)
    epsilon: float = 1e-4
    max_iter: int = 0
    deterministic_reductions: bool = False
    variant: PcgVariant = PcgVariant.sequential
    collect_trace: bool = False
    check_residual_drift: bool = False

    def to_c(self) -> _abi.PcgConfigC:
        return _abi.PcgConfigC(float(self.epsilon), int(self.max_iter),
                               int(bool(self.deterministic_reductions)), int(self.variant),
                               int(bool(self.collect_trace)),
                               int(bool(self.check_residual_drift)), 0)


@dataclass
class SolveReport:  # pcg.hpp:31-38
    iterations: int = 0
    exit_eta: float = 0.0
    converged: bool = False
    trace: list = field(default_factory=list)
    wall_time: float = 0.0
    max_residual_drift: float = 0.0

    @staticmethod
    def from_c(rep: _abi.SolveReportC, trace: np.ndarray | None = None) -> "SolveReport":
        tr = [] if trace is None else [float(x) for x in trace[: rep.trace_len]]
        return SolveReport(int(rep.iterations), float(rep.exit_eta), bool(rep.converged), tr,
                           float(rep.wall_time), float(rep.max_residual_drift))


class BatchReports:
    """Per-system SolveReports of a batched call, decoded lazily from the C
    array (a 4096-system batch would otherwise spend milliseconds building
    Python objects). Indexing / iteration yields SolveReport; the fields are
    also available whole as numpy arrays (.iterations, .converged, ...)."""

    def __init__(self, arr):
        self._c = arr
        self._np = np.ctypeslib.as_array(arr)

    def __len__(self) -> int:
        return len(self._c)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        return SolveReport.from_c(self._c[i])

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    def field(self, name: str) -> np.ndarray:
        return self._np[name].copy()

    @property
    def iterations(self) -> np.ndarray:
        return self.field("iterations")

    @property
    def converged(self) -> np.ndarray:
        return self.field("converged").astype(bool)

    @property
    def exit_eta(self) -> np.ndarray:
        return self.field("exit_eta")


@dataclass
class PcgResult:  # pcg.hpp:40-43
    lambda_: np.ndarray
    report: SolveReport

    @property
    def lam(self) -> np.ndarray:
        return self.lambda_


# ---------------------------------------------------------------- BlockTriMatrix
class BlockTriMatrix:
    """block_tri.hpp:18-75 — data[K][3][nb][nb], slot 0 left, 1 diag, 2 right."""

    def __init__(self, num_block_rows: int = 0, block_dim: int = 0, dtype=np.float64,
                 data: np.ndarray | None = None):
        if data is not None:
            data = np.ascontiguousarray(data)
            if data.ndim != 4 or data.shape[1] != 3 or data.shape[2] != data.shape[3]:
                raise ValueError("BlockTriMatrix: data must be [K][3][nb][nb]")
            self.data = data
            self.structurally_symmetric = False
            return
        if num_block_rows == 0 and block_dim == 0:
            self.data = np.zeros((0, 3, 0, 0), dtype=dtype)
        else:
            if num_block_rows < 1 or block_dim < 1:
                raise ValueError(
                    "BlockTriMatrix: need at least one block row and block_dim >= 1")
            self.data = np.zeros((num_block_rows, 3, block_dim, block_dim), dtype=dtype)
        self.structurally_symmetric = False

    def block_rows(self) -> int:
        return self.data.shape[0]

    def block_dim(self) -> int:
        return self.data.shape[2]

    def dim(self) -> int:
        return self.block_rows() * self.block_dim()

    def empty(self) -> bool:
        return self.block_rows() == 0

    def left(self, row):
        return self.data[row, 0]

    def diag(self, row):
        return self.data[row, 1]

    def right(self, row):
        return self.data[row, 2]

    def _check(self, row, b):
        if row < 0 or row >= self.block_rows():
            raise ValueError(
                f"BlockTriMatrix: block row {row} out of range [0, {self.block_rows()})")
        b = np.asarray(b)
        nb = self.block_dim()
        if b.shape != (nb, nb):
            raise ValueError(f"BlockTriMatrix: expected {nb}x{nb} block, got "
                             f"{b.shape[0] if b.ndim else 0}x{b.shape[1] if b.ndim > 1 else 0}")
        return b

    def set_left(self, row, b):  # block_tri.cpp:46-52
        b = self._check(row, b)
        if row == 0:
            raise ValueError("BlockTriMatrix: row 0 has no left block (boundary padding)")
        self.data[row, 0] = b

    def set_diag(self, row, b):
        self.data[row, 1] = self._check(row, b)

    def set_right(self, row, b):  # block_tri.cpp:60-67
        b = self._check(row, b)
        if row == self.block_rows() - 1:
            raise ValueError("BlockTriMatrix: last row has no right block (boundary padding)")
        self.data[row, 2] = b

    def to_dense(self) -> np.ndarray:  # block_tri.cpp:94-104
        K, nb = self.block_rows(), self.block_dim()
        D = np.zeros((K * nb, K * nb), dtype=self.data.dtype)
        for r in range(K):
            if r > 0:
                D[r * nb:(r + 1) * nb, (r - 1) * nb:r * nb] = self.left(r)
            D[r * nb:(r + 1) * nb, r * nb:(r + 1) * nb] = self.diag(r)
            if r + 1 < K:
                D[r * nb:(r + 1) * nb, (r + 1) * nb:(r + 2) * nb] = self.right(r)
        return D

    @staticmethod
    def from_dense(dense: np.ndarray, block_dim: int) -> "BlockTriMatrix":  # :106-119
        dense = np.asarray(dense)
        if dense.shape[0] != dense.shape[1] or dense.shape[0] % block_dim != 0:
            raise ValueError(f"BlockTriMatrix::from_dense: matrix size {dense.shape[0]}x"
                             f"{dense.shape[1]} is not square with block_dim {block_dim}")
        K = dense.shape[0] // block_dim
        nb = block_dim
        out = BlockTriMatrix(K, nb, dtype=dense.dtype)
        for r in range(K):
            if r > 0:
                out.set_left(r, dense[r * nb:(r + 1) * nb, (r - 1) * nb:r * nb])
            out.set_diag(r, dense[r * nb:(r + 1) * nb, r * nb:(r + 1) * nb])
            if r + 1 < K:
                out.set_right(r, dense[r * nb:(r + 1) * nb, (r + 1) * nb:(r + 2) * nb])
        return out

    def max_abs(self) -> float:  # block_tri.cpp:161-165
        return float(np.abs(self.data).max()) if self.data.size else 0.0

    def max_asymmetry(self) -> float:  # block_tri.cpp:167-177
        d = self.data
        w = float(np.abs(d[:, 1] - np.swapaxes(d[:, 1], 1, 2)).max()) if d.size else 0.0
        if d.shape[0] > 1:
            w = max(w, float(np.abs(d[:-1, 2] - np.swapaxes(d[1:, 0], 1, 2)).max()))
        return w

    def copy(self) -> "BlockTriMatrix":
        out = BlockTriMatrix(data=self.data.copy())
        out.structurally_symmetric = self.structurally_symmetric
        return out


# ---------------------------------------------------------------- KKT
@dataclass
class KKTSystem:
    """kkt.hpp:29-46 in the b2p_kkt SoA layout (optionally with a leading batch dim)."""

    N: int
    n: int
    m: int
    Q: np.ndarray
    q: np.ndarray
    R: np.ndarray
    r: np.ndarray
    A: np.ndarray
    B: np.ndarray
    e: np.ndarray
    x_s: np.ndarray
    x0: np.ndarray

    @property
    def batch(self) -> int | None:
        return None if self.Q.ndim == 3 else self.Q.shape[0]

    def primal_dim(self) -> int:
        return (self.N + 1) * self.n + self.N * self.m

    def dual_dim(self) -> int:
        return (self.N + 1) * self.n

    def arrays(self):
        return [getattr(self, f) for f in _abi.KKT_FIELDS]

    def astype(self, dtype) -> "KKTSystem":
        return KKTSystem(self.N, self.n, self.m,
                         *[np.ascontiguousarray(a, dtype=dtype) for a in self.arrays()])

    def system(self, i: int) -> "KKTSystem":
        return KKTSystem(self.N, self.n, self.m, *[a[i] for a in self.arrays()])

    def constraint_rhs(self) -> np.ndarray:  # kkt.cpp:32-39
        c = np.empty(self.dual_dim(), dtype=self.Q.dtype)
        c[: self.n] = self.x_s - self.x0
        c[self.n:] = (-self.e).reshape(-1)
        return c

    @staticmethod
    def allocate(N: int, n: int, m: int, batch: int | None = None, dtype=np.float64,
                 alloc=None) -> "KKTSystem":
        shapes = _abi.kkt_shapes(N, n, m)
        arrs = []
        for f in _abi.KKT_FIELDS:
            shp = shapes[f] if batch is None else (batch,) + shapes[f]
            arrs.append(alloc(shp, dtype) if alloc else np.zeros(shp, dtype=dtype))
        return KKTSystem(N, n, m, *arrs)

    def to_c(self, ptr=None) -> _abi.KktC:
        """b2p_kkt view. `ptr(array)` maps an array to an address (host default)."""
        arrs = self.arrays()
        for a in arrs:
            if isinstance(a, np.ndarray) and not a.flags["C_CONTIGUOUS"]:
                raise ValueError("KKTSystem arrays must be C-contiguous")
        get = ptr or (lambda a: a.ctypes.data)
        return _abi.KktC(self.N, self.n, self.m, 0, *[get(a) for a in arrs])


@dataclass
class SchurSystem:  # schur.hpp:19-24
    S: BlockTriMatrix
    gamma: np.ndarray
    theta_inv: np.ndarray  # [K][n][n]
    n: int = 0


@dataclass
class Preconditioner:  # schur.hpp:33-38
    kind: PrecondKind = PrecondKind.identity
    order: int = 0
    phi_inv: BlockTriMatrix = field(default_factory=BlockTriMatrix)
    # poly_split only: Psi and E = Psi - S are implied by S (kept for callers
    # that want them materialised).
    stair_psi: BlockTriMatrix | None = None
    remainder: BlockTriMatrix | None = None
    S: BlockTriMatrix | None = None  # the system the poly series splits
