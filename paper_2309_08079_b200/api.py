"""Reference-facing API of the B200 hot path (Python mirror of proj/include/trajopt).

Same names, argument meaning and error behaviour as the reference's C++ free
functions (block_tri.hpp, schur.hpp, pcg.hpp, random_problem.hpp); every
compute call goes through the C-ABI (include/b2p.h) into libb2p.so and runs
on the GPU. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _abi
from ._lib import load
from .types import (BatchReports, BlockTriMatrix, KKTSystem, PcgConfig, PcgResult, PcgVariant,
                    Preconditioner, PrecondKind, SchurSystem, SolveReport, raise_for)

_tls = threading.local()


class Context:
    """One b2p_ctx (device + stream + workspaces)."""

    def __init__(self, device: int = 0):
        L = load()
        self._lib = L
        self.device = device
        h = C.c_void_p()
        err = _abi.ErrorC()
        _check(L.b2p_ctx_create(device, C.byref(h), C.byref(err)), err)
        self.handle = h

    def set_stream(self, stream_ptr: int | None):
        self._lib.b2p_ctx_set_stream(self.handle, stream_ptr)

    @property
    def stream(self) -> int:
        return self._lib.b2p_ctx_stream(self.handle) or 0

    def kernel_launches(self) -> int:
        return int(self._lib.b2p_ctx_kernel_launches(self.handle))

    def last_path(self) -> int:
        """1 if the last fused solve ran the persistent K1+K3 kernel, 0 if split."""
        return int(self._lib.b2p_ctx_last_path(self.handle))

    def last_solve_ms(self) -> float:
        v = C.c_float()
        self._lib.b2p_ctx_last_solve_ms(self.handle, C.byref(v))
        return float(v.value)

    def last_h2d_bytes(self) -> int:
        """Host -> device bytes of the most recent solve_batched call (Q_k / R_k
        travel as lower triangles)."""
        v = C.c_ulonglong()
        self._lib.b2p_ctx_last_h2d_bytes(self.handle, C.byref(v))
        return int(v.value)

    def last_phase_ms(self) -> tuple[float, float]:
        """(K1 formation ms, K3 PCG ms) of the most recent fused solve."""
        v = (C.c_float * 2)()
        self._lib.b2p_ctx_last_phase_ms(self.handle, v, 2)
        return float(v[0]), float(v[1])

    def phase_accounting(self, enable: bool):
        self._lib.b2p_ctx_phase_accounting(self.handle, int(enable))

    def phase_totals(self) -> tuple[float, float, float, int]:
        """Summed (K1 ms, K3 ms, total ms, solves) since accounting was enabled."""
        v = (C.c_float * 3)()
        n = C.c_int()
        rc = self._lib.b2p_ctx_phase_totals(self.handle, v, 3, C.byref(n))
        if rc != 0:
            raise RuntimeError("b2p_ctx_phase_totals failed")
        return float(v[0]), float(v[1]), float(v[2]), int(n.value)

    def close(self):
        if self.handle:
            self._lib.b2p_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_count() -> int:
    return int(load().b2p_device_count())


def require_device():
    if device_count() < 1:
        raise RuntimeError("b2p: no CUDA device visible (the B200 path has no CPU fallback)")


def context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _check(rc: int, err: _abi.ErrorC):
    raise_for(rc, err.message.decode(errors="replace"), err.knot, err.iteration)


def _dt(dtype) -> int:
    return _abi.F32 if np.dtype(dtype) == np.float32 else _abi.F64


def _arr(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return None if a is None else a.ctypes.data


def _check_kkt(k: KKTSystem, batch: int | None = None):
    """Every array of a host KKTSystem must have the b2p_kkt shape for (N, n, m)
    (plus the leading batch dimension): the C side reads exactly that many bytes."""
    shapes = _abi.kkt_shapes(k.N, k.n, k.m)
    for f in _abi.KKT_FIELDS:
        a = getattr(k, f)
        want = shapes[f] if batch is None else (batch,) + shapes[f]
        if tuple(a.shape) != want:
            raise ValueError(f"KKTSystem.{f}: expected shape {want}, got {tuple(a.shape)}")


def _lambda0(lambda0, dt, dim: int, batch: int | None = None):
    """lambda0 as a contiguous dt vector of the dual dimension (pcg.cpp:34-35)."""
    if lambda0 is None:
        return None
    l0 = _arr(lambda0, dt)
    want = dim if batch is None else batch * dim
    if l0.size != want:
        raise ValueError(f"pcg: expected lambda0 of length {want}, got {l0.size}")
    return l0


def _compute_dtype(x, dtype):
    if dtype is not None:
        return np.dtype(dtype)
    return np.dtype(np.float32) if np.asarray(x).dtype == np.float32 else np.dtype(np.float64)


# ------------------------------------------------------------- random_problem.hpp
def _generate(family, seed, N, n, m, diag_floor=0.1, coupling=1.0) -> KKTSystem:
    kkt = KKTSystem.allocate(N, n, m)
    out = _abi.KktOutC(N, n, m, 0, *[a.ctypes.data for a in kkt.arrays()])
    err = _abi.ErrorC()
    _check(load().b2p_random_kkt(family, seed, N, n, m, diag_floor, coupling, C.byref(out),
                                 C.byref(err)), err)
    return kkt


def random_kkt(seed, N, n, m) -> KKTSystem:  # random_problem.cpp:42-44
    return _generate(0, seed, N, n, m)


def random_kkt_scaled(seed, N, n, m, diag_floor, coupling) -> KKTSystem:  # :46-49
    return _generate(1, seed, N, n, m, diag_floor, coupling)


def random_trajectory_kkt(seed, N, n, m) -> KKTSystem:  # :51-80
    return _generate(2, seed, N, n, m)


def random_kkt_batch(seed0: int, batch: int, N: int, n: int, m: int, family: int = 0,
                     diag_floor: float = 0.1, coupling: float = 1.0, threads: int = 0,
                     alloc=None) -> KKTSystem:
    """System i = random_kkt(seed0 + i, ...) (the bench-pcg seeding rule)."""
    kkt = KKTSystem.allocate(N, n, m, batch=batch, alloc=alloc)
    out = _abi.KktOutC(N, n, m, 0, *[a.ctypes.data for a in kkt.arrays()])
    err = _abi.ErrorC()
    _check(load().b2p_random_kkt_batch(family, seed0, batch, N, n, m, diag_floor, coupling,
                                       threads, C.byref(out), C.byref(err)), err)
    return kkt


# ------------------------------------------------------------- block_tri.hpp
def matvec(M: BlockTriMatrix, x, dtype=None) -> np.ndarray:
    dt = _compute_dtype(M.data, dtype)
    d = _arr(M.data, dt)
    x = _arr(x, dt)
    y = np.zeros(d.shape[0] * d.shape[2], dtype=dt)
    err = _abi.ErrorC()
    _check(load().b2p_blocktri_matvec(context().handle, _dt(dt), d.shape[0], d.shape[2],
                                      _ptr(d), _ptr(x), x.size, _ptr(y), C.byref(err)), err)
    return y


def max_asymmetry(M: BlockTriMatrix) -> float:
    d = _arr(M.data, _compute_dtype(M.data, None))
    a, m = C.c_double(), C.c_double()
    err = _abi.ErrorC()
    _check(load().b2p_blocktri_check(context().handle, _dt(d.dtype), d.shape[0], d.shape[2],
                                     _ptr(d), C.byref(a), C.byref(m), C.byref(err)), err)
    return a.value


def cholesky_solve(M: BlockTriMatrix, rhs, dtype=None) -> np.ndarray:
    dt = _compute_dtype(M.data, dtype)
    d = _arr(M.data, dt)
    rhs = _arr(rhs, dt)
    x = np.zeros(d.shape[0] * d.shape[2], dtype=dt)
    err = _abi.ErrorC()
    _check(load().b2p_blocktri_cholesky_solve(context().handle, _dt(dt), d.shape[0], d.shape[2],
                                              _ptr(d), _ptr(rhs), rhs.size, _ptr(x),
                                              C.byref(err)), err)
    return x


# ------------------------------------------------------------- schur.hpp
def build_schur(kkt: KKTSystem, dtype=np.float64) -> SchurSystem:  # schur.cpp:38-82
    dt = np.dtype(dtype)
    k = kkt.astype(dt)
    _check_kkt(k)
    K, n = k.N + 1, k.n
    S = np.zeros((K, 3, n, n), dtype=dt)
    gamma = np.zeros(K * n, dtype=dt)
    ti = np.zeros((K, n, n), dtype=dt)
    err = _abi.ErrorC()
    _check(load().b2p_build_schur(context().handle, _dt(dt), C.byref(k.to_c()), _ptr(S),
                                  _ptr(gamma), _ptr(ti), C.byref(err)), err)
    Sm = BlockTriMatrix(data=S)
    Sm.structurally_symmetric = True
    return SchurSystem(Sm, gamma, ti, n)


def stair_matrix(S: BlockTriMatrix) -> BlockTriMatrix:  # schur.cpp:84-94
    d = _arr(S.data, _compute_dtype(S.data, None))
    out = np.zeros_like(d)
    err = _abi.ErrorC()
    _check(load().b2p_stair_matrix(context().handle, _dt(d.dtype), d.shape[0], d.shape[2],
                                   _ptr(d), _ptr(out), C.byref(err)), err)
    return BlockTriMatrix(data=out)


def build_preconditioner(schur: SchurSystem, kind, order: int = 1,
                         dtype=None) -> Preconditioner:  # schur.cpp:164-173
    kind = PrecondKind(kind)
    dt = _compute_dtype(schur.S.data, dtype)
    S = _arr(schur.S.data, dt)
    ti = _arr(schur.theta_inv, dt)
    K, nb = S.shape[0], S.shape[2]
    phi = np.zeros_like(S)
    err = _abi.ErrorC()
    _check(load().b2p_build_preconditioner(context().handle, _dt(dt), int(kind), int(order), K,
                                           nb, _ptr(S), _ptr(ti), _ptr(phi), C.byref(err)), err)
    P = Preconditioner(kind=kind, order=order if kind == PrecondKind.poly_split else 0)
    if kind != PrecondKind.identity:
        P.phi_inv = BlockTriMatrix(data=phi)
        P.phi_inv.structurally_symmetric = kind in (PrecondKind.block_jacobi,
                                                    PrecondKind.symmetric_stair)
    if kind == PrecondKind.poly_split:
        P.S = schur.S
    return P


def build_identity() -> Preconditioner:  # schur.cpp:96
    return Preconditioner()


def build_block_jacobi(s: SchurSystem) -> Preconditioner:  # :98-107
    return build_preconditioner(s, PrecondKind.block_jacobi)


def build_stair(s: SchurSystem) -> Preconditioner:  # :109-127
    return build_preconditioner(s, PrecondKind.stair)


def build_symmetric_stair(s: SchurSystem) -> Preconditioner:  # :129-142
    return build_preconditioner(s, PrecondKind.symmetric_stair)


def build_poly_split(s: SchurSystem, order: int) -> Preconditioner:  # :144-162
    if order < 1:
        raise ValueError(f"build_poly_split: order must be >= 1, got {order}")
    return build_preconditioner(s, PrecondKind.poly_split, order)


def apply_preconditioner(P: Preconditioner, r, dtype=None) -> np.ndarray:  # :175-194
    if P.kind == PrecondKind.identity:
        return np.array(r, copy=True)
    dt = _compute_dtype(P.phi_inv.data, dtype)
    phi = _arr(P.phi_inv.data, dt)
    r = _arr(r, dt)
    K, nb = phi.shape[0], phi.shape[2]
    S = _arr(P.S.data, dt) if P.kind == PrecondKind.poly_split else None
    out = np.zeros(K * nb, dtype=dt)
    err = _abi.ErrorC()
    _check(load().b2p_apply_preconditioner(context().handle, _dt(dt), int(P.kind), int(P.order),
                                           K, nb, _ptr(S), _ptr(phi), _ptr(r), r.size, _ptr(out),
                                           C.byref(err)), err)
    return out


# ------------------------------------------------------------- pcg.hpp
def _max_iter(cfg, dim):
    return cfg.max_iter if cfg.max_iter > 0 else dim


def pcg_solve_auto(S: BlockTriMatrix, P: Preconditioner, gamma, lambda0,
                   cfg: PcgConfig | None = None, dtype=None) -> PcgResult:  # pcg.cpp:364-369
    cfg = cfg or PcgConfig()
    dt = _compute_dtype(S.data, dtype)
    d = _arr(S.data, dt)
    K, nb = (d.shape[0], d.shape[2]) if d.size else (0, 0)
    gamma = _arr(gamma, dt)
    lambda0 = _arr(lambda0, dt)
    phi = None
    pK = pnb = 0
    if P.kind != PrecondKind.identity:
        phi = _arr(P.phi_inv.data, dt)
        pK, pnb = phi.shape[0], phi.shape[2]
    lam = np.zeros(max(K * nb, 1), dtype=dt)
    rep = _abi.SolveReportC()
    trace = np.zeros(max(1, _max_iter(cfg, K * nb))) if cfg.collect_trace else None
    err = _abi.ErrorC()
    c = cfg.to_c()
    _check(load().b2p_pcg_solve(context().handle, _dt(dt), K, nb, _ptr(d), int(P.kind),
                                int(P.order), pK, pnb, _ptr(phi), _ptr(gamma), gamma.size,
                                _ptr(lambda0), lambda0.size, C.byref(c), _ptr(lam), C.byref(rep),
                                _ptr(trace), C.byref(err)), err)
    return PcgResult(lam[:K * nb], SolveReport.from_c(rep, trace))


def pcg_solve(S, P, gamma, lambda0, cfg=None, dtype=None) -> PcgResult:  # pcg.cpp:55-129
    cfg = PcgConfig(**{**(cfg or PcgConfig()).__dict__, "variant": PcgVariant.sequential})
    return pcg_solve_auto(S, P, gamma, lambda0, cfg, dtype)


def pcg_solve_block_parallel(S, P, gamma, lambda0, cfg=None, dtype=None) -> PcgResult:
    cfg = PcgConfig(**{**(cfg or PcgConfig()).__dict__, "variant": PcgVariant.block_parallel})
    return pcg_solve_auto(S, P, gamma, lambda0, cfg, dtype)


# ------------------------------------------------------------- fused hot path
def solve(kkt: KKTSystem, kind=PrecondKind.symmetric_stair, order: int = 1,
          cfg: PcgConfig | None = None, lambda0=None, dtype=np.float64) -> PcgResult:
    """build_schur -> build_preconditioner -> pcg_solve_auto in one device pass."""
    cfg = cfg or PcgConfig()
    dt = np.dtype(dtype)
    k = kkt.astype(dt)
    _check_kkt(k)
    D = k.dual_dim()
    lam = np.zeros(D, dtype=dt)
    l0 = _lambda0(lambda0, dt, D)
    rep = _abi.SolveReportC()
    trace = np.zeros(max(1, _max_iter(cfg, D))) if cfg.collect_trace else None
    err = _abi.ErrorC()
    c = cfg.to_c()
    _check(load().b2p_solve(context().handle, _dt(dt), C.byref(k.to_c()), int(kind), int(order),
                            C.byref(c), _ptr(l0), _ptr(lam), C.byref(rep), _ptr(trace),
                            C.byref(err)), err)
    return PcgResult(lam, SolveReport.from_c(rep, trace))


def solve_batched(kkt_batch: KKTSystem, kind=PrecondKind.symmetric_stair, order: int = 1,
                  cfg: PcgConfig | None = None, lambda0=None, dtype=np.float64,
                  lambda_out: np.ndarray | None = None, ctx: Context | None = None):
    """Independent systems from host buffers (pinned for full overlap).

    Returns (lambda [B, D], list[SolveReport])."""
    cfg = cfg or PcgConfig()
    dt = np.dtype(dtype)
    k = kkt_batch if all(a.dtype == dt for a in kkt_batch.arrays()) else kkt_batch.astype(dt)
    B = k.batch
    if B is None:
        raise ValueError("solve_batched: kkt_batch needs a leading batch dimension")
    _check_kkt(k, B)
    D = k.dual_dim()
    if lambda_out is not None:
        if (not isinstance(lambda_out, np.ndarray) or lambda_out.dtype != dt
                or tuple(lambda_out.shape) != (B, D) or not lambda_out.flags["C_CONTIGUOUS"]):
            raise ValueError(f"solve_batched: lambda_out must be a C-contiguous {dt.name} "
                             f"array of shape ({B}, {D})")
        lam = lambda_out
    else:
        lam = np.zeros((B, D), dtype=dt)
    l0 = _lambda0(lambda0, dt, D, B)
    reps = (_abi.SolveReportC * B)()
    err = _abi.ErrorC()
    c = cfg.to_c()
    ctx = ctx or context()
    _check(load().b2p_solve_batched(ctx.handle, _dt(dt), B, C.byref(k.to_c()), int(kind),
                                    int(order), C.byref(c), _ptr(l0), _ptr(lam), reps,
                                    C.byref(err)), err)
    return lam, BatchReports(reps)


def solve_batched_device(kkt_dev: KKTSystem, lambda_out_ptr: int, batch: int,
                         kind=PrecondKind.symmetric_stair, order: int = 1,
                         cfg: PcgConfig | None = None, lambda0_ptr: int | None = None,
                         dtype=np.float64, ctx: Context | None = None, want_reports=False,
                         status_ptr: int | None = None):
    """Device-resident batch: kkt_dev holds device tensors (anything with
    .data_ptr()). Launches on the context stream; no host sync unless
    want_reports. status_ptr: optional device int32[batch][4] (16-byte aligned)
    receiving {status, iterations, converged, aux} per system on the stream."""
    cfg = cfg or PcgConfig()
    ctx = ctx or context()
    kc = kkt_dev.to_c(ptr=lambda t: t.data_ptr())
    reps = (_abi.SolveReportC * batch)() if want_reports else None
    err = _abi.ErrorC()
    c = cfg.to_c()
    _check(load().b2p_solve_batched_device(ctx.handle, _dt(dtype), batch, C.byref(kc),
                                           int(kind), int(order), C.byref(c), lambda0_ptr,
                                           lambda_out_ptr, reps, status_ptr, C.byref(err)), err)
    return BatchReports(reps) if want_reports else None


def reconstruct_primal(kkt: KKTSystem, lam, dtype=np.float64) -> np.ndarray:  # kkt.cpp:153-181
    """dz = [x_0, u_0, ..., x_N] from the multipliers (one warp per knot block)."""
    dt = np.dtype(dtype)
    k = kkt.astype(dt)
    _check_kkt(k)
    lam = np.ascontiguousarray(np.asarray(lam), dtype=dt).reshape(-1)
    dz = np.zeros(k.primal_dim(), dtype=dt)
    err = _abi.ErrorC()
    _check(load().b2p_reconstruct_primal(context().handle, _dt(dt), C.byref(k.to_c()), _ptr(lam),
                                         int(lam.size), _ptr(dz), C.byref(err)), err)
    return dz


def sqp_step(kkt: KKTSystem, kind=PrecondKind.symmetric_stair, order: int = 1,
             cfg: PcgConfig | None = None, lambda0=None, dtype=np.float64):
    """The SQP linear step (sqp.cpp:171-176) on one upload: fused solve, then
    reconstruct_primal on the resident knots. Returns (PcgResult, dz)."""
    cfg = cfg or PcgConfig()
    dt = np.dtype(dtype)
    k = kkt.astype(dt)
    D = k.dual_dim()
    lam = np.zeros(D, dtype=dt)
    _check_kkt(k)
    dz = np.zeros(k.primal_dim(), dtype=dt)
    l0 = _lambda0(lambda0, dt, D)
    rep = _abi.SolveReportC()
    trace = np.zeros(max(1, _max_iter(cfg, D))) if cfg.collect_trace else None
    err = _abi.ErrorC()
    c = cfg.to_c()
    _check(load().b2p_sqp_step(context().handle, _dt(dt), C.byref(k.to_c()), int(kind),
                               int(order), C.byref(c), _ptr(l0), _ptr(lam), _ptr(dz),
                               C.byref(rep), _ptr(trace), C.byref(err)), err)
    return PcgResult(lam, SolveReport.from_c(rep, trace)), dz


def reconstruct_primal_batched_device(kkt_dev: KKTSystem, lambda_ptr: int, dz_ptr: int,
                                      batch: int, dtype=np.float64, ctx: Context | None = None):
    """Device-resident batch (tensors with .data_ptr()); no host sync."""
    ctx = ctx or context()
    kc = kkt_dev.to_c(ptr=lambda t: t.data_ptr())
    err = _abi.ErrorC()
    _check(load().b2p_reconstruct_primal_batched_device(ctx.handle, _dt(dtype), batch,
                                                        C.byref(kc), lambda_ptr, dz_ptr,
                                                        C.byref(err)), err)


def direct_solve_batched_device(kkt_dev: KKTSystem, lambda_ptr: int, status_ptr: int, batch: int,
                                dtype=np.float64, ctx: Context | None = None):
    """Direct baseline on a device-resident batch: build_schur then the block-Thomas
    cholesky_solve of S lambda = gamma (block_tri.cpp:121-159); no host sync."""
    ctx = ctx or context()
    kc = kkt_dev.to_c(ptr=lambda t: t.data_ptr())
    err = _abi.ErrorC()
    _check(load().b2p_direct_solve_batched_device(ctx.handle, _dt(dtype), batch, C.byref(kc),
                                                  lambda_ptr, status_ptr, C.byref(err)), err)


def solve_batched_multi(devices, kkt_batch: KKTSystem, kind=PrecondKind.symmetric_stair,
                        order: int = 1, cfg: PcgConfig | None = None, dtype=np.float64):
    """K4: contiguous batch-index shards, one host thread + context per device."""
    cfg = cfg or PcgConfig()
    dt = np.dtype(dtype)
    k = kkt_batch.astype(dt)
    _check_kkt(k, k.batch)
    B, D = k.batch, k.dual_dim()
    lam = np.zeros((B, D), dtype=dt)
    reps = (_abi.SolveReportC * B)()
    devs = (C.c_int * len(devices))(*devices)
    err = _abi.ErrorC()
    c = cfg.to_c()
    _check(load().b2p_solve_batched_multi(devs, len(devices), _dt(dt), B, C.byref(k.to_c()),
                                          int(kind), int(order), C.byref(c), None, _ptr(lam),
                                          reps, C.byref(err)), err)
    return lam, BatchReports(reps)
