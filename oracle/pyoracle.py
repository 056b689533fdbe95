"""TEST INFRASTRUCTURE — NOT PRODUCT CODE.

ctypes wrapper over oracle/build/liboracle.so, the Eigen-free CPU
restatement of the reference hot path (oracle/trajopt_oracle.hpp). Only
tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
It mirrors the reference API names (build_schur, build_preconditioner,
apply_preconditioner, pcg_solve, ...) so parity tests read like the
reference's doctest suites.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2309_08079_b200 import _abi
from paper_2309_08079_b200.types import (BlockTriMatrix, KKTSystem, PcgConfig, PcgResult,
                                         PrecondKind, SchurSystem, SolveReport, raise_for)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
# the labelled "-march=native" CPU row BASELINE.md §2 allows (bench.py only);
# built on the machine that runs it (the GPU box's host CPU)
LIB_NATIVE = os.path.join(HERE, "build", "liboracle_native.so")


def build(force: bool = False, native: bool = False) -> str:
    """g++ -O3 -DNDEBUG (the reference's Release flags, proj/CMakeLists.txt:6-8);
    native=True adds -march=native into a separate library."""
    out = LIB_NATIVE if native else LIB_PATH
    src = [os.path.join(HERE, "oracle_capi.cpp"), os.path.join(HERE, "trajopt_oracle.hpp")]
    stamp = out + ".cpu"
    same_cpu = not native or (os.path.exists(stamp) and open(stamp).read() == _cpu_signature())
    if (not force and same_cpu and os.path.exists(out)
            and os.path.getmtime(out) >= max(os.path.getmtime(s) for s in src)):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + f".{os.getpid()}.tmp"
    cmd = ["g++", "-std=c++20", "-O3", "-DNDEBUG", "-fPIC", "-shared", "-pthread"]
    cmd += ["-march=native"] if native else []
    subprocess.check_call(cmd + [src[0], "-o", tmp])
    os.replace(tmp, out)
    if native:
        open(stamp, "w").write(_cpu_signature())
    return out


def _cpu_signature() -> str:
    """Model name + ISA flags of this host: a -march=native build only runs here."""
    try:
        lines = open("/proc/cpuinfo").read().splitlines()
    except OSError:
        return "unknown"
    keep = [ln for ln in lines if ln.startswith(("model name", "flags"))][:2]
    return "\n".join(keep)


_libs = {}


def lib(native: bool = False):
    if native not in _libs:
        path = LIB_NATIVE if native else LIB_PATH
        if native:
            build(native=True)  # always for this host's CPU
        elif not os.path.exists(path):
            build()
        L = C.CDLL(path)
        vp, i32, dbl, u64 = C.c_void_p, C.c_int, C.c_double, C.c_uint64
        E = C.POINTER(_abi.ErrorC)
        L.orc_set_threads.argtypes = [i32]
        L.orc_uniform.argtypes = [u64, i32, dbl, dbl, vp]
        L.orc_uniform.restype = None
        L.orc_random_kkt.argtypes = [i32, u64, i32, i32, i32, dbl, dbl,
                                     C.POINTER(_abi.KktOutC), E]
        L.orc_build_schur.argtypes = [i32, C.POINTER(_abi.KktC), vp, vp, vp, E]
        L.orc_stair_matrix.argtypes = [i32, i32, vp, vp, E]
        L.orc_build_preconditioner.argtypes = [i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, E]
        L.orc_apply_preconditioner.argtypes = [i32, i32, i32, i32, i32, vp, vp, vp, vp, E]
        L.orc_matvec.argtypes = [i32, i32, vp, vp, i32, vp, E]
        L.orc_max_asymmetry.argtypes = [i32, i32, vp]
        L.orc_max_asymmetry.restype = dbl
        L.orc_max_abs.argtypes = [i32, i32, vp]
        L.orc_max_abs.restype = dbl
        L.orc_cholesky_solve.argtypes = [i32, i32, vp, vp, vp, E]
        L.orc_pcg_solve.argtypes = [i32, i32, i32, vp, i32, i32, vp, vp, i32, vp, i32,
                                    C.POINTER(_abi.PcgConfigC), vp,
                                    C.POINTER(_abi.SolveReportC), vp, E]
        L.orc_solve.argtypes = [i32, C.POINTER(_abi.KktC), i32, i32,
                                C.POINTER(_abi.PcgConfigC), vp, vp,
                                C.POINTER(_abi.SolveReportC), vp, E]
        L.orc_solve_batch.argtypes = [i32, i32, C.POINTER(_abi.KktC), i32, i32,
                                      C.POINTER(_abi.PcgConfigC), i32, vp,
                                      C.POINTER(_abi.SolveReportC), E]
        L.orc_solve_batch.restype = dbl
        L.orc_reconstruct_primal.argtypes = [i32, C.POINTER(_abi.KktC), vp, i32, vp, E]
        L.orc_random_kkt_batch.argtypes = [i32, u64, i32, i32, i32, i32, dbl, dbl, i32,
                                           C.POINTER(_abi.KktOutC), E]
        _libs[native] = L
    return _libs[native]


def _check(rc: int, err: _abi.ErrorC):
    raise_for(rc, err.message.decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _dt(dtype) -> int:
    return _abi.F32 if np.dtype(dtype) == np.float32 else _abi.F64


def set_threads(t: int) -> int:
    return lib().orc_set_threads(int(t))


# ---------------------------------------------------------------- generator
class UniformRng:
    """random_problem.hpp:13-37 — mt19937_64, u = (x>>11)*2^-53, row-major draws."""

    def __init__(self, seed: int):
        self.seed = seed
        self.pos = 0
        self.buf = np.zeros(0)

    def _take(self, count: int) -> np.ndarray:
        need = self.pos + count
        if need > self.buf.size:
            n = max(need, 2 * self.buf.size, 4096)
            self.buf = np.zeros(n)
            lib().orc_uniform(self.seed, n, 0.0, 1.0, self.buf.ctypes.data)
        out = self.buf[self.pos:need]
        self.pos = need
        return out

    def uniform(self, lo, hi):
        return lo + (hi - lo) * float(self._take(1)[0])

    def matrix(self, rows, cols, lo, hi):
        return (lo + (hi - lo) * self._take(rows * cols)).reshape(rows, cols)

    def vector(self, size, lo, hi):
        return lo + (hi - lo) * self._take(size)


def _generate(family, seed, N, n, m, diag_floor=0.1, coupling=1.0) -> KKTSystem:
    kkt = KKTSystem.allocate(N, n, m)
    out = _abi.KktOutC(N, n, m, 0, *[a.ctypes.data for a in kkt.arrays()])
    err = _abi.ErrorC()
    _check(lib().orc_random_kkt(family, seed, N, n, m, diag_floor, coupling, C.byref(out),
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
    _check(lib().orc_random_kkt_batch(family, seed0, batch, N, n, m, diag_floor, coupling,
                                      threads, C.byref(out), C.byref(err)), err)
    return kkt


def stack(kkts: list[KKTSystem]) -> KKTSystem:
    k0 = kkts[0]
    return KKTSystem(k0.N, k0.n, k0.m,
                     *[np.ascontiguousarray(np.stack([getattr(k, f) for k in kkts]))
                       for f in _abi.KKT_FIELDS])


# ---------------------------------------------------------------- schur.hpp
def build_schur(kkt: KKTSystem, dtype=np.float64) -> SchurSystem:
    kkt = kkt.astype(np.float64)
    K, n = kkt.N + 1, kkt.n
    S = np.zeros((K, 3, n, n))
    gamma = np.zeros(K * n)
    theta_inv = np.zeros((K, n, n))
    err = _abi.ErrorC()
    _check(lib().orc_build_schur(_dt(dtype), C.byref(kkt.to_c()), _ptr(S), _ptr(gamma),
                                 _ptr(theta_inv), C.byref(err)), err)
    Sm = BlockTriMatrix(data=S)
    Sm.structurally_symmetric = True
    return SchurSystem(Sm, gamma, theta_inv, n)


def stair_matrix(S: BlockTriMatrix) -> BlockTriMatrix:
    d = _f64(S.data)
    out = np.zeros_like(d)
    err = _abi.ErrorC()
    _check(lib().orc_stair_matrix(d.shape[0], d.shape[2], _ptr(d), _ptr(out), C.byref(err)), err)
    return BlockTriMatrix(data=out)


def build_preconditioner(schur: SchurSystem, kind, order: int = 1, dtype=np.float64):
    from paper_2309_08079_b200.types import Preconditioner
    S = _f64(schur.S.data)
    ti = _f64(schur.theta_inv)
    K, nb = S.shape[0], S.shape[2]
    phi = np.zeros_like(S)
    psi = np.zeros_like(S)
    rem = np.zeros_like(S)
    err = _abi.ErrorC()
    _check(lib().orc_build_preconditioner(_dt(dtype), int(kind), int(order), K, nb, _ptr(S),
                                          _ptr(ti), _ptr(phi), _ptr(psi), _ptr(rem),
                                          C.byref(err)), err)
    kind = PrecondKind(kind)
    P = Preconditioner(kind=kind, order=order if kind == PrecondKind.poly_split else 0)
    if kind != PrecondKind.identity:
        P.phi_inv = BlockTriMatrix(data=phi)
    if kind == PrecondKind.poly_split:
        P.stair_psi = BlockTriMatrix(data=psi)
        P.remainder = BlockTriMatrix(data=rem)
        P.S = schur.S
    return P


def build_identity():
    from paper_2309_08079_b200.types import Preconditioner
    return Preconditioner()


def build_block_jacobi(s):
    return build_preconditioner(s, PrecondKind.block_jacobi)


def build_stair(s):
    return build_preconditioner(s, PrecondKind.stair)


def build_symmetric_stair(s):
    return build_preconditioner(s, PrecondKind.symmetric_stair)


def build_poly_split(s, order):
    return build_preconditioner(s, PrecondKind.poly_split, order)


def _precond_args(P, K, nb):
    phi = None if P.kind == PrecondKind.identity else _f64(P.phi_inv.data)
    S = None
    if P.kind == PrecondKind.poly_split:
        S = _f64(P.S.data)
    return phi, S


def apply_preconditioner(P, r, dtype=np.float64) -> np.ndarray:
    r = _f64(r)
    if P.kind == PrecondKind.identity:
        return r.copy()
    K, nb = P.phi_inv.block_rows(), P.phi_inv.block_dim()
    if r.size != K * nb:
        raise ValueError(f"apply_preconditioner: expected vector of length {K * nb}, "
                         f"got {r.size}")
    phi, S = _precond_args(P, K, nb)
    out = np.zeros(K * nb)
    err = _abi.ErrorC()
    _check(lib().orc_apply_preconditioner(_dt(dtype), int(P.kind), int(P.order), K, nb,
                                          _ptr(S), _ptr(phi), _ptr(r), _ptr(out),
                                          C.byref(err)), err)
    return out


# ---------------------------------------------------------------- block_tri.hpp
def matvec(M: BlockTriMatrix, x) -> np.ndarray:
    d = _f64(M.data)
    x = _f64(x)
    y = np.zeros(d.shape[0] * d.shape[2])
    err = _abi.ErrorC()
    _check(lib().orc_matvec(d.shape[0], d.shape[2], _ptr(d), _ptr(x), x.size, _ptr(y),
                            C.byref(err)), err)
    return y


def max_asymmetry(M: BlockTriMatrix) -> float:
    d = _f64(M.data)
    return lib().orc_max_asymmetry(d.shape[0], d.shape[2], _ptr(d))


def cholesky_solve(M: BlockTriMatrix, rhs) -> np.ndarray:
    d = _f64(M.data)
    rhs = _f64(rhs)
    x = np.zeros(d.shape[0] * d.shape[2])
    err = _abi.ErrorC()
    _check(lib().orc_cholesky_solve(d.shape[0], d.shape[2], _ptr(d), _ptr(rhs), _ptr(x),
                                    C.byref(err)), err)
    return x


# ---------------------------------------------------------------- pcg.hpp
def _max_iter(cfg, dim):
    return cfg.max_iter if cfg.max_iter > 0 else dim


def pcg_solve_auto(S: BlockTriMatrix, P, gamma, lambda0, cfg: PcgConfig = None,
                   dtype=np.float64) -> PcgResult:
    cfg = cfg or PcgConfig()
    d = _f64(S.data)
    K, nb = d.shape[0], d.shape[2]
    gamma = _f64(gamma)
    lambda0 = _f64(lambda0)
    phi, Sp = _precond_args(P, K, nb)
    lam = np.zeros(K * nb)
    rep = _abi.SolveReportC()
    trace = np.zeros(max(1, _max_iter(cfg, K * nb)))
    err = _abi.ErrorC()
    c = cfg.to_c()
    _check(lib().orc_pcg_solve(_dt(dtype), K, nb, _ptr(d), int(P.kind), int(P.order),
                               _ptr(phi), _ptr(gamma), gamma.size, _ptr(lambda0), lambda0.size,
                               C.byref(c), _ptr(lam), C.byref(rep), _ptr(trace), C.byref(err)),
           err)
    return PcgResult(lam, SolveReport.from_c(rep, trace))


def pcg_solve(S, P, gamma, lambda0, cfg=None, dtype=np.float64) -> PcgResult:
    from paper_2309_08079_b200.types import PcgVariant
    cfg = PcgConfig(**{**(cfg or PcgConfig()).__dict__, "variant": PcgVariant.sequential})
    return pcg_solve_auto(S, P, gamma, lambda0, cfg, dtype)


def pcg_solve_block_parallel(S, P, gamma, lambda0, cfg=None, dtype=np.float64) -> PcgResult:
    from paper_2309_08079_b200.types import PcgVariant
    cfg = PcgConfig(**{**(cfg or PcgConfig()).__dict__, "variant": PcgVariant.block_parallel})
    return pcg_solve_auto(S, P, gamma, lambda0, cfg, dtype)


def solve(kkt: KKTSystem, kind=PrecondKind.symmetric_stair, order: int = 1,
          cfg: PcgConfig = None, lambda0=None, dtype=np.float64) -> PcgResult:
    """build_schur -> build_preconditioner -> pcg_solve_auto."""
    cfg = cfg or PcgConfig()
    kkt = kkt.astype(np.float64)
    D = kkt.dual_dim()
    lam = np.zeros(D)
    rep = _abi.SolveReportC()
    trace = np.zeros(max(1, _max_iter(cfg, D)))
    err = _abi.ErrorC()
    c = cfg.to_c()
    l0 = None if lambda0 is None else _f64(lambda0)
    _check(lib().orc_solve(_dt(dtype), C.byref(kkt.to_c()), int(kind), int(order), C.byref(c),
                           _ptr(l0), _ptr(lam), C.byref(rep), _ptr(trace), C.byref(err)), err)
    return PcgResult(lam, SolveReport.from_c(rep, trace))


def solve_batch(kkt_batch: KKTSystem, kind=PrecondKind.symmetric_stair, order: int = 1,
                cfg: PcgConfig = None, threads: int = 0, dtype=np.float64,
                want_lambda: bool = True, native: bool = False):
    """cmd_bench_pcg-style parallel_for over instances. Returns (seconds, lambda, reports)."""
    cfg = cfg or PcgConfig()
    kb = kkt_batch.astype(np.float64)
    B = kb.batch
    lam = np.zeros((B, kb.dual_dim())) if want_lambda else None
    reps = (_abi.SolveReportC * B)()
    err = _abi.ErrorC()
    c = cfg.to_c()
    secs = lib(native).orc_solve_batch(_dt(dtype), B, C.byref(kb.to_c()), int(kind), int(order),
                                 C.byref(c), int(threads), _ptr(lam), reps, C.byref(err))
    if secs < 0:
        _check(err.code, err)
    return secs, lam, [SolveReport.from_c(r) for r in reps]


def reconstruct_primal(kkt: KKTSystem, lam, dtype=np.float64) -> np.ndarray:
    kkt = kkt.astype(np.float64)
    lam = _f64(lam)
    dz = np.zeros(kkt.primal_dim())
    err = _abi.ErrorC()
    _check(lib().orc_reconstruct_primal(_dt(dtype), C.byref(kkt.to_c()), _ptr(lam), lam.size,
                                        _ptr(dz), C.byref(err)), err)
    return dz
