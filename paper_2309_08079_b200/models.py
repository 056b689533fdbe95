"""Dynamics models, tracking cost and the KKT linearisation — the host side of
named-model problem files (proj/include/trajopt/models.hpp, proj/src/models.cpp,
proj/src/kkt.cpp:83-127, proj/src/problem_io.cpp:194-216).

Host-side per-knot arithmetic on n <= 4 states, as in the reference; the C++
mirror (with the SQP / NMPC loops) is include/trajopt_b200_sqp.hpp. The solve
itself always goes through the C-ABI (api.py).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._lib import load
from .types import KKTSystem


def uniform_draws(seed: int, count: int, lo: float, hi: float) -> np.ndarray:
    """UniformRng(seed) draws in order (random_problem.hpp:13-37), from libb2p."""
    out = np.zeros(max(count, 1))
    err = _abi.ErrorC()
    rc = load().b2p_uniform_draws(int(seed), int(count), float(lo), float(hi),
                                  out.ctypes.data, C.byref(err))
    if rc:
        raise ValueError(err.message.decode())
    return out[:count]


class DynamicsModel:  # models.hpp:14-27
    n = 0
    m = 0
    model_name = ""

    def state_dim(self) -> int:
        return self.n

    def control_dim(self) -> int:
        return self.m

    def name(self) -> str:
        return self.model_name

    def step(self, x, u, h) -> np.ndarray:
        raise NotImplementedError

    def jacobians(self, x, u, h):
        raise NotImplementedError


class DoubleIntegrator(DynamicsModel):  # models.cpp:14-34
    n, m, model_name = 2, 1, "double_integrator"

    def step(self, x, u, h):
        return np.array([x[0] + h * x[1], x[1] + h * u[0]])

    def jacobians(self, x, u, h):
        A = np.eye(2)
        A[0, 1] = h
        B = np.zeros((2, 1))
        B[1, 0] = h
        return A, B


class Pendulum(DynamicsModel):  # models.cpp:36-66
    n, m, model_name = 2, 1, "pendulum"
    mass, length, gravity = 1.0, 1.0, 9.81

    def step(self, x, u, h):
        ml2 = self.mass * self.length * self.length
        return np.array([x[0] + h * x[1],
                         x[1] + h * (u[0] - self.mass * self.gravity * self.length *
                                     math.sin(x[0])) / ml2])

    def jacobians(self, x, u, h):
        A = np.eye(2)
        A[0, 1] = h
        A[1, 0] = -h * self.gravity * math.cos(x[0]) / self.length
        B = np.zeros((2, 1))
        B[1, 0] = h / (self.mass * self.length * self.length)
        return A, B


class Cartpole(DynamicsModel):  # models.cpp:68-149
    n, m, model_name = 4, 1, "cartpole"
    mc, mp, length, gravity = 1.0, 0.1, 0.5, 9.81

    def step(self, x, u, h):
        s, c = math.sin(x[1]), math.cos(x[1])
        total = self.mc + self.mp
        temp = (u[0] + self.mp * self.length * x[3] * x[3] * s) / total
        tdd = (self.gravity * s - c * temp) / (self.length * (4.0 / 3.0 - self.mp * c * c / total))
        xdd = temp - self.mp * self.length * tdd * c / total
        return np.array([x[0] + h * x[2], x[1] + h * x[3], x[2] + h * xdd, x[3] + h * tdd])

    def jacobians(self, x, u, h):
        theta, td, f = x[1], x[3], u[0]
        s, c = math.sin(theta), math.cos(theta)
        mp, L, g = self.mp, self.length, self.gravity
        total = self.mc + mp
        temp = (f + mp * L * td * td * s) / total
        num = g * s - c * temp
        den = L * (4.0 / 3.0 - mp * c * c / total)
        tdd = num / den
        dtemp_dtheta = mp * L * td * td * c / total
        dtemp_dtd = 2.0 * mp * L * td * s / total
        dtemp_df = 1.0 / total
        dnum_dtheta = g * c + s * temp - c * dtemp_dtheta
        dnum_dtd = -c * dtemp_dtd
        dnum_df = -c * dtemp_df
        dden_dtheta = 2.0 * L * mp * c * s / total
        dtdd_dtheta = (dnum_dtheta * den - num * dden_dtheta) / (den * den)
        dtdd_dtd = dnum_dtd / den
        dtdd_df = dnum_df / den
        scale = mp * L / total
        A = np.eye(4)
        A[0, 2] = h
        A[1, 3] = h
        A[2, 1] = h * (dtemp_dtheta - scale * (dtdd_dtheta * c - tdd * s))
        A[2, 3] = h * (dtemp_dtd - scale * c * dtdd_dtd)
        A[3, 1] = h * dtdd_dtheta
        A[3, 3] = 1.0 + h * dtdd_dtd
        B = np.zeros((4, 1))
        B[2, 0] = h * (dtemp_df - scale * c * dtdd_df)
        B[3, 0] = h * dtdd_df
        return A, B


_MODELS = {"double_integrator": DoubleIntegrator, "pendulum": Pendulum, "cartpole": Cartpole}


def make_model(name: str) -> DynamicsModel:  # models.cpp:155-161
    if name not in _MODELS:
        raise ValueError(f'unknown model "{name}" (expected double_integrator, pendulum, or '
                         'cartpole)')
    return _MODELS[name]()


@dataclass
class CostModel:  # models.hpp:35-50
    Wx: np.ndarray
    Wu: np.ndarray
    WN: np.ndarray
    goals: list = field(default_factory=list)  # 1 (broadcast) or N+1

    def goal(self, knot: int) -> np.ndarray:
        return self.goals[0] if len(self.goals) == 1 else self.goals[knot]


def quadratic_tracking_cost(Wx, Wu, WN, goal) -> CostModel:  # models.cpp:163-171
    return CostModel(np.asarray(Wx, float), np.asarray(Wu, float), np.asarray(WN, float),
                     [np.asarray(goal, float)])


@dataclass
class Trajectory:  # trajectory.hpp:9-17
    h: float = 0.01
    X: list = field(default_factory=list)
    U: list = field(default_factory=list)
    lam: np.ndarray | None = None

    def horizon(self) -> int:
        return len(self.U)


def eval_cost(cost: CostModel, X, U) -> float:  # models.cpp:173-189
    if len(X) != len(U) + 1:
        raise ValueError(f"eval_cost: need N+1 states and N controls, got {len(X)} states and "
                         f"{len(U)} controls")
    N = len(U)
    total = 0.0
    for k in range(N):
        dx = X[k] - cost.goal(k)
        total += 0.5 * dx @ (cost.Wx @ dx) + 0.5 * U[k] @ (cost.Wu @ U[k])
    dxN = X[N] - cost.goal(N)
    return float(total + 0.5 * dxN @ (cost.WN @ dxN))


def rollout(model: DynamicsModel, x0, controls, h) -> Trajectory:  # models.cpp:191-200
    t = Trajectory(h=h, X=[np.asarray(x0, float)], U=[np.asarray(u, float) for u in controls])
    for u in t.U:
        t.X.append(model.step(t.X[-1], u, h))
    return t


def _regularize_spd(W: np.ndarray) -> np.ndarray:  # kkt.cpp:20-25
    lower = np.tril(W) + np.tril(W, -1).T  # SelfAdjointEigenSolver reads the lower triangle
    if np.linalg.eigvalsh(lower).min() < 1e-8:
        W = W + 1e-6 * np.eye(W.shape[0])
    return W


def assemble_kkt(traj: Trajectory, model: DynamicsModel, cost: CostModel, x_s) -> KKTSystem:
    """kkt.cpp:83-127 — linearise the dynamics and expand the cost around traj."""
    N, n, m = traj.horizon(), model.state_dim(), model.control_dim()
    if len(traj.X) != N + 1:
        raise ValueError(f"assemble_kkt: trajectory needs N+1 states, got {len(traj.X)} for "
                         f"N = {N}")
    k = KKTSystem.allocate(N, n, m)
    k.x_s[:] = x_s
    k.x0[:] = traj.X[0]
    for i in range(N + 1):
        terminal = i == N
        Q = cost.WN if terminal else cost.Wx
        q = Q @ (traj.X[i] - cost.goal(i))
        Q = _regularize_spd(Q)
        if not terminal:
            R = _regularize_spd(cost.Wu)
            r = cost.Wu @ traj.U[i]
            A, B = model.jacobians(traj.X[i], traj.U[i], traj.h)
            e = traj.X[i + 1] - model.step(traj.X[i], traj.U[i], traj.h)
            if not all(np.isfinite(a).all() for a in (A, B, e, R, r)):
                raise RuntimeError(f"assemble_kkt: non-finite linearization at knot {i}")
            k.R[i], k.r[i], k.A[i], k.B[i], k.e[i] = R, r, A, B, e
        if not (np.isfinite(Q).all() and np.isfinite(q).all()):
            raise RuntimeError(f"assemble_kkt: non-finite cost expansion at knot {i}")
        k.Q[i], k.q[i] = Q, q
    return k


__all__ = ["uniform_draws", "DynamicsModel", "DoubleIntegrator", "Pendulum", "Cartpole",
           "make_model", "CostModel", "quadratic_tracking_cost", "Trajectory", "eval_cost",
           "rollout", "assemble_kkt"]
