"""Problem files and result rows of the reference's solve-qp / bench-pcg path
(proj/include/trajopt/problem_io.hpp, proj/src/problem_io.cpp:78-248,
proj/include/trajopt/format.hpp) — SURVEY §8(f) rank 4.

Host-side file formats only (no compute): the explicit-model JSON problem
document, the benchmark CSV row schema, and `solve_qp`, which mirrors
`cmd_solve_qp` (proj/tools/trajopt_cli.cpp:88-125) on the B200 path
(build_schur -> build_preconditioner -> pcg_solve_auto through the C-ABI).
Named dynamics models (model != "explicit") are linearised around the seeded
rollout (models.py, problem_io.cpp:194-216) and solved on the same path.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .types import KKTSystem, PcgConfig, PcgVariant, SolveReport, parse_precond


class InputError(RuntimeError):
    """problem_io.hpp:37-40 — malformed input files; the message carries line/column."""


def format9(v: float) -> str:
    """format.hpp:9-13 — locale-independent "%.9g"."""
    return "%.9g" % v


def result_row_header() -> str:  # problem_io.cpp:233-236
    return ("experiment,N,n,m,preconditioner,epsilon,variant,iterations,exit_eta,converged,"
            "wall_time_us,seed")


def result_row(experiment: str, knot_points: int, n: int, m: int, preconditioner: str,
               epsilon: float, variant: str, report: SolveReport, seed: int,
               zero_times: bool) -> str:  # problem_io.cpp:238-248
    wall_us = 0 if zero_times else int(report.wall_time * 1e6)
    return ",".join([experiment, str(knot_points), str(n), str(m), preconditioner,
                     format9(epsilon), variant, str(report.iterations), format9(report.exit_eta),
                     "true" if report.converged else "false", str(wall_us), str(seed)])


@dataclass
class ProblemFile:  # problem_io.hpp:16-31
    n: int = 0
    m: int = 0
    N: int = 0
    h: float = 0.01
    model: str = "explicit"
    seed: int = 0
    x_s: np.ndarray | None = None
    x0: np.ndarray | None = None
    wx: float = 1.0
    wu: float = 0.1
    wn: float = 10.0
    goal: np.ndarray | None = None
    knots: list = field(default_factory=list)  # dicts of Q, q (+ R, r, A, B, e for k < N)


def _matrix(j, what: str) -> np.ndarray:  # problem_io.cpp:35-49
    if not isinstance(j, list) or not j or not isinstance(j[0], list):
        raise InputError(f"problem file: {what} must be a nested list (row-major)")
    cols = len(j[0])
    for row in j:
        if len(row) != cols:
            raise InputError(f"problem file: ragged rows in {what}")
    return np.array(j, dtype=np.float64).reshape(len(j), cols)


def _vector(j, what: str) -> np.ndarray:  # problem_io.cpp:51-58
    if not isinstance(j, list):
        raise InputError(f"problem file: {what} must be a list")
    return np.array(j, dtype=np.float64).reshape(-1)


def load_problem(path: str) -> ProblemFile:  # problem_io.cpp:74-141
    try:
        with open(path, "rb") as fh:
            text = fh.read().decode()
    except OSError:
        raise InputError(f"cannot open problem file: {path}") from None
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise InputError(f"malformed JSON in {path} at line {e.lineno}, column {e.colno}: "
                         f"{e.msg}") from None
    try:
        pf = ProblemFile(n=int(doc["n"]), m=int(doc["m"]), N=int(doc["N"]))
        pf.h = float(doc.get("h", 0.01))
        pf.model = str(doc.get("model", "explicit"))
        pf.seed = int(doc.get("seed", 0))
        if "x_s" in doc:
            pf.x_s = _vector(doc["x_s"], "x_s")
        if "x0" in doc:
            pf.x0 = _vector(doc["x0"], "x0")
        if "cost" in doc:
            c = doc["cost"]
            pf.wx, pf.wu, pf.wn = (float(c.get("wx", 1.0)), float(c.get("wu", 0.1)),
                                   float(c.get("wn", 10.0)))
            if "goal" in c:
                pf.goal = _vector(c["goal"], "cost.goal")
        for kj in doc.get("knots", []):
            kd = {"Q": _matrix(kj["Q"], "knots.Q"), "q": _vector(kj["q"], "knots.q")}
            if "R" in kj:
                kd.update(R=_matrix(kj["R"], "knots.R"), r=_vector(kj["r"], "knots.r"),
                          A=_matrix(kj["A"], "knots.A"), B=_matrix(kj["B"], "knots.B"),
                          e=_vector(kj["e"], "knots.e"))
            pf.knots.append(kd)
    except (KeyError, TypeError, ValueError) as e:
        raise InputError(f"problem file {path}: {e}") from None
    if pf.n < 1 or pf.m < 0 or pf.N < 0:
        raise InputError(f"problem file: invalid dimensions n={pf.n} m={pf.m} N={pf.N}")
    if pf.model == "explicit" and len(pf.knots) != pf.N + 1:
        raise InputError(f"problem file: explicit model needs N+1 knots, got {len(pf.knots)} "
                         f"for N = {pf.N}")
    return pf


def problem_to_json(pf: ProblemFile) -> str:  # problem_io.cpp:143-176
    """nlohmann::json dump(2) layout: keys sorted (std::map), two-space indent."""
    doc = {"n": pf.n, "m": pf.m, "N": pf.N, "h": pf.h, "model": pf.model, "seed": pf.seed}
    if pf.x_s is not None and len(pf.x_s):
        doc["x_s"] = [float(x) for x in pf.x_s]
    if pf.x0 is not None and len(pf.x0):
        doc["x0"] = [float(x) for x in pf.x0]
    if pf.model != "explicit":
        doc["cost"] = {"wx": pf.wx, "wu": pf.wu, "wn": pf.wn}
        if pf.goal is not None and len(pf.goal):
            doc["cost"]["goal"] = [float(x) for x in pf.goal]
    if pf.knots:
        ks = []
        for kd in pf.knots:
            kj = {"Q": np.asarray(kd["Q"]).tolist(), "q": np.asarray(kd["q"]).tolist()}
            if "R" in kd and np.asarray(kd["R"]).size:
                for f in ("R", "r", "A", "B", "e"):
                    kj[f] = np.asarray(kd[f]).tolist()
            ks.append(kj)
        doc["knots"] = ks
    return json.dumps(doc, indent=2, sort_keys=True) + "\n"


def save_problem(pf: ProblemFile, path: str) -> None:  # problem_io.cpp:178-180
    with open(path, "w") as fh:
        fh.write(problem_to_json(pf))


def problem_to_kkt(pf: ProblemFile) -> KKTSystem:  # problem_io.cpp:182-216
    if pf.model != "explicit":
        return _named_model_kkt(pf)
    n, m, N = pf.n, pf.m, pf.N
    k = KKTSystem.allocate(N, n, m)
    for i, kd in enumerate(pf.knots):
        k.Q[i] = kd["Q"]
        k.q[i] = kd["q"]
        if i < N:
            k.R[i] = kd["R"]
            k.r[i] = kd["r"]
            k.A[i] = kd["A"]
            k.B[i] = kd["B"]
            k.e[i] = kd["e"]
    k.x_s[:] = pf.x_s if pf.x_s is not None and len(pf.x_s) else 0.0
    k.x0[:] = pf.x0 if pf.x0 is not None and len(pf.x0) else 0.0
    return k


def _named_model_kkt(pf: ProblemFile) -> KKTSystem:  # problem_io.cpp:194-216
    """Linearise a named model around the rollout from x_s: zero controls for seed 0,
    else controls drawn uniform in [-0.1, 0.1] from UniformRng(seed)."""
    from . import models
    try:
        model = models.make_model(pf.model)
    except ValueError as e:
        raise InputError(str(e)) from None
    if model.state_dim() != pf.n or model.control_dim() != pf.m:
        raise InputError(f"problem file: model {pf.model} has dims n={model.state_dim()} "
                         f"m={model.control_dim()}, file says n={pf.n} m={pf.m}")
    x_start = pf.x_s if pf.x_s is not None and len(pf.x_s) else np.zeros(pf.n)
    goal = pf.goal if pf.goal is not None and len(pf.goal) else np.zeros(pf.n)
    cost = models.quadratic_tracking_cost(pf.wx * np.eye(pf.n), pf.wu * np.eye(pf.m),
                                          pf.wn * np.eye(pf.n), goal)
    if pf.seed != 0:
        u = models.uniform_draws(pf.seed, pf.N * pf.m, -0.1, 0.1).reshape(pf.N, pf.m)
        controls = [u[k] for k in range(pf.N)]
    else:
        controls = [np.zeros(pf.m) for _ in range(pf.N)]
    traj = models.rollout(model, x_start, controls, pf.h)
    return models.assemble_kkt(traj, model, cost, x_start)


def problem_from_kkt(kkt: KKTSystem, seed: int) -> ProblemFile:  # problem_io.cpp:218-229
    pf = ProblemFile(n=kkt.n, m=kkt.m, N=kkt.N, model="explicit", seed=int(seed),
                     x_s=np.array(kkt.x_s, dtype=np.float64),
                     x0=np.array(kkt.x0, dtype=np.float64))
    for i in range(kkt.N + 1):
        kd = {"Q": np.array(kkt.Q[i]), "q": np.array(kkt.q[i])}
        if i < kkt.N:
            kd.update(R=np.array(kkt.R[i]), r=np.array(kkt.r[i]), A=np.array(kkt.A[i]),
                      B=np.array(kkt.B[i]), e=np.array(kkt.e[i]))
        pf.knots.append(kd)
    return pf


def parse_variant(name: str) -> PcgVariant:  # trajopt_cli.cpp:55-59
    if name == "sequential":
        return PcgVariant.sequential
    if name in ("parallel", "block_parallel"):
        return PcgVariant.block_parallel
    raise InputError(f'unknown variant "{name}" (expected sequential|parallel)')


def solve_qp(path: str, precond: str = "symstair", eps: float = 1e-4,
             variant: str = "sequential", max_iter: int = 0, seed: int = 0,
             deterministic: bool = False) -> str:
    """cmd_solve_qp (trajopt_cli.cpp:88-112) on the B200 path: header + one CSV row."""
    from . import api
    pf = load_problem(path)
    kkt = problem_to_kkt(pf)
    schur = api.build_schur(kkt)
    kind, order = parse_precond(precond)
    P = api.build_preconditioner(schur, kind, max(order, 1))
    var = parse_variant(variant)
    cfg = PcgConfig(epsilon=eps, max_iter=max_iter, variant=var,
                    deterministic_reductions=deterministic)
    res = api.pcg_solve_auto(schur.S, P, schur.gamma, np.zeros(schur.S.dim()), cfg)
    vname = "sequential" if var == PcgVariant.sequential else "block_parallel"
    return (result_row_header() + "\n" +
            result_row("solve_qp", kkt.N + 1, kkt.n, kkt.m, precond, eps, vname, res.report,
                       seed, deterministic) + "\n")


__all__ = ["InputError", "format9", "result_row_header", "result_row", "ProblemFile",
           "load_problem", "problem_to_json", "save_problem", "problem_to_kkt",
           "problem_from_kkt", "parse_variant", "solve_qp"]
