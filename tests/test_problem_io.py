"""Problem files and CSV rows (problem_io.cpp:78-248, format.hpp),
with the reference's CLI row KAT (test_cli.cpp:44-57)."""
import json

import numpy as np
import pytest

from paper_2309_08079_b200 import problem_io as pio
from paper_2309_08079_b200.types import SolveReport


def test_format9_and_row_schema():
    assert pio.format9(1e-12) == "1e-12"
    assert pio.format9(0.1) == "0.1"
    assert pio.format9(1.0 / 3.0) == "0.333333333"
    rep = SolveReport(iterations=7, exit_eta=1.5e-9, converged=True, wall_time=0.000123456)
    row = pio.result_row("solve_qp", 32, 14, 7, "symstair", 1e-8, "sequential", rep, 5, False)
    assert row == "solve_qp,32,14,7,symstair,1e-08,sequential,7,1.5e-09,true,123,5"
    assert pio.result_row("x", 1, 2, 0, "identity", 1e-4, "block_parallel", rep, 0,
                          True).endswith(",true,0,0")
    assert pio.result_row_header().split(",") == [
        "experiment", "N", "n", "m", "preconditioner", "epsilon", "variant", "iterations",
        "exit_eta", "converged", "wall_time_us", "seed"]


def test_problem_round_trip(tmp_path, orc):
    kkt = orc.random_trajectory_kkt(17, 8, 2, 1)
    path = str(tmp_path / "p.json")
    pio.save_problem(pio.problem_from_kkt(kkt, 17), path)
    doc = json.load(open(path))
    assert list(doc) == sorted(doc)  # nlohmann std::map key order
    pf = pio.load_problem(path)
    assert (pf.n, pf.m, pf.N, pf.seed, pf.model) == (2, 1, 8, 17, "explicit")
    back = pio.problem_to_kkt(pf)
    for a, b in zip(back.arrays(), kkt.arrays()):
        assert np.array_equal(a, b)


def test_input_errors(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text("{ not json")
    with pytest.raises(pio.InputError, match=r"malformed JSON in .* at line 1, column 3"):
        pio.load_problem(str(bad))
    short = tmp_path / "short.json"
    short.write_text(json.dumps({"n": 2, "m": 0, "N": 1, "knots": [{"Q": [[1, 0], [0, 1]],
                                                                    "q": [0, 0]}]}))
    with pytest.raises(pio.InputError, match="explicit model needs N\\+1 knots, got 1 for N = 1"):
        pio.load_problem(str(short))
    ragged = tmp_path / "ragged.json"
    ragged.write_text(json.dumps({"n": 2, "m": 0, "N": 0, "knots": [{"Q": [[1, 0], [0]],
                                                                     "q": [0, 0]}]}))
    with pytest.raises(pio.InputError, match="ragged rows in knots.Q"):
        pio.load_problem(str(ragged))
    with pytest.raises(pio.InputError, match='unknown variant "fast"'):
        pio.parse_variant("fast")
    with pytest.raises(pio.InputError, match="cannot open problem file"):
        pio.load_problem(str(tmp_path / "missing.json"))


@pytest.mark.gpu
def test_solve_qp_identity_system_row_kat(tmp_path):  # test_cli.cpp:44-57
    path = tmp_path / "identity.json"
    path.write_text('{"n": 2, "m": 0, "N": 0, "model": "explicit", "seed": 0,'
                    ' "x_s": [0.5, -0.2],'
                    ' "knots": [{"Q": [[1.0, 0.0], [0.0, 1.0]], "q": [1.0, 0.0]}]}')
    out = pio.solve_qp(str(path), eps=1e-12)
    assert out.startswith(pio.result_row_header())
    assert "solve_qp,1,2,0,symstair,1e-12,sequential,1," in out
    assert ",true," in out


@pytest.mark.gpu
def test_solve_qp_random_instance_agrees_with_oracle(tmp_path, orc):  # test_cli.cpp:59-64
    from paper_2309_08079_b200.types import PcgConfig, PrecondKind
    kkt = orc.random_trajectory_kkt(17, 8, 2, 1)
    path = str(tmp_path / "r.json")
    pio.save_problem(pio.problem_from_kkt(kkt, 17), path)
    out = pio.solve_qp(path, eps=1e-10, max_iter=2000, seed=17, deterministic=True)
    want = orc.solve(kkt, PrecondKind.symmetric_stair, cfg=PcgConfig(epsilon=1e-10,
                                                                     max_iter=2000))
    row = out.splitlines()[1].split(",")
    assert int(row[7]) == want.report.iterations and row[9] == "true" and row[10] == "0"


def test_uniform_draws_match_the_oracle_rng(orc):  # random_problem.hpp:13-37
    from paper_2309_08079_b200.models import uniform_draws
    assert np.array_equal(uniform_draws(5, 12, -0.1, 0.1), orc.UniformRng(5).vector(12, -0.1, 0.1))


def test_named_model_problem_linearizes_around_seeded_rollout(tmp_path):  # test_io.cpp:60-76
    pf = pio.ProblemFile(n=2, m=1, N=6, h=0.02, model="pendulum", seed=5, x_s=np.zeros(2))
    kkt = pio.problem_to_kkt(pf)
    assert (kkt.N, kkt.n, kkt.m) == (6, 2, 1)
    assert np.abs(kkt.e).max() <= 1e-14  # rollout linearization: defects vanish
    assert np.abs(kkt.x0 - kkt.x_s).max() == 0.0
    # seed 5 controls are nonzero and drive q/r through the default weights
    assert np.abs(kkt.r).max() > 0 and np.allclose(kkt.R, 0.1)
    # dims mismatch and unknown models are InputErrors
    with pytest.raises(pio.InputError, match="model cartpole has dims n=4 m=1, file says n=2 m=1"):
        pio.problem_to_kkt(pio.ProblemFile(n=2, m=1, N=3, model="cartpole"))
    with pytest.raises(pio.InputError, match='unknown model "segway"'):
        pio.problem_to_kkt(pio.ProblemFile(n=2, m=1, N=3, model="segway"))
    # the named-model document round-trips through the JSON writer
    pf.goal = np.array([0.5, 0.0])
    path = str(tmp_path / "named.json")
    pio.save_problem(pf, path)
    back = pio.load_problem(path)
    assert back.model == "pendulum" and back.seed == 5 and np.array_equal(back.goal, pf.goal)
    assert pio.problem_to_json(back) == open(path).read()


def test_models_jacobians_match_finite_differences(orc):  # test_models.cpp:112-122
    from paper_2309_08079_b200 import models
    rng = orc.UniformRng(77)
    for name in ("double_integrator", "pendulum", "cartpole"):
        mdl = models.make_model(name)
        for _ in range(100):
            x = rng.vector(mdl.state_dim(), -2.0, 2.0)
            u = rng.vector(mdl.control_dim(), -2.0, 2.0)
            A, B = mdl.jacobians(x, u, 0.02)
            eps = 1e-6
            Af = np.stack([(mdl.step(x + eps * e, u, 0.02) - mdl.step(x - eps * e, u, 0.02)) /
                           (2 * eps) for e in np.eye(len(x))], axis=1)
            Bf = np.stack([(mdl.step(x, u + eps * e, 0.02) - mdl.step(x, u - eps * e, 0.02)) /
                           (2 * eps) for e in np.eye(len(u))], axis=1)
            scale = max(1.0, np.abs(Af).max(), np.abs(Bf).max())
            assert max(np.abs(A - Af).max(), np.abs(B - Bf).max()) / scale <= 1e-5
    with pytest.raises(ValueError, match="unknown model"):
        models.make_model("segway")


def test_assemble_kkt_kats(orc):  # test_kkt.cpp:30-78,144-157 + kkt.cpp:20-25 ridge
    from paper_2309_08079_b200 import models
    di = models.make_model("double_integrator")
    I2, I1 = np.eye(2), np.eye(1)
    t = models.Trajectory(h=0.01, X=[np.zeros(2)] * 5, U=[np.zeros(1)] * 4)
    k = models.assemble_kkt(t, di, models.quadratic_tracking_cost(I2, I1, I2, np.zeros(2)),
                            np.zeros(2))
    assert np.abs(k.e).max() == 0.0 and np.abs(k.constraint_rhs()).max() == 0.0
    goal = np.array([0.5, -0.25])
    rng = orc.UniformRng(4)
    t = models.Trajectory(h=0.01, X=[rng.vector(2, -1.0, 1.0) for _ in range(3)],
                          U=[rng.vector(1, -1.0, 1.0) for _ in range(2)])
    k = models.assemble_kkt(t, di, models.quadratic_tracking_cost(I2, I1, I2, goal), t.X[0])
    for i in range(3):
        assert np.abs(k.q[i] - (t.X[i] - goal)).max() <= 1e-15
    t.X[1] = np.array([np.nan, 0.0])
    with pytest.raises(RuntimeError, match="knot"):
        models.assemble_kkt(t, di, models.quadratic_tracking_cost(I2, I1, I2, goal), t.X[0])
    Wx = np.diag([1.0, 0.0])  # singular: ridge after q is formed
    t = models.Trajectory(h=0.01, X=[np.ones(2)] * 2, U=[np.zeros(1)])
    k = models.assemble_kkt(t, di, models.quadratic_tracking_cost(Wx, I1, I2, np.zeros(2)),
                            np.zeros(2))
    assert k.Q[0][1, 1] == 1e-6 and k.Q[0][0, 0] == 1.0 + 1e-6 and k.q[0][1] == 0.0
    assert k.Q[1][0, 0] == 1.0 and k.R[0][0, 0] == 1.0


@pytest.mark.gpu
def test_solve_qp_named_model_agrees_with_oracle(tmp_path, orc):  # cmd_solve_qp on a model file
    from paper_2309_08079_b200.types import PcgConfig, PrecondKind
    pf = pio.ProblemFile(n=4, m=1, N=40, h=0.02, model="cartpole", seed=9,
                         x_s=np.array([0.0, 0.2, 0.0, 0.0]), goal=np.zeros(4))
    path = str(tmp_path / "cp.json")
    pio.save_problem(pf, path)
    out = pio.solve_qp(path, eps=1e-10, max_iter=2000, seed=9, deterministic=True)
    want = orc.solve(pio.problem_to_kkt(pf), PrecondKind.symmetric_stair,
                     cfg=PcgConfig(epsilon=1e-10, max_iter=2000))
    row = out.splitlines()[1].split(",")
    assert row[:4] == ["solve_qp", "41", "4", "1"]
    assert int(row[7]) == want.report.iterations and row[9] == "true"
