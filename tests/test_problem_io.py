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
