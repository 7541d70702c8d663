"""Drop-in names the reference package exports (qapswarm/__init__.py:6-58)
that run without a GPU: assignments and goal evaluation (core.py), QAPLIB
instance / solution I/O (qaplib.py), the bundled instances (datasets.py),
the stream keys (streams.py) and the CLI's validate / flag handling
(cli.py).  Behaviour follows the reference's own tests (pkg/tests/
test_core.py, test_qaplib.py, test_cli.py, test_streams.py), restated."""

import itertools

import numpy as np
import pytest

import paper_1504_05158_b200 as qsb
from paper_1504_05158_b200 import cli, streams
from oracle import oracle as orc


def test_reference_names_exported():
    names = ["QapInstance", "ReferenceSolution", "parse_instance", "parse_reference_solution",
             "format_instance", "format_reference_solution", "load_instance",
             "load_reference_solution", "Assignment", "evaluate_cost", "matrix_to_assignment",
             "gap", "PsoCoefficients", "SV_MODES", "SX_MODES", "SwarmBestTable",
             "MigrationEvent", "migrate", "SolverConfig", "PopulationState", "RunResult",
             "init_population", "step", "run", "projected_buffer_bytes", "IterationStats",
             "percentile", "pmf", "collect", "export_csv", "write_solution", "data_path",
             "list_bundled", "load_bundled", "load_bundled_solution"]
    missing = [n for n in names if not hasattr(qsb, n)]
    assert not missing, missing


# ------------------------------------------------------------------ core
def test_assignment_matrix_roundtrip():
    rng = np.random.default_rng(0)
    for n in (2, 5, 12):
        a = qsb.Assignment(rng.permutation(n))
        x = a.matrix
        assert x.dtype == np.int8 and (x.sum(0) == 1).all() and (x.sum(1) == 1).all()
        assert (np.argmax(x, axis=0) == a.perm).all()          # X[k, i] = 1 iff k == perm[i]
        assert np.array_equal(qsb.matrix_to_assignment(x).perm, a.perm)
        assert not a.perm.flags.writeable


@pytest.mark.parametrize("bad,match", [
    (np.array([[1, 0], [1, 0]]), "column 0 sums to 2"),
    (np.array([[1, 1], [0, 0]]), "row 0 sums to 2"),
    (np.array([[2, 0], [0, 1]]), "0 or 1"),
    (np.ones((2, 3)), "square"),
])
def test_matrix_to_assignment_rejects(bad, match):
    with pytest.raises(ValueError, match=match):
        qsb.matrix_to_assignment(bad)


def test_assignment_rejects_non_bijection():
    with pytest.raises(ValueError, match="bijection"):
        qsb.Assignment([0, 0, 1])


def test_evaluate_cost_quadruple_sum_and_types():
    inst = qsb.load_bundled("chr12a")
    sol = qsb.load_bundled_solution("chr12a")
    assert qsb.evaluate_cost(inst, sol.permutation) == 9552 == sol.cost
    assert isinstance(qsb.evaluate_cost(inst, qsb.Assignment(sol.permutation)), int)
    rng = np.random.default_rng(1)
    n = 6
    f, d = rng.integers(0, 9, (n, n)), rng.integers(0, 9, (n, n))
    small = qsb.QapInstance("s", n, f, d)
    for perm in itertools.islice(itertools.permutations(range(n)), 0, 720, 37):
        p = np.array(perm)
        q = sum(f[i, j] * d[p[i], p[j]] for i in range(n) for j in range(n))
        assert qsb.evaluate_cost(small, p) == q
    fl = qsb.QapInstance("f", n, f * 0.5, d.astype(float))
    assert isinstance(qsb.evaluate_cost(fl, np.arange(n)), float)
    with pytest.raises(ValueError, match="does not match"):
        qsb.evaluate_cost(small, np.arange(n + 1))


def test_gap():
    assert qsb.gap(110, 100) == pytest.approx(0.1)
    with pytest.raises(ValueError, match="positive"):
        qsb.gap(1, 0)


# ---------------------------------------------------------------- qaplib
def test_instance_format_parse_roundtrip():
    for inst in (qsb.load_bundled("esc32e"), qsb.taillard_uniform(9),
                 qsb.QapInstance("fl", 3, np.array([[0, 1.5, 2], [1.5, 0, 0.25], [2, 0.25, 0]]),
                                 np.eye(3))):
        back = qsb.parse_instance(qsb.format_instance(inst))
        assert back.n == inst.n
        assert np.array_equal(back.flow, inst.flow) and np.array_equal(back.distance, inst.distance)
        assert back.flow.dtype == (np.int64 if inst.is_integral else np.float64)


@pytest.mark.parametrize("text,match", [
    ("", "token 1"), ("x 1 2 3 4 5 6 7 8", "token 1"), ("2.5 0 0 0 0 0 0 0 0", "integer"),
    ("1 0 0", ">= 2"), ("2 0 1 1 0 0 3 3", "tokens"), ("2 0 1 1 0 0 3 3 -1", "token 9"),
    ("2 0 1 1 0 0 3 3 q", "token 9"),
])
def test_parse_instance_errors_name_the_token(text, match):
    with pytest.raises(ValueError, match=match):
        qsb.parse_instance(text)


def test_reference_solution_io():
    sol = qsb.parse_reference_solution("4 17\n2 4 1 3\n")
    assert sol.n == 4 and sol.cost == 17 and isinstance(sol.cost, int)
    assert sol.permutation.tolist() == [1, 3, 0, 2]
    assert qsb.parse_reference_solution(qsb.format_reference_solution(sol)).permutation.tolist() \
        == [1, 3, 0, 2]
    for bad, match in (("4", "two tokens"), ("4 1 1 2 3", "expected 6"),
                       ("4 1 1 2 3 9", "out of range"), ("4 1 1 2 2 3", "duplicate"),
                       ("4 1 1 2 3 3.5", "not an integer")):
        with pytest.raises(ValueError, match=match):
            qsb.parse_reference_solution(bad)
    with pytest.raises(ValueError, match="bijection"):
        qsb.ReferenceSolution(3, 1, [0, 0, 1])


def test_bundled_instances():
    assert qsb.list_bundled() == ["chr12a.dat", "esc32e.dat", "rand150.dat", "rand26.dat"]
    e = qsb.load_bundled("esc32e")
    assert e.n == 32 and e.known_best == 2
    assert qsb.evaluate_cost(e, qsb.load_bundled_solution("esc32e").permutation) == 2
    assert qsb.load_bundled("rand150").n == 150
    assert qsb.load_instance(qsb.data_path("rand26.dat")).n == 26
    with pytest.raises(FileNotFoundError):
        qsb.data_path("nope.dat")


def test_grey_pattern_generator():
    g = qsb.grey_pattern()
    assert g.n == 256 and g.is_integral
    assert g.flow.sum() == 92 * 91 and (g.flow == g.flow.T).all()
    assert (g.distance == g.distance.T).all() and g.distance.max() <= 100
    assert (np.diag(g.distance) == 0).all() and (g.distance[~np.eye(256, dtype=bool)] >= 0).all()


# --------------------------------------------------------------- streams
def test_stream_keys_match_the_reference_contract():
    a = streams.phase_rng(42, streams.PHASE_STEP, 7).random(8)
    assert np.array_equal(a, orc.phase_rng(42, orc.PHASE_STEP, 7).random(8))
    assert not np.array_equal(a, streams.phase_rng(42, streams.PHASE_HOST, 7).random(8))
    assert np.array_equal(streams.host_rng(3, 9).integers(0, 10, 5),
                          orc.phase_rng(3, orc.PHASE_HOST, 9).integers(0, 10, 5))
    with pytest.raises(ValueError, match="iteration"):
        streams.phase_rng(1, streams.PHASE_STEP, 2**32)
    with pytest.raises(ValueError, match="population"):
        streams.step_draws(1, 1, 2**24, 2)
    assert 0.0 <= streams.phase_rng(-1, streams.PHASE_INIT, 0).random() < 1.0


# -------------------------------------------------------------------- CLI
def test_cli_validate(tmp_path, capsys):
    dat, sln = str(qsb.data_path("chr12a.dat")), str(qsb.data_path("chr12a.sln"))
    assert cli.main(["validate", dat, sln]) == 0
    assert "9552" in capsys.readouterr().out
    bad = tmp_path / "bad.sln"
    bad.write_text("12 9553\n7 5 12 2 1 3 9 11 10 6 8 4\n")
    assert cli.main(["validate", dat, str(bad)]) == 1
    out = capsys.readouterr().out
    assert "9553" in out and "9552" in out
    bad.write_text("12 9552\n7 5 12 2 1 3 9 11 10 6 8 7\n")
    assert cli.main(["validate", dat, str(bad)]) == 3


def test_cli_flag_and_io_errors(tmp_path, capsys, monkeypatch):
    dat = str(qsb.data_path("chr12a.dat"))
    assert cli.main(["solve", dat, "--sx", "nonsense"]) == 2
    assert cli.main(["frobnicate"]) == 2
    assert cli.main(["solve", str(tmp_path / "missing.dat")]) == 3
    assert "missing.dat" in capsys.readouterr().err
    bad = tmp_path / "bad.dat"
    bad.write_text("3 0 1")
    assert cli.main(["solve", str(bad)]) == 3
    err = capsys.readouterr().err
    assert "bad.dat" in err and "tokens" in err
    assert cli.main(["sweep", str(tmp_path / "none.txt")]) == 3
    monkeypatch.setenv("QAPSWARM_WORKERS", "3")
    assert cli.build_parser().parse_args(["solve", "x.dat"]).workers == 3


def test_cli_memory_guard_refuses_before_touching_the_device(tmp_path, capsys):
    dat = str(qsb.data_path("chr12a.dat"))
    rc = cli.main(["solve", dat, "--swarms", "4", "--swarm-size", "10", "--mem-cap", "0.000001",
                   "--out", str(tmp_path)])
    assert rc == 2
    io = capsys.readouterr()
    assert "GiB projected" in io.out and "mem-cap" in io.err
