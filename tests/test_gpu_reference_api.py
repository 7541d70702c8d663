"""The reference's engine, migration and CLI test suites, restated against
this package (the reference itself cannot travel to the GPU box).  Each
test names the reference test it restates (paths under
/root/reference/pkg/tests/); the assertions are the reference's, the code
is this repo's."""

import numpy as np
import pytest

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import paper_1504_05158_b200 as qsb            # noqa: E402
from paper_1504_05158_b200 import cli           # noqa: E402


@pytest.fixture(scope="module")
def chr12a():
    return qsb.load_bundled("chr12a")


@pytest.fixture(scope="module")
def tiny():
    return qsb.parse_instance("2  0 1  1 0   0 3  3 0", name="tiny")


def cfg(**kw):
    base = dict(swarms=4, swarm_size=10, max_iterations=10, seed=5, workers=2)
    base.update(kw)
    return qsb.SolverConfig(**base)


def fingerprint(st):
    """test_engine.py:13-16."""
    return tuple(np.ascontiguousarray(a).tobytes() for a in (
        st.X, st.V, st.PL, st.perms, st.cost, st.pl_cost, st.bests.matrices, st.bests.costs))


def perm_matrices_ok(buf):
    return (buf.sum(axis=1) == 1).all() and (buf.sum(axis=2) == 1).all()


# ------------------------------------------------------- test_engine.py
def test_config_validation():                                   # test_engine.py:19-27
    for kw, match in ((dict(migration_factor=0.5), "migration_factor"), (dict(swarms=0), "positive"),
                      (dict(workers=0), "workers"), (dict(stats_stride=0), "stats_stride")):
        with pytest.raises(ValueError, match=match):
            cfg(**kw)


def test_init_shapes_and_singletons(tiny, chr12a):               # test_engine.py:30-46
    st = qsb.init_population(qsb.SolverConfig(swarms=1, swarm_size=1), tiny)
    assert np.array_equal(st.bests.matrices[0], st.X[0]) and np.array_equal(st.PL[0], st.X[0])
    assert st.bests.costs[0] == st.cost[0] == st.best_cost
    big = qsb.init_population(qsb.SolverConfig(swarms=200, swarm_size=50, seed=1), chr12a)
    X = big.X
    assert X.shape == big.V.shape == (10000, 12, 12) and big.num_particles == 10000
    assert perm_matrices_ok(X) and (np.argmax(X, axis=1) == big.perms).all()


def test_init_seed_and_amplitude(tiny, chr12a):                  # test_engine.py:49-63
    a, b, c = (qsb.init_population(cfg(seed=s), tiny) for s in (9, 9, 10))
    assert fingerprint(a) == fingerprint(b) != fingerprint(c)
    assert np.abs(qsb.init_population(cfg(init_velocity_amplitude=0.25), chr12a).V).max() <= 0.25
    v = np.abs(qsb.init_population(cfg(), chr12a).V).max()
    assert 0.5 < v <= 1.0


def test_zero_coefficients_and_inertia_collapse(chr12a):         # test_engine.py:66-86
    c0 = qsb.PsoCoefficients(c1=0.0, c2=0.0, c3=0.0, sv_mode="raw", sx_mode="global-max")
    conf = cfg(coefficients=c0)
    st = qsb.init_population(conf, chr12a)
    before = st.X.copy()
    qsb.step(st, chr12a, conf)
    assert np.array_equal(st.X, before)
    c1 = qsb.PsoCoefficients(c1=0.0, c2=0.5, c3=0.5, sv_mode="raw", sx_mode="global-max")
    conf = qsb.SolverConfig(swarms=1, swarm_size=1, coefficients=c1, seed=3)
    st = qsb.init_population(conf, chr12a)
    qsb.step(st, chr12a, conf)
    assert np.array_equal(st.V[0], np.zeros((12, 12)))


def test_worker_count_does_not_change_states(chr12a):            # test_engine.py:89-98
    fps = []
    for workers in (1, 2, 8):
        conf = cfg(workers=workers, migration_factor=0.25)
        st = qsb.init_population(conf, chr12a)
        for _ in range(5):
            qsb.step(st, chr12a, conf)
        fps.append(fingerprint(st))
    assert fps[0] == fps[1] == fps[2]


def test_bests_monotone_and_consistent(chr12a):                  # test_engine.py:101-151
    conf = cfg(migration_factor=0.25, max_iterations=30)
    st = qsb.init_population(conf, chr12a)
    series, prev_pl = [st.best_cost], st.pl_cost.copy()
    for _ in range(30):
        qsb.step(st, chr12a, conf)
        series.append(st.best_cost)
        assert st.best_cost == qsb.evaluate_cost(chr12a, st.best_perm)
        assert (st.pl_cost <= prev_pl).all()                      # local bests, with migration
        prev_pl = st.pl_cost.copy()
        b = st.bests
        for k in range(conf.swarms):                              # migrated bests stay consistent
            assert b.costs[k] == qsb.evaluate_cost(chr12a, b.perms[k])
    assert all(y <= x for x, y in zip(series, series[1:]))
    conf = cfg(max_iterations=20)
    st = qsb.init_population(conf, chr12a)
    prev = st.bests.costs.copy()
    for _ in range(20):                                           # no migration: swarm bests
        qsb.step(st, chr12a, conf)
        b = st.bests
        b.check()
        assert (b.costs <= prev).all()
        prev = b.costs.copy()
        assert perm_matrices_ok(st.X) and perm_matrices_ok(st.PL)
        pl = st.pl_cost
        for k in range(conf.swarms):
            span = slice(k * conf.swarm_size, (k + 1) * conf.swarm_size)
            assert b.costs[k] == qsb.evaluate_cost(chr12a, b.perms[k])
            assert b.costs[k] <= pl[span].min()


def test_swarm_membership(chr12a):                               # test_engine.py:168-173
    st = qsb.init_population(cfg(), chr12a)
    assert [st.swarm_of(p) for p in (0, 9, 10, 39)] == [0, 0, 1, 3]


def test_run_edges(chr12a):                                      # test_engine.py:176-205
    r = qsb.run(cfg(max_iterations=0), chr12a)
    st = qsb.init_population(cfg(max_iterations=0), chr12a)
    assert (r.best_cost, r.best_iteration, r.iterations_run, len(r.stats)) == \
        (st.cost.min(), 0, 0, 1)
    assert qsb.run(cfg(max_iterations=50, target_cost=10**9), chr12a).iterations_run == 0
    assert [s.t for s in qsb.run(cfg(max_iterations=10, stats_stride=5), chr12a).stats] == [0, 5, 10]
    r = qsb.run(qsb.SolverConfig(swarms=50, swarm_size=40, max_iterations=60, seed=2, workers=2,
                                 target_cost=9552), chr12a)
    assert r.gap == qsb.gap(r.best_cost, 9552)


def test_depth_below_problem_size(tiny):                         # test_engine.py:208-214
    conf = qsb.SolverConfig(swarms=1, swarm_size=2, coefficients=qsb.PsoCoefficients(depth=2))
    st = qsb.init_population(conf, tiny)
    with pytest.raises(ValueError, match="depth"):
        qsb.step(st, tiny, conf)


def test_projected_bytes_close_to_actual(chr12a):                # test_engine.py:217-226
    conf = cfg()
    st = qsb.init_population(conf, chr12a)
    b = st.bests
    actual = sum(a.nbytes for a in (st.X, st.X_new, st.V, st.PL, st.perms, st.perms_new,
                                    st.pl_perms, st.cost, st.pl_cost, b.matrices, b.perms, b.costs))
    assert qsb.projected_buffer_bytes(conf, chr12a.n) == pytest.approx(actual, rel=0.05)


def test_migration_off_and_float_instances(chr12a):             # test_engine.py:229-251
    a = qsb.run(cfg(migration_factor=0.0, max_iterations=8), chr12a)
    b = qsb.run(cfg(max_iterations=8), chr12a)
    assert a.best_cost == b.best_cost and np.array_equal(a.best_perm, b.best_perm)
    assert [s.p50 for s in a.stats] == [s.p50 for s in b.stats]
    rng = np.random.default_rng(2)
    f = np.triu(rng.uniform(0, 10, (6, 6)), 1)
    d = np.triu(rng.uniform(0, 10, (6, 6)), 1)
    inst = qsb.QapInstance("float6", 6, f + f.T, d + d.T)
    r = qsb.run(cfg(max_iterations=5), inst)
    assert isinstance(r.best_cost, float)
    assert r.best_cost == qsb.evaluate_cost(inst, r.best_perm)


# ---------------------------------------------------- test_migration.py
def population(rng, m, S, n, cost_per_swarm):
    p = m * S
    perms = np.array([rng.permutation(n) for _ in range(p)])
    mats = np.zeros((p, n, n), dtype=np.int8)
    mats[np.arange(p)[:, None], perms, np.arange(n)[None, :]] = 1
    return perms, mats, np.repeat(np.asarray(cost_per_swarm, dtype=np.int64), S)


def table(rng, m, n, costs):
    perms = np.array([rng.permutation(n) for _ in range(m)])
    mats = np.zeros((m, n, n), dtype=np.int8)
    mats[np.arange(m)[:, None], perms, np.arange(n)[None, :]] = 1
    return qsb.SwarmBestTable(matrices=mats, perms=perms, costs=np.asarray(costs, dtype=np.int64))


def test_migrate_depth_zero_and_hand_trace():                    # test_migration.py:24-52
    rng = np.random.default_rng(0)
    t = table(rng, 4, 5, [10, 20, 30, 40])
    before = t.costs.copy()
    assert qsb.migrate(0, t, *population(rng, 4, 3, 5, [11, 21, 31, 41]), 3,
                       np.random.default_rng(1)) == []
    assert np.array_equal(t.costs, before)
    rng = np.random.default_rng(2)
    t = table(rng, 4, 5, [10, 20, 30, 40])
    keep = t.perms.copy()
    perms, mats, costs = population(rng, 4, 3, 5, [12, 22, 32, 42])
    ev = qsb.migrate(1, t, perms, mats, costs, 3, np.random.default_rng(7))
    assert len(ev) == 1 and (ev[0].source_swarm, ev[0].target_swarm) == (0, 3)
    assert 0 <= ev[0].particle < 3 and t.costs[3] == 12
    assert np.array_equal(t.perms[3], perms[ev[0].particle])
    assert all(np.array_equal(t.perms[k], keep[k]) for k in (0, 1, 2))
    t.check()


def test_migrate_rank_sets_and_factor():                         # test_migration.py:55-86
    rng = np.random.default_rng(3)
    m, S, n = 250, 2, 4
    t = table(rng, m, n, rng.integers(100, 10000, m))
    d = int(0.33 * m)
    assert d == 82
    assert len(qsb.migrate(d, t, *population(rng, m, S, n, rng.integers(100, 10000, m)), S,
                           np.random.default_rng(4))) == 82
    t.check()
    rng = np.random.default_rng(5)
    m, S, n = 10, 4, 5
    t = table(rng, m, n, np.arange(10, 10 + m) * 100)
    perms, mats, costs = population(rng, m, S, n, rng.integers(0, 10**6, m))
    ev = qsb.migrate(4, t, perms, mats, costs, S, np.random.default_rng(6))
    src, dst = {e.source_swarm for e in ev}, {e.target_swarm for e in ev}
    assert src == {0, 1, 2, 3} and dst == {9, 8, 7, 6}
    for e in ev:
        assert e.particle // S == e.source_swarm
        assert np.array_equal(t.perms[e.target_swarm], perms[e.particle])


def test_migrate_worse_values_bounds_and_ties():                 # test_migration.py:89-122
    rng = np.random.default_rng(8)
    t = table(rng, 4, 5, [10, 20, 30, 40])
    ev = qsb.migrate(1, t, *population(rng, 4, 3, 5, [999] * 4), 3, np.random.default_rng(9))
    assert t.costs[3] == 999 and ev[0].new_cost > ev[0].old_cost
    rng = np.random.default_rng(10)
    t = table(rng, 4, 5, [1, 2, 3, 4])
    with pytest.raises(ValueError, match="m/2"):
        qsb.migrate(2, t, *population(rng, 4, 2, 5, [1, 2, 3, 4]), 2, np.random.default_rng(0))
    with pytest.raises(ValueError, match="population"):
        qsb.migrate(1, t, *population(rng, 3, 2, 5, [1, 2, 3]), 2, np.random.default_rng(0))
    rng = np.random.default_rng(12)
    t = table(rng, 4, 5, [7, 7, 7, 7])
    ev = qsb.migrate(1, t, *population(rng, 4, 2, 5, [5] * 4), 2, np.random.default_rng(1))
    assert (ev[0].source_swarm, ev[0].target_swarm) == (0, 3)


# ---------------------------------------------------------- test_cli.py
def solve_argv(tmp_path, **extra):
    argv = ["solve", str(qsb.data_path("chr12a.dat")), "--swarms", "4", "--swarm-size", "10",
            "--max-iters", "5", "--seed", "3", "--out", str(tmp_path)]
    for k, v in extra.items():
        argv += [f"--{k.replace('_', '-')}", str(v)]
    return argv


def test_cli_solve_outputs(tmp_path, capsys):                    # test_cli.py:24-50,182-187
    assert cli.main(solve_argv(tmp_path)) == 0
    out = capsys.readouterr().out
    assert all(k in out for k in ("goal=", "iteration=", "time/iter=", "GiB projected"))
    d = tmp_path / "chr12a-s3"
    assert all((d / f).is_file() for f in ("stats.csv", "pmf.csv", "solution.txt"))
    sol = qsb.load_reference_solution(d / "solution.txt")
    assert qsb.evaluate_cost(qsb.load_bundled("chr12a"), sol.permutation) == sol.cost
    assert int(out.split("goal=")[1].split()[0]) == sol.cost
    assert cli.main(solve_argv(tmp_path, sln=qsb.data_path("chr12a.sln"))) == 0
    assert "gap=" in capsys.readouterr().out
    assert cli.main(solve_argv(tmp_path, repeats=3)) == 0
    assert capsys.readouterr().out.count("goal=") == 3
    assert all((tmp_path / f"chr12a-s{s}").is_dir() for s in (3, 4, 5))


def test_cli_sweep(tmp_path):                                    # test_cli.py:110-170
    dat = qsb.data_path("chr12a.dat")
    m = tmp_path / "m.txt"
    m.write_text(f"{dat} --swarms 2 --swarm-size 5 --max-iters 2 --seed 1 --out {tmp_path}\n"
                 f"{tmp_path}/nope.dat --swarms 2\n"
                 f"{dat} --sln {qsb.data_path('chr12a.sln')} --swarms 2 --swarm-size 5 "
                 f"--max-iters 2 --out {tmp_path}\n")
    assert cli.main(["sweep", str(m), "--out", str(tmp_path)]) == 0
    lines = (tmp_path / "sweep_results.csv").read_text().splitlines()
    assert len(lines) == 4 and lines[0].startswith("instance,swarms,swarm_size,total_particles")
    assert all(len(x.split(",")) == len(lines[0].split(",")) for x in lines)
    err = [x for x in lines[1:] if "nope" in x]
    assert len(err) == 1 and err[0].split(",")[-1] != ""
    ref = lines[3].split(",")
    assert ref[0] == "chr12a" and ref[10] == "9552" and ref[11] != ""
    rows = [f"{qsb.data_path(('chr12a', 'esc32e', 'rand26')[i % 3] + '.dat')} --swarms 2 "
            f"--swarm-size 4 --max-iters 1 --seed {i} --out {tmp_path}" for i in range(18)]
    m.write_text("\n".join(rows) + "\n")
    assert cli.main(["sweep", str(m), "--out", str(tmp_path)]) == 0
    assert len((tmp_path / "sweep_results.csv").read_text().splitlines()) == 19
    m.write_text(f"{tmp_path}/nope.dat --swarms 2\n")
    assert cli.main(["sweep", str(m), "--out", str(tmp_path)]) == 3


def test_cli_extension_flags(tmp_path, capsys):
    """The engine's extensions: fp32 throughput mode, migration period,
    2-opt and device init run through the same front end."""
    argv = solve_argv(tmp_path, precision="fp32", migration=0.25, migration_period=2, two_opt=1,
                      init="device")
    assert cli.main(argv) == 0
    sol = qsb.load_reference_solution(tmp_path / "chr12a-s3" / "solution.txt")
    assert qsb.evaluate_cost(qsb.load_bundled("chr12a"), sol.permutation) == sol.cost
