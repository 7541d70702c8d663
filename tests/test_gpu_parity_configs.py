"""Parity on the configurations bench.py actually runs, plus the pieces the
round-1 suite left unpinned:

* the n > 160 kernel variants (fp32 n = 256 keeps its tile in global memory:
  ``step_kernel<float, u16, 8, 1, 1, true>``; fp64 likewise above ~160),
  one step replayed on the CPU oracle;
* a whole-swarm replay at the full config-3 shape (80k particles, fp32,
  migration every 10 iterations) after 12 steps;
* the device-drawn migration picks against the reference's host stream;
* the throughput-mode device initialisation against its oracle restatement
  and its distribution;
* CUDA-graph replay against eager steps when the first step's velocity
  bound differs from the later steps'.

The oracle (oracle/) is the checker only; every result under test comes from
libqsb.so through the package."""

import math

import numpy as np
import pytest

from conftest import GOLDEN, cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import torch                                    # noqa: E402

import paper_1504_05158_b200 as qsb            # noqa: E402
from paper_1504_05158_b200 import _lib, engine  # noqa: E402
from oracle import oracle as orc                # noqa: E402

MODES = {"global-max": 0, "pick-column": 1, "second-target": 2}


def v_rows(st, idx):
    """float64 velocities of local particles ``idx`` (exact u * s for the
    column-scaled fp32 layouts)."""
    n = st.n
    it = torch.as_tensor(np.asarray(idx), dtype=torch.int64, device=st.device)
    u = st.d_V.index_select(0, it)[:, :n * n].reshape(len(idx), n, n)
    if st.d_vcol is not None:
        s = st.d_vcol.index_select(0, it)[:, 0, :n]
        return (st.v_decode(u) * st.v_decode(s).unsqueeze(1)).cpu().numpy()
    return u.double().cpu().numpy()


def rows(t, idx):
    it = torch.as_tensor(np.asarray(idx), dtype=torch.int64, device=t.device)
    return t.index_select(0, it).cpu().numpy()


def col_scaled_err(got, ref):
    scale = np.abs(ref).max(axis=1, keepdims=True)
    return (np.abs(got - ref) / np.where(scale > 0, scale, 1.0)).max()


def replay_swarms(st, inst, cfg, swarms):
    """Step the device state once and replay that step for the listed
    swarms on the oracle, from the device's own pre-step state.  Draws use
    the global particle offsets (streams.py:53-64 row p = particle p).
    Returns the comparisons as a dict of booleans / errors."""
    n, S = st.n, st.swarm_size
    c = cfg.coefficients
    t = st.t + 1
    idx = np.concatenate([np.arange(k * S, (k + 1) * S) for k in swarms])
    X = rows(st.d_perm, idx).astype(np.int64)
    PL = rows(st.d_pl_perm, idx).astype(np.int64)
    pl_cost = rows(st.d_pl_cost, idx)
    PG = rows(st.d_pg_perm, swarms).astype(np.int64)
    pg_cost = rows(st.d_pg_cost, swarms)
    V = v_rows(st, idx)
    qsb.step(st, inst, cfg)
    out = {}
    xm = orc.matrices_from_perms(X, n)
    plm = orc.matrices_from_perms(PL, n)
    pgm = orc.matrices_from_perms(PG, n)
    v_ref = V.copy()
    draws = np.concatenate([orc.step_draws(cfg.seed, t, S, n, p0=k * S) for k in swarms])
    orc.velocity_many(v_ref, xm, plm, pgm, S, c.c1, c.c2 * draws[:, 0].copy(),
                      c.c3 * draws[:, 1].copy(), c.v_max, c.sv_mode == "norm")
    v_got = v_rows(st, idx)
    out["v_err"] = col_scaled_err(v_got, v_ref)
    if st.precision == "fp64":
        out["v_exact"] = v_got.tobytes() == v_ref.tobytes()
    # aggregation + goal: exact against the oracle fed the device's own V
    got_perm = rows(st.d_perm, idx).astype(np.int64)     # post-swap current positions
    om = np.zeros_like(xm)
    op = np.zeros((len(idx), n), np.int64)
    orc.aggregate_many(xm, np.ascontiguousarray(v_got), MODES[c.sx_mode], c.depth,
                       np.ascontiguousarray(draws[:, 2:]), om, op)
    out["perm_exact"] = np.array_equal(op, got_perm)
    cost = np.zeros(len(idx), np.int64)
    orc.cost_many(op, inst.flow, inst.distance, cost)
    out["cost_exact"] = np.array_equal(cost, rows(st.d_cost, idx))
    # personal and swarm bests (engine.py:210-229)
    imp = cost < pl_cost
    pl_ref = np.where(imp, cost, pl_cost)
    out["pbest_exact"] = (np.array_equal(pl_ref, rows(st.d_pl_cost, idx))
                          and np.array_equal(np.where(imp[:, None], op, PL),
                                             rows(st.d_pl_perm, idx).astype(np.int64)))
    pg_ref = pg_cost.copy()
    for i, k in enumerate(swarms):
        sl = slice(i * S, (i + 1) * S)
        cand = np.nonzero(imp[sl])[0]
        if cand.size:
            j = cand[np.argmin(cost[sl][cand])]
            if cost[sl][j] < pg_ref[i]:
                pg_ref[i] = cost[sl][j]
    out["pg_exact"] = np.array_equal(pg_ref, rows(st.d_pg_cost, swarms))
    return out


# ------------------------------------------------- n > 160 kernel variants
@pytest.mark.parametrize("n", [161, 200, 255, 256])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_large_n_step_replay(n, precision):
    """fp32 n = 256 is the config-5 kernel (tile in global memory); fp64
    keeps its tile in global memory above ~160 too.  fp64 is bit-exact;
    fp32 meets the column-scaled 1e-5 rule; aggregation, goal and bests are
    exact in both."""
    inst = qsb.taillard_uniform(n)
    cfg = qsb.SolverConfig(swarms=3, swarm_size=8, seed=n, precision=precision,
                           migration_factor=0.34, migration_period=2,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, inst)
    for _ in range(4):
        qsb.step(st, inst, cfg)
    r = replay_swarms(st, inst, cfg, [0, 1, 2])
    assert r["v_err"] <= 1e-5, r
    if precision == "fp64":
        assert r["v_exact"], r
    assert r["perm_exact"] and r["cost_exact"] and r["pbest_exact"] and r["pg_exact"], r


@pytest.mark.parametrize("n", [170, 200, 256])
def test_fp64_large_n_trajectory_bit_exact(n):
    """fp64 parity mode above the shared-memory tile limit: the whole state
    (X, V, PL, costs, swarm bests) equals the oracle's bit for bit over
    several steps with migration."""
    inst = qsb.taillard_uniform(n)
    cfg = qsb.SolverConfig(swarms=4, swarm_size=3, seed=7, migration_factor=0.25,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, inst)
    ost = orc.init_population(4, 3, n, inst.flow, inst.distance, seed=7)
    kw = orc.coeff_kwargs(cfg)
    for t in range(3):
        qsb.step(st, inst, cfg)
        orc.step(ost, inst.flow, inst.distance, **kw)
        assert st.V.tobytes() == ost.V.tobytes(), f"step {t + 1}"
        assert np.array_equal(st.perms, ost.perms)
        assert np.array_equal(st.cost, ost.cost)
        assert np.array_equal(st.pl_cost, ost.pl_cost)
        assert np.array_equal(st.bests.costs, ost.pg_costs)
    assert st.best_cost == ost.best_cost


# -------------------------------------------------- full config-3 shape
def test_config3_full_size_swarm_replay():
    """The bench's headline state (n = 50, 800 x 100 = 80k particles, fp32,
    device init, migration 0.33 every 10 iterations) after 12 steps: step
    13 replayed on the oracle for 12 whole swarms spread over the population
    (first, last, and around the dynamic-scheduling tail), with their global
    draw offsets."""
    inst = qsb.taillard_uniform(50)
    cfg = qsb.SolverConfig(swarms=800, swarm_size=100, seed=1, precision="fp32", init="device",
                           migration_factor=0.33, migration_period=10,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, inst)
    for _ in range(12):
        qsb.step(st, inst, cfg)
    assert len(st.migration_log) == cfg.migration_depth
    swarms = [0, 1, 97, 255, 256, 399, 400, 511, 640, 777, 798, 799]
    r = replay_swarms(st, inst, cfg, swarms)
    assert r["v_err"] <= 1e-5, r
    assert r["perm_exact"] and r["cost_exact"] and r["pbest_exact"] and r["pg_exact"], r


# ------------------------------------------------------- migration picks
def _picks_device(seed, t, d, S):
    out = torch.empty(max(d, 1), dtype=torch.int32, device="cuda")
    _lib.call("qsb_migration_picks", int(seed) & (2**64 - 1), int(t), int(d), int(S),
              out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    return out[:d].cpu().numpy()


def test_device_migration_picks_equal_reference_host_stream():
    g = np.load(GOLDEN / "draws.npz")
    for i, (seed, t, S, d) in enumerate([(1, 10, 100, 264), (3, 5, 20, 16), (5, 1, 10, 1)]):
        assert np.array_equal(_picks_device(seed, t, d, S), g[f"host{i}"])
    rng = np.random.default_rng(1)
    for _ in range(25):
        seed = int(rng.integers(-2**40, 2**40))
        t = int(rng.integers(0, 2**32))
        S = int(rng.choice([1, 2, 3, 7, 100, 1000, 65536, 3 * 2**20 + 1]))
        d = int(rng.integers(1, 600))
        assert np.array_equal(_picks_device(seed, t, d, S), orc.migration_picks(seed, t, d, S))
    # S = 14316558 rejects about 1 draw in 300: 2000 draws exercise the
    # sequential redraw path of host_picks
    S, d = 14316558, 2000
    ref = orc.migration_picks(9, 77, d, S)
    thr = ((1 << 32) - S) % S
    key = (9, (3 << 56) | (77 << 24))
    no_reject = []
    for j in range(d):
        w = int(orc.philox_block([j // 8 + 1, 0, 0, 0], key)[(j >> 1) & 3])
        no_reject.append(((w >> 32) if j & 1 else (w & 0xFFFFFFFF)) * S >> 32)
    assert not np.array_equal(ref, no_reject), "case must include a rejected draw"
    assert thr > 0
    assert np.array_equal(_picks_device(9, 77, d, S), ref)


def test_migration_events_equal_oracle_at_long_periods(golden_instances):
    """Device picks inside migrate_kernel: the event log and swarm bests
    equal the oracle's (reference host stream) over many epochs."""
    inst = golden_instances["tai30"]
    cfg = qsb.SolverConfig(swarms=10, swarm_size=12, seed=-5, migration_factor=0.34,
                           migration_period=4, coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, inst)
    ost = orc.init_population(10, 12, inst.n, inst.flow, inst.distance, seed=-5)
    kw = orc.coeff_kwargs(cfg)
    for _ in range(41):
        qsb.step(st, inst, cfg)
        orc.step(ost, inst.flow, inst.distance, **kw)
    assert st.V.tobytes() == ost.V.tobytes()
    assert np.array_equal(st.bests.costs, ost.pg_costs)
    assert [tuple(e) for e in st.migration_log] == [tuple(e) for e in ost.migration_log]


# ------------------------------------------------------------ device init
@pytest.mark.parametrize("precision,n", [("fp64", 12), ("fp32", 30), ("fp32", 64), ("fp32", 80),
                                         ("fp64", 50)])
def test_device_init_equals_restatement(precision, n):
    """init="device" (csrc/aux_kernels.cuh init_kernel) equals its oracle
    restatement bit for bit, including a sharded slice (global offsets)."""
    inst = qsb.taillard_uniform(n)
    cfg = qsb.SolverConfig(swarms=6, swarm_size=7, seed=123, precision=precision, init="device",
                           init_velocity_amplitude=0.75)
    for rng_ in (None, (2, 5)):
        st = qsb.init_population(cfg, inst, swarm_range=rng_)
        p0, P = st.particle_offset, st.local_particles
        perms, V = orc.device_init(cfg.seed, p0, P, n, 0.75)
        assert np.array_equal(st.perms, perms)
        words = st.d_V[:, :n * n].reshape(P, n, n)
        if precision == "fp64":
            assert words.cpu().numpy().tobytes() == V.tobytes()
        elif st.v_wide:
            want = engine.wide_encode(torch.from_numpy(V).to(st.device))
            assert torch.equal(words.view(torch.int32), want.view(torch.int32))
        else:
            assert np.array_equal(words.cpu().numpy(), V.astype(np.float32))
        cost = np.zeros(P, np.int64)
        orc.cost_many(perms, inst.flow, inst.distance, cost)
        assert np.array_equal(st.cost, cost)
        assert np.array_equal(st.pl_cost, cost)


def test_device_init_distribution():
    """Positions: every (row, column) cell of X occupied uniformly (chi^2 over
    the n x n count table, 0.1 % level); velocities: U(-amp, amp) (KS)."""
    from scipy import stats as ss
    n = 12
    inst = qsb.taillard_uniform(n)
    cfg = qsb.SolverConfig(swarms=200, swarm_size=100, seed=99, precision="fp64", init="device",
                           init_velocity_amplitude=2.0)
    st = qsb.init_population(cfg, inst)
    perms = st.perms
    P = perms.shape[0]
    assert (np.sort(perms, axis=1) == np.arange(n)).all()
    counts = np.zeros((n, n), np.int64)
    for c in range(n):
        counts[:, c] = np.bincount(perms[:, c], minlength=n)
    chi = ss.chisquare(counts.ravel(), np.full(n * n, P / n))
    assert chi.pvalue > 1e-3, chi
    v = st.V.ravel()
    assert v.min() >= -2.0 and v.max() < 2.0
    ks = ss.kstest(v[::7], ss.uniform(loc=-2.0, scale=4.0).cdf)
    assert ks.pvalue > 1e-3, ks


# ------------------------------------------------------------- graph hints
def test_graph_replay_after_velocity_bound_changes(golden_instances):
    """the first eager step runs with the init amplitude's bound
    (|c1 v| <= v_max holds), later steps do not (|v| reaches 1 > v_max / c1).
    Graph replay must use the later steps' hints and equal eager stepping."""
    inst = golden_instances["tai30"]
    for precision in ("fp64", "fp32"):
        cfg = qsb.SolverConfig(swarms=6, swarm_size=10, seed=4, precision=precision,
                               init_velocity_amplitude=0.5, migration_factor=0.34,
                               migration_period=3,
                               coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5, v_max=0.5))
        a = qsb.init_population(cfg, inst)
        b = qsb.init_population(cfg, inst)
        for _ in range(17):
            qsb.step(a, inst, cfg)
        qsb.step_many(b, inst, cfg, 17)
        assert a.t == b.t == 17
        assert a.d_V.cpu().numpy().tobytes() == b.d_V.cpu().numpy().tobytes(), precision
        assert np.array_equal(a.perms, b.perms)
        assert np.array_equal(a.bests.costs, b.bests.costs)
        assert [tuple(e) for e in a.migration_log] == [tuple(e) for e in b.migration_log]
        # the cached graph is reused by a second call
        qsb.step_many(a, inst, cfg, 12)
        qsb.step_many(b, inst, cfg, 12)
        assert a.d_V.cpu().numpy().tobytes() == b.d_V.cpu().numpy().tobytes()
        assert [tuple(e) for e in a.migration_log] == [tuple(e) for e in b.migration_log]


def test_step_many_period10_config3_shape_small():
    """Graph span lcm(2, 10) = 10 with the migration launch captured at its
    slot: identical to eager steps, events included."""
    inst = qsb.taillard_uniform(50)
    cfg = qsb.SolverConfig(swarms=40, swarm_size=25, seed=1, precision="fp32", init="device",
                           migration_factor=0.33, migration_period=10,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    a = qsb.init_population(cfg, inst)
    b = qsb.init_population(cfg, inst)
    for _ in range(47):
        qsb.step(a, inst, cfg)
    qsb.step_many(b, inst, cfg, 47)
    assert a.d_V.cpu().numpy().tobytes() == b.d_V.cpu().numpy().tobytes()
    assert np.array_equal(a.perms, b.perms)
    assert (a.best_cost, a.best_iteration) == (b.best_cost, b.best_iteration)
    assert [tuple(e) for e in a.migration_log] == [tuple(e) for e in b.migration_log]
    assert len(a.migration_log) == 4 * cfg.migration_depth


def test_runtime_follows_the_instance_object():
    """A state stepped with a different instance object (same n) evaluates
    the goal against that instance (the runtime is keyed on the object)."""
    a = qsb.taillard_uniform(20)
    b = qsb.taillard_uniform(20, seed=77)
    cfg = qsb.SolverConfig(swarms=2, swarm_size=5, seed=1,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, a)
    qsb.step(st, a, cfg)
    qsb.step(st, b, cfg)
    cost = np.zeros(10, np.int64)
    orc.cost_many(st.perms, b.flow, b.distance, cost)
    assert np.array_equal(st.cost, cost)


# ----------------------------------------- fp32 statistical equivalence
def _final_bests(n, precision, seeds, swarms, S, iters):
    inst = qsb.taillard_uniform(n)
    best, when = [], []
    for seed in seeds:
        cfg = qsb.SolverConfig(swarms=swarms, swarm_size=S, seed=seed, precision=precision,
                               migration_factor=0.33, migration_period=10,
                               max_iterations=iters,
                               coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
        r = qsb.run(cfg, inst, collect_stats=False)
        best.append(r.best_cost)
        when.append(r.best_iteration)
    return np.array(best, np.float64), np.array(when, np.float64)


@pytest.mark.parametrize("n,swarms,S,iters", [(30, 20, 25, 200), (50, 20, 25, 200)])
def test_fp32_final_best_distribution_matches_fp64(n, swarms, S, iters):
    """north_star / BASELINE.md: the fp32 throughput mode's final best-cost
    distribution must be statistically indistinguishable from the reference
    arithmetic (fp64 parity mode, bit-identical to the reference).  40
    independent seeds per arm (disjoint seed sets, so the samples are
    independent), two-sample KS and Mann-Whitney U at alpha = 0.01 on the
    final best cost and on the iteration that found it."""
    from scipy import stats as ss
    b64, w64 = _final_bests(n, "fp64", range(0, 40), swarms, S, iters)
    b32, w32 = _final_bests(n, "fp32", range(1000, 1040), swarms, S, iters)
    for a, b, what in ((b64, b32, "best cost"), (w64, w32, "best iteration")):
        ks = ss.ks_2samp(a, b)
        mw = ss.mannwhitneyu(a, b, alternative="two-sided")
        assert ks.pvalue > 0.01, (what, ks, a.mean(), b.mean())
        assert mw.pvalue > 0.01, (what, mw, a.mean(), b.mean())
