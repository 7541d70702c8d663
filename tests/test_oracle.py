"""Pins the CPU oracle (oracle/) to the reference's own outputs.

The golden vectors were produced by running the reference package
(tests/golden/make_golden.py); the oracle must reproduce every one of them
bit for bit before it is trusted as the checker of the CUDA path.
"""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as orc


def digest(st):
    h = hashlib.sha256()
    for b in st.fingerprint():
        h.update(b)
    return h.hexdigest()


def test_philox_matches_numpy_generator():
    for seed, word in [(0, 0), (12345, (2 << 56) | (7 << 24)), (2**64 - 1, 3 << 56)]:
        g = np.random.Generator(np.random.Philox(key=np.array([seed, word], np.uint64)))
        ref = g.random(41)
        got = [orc.lib().orc_uniform_at(seed, word, i) for i in range(41)]
        assert np.array_equal(ref, np.array(got))


def test_step_draws_golden():
    g = np.load(GOLDEN / "draws.npz")
    for i, (seed, t, P, n) in enumerate(g["cases"].tolist()):
        got = orc.step_draws(int(seed), int(t), int(P), int(n))
        assert np.array_equal(got, g[f"case{i}"]), f"case {i}"


def test_step_draws_particle_offset():
    full = orc.step_draws(3, 9, 40, 7)
    part = orc.step_draws(3, 9, 15, 7, p0=25)
    assert np.array_equal(full[25:], part)


def test_step_draws_bounds():
    with pytest.raises(ValueError, match="population"):
        orc.step_draws(1, 1, 2**24, 2)
    with pytest.raises(ValueError, match="iteration"):
        orc.step_draws(1, 2**32, 1, 2)


def test_host_stream_picks_golden():
    g = np.load(GOLDEN / "draws.npz")
    for i, (seed, t, S, d) in enumerate([(1, 10, 100, 264), (3, 5, 20, 16), (5, 1, 10, 1)]):
        rng = orc.phase_rng(seed, orc.PHASE_HOST, t)
        got = np.array([rng.integers(0, S) for _ in range(d)])
        assert np.array_equal(got, g[f"host{i}"])


def _velocity_case(g, k):
    n, P, S, norm = g[f"v{k}_meta"].tolist()
    c1, c2, c3, vmax = g[f"v{k}_coef"].tolist()
    x = orc.matrices_from_perms(g[f"v{k}_perm"], n)
    pl = orc.matrices_from_perms(g[f"v{k}_plperm"], n)
    pg = orc.matrices_from_perms(g[f"v{k}_pgperm"], n)
    return n, P, S, bool(norm), (c1, c2, c3, vmax), x, pl, pg


def test_velocity_golden_bit_exact():
    g = np.load(GOLDEN / "velocity.npz")
    for k in range(int(g["count"])):
        n, P, S, norm, (c1, c2, c3, vmax), x, pl, pg = _velocity_case(g, k)
        v = g[f"v{k}_in"].copy()
        orc.velocity_many(v, x, pl, pg, S, c1, c2 * g[f"v{k}_r2"], c3 * g[f"v{k}_r3"], vmax, norm)
        assert v.tobytes() == g[f"v{k}_out"].tobytes(), f"case {k}"


def test_aggregate_golden_bit_exact():
    g = np.load(GOLDEN / "aggregate.npz")
    for k in range(int(g["count"])):
        mode, depth, n, p = g[f"a{k}_meta"].tolist()
        x = orc.matrices_from_perms(g[f"a{k}_perm"], n)
        out_mat = np.zeros_like(x)
        out_perm = np.zeros((p, n), np.int64)
        orc.aggregate_many(x, g[f"a{k}_v"], mode, depth, g[f"a{k}_draws"], out_mat, out_perm)
        assert np.array_equal(out_perm, g[f"a{k}_out"]), f"case {k}"
        assert np.array_equal(out_mat, orc.matrices_from_perms(out_perm, n))


def test_aggregate_thread_count_invariance():
    g = np.load(GOLDEN / "aggregate.npz")
    mode, depth, n, p = g["a0_meta"].tolist()
    x = orc.matrices_from_perms(g["a0_perm"], n)
    outs = []
    for k in (1, 3):
        orc.set_threads(k)
        out_perm = np.zeros((p, n), np.int64)
        orc.aggregate_many(x, g["a0_v"], mode, depth, g["a0_draws"], np.zeros_like(x), out_perm)
        outs.append(out_perm)
    orc.set_threads(0)
    assert np.array_equal(outs[0], outs[1])


def test_cost_golden(golden_instances):
    g = np.load(GOLDEN / "cost.npz")
    for name in ("chr12a", "tai30", "float6", "esc32e"):
        inst = golden_instances[name]
        perms = g[f"{name}_perms"]
        out = np.zeros(perms.shape[0], g[f"{name}_cost"].dtype)
        orc.cost_many(perms, inst.flow, inst.distance, out)
        assert out.tobytes() == g[f"{name}_cost"].tobytes()


def test_chr12a_known_optimum(golden_instances, golden_meta):
    inst = golden_instances["chr12a"]
    sln = golden_meta["chr12a_sln"]
    assert orc.evaluate_cost(inst.flow, inst.distance, sln["perm"]) == 9552 == sln["cost"]


@pytest.mark.parametrize("name", ["A_chr12a_mig", "B_chr12a_raw_gm", "C_chr12a_pc_mig",
                                  "D_tai30_st_mig", "E_float6", "F_tiny_gm", "G_zero_coeffs",
                                  "H_esc32e_st3", "I_tai50_norm"])
def test_trajectory_golden(name, trajectories, golden_instances):
    tr = trajectories[name]
    inst = golden_instances[tr["instance"]]
    ck = dict(c1=0.5, c2=0.5, c3=0.5, v_max=4.0, sv_mode="norm", sx_mode="second-target",
              depth=2)
    ck.update(tr["coefficients"])
    cfg = dict(tr["config"])
    st = orc.init_population(cfg["swarms"], cfg["swarm_size"], inst.n, inst.flow,
                             inst.distance, seed=cfg.get("seed", 0),
                             amp=cfg.get("init_velocity_amplitude", 1.0))
    assert digest(st) == tr["digests"][0]
    for t in range(tr["iterations"]):
        orc.step(st, inst.flow, inst.distance, seed=cfg.get("seed", 0),
                 migration_factor=cfg.get("migration_factor", 0.0), **ck)
        assert digest(st) == tr["digests"][t + 1], f"step {t + 1}"
        assert [st.best_cost, st.best_iteration] == tr["bests"][t + 1]
    assert st.best_perm.tolist() == tr["best_perm"]
    assert [list(e) for e in st.migration_log] == tr["migration_log"]


def test_twoopt_oracle_against_bruteforce(golden_instances):
    """2-opt has no reference symbol: its oracle is pinned by brute force --
    every applied move is the best (lexicographically first) exchange and
    the costs equal evaluate_cost."""
    rng = np.random.default_rng(3)
    for name in ("chr12a", "tai30"):
        inst = golden_instances[name]
        n = inst.n
        perms = np.array([rng.permutation(n) for _ in range(6)], dtype=np.int64)
        costs = np.zeros(6, np.int64)
        orc.cost_many(perms, inst.flow, inst.distance, costs)
        for p in range(6):
            q = perms[p:p + 1].copy()
            c = costs[p:p + 1].copy()
            orc.twoopt_many(q, inst.flow, inst.distance, c, 1)
            base = orc.evaluate_cost(inst.flow, inst.distance, perms[p])
            best, arg = 0, None
            for r in range(n):
                for s in range(r + 1, n):
                    t = perms[p].copy()
                    t[r], t[s] = t[s], t[r]
                    dlt = orc.evaluate_cost(inst.flow, inst.distance, t) - base
                    if dlt < best:
                        best, arg = dlt, t
            expect = arg if arg is not None else perms[p]
            assert np.array_equal(q[0], expect)
            assert c[0] == orc.evaluate_cost(inst.flow, inst.distance, q[0])
        # many passes never increase the cost and stay consistent
        q = perms.copy()
        c = costs.copy()
        orc.twoopt_many(q, inst.flow, inst.distance, c, 50)
        assert (c <= costs).all()
        for p in range(6):
            assert c[p] == orc.evaluate_cost(inst.flow, inst.distance, q[p])
