"""qsb_step_host (the host-buffer, reference-layout engine.step) against the
CPU oracle: the whole reference PopulationState -- X, V, PL, perms, costs,
swarm bests (matrices, perms, costs), the global best and the migration log
-- bit for bit after every step, with the particles streamed through the
device in several chunk counts."""

import os

import numpy as np
import pytest

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import paper_1504_05158_b200 as qsb            # noqa: E402
from paper_1504_05158_b200 import host          # noqa: E402
from oracle import oracle as orc                # noqa: E402


def host_from_oracle(ost, cfg, integral):
    hp = host.HostPopulation(cfg, ost.n, integral)
    for name in ("X", "X_new", "V", "PL", "perms", "perms_new", "pl_perms", "cost", "pl_cost"):
        getattr(hp, name)[...] = getattr(ost, name)
    hp.bests.matrices[...] = ost.pg_mats
    hp.bests.perms[...] = ost.pg_perms
    hp.bests.costs[...] = ost.pg_costs
    hp._best_perm[...] = ost.best_perm
    hp._best_cost[0] = ost.best_cost
    hp._best_iter[0] = ost.best_iteration
    return hp


def assert_same(hp, ost, where):
    for name in ("X", "V", "PL", "perms", "cost", "pl_cost", "pl_perms"):
        a, b = getattr(hp, name), getattr(ost, name)
        assert a.tobytes() == np.ascontiguousarray(b).astype(a.dtype).tobytes(), (where, name)
    assert hp.bests.matrices.tobytes() == ost.pg_mats.tobytes(), where
    assert np.array_equal(hp.bests.perms, ost.pg_perms), where
    assert hp.bests.costs.tobytes() == ost.pg_costs.tobytes(), where
    assert (hp.best_cost, hp.best_iteration) == (ost.best_cost, ost.best_iteration), where
    assert np.array_equal(hp.best_perm, ost.best_perm), where


@pytest.mark.parametrize("name,chunks,kw", [
    ("chr12a", "8", dict(migration_factor=0.34, coefficients=qsb.PsoCoefficients(0.5, 0.5, 0.5))),
    ("tai30", "3", dict(migration_factor=0.25, migration_period=3,
                        coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))),
    ("tai30", "1", dict(coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5, sv_mode="raw",
                                                          sx_mode="pick-column"))),
    ("float6", "5", dict(migration_factor=0.3,
                         coefficients=qsb.PsoCoefficients(0.7, 0.5, 0.9, sx_mode="global-max"))),
    ("tai50", "64", dict(migration_factor=0.2, coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))),
])
def test_step_host_equals_oracle(name, chunks, kw, golden_instances, monkeypatch):
    monkeypatch.setenv("QSB_HOST_CHUNKS", chunks)
    inst = golden_instances[name]
    cfg = qsb.SolverConfig(swarms=11, swarm_size=7, seed=13, **kw)
    ost = orc.init_population(11, 7, inst.n, inst.flow, inst.distance, seed=13)
    integral = inst.flow.dtype.kind in "iu"
    hp = host_from_oracle(ost, cfg, integral)
    okw = orc.coeff_kwargs(cfg)
    for t in range(1, 9):
        host.step_host(hp, inst, cfg)
        orc.step(ost, inst.flow, inst.distance, **okw)
        assert hp.t == ost.t == t
        assert_same(hp, ost, f"step {t}")
    assert [tuple(e) for e in hp.migration_log] == [tuple(e) for e in ost.migration_log]


def test_step_host_from_device_state_continues_the_device_trajectory():
    """A device population downloaded into host buffers and stepped there
    follows the same fp64 trajectory as the device engine."""
    inst = qsb.taillard_uniform(40)
    cfg = qsb.SolverConfig(swarms=9, swarm_size=6, seed=2, migration_factor=0.34,
                           migration_period=2, coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, inst)
    for _ in range(3):
        qsb.step(st, inst, cfg)
    hp = host.HostPopulation.from_state(st, cfg)
    for _ in range(4):
        qsb.step(st, inst, cfg)
        host.step_host(hp, inst, cfg)
    assert hp.V.tobytes() == st.V.tobytes()
    assert np.array_equal(hp.perms, st.perms) and np.array_equal(hp.X, st.X)
    assert np.array_equal(hp.PL, st.PL) and np.array_equal(hp.cost, st.cost)
    assert np.array_equal(hp.bests.costs, st.bests.costs)
    assert np.array_equal(hp.bests.matrices, st.bests.matrices)
    assert (hp.best_cost, hp.best_iteration) == (st.best_cost, st.best_iteration)
    assert [tuple(e) for e in hp.migration_log] == [tuple(e) for e in st.migration_log[-2 * 3:]]


def test_step_reference_state_on_reference_layout_object(golden_instances):
    """host.step_reference_state on an object with exactly the reference's
    PopulationState fields (engine.py:85-124), as the Level-1b drop-in binds
    it: every field equals the oracle after every step, including the
    scalar best record, the X / perms swaps and the migration log."""
    from types import SimpleNamespace
    inst = golden_instances["tai30"]
    cfg = qsb.SolverConfig(swarms=6, swarm_size=7, seed=19, migration_factor=0.34,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    ost = orc.init_population(6, 7, inst.n, inst.flow, inst.distance, seed=19)
    ref = SimpleNamespace(
        X=ost.X.copy(), X_new=ost.X_new.copy(), V=ost.V.copy(), PL=ost.PL.copy(),
        perms=ost.perms.copy(), perms_new=ost.perms_new.copy(), pl_perms=ost.pl_perms.copy(),
        cost=ost.cost.copy(), pl_cost=ost.pl_cost.copy(),
        bests=qsb.SwarmBestTable(matrices=ost.pg_mats.copy(), perms=ost.pg_perms.copy(),
                                 costs=ost.pg_costs.copy()),
        n=inst.n, num_particles=42, swarms=6, swarm_size=7, t=0,
        best_perm=ost.best_perm.copy(), best_cost=ost.best_cost, best_iteration=0,
        pmf_range=(0.0, 1.0), migration_log=[])
    kw = orc.coeff_kwargs(cfg)
    for k in range(5):
        host.step_reference_state(ref, inst, cfg)
        orc.step(ost, inst.flow, inst.distance, **kw)
        for name in ("X", "V", "PL", "perms", "cost", "pl_cost", "pl_perms"):
            assert getattr(ref, name).tobytes() == getattr(ost, name).tobytes(), (k, name)
        assert ref.bests.matrices.tobytes() == ost.pg_mats.tobytes()
        assert np.array_equal(ref.bests.costs, ost.pg_costs)
        assert (ref.best_cost, ref.best_iteration, ref.t) == (ost.best_cost, ost.best_iteration, ost.t)
        assert np.array_equal(ref.best_perm, ost.best_perm)
    assert [tuple(e) for e in ref.migration_log] == [tuple(e) for e in ost.migration_log]
