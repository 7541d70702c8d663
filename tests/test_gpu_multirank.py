"""The sharded (multi-rank) engine with its real kernels: world-size-2
process groups share this box's GPU over gloo (host-level collectives only,
no kernel waits on another rank), run migration epochs through
``shard.make_exchange`` (qsb_migrate modes 1 / 2) and must reproduce the
single-rank trajectory bit for bit in fp64 parity mode."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

STEPS = 7


def _cfg(qsb, precision):
    return qsb.SolverConfig(swarms=6, swarm_size=12, seed=17, precision=precision,
                            migration_factor=0.34, migration_period=2,
                            coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))


def _worker(rank, world, port, precision, out):
    import paper_1504_05158_b200 as qsb
    from paper_1504_05158_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = qsb.taillard_uniform(20)
        cfg = _cfg(qsb, precision)
        lo, hi = shard.swarm_range(cfg.swarms, world, rank)
        st = qsb.init_population(cfg, inst, device="cuda:0", swarm_range=(lo, hi))
        ex = shard.make_exchange(world)
        for _ in range(STEPS):
            qsb.step(st, inst, cfg, exchange=ex)
        torch.cuda.synchronize()
        best = shard.merge_best(st.best_cost, st.best_iteration, 0, st.best_perm, world,
                                torch.device("cpu"))
        out[rank] = dict(perms=st.perms, cost=st.cost, pl_cost=st.pl_cost,
                         pg=st.bests.costs, pg_perms=st.bests.perms,
                         V=st.V, best=(int(best.cost), int(best.iteration)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_two_ranks_match_one(precision):
    import paper_1504_05158_b200 as qsb
    inst = qsb.taillard_uniform(20)
    cfg = _cfg(qsb, precision)
    ref = qsb.init_population(cfg, inst)
    for _ in range(STEPS):
        qsb.step(ref, inst, cfg)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, 2, port, precision, out)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(300)
        assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
        res = [out[0], out[1]]
    cat = lambda k: np.concatenate([res[0][k], res[1][k]])
    assert np.array_equal(cat("perms"), ref.perms)
    assert np.array_equal(cat("cost"), ref.cost)
    assert np.array_equal(cat("pl_cost"), ref.pl_cost)
    assert np.array_equal(cat("pg"), ref.bests.costs)
    assert np.array_equal(cat("pg_perms"), ref.bests.perms)
    assert cat("V").tobytes() == ref.V.tobytes()
    assert res[0]["best"] == res[1]["best"] == (int(ref.best_cost), int(ref.best_iteration))


# ------------------------------------------------------------ ring mode
RING_STEPS = 9


def _ring_cfg(qsb, precision="fp64", seed=17, iters=RING_STEPS):
    return qsb.SolverConfig(swarms=10, swarm_size=8, seed=seed, precision=precision,
                            migration_factor=0.4, migration_period=3, max_iterations=iters,
                            coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))


def _ring_worker(rank, world, port, out, seeds, iters):
    import paper_1504_05158_b200 as qsb
    from paper_1504_05158_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inst = qsb.taillard_uniform(20)
        res = {}
        for seed in seeds:
            cfg = _ring_cfg(qsb, seed=seed, iters=iters)
            lo, hi = shard.swarm_range(cfg.swarms, world, rank)
            st = qsb.init_population(cfg, inst, device="cuda:0", swarm_range=(lo, hi))
            ex = shard.make_ring_exchange(world, rank, cfg)
            for _ in range(iters):
                qsb.step(st, inst, cfg, exchange=ex)
            torch.cuda.synchronize()
            best = shard.merge_best(st.best_cost, st.best_iteration, 0, st.best_perm, world,
                                    torch.device("cpu"))
            res[seed] = dict(perms=st.perms, cost=st.cost, pg=st.bests.costs,
                             pg_perms=st.bests.perms, best=int(best.cost))
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _run_ring(world, seeds, iters):
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        port = _free_port()
        procs = [ctx.Process(target=_ring_worker, args=(r, world, port, out, seeds, iters))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(600)
        assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
        return [dict(out[r]) for r in range(world)]


def test_ring_two_ranks_equal_oracle():
    """Two ranks, ring migration every 3 iterations: positions, costs and
    swarm bests equal the oracle (fp64 steps, oracle.ring_migrate epochs)."""
    import paper_1504_05158_b200 as qsb
    from paper_1504_05158_b200 import shard
    from oracle import oracle as orc
    inst = qsb.taillard_uniform(20)
    cfg = _ring_cfg(qsb)
    res = _run_ring(2, [cfg.seed], RING_STEPS)
    kw = orc.coeff_kwargs(cfg)
    kw["migration_factor"] = 0.0
    st = orc.init_population(cfg.swarms, cfg.swarm_size, 20, inst.flow, inst.distance,
                             seed=cfg.seed)
    d = shard.ring_depth(cfg, 2)
    S = cfg.swarm_size
    for _ in range(RING_STEPS):
        orc.step(st, inst.flow, inst.distance, **kw)
        if st.t % cfg.migration_period == 0:
            shards = []
            for r in range(2):
                lo, hi = shard.swarm_range(cfg.swarms, 2, r)
                shards.append(dict(pg_costs=st.pg_costs[lo:hi], pg_perms=st.pg_perms[lo:hi],
                                   perms=st.perms[lo * S:hi * S], cost=st.cost[lo * S:hi * S]))
            orc.ring_migrate(shards, d, cfg.seed, st.t, S)
            st.pg_mats = orc.matrices_from_perms(st.pg_perms, 20)
    got = [res[0][cfg.seed], res[1][cfg.seed]]
    cat = lambda k: np.concatenate([got[0][k], got[1][k]])
    assert np.array_equal(cat("perms"), st.perms)
    assert np.array_equal(cat("cost"), st.cost)
    assert np.array_equal(cat("pg"), st.pg_costs)
    assert np.array_equal(cat("pg_perms"), st.pg_perms)


def test_ring_one_rank_is_reference_migration():
    """world == 1: the ring closes on the rank itself and every epoch is the
    reference migration (migration.py:55-86) bit for bit."""
    import paper_1504_05158_b200 as qsb
    from paper_1504_05158_b200 import shard
    inst = qsb.taillard_uniform(20)
    cfg = _ring_cfg(qsb)
    a = qsb.init_population(cfg, inst)
    b = qsb.init_population(cfg, inst)
    ex = shard.make_ring_exchange(1, 0, cfg)
    for _ in range(RING_STEPS):
        qsb.step(a, inst, cfg)
        qsb.step(b, inst, cfg, exchange=ex)
    assert np.array_equal(a.perms, b.perms)
    assert np.array_equal(a.bests.costs, b.bests.costs)
    assert a.V.tobytes() == b.V.tobytes()


def test_ring_final_best_distribution_matches_rank_migration():
    """Non-parity mode, statistical check over 24 seeds: the final global
    best of the two-rank ring is not distinguishable from the reference's
    rank-based migration at alpha = 0.01 (two-sided Mann-Whitney U)."""
    from scipy.stats import mannwhitneyu
    import paper_1504_05158_b200 as qsb
    inst = qsb.taillard_uniform(20)
    seeds = list(range(100, 124))
    iters = 60
    ring = _run_ring(2, seeds, iters)
    ring_best = np.array([ring[0][s]["best"] for s in seeds])
    assert all(ring[0][s]["best"] == ring[1][s]["best"] for s in seeds)
    ref_best = np.array([qsb.run(_ring_cfg(qsb, seed=s, iters=iters), inst,
                                 collect_stats=False).best_cost for s in seeds])
    p = mannwhitneyu(ring_best, ref_best, alternative="two-sided").pvalue
    assert p > 0.01, (p, np.median(ring_best), np.median(ref_best))


def test_nccl_exchange_captured_in_graph_equals_eager():
    """The NCCL path of the sharded exchange, captured in step_many's CUDA
    graph: a one-rank NCCL process group (the only NCCL world one GPU
    allows) runs shard.make_exchange -- mode-1 plan/pack, an NCCL all-reduce
    of the donor records, mode-2 apply -- inside the captured graph, and the
    trajectory equals eager single-device steps bit for bit."""
    import paper_1504_05158_b200 as qsb
    from paper_1504_05158_b200 import shard
    if not dist.is_nccl_available():
        pytest.skip("NCCL backend not built")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        inst = qsb.taillard_uniform(20)
        cfg = qsb.SolverConfig(swarms=6, swarm_size=12, seed=17, precision="fp32",
                               migration_factor=0.34, migration_period=2,
                               coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
        ref = qsb.init_population(cfg, inst)
        for _ in range(13):
            qsb.step(ref, inst, cfg)
        st = qsb.init_population(cfg, inst)
        qsb.step_many(st, inst, cfg, 13, exchange=shard.make_exchange(1))
        torch.cuda.synchronize()
        assert np.array_equal(st.perms, ref.perms)
        assert np.array_equal(st.bests.costs, ref.bests.costs)
        assert np.array_equal(st.bests.perms, ref.bests.perms)
        assert st.V.tobytes() == ref.V.tobytes()
    finally:
        dist.destroy_process_group()
