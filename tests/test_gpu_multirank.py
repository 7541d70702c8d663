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
