"""Multi-rank swarm sharding on CPU: world-size-2 gloo process groups run the
product's collective choreography (paper_1504_05158_b200/shard.py) with CPU
stand-ins for the two device kernels of a sharded migration epoch, and must
reproduce the single-process reference migration (migration.py:55-86)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1504_05158_b200 import engine, shard
from oracle import oracle as orc


def test_swarm_range_partitions():
    for m, w in [(800, 8), (800, 3), (5, 2), (7, 7)]:
        spans = [shard.swarm_range(m, w, r) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(hi - lo for lo, hi in spans) - min(hi - lo for lo, hi in spans) <= 1
    with pytest.raises(ValueError):
        shard.swarm_range(3, 4, 0)


# ------------------------------------------- CPU stand-ins of the kernels
def plan_pack(all_costs, picks, S, m0, m_local, perms_local, costs_local, n):
    """migrate_kernel mode 1: stable ranking, plan, pack local donors."""
    m = all_costs.size
    order = np.argsort(all_costs, kind="stable")
    d = picks.size
    plan = np.zeros((d, 3), np.int64)
    rec = np.zeros((d, n + 1), np.int64)
    for k in range(d):
        src, dst = int(order[k]), int(order[m - 1 - k])
        particle = src * S + int(picks[k])
        plan[k] = (src, dst, particle)
        if m0 <= src < m0 + m_local:
            lp = particle - m0 * S
            rec[k, 0] = costs_local[lp]
            rec[k, 1:] = perms_local[lp]
    return plan, rec


def apply(plan, rec, m0, m_local, pg_perms_local, pg_costs_local):
    """migrate_kernel mode 2: write the records of the swarms owned here."""
    for k in range(plan.shape[0]):
        dst = int(plan[k, 1]) - m0
        if 0 <= dst < m_local:
            pg_costs_local[dst] = rec[k, 0]
            pg_perms_local[dst] = rec[k, 1:]


def _worker(rank, world, port, swarms, S, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1504_05158_b200 as qsb
        inst = qsb.taillard_uniform(12, seed=77)
        n = 12
        kw = dict(c1=0.8, c2=0.5, c3=0.5, v_max=4.0, sv_mode="norm", sx_mode="second-target",
                  depth=2, seed=seed)
        st = orc.init_population(swarms, S, n, inst.flow, inst.distance, seed=seed)
        for _ in range(3):
            orc.step(st, inst.flow, inst.distance, **kw)
        t = st.t
        d = int(0.4 * swarms)
        # single-process reference migration on a copy
        ref = orc.init_population(swarms, S, n, inst.flow, inst.distance, seed=seed)
        for _ in range(3):
            orc.step(ref, inst.flow, inst.distance, **kw)
        orc.migrate(d, ref, orc.phase_rng(seed, orc.PHASE_HOST, t), iteration=t)

        # sharded: this rank's swarms and particles only
        m0, m1 = shard.swarm_range(swarms, world, rank)
        ml = m1 - m0
        perms_l = st.perms[m0 * S:m1 * S].copy()
        costs_l = st.cost[m0 * S:m1 * S].copy()
        pg_perms_l = st.pg_perms[m0:m1].copy()
        pg_costs_l = st.pg_costs[m0:m1].copy()
        full = shard.gather_swarm_costs(torch.from_numpy(pg_costs_l), swarms, world).numpy()
        assert np.array_equal(full, st.pg_costs)
        picks = orc.migration_picks(seed, t, d, S)
        plan, rec = plan_pack(full, picks, S, m0, ml, perms_l, costs_l, n)
        rec_t = shard.exchange_records(torch.from_numpy(rec))
        apply(plan, rec_t.numpy(), m0, ml, pg_perms_l, pg_costs_l)
        got_costs = shard.gather_swarm_costs(torch.from_numpy(pg_costs_l), swarms, world).numpy()
        perm_rows = [torch.zeros((shard.swarm_range(swarms, world, r)[1] -
                                  shard.swarm_range(swarms, world, r)[0], n), dtype=torch.int64)
                     for r in range(world)]
        pad = max(p.shape[0] for p in perm_rows)
        buf = torch.zeros((pad, n), dtype=torch.int64)
        buf[:ml] = torch.from_numpy(pg_perms_l)
        allp = [torch.zeros((pad, n), dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allp, buf)
        got_perms = np.concatenate([allp[r][:perm_rows[r].shape[0]].numpy() for r in range(world)])
        ok_mig = np.array_equal(got_costs, ref.pg_costs) and np.array_equal(got_perms, ref.pg_perms)

        # global best: lexicographic (cost, iteration, index) over the ranks
        lc = st.cost[m0 * S:m1 * S]
        li = int(np.argmin(lc))
        best = shard.merge_best(int(lc[li]), t, m0 * S + li, st.perms[m0 * S + li], world,
                                torch.device("cpu"))
        gi = int(np.argmin(st.cost))
        ok_best = best.cost == int(st.cost[gi]) and best.index == gi and \
            np.array_equal(best.perm, st.perms[gi])
        out[rank] = (ok_mig, ok_best)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("swarms,S", [(10, 6), (7, 5)])
def test_sharded_migration_equals_single_process(swarms, S):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, swarms, S, 13, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert out[0] == (True, True) and out[1] == (True, True)


# ------------------------------------------------------------ ring mode
def _ring_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rows = torch.full((3, 5), 10 * rank, dtype=torch.int64) + torch.arange(5)
        got = shard.send_recv_ring(rows.clone(), (rank + 1) % world, (rank - 1) % world)
        prev = (rank - 1) % world
        out[rank] = bool(torch.equal(got, torch.full((3, 5), 10 * prev, dtype=torch.int64)
                                     + torch.arange(5)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ring_send_recv_moves_records_to_next_rank(world):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert all(out[r] for r in range(world))


def test_ring_depth_and_world1_oracle_equals_reference_migration():
    from types import SimpleNamespace
    cfg = SimpleNamespace(migration_factor=0.33, swarms=800)
    assert shard.ring_depth(cfg, 1) == int(0.33 * 800)
    assert shard.ring_depth(cfg, 8) == int(0.33 * 100)
    # one rank: the ring closes on itself and the epoch is migration.migrate
    import paper_1504_05158_b200 as qsb
    inst = qsb.taillard_uniform(12, seed=5)
    kw = dict(c1=0.8, c2=0.5, c3=0.5, v_max=4.0, sv_mode="norm", sx_mode="second-target",
              depth=2, seed=21)
    st = orc.init_population(9, 4, 12, inst.flow, inst.distance, seed=21)
    for _ in range(2):
        orc.step(st, inst.flow, inst.distance, **kw)
    ref_c, ref_p = st.pg_costs.copy(), st.pg_perms.copy()
    d = int(0.34 * 9)
    sh = dict(pg_costs=st.pg_costs.copy(), pg_perms=st.pg_perms.copy(), perms=st.perms,
              cost=st.cost)
    orc.ring_migrate([sh], d, 21, st.t, 4)
    orc.migrate(d, st, orc.phase_rng(21, orc.PHASE_HOST, st.t), iteration=st.t)
    assert np.array_equal(sh["pg_costs"], st.pg_costs)
    assert np.array_equal(sh["pg_perms"], st.pg_perms)
    assert not np.array_equal(ref_c, st.pg_costs) or not np.array_equal(ref_p, st.pg_perms)
