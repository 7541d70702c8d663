"""Best-solution exchange between swarms (the reference's migration.py).

Rank-based scheme of migration.py:55-86: swarms are ranked by their best
cost (stable sort), the d best-ranked swarms each donate the CURRENT
solution of one uniformly drawn particle (anti-cloning), which replaces the
stored best of the d worst-ranked swarms (rank m-1-k receives from rank k),
accepting worse values.

Inside the engine the ranking and copies run in ``migrate_kernel``; only the
donor offsets -- ``rng.integers(0, S)`` once per replacement, a pure
function of (seed, t) -- are drawn on the host.  :func:`migrate` below is
the reference-layout entry point on host numpy buffers.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np


@dataclass
class SwarmBestTable:
    """Per-swarm bests: matrix view, vector view and cost (migration.py:23-41)."""

    matrices: np.ndarray   # (m, n, n) int8
    perms: np.ndarray      # (m, n) int64
    costs: np.ndarray      # (m,) int64 or float64

    @property
    def num_swarms(self) -> int:
        return self.costs.shape[0]

    def check(self):
        """Permutation-matrix invariants (used by tests)."""
        m = self.matrices
        if not ((m.sum(axis=1) == 1).all() and (m.sum(axis=2) == 1).all()):
            raise AssertionError("swarm best is not a permutation matrix")
        if not (np.argmax(m, axis=1) == self.perms).all():
            raise AssertionError("matrix and vector views disagree")


class MigrationEvent(NamedTuple):
    """One replacement: which particle's solution went to which swarm."""

    iteration: int
    source_swarm: int
    target_swarm: int
    particle: int
    old_cost: float
    new_cost: float


def migrate(d: int, bests: SwarmBestTable, perms: np.ndarray, matrices: np.ndarray,
            costs: np.ndarray, swarm_size: int, rng: np.random.Generator,
            iteration: int = 0, device=None) -> list[MigrationEvent]:
    """Reference-layout migration on host buffers (migration.py:55-86), run by
    the device kernel.  Mutates ``bests`` in place; returns the events."""
    import torch
    from . import _lib

    m = bests.num_swarms
    if not 0 <= d < m / 2:
        raise ValueError(f"migration depth must satisfy 0 <= d < m/2 = {m / 2}, got {d}")
    if swarm_size < 1 or perms.shape[0] != m * swarm_size:
        raise ValueError("population shape does not match swarms * swarm_size")
    if d == 0:
        return []
    picks = np.array([rng.integers(0, swarm_size) for _ in range(d)], dtype=np.int32)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = perms.shape[1]
    integral = costs.dtype.kind in "iu"
    cdt = torch.int64 if integral else torch.float64
    d_perm = torch.from_numpy(np.ascontiguousarray(perms, dtype=np.int16)).to(dev)
    d_cost = torch.from_numpy(np.ascontiguousarray(costs)).to(dev, cdt)
    d_pg_perm = torch.from_numpy(np.ascontiguousarray(bests.perms, dtype=np.int16)).to(dev)
    d_pg_cost = torch.from_numpy(np.ascontiguousarray(bests.costs)).to(dev, cdt)
    t_dev = torch.tensor([iteration], dtype=torch.int64, device=dev)
    plan = torch.zeros((d, 4), dtype=torch.int64, device=dev)
    log = torch.zeros((1, d, 6), dtype=torch.float64, device=dev)
    log_count = torch.zeros(1, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    d_picks = torch.from_numpy(picks).to(dev)

    st = _lib.QsbState()
    st.n, st.vstride = n, n * n
    st.v_dtype = _lib.F64
    st.cost_dtype = _lib.I64 if integral else _lib.F64
    st.num_particles, st.swarm_size, st.num_swarms = m * swarm_size, swarm_size, m
    st.perm, st.cost = d_perm.data_ptr(), d_cost.data_ptr()
    st.pg_perm, st.pg_cost = d_pg_perm.data_ptr(), d_pg_cost.data_ptr()
    st.iteration = t_dev.data_ptr()
    mig = _lib.QsbMigration()
    mig.d, mig.period, mig.mode = d, 0, 0
    mig.num_swarms_total = m
    mig.picks, mig.picks_epoch0, mig.picks_rows = d_picks.data_ptr(), iteration, 1
    mig.all_pg_cost = d_pg_cost.data_ptr()
    mig.plan = plan.data_ptr()
    mig.log, mig.log_rows, mig.log_count = log.data_ptr(), 1, log_count.data_ptr()
    mig.status = status.data_ptr()
    _lib.call("qsb_migrate", st, mig, torch.cuda.current_stream(dev).cuda_stream)
    new_perms = d_pg_perm.cpu().numpy().astype(np.int64)
    new_costs = d_pg_cost.cpu().numpy()
    rows = log[0].cpu().numpy()
    changed = rows[:, 2].astype(np.int64)
    bests.perms[changed] = new_perms[changed]
    bests.costs[changed] = new_costs[changed].astype(bests.costs.dtype)
    mats = np.zeros((changed.size, n, n), dtype=bests.matrices.dtype)
    mats[np.arange(changed.size)[:, None], new_perms[changed], np.arange(n)[None, :]] = 1
    bests.matrices[changed] = mats
    return [MigrationEvent(int(r[0]), int(r[1]), int(r[2]), int(r[3]), float(r[4]), float(r[5]))
            for r in rows]
