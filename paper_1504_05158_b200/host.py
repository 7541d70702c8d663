"""The reference's population in HOST memory, stepped on the GPU.

:class:`HostPopulation` holds exactly the reference's PopulationState buffers
(engine.py:85-124): float64 V, int8 0/1 matrices X / X_new / PL and the
swarm-best matrices, int64 permutations and costs.  :func:`step_host` is
engine.step (engine.py:181-244) with phases 1-5 in one C-ABI call,
``qsb_step_host`` (include/qapswarm_b200.h): every call ships the state to
the device and back (swarm-aligned chunks, copies overlapped with the fused
fp64 kernels), so the results are the reference's, bit for bit, and the
PCIe traffic is the price of keeping the state on the host.  This is the
binding a maintainer of the reference would add (Level 1);
the device-resident engine (engine.py) is the fast path.

The buffers are allocated in pinned host memory when CUDA is available.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .config import SX_CODES, SolverConfig
from .migration import MigrationEvent, SwarmBestTable


def _host_empty(shape, dtype, pinned: bool):
    if pinned:
        import torch
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64,
               np.dtype(np.int8): torch.int8, np.dtype(np.uint8): torch.uint8}[np.dtype(dtype)]
        return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()
    return np.empty(shape, dtype=dtype)


class HostPopulation:
    """engine.PopulationState (engine.py:85-124) in host memory."""

    def __init__(self, config: SolverConfig, n: int, integral: bool = True, pinned=None):
        if pinned is None:
            import torch
            pinned = torch.cuda.is_available()
        m, S = config.swarms, config.swarm_size
        p = m * S
        self.n, self.swarms, self.swarm_size = n, m, S
        ct = np.int64 if integral else np.float64
        e = lambda shape, dt: _host_empty(shape, dt, pinned)   # noqa: E731
        self.X, self.X_new, self.PL = (e((p, n, n), np.int8) for _ in range(3))
        self.V = e((p, n, n), np.float64)
        self.perms, self.perms_new, self.pl_perms = (e((p, n), np.int64) for _ in range(3))
        self.cost, self.pl_cost = e((p,), ct), e((p,), ct)
        self.improved = e((p,), np.uint8)
        self.bests = SwarmBestTable(matrices=e((m, n, n), np.int8), perms=e((m, n), np.int64),
                                    costs=e((m,), ct))
        self._best_perm = e((n,), np.int64)
        self._best_cost = e((1,), ct)
        self._best_iter = e((1,), np.int64)
        self.t = 0
        self.pmf_range = (0.0, 1.0)
        self.migration_log: list[MigrationEvent] = []
        self._log = np.zeros((max(1, config.migration_depth), 6), dtype=np.float64)

    @property
    def num_particles(self) -> int:
        return self.swarms * self.swarm_size

    def swarm_of(self, particle: int) -> int:
        return particle // self.swarm_size

    @property
    def best_cost(self):
        return self._best_cost[0].item()

    @property
    def best_iteration(self) -> int:
        return int(self._best_iter[0])

    @property
    def best_perm(self) -> np.ndarray:
        return self._best_perm

    @classmethod
    def from_state(cls, state, config: SolverConfig, pinned=None) -> "HostPopulation":
        """Download a device PopulationState into the reference layout."""
        hp = cls(config, state.n, state.integral, pinned)
        hp.X[...] = state.X
        hp.X_new[...] = state.X_new
        hp.PL[...] = state.PL
        hp.V[...] = state.V
        hp.perms[...] = state.perms
        hp.perms_new[...] = state.perms_new
        hp.pl_perms[...] = state.pl_perms
        hp.cost[...] = state.cost
        hp.pl_cost[...] = state.pl_cost
        b = state.bests
        hp.bests.matrices[...] = b.matrices
        hp.bests.perms[...] = b.perms
        hp.bests.costs[...] = b.costs
        hp._best_perm[...] = state.best_perm
        hp._best_cost[0] = state.best_cost
        hp._best_iter[0] = state.best_iteration
        hp.t = state.t
        hp.pmf_range = state.pmf_range
        return hp

    def c_struct(self) -> _lib.QsbHostPopulation:
        s = _lib.QsbHostPopulation()
        s.n = self.n
        s.cost_dtype = _lib.I64 if self.cost.dtype == np.int64 else _lib.F64
        s.num_particles, s.swarm_size, s.num_swarms = self.num_particles, self.swarm_size, self.swarms
        for name, arr in (("V", self.V), ("X_new", self.X_new), ("PL", self.PL),
                          ("perms", self.perms), ("perms_new", self.perms_new),
                          ("pl_perms", self.pl_perms), ("cost", self.cost), ("pl_cost", self.pl_cost),
                          ("improved", self.improved), ("pg_mats", self.bests.matrices),
                          ("pg_perms", self.bests.perms), ("pg_costs", self.bests.costs),
                          ("best_perm", self._best_perm), ("best_cost", self._best_cost),
                          ("best_iteration", self._best_iter)):
            assert arr.flags["C_CONTIGUOUS"]
            setattr(s, name, arr.ctypes.data)
        return s

    def transfer_bytes(self, instance, migrate: bool = False) -> tuple[int, int]:
        """(host->device, device->host) bytes one step_host call moves."""
        p, n, m = self.num_particles, self.n, self.swarms
        nn = n * n
        f, d = np.asarray(instance.flow), np.asarray(instance.distance)
        narrow = (f.dtype.kind in "iu" and d.dtype.kind in "iu" and min(f.min(), d.min()) >= 0
                  and max(f.max(), d.max()) < 1 << 16)
        h2d = (p * (8 * nn + 8 * n + 8 * n + 8) + m * (8 * n + 8) + 8 * n + 16
               + 2 * nn * (2 if narrow else 8))
        d2h = p * (8 * nn + nn + 8 * n + 8 * n + 8 + 8 + 1) + m * (8 * n + 8) + 8 * n + 16
        if migrate:
            d2h += self._log.nbytes
        return h2d, d2h


def _instance_struct(instance):
    f = np.asarray(instance.flow)
    d = np.asarray(instance.distance)
    integral = f.dtype.kind in "iu" and d.dtype.kind in "iu"
    dt = np.int64 if integral else np.float64
    f = np.ascontiguousarray(f, dtype=dt)
    d = np.ascontiguousarray(d, dtype=dt)
    hi = _lib.QsbHostInstance(int(instance.n), _lib.I64 if integral else _lib.F64,
                              f.ctypes.data, d.ctypes.data)
    return hi, (f, d)


def step_host(hp: HostPopulation, instance, config: SolverConfig) -> HostPopulation:
    """engine.step (engine.py:181-244) on host buffers: one ``qsb_step_host``
    call (draws, velocity, aggregation, goal, bests, migration on the device,
    fp64 reference arithmetic), then the X / X_new swap on the host."""
    c = config.coefficients
    if c.sx_mode == "second-target" and not c.depth < hp.n:
        raise ValueError(f"depth {c.depth} must be below the problem size {hp.n}")
    if config.two_opt_passes:
        raise ValueError("two_opt_passes is not available on host buffers (use the device engine)")
    t = hp.t + 1
    if not 0 <= t < 1 << 32:
        raise ValueError(f"iteration {t} outside supported range")
    d = config.migration_depth if (config.migration_factor > 0.0
                                   and t % config.migration_period == 0) else 0
    co = _lib.QsbCoeffs(c.c1, c.c2, c.c3, c.v_max, int(c.sv_mode == "norm"), SX_CODES[c.sx_mode],
                        c.depth, 0, int(config.seed) & (2**64 - 1))
    hi, keep = _instance_struct(instance)
    if d > hp._log.shape[0]:
        hp._log = np.zeros((d, 6), dtype=np.float64)
    _lib.call("qsb_step_host", hp.c_struct(), hi, co, t, d, hp._log.ctypes.data)
    del keep
    hp.X, hp.X_new = hp.X_new, hp.X
    hp.perms, hp.perms_new = hp.perms_new, hp.perms
    for r in hp._log[:d]:
        hp.migration_log.append(MigrationEvent(int(r[0]), int(r[1]), int(r[2]), int(r[3]),
                                               float(r[4]), float(r[5])))
    hp.t = t
    return hp


def step_reference_state(state, instance, config) -> object:
    """``engine.step(state, instance, config)`` for an object laid out like the
    reference's own ``PopulationState`` (engine.py:85-124: X, X_new, V, PL,
    perms, perms_new, pl_perms, cost, pl_cost, bests, best_perm, best_cost,
    best_iteration, t, migration_log) -- the one-line drop-in of
    INTEGRATION.md Level 1b.  The reference's buffers are used in place (no
    copies on the host); the scalar best-so-far fields go through small
    arrays and are written back, X / X_new and perms / perms_new are swapped
    as engine.py:231-232 does."""
    hp = object.__new__(HostPopulation)
    hp.n, hp.swarms, hp.swarm_size = state.n, state.swarms, state.swarm_size
    for name in ("X", "X_new", "V", "PL", "perms", "perms_new", "pl_perms", "cost", "pl_cost",
                 "bests"):
        setattr(hp, name, getattr(state, name))
    ct = state.cost.dtype
    hp.improved = getattr(state, "_b200_improved", None)
    if hp.improved is None or hp.improved.shape[0] != state.cost.shape[0]:
        hp.improved = np.empty(state.cost.shape[0], dtype=np.uint8)
        try:
            state._b200_improved = hp.improved
        except AttributeError:
            pass
    hp._best_perm = np.ascontiguousarray(state.best_perm, dtype=np.int64)
    hp._best_cost = np.array([state.best_cost], dtype=ct)
    hp._best_iter = np.array([state.best_iteration], dtype=np.int64)
    hp.t = state.t
    hp.pmf_range = getattr(state, "pmf_range", (0.0, 1.0))
    hp.migration_log = state.migration_log
    hp._log = np.zeros((max(1, config.migration_depth), 6), dtype=np.float64)
    step_host(hp, instance, config)
    state.X, state.X_new = hp.X, hp.X_new
    state.perms, state.perms_new = hp.perms, hp.perms_new
    if state.best_perm is not hp._best_perm:
        state.best_perm = hp._best_perm
    state.best_cost = hp._best_cost[0].item()
    state.best_iteration = int(hp._best_iter[0])
    state.t = hp.t
    return state
