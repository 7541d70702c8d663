"""The B200 solver engine: device-resident population, the fused step, runs.

Mirrors the reference engine (engine.py:29-307) -- same public functions,
signatures, field names and error messages -- while the particle state
lives in HBM as structure-of-arrays torch tensors and every phase of an
iteration runs in the sm_100a kernels of libqsb.so:

    reference phase (engine.step)          here
    -------------------------------------  ------------------------------------
    streams.step_draws   (engine.py:189)   in-kernel Philox, zero HBM bytes
    velocity_many        (engine.py:197)   \
    aggregate_many       (engine.py:203)    > one fused kernel (qsb_step)
    cost_many            (engine.py:207)    |
    personal bests       (engine.py:211)   /
    swarm/global bests   (engine.py:216)   best_kernel (one launch)
    X <-> X_new swap     (engine.py:231)   pointer swap of perm / perm_new
    migrate              (engine.py:235)   migrate_kernel (+ host picks)

Positions are int16 permutations (perm[c] = row of the 1 in column c,
core.py:5-6); the reference's 0/1 matrices, float64 velocities and int64
permutations are materialised on demand by the host-view properties of
:class:`PopulationState` (``X``, ``V``, ``PL``, ``perms``, ``bests`` ...).
"""

from __future__ import annotations

import math
import os as _os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import SX_CODES, PsoCoefficients, SolverConfig
from .core import gap
from .instance import device_format, is_integral
from .migration import MigrationEvent, SwarmBestTable
from .stats import PERCENTILE_RANKS, IterationStats, _ranks_sorted, collect

from .streams import PHASE_HOST, PHASE_INIT, PHASE_STEP, _ITER_LIMIT, _PARTICLE_LIMIT, phase_rng  # noqa: F401

_LOG_EPOCHS = 256


def projected_buffer_bytes(config: SolverConfig, n: int) -> int:
    """The reference's host-buffer estimate (engine.py:71-82), kept for
    drop-in memory guards."""
    p = config.num_particles
    mats = 3 * p * n * n * 1 + p * n * n * 8
    perms = 3 * p * n * 8
    tables = 3 * p * 8
    swarm = config.swarms * (n * n + n * 8 + 8)
    return mats + perms + tables + swarm


# fp32 states up to this n carry the lazily scaled layout (wide words, five
# column-state rows); the one-warp kernels since round 1, the multi-warp
# kernels (n <= 256) since round 2.  QSB_MW_DEFER=1 keeps n > 64 on the
# deferred column scale (A/B; read by libqsb too).
# first iteration run by the late-iteration kernel variant (QSB_HINT_LATE)
_CHAIN_T0 = int(_os.environ.get("QSB_CHAIN_T0", "120"))
# QSB_NO_COEF_FOLD=1: a separate draw pre-pass every step (A/B measurements)
_COEF_FOLD = _os.environ.get("QSB_NO_COEF_FOLD", "") != "1"
_LAZY_MAX_N = 64 if _os.environ.get("QSB_MW_DEFER", "") == "1" else 256


def _vcs(n: int) -> int:
    return (n + 3) // 4 * 4


def device_buffer_bytes(config: SolverConfig, n: int) -> int:
    """HBM bytes of this engine's state for one device holding every particle."""
    p = config.num_particles
    sv = 8 if config.precision == "fp64" else 4
    vstride = -(-n * n // (16 // sv)) * (16 // sv)
    vcol = 20 * _vcs(n) if sv == 4 else 0
    return p * (vstride * sv + vcol + 3 * n * 2 + 2 * 8 + 16 + 1) + config.swarms * (n * 2 + 3 * 8)


def _dev(device):
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise RuntimeError("the qapswarm-b200 engine runs on CUDA devices only")
    return device


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def wide_decode(w: torch.Tensor) -> torch.Tensor:
    """Wide 32-bit velocity words (held in a float32 tensor) -> float64: the
    word is the high half of the double (csrc/common.cuh wdec)."""
    return (w.contiguous().view(torch.int32).to(torch.int64) << 32).view(torch.float64)


def wide_encode(v: torch.Tensor) -> torch.Tensor:
    """float64 -> wide words, rounded to nearest (csrc/common.cuh wenc)."""
    b = (v.contiguous().view(torch.int64) + 0x80000000) >> 32
    return b.to(torch.int32).view(torch.float32)


class PopulationState:
    """Device-resident population (the reference's flat buffers,
    engine.py:85-124, as int16 permutations plus the velocity tensor).

    ``swarm_range`` selects the swarms this device owns (multi-GPU
    sharding); particle ids and random streams stay global, so any split
    reproduces the single-device trajectory.
    """

    def __init__(self, config: SolverConfig, instance, device=None, swarm_range=None):
        n = int(instance.n)
        dev = _dev(device)
        m_total = config.swarms
        m0, m1 = swarm_range if swarm_range is not None else (0, m_total)
        if not 0 <= m0 < m1 <= m_total:
            raise ValueError("swarm_range must be a non-empty sub-range of the swarms")
        if m_total * config.swarm_size >= _PARTICLE_LIMIT:
            raise ValueError(f"population {m_total * config.swarm_size} exceeds supported size")
        S = config.swarm_size
        p = (m1 - m0) * S
        self.n = n
        self.device = dev
        self.swarms = m_total
        self.swarm_size = S
        self.num_particles = m_total * S
        self.local_swarms = m1 - m0
        self.local_particles = p
        self.swarm_offset = m0
        self.particle_offset = m0 * S
        self.precision = config.precision
        self.v_code = _lib.F64 if config.precision == "fp64" else _lib.F32
        self.vstride = int(_lib.lib().qsb_vstride(n, self.v_code))
        self.integral = is_integral(instance)
        self.cost_code = _lib.I64 if self.integral else _lib.F64
        vdt = torch.float64 if self.v_code == _lib.F64 else torch.float32
        cdt = torch.int64 if self.integral else torch.float64
        z = dict(device=dev)
        try:
            self.d_V = torch.zeros((p, self.vstride), dtype=vdt, **z)
            self.d_perm = torch.zeros((p, n), dtype=torch.int16, **z)
            self.d_perm_new = torch.zeros((p, n), dtype=torch.int16, **z)
            self.d_pl_perm = torch.zeros((p, n), dtype=torch.int16, **z)
            self.d_cost = torch.zeros(p, dtype=cdt, **z)
            self.d_pl_cost = torch.zeros(p, dtype=cdt, **z)
            self.d_improved = torch.zeros(p, dtype=torch.uint8, **z)
            self.d_pg_perm = torch.zeros((self.local_swarms, n), dtype=torch.int16, **z)
            self.d_pg_cost = torch.zeros(self.local_swarms, dtype=cdt, **z)
            self.d_best_perm = torch.zeros(n, dtype=torch.int16, **z)
            self.d_best_cost = torch.zeros(1, dtype=cdt, **z)
            self.d_best_iter = torch.zeros(1, dtype=torch.int64, **z)
            self.d_best_idx = torch.zeros(1, dtype=torch.int64, **z)
            self.d_iteration = torch.zeros(1, dtype=torch.int64, **z)
            self.d_swarm_min = torch.zeros(self.local_swarms, dtype=cdt, **z)
            self.d_swarm_min_idx = torch.zeros(self.local_swarms, dtype=torch.int64, **z)
            self.d_done = torch.zeros(1, dtype=torch.int32, **z)
            self.d_work = torch.zeros(1, dtype=torch.int32, **z)
            self.d_step_coef = torch.zeros((p, 2), dtype=torch.float64, **z)
            # fp32 column state: the lazily scaled layout (one-warp kernel
            # variants, n <= 64) or, for n > 64, the deferred column scale
            # (row 0 only); V holds u, v = u * s per column; see
            # include/qapswarm_b200.h
            self.d_vcol = None
            # (QSB_NO_DEFER=1: multi-warp fp32 tiles normalised in place
            # instead, the pre-deferral layout, for A/B measurements)
            if self.v_code == _lib.F32 and (n <= _LAZY_MAX_N or not _os.environ.get("QSB_NO_DEFER")):
                self.d_vcol = torch.empty((p, 5, _vcs(n)), dtype=torch.float32, **z)
                self.reset_vcol()
        except torch.OutOfMemoryError:
            raise MemoryError(
                f"cannot allocate population buffers: {p} particles of size {n}x{n} need about "
                f"{device_buffer_bytes(config, n)} bytes") from None
        self.t = 0
        self.pmf_range = (0.0, 1.0)
        self._migration_log: list[MigrationEvent] = []
        self._mig = None          # migration scratch, allocated on first use
        self._host_best = None    # cached (cost, iteration, perm) of the device record
        self._inst = None
        self._cs = None
        self._stats_scratch = None
        self.launches = 0         # kernels launched by step() (bench accounting)
        self.v_bound = float("inf")   # proven bound on max |V| (enables QSB_HINT_V_BOUNDED)
        self.cost_current = False     # cost[p] == goal(perm[p]) (enables QSB_HINT_COST_CURRENT)
        # (t, c2, c3, seed): step_coef holds iteration t's draws, drawn by the
        # previous best update (enables QSB_HINT_COEF_READY)
        self.coef_ready = None

    # ---------------------------------------------------------- C structs
    def c_state(self) -> _lib.QsbState:
        s = self._cs
        if s is not None:
            s.perm, s.perm_new = self.d_perm.data_ptr(), self.d_perm_new.data_ptr()
            return s
        s = _lib.QsbState()
        s.n, s.vstride, s.v_dtype, s.cost_dtype = self.n, self.vstride, self.v_code, self.cost_code
        s.num_particles = self.local_particles
        s.swarm_size = self.swarm_size
        s.num_swarms = self.local_swarms
        s.particle_offset = self.particle_offset
        s.swarm_offset = self.swarm_offset
        for name in ("V", "perm", "perm_new", "pl_perm", "cost", "pl_cost", "improved",
                     "pg_perm", "pg_cost", "best_perm", "best_cost", "best_iter", "best_idx",
                     "swarm_min", "swarm_min_idx", "done", "work", "vcol", "step_coef"):
            setattr(s, name, _ptr(getattr(self, "d_" + name)))
        s.iteration = _ptr(self.d_iteration)
        self._cs = s
        return s

    def stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def swap_positions(self):
        self.d_perm, self.d_perm_new = self.d_perm_new, self.d_perm

    @property
    def migration_log(self) -> list:
        _drain_log(self)
        return self._migration_log

    def swarm_of(self, particle: int) -> int:
        return particle // self.swarm_size

    # ------------------------------------------- reference-layout host views
    def _mats(self, perms_t: torch.Tensor) -> np.ndarray:
        p = perms_t.shape[0]
        out = torch.empty((p, self.n, self.n), dtype=torch.int8, device=self.device)
        if p:
            _lib.call("qsb_perm_to_matrix", perms_t.data_ptr(), p, self.n, out.data_ptr(),
                      self.stream())
        return out.cpu().numpy()

    @property
    def X(self):
        return self._mats(self.d_perm)

    @property
    def X_new(self):
        return self._mats(self.d_perm_new)

    @property
    def PL(self):
        return self._mats(self.d_pl_perm)

    def reset_vcol(self):
        """Column state of the lazily scaled layout after V was written from
        outside the step: scale 1, statistics unknown (the next step runs
        the full pass)."""
        if self.d_vcol is not None:
            if self.v_wide:
                self.d_vcol[:, 0].view(torch.int32).fill_(0x3FF00000)   # the wide word of 1.0
            else:
                self.d_vcol[:, 0].fill_(1.0)
            self.d_vcol[:, 1:3].zero_()
            self.d_vcol[:, 3].fill_(float("nan"))
            self.d_vcol[:, 4].zero_()

    @property
    def v_wide(self) -> bool:
        """Lazily scaled fp32 tiles hold wide 32-bit words: the high word of
        the float64 value, rounded to nearest (fp32's size, fp64's exponent
        range; csrc/common.cuh wdec / wenc).  Stored-v fp32 tiles hold
        floats."""
        return (self.v_code == _lib.F32 and self.n <= _LAZY_MAX_N
                and getattr(self, "d_vcol", None) is not None)

    def v_decode(self, u: torch.Tensor) -> torch.Tensor:
        """Stored fp32-state words -> float64 values (exact)."""
        return wide_decode(u) if self.v_wide else u.double()

    def v_encode(self, v: torch.Tensor) -> torch.Tensor:
        """float64 values -> stored fp32-state words (rounded to nearest)."""
        return wide_encode(v) if self.v_wide else v.float()

    def set_lazy_scale(self, enabled: bool):
        """Switch the fp32 state to (or from) the lazily scaled layout; V is
        materialised (u * s, rounded to the stored format) when leaving it."""
        if self.n > _LAZY_MAX_N:
            return      # multi-warp kernels: the deferred column scale stays
        if not enabled and self.d_vcol is not None:
            p, n = self.local_particles, self.n
            u = self.d_V[:, :n * n].view(p, n, n)
            v = self.v_decode(u) * self.v_decode(self.d_vcol[:, 0, :n]).unsqueeze(1)
            self.d_vcol = None                # stored-v: plain floats
            u.copy_(v.float())
        elif enabled and self.d_vcol is None and self.v_code == _lib.F32 and self.n <= _LAZY_MAX_N:
            p, n = self.local_particles, self.n
            u = self.d_V[:, :n * n].view(p, n, n)
            v = u.double()
            self.d_vcol = torch.empty((p, 5, _vcs(n)), dtype=torch.float32, device=self.device)
            u.copy_(self.v_encode(v))         # lazily scaled: wide words
            self.reset_vcol()
        self._cs = None
        self._graph_cache = None

    @property
    def V(self):
        """Velocities (P, n, n); fp32 states return float64 when lazily
        scaled (u * s is exact in float64)."""
        p, n, nn = self.local_particles, self.n, self.n * self.n
        u = self.d_V[:, :nn].view(p, n, n)
        if self.d_vcol is not None:
            return (self.v_decode(u) * self.v_decode(self.d_vcol[:, 0, :n]).unsqueeze(1)).cpu().numpy()
        return u.cpu().numpy()

    @property
    def perms(self):
        return self.d_perm.cpu().numpy().astype(np.int64)

    @property
    def perms_new(self):
        return self.d_perm_new.cpu().numpy().astype(np.int64)

    @property
    def pl_perms(self):
        return self.d_pl_perm.cpu().numpy().astype(np.int64)

    @property
    def cost(self):
        return self.d_cost.cpu().numpy()

    @property
    def pl_cost(self):
        return self.d_pl_cost.cpu().numpy()

    @property
    def bests(self) -> SwarmBestTable:
        return SwarmBestTable(matrices=self._mats(self.d_pg_perm),
                              perms=self.d_pg_perm.cpu().numpy().astype(np.int64),
                              costs=self.d_pg_cost.cpu().numpy())

    def _best(self):
        if self._host_best is None:
            c = self.d_best_cost.cpu().numpy()[0].item()
            it = int(self.d_best_iter.cpu()[0])
            self._host_best = (c, it, self.d_best_perm.cpu().numpy().astype(np.int64))
        return self._host_best

    @property
    def best_cost(self):
        return self._best()[0]

    @property
    def best_iteration(self):
        return self._best()[1]

    @property
    def best_perm(self):
        return self._best()[2]


# ---------------------------------------------------------------- runtime
class _Runtime:
    """Per-(state, instance, coefficients) C structs, rebuilt only on change."""

    def __init__(self, state: PopulationState, instance, config: SolverConfig):
        f, d, code = device_format(instance)
        self.flow = torch.from_numpy(f.view(np.int16) if code == _lib.U16 else f).to(state.device)
        self.dist = torch.from_numpy(d.view(np.int16) if code == _lib.U16 else d).to(state.device)
        acc32 = 0
        if code == _lib.U16:
            acc32 = int(state.n * int(f.max()) * int(d.max()) < 2**32)
        self.inst = _lib.QsbInstance(state.n, code, self.flow.data_ptr(), self.dist.data_ptr(),
                                     acc32, 0)
        self.mat_code = code
        fa, da = np.asarray(instance.flow), np.asarray(instance.distance)
        sym = bool((fa == fa.T).all() and (da == da.T).all())
        self.symmetric = sym and code == _lib.U16          # 2-opt kernels' symmetric sweep
        self.symmetric_int = sym and code != _lib.F64      # incremental goal halving
        # byte-sized entries with int32-safe sums: the 2-opt dp4a kernel
        mf, md = (int(fa.max()), int(da.max())) if fa.size else (0, 0)
        self.twoopt_bytes = bool(code == _lib.U16 and max(mf, md) < 256 and state.n * mf * md < 2**31)
        self.instance = instance
        self.key = (config.coefficients, config.seed)
        c = config.coefficients
        self.coeffs = _lib.QsbCoeffs(c.c1, c.c2, c.c3, c.v_max, int(c.sv_mode == "norm"),
                                     SX_CODES[c.sx_mode], c.depth, 0, int(config.seed) & (2**64 - 1))
        if not _lib.lib().qsb_supported(state.n, state.v_code, code):
            raise ValueError(f"problem size {state.n} is not supported by the fused kernel "
                             f"at precision {config.precision}")


def _runtime(state: PopulationState, instance, config: SolverConfig) -> _Runtime:
    key = (config.coefficients, config.seed)
    rt = state._inst
    # keyed on the instance object itself (held by the runtime), not id():
    # a collected instance's id can be reused by a different one
    if rt is None or rt.instance is not instance or rt.key != key:
        if rt is not None and rt.instance is not instance:
            # the stored goals belong to the previous instance: the next
            # step evaluates the full goal (no incremental update)
            state.cost_current = False
        rt = _Runtime(state, instance, config)
        state._inst = rt
    return rt


# ----------------------------------------------------------------- init
def _reference_init_arrays(config: SolverConfig, n: int):
    """The reference's initial population (engine.py:150-156): row-wise
    numpy ``permuted`` then ``uniform(-amp, amp)`` from init_rng(seed)."""
    p = config.num_particles
    rng = phase_rng(config.seed, PHASE_INIT, 0)
    perms = rng.permuted(np.tile(np.arange(n, dtype=np.int64), (p, 1)), axis=1)
    amp = config.init_velocity_amplitude
    V = rng.uniform(-amp, amp, (p, n, n))
    return perms, V


def init_population(config: SolverConfig, instance, device=None, swarm_range=None) -> PopulationState:
    """Seeded population: random permutations, uniform velocities; personal
    bests = initial solutions; each swarm's best is its cheapest particle
    (engine.py:139-178)."""
    state = PopulationState(config, instance, device, swarm_range)
    n, p = state.n, state.local_particles
    lo_p = state.particle_offset
    rt = _runtime(state, instance, config)
    stream = state.stream()
    if config.init == "reference":
        perms, V = _reference_init_arrays(config, n)
        perms = perms[lo_p:lo_p + p]
        V = V[lo_p:lo_p + p]
        state.d_perm.copy_(torch.from_numpy(perms.astype(np.int16)))
        Vt = torch.from_numpy(np.ascontiguousarray(V.reshape(p, n * n), dtype=np.float64))
        state.d_V[:, :n * n].copy_(state.v_encode(Vt) if state.v_wide else Vt)
        del V
    else:
        _lib.call("qsb_init_population_device", state.c_state(), int(config.seed) & (2**64 - 1),
                  float(config.init_velocity_amplitude), stream)
    state.reset_vcol()
    _lib.call("qsb_cost", state.d_perm.data_ptr(), p, rt.inst, state.d_cost.data_ptr(), stream)
    state.d_pl_perm.copy_(state.d_perm)
    state.d_pl_cost.copy_(state.d_cost)
    # swarm / global bests of the initial population = one best-kernel pass
    # with every particle "improved" against +inf tables, at iteration 0
    big = torch.finfo(torch.float64).max if not state.integral else torch.iinfo(torch.int64).max
    state.d_pg_cost.fill_(big)
    state.d_best_cost.fill_(big)
    state.d_improved.fill_(1)
    state.d_iteration.fill_(-1)
    cs = state.c_state()
    cs.perm_new = state.d_perm.data_ptr()
    # (the pass also draws iteration 1's coefficients: *t_dev + 2 = 1)
    _best_update(cs, rt, stream)
    state.coef_ready = _coef_key(config, 1)
    state.t = 0
    state._host_best = None
    state.v_bound = float(config.init_velocity_amplitude)
    state.cost_current = True
    # the migration scratch (plan, device event log) is allocated here, not at
    # the first migration: a step() then never allocates device memory
    if config.migration_factor > 0.0 and config.migration_depth > 0:
        state._mig = _MigrationScratch(state, config.migration_depth)
    costs = state.d_cost.cpu().numpy()
    if state.local_particles != state.num_particles and torch.distributed.is_initialized():
        lo = torch.tensor([costs.min(), -costs.max()], dtype=torch.float64, device=state.device)
        torch.distributed.all_reduce(lo, op=torch.distributed.ReduceOp.MIN)
        lo_v, hi_v = float(lo[0]), float(-lo[1])
    else:
        lo_v, hi_v = float(costs.min()), float(costs.max())
    state.pmf_range = (lo_v, hi_v) if hi_v > lo_v else (lo_v, lo_v + 1.0)
    return state


# ------------------------------------------------------------- migration
class _MigrationScratch:
    """Device buffers of the migration phase.  The donor picks are drawn
    inside migrate_kernel from the reference's host stream (seed, t), so no
    host work is left in a migration epoch."""

    def __init__(self, state: PopulationState, d: int, log_rows: int = _LOG_EPOCHS):
        dev = state.device
        self.d = d
        self.device = dev
        self.plan = torch.zeros((d, 4), dtype=torch.int64, device=dev)
        self.log = torch.zeros((log_rows, d, 6), dtype=torch.float64, device=dev)
        self.log_count = torch.zeros(1, dtype=torch.int64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.records = torch.zeros((d, state.n + 1), dtype=torch.int64, device=dev)
        self.pending = 0          # epochs logged on the device, not yet drained

    def struct(self, state: PopulationState, config: SolverConfig) -> _lib.QsbMigration:
        mig = _lib.QsbMigration()
        mig.d, mig.period, mig.mode, mig.reserved = self.d, config.migration_period, 0, 0
        mig.num_swarms_total = state.swarms
        mig.picks, mig.picks_epoch0, mig.picks_rows = None, 0, 0    # drawn on the device
        mig.seed = int(config.seed) & (2**64 - 1)
        mig.all_pg_cost = state.d_pg_cost.data_ptr()
        mig.plan, mig.records = self.plan.data_ptr(), self.records.data_ptr()
        mig.log, mig.log_rows = self.log.data_ptr(), self.log.shape[0]
        mig.log_count = self.log_count.data_ptr()
        mig.status = self.status.data_ptr()
        return mig


def _drain_log(state: PopulationState):
    ms = state._mig
    if ms is None or ms.pending == 0:
        return
    if int(ms.status.item()) != 0:
        raise RuntimeError("migrate_kernel reported a missing donor-picks row (status "
                           f"{int(ms.status.item())}); migration events were dropped")
    rows = ms.log[:ms.pending].cpu().numpy().reshape(-1, 6)
    for r in rows:
        state._migration_log.append(MigrationEvent(int(r[0]), int(r[1]), int(r[2]), int(r[3]),
                                                   float(r[4]), float(r[5])))
    ms.log_count.zero_()
    ms.pending = 0


def migration_struct(state: PopulationState, config: SolverConfig, t: int) -> _lib.QsbMigration:
    """C descriptor of the migration event at iteration t."""
    d = config.migration_depth
    if state._mig is None or state._mig.d != d:
        _drain_log(state)
        state._mig = _MigrationScratch(state, d)
    ms = state._mig
    if ms.pending >= ms.log.shape[0]:
        _drain_log(state)
    return ms.struct(state, config)


def _migrate_device(state: PopulationState, config: SolverConfig, t: int, exchange=None):
    mig = migration_struct(state, config, t)
    if exchange is None:
        _lib.call("qsb_migrate", state.c_state(), mig, state.stream())
    else:
        exchange(state, mig)
    if getattr(exchange, "logs_events", True):
        state._mig.pending += 1


# ------------------------------------------------------------ statistics
def collect_device(state: PopulationState, time_ms: float, bins: int = 60,
                   all_swarms: bool = False) -> IterationStats:
    """stats.collect (stats.py:72-100) with the O(P) parts on the device: the
    PMF histogram, the minimum and the four nearest-rank percentiles come
    from qsb_population_stats; only the swarm-best table and the best
    swarm's costs cross to the host.  Field values and types are identical to
    :func:`stats.collect` (same float64 binning, same k-th smallest)."""
    import ctypes
    P = state.local_particles
    lo, hi = state.pmf_range
    if bins < 1:
        raise ValueError(f"bins must be >= 1, got {bins}")
    if not lo < hi:
        raise ValueError(f"invalid range: [{lo}, {hi}]")
    width = (hi - lo) / bins
    ks = [math.ceil(r / 100.0 * P) - 1 for r in PERCENTILE_RANKS]
    sc = state._stats_scratch
    if sc is None or sc[1].numel() < bins:
        work = torch.empty(int(_lib.lib().qsb_stats_work_bytes()), dtype=torch.uint8, device=state.device)
        sc = (work, torch.empty(max(bins, 64), dtype=torch.int32, device=state.device),
              torch.empty(8, dtype=torch.int64, device=state.device))
        state._stats_scratch = sc
    work, hist, out = sc
    karr = (ctypes.c_int64 * 4)(*ks)
    _lib.call("qsb_population_stats", state.d_cost.data_ptr(), state.cost_code, P, float(lo),
              float(width), bins, karr, 4, work.data_ptr(), hist.data_ptr(), out.data_ptr(),
              state.stream())
    vals = out.cpu().numpy()[:5]
    if state.cost_code == _lib.F64:
        vals = vals.view(np.float64)
    counts = hist[:bins].cpu().numpy().astype(np.int64)
    freq = counts / P
    edges = lo + width * np.arange(bins + 1)
    table = state.d_pg_cost.cpu().numpy()
    best_swarm = int(np.argmin(table))
    S = state.swarm_size
    mine = state.d_cost[best_swarm * S:(best_swarm + 1) * S].cpu().numpy()
    all_ranks = None
    if all_swarms:
        srt = np.sort(state.d_cost.cpu().numpy().reshape(state.swarms, S), axis=1)
        all_ranks = np.array([_ranks_sorted(row) for row in srt], dtype=np.float64)
    p5, p25, p50, p75 = (vals[1 + i].item() for i in range(4))
    return IterationStats(
        t=state.t, p5=p5, p25=p25, p50=p50, p75=p75, best=vals[0].item(),
        global_best=state.best_cost, per_swarm_best=table.copy(), pmf_edges=edges, pmf_freq=freq,
        time_ms=time_ms, best_swarm=best_swarm,
        best_swarm_percentiles=tuple(_ranks_sorted(np.sort(mine))), all_swarm_percentiles=all_ranks)


# ------------------------------------------------------------------ step
def _hints(state: PopulationState, rt: "_Runtime", coeffs: PsoCoefficients) -> int:
    """Launch hints the state guarantees for its next step (QSB_HINT_*)."""
    # |c1 v| <= v_max for every stored v => the bulk-row clamp is a no-op
    hints = _lib.HINT_V_BOUNDED if coeffs.c1 * state.v_bound * (1 + 1e-6) <= coeffs.v_max else 0
    if state.cost_current and state.integral:
        hints |= _lib.HINT_COST_CURRENT
        if rt.symmetric_int:
            hints |= _lib.HINT_SYMMETRIC
    # past the first iterations the aggregation's bulk steps leave more free
    # columns (performance only; QSB_HINT_LATE in include/qapswarm_b200.h)
    if state.t + 1 >= _CHAIN_T0:
        hints |= _lib.HINT_LATE
    return hints


def _coef_key(config: SolverConfig, t: int):
    if not _COEF_FOLD:
        return None
    c = config.coefficients
    return (t, float(c.c2), float(c.c3), int(config.seed) & (2**64 - 1))


def _best_update(cs, rt: "_Runtime", stream) -> None:
    """Swarm / global best update; it also draws the next iteration's
    coefficients (qsb_best_update_next), so that step runs no pre-pass."""
    if _COEF_FOLD:
        _lib.call("qsb_best_update_next", cs, rt.coeffs, stream)
    else:
        _lib.call("qsb_best_update", cs, stream)


def _post_step_v_bound(coeffs: PsoCoefficients) -> float:
    """After S_v every entry is clamped to v_max, or normalised to |v| <= 1."""
    return (1.0 + 1e-6) if coeffs.sv_mode == "norm" else coeffs.v_max


def step(state: PopulationState, instance, config: SolverConfig, exchange=None,
         timer=None) -> PopulationState:
    """Advance one iteration (engine.py:181-244): the fused velocity /
    aggregation / goal / personal-best kernel, the swarm and global best
    reduction, the position swap and, when due, migration.

    ``exchange`` performs the cross-device part of migration when the
    swarms are sharded (see shard.py); ``timer`` (optional) brackets the
    fused kernel launch with CUDA events for roofline measurement."""
    coeffs = config.coefficients
    n = state.n
    if coeffs.sx_mode == "second-target" and not coeffs.depth < n:
        raise ValueError(f"depth {coeffs.depth} must be below the problem size {n}")
    t = state.t + 1
    if not 0 <= t < _ITER_LIMIT:
        raise ValueError(f"iteration {t} outside supported range")
    rt = _runtime(state, instance, config)
    stream = state.stream()
    cs = state.c_state()
    ready = _COEF_FOLD and state.coef_ready == _coef_key(config, t)
    rt.coeffs.hints = _hints(state, rt, coeffs) | (_lib.HINT_COEF_READY if ready else 0)
    passes = config.two_opt_passes
    if passes and not state.integral:
        raise ValueError("two_opt_passes requires an integral instance")
    flags = _lib.PHASE_ALL if not passes else _lib.PHASE_ALL & ~_lib.PHASE_PBEST
    if timer is not None:
        timer.before(stream)
    _lib.call("qsb_step_phases", cs, rt.inst, rt.coeffs, flags, None, 0, 2, None, 0, stream)
    if timer is not None:
        timer.after(stream)
    if passes:
        tf = (_lib.TWOOPT_PBEST | (_lib.TWOOPT_SYMMETRIC if rt.symmetric else 0)
              | (_lib.TWOOPT_BYTES if rt.twoopt_bytes else 0))
        tb = getattr(timer, "before_twoopt", None) if timer is not None else None
        if tb is not None:
            tb(stream)
        _lib.call("qsb_twoopt", cs, rt.inst, passes, tf, stream)
        if tb is not None:
            timer.after_twoopt(stream)
        state.launches += 1
    # the best update also draws iteration t + 1's coefficients
    _best_update(cs, rt, stream)
    state.coef_ready = _coef_key(config, t + 1)
    state.launches += 2 if ready else 3      # [draw pre-pass +] fused step + best update
    state.v_bound = _post_step_v_bound(coeffs)
    state.cost_current = True     # cost[p] is now the goal of the new position
    state.swap_positions()
    state._host_best = None
    if config.migration_factor > 0.0 and t % config.migration_period == 0:
        if config.migration_depth > 0:
            _migrate_device(state, config, t, exchange)
            state.launches += 1 if exchange is None else 2
    state.t = t
    return state


def _due_epochs(config: SolverConfig, t0: int, t1: int) -> int:
    """Migration events in iterations t0+1 .. t1."""
    if config.migration_factor <= 0.0 or config.migration_depth <= 0:
        return 0
    P = config.migration_period
    return t1 // P - t0 // P


def _graph_span(config: SolverConfig) -> int:
    """Iterations held by one captured graph: even (perm / perm_new return
    to their buffers) and a multiple of the migration period, so a graph
    that starts at t % span == 0 has its migration launches at fixed slots.
    Without migration any even t works, and 8 steps per replay keep a small
    population's device time ahead of the host's graph launches."""
    if config.migration_factor <= 0.0 or config.migration_depth <= 0:
        return 8
    return math.lcm(2, config.migration_period)


def step_many(state: PopulationState, instance, config: SolverConfig, steps: int,
              exchange=None) -> PopulationState:
    """Advance ``steps`` iterations by replaying a CUDA graph of
    :func:`_graph_span` iterations, with the migration launches (and, for
    sharded states, the ``exchange`` collectives) captured at their slots.
    Results are identical to calling :func:`step` ``steps`` times; the host
    only launches the graph.  Steps before the first aligned iteration and
    after the last whole graph run eagerly."""
    if steps <= 0:
        return state
    sharded = state.local_particles != state.num_particles
    if sharded and exchange is None and _due_epochs(config, state.t, state.t + steps):
        raise ValueError("a sharded state with migration needs the cross-device exchange")
    span = _graph_span(config)
    # eager steps up to an aligned start (the first one also settles the
    # launch hints: velocity bound and current costs)
    align = span if _due_epochs(config, 0, span) else 2
    while steps > 0 and (state.t == 0 or state.t % align != 0 or not state.cost_current
                         or state.coef_ready != _coef_key(config, state.t + 1)):
        step(state, instance, config, exchange=exchange)
        steps -= 1
    reps = steps // span
    if reps >= 1:
        rt = _runtime(state, instance, config)
        coeffs = config.coefficients
        # valid for every later step (post-S_v bound; each step's best update
        # draws the next step's coefficients)
        base = (_hints(state, rt, coeffs) & ~_lib.HINT_LATE) | (_lib.HINT_COEF_READY if _COEF_FOLD else 0)
        d = config.migration_depth if config.migration_factor > 0.0 else 0
        graphs = getattr(state, "_graph_cache", None)
        if not isinstance(graphs, dict):
            graphs = {}
        if d > 0:
            if state._mig is None or state._mig.d != d:
                _drain_log(state)
                state._mig = _MigrationScratch(state, d)
            # room in the device log for every epoch of this call
            need = state._mig.pending + _due_epochs(config, state.t, state.t + reps * span)
            if need > state._mig.log.shape[0]:
                _drain_log(state)
                need = _due_epochs(config, state.t, state.t + reps * span)
                if need > state._mig.log.shape[0]:
                    state._mig = _MigrationScratch(state, d, log_rows=need)
        if graphs.get("_mig", state._mig) is not state._mig or len(graphs) > 8:
            graphs = {}          # the captured migration scratch changed
        graphs["_mig"] = state._mig
        state._graph_cache = graphs

        def graph_for(hints):
            # rt: the runtime object itself (its device instance is captured)
            key = (rt, hints, config, state.d_perm.data_ptr(), state.d_perm_new.data_ptr(), exchange)
            hit = graphs.get(key)
            if hit is not None:
                return hit[0]
            rt.coeffs.hints = hints
            passes = config.two_opt_passes
            flags = _lib.PHASE_ALL if not passes else _lib.PHASE_ALL & ~_lib.PHASE_PBEST
            tf = (_lib.TWOOPT_PBEST | (_lib.TWOOPT_SYMMETRIC if rt.symmetric else 0)
                  | (_lib.TWOOPT_BYTES if rt.twoopt_bytes else 0))
            cs_a = state.c_state()
            cs_b = _lib.QsbState.from_buffer_copy(cs_a)
            cs_b.perm, cs_b.perm_new = cs_a.perm_new, cs_a.perm
            mig = state._mig.struct(state, config) if d > 0 else None
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(state.device)
            side.wait_stream(torch.cuda.current_stream(state.device))
            with torch.cuda.stream(side):
                with torch.cuda.graph(graph, stream=side):
                    s = side.cuda_stream
                    for i in range(span):
                        cs = cs_a if i % 2 == 0 else cs_b
                        _lib.call("qsb_step_phases", cs, rt.inst, rt.coeffs, flags, None, 0, 2,
                                  None, 0, s)
                        if passes:
                            _lib.call("qsb_twoopt", cs, rt.inst, passes, tf, s)
                        _best_update(cs, rt, s)
                        if mig is not None and (i + 1) % config.migration_period == 0:
                            mst = _lib.QsbState.from_buffer_copy(cs)
                            mst.perm = cs.perm_new           # migration reads the post-swap positions
                            if exchange is None:
                                _lib.call("qsb_migrate", mst, mig, s)
                            else:
                                exchange(state, mig, cstate=mst)
            torch.cuda.current_stream(state.device).wait_stream(side)
            graphs[key] = (graph, mig)
            return graph

        # the late-iteration kernel variant (QSB_HINT_LATE, performance only)
        # is picked per replay: both graphs are captured once and cached
        for r in range(reps):
            late = state.t + r * span + 1 >= _CHAIN_T0
            graph_for(base | (_lib.HINT_LATE if late else 0)).replay()
        passes = config.two_opt_passes
        epochs = _due_epochs(config, state.t, state.t + reps * span)
        state.launches += reps * span * (2 + (0 if _COEF_FOLD else 1) + (1 if passes else 0)) \
            + epochs * (1 if exchange is None else 2)
        state.t += reps * span
        state.coef_ready = _coef_key(config, state.t + 1)
        if state._mig is not None and getattr(exchange, "logs_events", True):
            state._mig.pending += epochs
        state.v_bound = _post_step_v_bound(coeffs)
        state._host_best = None
        steps -= reps * span
    for _ in range(steps):
        step(state, instance, config, exchange=exchange)
    return state


@dataclass
class RunResult:
    """Outcome of a full run plus the collected statistics (engine.py:247-265)."""

    instance_name: str
    best_perm: np.ndarray
    best_cost: float
    best_iteration: int
    gap: float | None
    iterations_run: int
    stats: list[IterationStats]
    total_seconds: float
    migration_events: list[MigrationEvent] = field(default_factory=list)

    @property
    def mean_ms_per_iteration(self) -> float:
        if self.iterations_run == 0:
            return 0.0
        return 1000.0 * self.total_seconds / self.iterations_run


def run(config: SolverConfig, instance, collect_stats: bool = True, device=None) -> RunResult:
    """Iterate until ``max_iterations`` or until the best reaches
    ``target_cost`` (engine.py:268-307).  Statistics at iteration 0 and
    every ``stats_stride``-th iteration."""
    t_start = time.perf_counter()
    state = init_population(config, instance, device)
    series: list[IterationStats] = []
    if collect_stats:
        series.append(collect_device(state, 1000.0 * (time.perf_counter() - t_start),
                                     bins=config.pmf_bins,
                                     all_swarms=config.record_all_swarm_percentiles))
    if not collect_stats and config.target_cost is None:
        # nothing is read back per iteration: replay CUDA graphs
        step_many(state, instance, config, config.max_iterations)
    for _ in range(config.max_iterations if (collect_stats or config.target_cost is not None) else 0):
        if config.target_cost is not None and state.best_cost <= config.target_cost:
            break
        it_start = time.perf_counter()
        step(state, instance, config)
        if collect_stats and state.t % config.stats_stride == 0:
            torch.cuda.current_stream(state.device).synchronize()
            elapsed_ms = 1000.0 * (time.perf_counter() - it_start)
            series.append(collect_device(state, elapsed_ms, bins=config.pmf_bins,
                                         all_swarms=config.record_all_swarm_percentiles))
    torch.cuda.current_stream(state.device).synchronize()
    total = time.perf_counter() - t_start
    _drain_log(state)
    g = None
    known = getattr(instance, "known_best", None)
    if known is not None and known > 0:
        g = gap(state.best_cost, known)
    return RunResult(instance_name=getattr(instance, "name", ""), best_perm=state.best_perm.copy(),
                     best_cost=state.best_cost, best_iteration=state.best_iteration, gap=g,
                     iterations_run=state.t, stats=series, total_seconds=total,
                     migration_events=list(state.migration_log))
