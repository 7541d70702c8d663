"""Run configuration: the reference's PsoCoefficients and SolverConfig.

Field names, defaults and ValueError messages follow the reference
(kernels.py:47-76 and engine.py:29-68) so existing configs and tests carry
over unchanged.  SolverConfig adds optional fields whose defaults preserve
reference behaviour:

* ``migration_period`` -- migrate only when ``t % migration_period == 0``
  (1 = every iteration, the reference; the north-star runs use 10);
* ``precision`` -- ``"fp64"`` keeps the velocity state in float64 and is
  bit-identical to the reference; ``"fp32"`` is the throughput mode;
* ``two_opt_passes`` -- after S_x, apply up to this many best-improvement
  pairwise-exchange moves per particle (0 = off, the reference; the
  north-star's 2-opt local search, integral instances only);
* ``init`` -- ``"reference"`` draws the initial population from the
  reference's numpy init stream on the host (bit-identical); ``"device"``
  draws it on the GPU from a documented Philox stream (not the reference's).
"""

from __future__ import annotations

from dataclasses import dataclass, field

SV_MODES = ("raw", "norm")
SX_MODES = ("global-max", "pick-column", "second-target")
SX_CODES = {"global-max": 0, "pick-column": 1, "second-target": 2}
PRECISIONS = ("fp64", "fp32")
INITS = ("reference", "device")


@dataclass(frozen=True)
class PsoCoefficients:
    """c1 weighs the inertia, c2 the pull to the personal best, c3 the pull
    to the swarm best; sv_mode shapes the velocity, sx_mode aggregates
    X + V into the next permutation (kernels.py:47-76)."""

    c1: float = 0.5
    c2: float = 0.5
    c3: float = 0.5
    v_max: float = 4.0
    sv_mode: str = "norm"
    sx_mode: str = "second-target"
    depth: int = 2

    def __post_init__(self):
        for label, c in (("c1", self.c1), ("c2", self.c2), ("c3", self.c3)):
            if not 0.0 <= c <= 1.0:
                raise ValueError(f"{label} must be in [0, 1], got {c}")
        if self.v_max <= 0:
            raise ValueError(f"v_max must be positive, got {self.v_max}")
        if self.sv_mode not in SV_MODES:
            raise ValueError(f"sv_mode must be one of {SV_MODES}, got {self.sv_mode!r}")
        if self.sx_mode not in SX_MODES:
            raise ValueError(f"sx_mode must be one of {SX_MODES}, got {self.sx_mode!r}")
        if self.depth < 1:
            raise ValueError(f"depth must be >= 1, got {self.depth}")


@dataclass(frozen=True)
class SolverConfig:
    """A complete, reproducible run description (engine.py:29-68)."""

    swarms: int
    swarm_size: int
    coefficients: PsoCoefficients = field(default_factory=PsoCoefficients)
    migration_factor: float = 0.0
    max_iterations: int = 200
    target_cost: float | None = None
    seed: int = 0
    workers: int = 1
    stats_stride: int = 1
    pmf_bins: int = 60
    record_all_swarm_percentiles: bool = False
    init_velocity_amplitude: float = 1.0
    # ---- extensions (defaults = reference behaviour)
    migration_period: int = 1
    precision: str = "fp64"
    init: str = "reference"
    two_opt_passes: int = 0

    def __post_init__(self):
        if self.swarms < 1 or self.swarm_size < 1:
            raise ValueError("swarms and swarm_size must be positive")
        if not 0.0 <= self.migration_factor < 0.5:
            raise ValueError(
                f"migration_factor must be in [0, 0.5), got {self.migration_factor}")
        if self.max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        if self.workers < 1:
            raise ValueError("workers must be positive")
        if self.stats_stride < 1 or self.pmf_bins < 1:
            raise ValueError("stats_stride and pmf_bins must be positive")
        if self.init_velocity_amplitude <= 0:
            raise ValueError("init_velocity_amplitude must be positive")
        if self.migration_period < 1:
            raise ValueError("migration_period must be positive")
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}, got {self.precision!r}")
        if self.two_opt_passes < 0:
            raise ValueError("two_opt_passes must be non-negative")
        if self.init not in INITS:
            raise ValueError(f"init must be one of {INITS}, got {self.init!r}")

    @property
    def num_particles(self) -> int:
        return self.swarms * self.swarm_size

    @property
    def migration_depth(self) -> int:
        return int(self.migration_factor * self.swarms)
