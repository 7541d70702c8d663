"""qapswarm-b200: B200-native multi-swarm PSO for the Quadratic Assignment
Problem (arXiv 1504.05158), drop-in for the reference package's solver API.

The public names mirror ``qapswarm/__init__.py``: configs, population
state, ``init_population`` / ``step`` / ``run``, migration and statistics.
The per-iteration work runs in hand-written sm_100a kernels (libqsb.so,
C ABI in include/qapswarm_b200.h); there is no CPU fallback.
"""

from .config import PsoCoefficients, SolverConfig, SV_MODES, SX_MODES
from .instance import (
    QapInstance,
    ReferenceSolution,
    parse_instance,
    parse_reference_solution,
    format_instance,
    format_reference_solution,
    load_instance,
    load_reference_solution,
    taillard_uniform,
    grey_pattern,
)
from .core import Assignment, evaluate_cost, matrix_to_assignment
from .migration import SwarmBestTable, MigrationEvent, migrate
from .stats import IterationStats, percentile, pmf, collect, export_csv, write_solution
from .engine import (
    PopulationState,
    RunResult,
    init_population,
    step,
    step_many,
    run,
    projected_buffer_bytes,
    device_buffer_bytes,
    gap,
    collect_device,
)
from .datasets import data_path, list_bundled, load_bundled, load_bundled_solution
from . import batch

__version__ = "0.1.0"

__all__ = [
    "PsoCoefficients", "SolverConfig", "SV_MODES", "SX_MODES",
    "QapInstance", "ReferenceSolution", "parse_instance", "parse_reference_solution",
    "format_instance", "format_reference_solution", "load_instance", "load_reference_solution",
    "taillard_uniform", "grey_pattern",
    "Assignment", "evaluate_cost", "matrix_to_assignment",
    "SwarmBestTable", "MigrationEvent", "migrate",
    "IterationStats", "percentile", "pmf", "collect", "export_csv", "write_solution",
    "PopulationState", "RunResult", "init_population", "step", "step_many", "run",
    "projected_buffer_bytes", "device_buffer_bytes", "gap", "batch", "collect_device",
    "data_path", "list_bundled", "load_bundled", "load_bundled_solution",
]
