"""ctypes binding of libqsb.so (the C ABI declared in include/qapswarm_b200.h).

The shared library is built in-tree (``python -m paper_1504_05158_b200.build``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or a call fails, an exception is raised.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("QSB_LIB", PKG / "libqsb.so"))
HEADER = PKG.parent / "include" / "qapswarm_b200.h"

QSB_OK, QSB_EINVAL, QSB_EUNSUPPORTED, QSB_ECUDA, QSB_EPERM = 0, 1, 2, 3, 4
F32, F64, I64, U16 = 1, 2, 3, 4
PHASE_VELOCITY, PHASE_AGGREGATE, PHASE_COST, PHASE_PBEST, PHASE_STORE_V = 1, 2, 4, 8, 16
HINT_V_BOUNDED = 1
HINT_COST_CURRENT = 2
HINT_SYMMETRIC = 4
HINT_COEF_READY = 8
HINT_LATE = 16
TWOOPT_PBEST, TWOOPT_SYMMETRIC = 1, 2
TWOOPT_BYTES = 4
PHASE_ALL = PHASE_VELOCITY | PHASE_AGGREGATE | PHASE_COST | PHASE_PBEST | PHASE_STORE_V

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double


class QsbState(ctypes.Structure):
    _fields_ = [
        ("n", _i32), ("vstride", _i32), ("v_dtype", _i32), ("cost_dtype", _i32),
        ("num_particles", _i64), ("swarm_size", _i64), ("num_swarms", _i64),
        ("particle_offset", _i64), ("swarm_offset", _i64),
        ("V", _vp), ("perm", _vp), ("perm_new", _vp), ("pl_perm", _vp),
        ("cost", _vp), ("pl_cost", _vp), ("improved", _vp),
        ("pg_perm", _vp), ("pg_cost", _vp),
        ("best_perm", _vp), ("best_cost", _vp), ("best_iter", _vp), ("best_idx", _vp),
        ("iteration", _vp), ("swarm_min", _vp), ("swarm_min_idx", _vp), ("done", _vp),
        ("work", _vp), ("vcol", _vp), ("step_coef", _vp),
    ]


class QsbInstance(ctypes.Structure):
    _fields_ = [("n", _i32), ("mat_dtype", _i32), ("flow", _vp), ("distance", _vp),
                ("acc32", _i32), ("reserved", _i32)]


class QsbCoeffs(ctypes.Structure):
    _fields_ = [("c1", _dbl), ("c2", _dbl), ("c3", _dbl), ("v_max", _dbl),
                ("normalize", _i32), ("sx_mode", _i32), ("depth", _i32), ("hints", _i32),
                ("seed", _u64)]


class QsbMigration(ctypes.Structure):
    _fields_ = [("d", _i32), ("period", _i32), ("mode", _i32), ("reserved", _i32),
                ("num_swarms_total", _i64), ("picks", _vp), ("picks_epoch0", _i64),
                ("picks_rows", _i64), ("all_pg_cost", _vp), ("plan", _vp), ("records", _vp),
                ("log", _vp), ("log_rows", _i64), ("log_count", _vp), ("status", _vp),
                ("seed", _u64)]


class QsbHostPopulation(ctypes.Structure):
    _fields_ = [("n", _i32), ("cost_dtype", _i32), ("num_particles", _i64), ("swarm_size", _i64),
                ("num_swarms", _i64), ("V", _vp), ("X_new", _vp), ("PL", _vp), ("perms", _vp),
                ("perms_new", _vp), ("pl_perms", _vp), ("cost", _vp), ("pl_cost", _vp),
                ("improved", _vp), ("pg_mats", _vp), ("pg_perms", _vp), ("pg_costs", _vp),
                ("best_perm", _vp), ("best_cost", _vp), ("best_iteration", _vp)]


class QsbHostInstance(ctypes.Structure):
    _fields_ = [("n", _i32), ("mat_dtype", _i32), ("flow", _vp), ("distance", _vp)]


# name -> (restype, argtypes); every symbol of include/qapswarm_b200.h
SIGNATURES = {
    "qsb_version": (ctypes.c_int, []),
    "qsb_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "qsb_last_cuda_error": (ctypes.c_int, []),
    "qsb_supported": (ctypes.c_int, [_i32, _i32, _i32]),
    "qsb_stream_gate": (ctypes.c_int, [_vp, ctypes.c_int64, _vp, _vp]),
    "qsb_vstride": (_i32, [_i32, _i32]),
    "qsb_step_phases": (ctypes.c_int, [ctypes.POINTER(QsbState), ctypes.POINTER(QsbInstance),
                                       ctypes.POINTER(QsbCoeffs), _i32, _vp, _i64, _i32, _vp,
                                       _u64, _vp]),
    "qsb_best_update": (ctypes.c_int, [ctypes.POINTER(QsbState), _vp]),
    "qsb_best_update_next": (ctypes.c_int, [ctypes.POINTER(QsbState), ctypes.POINTER(QsbCoeffs), _vp]),
    "qsb_step": (ctypes.c_int, [ctypes.POINTER(QsbState), ctypes.POINTER(QsbInstance),
                                ctypes.POINTER(QsbCoeffs), _vp]),
    "qsb_migrate": (ctypes.c_int, [ctypes.POINTER(QsbState), ctypes.POINTER(QsbMigration), _vp]),
    "qsb_cost": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(QsbInstance), _vp, _vp]),
    "qsb_twoopt": (ctypes.c_int, [ctypes.POINTER(QsbState), ctypes.POINTER(QsbInstance), _i32,
                                  _i32, _vp]),
    "qsb_twoopt_many": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i32]),
    "qsb_step_draws": (ctypes.c_int, [_u64, _u64, _i64, _i64, _i32, _vp, _vp]),
    "qsb_migration_picks": (ctypes.c_int, [_u64, _u64, _i32, _i64, _vp, _vp]),
    "qsb_stats_work_bytes": (ctypes.c_size_t, []),
    "qsb_population_stats": (ctypes.c_int, [_vp, _i32, _i64, _dbl, _dbl, _i32, _vp, _i32, _vp,
                                            _vp, _vp, _vp]),
    "qsb_init_population_device": (ctypes.c_int, [ctypes.POINTER(QsbState), _u64, _dbl, _vp]),
    "qsb_perm_to_matrix": (ctypes.c_int, [_vp, _i64, _i32, _vp, _vp]),
    "qsb_velocity_many": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i32, _i64, _dbl, _vp, _vp,
                                         _dbl, _i32]),
    "qsb_aggregate_many": (ctypes.c_int, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i64, _vp,
                                          _vp]),
    "qsb_cost_many_i64": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i32]),
    "qsb_cost_many_f64": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i32]),
    "qsb_step_draws_host": (ctypes.c_int, [_u64, _u64, _i64, _i32, _vp]),
    "qsb_step_host": (ctypes.c_int, [ctypes.POINTER(QsbHostPopulation),
                                     ctypes.POINTER(QsbHostInstance), ctypes.POINTER(QsbCoeffs),
                                     _u64, _i32, _vp]),
}

_lib = None


class QsbError(RuntimeError):
    """A libqsb call returned an error status."""

    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} failed: {msg} (status {code})")
        self.code = code


def build(verbose: bool = False) -> Path:
    """Compile libqsb.so for sm_100a with nvcc (csrc/Makefile)."""
    cmd = ["make", "-C", str(PKG / "csrc")]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"libqsb build failed:\n{out.stdout}\n{out.stderr}")
    return LIB_PATH


def lib():
    """Load libqsb.so.  Raises if it has not been built: no CPU fallback."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(fn: str, code: int):
    if code != QSB_OK:
        msg = lib().qsb_strerror(code).decode()
        raise QsbError(fn, code, msg)


def call(fn: str, *args):
    check(fn, getattr(lib(), fn)(*args))
