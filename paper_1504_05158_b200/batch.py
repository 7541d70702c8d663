"""Reference-layout, host-buffer drop-ins for ``qapswarm._batch`` and
``qapswarm.streams.step_draws``.

Same signatures, layouts and in-place semantics as _batch.py:30-197 and
streams.py:53-64; each call goes through the tier-1 C ABI
(include/qapswarm_b200.h), which copies to the device, runs the sm_100a
kernels and copies back.  The velocity and aggregation entry points require
x / pl / pg to be permutation matrices (the only inputs the engine
produces); anything else raises ValueError.
"""

from __future__ import annotations

import numpy as np

from . import _lib

MODE_GLOBAL_MAX = 0
MODE_PICK_COLUMN = 1
MODE_SECOND_TARGET = 2
MODE_CODES = {"global-max": MODE_GLOBAL_MAX, "pick-column": MODE_PICK_COLUMN,
              "second-target": MODE_SECOND_TARGET}


def _c(a, dtype):
    a = np.asarray(a)
    if a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"expected a C-contiguous {np.dtype(dtype)} array, got {a.dtype}")
    return a


def _call(fn, *args):
    code = getattr(_lib.lib(), fn)(*args)
    if code == _lib.QSB_EPERM:
        raise ValueError(f"{fn}: input is not a permutation matrix")
    _lib.check(fn, code)


def velocity_many(v, x, pl, pg, swarm_size, c1, c2r2, c3r3, v_max, normalize):
    """_batch.velocity_many (_batch.py:30-58): in place on v (P, n, n) f64."""
    v = _c(v, np.float64)
    P, n = v.shape[0], v.shape[1]
    x, pl, pg = (_c(a, np.int8) for a in (x, pl, pg))
    c2r2 = np.ascontiguousarray(np.broadcast_to(c2r2, (P,)), dtype=np.float64)
    c3r3 = np.ascontiguousarray(np.broadcast_to(c3r3, (P,)), dtype=np.float64)
    _call("qsb_velocity_many", v.ctypes.data, x.ctypes.data, pl.ctypes.data, pg.ctypes.data, P,
          n, int(swarm_size), float(c1), c2r2.ctypes.data, c3r3.ctypes.data, float(v_max),
          int(bool(normalize)))


def aggregate_many(x, v, mode, depth, draws, out_mat, out_perm):
    """_batch.aggregate_many (_batch.py:178-183); draws (P, >=2n) rows."""
    x = _c(x, np.int8)
    v = _c(v, np.float64)
    P, n = x.shape[0], x.shape[1]
    draws = np.asarray(draws, dtype=np.float64)
    if draws.ndim != 2 or draws.strides[1] != 8:
        draws = np.ascontiguousarray(draws)
    out_mat = _c(out_mat, np.int8)
    out_perm = _c(out_perm, np.int64)
    if isinstance(mode, str):
        mode = MODE_CODES[mode]
    _call("qsb_aggregate_many", x.ctypes.data, v.ctypes.data, P, n, int(mode), int(depth),
          draws.ctypes.data, draws.strides[0] // 8, out_mat.ctypes.data, out_perm.ctypes.data)


def cost_many(perms, flow, distance, out):
    """_batch.cost_many (_batch.py:186-197)."""
    perms = np.ascontiguousarray(perms, dtype=np.int64)
    P, n = perms.shape
    if out.dtype == np.int64:
        f = np.ascontiguousarray(flow, dtype=np.int64)
        d = np.ascontiguousarray(distance, dtype=np.int64)
        _call("qsb_cost_many_i64", perms.ctypes.data, f.ctypes.data, d.ctypes.data,
              out.ctypes.data, P, n)
    else:
        f = np.ascontiguousarray(flow, dtype=np.float64)
        d = np.ascontiguousarray(distance, dtype=np.float64)
        _call("qsb_cost_many_f64", perms.ctypes.data, f.ctypes.data, d.ctypes.data,
              out.ctypes.data, P, n)


def step_draws(seed: int, iteration: int, num_particles: int, n: int) -> np.ndarray:
    """streams.step_draws (streams.py:53-64), computed on the device."""
    if num_particles >= 1 << 24:
        raise ValueError(f"population {num_particles} exceeds supported size")
    if not 0 <= iteration < 1 << 32:
        raise ValueError(f"iteration {iteration} outside supported range")
    out = np.empty((num_particles, 2 + 2 * n), dtype=np.float64)
    _call("qsb_step_draws_host", int(seed) & (2**64 - 1), int(iteration), int(num_particles),
          int(n), out.ctypes.data)
    return out


def twoopt_many(perms, flow, distance, costs, passes):
    """2-opt extension (no reference symbol): in place on int64 perms (P, n)
    and int64 costs (P,); integral instances only."""
    perms = _c(perms, np.int64)
    costs = _c(costs, np.int64)
    P, n = perms.shape
    f = np.ascontiguousarray(flow, dtype=np.int64)
    d = np.ascontiguousarray(distance, dtype=np.int64)
    _call("qsb_twoopt_many", perms.ctypes.data, f.ctypes.data, d.ctypes.data, costs.ctypes.data,
          P, n, int(passes))
