"""Swarm sharding across the GPUs of one node (one process per GPU).

Each rank owns a contiguous block of swarms, hence a contiguous range of
GLOBAL particle ids; the in-kernel random streams are keyed by global ids,
so any world size reproduces the single-device trajectory bit for bit.

The data path needs no collective inside an iteration.  Cross-rank traffic
happens only at:

* migration epochs (migration.py:55-86 semantics, every
  ``migration_period`` iterations): all-gather of the m swarm-best costs
  (m x 8 B), every rank ranks them identically on the device and packs the
  donor records it owns, one all-reduce(sum) of the d x (n+1) record buffer
  (28.6 KB at n=50, d=264), then each rank applies the records of the
  swarms it owns;
* the global best (engine.py:225-229): an all-gather of each rank's
  (cost, first iteration, global particle id, permutation) record and a
  lexicographic minimum, which reproduces the reference's strict-< /
  first-index rule because ranks own ascending id ranges.

The collective sequence is written against ``torch.distributed`` so the
same code runs over NCCL (GPU tensors) and gloo (CPU tensors, used by the
world-size-2 tests with CPU stand-ins for the pack/apply kernels).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def swarm_range(swarms: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block of swarms owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    if swarms < world:
        raise ValueError(f"cannot shard {swarms} swarms over {world} ranks")
    base, extra = divmod(swarms, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_swarm_costs(local: torch.Tensor, swarms: int, world: int, group=None) -> torch.Tensor:
    """All-gather the per-rank swarm-best cost blocks into global order."""
    if world == 1:
        return local
    sizes = [swarm_range(swarms, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[:local.numel()] = local
    out = torch.empty(world * width, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return torch.cat([out[r * width: r * width + (hi - lo)] for r, (lo, hi) in enumerate(sizes)])


def exchange_records(records: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the donor-record buffers: each donor row is non-zero on exactly
    one rank (its owner), so the sum is the full record set."""
    dist.all_reduce(records, op=dist.ReduceOp.SUM, group=group)
    return records


def make_exchange(world: int, group=None):
    """Cross-device migration hook for ``engine.step(..., exchange=...)``."""
    from . import _lib

    def exchange(state, mig, cstate=None):
        """``cstate``: the C state to migrate on (post-swap positions); the
        state's current one by default.  CUDA-graph capture (engine.step_many)
        passes the captured slot's state; the collectives are then captured
        too, which needs NCCL (gloo runs eagerly only)."""
        cs = cstate if cstate is not None else state.c_state()
        full = gather_swarm_costs(state.d_pg_cost, state.swarms, world, group)
        mig.all_pg_cost = full.data_ptr()
        stream = torch.cuda.current_stream(state.device).cuda_stream
        mig.mode = 1
        _lib.call("qsb_migrate", cs, mig, stream)
        exchange_records(state._mig.records, group)
        mig.mode = 2
        _lib.call("qsb_migrate", cs, mig, stream)
        state._keep_alive = full

    return exchange


_RING_SEED_STRIDE = 0x9E3779B97F4A7C15   # golden-ratio odd constant: rank r's picks key


def ring_depth(config, world: int) -> int:
    """Donors every rank sends per ring epoch: int(f * floor(m / world)),
    the reference's depth rule (engine.py:66-68) over the smallest shard, so
    every rank sends and receives the same number of records."""
    return int(config.migration_factor * (config.swarms // world))


def make_ring_exchange(world: int, rank: int, config, group=None):
    """Ring migration (north_star: "ring-exchanges best particles"; SURVEY
    §8(e) optional mode, NOT the reference's semantics).

    At every migration epoch rank g ranks its OWN swarms by swarm-best cost
    (stable, as migration.py:64), picks a random current particle of each of
    its d_g = int(f * m_g) best swarms (the reference's donor rule,
    migration.py:74-80, with the picks stream keyed by (seed + g * c, t)),
    sends those d records to rank g+1 and writes the d records it
    receives from rank g-1 into its own d worst swarm bests (k-th best
    donor -> k-th worst swarm, worse values accepted as in the reference).
    Only the donor records (d x (n + 1) int64) cross the ring: one NCCL
    send/recv pair per epoch instead of the all-gather + all-reduce of the
    rank-based scheme.  With world == 1 the ring closes on the rank itself
    and the epoch is exactly the reference migration (same seed, same d).

    The donor kernel is qsb_migrate on a rank-local view of the state
    (swarm offset 0, m = m_local): mode 1 plans and packs, the records move
    over the ring, mode 2 applies them to the planned destinations.  No
    MigrationEvent rows are logged in this mode."""
    from . import _lib

    nxt, prv = (rank + 1) % world, (rank - 1) % world

    def exchange(state, mig, cstate=None):
        cs = cstate if cstate is not None else state.c_state()
        local = _lib.QsbState.from_buffer_copy(cs)
        local.swarm_offset = 0
        d = ring_depth(config, world)
        if d == 0:
            return
        m = _lib.QsbMigration.from_buffer_copy(mig)
        m.d = d
        m.num_swarms_total = state.local_swarms
        m.all_pg_cost = state.d_pg_cost.data_ptr()
        m.log, m.log_rows, m.log_count = None, 0, None
        m.seed = (int(config.seed) + rank * _RING_SEED_STRIDE) & (2**64 - 1)
        stream = torch.cuda.current_stream(state.device).cuda_stream
        if world == 1:
            m.mode = 0
            _lib.call("qsb_migrate", local, m, stream)
            return
        rec = state._mig.records[:d]
        m.mode = 1
        _lib.call("qsb_migrate", local, m, stream)
        send_recv_ring(rec, nxt, prv, group)
        m.mode = 2
        _lib.call("qsb_migrate", local, m, stream)

    exchange.logs_events = False
    return exchange


def send_recv_ring(buf: torch.Tensor, nxt: int, prv: int, group=None) -> torch.Tensor:
    """Send ``buf`` to rank ``nxt`` and overwrite it with ``prv``'s buffer
    (every rank sends the same d rows).  NCCL moves device tensors directly (capturable in a CUDA
    graph); gloo, which has no device point-to-point, goes through host
    copies."""
    on_dev = buf.device.type == "cuda" and dist.get_backend(group) == "nccl"
    out = buf if on_dev else buf.cpu()
    inc = torch.empty_like(out)
    reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, out.contiguous(), nxt, group),
                                   dist.P2POp(dist.irecv, inc, prv, group)])
    for r in reqs:
        r.wait()
    buf.copy_(inc)
    return buf


@dataclass
class BestRecord:
    cost: float
    iteration: int
    index: int
    perm: np.ndarray


def merge_best(cost, iteration: int, index: int, perm, world: int, device, group=None,
               integral: bool = True) -> BestRecord:
    """Global best over ranks: lexicographic min of (cost, iteration, index)."""
    n = len(perm)
    rec = torch.zeros(4 + n, dtype=torch.float64 if not integral else torch.int64, device=device)
    rec[0] = cost
    rec[1] = iteration
    rec[2] = index
    rec[4:] = torch.as_tensor(np.asarray(perm), dtype=rec.dtype)
    if world > 1:
        out = torch.empty(world * (4 + n), dtype=rec.dtype, device=device)
        dist.all_gather_into_tensor(out, rec, group=group)
        rows = out.view(world, 4 + n).cpu().numpy()
    else:
        rows = rec.view(1, 4 + n).cpu().numpy()
    best = min(range(rows.shape[0]), key=lambda r: (rows[r, 0], rows[r, 1], rows[r, 2]))
    r = rows[best]
    c = r[0].item()
    return BestRecord(int(c) if integral else float(c), int(r[1]), int(r[2]),
                      r[4:].astype(np.int64))
