"""Benchmark of the fused PSO step (BASELINE.json north-star workload).

Workload (BASELINE.json configs[2]): synthetic Taillard-style QAP n=50,
800 swarms x 100 particles (80k particles), c = (0.8, 0.5, 0.5), v_max 4,
sv = norm, sx = second-target depth 2, migration factor 0.33 every 10
iterations, seed 1, fp32 velocity state (the north-star throughput mode).
A "step" is one PSO iteration over every particle.  Strong scaling: the 80k
particles are split by swarms across the N ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Rank 0 prints one JSON line.  ``--impl reference`` times the CPU restatement
of the reference's hot path (oracle/, kind "port") on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-iterations/sec (QAP n=50, 80k particles)"   # the headline (config3)
UNIT = "particle-iterations/s"
N_DEFAULT, SWARMS, SWARM_SIZE = 50, 800, 100
PERIOD, FACTOR, SEED = 10, 0.33, 1
L2_BYTES = 126 << 20     # B200 L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--swarms", type=int, default=SWARMS)
    ap.add_argument("--swarm-size", type=int, default=SWARM_SIZE)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--e2e-steps", type=int, default=-1,
                    help="steps of the end-to-end (public API) measurement; default = --steps, "
                         "run on a fresh population over the same iterations as the device-timed "
                         "window (0 = skip)")
    ap.add_argument("--host-steps", type=int, default=20,
                    help="steps of the host-buffer end-to-end leg (qsb_step_host); 0 = skip")
    ap.add_argument("--fp64-steps", type=int, default=20,
                    help="steps of the fp64 parity-mode throughput window (value_fp64); 0 = skip")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--velocity-only", action="store_true",
                    help="time only the velocity/normalise phase of the fused kernel")
    ap.add_argument("--preset", default="config3",
                    choices=["config1", "config2", "config3", "config4", "config5"],
                    help="BASELINE.json configs: 1 n=12 1x100; 2 n=30 100x100 2-opt; "
                         "3 n=50 800x100 migration/10 (the headline, default); "
                         "4 n=100 10k; 5 n=256 2k/GPU 2-opt + migration")
    ap.add_argument("--two-opt", type=int, default=None)
    ap.add_argument("--graph", action="store_true",
                    help="time the K steps as CUDA-graph replays (step_many); the roofline "
                         "kernel time then comes from an eager window of the same length after")
    args = ap.parse_args()
    presets = {
        "config1": dict(n=12, swarms=1, swarm_size=100, two_opt=0, factor=0.0),
        "config2": dict(n=30, swarms=100, swarm_size=100, two_opt=1, factor=0.0),
        "config3": dict(n=50, swarms=800, swarm_size=100, two_opt=0, factor=FACTOR),
        "config4": dict(n=100, swarms=100, swarm_size=100, two_opt=0, factor=FACTOR),
        "config5": dict(n=256, swarms=20, swarm_size=100, two_opt=1, factor=FACTOR),
    }
    pr = presets[args.preset]
    if args.preset != "config3":
        args.n, args.swarms, args.swarm_size = pr["n"], pr["swarms"], pr["swarm_size"]
    args.factor = pr["factor"]
    if args.two_opt is None:
        args.two_opt = pr["two_opt"]
    return args


def config(args, swarms=None, precision=None):
    import paper_1504_05158_b200 as qsb
    return qsb.SolverConfig(
        swarms=swarms or args.swarms, swarm_size=args.swarm_size, seed=SEED,
        coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5, v_max=4.0, sv_mode="norm",
                                          sx_mode="second-target", depth=2),
        migration_factor=getattr(args, "factor", FACTOR), migration_period=PERIOD,
        precision=precision or args.precision, init="device",
        two_opt_passes=getattr(args, "two_opt", 0))


def workload(args, n_gpus):
    mig = (f"migration f={args.factor} every {PERIOD} iterations" if args.factor
           else "independent swarms")
    return {"workload": f"synthetic Taillard-style QAP n={args.n}, {args.swarms} swarms x "
                        f"{args.swarm_size} particles, {mig}, sv=norm, sx=second-target(2), "
                        f"c=(0.8,0.5,0.5), 2-opt passes={args.two_opt} ({args.preset})",
            "n": args.n, "particles": args.swarms * args.swarm_size, "swarms": args.swarms,
            "swarm_size": args.swarm_size, "precision": args.precision,
            "parallelism": f"swarm-shard x{n_gpus}",
            "l2": "inputs larger than L2 (velocity state "
                  f"{args.swarms * args.swarm_size * args.n * args.n * (4 if args.precision == 'fp32' else 8) / 1e6:.0f} MB > 126 MB)"}


def bytes_per_particle(n, S, sv, lazy=False, incremental_cost=True):
    """HBM bytes one fused step has to move per particle-iteration (the
    ``moved_bytes`` beside the roofline; the roofline itself uses SURVEY
    §8(d)'s B_vel).

    Stored-v layout (fp64, or fp32 without the column state): V read +
    write (2 n^2 sV).  Lazily scaled fp32 layout: the tile is
    read when it is staged in shared memory (4 n^2; n = 256 keeps it in
    global memory and reads only the <= 3n touched entries), only the
    touched entries are written (12n), and the column state is read and
    written (2 * 20 * ceil4(n)); column rescans are not counted.  Both:
    perm / pl_perm read + perm_new write (6n), swarm best row amortised
    (2n/S), (c2 r2, c3 r3) written by the draw pre-pass and read (32), cost
    read (incremental goal) and written, pl_cost read, improved flag (25)."""
    common = 6 * n + 2 * n / S + 32 + (25 if incremental_cost else 17)
    if lazy:
        vcs = (n + 3) // 4 * 4
        tile = 4 * n * n if 4 * n * n <= 200 * 1024 else 12 * n
        return tile + 12 * n + 40 * vcs + common
    return 2 * n * n * sv + common


# ------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.rows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r for r in self.rows if r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[0]) for r in rows]
        load = [s for s in sm if s > 600] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": int(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# -------------------------------------------------------- kernel timer
class KernelTimer:
    """CUDA events around every fused-kernel launch on its own stream."""

    def __init__(self):
        import torch
        self.torch = torch
        self.pairs = []
        self.active = False

    def before(self, stream):
        # the engine launches on torch's current stream (state.stream())
        if self.active:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record(self.torch.cuda.current_stream())
            self.pairs.append([e, None])

    def after(self, stream):
        if self.active:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record(self.torch.cuda.current_stream())
            self.pairs[-1][1] = e

    def mean_ms(self):
        d = [a.elapsed_time(b) for a, b in self.pairs]
        return sum(d) / len(d) if d else None

    # the 2-opt launch (tensor cores), when the config runs one
    def before_twoopt(self, stream):
        if self.active:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record(self.torch.cuda.current_stream())
            self.pairs2 = getattr(self, "pairs2", [])
            self.pairs2.append([e, None])

    def after_twoopt(self, stream):
        if self.active:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record(self.torch.cuda.current_stream())
            self.pairs2[-1][1] = e

    def mean_twoopt_ms(self):
        d = [a.elapsed_time(b) for a, b in getattr(self, "pairs2", [])]
        return sum(d) / len(d) if d else None


def traffic_from_profile(n, precision, particles, prefix=""):
    """ncu DRAM bytes per launch of the fused kernel, from profiles/ (or None)."""
    p = ROOT / "profiles" / "ncu_step_summary.json"
    if not p.exists():
        return None
    try:
        rec = json.loads(p.read_text())
        key = f"{prefix}n{n}_{precision}_P{particles}"
        return rec.get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------- CPU baseline
def cpu_sample(args, seconds, swarms=8, steps_cap=1000, warm=1):
    """The CPU restatement (oracle/, all host threads) on a bounded sample."""
    import numpy as np
    from oracle import oracle as orc
    import paper_1504_05158_b200 as qsb
    inst = qsb.taillard_uniform(args.n)
    cfg = config(args, swarms=swarms, precision="fp64")
    st = orc.init_population(cfg.swarms, cfg.swarm_size, args.n, inst.flow, inst.distance,
                             seed=cfg.seed, amp=cfg.init_velocity_amplitude)
    kw = orc.coeff_kwargs(cfg)
    for _ in range(warm):
        orc.step(st, inst.flow, inst.distance, **kw)
    t0 = time.perf_counter()
    k = 0
    while k < steps_cap and (time.perf_counter() - t0) < seconds:
        orc.step(st, inst.flow, inst.distance, **kw)
        k += 1
    dt = time.perf_counter() - t0
    P = cfg.num_particles
    return {"value": P * k / dt, "unit": UNIT, "cores": orc.num_threads(), "kind": "port",
            "sample": f"oracle/ (C+OpenMP restatement of the reference numba path, fp64, "
                      f"O(n^3) aggregation as in _batch.py) on {cfg.swarms} swarms x "
                      f"{cfg.swarm_size} particles of the same n={args.n} workload, {k} "
                      f"iterations in {dt:.2f} s"}


def run_reference(args, rank, world):
    """The reference arm: the CPU restatement of the reference's step
    (oracle/, C + OpenMP over particles like the numba prange, fp64, the
    O(n^3) aggregation of _batch.py) on the SAME workload -- every particle
    of the config -- with all host threads.  Steps and warm-up are the
    caller's, capped (40 / 5) so a default run stays within minutes."""
    if rank != 0:
        return
    from oracle import oracle as orc
    import paper_1504_05158_b200 as qsb
    inst = qsb.taillard_uniform(args.n)
    cfg = config(args, precision="fp64")
    st = orc.init_population(cfg.swarms, cfg.swarm_size, args.n, inst.flow, inst.distance,
                             seed=cfg.seed, amp=cfg.init_velocity_amplitude)
    kw = orc.coeff_kwargs(cfg)
    steps = min(args.steps, 40)
    warm = min(args.warmup, 5)
    for _ in range(warm):
        orc.step(st, inst.flow, inst.distance, **kw)
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.step(st, inst.flow, inst.distance, **kw)
    dt = time.perf_counter() - t0
    P = cfg.num_particles
    value = P * steps / dt
    wl = workload(args, world)
    wl["precision"] = "fp64"
    wl["init"] = "reference (numpy init stream)"
    line = {"impl": "reference", "metric": METRIC if args.preset == "config3" else
            f"particle-iterations/sec (QAP n={args.n}, {P} particles, {args.preset})",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": 1000 * dt / steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": wl,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": orc.num_threads(),
                             "kind": "port",
                             "sample": f"the full workload: {cfg.swarms} swarms x {cfg.swarm_size} "
                                       f"particles, iterations {warm + 1}-{warm + steps}, fp64 "
                                       "reference arithmetic, all host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- main
def preload_kernels(cfg, inst, dev):
    """Launch every kernel a timed step can launch once, on a throwaway
    16-particle population of the same n / precision / 2-opt setting with
    migration every iteration, so that CUDA's lazy module loading happens
    here and not at the first migration epoch inside a timed window (the
    warmup steps alone never reach t = migration_period)."""
    import dataclasses
    import torch
    import paper_1504_05158_b200 as qsb
    small = dataclasses.replace(cfg, swarms=4, swarm_size=4, migration_period=1,
                                migration_factor=max(cfg.migration_factor, 0.25))
    from paper_1504_05158_b200 import engine
    st = qsb.init_population(small, inst, device=dev)
    for _ in range(3):
        qsb.step(st, inst, small)
    # and the late-iteration variant of the fused kernel (QSB_HINT_LATE)
    saved = engine._CHAIN_T0
    try:
        engine._CHAIN_T0 = 1
        qsb.step(st, inst, small)
    finally:
        engine._CHAIN_T0 = saved
    torch.cuda.synchronize()
    del st


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1504_05158_b200 as qsb
    from paper_1504_05158_b200 import engine, shard

    # functional check of the multi-rank path on a one-GPU box (not a
    # measurement): QSB_BENCH_BACKEND=gloo QSB_BENCH_SAME_DEVICE=1 puts every
    # rank on cuda:0 with host-level collectives (no kernel waits on another
    # rank); the driver's runs use NCCL, one GPU per rank
    backend = os.environ.get("QSB_BENCH_BACKEND", "nccl")
    if os.environ.get("QSB_BENCH_SAME_DEVICE"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    inst = qsb.taillard_uniform(args.n)
    cfg = config(args)
    preload_kernels(cfg, inst, dev)
    lo, hi = shard.swarm_range(cfg.swarms, world, rank)
    state = qsb.init_population(cfg, inst, device=dev, swarm_range=(lo, hi))
    exchange = shard.make_exchange(world) if world > 1 else None
    timer = KernelTimer()
    flags = None
    if args.velocity_only:
        from paper_1504_05158_b200 import _lib
        flags = _lib.PHASE_VELOCITY | _lib.PHASE_STORE_V
        state.set_lazy_scale(False)   # the streaming velocity pass over the stored-v layout

    def one_step():
        if flags is None:
            qsb.step(state, inst, cfg, exchange=exchange, timer=timer)
        else:
            from paper_1504_05158_b200 import _lib
            rt = engine._runtime(state, inst, cfg)
            rt.coeffs.hints &= ~_lib.HINT_COEF_READY   # this leg draws its own coefficients
            s = state.stream()
            timer.before(s)
            _lib.call("qsb_step_phases", state.c_state(), rt.inst, rt.coeffs, flags, None, 0, 2,
                      None, 1, s)
            timer.after(s)
            state.launches += 1

    for _ in range(args.warmup):
        one_step()
    if args.graph and world == 1 and flags is None and cfg.migration_factor == 0.0:
        qsb.step_many(state, inst, cfg, args.steps + (args.steps % 2))   # capture outside the timing
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local) if rank == 0 else None
    if clocks:
        clocks.start()
    stream = torch.cuda.current_stream()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = state.launches
    # no per-kernel events in the timed region: an event recorded between two
    # kernels breaks their programmatic-dependent-launch overlap (about 10 us
    # per step at config 3, scripts/diag_overhead.py); the kernel durations
    # for the roofline come from a second pass below
    timer.active = False
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # inputs smaller than L2: flush it (write a 256 MB buffer) before every
    # timed step and time the steps one by one, outside the flushes
    vbytes = state.local_particles * state.vstride * (4 if cfg.precision == "fp32" else 8)
    use_graph = args.graph and world == 1 and flags is None
    flush_l2 = vbytes < 2 * L2_BYTES and not use_graph
    step_ms = None
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush_l2 else None
    # one GPU: the window's first GATE_STEPS steps are enqueued behind a
    # host-released gate (qsb_stream_gate), so a host stall while they are
    # being launched (scheduler, allocator, the clock sampler) cannot leave
    # the GPU idle inside the timed region; the gate opens after them (the
    # launch queue stays far from full) and the host stays that far ahead.
    # Nothing in a step synchronises with the host.
    GATE_STEPS = 32
    if flush_l2:
        scratch.fill_(1)          # its kernel loaded before the window (lazy loading blocks the host)
    gate_note = None
    use_gate = world == 1 and not use_graph
    if use_gate:
        # a profiler (ncu) runs every launch to completion before returning;
        # there a gate could only time out: probe with a 2 ms one first
        from paper_1504_05158_b200 import _lib as _gl
        probe = torch.zeros(2, dtype=torch.int32, pin_memory=True)
        w0 = time.perf_counter()
        _gl.call("qsb_stream_gate", probe.data_ptr(), int(2e6), probe.data_ptr() + 4, stream.cuda_stream)
        serialized = time.perf_counter() - w0 > 1e-3
        torch.cuda.synchronize()
        use_gate = not serialized
    for attempt in (0, 1):
        gate = None
        if use_gate and attempt == 0:
            from paper_1504_05158_b200 import _lib as _gl
            gate = (torch.zeros(1, dtype=torch.int32, pin_memory=True),
                    torch.zeros(1, dtype=torch.int32, pin_memory=True))
            _gl.call("qsb_stream_gate", gate[0].data_ptr(), int(10e9), gate[1].data_ptr(),
                     stream.cuda_stream)
        t_start.record(stream)
        if use_graph:
            timer.active = False
            qsb.step_many(state, inst, cfg, args.steps)
        elif flush_l2:
            pairs = []
            for i in range(args.steps):
                if gate is not None and i == GATE_STEPS:
                    gate[0][0] = 1
                scratch.fill_(1)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                one_step()
                e1.record(stream)
                pairs.append((e0, e1))
        else:
            for i in range(args.steps):
                if gate is not None and i == GATE_STEPS:
                    gate[0][0] = 1
                one_step()
        t_end.record(stream)
        if gate is not None:
            gate[0][0] = 1
        torch.cuda.synchronize()
        if gate is None or int(gate[1][0]) == 0:
            break
        # the gate gave up (something in the window waited on the host): the
        # window is measured again, ungated, on a fresh population
        gate_note = "gate timed out; window re-measured without it"
        print("bench: " + gate_note, file=sys.stderr)
        del state
        torch.cuda.empty_cache()
        state = qsb.init_population(cfg, inst, device=dev, swarm_range=(lo, hi))
        if flags is not None:
            state.set_lazy_scale(False)
        for _ in range(args.warmup):
            one_step()
        torch.cuda.synchronize()
        launches0 = state.launches
    if flush_l2:
        step_ms = sum(a.elapsed_time(b) for a, b in pairs)
    if world > 1:
        dist.barrier()
    clock_rec = clocks.stop() if clocks else None
    ms = step_ms if step_ms is not None else t_start.elapsed_time(t_end)
    launches = state.launches - launches0
    # the kernel-timing pass: CUDA events around every fused-kernel (and 2-opt)
    # launch, over the same iterations on a fresh population (eager steps after
    # the graph replays in graph mode), with the same L2 flushes
    if args.graph and world == 1 and flags is None:
        timer.active = True
        for _ in range(args.steps):
            one_step()
        torch.cuda.synchronize()
    else:
        del state
        torch.cuda.empty_cache()
        state = qsb.init_population(cfg, inst, device=dev, swarm_range=(lo, hi))
        if flags is not None:
            state.set_lazy_scale(False)
        for _ in range(args.warmup):
            one_step()
        torch.cuda.synchronize()
        timer.active = True
        for _ in range(args.steps):
            if flush_l2:
                scratch.fill_(1)
            one_step()
        torch.cuda.synchronize()
    timer.active = False
    kern_ms = timer.mean_ms()
    tm = torch.tensor([ms, kern_ms or 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms_max, kern_max = float(tm[0]), float(tm[1])
    P_total = cfg.num_particles
    value = P_total * args.steps / (ms_max / 1000.0)

    # ---- end to end through the public API: step() + D2H of the step's
    # per-particle costs and best record, synchronised every step
    e2e_steps = (args.steps if args.e2e_steps < 0 else args.e2e_steps) if flags is None else 0
    e2e_resident = None
    if e2e_steps:
        # a fresh population, warmed up like the device-timed run, so the
        # end-to-end window covers the same iterations (W+1 .. W+K)
        del state
        torch.cuda.empty_cache()
        state = qsb.init_population(cfg, inst, device=dev, swarm_range=(lo, hi))
        for _ in range(args.warmup):
            qsb.step(state, inst, cfg, exchange=exchange)
        # double-buffered pinned results: the host reads step i's costs while
        # step i+1 runs (every step's result still crosses to the host)
        host_cost = [torch.empty(state.local_particles, dtype=state.d_cost.dtype, pin_memory=True)
                     for _ in range(2)]
        host_best = [torch.empty(1, dtype=state.d_best_cost.dtype, pin_memory=True)
                     for _ in range(2)]
        evs = [torch.cuda.Event() for _ in range(2)]
        # the D2H runs on a copy stream so it overlaps the next step: the
        # compute stream snapshots the results into a device staging buffer
        # (a 640 KB D2D at config 3), the copy stream drains it to the host
        main = torch.cuda.current_stream()
        cstream = torch.cuda.Stream()
        dev_cost = [torch.empty_like(state.d_cost) for _ in range(2)]
        dev_best = [torch.empty_like(state.d_best_cost) for _ in range(2)]
        snap = [torch.cuda.Event() for _ in range(2)]
        checksum = 0
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        for i in range(e2e_steps):
            qsb.step(state, inst, cfg, exchange=exchange)
            b = i % 2
            if i >= 2:
                main.wait_event(evs[b])          # staging buffer b drained
            dev_cost[b].copy_(state.d_cost, non_blocking=True)
            dev_best[b].copy_(state.d_best_cost, non_blocking=True)
            snap[b].record(main)
            cstream.wait_event(snap[b])
            with torch.cuda.stream(cstream):
                host_cost[b].copy_(dev_cost[b], non_blocking=True)
                host_best[b].copy_(dev_best[b], non_blocking=True)
                evs[b].record(cstream)
            if i:
                evs[1 - b].synchronize()
                checksum += int(host_best[1 - b][0]) + int(host_cost[1 - b][0])
        evs[(e2e_steps - 1) % 2].synchronize()
        checksum += int(host_best[(e2e_steps - 1) % 2][0])
        w = time.perf_counter() - w0
        wt = torch.tensor([w], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        e2e_resident = {"value": P_total * e2e_steps / float(wt[0]), "unit": UNIT,
               "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(host_cost[0].numel() * host_cost[0].element_size()
                                         + host_best[0].element_size()),
               "steps": e2e_steps,
               "how": "public step() per iteration + D2H of that iteration's per-particle cost "
                      "vector and best cost into pinned memory, read on the host one step behind "
                      "(double-buffered; the D2H runs on a copy stream from a device snapshot, overlapping the next step), wall clock, max over ranks, on a fresh population over "
                      "the same iterations as the device-timed window; the population stays "
                      "resident (the random streams are generated in-kernel, so an iteration has "
                      "no host inputs)"}

    # ---- roofline of the fused kernel
    sv = 4 if cfg.precision == "fp32" else 8
    lazy = getattr(state, "d_vcol", None) is not None
    B = bytes_per_particle(args.n, args.swarm_size, sv, lazy=lazy)
    if flags is not None:
        B = 2 * args.n * args.n * sv + 4 * args.n + 2 * args.n / args.swarm_size + 32
    moved_per_launch = B * state.local_particles
    # roofline.achieved uses SURVEY.md §8(d)'s algorithmic bytes of the
    # velocity/normalise phase, B_vel = 2 n^2 s_V + 2 n 2 + 2 n / S per
    # particle-iteration (read + write V, X and PL perms, PG amortised); the
    # bytes this layout actually has to move (lazy column scale: the tile
    # read, <= 3n entries written, column state) are reported beside it
    B_vel = 2 * args.n * args.n * sv + 4 * args.n + 2 * args.n / args.swarm_size
    per_launch = B_vel * state.local_particles if flags is None else moved_per_launch
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = per_launch / (kern_max / 1000.0) / 1e9 if kern_max else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic_from_profile(args.n, cfg.precision, state.local_particles,
                                                "velocity_only_" if flags is not None else ""),
                "kernel": ("step_kernel (fused velocity+aggregation+goal+pbest; draws made by the previous best_kernel)"
                           if engine._COEF_FOLD else
                           "coef_kernel + step_kernel (draw pre-pass; fused velocity+aggregation+goal+pbest)") if flags is None
                          else "step_kernel velocity-only build",
                "kernel_ms": kern_max,
                "kernel_timing": ("CUDA events around every launch on its stream, in a second pass "
                                  "over the same iterations (not in the timed region: an event "
                                  "between kernels breaks the PDL chain)"),
                "algorithmic_bytes_per_launch": per_launch,
                "algorithmic_bytes_per_particle": "SURVEY §8(d) B_vel = 2 n^2 s_V + 4 n + 2 n / S"
                                                  if flags is None else "velocity-only build: V read + write",
                "moved_bytes_per_launch": moved_per_launch,
                "moved_frac": (moved_per_launch / (kern_max / 1000.0) / 1e9 / peak) if kern_max else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk.exists() else "fallback"}

    # ---- the 2-opt kernel's tensor-core roofline (configs with 2-opt):
    # algorithmic work of a pass is the GEMM H = [F|P][P|F]^T, 2 * n * n * 2n
    # ops per particle; peak = 2 x the measured dense bf16 rate (B200's dense
    # int8 rate is twice its bf16 rate)
    roofline2 = None
    t2 = timer.mean_twoopt_ms()
    if args.two_opt and t2:
        ops = 4.0 * args.n ** 3 * state.local_particles * args.two_opt
        bf16 = peaks.get("bf16_tflops")
        peak2 = 2.0 * bf16 if bf16 else 4500.0
        tmax = torch.tensor([t2], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        ach2 = ops / (float(tmax[0]) / 1000.0) / 1e12
        roofline2 = {"bound": "tensor", "achieved": ach2, "peak": peak2, "unit": "TOP/s",
                     "frac": ach2 / peak2, "traffic": None,
                     "kernel": "twoopt_tc kernels (tcgen05.mma kind::i8, u8 x u8 -> s32)",
                     "kernel_ms": float(tmax[0]),
                     "algorithmic_ops_per_launch": ops,
                     "note": "upper bound on passes (a particle stops early when no swap improves)",
                     "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops" if bf16 else "nominal int8 dense"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample(args, args.cpu_seconds)

    best = shard.merge_best(state.best_cost, state.best_iteration, 0, state.best_perm, world,
                            dev) if world > 1 else None
    best_cost = best.cost if best else state.best_cost
    # ---- end to end through the reference-facing C-ABI on HOST buffers:
    # host.step_host (qsb_step_host) on the reference's PopulationState
    # layout in pinned host memory -- f64 V, int8 0/1 matrices, int64 perms
    # -- shipped to the device and back every step (fp64 reference
    # arithmetic: the host layout is the reference's float64 state)
    e2e = None
    value_fp64 = None
    host_steps = min(args.host_steps, args.steps) if (flags is None and world == 1) else 0
    fp64_steps = args.fp64_steps if (flags is None and world == 1) else 0
    if (host_steps and args.two_opt == 0) or fp64_steps:
        del state
        torch.cuda.empty_cache()
        cfg64 = config(args, precision="fp64")
        st64 = qsb.init_population(cfg64, inst, device=dev, swarm_range=(lo, hi))
        for _ in range(args.warmup):
            qsb.step(st64, inst, cfg64, exchange=exchange)
        if fp64_steps:
            # ---- the fp64 parity mode (bit-identical to the reference),
            # device-resident, same workload, iterations W+1 .. W+K64
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(fp64_steps):
                qsb.step(st64, inst, cfg64, exchange=exchange)
            e1.record()
            torch.cuda.synchronize()
            ms64 = e0.elapsed_time(e1)
            value_fp64 = {"value": P_total * fp64_steps / (ms64 / 1000.0), "unit": UNIT,
                          "ms_per_step": ms64 / fp64_steps, "steps": fp64_steps,
                          "iterations": f"{args.warmup + 1}-{args.warmup + fp64_steps}",
                          "how": "precision='fp64' (bit-identical to the reference), device-"
                                 "resident, CUDA events around the steps"}
    if host_steps and args.two_opt == 0:
        from paper_1504_05158_b200 import host
        hp = host.HostPopulation.from_state(st64, cfg64)
        del st64
        torch.cuda.empty_cache()
        host.step_host(hp, inst, cfg64)            # first call allocates the device buffers
        torch.cuda.synchronize()
        bytes_in = bytes_out = 0
        w0 = time.perf_counter()
        for _ in range(host_steps):
            mig = cfg64.migration_factor > 0 and (hp.t + 1) % cfg64.migration_period == 0
            bi, bo = hp.transfer_bytes(inst, migrate=mig)
            bytes_in += bi
            bytes_out += bo
            host.step_host(hp, inst, cfg64)
        w = time.perf_counter() - w0
        e2e = {"value": P_total * host_steps / w, "unit": UNIT,
               "h2d_bytes_per_step": int(bytes_in / host_steps),
               "d2h_bytes_per_step": int(bytes_out / host_steps),
               "steps": host_steps, "iterations": f"{hp.t - host_steps + 1}-{hp.t}",
               "pcie_gb_s": (bytes_in + bytes_out) / w / 1e9,
               "how": "host.step_host -> qsb_step_host (include/qapswarm_b200.h): one reference "
                      "engine.step on the reference's host PopulationState (pinned numpy buffers: "
                      "f64 V, int8 X/X_new/PL and swarm-best matrices, int64 perms/costs); every "
                      "step copies the state host->device and the results device->host (16 "
                      "swarm-aligned chunks, copies overlapped with the fused fp64 step, "
                      "migration on the device); wall clock, synchronous calls; fp64 reference "
                      "arithmetic (the host layout is the reference's float64 state)"}

    if rank == 0:
        metric = METRIC if args.preset == "config3" else \
            f"particle-iterations/sec (QAP n={args.n}, {P_total} particles, {args.preset})"
        line = {"metric": metric, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32" if cfg.precision == "fp32" else "f64", "data": "synthetic",
                "config": dict(workload(args, world), l2=(
                    f"velocity state {vbytes / 1e6:.0f} MB per GPU "
                    + ("< 2 x L2: L2 flushed (256 MB write) before every timed step, steps timed "
                       "one by one" if flush_l2 else
                       "< 2 x L2, CUDA-graph replay without flushes (launch-latency bound)"
                       if use_graph and vbytes < 2 * L2_BYTES else
                       "> 2 x L2 (126 MB): inputs larger than L2")),
                    timed_window=(gate_note if gate_note else
                                  f"the first {min(GATE_STEPS, args.steps)} of the K steps "
                                  "enqueued behind a host-released gate (qsb_stream_gate), CUDA "
                                  "events around all K; per-kernel events only in a second pass"
                                  if gate is not None else
                                  "CUDA events around the K steps")),
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "e2e_resident": e2e_resident, "value_fp64": value_fp64,
                "gpu_launches": launches, "clocks": clock_rec,
                "roofline_twoopt": roofline2,
                "best_cost": best_cost}
        if flags is not None:
            line["metric"] = "velocity/normalise phase HBM throughput"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
