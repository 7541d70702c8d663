"""Small invocations of every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck; scripts/gpu_sanitize.sh).

Each case launches the kernels a user call launches: init, the draw
pre-pass, the fused step (one-warp lazy fp32, one-warp fp64, multi-warp
fp32 deferred / fp64, the global-memory tile), best update, migration,
the 2-opt kernels (tensor-core and dp4a) and the device statistics.
Sizes are tiny so the instrumented run finishes in minutes."""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1504_05158_b200 as qsb  # noqa: E402

CASES = {
    # name: (n, swarms, swarm_size, precision, migration, two_opt, init)
    "lazy_fp32_n30": (30, 3, 5, "fp32", 0.34, 0, "device"),
    "fp64_n30": (30, 3, 5, "fp64", 0.34, 0, "reference"),
    "lazy_fp32_n50_2opt": (50, 2, 4, "fp32", 0.0, 1, "device"),
    "multiwarp_fp32_n100": (100, 2, 3, "fp32", 0.0, 0, "device"),
    "multiwarp_fp64_n100": (100, 2, 3, "fp64", 0.0, 0, "device"),
    "gtile_fp32_n256_2opt": (256, 2, 2, "fp32", 0.0, 1, "device"),
    "twoopt_fp32_n30": (30, 2, 4, "fp32", 0.0, 2, "device"),
}


def run_case(name: str, steps: int = 3) -> None:
    n, m, S, prec, mig, two, init = CASES[name]
    inst = qsb.taillard_uniform(n)
    cfg = qsb.SolverConfig(swarms=m, swarm_size=S, seed=5, migration_factor=mig, precision=prec,
                           init=init, two_opt_passes=two,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, inst)
    for _ in range(steps):
        qsb.step(st, inst, cfg)
    qsb.engine.collect_device(st, 0.0)
    torch.cuda.synchronize()
    print(f"{name}: t={st.t} best={st.best_cost}", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        run_case(nm)
