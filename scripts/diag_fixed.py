"""Fixed (per-launch) versus per-particle cost of the fused step kernel at
config 3's shape (diagnostic): the kernel time at t = 10..14 for several
population sizes, CUDA events around each launch, no L2 flush."""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_1504_05158_b200 as qsb

inst = qsb.taillard_uniform(50)
out = {}
for m in (100, 200, 400, 800, 1600):
    cfg = qsb.SolverConfig(swarms=m, swarm_size=100, seed=1, precision="fp32", init="device",
                           migration_factor=0.33, migration_period=10,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    st = qsb.init_population(cfg, inst)
    for _ in range(9):
        qsb.step(st, inst, cfg)

    class T:
        def __init__(s): s.p = []
        def before(s, _):
            e = torch.cuda.Event(enable_timing=True); e.record(); s.p.append([e, None])
        def after(s, _):
            e = torch.cuda.Event(enable_timing=True); e.record(); s.p[-1][1] = e
    tm = T()
    for _ in range(5):
        qsb.step(st, inst, cfg, timer=tm)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in tm.p]
    out[m * 100] = round(sum(ms) / len(ms), 5)
    del st
    torch.cuda.empty_cache()
ps = sorted(out)
fits = {}
for a, b in zip(ps, ps[1:]):
    slope = (out[b] - out[a]) / (b - a)
    fits[f"{a}-{b}"] = {"us_per_1k": round(slope * 1e6, 3), "fixed_us": round((out[a] - slope * a) * 1000, 2)}
print(json.dumps({"kernel_ms": out, "fit": fits}))
