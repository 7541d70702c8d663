"""Every iteration's fused-kernel time over a long run (config 3, fp32)."""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_1504_05158_b200 as qsb
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 500
mig = float(sys.argv[2]) if len(sys.argv) > 2 else 0.33
period = int(sys.argv[3]) if len(sys.argv) > 3 else 10
inst = qsb.taillard_uniform(50)
cfg = qsb.SolverConfig(swarms=800, swarm_size=100, seed=1, precision="fp32", init="device",
                       migration_factor=mig, migration_period=period,
                       coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
st = qsb.init_population(cfg, inst)
class T:
    def __init__(s): s.p = []
    def before(s, _):
        e = torch.cuda.Event(enable_timing=True); e.record(); s.p.append([e, None])
    def after(s, _):
        e = torch.cuda.Event(enable_timing=True); e.record(); s.p[-1][1] = e
tm = T()
for t in range(iters):
    qsb.step(st, inst, cfg, timer=tm)
torch.cuda.synchronize()
print(json.dumps({"mig": mig, "ms": [round(a.elapsed_time(b), 3) for a, b in tm.p]}))
