"""Per-iteration fused-kernel time, every iteration (diagnostic)."""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_1504_05158_b200 as qsb
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
inst = qsb.taillard_uniform(50)
cfg = qsb.SolverConfig(swarms=800, swarm_size=100, seed=1, precision="fp32", init="device",
                       migration_factor=0.33, migration_period=10,
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
ms = [round(a.elapsed_time(b), 3) for a, b in tm.p]
print(json.dumps(ms))
