"""Per-iteration fused-kernel time with the lazily scaled layout switched off
(stored-v streaming passes), for comparison with diag_steps.py."""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_1504_05158_b200 as qsb
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 500
inst = qsb.taillard_uniform(50)
cfg = qsb.SolverConfig(swarms=800, swarm_size=100, seed=1, precision="fp32", init="device",
                       migration_factor=0.33, migration_period=10,
                       coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
st = qsb.init_population(cfg, inst)
st.set_lazy_scale(False)
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
ms = [a.elapsed_time(b) for a, b in tm.p]
print(json.dumps({"nolazy_kernel_ms": {str(i + 1): round(sum(ms[i:i + 20]) / 20, 3) for i in range(0, iters, 20)}}))
