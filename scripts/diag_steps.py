"""Per-iteration fused-kernel time over a long run (diagnostic)."""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1504_05158_b200 as qsb
from paper_1504_05158_b200 import _lib, engine

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 500
swarms = int(sys.argv[3]) if len(sys.argv) > 3 else 800
inst = qsb.taillard_uniform(50)
cfg = qsb.SolverConfig(swarms=swarms, swarm_size=100, seed=1, precision=prec, init="device",
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
w0 = time.perf_counter()
for t in range(iters):
    qsb.step(st, inst, cfg, timer=tm)
torch.cuda.synchronize()
wall = time.perf_counter() - w0
ms = [a.elapsed_time(b) for a, b in tm.p]
out = {"prec": prec, "wall_ms_per_step": 1000 * wall / iters,
       "kernel_ms": {str(i + 1): round(ms[i], 3) for i in range(0, iters, max(1, iters // 25))}}
V = st.V
out["zero_frac"] = float((V == 0).mean())
out["denorm_frac"] = float(((V != 0) & (np.abs(V) < np.finfo(V.dtype).tiny)).mean())
dup = np.mean([50 - len(np.unique(V[p, :, c])) for p in range(0, st.local_particles, 997) for c in range(50)])
out["dups_per_col"] = float(dup)
print(json.dumps(out))
