"""Per-step overhead outside the fused kernel at config 3 (diagnostic):
the same 20 iterations timed as (A) pre-pass + fused kernel only, (B) A plus
the best update, (C) the public step() with the folded pre-pass, (D) C with
CUDA events recorded around every fused-kernel launch (bench.py's kernel
timer).  A and B
leave the population inconsistent and exist only for timing."""
import sys, json
sys.path.insert(0, '.')
import torch
import paper_1504_05158_b200 as qsb
from paper_1504_05158_b200 import _lib, engine

inst = qsb.taillard_uniform(50)
cfg = qsb.SolverConfig(swarms=800, swarm_size=100, seed=1, precision="fp32", init="device",
                       migration_factor=0.33, migration_period=10,
                       coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
out = {}
class T:
    def __init__(s): s.p = []
    def before(s, _):
        e = torch.cuda.Event(enable_timing=True); e.record(); s.p.append([e, None])
    def after(s, _):
        e = torch.cuda.Event(enable_timing=True); e.record(); s.p[-1][1] = e
for mode in ("A", "B", "C", "C2", "D"):
    st = qsb.init_population(cfg, inst)
    for _ in range(5):
        qsb.step(st, inst, cfg)
    torch.cuda.synchronize()
    rt = engine._runtime(st, inst, cfg)
    s = st.stream()
    tm = T()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        if mode in ("C", "C2"):
            qsb.step(st, inst, cfg)
        elif mode == "D":
            qsb.step(st, inst, cfg, timer=tm)
        else:
            rt.coeffs.hints = engine._hints(st, rt, cfg.coefficients)
            _lib.call("qsb_step_phases", st.c_state(), rt.inst, rt.coeffs, _lib.PHASE_ALL, None, 0, 2, None, 0, s)
            if mode == "B":
                _lib.call("qsb_best_update", st.c_state(), s)
            st.swap_positions()
    e1.record()
    torch.cuda.synchronize()
    out[mode] = round(e0.elapsed_time(e1) / 20, 5)
print(json.dumps(out))
