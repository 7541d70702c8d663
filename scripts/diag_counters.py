"""Aggregation event counters per particle-iteration (diagnosis build)."""
import ctypes, os, sys
os.environ["QSB_LIB"] = os.path.join(os.path.dirname(__file__), "..", "paper_1504_05158_b200", "libqsb_counters.so")
sys.path.insert(0, ".")
import torch
import paper_1504_05158_b200 as qsb
from paper_1504_05158_b200 import _lib
L = _lib.lib()
L.qsb_debug_counters.argtypes = [ctypes.c_void_p]
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
inst = qsb.taillard_uniform(50)
cfg = qsb.SolverConfig(swarms=80, swarm_size=100, seed=1, precision=prec, init="device",
                       migration_factor=0.33, migration_period=10,
                       coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
st = qsb.init_population(cfg, inst)
buf = (ctypes.c_ulonglong * 12)()
names = ["particles", "normal_rounds", "bulk_steps", "bulk_cells", "tie_rounds", "warp_tie", "slow_tie",
         "rescans", "full_pass", "incr_rescans", "incr_unknown", "renorm"]
L.qsb_debug_counters(buf)
for t in range(1, 401):
    qsb.step(st, inst, cfg)
    if t in (1, 10, 50, 100, 150, 200, 300, 400):
        torch.cuda.synchronize()
        L.qsb_debug_counters(buf)
        P = buf[0]
        print(t, {names[i]: round(buf[i] / P, 3) for i in range(1, 12)})
    else:
        torch.cuda.synchronize()
        L.qsb_debug_counters(buf)
