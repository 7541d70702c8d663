"""Host-buffer e2e leg (qsb_step_host) at config 3 for several chunk counts,
plus the raw pinned PCIe bandwidth (H2D, D2H, both at once) for the bound."""
import json, os, sys, time
sys.path.insert(0, ".")
import torch
import paper_1504_05158_b200 as qsb
from paper_1504_05158_b200 import host

inst = qsb.taillard_uniform(50)
cfg = qsb.SolverConfig(swarms=800, swarm_size=100, seed=1, precision="fp64", init="device",
                       migration_factor=0.33, migration_period=10,
                       coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
out = {}
# raw PCIe: 1 GB pinned buffers
N = 1 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name in ("h2d", "d2h", "duplex"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        if name in ("h2d", "duplex"):
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
        if name in ("d2h", "duplex"):
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out[f"pcie_{name}_gb_s"] = round((2 if name == "duplex" else 1) * 3 * N / dt / 1e9, 1)
del h, h2, d, d2
torch.cuda.empty_cache()
st = qsb.init_population(cfg, inst)
for _ in range(5):
    qsb.step(st, inst, cfg)
hp = host.HostPopulation.from_state(st, cfg)
del st
torch.cuda.empty_cache()
for k in [int(x) for x in (sys.argv[1:] or ["8", "16", "32"])]:
    os.environ["QSB_HOST_CHUNKS"] = str(k)
    host.step_host(hp, inst, cfg)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    steps = 8
    for _ in range(steps):
        host.step_host(hp, inst, cfg)
    w = time.perf_counter() - w0
    out[f"chunks{k}_ms_per_step"] = round(1000 * w / steps, 2)
    out[f"chunks{k}_M_particle_iter_s"] = round(80000 * steps / w / 1e6, 3)
print(json.dumps(out))
