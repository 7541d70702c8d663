"""Repro / diagnosis: fp32 steps at size n with migration, synchronising every step."""
import sys; sys.path.insert(0, '.')
import torch, paper_1504_05158_b200 as qsb
n = int(sys.argv[1]); sw = int(sys.argv[2]); iters = int(sys.argv[3]) if len(sys.argv) > 3 else 12
mig = float(sys.argv[4]) if len(sys.argv) > 4 else 0.33
inst = qsb.taillard_uniform(n)
cfg = qsb.SolverConfig(swarms=sw, swarm_size=100, seed=1, precision="fp32", init="device",
                       migration_factor=mig, migration_period=10,
                       coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
st = qsb.init_population(cfg, inst)
for t in range(iters):
    try:
        qsb.step(st, inst, cfg)
        torch.cuda.synchronize()
        if "--check" in sys.argv:
            p_, nn = st.local_particles, n * n
            u = st.d_V[:, :nn].float()
            sc = st.d_vcol[:, 0, :n] if st.d_vcol is not None else None
            bad_u = (~torch.isfinite(u)).sum().item()
            mx = u.abs().max().item()
            smin = sc.min().item() if sc is not None else None
            smax = sc.max().item() if sc is not None else None
            bad_s = (~torch.isfinite(sc)).sum().item() if sc is not None else None
            perm = st.d_perm.long()
            ok_perm = bool(((perm.sort(dim=1).values - torch.arange(n, device=perm.device)) == 0).all())
            print(t + 1, "u nonfinite", bad_u, "max|u|", mx, "s", smin, smax, "s nonfinite", bad_s, "perms ok", ok_perm)
    except Exception as e:
        print("failed at step", t + 1, repr(e)[:200]); raise
print("ok", st.best_cost)
