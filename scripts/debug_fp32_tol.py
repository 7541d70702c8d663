"""Debug: worst entry of the fp32 single-step tolerance check."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np, torch
import paper_1504_05158_b200 as qsb
from oracle import oracle as orc
from conftest import load_instances

name, warm = sys.argv[1], int(sys.argv[2])
inst = load_instances()[0][name]
cfg = qsb.SolverConfig(swarms=20, swarm_size=25, seed=1, precision="fp32",
                       coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
st = qsb.init_population(cfg, inst)
for _ in range(warm):
    qsb.step(st, inst, cfg)
n = inst.n
ost = orc.init_population(20, 25, n, inst.flow, inst.distance, seed=1)
ost.X, ost.perms = st.X, st.perms
ost.PL, ost.pl_perms, ost.pl_cost = st.PL, st.pl_perms, st.pl_cost
b = st.bests
ost.pg_mats, ost.pg_perms, ost.pg_costs = b.matrices, b.perms, b.costs
ost.V = st.V.astype(np.float64)
ost.t = st.t
v0 = ost.V.copy()
vc0 = st.d_vcol.clone().cpu()
u0 = st.d_V[:, :n * n].view(-1, n, n).clone().cpu().numpy()
perm0, pl0 = st.perms, st.pl_perms
pg0 = st.bests.perms
qsb.step(st, inst, cfg)
orc.step(ost, inst.flow, inst.distance, **orc.coeff_kwargs(cfg))
got = st.V.astype(np.float64)
ref = ost.V
scale = np.abs(ref).max(axis=1, keepdims=True)
err = np.abs(got - ref) / np.where(scale > 0, scale, 1.0)
p, r, c = np.unravel_index(err.argmax(), err.shape)
print("max err", err.max(), "at", p, r, c)
print("x row", perm0[p, c], "pl row", pl0[p, c], "pg row", pg0[p // 25, c])
print("got", got[p, r, c], "ref", ref[p, r, c], "colmax", scale[p, 0, c], "v0", v0[p, r, c])
u1 = st.d_V[:, :n * n].view(-1, n, n).cpu().numpy()
vc1 = st.d_vcol.cpu()
print("u0", u0[p, r, c], "u1", u1[p, r, c], "s0", float(vc0[p, 0, c]), "s1", float(vc1[p, 0, c]))
w0 = vc0.view(torch.int32)[p, :, c].tolist(); w1 = vc1.view(torch.int32)[p, :, c].tolist()
print("col words before", w0, "after", w1)
colref = ref[p, :, c]; colgot = got[p, :, c]
print("ref col sum|.|", np.abs(colref).sum(), "got", np.abs(colgot).sum())
print("rel err per row (top 5):", sorted(zip(err[p, :, c], range(n)))[-5:])
print("sum |u1|", np.abs(u1[p, :, c].astype(np.float64)).sum())
