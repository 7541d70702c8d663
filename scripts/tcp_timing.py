"""Pipeline stamps of the pipelined 2-opt kernel (diagnosis build
libqsb_tt.so, -DQSB_TCP_TIMING): per particle of CTA 0, cycles between the
events (builders start / P built / issuer ready / full / hfree / commit,
epilogue start / TMEM done (q0, q3) / apply done)."""
import ctypes, os, sys
sys.path.insert(0, ".")
os.environ["QSB_LIB"] = os.path.abspath("paper_1504_05158_b200/libqsb_tt.so")
import numpy as np, torch
from paper_1504_05158_b200 import batch, _lib
from oracle import oracle as orc
n = 256
rng = np.random.default_rng(3)
f = np.triu(rng.integers(0, 100, (n, n)), 1); d = np.triu(rng.integers(0, 100, (n, n)), 1)
f, d = f + f.T, d + d.T
P = 148 * 14
perms = np.array([rng.permutation(n) for _ in range(P)], dtype=np.int64)
costs = np.zeros(P, np.int64)
orc.cost_many(perms, f, d, costs)
batch.twoopt_many(perms.copy(), f, d, costs.copy(), 1)
ts = np.zeros((64, 10), np.int64)
_lib.lib().qsb_debug_tcp_stamps(ts.ctypes.data_as(ctypes.c_void_p))
names = ["bld_start", "P_built", "iss_ready", "full", "hfree", "commit", "epi_start", "epi_tmem_q0", "epi_tmem_q3", "epi_done"]
t0 = ts[0, 0]
for i in range(14):
    print(i, " ".join(f"{nm}={(ts[i, k] - t0) / 1000:7.2f}k" for k, nm in enumerate(names)))
per = (ts[13, 9] - ts[3, 9]) / 10
print("cycles per particle (steady)", per, "->", per / 1.9e3, "us")
