"""Pipeline stamps of the CTA-pair 2-opt kernel (diagnosis build libqsb_tt.so,
-DQSB_TCP_TIMING): per particle of CTA 0, cycles of the events."""
import ctypes, os, sys
sys.path.insert(0, ".")
os.environ["QSB_LIB"] = os.path.abspath("paper_1504_05158_b200/libqsb_tt.so")
import numpy as np
from paper_1504_05158_b200 import batch, _lib
from oracle import oracle as orc
n = 256
rng = np.random.default_rng(3)
f = np.triu(rng.integers(0, 100, (n, n)), 1); d = np.triu(rng.integers(0, 100, (n, n)), 1)
f, d = f + f.T, d + d.T
P = 74 * 14
perms = np.array([rng.permutation(n) for _ in range(P)], dtype=np.int64)
costs = np.zeros(P, np.int64)
orc.cost_many(perms, f, d, costs)
batch.twoopt_many(perms.copy(), f, d, costs.copy(), 1)
ts = np.zeros((64, 12), np.int64)
L = _lib.lib()
fn = getattr(L, "qsb_debug_pair_stamps")
fn(ts.ctypes.data_as(ctypes.c_void_p))
names = ["bld", "list", "built", "iss_full", "iss_hfree", "commit", "epi_mma", "epi_tmem0", "epi_tmem3", "epi_red", "epi_pair", "epi_done"]
t0 = ts[0, 0]
for i in range(14):
    print(i, " ".join(f"{nm}={(ts[i, k] - t0) / 1000:6.1f}" for k, nm in enumerate(names)))
print("cycles per particle (steady)", (ts[13, 11] - ts[3, 11]) / 10)
