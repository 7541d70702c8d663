"""Pack the reference's bundled instances (pkg/src/qapswarm/data/, see its
README for provenance) into paper_1504_05158_b200/data/bundled.npz, read by
paper_1504_05158_b200.datasets.  Run in the build container (it reads
/root/reference); the .npz is committed, the reference files are not."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1504_05158_b200 import instance as I   # noqa: E402

SRC = Path("/root/reference/pkg/src/qapswarm/data")
arrays = {}
for dat in sorted(SRC.glob("*.dat")):
    inst = I.load_instance(dat)
    arrays[f"{inst.name}__flow"] = inst.flow
    arrays[f"{inst.name}__distance"] = inst.distance
    sln = dat.with_suffix(".sln")
    if sln.exists():
        sol = I.load_reference_solution(sln)
        arrays[f"{inst.name}__sln_perm"] = sol.permutation
        arrays[f"{inst.name}__sln_cost"] = np.array(sol.cost)
np.savez_compressed(ROOT / "paper_1504_05158_b200" / "data" / "bundled.npz", **arrays)
print(sorted(arrays))
