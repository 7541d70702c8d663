"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run once in the build container (the reference is importable only there):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

The outputs are small .npz / .json / .csv files committed next to this
script; tests read them on any box (the GPU box has no /root/reference).
Nothing here is imported by the product or by the tests.
"""

from __future__ import annotations

import hashlib
import io
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = os.environ.get("QAPSWARM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import qapswarm as qs                      # noqa: E402
from qapswarm import _batch, streams      # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(state) -> str:
    h = hashlib.sha256()
    for a in (state.X, state.V, state.PL, state.perms, state.cost, state.pl_cost,
              state.bests.matrices, state.bests.costs):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def taillard(n: int):
    """Synthetic Taillard-style uniform instance."""
    rng = np.random.default_rng(1000 + n)

    def sym():
        m = np.triu(rng.integers(0, 100, (n, n)), 1)
        return (m + m.T).astype(np.int64)
    f = sym()
    d = sym()
    return qs.QapInstance(f"tai{n}-synthetic", n, f, d)


def float_instance():
    rng = np.random.default_rng(2)
    n = 6
    f = rng.uniform(0, 10, (n, n))
    f = np.triu(f, 1) + np.triu(f, 1).T
    d = rng.uniform(0, 10, (n, n))
    d = np.triu(d, 1) + np.triu(d, 1).T
    return qs.QapInstance("float6", n, f, d)


def instances():
    chr12a = qs.load_bundled("chr12a")
    return {
        "chr12a": chr12a,
        "esc32e": qs.load_bundled("esc32e"),
        "rand26": qs.load_bundled("rand26"),
        "tiny": qs.parse_instance("2  0 1  1 0   0 3  3 0", name="tiny"),
        "tai30": taillard(30),
        "tai50": taillard(50),
        "float6": float_instance(),
    }


def save_instances(insts):
    arrays = {}
    meta = {}
    for k, inst in insts.items():
        arrays[f"{k}__flow"] = np.asarray(inst.flow)
        arrays[f"{k}__distance"] = np.asarray(inst.distance)
        meta[k] = {"name": inst.name, "n": inst.n,
                   "known_best": inst.known_best}
    np.savez_compressed(OUT / "instances.npz", **arrays)
    sln = qs.load_bundled_solution("chr12a")
    meta["chr12a_sln"] = {"cost": sln.cost, "perm": sln.permutation.tolist()}
    (OUT / "instances.json").write_text(json.dumps(meta, indent=1))


def gen_draws():
    cases = [(1, 3, 50, 12), (42, 7, 9, 5), (-1, 1, 4, 3), (7, 2**32 - 1, 3, 30),
             (2**63 + 5, 12345, 17, 50)]
    arrays = {}
    for i, (seed, t, P, n) in enumerate(cases):
        arrays[f"case{i}"] = streams.step_draws(seed, t, P, n)
    arrays["cases"] = np.array([[c[0] & (2**64 - 1), c[1], c[2], c[3]] for c in cases],
                               dtype=np.uint64)
    # host stream: the migration picks (integers) for a few keys
    picks = []
    for seed, t, S, d in [(1, 10, 100, 264), (3, 5, 20, 16), (5, 1, 10, 1)]:
        rng = streams.host_rng(seed, t)
        picks.append(np.array([rng.integers(0, S) for _ in range(d)], dtype=np.int64))
    for i, p in enumerate(picks):
        arrays[f"host{i}"] = p
    np.savez_compressed(OUT / "draws.npz", **arrays)


def gen_velocity():
    rng = np.random.default_rng(31)
    arrays = {}
    k = 0
    for n, P, S in [(6, 8, 4), (13, 6, 3), (50, 4, 2)]:
        for sv in ("raw", "norm"):
            for c1, c2, c3 in [(0.8, 0.5, 0.5), (0.0, 0.0, 1.0), (1.0, 0.3, 0.0)]:
                perms = np.array([rng.permutation(n) for _ in range(P)])
                x = np.zeros((P, n, n), np.int8)
                x[np.arange(P)[:, None], perms, np.arange(n)[None, :]] = 1
                plp = np.array([rng.permutation(n) for _ in range(P)])
                pl = np.zeros_like(x)
                pl[np.arange(P)[:, None], plp, np.arange(n)[None, :]] = 1
                m = P // S
                pgp = np.array([rng.permutation(n) for _ in range(m)])
                pg = np.zeros((m, n, n), np.int8)
                pg[np.arange(m)[:, None], pgp, np.arange(n)[None, :]] = 1
                v = rng.uniform(-4.5, 4.5, (P, n, n))
                v[0, :, 0] = 0.0            # a dead column
                v[-1, 1, :] = -0.0          # negative zeros
                r2 = rng.random(P)
                r3 = rng.random(P)
                out = v.copy()
                _batch.velocity_many(out, x, pl, pg, S, c1, c2 * r2, c3 * r3, 4.0, sv == "norm")
                arrays.update({f"v{k}_in": v, f"v{k}_perm": perms, f"v{k}_plperm": plp,
                               f"v{k}_pgperm": pgp, f"v{k}_r2": r2, f"v{k}_r3": r3,
                               f"v{k}_out": out,
                               f"v{k}_meta": np.array([n, P, S, sv == "norm"], np.int64),
                               f"v{k}_coef": np.array([c1, c2, c3, 4.0])})
                k += 1
    arrays["count"] = np.array(k)
    np.savez_compressed(OUT / "velocity.npz", **arrays)


def gen_aggregate():
    """Batched aggregation on tie-heavy integer V, uniform V, all-zero V,
    replayed draws (the test_kernels.py:262-282 style)."""
    rng = np.random.default_rng(21)
    arrays = {}
    k = 0
    kinds = ["int", "uniform", "zero", "small-int"]
    for mode in ("global-max", "pick-column", "second-target"):
        for kind in kinds:
            for case in range(6):
                n = int(rng.integers(2, 14)) if case < 5 else 64
                if case == 4:
                    n = 33
                p = 7
                perms = np.array([rng.permutation(n) for _ in range(p)])
                x = np.zeros((p, n, n), np.int8)
                x[np.arange(p)[:, None], perms, np.arange(n)[None, :]] = 1
                if kind == "int":
                    v = rng.integers(-2, 3, (p, n, n)).astype(np.float64)
                elif kind == "small-int":
                    v = rng.integers(-1, 1, (p, n, n)).astype(np.float64)
                elif kind == "zero":
                    v = np.zeros((p, n, n))
                else:
                    v = rng.uniform(-1, 1, (p, n, n))
                draws = rng.random((p, 2 * n))
                depth = int(min(int(rng.integers(1, 4)), n - 1))
                out_mat = np.zeros_like(x)
                out_perm = np.zeros((p, n), np.int64)
                _batch.aggregate_many(x, v, _batch.MODE_CODES[mode], depth, draws,
                                      out_mat, out_perm)
                arrays.update({f"a{k}_perm": perms, f"a{k}_v": v, f"a{k}_draws": draws,
                               f"a{k}_out": out_perm,
                               f"a{k}_meta": np.array([_batch.MODE_CODES[mode], depth, n, p])})
                k += 1
    arrays["count"] = np.array(k)
    np.savez_compressed(OUT / "aggregate.npz", **arrays)


def gen_cost(insts):
    arrays = {}
    for name in ("chr12a", "tai30", "float6", "esc32e"):
        inst = insts[name]
        rng = np.random.default_rng(41)
        perms = np.array([rng.permutation(inst.n) for _ in range(40)])
        ct = np.int64 if inst.is_integral else np.float64
        out = np.zeros(40, ct)
        _batch.cost_many(perms, inst.flow, inst.distance, out)
        arrays[f"{name}_perms"] = perms
        arrays[f"{name}_cost"] = out
    np.savez_compressed(OUT / "cost.npz", **arrays)


TRAJ = {
    # name: (instance, config kwargs, coefficient kwargs, iterations)
    "A_chr12a_mig": ("chr12a", dict(swarms=4, swarm_size=10, seed=5, migration_factor=0.25),
                     dict(), 10),
    "B_chr12a_raw_gm": ("chr12a", dict(swarms=3, swarm_size=7, seed=9),
                        dict(c1=0.8, c2=0.5, c3=0.5, sv_mode="raw", sx_mode="global-max"), 12),
    "C_chr12a_pc_mig": ("chr12a", dict(swarms=3, swarm_size=5, seed=3, migration_factor=0.4),
                        dict(sx_mode="pick-column"), 8),
    "D_tai30_st_mig": ("tai30", dict(swarms=5, swarm_size=20, seed=1, migration_factor=0.33),
                       dict(c1=0.8, c2=0.5, c3=0.5, depth=2), 6),
    "E_float6": ("float6", dict(swarms=4, swarm_size=10, seed=5), dict(), 5),
    "F_tiny_gm": ("tiny", dict(swarms=2, swarm_size=3, seed=4), dict(sx_mode="global-max"), 4),
    "G_zero_coeffs": ("chr12a", dict(swarms=4, swarm_size=10, seed=5),
                      dict(c1=0.0, c2=0.0, c3=0.0, sv_mode="raw", sx_mode="global-max"), 2),
    "H_esc32e_st3": ("esc32e", dict(swarms=2, swarm_size=8, seed=7, init_velocity_amplitude=0.25),
                     dict(depth=3, sv_mode="raw"), 5),
    "I_tai50_norm": ("tai50", dict(swarms=4, swarm_size=16, seed=1, migration_factor=0.3),
                     dict(c1=0.8, c2=0.5, c3=0.5), 4),
}


def gen_trajectories(insts):
    meta = {}
    for name, (iname, ckw, kkw, iters) in TRAJ.items():
        inst = insts[iname]
        cfg = qs.SolverConfig(coefficients=qs.PsoCoefficients(**kkw), workers=2, **ckw)
        st = qs.init_population(cfg, inst)
        digs = [digest(st)]
        bests = [[st.best_cost, st.best_iteration]]
        for _ in range(iters):
            qs.step(st, inst, cfg)
            digs.append(digest(st))
            bests.append([st.best_cost, st.best_iteration])
        meta[name] = {
            "instance": iname, "config": ckw, "coefficients": kkw, "iterations": iters,
            "digests": digs, "bests": bests, "best_perm": st.best_perm.tolist(),
            "final_costs": st.cost.tolist(), "pg_costs": st.bests.costs.tolist(),
            "migration_log": [list(e) for e in st.migration_log],
        }
    (OUT / "trajectories.json").write_text(json.dumps(meta, indent=0))


def gen_demo05(insts):
    """pkg/demos/05_statistics.py configuration (demos/05_statistics.py:13-19)."""
    inst = qs.load_bundled("chr12a")
    config = qs.SolverConfig(
        swarms=50, swarm_size=50,
        coefficients=qs.PsoCoefficients(0.5, 0.5, 0.5, sv_mode="norm",
                                        sx_mode="second-target", depth=2),
        max_iterations=80, seed=11, workers=2, pmf_bins=40,
    )
    result = qs.run(config, inst)
    with tempfile.TemporaryDirectory() as d:
        qs.export_csv(result.stats, d)
        qs.write_solution(Path(d) / "solution.txt", inst.n, result.best_cost, result.best_perm)
        stats = (Path(d) / "stats.csv").read_text().splitlines()
        # drop the wall-time column: it is the only non-deterministic field
        stats = [",".join(line.split(",")[:-1]) for line in stats]
        (OUT / "demo05_stats_notime.csv").write_text("\n".join(stats) + "\n")
        (OUT / "demo05_pmf.csv").write_text((Path(d) / "pmf.csv").read_text())
        (OUT / "demo05_solution.txt").write_text((Path(d) / "solution.txt").read_text())


if __name__ == "__main__":
    insts = instances()
    save_instances(insts)
    gen_draws()
    gen_velocity()
    gen_aggregate()
    gen_cost(insts)
    gen_trajectories(insts)
    gen_demo05(insts)
    print("golden fixtures written to", OUT)
