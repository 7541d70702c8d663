"""CPU tests of the host layer: config validation (the reference's messages),
statistics and CSV output (pinned to the reference's golden demo run via the
oracle trajectory), instances, migration picks and the C ABI surface."""

import ctypes
import re
import tempfile
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

import paper_1504_05158_b200 as qsb
from paper_1504_05158_b200 import _lib, engine, stats
from oracle import oracle as orc


# ---------------------------------------------------------------- configs
def test_coefficient_validation_messages():
    # the reference's test_kernels.py:31-41 message substrings
    with pytest.raises(ValueError, match="c1"):
        qsb.PsoCoefficients(c1=1.2)
    with pytest.raises(ValueError, match="v_max"):
        qsb.PsoCoefficients(v_max=0)
    with pytest.raises(ValueError, match="sv_mode"):
        qsb.PsoCoefficients(sv_mode="soft")
    with pytest.raises(ValueError, match="sx_mode"):
        qsb.PsoCoefficients(sx_mode="argmax")
    with pytest.raises(ValueError, match="depth"):
        qsb.PsoCoefficients(depth=0)


def test_config_validation_messages():
    base = dict(swarms=4, swarm_size=10, max_iterations=10, seed=5, workers=2)
    with pytest.raises(ValueError, match="migration_factor"):
        qsb.SolverConfig(**{**base, "migration_factor": 0.5})
    with pytest.raises(ValueError, match="positive"):
        qsb.SolverConfig(**{**base, "swarms": 0})
    with pytest.raises(ValueError, match="workers"):
        qsb.SolverConfig(**{**base, "workers": 0})
    with pytest.raises(ValueError, match="stats_stride"):
        qsb.SolverConfig(**{**base, "stats_stride": 0})
    with pytest.raises(ValueError, match="migration_period"):
        qsb.SolverConfig(**{**base, "migration_period": 0})
    with pytest.raises(ValueError, match="precision"):
        qsb.SolverConfig(**{**base, "precision": "bf16"})
    with pytest.raises(ValueError, match="init"):
        qsb.SolverConfig(**{**base, "init": "gpu"})


def test_config_defaults_match_reference():
    c = qsb.PsoCoefficients()
    assert (c.c1, c.c2, c.c3, c.v_max, c.sv_mode, c.sx_mode, c.depth) == \
        (0.5, 0.5, 0.5, 4.0, "norm", "second-target", 2)
    s = qsb.SolverConfig(swarms=800, swarm_size=100, migration_factor=0.33)
    assert s.num_particles == 80000 and s.migration_depth == 264
    assert (s.max_iterations, s.seed, s.stats_stride, s.pmf_bins) == (200, 0, 1, 60)
    assert (s.migration_period, s.precision, s.init) == (1, "fp64", "reference")


def test_projected_buffer_bytes_reference_formula():
    cfg = qsb.SolverConfig(swarms=4, swarm_size=10)
    n, p = 12, 40
    expect = 3 * p * n * n + p * n * n * 8 + 3 * p * n * 8 + 3 * p * 8 + 4 * (n * n + n * 8 + 8)
    assert qsb.projected_buffer_bytes(cfg, n) == expect
    # the device layout is far smaller: int16 permutations, no 0/1 matrices
    assert qsb.device_buffer_bytes(cfg, n) < expect


# -------------------------------------------------------------- instances
def test_taillard_generator_matches_golden(golden_instances):
    for n in (30, 50):
        inst = qsb.taillard_uniform(n)
        g = golden_instances[f"tai{n}"]
        assert np.array_equal(inst.flow, g.flow) and np.array_equal(inst.distance, g.distance)
        assert (inst.flow == inst.flow.T).all() and (np.diag(inst.flow) == 0).all()


def test_parse_instance_roundtrip_and_errors(golden_instances):
    tiny = qsb.parse_instance("2  0 1  1 0   0 3  3 0", name="tiny")
    assert tiny.n == 2 and tiny.is_integral and tiny.flow.tolist() == [[0, 1], [1, 0]]
    with pytest.raises(ValueError, match="tokens"):
        qsb.parse_instance("2 0 1 1")
    with pytest.raises(ValueError, match="negative"):
        qsb.QapInstance("bad", 2, np.array([[0, -1], [1, 0]]), np.zeros((2, 2)))
    f = qsb.parse_instance("2 0 1.5 1 0 0 3 3 0")
    assert not f.is_integral


def test_device_format_selection():
    from paper_1504_05158_b200.instance import device_format
    inst = qsb.taillard_uniform(20)
    assert device_format(inst)[2] == _lib.U16
    wide = qsb.QapInstance("w", 3, np.full((3, 3), 70000), np.ones((3, 3), np.int64))
    assert device_format(wide)[2] == _lib.I64
    fl = qsb.QapInstance("f", 3, np.full((3, 3), 0.5), np.ones((3, 3)))
    assert device_format(fl)[2] == _lib.F64


# ------------------------------------------------------------- statistics
def test_percentile_nearest_rank():
    vals = [15, 20, 35, 40, 50]
    assert [stats.percentile(vals, r) for r in (5, 30, 40, 50, 100 - 1e-9)] == [15, 20, 20, 35, 50]
    with pytest.raises(ValueError, match="empty"):
        stats.percentile([], 50)
    with pytest.raises(ValueError, match="rank"):
        stats.percentile([1], 100)


def test_pmf_folds_out_of_range():
    edges, freq = stats.pmf([-5, 0, 1, 2, 10], 2, 0.0, 2.0)
    assert edges.tolist() == [0.0, 1.0, 2.0]
    assert freq.tolist() == [0.4, 0.6]
    with pytest.raises(ValueError, match="range"):
        stats.pmf([1], 2, 1.0, 1.0)


class _OracleView:
    """The oracle state seen through the attributes stats.collect reads."""

    def __init__(self, st):
        self.st = st

    def __getattr__(self, k):
        return getattr(self.st, k)

    @property
    def bests(self):
        return qsb.SwarmBestTable(self.st.pg_mats, self.st.pg_perms, self.st.pg_costs)


def test_stats_and_csv_reproduce_reference_golden_run(golden_instances):
    """demos/05_statistics.py configuration: the oracle trajectory fed to this
    package's collect/export_csv/write_solution reproduces the reference's
    stats.csv (minus wall time), pmf.csv and solution.txt byte for byte."""
    inst = golden_instances["chr12a"]
    cfg = qsb.SolverConfig(swarms=50, swarm_size=50, max_iterations=80, seed=11, workers=2,
                           pmf_bins=40,
                           coefficients=qsb.PsoCoefficients(0.5, 0.5, 0.5, sv_mode="norm",
                                                            sx_mode="second-target", depth=2))
    st = orc.init_population(50, 50, 12, inst.flow, inst.distance, seed=11)
    view = _OracleView(st)
    series = [stats.collect(view, 0.0, bins=40)]
    kw = orc.coeff_kwargs(cfg)
    for _ in range(80):
        orc.step(st, inst.flow, inst.distance, **kw)
        series.append(stats.collect(view, 0.0, bins=40))
    with tempfile.TemporaryDirectory() as d:
        stats.export_csv(series, d)
        stats.write_solution(Path(d) / "solution.txt", 12, st.best_cost, st.best_perm)
        rows = [",".join(r.split(",")[:-1]) for r in (Path(d) / "stats.csv").read_text().splitlines()]
        assert "\n".join(rows) + "\n" == (GOLDEN / "demo05_stats_notime.csv").read_text()
        assert (Path(d) / "pmf.csv").read_text() == (GOLDEN / "demo05_pmf.csv").read_text()
        assert (Path(d) / "solution.txt").read_text() == (GOLDEN / "demo05_solution.txt").read_text()


def test_collect_all_swarms_shape(golden_instances):
    inst = golden_instances["chr12a"]
    st = orc.init_population(3, 4, 12, inst.flow, inst.distance, seed=2)
    s = stats.collect(_OracleView(st), 1.0, bins=5, all_swarms=True)
    assert s.all_swarm_percentiles.shape == (3, 4)
    assert s.best_swarm == int(np.argmin(st.pg_costs))


# ------------------------------------------------------------- migration
def test_device_picks_algorithm_matches_reference_host_stream():
    """migrate_kernel's in-kernel donor draw (Lemire over the Philox halves,
    restated in oracle.lemire_picks) equals the reference's scalar
    rng.integers(0, S) calls: golden vectors plus random keys, including a
    swarm size whose rejection threshold is non-zero and a wrapped seed."""
    g = np.load(GOLDEN / "draws.npz")
    for i, (seed, t, S, d) in enumerate([(1, 10, 100, 264), (3, 5, 20, 16), (5, 1, 10, 1)]):
        assert np.array_equal(orc.lemire_picks(seed, t, d, S), g[f"host{i}"])
    rng = np.random.default_rng(0)
    for _ in range(20):
        seed = int(rng.integers(-2**40, 2**40))
        t = int(rng.integers(0, 2**32))
        S = int(rng.choice([1, 2, 3, 7, 100, 1000, 65535, 65536, 3 * 2**20 + 1]))
        d = int(rng.integers(1, 300))
        assert np.array_equal(orc.lemire_picks(seed, t, d, S), orc.migration_picks(seed, t, d, S))


def test_migrate_validation_messages():
    t = qsb.SwarmBestTable(np.zeros((4, 3, 3), np.int8), np.zeros((4, 3), np.int64),
                           np.arange(4, dtype=np.int64))
    perms = np.zeros((8, 3), np.int64)
    with pytest.raises(ValueError, match="m/2"):
        qsb.migrate(2, t, perms, None, np.zeros(8, np.int64), 2, np.random.default_rng(0))
    with pytest.raises(ValueError, match="population"):
        qsb.migrate(1, t, perms[:6], None, np.zeros(6, np.int64), 2, np.random.default_rng(0))
    assert qsb.migrate(0, t, perms, None, np.zeros(8, np.int64), 2, np.random.default_rng(0)) == []


# ------------------------------------------------------------------- C ABI
def _header_functions():
    text = (ROOT / "include" / "qapswarm_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qsb_[a-z0-9_]+)\s*\(", text)))


def test_c_abi_library_exports_every_header_symbol():
    L = ctypes.CDLL(str(_lib.LIB_PATH))
    names = _header_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(L, name), f"{name} declared in include/qapswarm_b200.h but not exported"
    assert set(names) == set(_lib.SIGNATURES), "ctypes signatures out of sync with the header"


def test_c_abi_pure_helpers_without_gpu():
    L = _lib.lib()
    assert L.qsb_version() >= 10000
    assert L.qsb_vstride(13, _lib.F32) == 172 and L.qsb_vstride(13, _lib.F64) == 170
    assert L.qsb_vstride(50, _lib.F32) == 2500
    assert L.qsb_strerror(_lib.QSB_EINVAL) == b"invalid argument"
    # argument validation fails before touching the device
    assert L.qsb_step_phases(None, None, None, 0, None, 0, 0, None, 0, None) == _lib.QSB_EINVAL
    assert L.qsb_velocity_many(None, None, None, None, 1, 4, 1, 0.5, None, None, 4.0, 1) == _lib.QSB_EINVAL


def test_ctypes_struct_layouts_match_header():
    """Field offsets and sizes of the ctypes mirrors equal the C structs of
    include/qapswarm_b200.h, as compiled by the host C compiler."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"qsb_state": _lib.QsbState, "qsb_instance": _lib.QsbInstance,
               "qsb_coeffs": _lib.QsbCoeffs, "qsb_migration": _lib.QsbMigration,
               "qsb_host_population": _lib.QsbHostPopulation,
               "qsb_host_instance": _lib.QsbHostInstance}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "qapswarm_b200.h"',
             "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    with tempfile.TemporaryDirectory() as d:
        src = Path(d) / "layout.c"
        src.write_text("\n".join(lines))
        exe = Path(d) / "layout"
        subprocess.run([cc, "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
        out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for cname, py in structs.items():
        assert int(got[f"{cname} size"]) == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, f"{cname}.{fname}"


def test_wide_velocity_words_roundtrip():
    """The lazily scaled layout's wide words (high word of the double,
    rounded to nearest): relative error <= 2^-21, the raw words order like
    the values under float compares, no flush to zero over fp64's range."""
    import torch
    from paper_1504_05158_b200.engine import wide_decode, wide_encode
    rng = np.random.default_rng(5)
    mag = 2.0 ** rng.uniform(-1000, 120, 20000)
    v = torch.from_numpy(np.where(rng.random(20000) < 0.5, -mag, mag))
    w = wide_encode(v)
    back = wide_decode(w)
    rel = ((back - v).abs() / v.abs()).max().item()
    assert rel <= 2.0 ** -21
    assert (back != 0).all()                       # 2^-1000 survives (fp32 would flush)
    # exactly representable values round-trip bit for bit
    assert torch.equal(wide_decode(wide_encode(back)), back)
    # float compares of the raw words order like the values
    i = torch.randperm(20000)
    j = torch.randperm(20000)
    assert torch.equal(w[i] > w[j], back[i] > back[j])
    assert torch.equal(w[i] == w[j], back[i] == back[j])
    # signed zeros compare equal, as in the double domain
    z = wide_encode(torch.tensor([0.0, -0.0], dtype=torch.float64))
    assert z[0] == z[1]


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` runs on the host cores alone (the oracle
    port; no GPU) and prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--n", "12", "--swarms", "80"],
                         capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
