"""The draw pre-pass folded into the previous step's best update
(qsb_best_update_next + QSB_HINT_COEF_READY): the coefficients it leaves in
step_coef are the ones coef_kernel would draw, a change of c2 / c3 / seed
between steps falls back to the pre-pass, and eager steps, graph replays
and the C-ABI sequence agree with the pre-pass path bit for bit."""

import dataclasses
import time

import numpy as np
import pytest

from conftest import cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

import torch                                    # noqa: E402

import paper_1504_05158_b200 as qsb            # noqa: E402
from paper_1504_05158_b200 import engine        # noqa: E402
from oracle import oracle as orc                # noqa: E402


def _state_bytes(st):
    torch.cuda.synchronize()
    return (st.d_V.cpu().numpy().tobytes(), st.d_perm.cpu().numpy().tobytes(),
            st.d_pl_perm.cpu().numpy().tobytes(), st.d_cost.cpu().numpy().tobytes(),
            st.d_pg_perm.cpu().numpy().tobytes(), st.best_cost)


def test_coefficient_change_between_steps_matches_oracle(golden_instances):
    """c2 / c3 change after step 3 and the seed after step 6: the folded
    draws of the old coefficients are discarded (fp64 parity mode against
    the oracle, which draws every step from scratch)."""
    inst = golden_instances["tai30"]
    base = qsb.SolverConfig(swarms=6, swarm_size=10, seed=3, migration_factor=0.34,
                            coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    cfgs = [base,
            dataclasses.replace(base, coefficients=qsb.PsoCoefficients(0.8, 0.7, 0.3)),
            dataclasses.replace(base, seed=11, coefficients=qsb.PsoCoefficients(0.8, 0.7, 0.3))]
    st = qsb.init_population(base, inst)
    ost = orc.init_population(6, 10, inst.n, inst.flow, inst.distance, seed=3)
    for t in range(9):
        cfg = cfgs[t // 3]
        qsb.step(st, inst, cfg)
        orc.step(ost, inst.flow, inst.distance, **orc.coeff_kwargs(cfg))
        assert np.array_equal(st.perms, ost.perms), f"step {t + 1}"
        assert st.V.tobytes() == np.ascontiguousarray(ost.V).tobytes(), f"step {t + 1}"


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_fold_equals_prepass(precision, golden_instances):
    """The same run with the fold (default) and with the pre-pass forced
    before every step (coef_ready cleared): identical device state."""
    inst = golden_instances["tai50"]
    cfg = qsb.SolverConfig(swarms=8, swarm_size=25, seed=5, precision=precision, init="device",
                           migration_factor=0.33, migration_period=4,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    a = qsb.init_population(cfg, inst)
    b = qsb.init_population(cfg, inst)
    for t in range(12):
        qsb.step(a, inst, cfg)
        b.coef_ready = None
        qsb.step(b, inst, cfg)
        assert _state_bytes(a) == _state_bytes(b), f"step {t + 1}"


def test_graph_replay_with_fold_equals_eager(golden_instances):
    """step_many (graphs captured with QSB_HINT_COEF_READY and the folded best
    update) against eager steps with the pre-pass forced."""
    inst = golden_instances["tai50"]
    cfg = qsb.SolverConfig(swarms=8, swarm_size=25, seed=9, precision="fp32", init="device",
                           migration_factor=0.33, migration_period=5,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    a = qsb.init_population(cfg, inst)
    b = qsb.init_population(cfg, inst)
    qsb.engine.step_many(a, inst, cfg, 23)
    for _ in range(23):
        b.coef_ready = None
        qsb.step(b, inst, cfg)
    assert a.t == b.t == 23
    assert _state_bytes(a) == _state_bytes(b)


def test_c_abi_best_update_next_leaves_prepass_coefficients(golden_instances):
    """qsb_best_update_next writes exactly the pre-pass's (c2 r2, c3 r3) for
    the next iteration -- the reference draw stream times c2, c3 -- and zeroes
    the particle counter."""
    inst = golden_instances["tai30"]
    cfg = qsb.SolverConfig(swarms=4, swarm_size=16, seed=21, precision="fp32", init="device",
                           coefficients=qsb.PsoCoefficients(0.8, 0.45, 0.65))
    st = qsb.init_population(cfg, inst)
    for _ in range(3):
        qsb.step(st, inst, cfg)
    torch.cuda.synchronize()
    folded = st.d_step_coef.clone()
    assert st.coef_ready == engine._coef_key(cfg, st.t + 1)
    assert int(st.d_work.item()) == 0
    # the reference draw stream (streams.step_draws restated): columns 0 and
    # 1 of a particle's row are r2, r3 of iteration t + 1
    draws = orc.step_draws(cfg.seed, st.t + 1, cfg.num_particles, inst.n)
    c = folded.cpu().numpy()
    assert np.array_equal(c[:, 0], 0.45 * draws[:, 0])
    assert np.array_equal(c[:, 1], 0.65 * draws[:, 1])


@pytest.mark.parametrize("n", [34, 50, 64])
def test_late_kernel_variant_equals_default(n):
    """QSB_HINT_LATE selects the fused-kernel variant that chains bulk steps
    against stale column maxima; its results must equal the default kernel's
    bit for bit.  300 iterations (where bulk steps leave more than five free
    columns often) with the variant from iteration 1 against the default."""
    inst = qsb.taillard_uniform(n)
    cfg = qsb.SolverConfig(swarms=20, swarm_size=100, seed=3, precision="fp32", init="device",
                           migration_factor=0.33, migration_period=10,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    saved = engine._CHAIN_T0
    try:
        engine._CHAIN_T0 = 1
        a = qsb.init_population(cfg, inst)
        engine.step_many(a, inst, cfg, 300)
        engine._CHAIN_T0 = 1 << 40
        b = qsb.init_population(cfg, inst)
        engine.step_many(b, inst, cfg, 300)
    finally:
        engine._CHAIN_T0 = saved
    assert a.t == b.t == 300
    assert _state_bytes(a) == _state_bytes(b)
    assert a.best_perm.tolist() == b.best_perm.tolist()


def test_step_many_switches_to_late_variant_mid_call():
    """step_many picks the late variant per graph replay (QSB_HINT_LATE from
    _CHAIN_T0 on), caching both graphs: a call that crosses the threshold
    equals eager steps."""
    inst = qsb.taillard_uniform(50)
    cfg = qsb.SolverConfig(swarms=10, swarm_size=100, seed=5, precision="fp32", init="device",
                           migration_factor=0.33, migration_period=5,
                           coefficients=qsb.PsoCoefficients(0.8, 0.5, 0.5))
    saved = engine._CHAIN_T0
    try:
        engine._CHAIN_T0 = 23
        a = qsb.init_population(cfg, inst)
        engine.step_many(a, inst, cfg, 47)
        engine.step_many(a, inst, cfg, 20)          # both graphs cached now
        b = qsb.init_population(cfg, inst)
        for _ in range(67):
            qsb.step(b, inst, cfg)
    finally:
        engine._CHAIN_T0 = saved
    assert a.t == b.t == 67
    assert _state_bytes(a) == _state_bytes(b)
    assert [tuple(e) for e in a.migration_log] == [tuple(e) for e in b.migration_log]


def test_stream_gate_holds_and_times_out():
    """qsb_stream_gate (bench.py's timed-window gate): work queued behind it
    waits for the host flag; an unreleased gate gives up after its timeout
    and reports it."""
    from paper_1504_05158_b200 import _lib
    s = torch.cuda.current_stream()
    flag = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    to = torch.zeros(1, dtype=torch.int32, pin_memory=True)
    x = torch.zeros(1, device="cuda")
    x += 1                          # the add kernel loaded now: lazy module
    x -= 1                          # loading inside the gate would block the host
    torch.cuda.synchronize()
    _lib.call("qsb_stream_gate", flag.data_ptr(), int(5e9), to.data_ptr(), s.cuda_stream)
    x += 1
    ev = torch.cuda.Event()
    ev.record(s)
    time.sleep(0.05)
    assert not ev.query(), (int(to[0]), int(flag[0]))          # held
    flag[0] = 1
    ev.synchronize()
    assert int(to[0]) == 0 and float(x.item()) == 1.0
    flag[0] = 0
    _lib.call("qsb_stream_gate", flag.data_ptr(), int(2e6), to.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    assert int(to[0]) == 1
