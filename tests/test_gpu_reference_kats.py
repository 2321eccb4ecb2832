"""The reference's own behavioural tests of the hot path, re-run on the device
path (same assertions as pkg/tests/test_engine.py:79-117,
test_restarts.py:22-42 and test_diagnostics.py:87-89 of the reference, on the
same instances: its conftest random_qcqp(20, 3, seed=3) and the analytic
suite, both stored in tests/golden)."""

import math

import numpy as np
import pytest

from conftest import ANALYTIC_NAMES, analytic_arrays, load_golden
import paper_2605_29291_b200 as R
from test_gpu_parity import inst_from

pytestmark = pytest.mark.gpu

GOLDEN_RATIO = (1 + 5 ** 0.5) / 2


@pytest.fixture(scope="module")
def small_qcqp():
    g = load_golden("small_qcqp")
    return inst_from(g["Q"], g["q"], g["r"], g["lower"], g["upper"])


@pytest.mark.parametrize("mode", ["xy", "yx"])
@pytest.mark.parametrize("nonmonotone", [False, True])
def test_stepsize_laws(small_qcqp, mode, nonmonotone):            # test_engine.py:79-97
    cfg = R.SolverConfig(mode=mode, nonmonotone=nonmonotone)
    avg, last, trace, eng = R.run(small_qcqp, cfg, R.initial_iterate(small_qcqp), 200)
    taus = [r.tau for r in trace]
    if not nonmonotone:
        for k in range(len(taus) - 1):
            assert taus[k + 1] <= taus[k] + 1e-15
            assert abs(trace[k + 1].tau_start - taus[k]) <= 1e-15
    else:
        for k in range(len(taus) - 1):
            assert taus[k + 1] / taus[k] <= GOLDEN_RATIO + 1e-12
            prev = taus[k - 1] if k > 0 else trace[0].tau_start
            expect = taus[k] * math.sqrt(1.0 + taus[k] / prev)
            assert abs(trace[k + 1].tau_start - expect) <= 1e-12


def test_eval_counter_identity(small_qcqp):                       # test_engine.py:108-117
    for mode in ("xy", "yx"):
        for nm in (False, True):
            cfg = R.SolverConfig(mode=mode, nonmonotone=nm)
            _, _, trace, eng = R.run(small_qcqp, cfg, R.initial_iterate(small_qcqp), 150)
            eta = cfg.resolved().eta
            recon = sum(1 + round(math.log(r.tau_start / r.tau) / math.log(1.0 / eta)) for r in trace)
            assert recon == eng.evals_total


def test_no_restart_is_passthrough(small_qcqp):                   # test_restarts.py:22-32
    cfg = R.SolverConfig(mode="yx", nonmonotone=True)
    z0 = R.initial_iterate(small_qcqp)
    _, last, trace, _ = R.run(small_qcqp, cfg, z0, 120)
    res = R.run_restarted(small_qcqp, cfg, R.NoRestart(), z_init=z0, budget=120)
    assert len(res.trace) == len(trace)
    for a, b in zip(trace, res.trace):
        assert a.tau == b.tau and a.sigma == b.sigma
        assert a.evals_total == b.evals_total
    np.testing.assert_array_equal(last.x, res.solution.x)
    np.testing.assert_array_equal(last.lam, res.solution.lam)


def _analytic(name):
    return inst_from(**analytic_arrays(load_golden("analytic"), name))


def test_fixed_restart_bookkeeping():                             # test_restarts.py:35-42
    inst = _analytic("ball")
    res = R.run_restarted(inst, R.SolverConfig(mode="yx"), R.FixedRestart(5), budget=23)
    assert [e.iteration for e in res.restart_log] == [5, 10, 15, 20]
    assert [e.outer for e in res.restart_log] == [1, 2, 3, 4]
    assert [r.iter for r in res.trace if r.restart_flag] == [5, 10, 15, 20]


@pytest.mark.parametrize("name", ANALYTIC_NAMES)
def test_kkt_zero_at_analytic_solutions(name):                    # test_diagnostics.py:87-89
    g = load_golden("analytic")
    inst = _analytic(name)
    z = R.Iterate(g[f"{name}/x_star"], g[f"{name}/v_star"], g[f"{name}/lam_star"])
    assert R.kkt_residual(inst, z).kkt_residual <= 1e-9
