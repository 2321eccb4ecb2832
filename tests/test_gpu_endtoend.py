"""End-of-run parity at the configurations the bench times (BASELINE.json
north_star bars), against goldens the REAL reference (C1) or the pinned
factored restatement (C3f) wrote offline:

* accepted step sizes / evaluation counts / restart points identical while
  the runs coincide (here: over the whole run), iterates within 1e-9 over
  the first 200 iterations;
* final KKT residual, infeasibility and objective within 1e-6 relative;
* total iteration counts within 2 %.

Reference: restarts.py:111-170 (loop, KKT cadence, fixed / adaptive restart),
diagnostics.py:96-113 (metrics), engine.py:198-259 (step).
Goldens: tests/golden/make_golden.py --c1-kkt (c1_kkt.npz),
tests/golden/make_c3f_golden.py (c3f_full.npz).
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from test_gpu_parity import TAU, crit, rel, trace_arr

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _end_bars(res, g, key):
    """The north_star end-of-run bars of one run_restarted result."""
    tr_g = g[f"{key}/trace"]
    tr = trace_arr(res.trace)
    it_g = int(g[f"{key}/iterations"])
    assert abs(res.iterations - it_g) <= 0.02 * it_g, (res.iterations, it_g)
    assert bool(res.converged) == bool(int(g[f"{key}/converged"]))
    k = min(len(tr), len(tr_g))
    np.testing.assert_array_equal(tr[:k, TAU], tr_g[:k, TAU])          # tau, sigma, gamma, evals
    np.testing.assert_array_equal(tr[:k, 10], tr_g[:k, 10])            # restart flags
    np.testing.assert_array_equal([e.iteration for e in res.restart_log], g[f"{key}/restart_iters"])
    met = g[f"{key}/metrics"]
    m = res.metrics
    for got, want in ((m.kkt_residual, met[0]), (m.infeas, met[4]), (m.f_value, met[5])):
        assert abs(got - want) <= 1e-6 * max(abs(want), 1e-300) or abs(got - want) <= 1e-12, (got, want)
    # KKT checkpoints along the run (every metrics_every iterations)
    ok = ~np.isnan(tr_g[:k, 7])
    np.testing.assert_allclose(tr[:k, 7][ok], tr_g[:k, 7][ok], rtol=1e-6)


@pytest.fixture(scope="module")
def c1():
    g = load_golden("c1_kkt")
    arr = instances.config_instance("C1")
    np.testing.assert_allclose([float(np.sum(arr.Q[i])) for i in range(0, arr.m + 1, 20)],
                               g["Q_checksum"][::20], rtol=1e-12)
    return g, R.ProblemInstance.from_arrays(arr, validate=False)


def test_c1_bench_config_to_kkt(c1):
    """The bench workload itself: C1, yx monotone + FixedRestart(500) to conic
    KKT 1e-6 -- the reference takes 570 iterations with a restart at 500."""
    g, inst = c1
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.FixedRestart(500),
                          budget=3000, criteria=crit(1e-6))
    _end_bars(res, g, "mono_fixed500")
    assert rel(res.solution.x, g["mono_fixed500/final_x"]) <= 1e-6
    assert rel(res.solution.lam, g["mono_fixed500/final_lam"]) <= 1e-6
    assert rel(res.average.x, g["mono_fixed500/avg_x"]) <= 1e-6


def test_c1_bench_config_iterates(c1):
    """Iterates of the same run at the golden's snapshots (the fixed restart at
    500 included): within 1e-9 over the first 200 iterations, 1e-6 after."""
    g, inst = c1
    key = "mono_fixed500"
    snaps = [int(k) for k in g[f"{key}/snap_iters"]]
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.initial_iterate(inst))
    done = 0
    for idx, k in enumerate(snaps):
        if k > 500 and done <= 500:          # FixedRestart(500): restart from the last iterate
            eng.run_block(500 - done)
            done = 500
            eng.reinit(eng.last)
        eng.run_block(k - done)
        done = k
        bar = 1e-9 if k <= 200 else 1e-6
        assert rel(eng.last.x, g[f"{key}/snap_x"][idx]) <= bar, k
        assert rel(eng.last.lam, g[f"{key}/snap_lam"][idx]) <= bar, k
    np.testing.assert_array_equal(trace_arr(eng.trace)[:, TAU], g[f"{key}/trace"][:done, TAU])


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c1_kkt.npz")) or
                    "mono_ada/trace" not in np.load(os.path.join(GOLDEN, "c1_kkt.npz")).files,
                    reason="C1 adaptive golden not generated")
def test_c1_adaptive_to_kkt(c1):
    g, inst = c1
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=False),
                          R.AdaptiveRestart(xi=0.04, q=0.5, warmup=50, check_period=200),
                          budget=3000, criteria=crit(1e-6))
    _end_bars(res, g, "mono_ada")
    gaps = g["mono_ada/trace"][:, 9]
    got = trace_arr(res.trace)[:, 9]
    ok = ~np.isnan(gaps)
    np.testing.assert_allclose(got[:len(gaps)][ok], gaps[ok], rtol=1e-6, atol=1e-12)
