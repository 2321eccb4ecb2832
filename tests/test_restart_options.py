"""Rows a6 (``warm_tau``) and a13 (``criterion="paper51"`` with ``f_star``,
plus the ``subopt`` trace column) against goldens the REAL reference wrote
(tests/golden/make_golden.py --restart-opts -> restart_opts.npz/.json).

Reference paths: engine.py:111-113 (``tau0 = tau_cand`` when ``warm_tau``),
used at restarts.py:129 and :153 and tested by pkg/tests/test_restarts.py:57-65;
diagnostics.py:254-258 (paper51: max(|f - f*| / (1 + |f*|), mean positive
violation) <= eps), diagnostics.py:113 (``subopt_abs = f - f*``) and
restarts.py:120 (``rec.subopt``).

The oracle pin runs on CPU; the ``gpu`` tests run the CUDA path through the
C ABI (``run_restarted``) and compare it with the same goldens.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, analytic_arrays, load_golden
from oracle import rapdb_oracle as O
from paper_2605_29291_b200 import instances

TAU = slice(1, 7)          # tau_start, tau, sigma, gamma, evals_iter, evals_total

with open(os.path.join(GOLDEN, "restart_opts.json")) as fh:
    META = json.load(fh)["cases"]
CASES = sorted(k for k in META if not k.startswith("fstar/"))


@pytest.fixture(scope="module")
def gold():
    return load_golden("restart_opts")


def _arrays(which):
    """(Q, q, r, A, b, lower, upper, mu) of the case's instance."""
    if which == "small":
        g = load_golden("small_qcqp")
        n = g["Q"].shape[1]
        return g["Q"], g["q"], g["r"], np.zeros((0, n)), np.zeros(0), g["lower"], g["upper"], 0.0
    if which == "c0":
        arr = instances.config_instance("C0")
        return arr.Q, arr.q, arr.r, arr.A, arr.b, arr.lower, arr.upper, arr.mu
    a = analytic_arrays(load_golden("analytic"), which)
    return a["Q"], a["q"], a["r"], a["A"], a["b"], a["lower"], a["upper"], a["mu"]


def _criteria(case):
    if case.get("eps") is None:
        return None
    if case.get("criterion", "conic") == "conic":
        return dict(criterion="conic", eps_kkt=case["eps"], eps_feas=case["eps"],
                    f_star=case.get("f_star"))
    return dict(criterion="paper51", eps=case["eps"], f_star=case.get("f_star"))


def _trace(rows):
    nan = np.nan
    return np.array([[r.iter, r.tau_start, r.tau, r.sigma, r.gamma, r.evals_iter, r.evals_total,
                      nan if r.kkt is None else r.kkt, nan if r.infeas is None else r.infeas,
                      nan if r.gap_xi is None else r.gap_xi, r.restart_flag] for r in rows])


def _subopt(rows):
    return np.array([np.nan if r.subopt is None else r.subopt for r in rows])


def _check_subopt(got, want, f_star):
    """Same checkpoints, values within 1e-9 of (1 + |f*|)."""
    np.testing.assert_array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    if f_star is not None:
        np.testing.assert_allclose(got[ok], want[ok], rtol=0, atol=1e-9 * (1 + abs(f_star)))


def _check_against_golden(g, key, case, tr, sub, iterations, converged, restart_iters,
                          x, lam, metrics_f, prefix_only=False):
    tr_g = g[f"{key}/trace"]
    k = min(200, len(tr_g))
    # step sizes / evaluation counts bit-identical over the first 200 iterations
    np.testing.assert_array_equal(tr[:k, TAU], tr_g[:k, TAU])
    if prefix_only:
        return
    assert iterations == int(g[f"{key}/iterations"])
    assert bool(converged) == bool(int(g[f"{key}/converged"]))
    np.testing.assert_array_equal(tr[:, 10], tr_g[:, 10])       # restart flags, every iteration
    np.testing.assert_array_equal(restart_iters, g[f"{key}/restart_iters"])
    _check_subopt(sub, g[f"{key}/subopt"], case.get("f_star"))
    np.testing.assert_allclose(x, g[f"{key}/final_x"], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(lam, g[f"{key}/final_lam"], rtol=1e-6, atol=1e-9)
    f_g = float(g[f"{key}/metrics"][5])
    assert abs(metrics_f - f_g) <= 1e-6 * max(1.0, abs(f_g))


def _oracle_policy(p):
    if p["kind"] == "none":
        return O.Policy()
    if p["kind"] == "fixed":
        return O.Policy(kind="fixed", period=p["period"], point=p.get("point", "last"))
    return O.Policy(kind="adaptive", xi=p.get("xi", 0.04), q=p.get("q", 0.5),
                    warmup=p.get("warmup", 50), check_period=p.get("check_period", 200),
                    point=p.get("point", "last"))


@pytest.mark.parametrize("key", CASES)
def test_oracle_pin_restart_options(gold, key):
    case = META[key]
    Q, q, r, A, b, lo, hi, mu = _arrays(case["instance"])
    P = O.Problem(list(Q), list(q), r, A, b, lo, hi, mu)
    opt = O.Options(mode=case.get("mode", "yx"), nonmonotone=case["nm"])
    res = O.run_restarted(P, opt, _oracle_policy(case["policy"]), budget=case["budget"],
                          criteria=_criteria(case), warm_tau=case.get("warm_tau", False))
    _check_against_golden(gold, key, case, _trace(res.trace), _subopt(res.trace),
                          res.iterations, res.converged, [e[1] for e in res.restarts],
                          res.x, res.lam, res.metrics.f_value)


def test_warm_tau_golden_matches_reference_test(gold):
    """pkg/tests/test_restarts.py:57-65 on the golden traces themselves: after
    the restart at iteration 30 the cold run re-enters at tau_bar, the warm
    run does not."""
    cold, warm = gold["ball/cold_fixed30/trace"], gold["ball/warm_fixed30/trace"]
    assert cold[30, 1] == 1.0
    assert warm[30, 1] != 1.0


# --------------------------------------------------------------------------- GPU


def _policy(R, p):
    if p["kind"] == "none":
        return R.NoRestart()
    if p["kind"] == "fixed":
        return R.FixedRestart(p["period"], point=p.get("point", "last"))
    return R.AdaptiveRestart(xi=p.get("xi", 0.04), q=p.get("q", 0.5), warmup=p.get("warmup", 50),
                             check_period=p.get("check_period", 200), point=p.get("point", "last"))


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
def test_gpu_restart_options(gold, key):
    import paper_2605_29291_b200 as R
    from paper_2605_29291_b200.geometry import Box, NonnegOrthant
    case = META[key]
    Q, q, r, A, b, lo, hi, mu = _arrays(case["instance"])
    Q = np.asarray(Q, float)
    m = Q.shape[0] - 1
    inst = R.ProblemInstance(n=Q.shape[1], m=m, p=A.shape[0], Q=Q, q=np.asarray(q, float), r=r,
                             A=np.asarray(A, float), b=np.asarray(b, float),
                             primal_set=Box(lo, hi), cone=NonnegOrthant(m), mu=mu)
    crit = _criteria(case)
    criteria = None if crit is None else R.TerminationCriteria(**crit)
    cfg = R.SolverConfig(mode=case.get("mode", "yx"), nonmonotone=case["nm"])
    res = R.run_restarted(inst, cfg, _policy(R, case["policy"]), budget=case["budget"],
                          criteria=criteria, warm_tau=case.get("warm_tau", False))
    _check_against_golden(gold, key, case, _trace(res.trace), _subopt(res.trace),
                          res.iterations, res.converged,
                          [e.iteration for e in res.restart_log],
                          res.solution.x, res.solution.lam, res.metrics.f_value)
    if case.get("f_star") is not None:
        g_sub = float(gold[f"{key}/subopt_final"])
        assert abs(res.metrics.subopt_abs - g_sub) <= 1e-6 * (1 + abs(case["f_star"]))
