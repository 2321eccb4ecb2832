"""Pin the CPU oracle against the golden traces the REAL reference produced
(tests/golden/make_golden.py).  Same machine as the fixture generation ->
bit-for-bit; elsewhere (different BLAS kernels) -> tight tolerances, with the
first 200 accepted step sizes still required to be identical."""

import numpy as np
import pytest

from conftest import ANALYTIC_NAMES, analytic_arrays
from oracle import rapdb_oracle as O
from paper_2605_29291_b200 import instances

TRACE_TAU = slice(1, 7)   # tau_start, tau, sigma, gamma, evals_iter, evals_total


def _policy(kind, **kw):
    return O.Policy(kind=kind, **kw)


def _run(P, mode, nm, policy, budget, eps=None, ball=None, snaps=None):
    opt = O.Options(mode=mode, nonmonotone=nm, ball=ball or O.Ball())
    crit = None if eps is None else dict(criterion="conic", eps_kkt=eps, eps_feas=eps)
    cap = {}

    def hook(total, eng):
        if snaps is not None and eng.iters in snaps:
            cap[eng.iters] = (eng.x.copy(), eng.lam.copy())
    res = O.run_restarted(P, opt, policy, budget=budget, criteria=crit, on_iter=hook)
    return res, cap


def _trace(res):
    nan = np.nan
    return np.array([[r.iter, r.tau_start, r.tau, r.sigma, r.gamma, r.evals_iter, r.evals_total,
                      nan if r.kkt is None else r.kkt, nan if r.infeas is None else r.infeas,
                      nan if r.gap_xi is None else r.gap_xi, r.restart_flag] for r in res.trace])


def _check_prefix(tr_o, tr_g, k=200):
    k = min(k, len(tr_g))
    np.testing.assert_array_equal(tr_o[:k, TRACE_TAU], tr_g[:k, TRACE_TAU])


SMALL_CASES = {
    "yx_mono": dict(mode="yx", nm=False, policy=("none", {}), budget=200),
    "yx_nm": dict(mode="yx", nm=True, policy=("none", {}), budget=200),
    "xy_mono": dict(mode="xy", nm=False, policy=("none", {}), budget=200),
    "xy_nm": dict(mode="xy", nm=True, policy=("none", {}), budget=200),
    "yx_nm_joint5": dict(mode="yx", nm=True, policy=("none", {}), budget=200, ball=O.Ball(1, 5.0)),
    "yx_nm_split": dict(mode="yx", nm=True, policy=("none", {}), budget=150, ball=O.Ball(2, 1.0, 0.7)),
    "yx_nm_fixed40avg": dict(mode="yx", nm=True, policy=("fixed", dict(period=40, point="average")),
                             budget=200),
    "yx_nm_ada": dict(mode="yx", nm=True, policy=("adaptive", dict(warmup=50, check_period=100)),
                      budget=1500, eps=1e-8),
}


@pytest.mark.parametrize("key", list(SMALL_CASES))
def test_oracle_matches_reference_small_qcqp(golden_small, key):
    g = golden_small
    P = O.Problem(list(g["Q"]), list(g["q"]), g["r"], np.zeros((0, 20)), np.zeros(0),
                  g["lower"], g["upper"])
    c = SMALL_CASES[key]
    kind, kw = c["policy"]
    res, _ = _run(P, c["mode"], c["nm"], _policy(kind, **kw), c["budget"], c.get("eps"),
                  c.get("ball"))
    tr_g = g[f"{key}/trace"]
    tr_o = _trace(res)
    _check_prefix(tr_o, tr_g)
    assert len(tr_o) == len(tr_g)
    np.testing.assert_allclose(res.x, g[f"{key}/final_x"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(res.lam, g[f"{key}/final_lam"], rtol=1e-9, atol=1e-12)
    np.testing.assert_array_equal([e[1] for e in res.restarts], g[f"{key}/restart_iters"])


@pytest.mark.parametrize("name", ANALYTIC_NAMES)
@pytest.mark.parametrize("key", ["nm_fixed500", "mono_fixed5", "xy_nm"])
def test_oracle_matches_reference_analytic(golden_analytic, name, key):
    g = golden_analytic
    a = analytic_arrays(g, name)
    P = O.Problem(list(a["Q"]), list(a["q"]), a["r"], a["A"], a["b"], a["lower"], a["upper"], a["mu"])
    spec = {"nm_fixed500": ("yx", True, _policy("fixed", period=500), 5000, 1e-7),
            "mono_fixed5": ("yx", False, _policy("fixed", period=5), 23, None),
            "xy_nm": ("xy", True, _policy("none"), 300, None)}[key]
    res, _ = _run(P, spec[0], spec[1], spec[2], spec[3], spec[4])
    pre = f"{name}/{key}/"
    tr_g = g[pre + "trace"]
    _check_prefix(_trace(res), tr_g, k=len(tr_g))
    np.testing.assert_allclose(res.x, g[pre + "final_x"], rtol=1e-9, atol=1e-13)
    met = g[pre + "metrics"]
    assert abs(res.metrics.kkt_residual - met[0]) <= 1e-9 * max(1.0, abs(met[0]))


def test_oracle_analytic_kats(golden_analytic):
    """KKT <= 1e-9 at the hand-verified solutions (test_diagnostics.py:87-89)."""
    g = golden_analytic
    for name in ANALYTIC_NAMES:
        a = analytic_arrays(g, name)
        P = O.Problem(list(a["Q"]), list(a["q"]), a["r"], a["A"], a["b"], a["lower"], a["upper"], a["mu"])
        met = O.kkt(P, g[f"{name}/x_star"], g[f"{name}/v_star"], g[f"{name}/lam_star"])
        assert met.kkt_residual <= 1e-9
        assert abs(met.f_value - float(g[f"{name}/f_star"])) <= 1e-12


def test_generator_matches_reference_c0(golden_c0):
    arr = instances.config_instance("C0")
    g = golden_c0
    np.testing.assert_array_equal(arr.Q[:, :3, :5], g["Q_sample"])
    np.testing.assert_allclose([float(np.sum(arr.Q[i])) for i in range(arr.m + 1)],
                               g["Q_checksum"], rtol=1e-12)
    P = O.Problem.from_arrays(arr)
    x = g["probe_x"]
    np.testing.assert_allclose(P.g(x), g["probe_g"], rtol=1e-13)
    assert abs(P.f(x) - float(g["probe_f"])) <= 1e-13 * abs(float(g["probe_f"]))


@pytest.mark.parametrize("key", ["mono_none", "nm_fixed500", "mono_ada", "xy_nm_none"])
def test_oracle_matches_reference_c0(golden_c0, key):
    arr = instances.config_instance("C0")
    P = O.Problem.from_arrays(arr)
    spec = {"mono_none": ("yx", False, _policy("none"), 50000, 1e-6),
            "nm_fixed500": ("yx", True, _policy("fixed", period=500), 50000, 1e-6),
            "mono_ada": ("yx", False, _policy("adaptive"), 50000, 1e-6),
            "xy_nm_none": ("xy", True, _policy("none"), 200, None)}[key]
    res, cap = _run(P, *spec, snaps={1, 10, 100, 200})
    g = golden_c0
    tr_g = g[f"{key}/trace"]
    tr_o = _trace(res)
    _check_prefix(tr_o, tr_g)
    snaps = list(g[f"{key}/snap_iters"])
    for k, (x, lam) in cap.items():
        idx = snaps.index(k)
        np.testing.assert_allclose(x, g[f"{key}/snap_x"][idx], rtol=1e-9, atol=1e-12)
    assert res.iterations == int(g[f"{key}/iterations"])
    np.testing.assert_array_equal([e[1] for e in res.restarts], g[f"{key}/restart_iters"])
    np.testing.assert_allclose(res.metrics.kkt_residual, g[f"{key}/metrics"][0], rtol=1e-6)


def test_oracle_matches_reference_kml_small(golden_kml):
    arr = instances.kml_epigraph(N=120, d=10)
    g = golden_kml
    np.testing.assert_allclose([float(np.sum(arr.Q[i])) for i in range(arr.m + 1)],
                               g["Q_checksum"], rtol=1e-12)
    P = O.Problem.from_arrays(arr)
    res, _ = _run(P, "yx", True, _policy("fixed", period=500), 3000, 1e-6)
    _check_prefix(_trace(res), g["nm_fixed500/trace"])
    assert res.iterations == int(g["nm_fixed500/iterations"])
