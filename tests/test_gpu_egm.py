"""The extragradient baseline on the device (egm.py, csrc/egm.cuh) against
the REAL reference's run_egm / tune_egm (tests/golden/egm.npz, made by
tests/golden/make_egm_golden.py).  EGM has no accept/reject decisions, so the
device and NumPy orders of summation only drift at rounding level: iterates
to 1e-10 relative, identical iteration counts and divergence points."""

import numpy as np
import pytest

from conftest import load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import egm
from paper_2605_29291_b200.geometry import JointBall
from test_gpu_parity import inst_from, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return load_golden("egm")


@pytest.fixture(scope="module")
def rq():
    g = load_golden("small_qcqp")
    return inst_from(g["Q"], g["q"], g["r"], g["lower"], g["upper"])


@pytest.fixture(scope="module")
def eqqp():
    g = load_golden("analytic")
    k = "eq-qp"
    return inst_from(g[f"{k}/Q"], g[f"{k}/q"], g[f"{k}/r"], g[f"{k}/lower"], g[f"{k}/upper"],
                     A=g[f"{k}/A"], b=g[f"{k}/b"], mu=float(g[f"{k}/mu"]))


CASES = {"rq_s01": (0.1, 300, None, 50), "rq_s003": (0.03, 300, None, 0), "rq_s1": (1.0, 300, None, 10),
         "rq_s10_div": (10.0, 300, None, 5), "rq_joint": (0.1, 200, 2.0, 0)}


@pytest.mark.parametrize("key", list(CASES))
def test_egm_vs_reference(gold, rq, key):
    s, K, ball, te = CASES[key]
    res = egm.run_egm(rq, s, R.initial_iterate(rq), K, dual_ball=None if ball is None else JointBall(ball),
                      trace_every=te)
    assert res.iterations == int(gold[f"{key}/iterations"])
    assert res.diverged == bool(gold[f"{key}/diverged"])
    tol = 1e-6 if res.diverged else 1e-10     # a diverging run amplifies rounding by |z| ~ 1e8
    assert rel(res.last.x, gold[f"{key}/last_x"]) <= tol
    assert rel(res.last.lam, gold[f"{key}/last_lam"]) <= tol
    assert rel(res.average.x, gold[f"{key}/avg_x"]) <= tol
    assert rel(res.average.lam, gold[f"{key}/avg_lam"]) <= tol
    tr = np.array([[t["iter"], t["norm"]] for t in res.trace]).reshape(-1, 2)
    g = gold[f"{key}/trace"]
    assert tr.shape == g.shape
    if tr.size:
        np.testing.assert_array_equal(tr[:, 0], g[:, 0])
        np.testing.assert_allclose(tr[:, 1], g[:, 1], rtol=tol)


def test_egm_equality_block(gold, eqqp):
    res = egm.run_egm(eqqp, 0.2, R.initial_iterate(eqqp), 200, trace_every=20)
    assert res.iterations == 200 and not res.diverged
    assert rel(res.last.x, gold["eq_s02/last_x"]) <= 1e-10
    assert rel(res.last.v, gold["eq_s02/last_v"]) <= 1e-10
    assert rel(res.average.v, gold["eq_s02/avg_v"]) <= 1e-10


def test_tune_egm(gold, rq):
    def score(z):
        return R.kkt_residual(rq, z).kkt_residual
    s, best = egm.tune_egm(rq, R.initial_iterate(rq), 100, score)
    assert s == float(gold["tune/best_s"])
    assert rel(best.last.x, gold["tune/last_x"]) <= 1e-10


def test_egm_rejects_bad_arguments(rq):
    with pytest.raises(R.ConfigurationError):
        egm.run_egm(rq, -1.0, R.initial_iterate(rq), 10)
    with pytest.raises(R.ConfigurationError):
        egm.run_egm(rq, 0.1, R.initial_iterate(rq), 0)


def test_egm_factored_matches_dense_equivalent():
    """EGM on a factored instance (host-assisted sweeps / gradients inside the
    EGM op) against EGM on the explicit dense form of the same problem."""
    from conftest import FACTORED_SMALL
    from paper_2605_29291_b200 import instances
    from paper_2605_29291_b200.factored import FactoredInstance
    arr = instances.factored_qcqp(**FACTORED_SMALL)
    finst = FactoredInstance.from_arrays(arr)
    Q, q, r = arr.dense_lists()
    dinst = inst_from(np.stack([np.asarray(M.toarray() if hasattr(M, "toarray") else M) for M in Q]),
                      np.stack(q), np.asarray(r), arr.lower, arr.upper)
    a = egm.run_egm(finst, 0.05, R.initial_iterate(finst), 120, trace_every=30)
    b = egm.run_egm(dinst, 0.05, R.initial_iterate(dinst), 120, trace_every=30)
    assert a.iterations == b.iterations and a.diverged == b.diverged
    assert rel(a.last.x, b.last.x) <= 1e-10
    assert rel(a.last.lam, b.last.lam) <= 1e-9
    assert rel(a.average.x, b.average.x) <= 1e-10
