"""The operator contract (problem.py:196-223) evaluated on the device,
checked with the reference's own operator tests (pkg/tests/test_problem.py:
36-110): hand examples, zero multipliers = objective, term-by-term oracle,
finite differences of grad_x Phi, dimension checks.  Random instances come
from instances.dense_qcqp (the reference's random_qcqp is not importable on
the GPU box); both layouts of the Q stack are exercised."""

import numpy as np
import pytest

import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.geometry import Box, NonnegOrthant

pytestmark = pytest.mark.gpu


def make_instance(n, Q0, cons=()):
    m = len(cons)
    Q = [Q0] + [c[0] for c in cons]
    q = [np.zeros(n)] + [c[1] for c in cons]
    r = np.array([0.0] + [c[2] for c in cons])
    return R.ProblemInstance(n=n, m=m, p=0, Q=Q, q=q, r=r, A=np.zeros((0, n)), b=np.zeros(0),
                             primal_set=Box(np.full(n, -10.0), np.full(n, 10.0)), cone=NonnegOrthant(m))


@pytest.fixture(params=["packed", "rows"])
def layout(request, monkeypatch):
    monkeypatch.setenv("RAPDB_LAYOUT", request.param)
    return request.param


def ball():
    return make_instance(2, np.eye(2), [(np.eye(2), np.zeros(2), -0.5)])


def test_hand_examples(layout):
    z = R.Iterate(np.array([1.0, 0.0]), np.zeros(0), np.array([3.0]))
    assert abs(R.coupling_value(ball(), z) - 0.5) <= 1e-10
    np.testing.assert_allclose(R.grad_x_coupling(ball(), z), [4.0, 0.0])
    one = make_instance(1, np.array([[1.0]]))
    assert R.coupling_value(one, R.Iterate(np.array([2.0]), np.zeros(0), np.zeros(0))) == 2.0
    eq, g = R.grad_y_coupling(ball(), R.Iterate(np.array([1.0, 0.0]), np.zeros(0), np.zeros(1)))
    assert eq.size == 0 and abs(g[0]) <= 1e-15


def test_zero_multipliers_and_term_by_term(layout):
    arr = instances.dense_qcqp(8, 3, 4, seed=5)
    inst = R.ProblemInstance.from_arrays(arr)
    rng = np.random.default_rng(0)
    for _ in range(10):
        x = rng.normal(size=8)
        z0 = R.Iterate(x, np.zeros(0), np.zeros(3))
        f = 0.5 * x @ arr.Q[0] @ x + arr.q[0] @ x + arr.r[0]
        assert abs(R.coupling_value(inst, z0) - f) <= 1e-12 * (1 + abs(f))
        lam = np.abs(rng.normal(size=3))
        g = np.array([0.5 * x @ arr.Q[i] @ x + arr.q[i] @ x + arr.r[i] for i in range(1, 4)])
        oracle = f + float(lam @ g)
        assert abs(R.coupling_value(inst, R.Iterate(x, np.zeros(0), lam)) - oracle) <= 1e-10 * (1 + abs(oracle))


def test_grad_x_finite_differences(layout):
    for seed in range(20):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(2, 11))
        m = int(rng.integers(1, 5))
        arr = instances.dense_qcqp(n, m, max(1, n // 2), seed=seed)
        inst = R.ProblemInstance.from_arrays(arr)
        x = rng.normal(size=n)
        lam = np.abs(rng.normal(size=m))
        z = R.Iterate(x, np.zeros(0), lam)
        g = R.grad_x_coupling(inst, z)
        h = 1e-5 * (1.0 + np.linalg.norm(x))
        fd = np.empty(n)
        for j in range(n):
            e = np.zeros(n)
            e[j] = h
            fd[j] = (R.coupling_value(inst, R.Iterate(x + e, z.v, lam))
                     - R.coupling_value(inst, R.Iterate(x - e, z.v, lam))) / (2 * h)
        assert np.linalg.norm(g - fd) <= 1e-6 * (1.0 + np.linalg.norm(g))


def test_dimension_mismatch():
    with pytest.raises(R.InputError):
        R.coupling_value(ball(), R.Iterate(np.zeros(3), np.zeros(0), np.zeros(1)))


@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (40, 40), (300, 123), (123, 300)])
def test_spectral_norm_vs_oracle(shape):
    """problem.spectral_norm (problem.py:47-68) on the device vs the oracle's
    restatement: same start vector, stop rule and 1.01 inflation."""
    from oracle import rapdb_oracle as O
    from paper_2605_29291_b200.problem import spectral_norm
    rng = np.random.default_rng(sum(shape))
    M = rng.standard_normal(shape)
    M[rng.random(shape) < 0.3] = 0.0
    got = spectral_norm(M)
    want = O.spectral_norm(M)
    assert abs(got - want) <= 1e-9 * want, (got, want)
    assert abs(got - 1.01 * np.linalg.norm(M, 2)) <= 1e-3 * got   # converged to ||M||_2
    assert spectral_norm(np.zeros((3, 4))) == 0.0
