"""Sparse quadratic forms kept sparse (factored.SparseQInstance): the
reference stores a Q_i below 25 % density as CSR (_as_operator,
problem.py:31-40) and applies it with scipy's csr_matvec.  Golden:
tests/golden/make_sparse_golden.py ran the REAL reference on
instances.sparse_qcqp (all forms CSR there).

CPU: the oracle restatement reproduces the golden traces bit for bit and the
instance's Sell stack walks to the CSR products.  GPU: the device path through
the C ABI -- grad_x Phi bit-identical to the reference (same products, same
operation order), accepted step sizes / evaluation counts identical, iterates
within 1e-9 -- and the densified ProblemInstance agrees with it to rounding."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.factored import SellMatrix, SparseQInstance
from oracle import rapdb_oracle as O

SPARSE_SMALL = dict(n=400, m=6, rows=60, nnz_row=4, seed=3)
TAU = slice(1, 7)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)) if b.size else 0.0


def trace_arr(trace):
    return np.array([[t.iter, t.tau_start, t.tau, t.sigma, t.gamma, t.evals_iter, t.evals_total] for t in trace])


@pytest.fixture(scope="module")
def case():
    Q, q, r, lo, hi = instances.sparse_qcqp(**SPARSE_SMALL)
    g = load_golden("sparse_qcqp")
    np.testing.assert_allclose([float(M.data.sum()) for M in Q], g["Q_checksum"], rtol=1e-13)
    np.testing.assert_array_equal([M.nnz for M in Q], g["Q_nnz"])
    assert float(g["density_max"]) < 0.25
    return Q, q, r, lo, hi, g


@pytest.mark.parametrize("key,nm", [("mono", False), ("nm", True)])
def test_oracle_pin_sparse_forms(case, key, nm):
    Q, q, r, lo, hi, g = case
    n = SPARSE_SMALL["n"]
    P = O.Problem(Q, [q[i] for i in range(len(Q))], r, np.zeros((0, n)), np.zeros(0), lo, hi, 0.0)
    assert all(sp.issparse(M) for M in P.Q)
    res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=nm), O.Policy("fixed", period=60), budget=150)
    tr = np.array([[t.iter, t.tau_start, t.tau, t.sigma, t.gamma, t.evals_iter, t.evals_total] for t in res.trace])
    np.testing.assert_array_equal(tr, g[f"{key}/trace"])
    np.testing.assert_array_equal(res.x, g[f"{key}/final_x"])
    np.testing.assert_array_equal(res.lam, g[f"{key}/final_lam"])


def test_instance_layout_and_validation(case):
    Q, q, r, lo, hi, g = case
    n, m = SPARSE_SMALL["n"], SPARSE_SMALL["m"]
    inst = SparseQInstance(n, m, Q, q, r, lo, hi)
    assert inst.sym and inst.mq == m and inst.L == 0 and inst.m == m and inst.p == 0
    np.testing.assert_array_equal(inst.rblk, np.arange(m + 2) * n)
    S = SellMatrix.by_block_chunks(inst.R, inst.rblk)
    x = g["probe_x"]
    chunks = -(-n // 128)
    for i in (0, m):                                       # block i's slots walk to Q_i x in CSR order
        u = np.zeros(n)
        for k in range(n):
            s_ = i * chunks * 128 + k
            acc = 0.0
            for t in range(int(S.len[s_])):
                pos = int(S.sp[s_ >> 5]) + 32 * t + (s_ & 31)
                acc = acc + S.val[pos] * x[S.idx[pos]]
            u[k] = acc
        np.testing.assert_array_equal(u, Q[i] @ x)
    bad = [M.copy() for M in Q]
    bad[1] = bad[1] + sp.csr_matrix(([1.0], ([0], [5])), shape=(n, n))
    with pytest.raises(R.InputError):
        SparseQInstance(n, m, bad, q, r, lo, hi)
    with pytest.raises(R.InputError):
        SparseQInstance(n, m, Q[:-1], q, r, lo, hi)


@pytest.mark.gpu
def test_probe_point_matches_reference(case):
    Q, q, r, lo, hi, g = case
    inst = SparseQInstance(SPARSE_SMALL["n"], SPARSE_SMALL["m"], Q, q, r, lo, hi)
    x, lam = g["probe_x"], g["probe_lam"]
    assert abs(inst.f_value(x) - float(g["probe_f"])) <= 1e-13 * (1 + abs(float(g["probe_f"])))
    np.testing.assert_allclose(inst.g_value(x), g["probe_g"], rtol=1e-13, atol=1e-13)
    gx = np.asarray(R.grad_x_coupling(inst, R.Iterate(x, np.zeros(0), lam)))
    np.testing.assert_array_equal(gx, g["probe_gradx"])    # same products, same operation order


@pytest.mark.gpu
@pytest.mark.parametrize("key,nm", [("mono", False), ("nm", True)])
def test_run_matches_reference(case, key, nm):
    Q, q, r, lo, hi, g = case
    inst = SparseQInstance(SPARSE_SMALL["n"], SPARSE_SMALL["m"], Q, q, r, lo, hi)
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.FixedRestart(60), budget=150)
    np.testing.assert_array_equal(trace_arr(res.trace)[:, TAU], g[f"{key}/trace"][:, TAU])
    np.testing.assert_array_equal([e.iteration for e in res.restart_log], g[f"{key}/restart_iters"])
    assert rel(res.solution.x, g[f"{key}/final_x"]) <= 1e-9
    assert rel(res.solution.lam, g[f"{key}/final_lam"]) <= 1e-9
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.initial_iterate(inst))
    done = 0
    for idx, k in enumerate(int(v) for v in g[f"{key}/snap_iters"]):
        if k > 60:
            break                                           # the run above covers the restart
        eng.run_block(k - done)
        done = k
        assert rel(eng.last.x, g[f"{key}/snap_x"][idx]) <= 1e-9, k
        assert rel(eng.last.lam, g[f"{key}/snap_lam"][idx]) <= 1e-9, k


@pytest.mark.gpu
def test_dense_and_sparse_paths_agree(case):
    Q, q, r, lo, hi, g = case
    n, m = SPARSE_SMALL["n"], SPARSE_SMALL["m"]
    dense = R.ProblemInstance(n=n, m=m, p=0, Q=[M.toarray() for M in Q], q=q, r=r, A=np.zeros((0, n)),
                              b=np.zeros(0), primal_set=R.geometry.Box(lo, hi),
                              cone=R.geometry.NonnegOrthant(m))
    sparse = SparseQInstance.from_problem(dense)
    cfg = R.SolverConfig(mode="yx", nonmonotone=True)
    a = R.run_restarted(dense, cfg, R.FixedRestart(60), budget=120)
    b = R.run_restarted(sparse, cfg, R.FixedRestart(60), budget=120)
    np.testing.assert_array_equal(trace_arr(a.trace)[:, TAU], trace_arr(b.trace)[:, TAU])
    assert rel(a.solution.x, b.solution.x) <= 1e-9 and rel(a.solution.lam, b.solution.lam) <= 1e-9
    za = R.kkt_residual(dense, a.solution)
    zb = R.kkt_residual(sparse, b.solution)
    assert abs(za.kkt_residual - zb.kkt_residual) <= 1e-9 * max(1.0, abs(za.kkt_residual))


@pytest.mark.gpu
def test_sharded_sparse_stack(case):
    """Constraint shards of the sparse stack (matrix ranges; emulated 2-rank
    cluster on one GPU): the unsharded run's step sizes, iterates to rounding."""
    from paper_2605_29291_b200.sharding import EmulatedCluster
    Q, q, r, lo, hi, g = case
    inst = SparseQInstance(SPARSE_SMALL["n"], SPARSE_SMALL["m"], Q, q, r, lo, hi)
    cfg = R.SolverConfig(mode="yx", nonmonotone=True)
    fused = R.run_restarted(inst, cfg, R.FixedRestart(60), budget=100)
    emu = EmulatedCluster(2).run(inst, lambda sh: R.run_restarted(inst, cfg, R.FixedRestart(60), budget=100, shard=sh))
    for res in emu:
        np.testing.assert_array_equal(trace_arr(res.trace)[:, TAU], trace_arr(fused.trace)[:, TAU])
        assert rel(res.solution.x, fused.solution.x) <= 1e-12
    np.testing.assert_array_equal(emu[0].solution.x, emu[1].solution.x)


@pytest.mark.gpu
@pytest.mark.parametrize("mode,nm,ball", [("xy", False, None), ("xy", True, None), ("yx", True, ("joint", 0.6)),
                                          ("xy", False, ("split", 1.0, 0.5))])
def test_modes_and_dual_balls_vs_oracle(case, mode, nm, ball):
    """APDB-xy and the dual balls (geometry.py:263-311) on the sparse stack,
    against the oracle run on the same CSR forms: step sizes and evaluation
    counts identical, iterates within 1e-9."""
    from paper_2605_29291_b200.geometry import JointBall, SplitBall
    Q, q, r, lo, hi, g = case
    n, m = SPARSE_SMALL["n"], SPARSE_SMALL["m"]
    inst = SparseQInstance(n, m, Q, q, r, lo, hi)
    dev_ball = None if ball is None else (JointBall(ball[1]) if ball[0] == "joint" else SplitBall(ball[1], ball[2]))
    ob = O.Ball() if ball is None else (O.Ball(1, ball[1]) if ball[0] == "joint" else O.Ball(2, ball[1], ball[2]))
    kw = {} if dev_ball is None else {"dual_ball": dev_ball}
    cfg = R.SolverConfig(mode=mode, nonmonotone=nm, **kw)
    res = R.run_restarted(inst, cfg, R.FixedRestart(50), budget=120)
    P = O.Problem(Q, [q[i] for i in range(m + 1)], r, np.zeros((0, n)), np.zeros(0), lo, hi, 0.0)
    ref = O.run_restarted(P, O.Options(mode=mode, nonmonotone=nm, ball=ob), O.Policy("fixed", period=50), budget=120)
    tr = np.array([[t.iter, t.tau_start, t.tau, t.sigma, t.gamma, t.evals_iter, t.evals_total] for t in ref.trace])
    np.testing.assert_array_equal(trace_arr(res.trace)[:, TAU], tr[:, TAU])
    assert rel(res.solution.x, ref.x) <= 1e-9
    assert rel(res.solution.lam, ref.lam) <= 1e-9
    if ball is not None:                                   # the ball binds somewhere along the run
        assert np.linalg.norm(res.solution.lam) <= (ball[1] if ball[0] == "joint" else ball[2]) * (1 + 1e-12)
