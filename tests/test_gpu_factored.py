"""Config-3 factored path (Q_i = R_i^T R_i + sparse linear rows) on the GPU,
through the C ABI, against the reference's golden run of the densified
instance and the oracle's factored restatement.

Tolerances: the device sums some CSR products in a different order than
scipy (the R^T gather per column, fixed chunk trees for the dot products),
so iterates agree to rounding (1e-8 relative over 200 iterations); the
accepted step sizes depend on the data only through the accept decisions,
so they -- and the backtrack counts -- must be identical.
"""

import numpy as np
import pytest

from conftest import FACTORED_SMALL, load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.factored import FactoredInstance
from oracle import rapdb_oracle as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)) if b.size else 0.0


def trace_arr(trace):
    return np.array([[t.iter, t.tau_start, t.tau, t.sigma, t.gamma, t.evals_iter, t.evals_total]
                     for t in trace])


def oracle_trace(P, nm, iters, mode="yx"):
    # a few BLAS threads: with the default (one per host core) OpenBLAS spends
    # milliseconds waking threads for every length-1e4+ dot product
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=4):
        res = O.run_restarted(P, O.Options(mode=mode, nonmonotone=nm), O.Policy(kind="none"),
                              budget=iters)
    tr = np.array([[r.iter, r.tau_start, r.tau, r.sigma, r.gamma, r.evals_iter, r.evals_total]
                   for r in res.trace])
    return tr, res


@pytest.fixture(scope="module")
def small():
    arr = instances.factored_qcqp(**FACTORED_SMALL)
    return arr, FactoredInstance.from_arrays(arr), load_golden("factored_small")


def test_factored_probe_and_gradient(small):
    arr, inst, g = small
    x, lam = g["probe_x"], g["probe_lam"]
    f = float(g["probe_f"])
    assert abs(inst.f_value(x) - f) <= 1e-12 * (1 + abs(f))
    np.testing.assert_allclose(inst.g_value(x), g["probe_g"], rtol=1e-12, atol=1e-12)
    gx = R.grad_x_coupling(inst, R.Iterate(x, np.zeros(0), lam))
    assert rel(gx, g["probe_gradx"]) <= 1e-12
    # the W-cache itself: W = R x
    u, _ = inst._evaluator().sweep(x)
    assert rel(u.cpu().numpy(), arr.R @ x) <= 1e-13


@pytest.mark.parametrize("key,nm", [("mono", False), ("nm", True)])
def test_factored_200_vs_reference(small, key, nm):
    arr, inst, g = small
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.initial_iterate(inst))
    snaps = list(g[f"{key}/snap_iters"])
    done = 0
    for k in (1, 10, 50, 100, 200):
        eng.run_block(k - done)
        done = k
        z = eng.last
        idx = snaps.index(k)
        assert rel(z.x, g[f"{key}/snap_x"][idx]) <= 1e-8, k
        assert rel(z.lam, g[f"{key}/snap_lam"][idx]) <= 1e-8, k
    tr = trace_arr(eng.trace)
    tg = g[f"{key}/trace"]
    np.testing.assert_array_equal(tr[:, 5], tg[:, 5])
    np.testing.assert_array_equal(tr[:, 1:5], tg[:, 1:5])
    assert rel(eng.average().x, g[f"{key}/avg_x"]) <= 1e-8


def test_factored_xy_vs_oracle(small):
    arr, inst, _ = small
    tr_o, res = oracle_trace(O.factored_problem(arr), True, 150, mode="xy")
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="xy", nonmonotone=True), R.initial_iterate(inst))
    eng.run_block(150)
    tr = trace_arr(eng.trace)
    np.testing.assert_array_equal(tr[:, 5], tr_o[:, 5])
    np.testing.assert_array_equal(tr[:, 1:5], tr_o[:, 1:5])
    assert rel(eng.last.x, res.x) <= 1e-8


def test_factored_fixed_restart_kkt(small):
    """run_restarted with device FixedRestart(200) and KKT every 10 iterations
    over the reference's 4000-iteration budget (the instance is degenerate --
    neither side reaches 1e-6): same stop, KKT residual within a factor 2."""
    arr, inst, g = small
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(200),
                          budget=4000, criteria=R.TerminationCriteria(criterion="conic", eps_kkt=1e-6,
                                                                      eps_feas=1e-6))
    assert res.iterations == int(g["nm_fixed200/iterations"])
    assert bool(res.converged) == bool(g["nm_fixed200/converged"])
    k_ref = float(g["nm_fixed200/metrics"][0])
    assert 0.5 * k_ref <= res.metrics.kkt_residual <= 2.0 * k_ref
    # device KKT at the final point vs the host-side evaluation of the same point
    m = R.kkt_residual(inst, res.solution)
    P = O.factored_problem(arr)
    mo = O.kkt(P, res.solution.x, np.zeros(0), res.solution.lam)
    assert abs(m.kkt_residual - mo.kkt_residual) <= 1e-9 * (1 + mo.kkt_residual)
    assert abs(m.f_value - mo.f_value) <= 1e-11 * (1 + abs(mo.f_value))


SHAPES = [
    dict(n=1000, mq=0, rows=100, nnz_row=10, lin_rows=500, lin_nnz=5, seed=2, x0_scale=0.1),   # objective only
    dict(n=2000, mq=3, rows=50, nnz_row=10, lin_rows=0, lin_nnz=5, seed=3),                     # no linear block
    dict(n=1025, mq=2, rows=1030, nnz_row=7, lin_rows=7, lin_nnz=3, seed=4, x0_scale=0.05),     # ragged chunks
    dict(n=50_000, mq=8, rows=5000, nnz_row=10, lin_rows=20_000, lin_nnz=5, seed=1, x0_scale=0.02),
]


@pytest.mark.parametrize("shape", SHAPES, ids=["mq0", "L0", "ragged", "n50k"])
@pytest.mark.parametrize("nm", [False, True])
def test_factored_shapes_vs_oracle(shape, nm):
    arr = instances.factored_qcqp(**shape)
    inst = FactoredInstance.from_arrays(arr)
    iters = 60
    tr_o, res = oracle_trace(O.FactoredProblem(arr), nm, iters)
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.initial_iterate(inst))
    eng.run_block(iters)
    tr = trace_arr(eng.trace)
    np.testing.assert_array_equal(tr[:, 5], tr_o[:, 5])
    np.testing.assert_array_equal(tr[:, 1:5], tr_o[:, 1:5])
    z = eng.last
    assert rel(z.x, res.x) <= 1e-8
    if arr.m:
        assert rel(z.lam, res.lam) <= 1e-8, rel(z.lam, res.lam)
    np.testing.assert_allclose(inst.g_value(z.x), O.FactoredProblem(arr).g(z.x), rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("kind", ["joint", "split"])
@pytest.mark.parametrize("mode,nm", [("yx", False), ("yx", True), ("xy", True)])
def test_factored_dual_ball_vs_oracle(small, kind, mode, nm):
    """JointBall / SplitBall on the factored path (geometry.py:263-311): the
    radius is half the unbounded run's multiplier norm after 200 iterations,
    so the ball binds.  The device scales y~ from a fixed-order norm, numpy
    from np.linalg.norm: rounding-level differences, same tolerances as the
    unbounded traces."""
    from paper_2605_29291_b200.geometry import JointBall, SplitBall
    arr, inst, g = small
    r = 0.5 * float(np.linalg.norm(g["mono/snap_lam"][-1]))
    assert r > 0
    ball = JointBall(r) if kind == "joint" else SplitBall(1.0, r)
    oball = O.Ball(1, r) if kind == "joint" else O.Ball(2, 1.0, r)
    iters = 120
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=4):
        res = O.run_restarted(O.factored_problem(arr), O.Options(mode=mode, nonmonotone=nm, ball=oball),
                              O.Policy(kind="none"), budget=iters)
    tr_o = np.array([[t.iter, t.tau_start, t.tau, t.sigma, t.gamma, t.evals_iter, t.evals_total]
                     for t in res.trace])
    cfg = R.SolverConfig(mode=mode, nonmonotone=nm, dual_ball=ball)
    eng = R.ApdbEngine(inst, cfg, R.initial_iterate(inst, ball))
    eng.run_block(iters)
    tr = trace_arr(eng.trace)
    np.testing.assert_array_equal(tr[:, 5], tr_o[:, 5])
    np.testing.assert_array_equal(tr[:, 1:5], tr_o[:, 1:5])
    z = eng.last
    assert rel(z.x, res.x) <= 1e-8
    assert rel(z.lam, res.lam) <= 1e-8
    assert np.linalg.norm(z.lam) <= r * (1 + 1e-12)
    assert np.linalg.norm(res.lam) >= 0.999 * r   # the ball is active at the end


def test_factored_rejects_unsupported(small):
    arr, inst, _ = small
    with pytest.raises(R.ConfigurationError):
        R.run_restarted(inst, R.SolverConfig(), R.AdaptiveRestart(warmup=5, check_period=5), budget=30)


# ------------------------------------------------------- constraint sharding (section 8(e))

def test_factored_forced_split_is_bitwise_identical(small):
    """One rank in split mode (kernel stops at every exchange point, host
    'all-reduces' a single buffer) == the fused single-launch run."""
    from paper_2605_29291_b200.sharding import Shard
    arr, inst, _ = small
    cfg = R.SolverConfig(mode="yx", nonmonotone=True)
    fused = R.run_restarted(inst, cfg, R.FixedRestart(40), budget=120)
    calls = []
    shard = Shard(rank=0, nranks=1, k0=0, k1=arr.mq + 1, l0=0, l1=arr.L, force_split=True,
                  exchange=lambda views: calls.append(len(views)))
    split = R.run_restarted(inst, cfg, R.FixedRestart(40), budget=120, shard=shard)
    assert calls
    np.testing.assert_array_equal(trace_arr(split.trace), trace_arr(fused.trace))
    np.testing.assert_array_equal(split.solution.x, fused.solution.x)
    np.testing.assert_array_equal(split.solution.lam, fused.solution.lam)


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("nm", [False, True])
def test_factored_emulated_shards(small, nranks, nm):
    """R ranks, each holding a block range and a linear-row range, exchanging
    the gradient partial and g per trial: same accepted steps as the
    unsharded device run, iterates to 1e-12, and the oracle to 1e-9."""
    from paper_2605_29291_b200.sharding import EmulatedCluster
    arr, inst, _ = small
    cfg = R.SolverConfig(mode="yx", nonmonotone=nm)
    iters = 80
    ref = R.ApdbEngine(inst, cfg, R.initial_iterate(inst))
    ref.run_block(iters)
    tr_ref = trace_arr(ref.trace)
    tr_o, res_o = oracle_trace(O.FactoredProblem(arr), nm, iters)
    cluster = EmulatedCluster(nranks)
    shards = cluster.shards(inst)
    assert [s.k0 for s in shards][0] == 0 and shards[-1].k1 == arr.mq + 1
    assert shards[0].l0 == 0 and shards[-1].l1 == arr.L

    def body(shard):
        eng = R.ApdbEngine(inst, cfg, R.initial_iterate(inst), shard=shard)
        eng.run_block(iters)
        return trace_arr(eng.trace), eng.last

    for tr, z in cluster.run(inst, body):
        np.testing.assert_array_equal(tr[:, 5], tr_ref[:, 5])
        np.testing.assert_array_equal(tr[:, 1:5], tr_ref[:, 1:5])
        assert rel(z.x, ref.last.x) <= 1e-12
        assert rel(z.lam, ref.last.lam) <= 1e-11
        np.testing.assert_array_equal(tr[:, 5], tr_o[:, 5])
        np.testing.assert_array_equal(tr[:, 1:5], tr_o[:, 1:5])


def test_factored_emulated_shards_with_ball(small):
    """Two constraint shards with a binding JointBall: the multipliers are
    replicated, so each rank's norm is complete and the scaled y~ agrees with
    the unsharded run (same steps, iterates to 1e-11)."""
    from paper_2605_29291_b200.geometry import JointBall
    from paper_2605_29291_b200.sharding import EmulatedCluster
    arr, inst, g = small
    ball = JointBall(0.5 * float(np.linalg.norm(g["mono/snap_lam"][-1])))
    cfg = R.SolverConfig(mode="yx", nonmonotone=True, dual_ball=ball)
    iters = 80
    ref = R.ApdbEngine(inst, cfg, R.initial_iterate(inst, ball))
    ref.run_block(iters)
    tr_ref = trace_arr(ref.trace)
    cluster = EmulatedCluster(2)

    def body(shard):
        eng = R.ApdbEngine(inst, cfg, R.initial_iterate(inst, ball), shard=shard)
        eng.run_block(iters)
        return trace_arr(eng.trace), eng.last

    for tr, z in cluster.run(inst, body):
        np.testing.assert_array_equal(tr[:, 5], tr_ref[:, 5])
        np.testing.assert_array_equal(tr[:, 1:5], tr_ref[:, 1:5])
        assert rel(z.x, ref.last.x) <= 1e-12
        assert rel(z.lam, ref.last.lam) <= 1e-11


@pytest.mark.slow
def test_c3_full_size_first_iterations():
    """BASELINE C3 at full size (n = 10^6, 64 factored constraints, 5e5
    linear rows): the first 3 accepted iterations (11 test evaluations, incl.
    the initial backtracking from tau_bar) against the oracle's factored
    restatement -- identical backtrack counts and step sizes to rounding,
    iterates to 1e-9.  (~1 min of CPU oracle time.)"""
    arr = instances.factored_qcqp()
    inst = FactoredInstance.from_arrays(arr)
    tr_o, res_o = oracle_trace(O.FactoredProblem(arr), False, 3)
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.initial_iterate(inst))
    eng.run_block(3)
    tr = trace_arr(eng.trace)
    np.testing.assert_array_equal(tr[:, 5], tr_o[:, 5])
    np.testing.assert_array_equal(tr[:, 1:5], tr_o[:, 1:5])
    assert rel(eng.last.x, res_o.x) <= 1e-9
    assert rel(eng.last.lam, res_o.lam) <= 1e-9


def test_row_phases_do_not_change_bits(monkeypatch):
    """The R^T gather continues every column's sum across the row phases in
    row order (one launch per phase), and the c_i part continues its block
    chain the same way: any phase count gives the same bits."""
    arr = instances.factored_qcqp(n=1500, mq=5, rows=200, nnz_row=7, lin_rows=300, lin_nnz=4, seed=8,
                                  x0_scale=0.1)
    outs = []
    for rows in ("100000", "500", "170"):            # 1, 3 and 8 phases of the 1200 stacked rows
        monkeypatch.setenv("RAPDB_RT_PHASE_ROWS", rows)
        inst = FactoredInstance.from_arrays(arr)
        lam = np.abs(np.linspace(0.0, 1.0, inst.m))
        lam[1] = 0.0                                  # a zero block weight: its gathers are skipped
        x = np.linspace(-0.3, 0.4, arr.n)
        gx = R.grad_x_coupling(inst, R.Iterate(x, np.zeros(0), lam))
        eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.initial_iterate(inst))
        eng.run_block(25)
        outs.append((np.asarray(gx), trace_arr(eng.trace), np.asarray(eng.last.x), np.asarray(eng.last.lam),
                     inst.device_data().rt_nph))
    assert [o[4] for o in outs] == [1, 3, 8]
    for o in outs[1:]:
        for a, b in zip(outs[0][:4], o[:4]):
            np.testing.assert_array_equal(a, b)


def test_gradient_matches_scipy_order(small):
    """The three column parts of the device gradient -- sum_i w_i c_i (block
    order), the R^T gather (row order, no FMA) and A^T mu -- restated with
    scipy in the same order give the same bits."""
    import scipy.sparse as sp
    arr, inst, g = small
    x, lam = g["probe_x"], g["probe_lam"]
    gx = np.asarray(R.grad_x_coupling(inst, R.Iterate(x, np.zeros(0), lam)))
    Rm = sp.csr_matrix(arr.R)
    W = Rm @ x
    wq = np.concatenate([[1.0], lam[:arr.mq]])
    rmat = np.repeat(np.arange(arr.mq + 1), arr.rows)
    Rt = Rm.T.tocsr()
    Rt.sort_indices()
    s = Rt @ (wq[rmat] * W)
    acc = np.zeros(arr.n)
    for i in range(arr.mq + 1):
        if wq[i] != 0.0:
            acc = acc + wq[i] * np.asarray(arr.C[i])
    At = sp.csr_matrix(arr.A).T.tocsr()
    At.sort_indices()
    t = At @ lam[arr.mq:]
    np.testing.assert_array_equal(gx, (acc + s) + t)


def test_ragged_blocks_and_variable_rows_match_scipy():
    """A factored instance that is not the generator's regular shape: blocks of
    70 / 200 / 0 / 33 rows (no multiple of the 32-slot slice or the 128-row
    chunk, one empty block), rows with 0..25 entries, empty columns, a linear
    block with empty rows.  g and the gradient against scipy in the device's
    order (gradient bitwise, g to rounding: the |W_i|^2 chunk sums differ)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(12)
    n, rows = 257, [70, 200, 0, 33]
    rblk = np.concatenate([[0], np.cumsum(rows)])
    dens = rng.uniform(0.0, 0.1, size=rblk[-1])
    mask = rng.uniform(size=(rblk[-1], n)) < dens[:, None]
    mask[5] = False                                   # an empty row
    mask[:, 100:110] = False                          # empty columns
    Rm = sp.csr_matrix(np.where(mask, rng.normal(size=mask.shape), 0.0))
    Am = sp.random(40, n, density=0.05, format="csr", random_state=3)
    Am = sp.vstack([Am[:20], sp.csr_matrix((3, n)), Am[20:]], format="csr")   # empty rows inside
    mq = len(rows) - 1
    C = rng.normal(size=(mq + 1, n)) / np.sqrt(n)
    d = np.concatenate([[0.0], -rng.uniform(1, 2, mq)])
    b = rng.uniform(0.5, 1.5, Am.shape[0])
    inst = FactoredInstance(n, mq, Rm, rblk, C, d, Am, b, np.full(n, -10.0), np.full(n, 10.0))
    x = rng.uniform(-0.5, 0.5, n)
    lam = np.abs(rng.normal(size=inst.m))
    lam[1] = 0.0
    W = Rm @ x
    g_ref = np.array([0.5 * float(W[rblk[i]:rblk[i + 1]] @ W[rblk[i]:rblk[i + 1]]) + float(C[i] @ x) + d[i]
                      for i in range(mq + 1)])
    g = inst.g_value(x)
    np.testing.assert_allclose(inst.f_value(x), g_ref[0], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(g[:mq], g_ref[1:], rtol=1e-13, atol=1e-13)
    np.testing.assert_array_equal(g[mq:], Am @ x - b)
    wq = np.concatenate([[1.0], lam[:mq]])
    rmat = np.repeat(np.arange(mq + 1), rows)
    Rt = Rm.T.tocsr()
    Rt.sort_indices()
    acc = np.zeros(n)
    for i in range(mq + 1):
        if wq[i] != 0.0:
            acc = acc + wq[i] * C[i]
    At = Am.T.tocsr()
    At.sort_indices()
    gx = np.asarray(R.grad_x_coupling(inst, R.Iterate(x, np.zeros(0), lam)))
    np.testing.assert_array_equal(gx, (acc + Rt @ (wq[rmat] * W)) + At @ lam[mq:])
    # and it runs: a few accepted iterations, deterministic
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.initial_iterate(inst))
    eng.run_block(15)
    eng2 = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.initial_iterate(inst))
    eng2.run_block(15)
    np.testing.assert_array_equal(trace_arr(eng.trace), trace_arr(eng2.trace))
    np.testing.assert_array_equal(eng.last.x, eng2.last.x)
