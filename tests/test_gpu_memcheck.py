"""Memory-safety and race checks of every device op, in place of
compute-sanitizer (closed on the test pool: runs under it left GPUs needing a
reset).

1. Guard zones: with RAPDB_GUARD=1 the workspace gets a 4 KB patterned zone
   after every buffer (rapdb_check_guards); each case runs its ops and
   asserts that no zone was written -- an out-of-bounds store into a
   neighbouring buffer would show up here.
2. Run-to-run determinism: each case runs twice from scratch and must give
   the same bits (trace, iterates, metrics) -- a race in a grid reduction, a
   stale ring-slot read or an unordered cross-CTA sum would not.

Small instances of: yx / xy, monotone / non-monotone, fixed restarts, KKT,
the smoothed gap (adaptive), the packed sweep's early reduction, the
row-major layout, the factored path (fused host-launched trial, generic
stops, several row phases of R^T), the peer exchange and the native NCCL exchange at world
size 1, EGM and the point evaluations.
"""

import os

import numpy as np
import pytest

import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import _capi, instances
from paper_2605_29291_b200.sharding import Shard

pytestmark = pytest.mark.gpu

CASES = ["yx_nm", "xy_nm", "yx_mono_kkt", "adaptive_gap", "early", "rows", "factored_yx", "factored_xy",
         "factored_phased", "peer", "comm", "egm", "points"]


def _dense(n=130, m=9, rank=8, seed=3):
    arr = instances.dense_qcqp(n, m, rank, seed=seed)
    return arr, R.ProblemInstance.from_arrays(arr, validate=False)


def _factored():
    from paper_2605_29291_b200.factored import FactoredInstance
    arr = instances.factored_qcqp(n=1500, mq=5, rows=200, nnz_row=7, lin_rows=300, lin_nnz=4, seed=8,
                                  x0_scale=0.1)
    return arr, FactoredInstance.from_arrays(arr)


def _snapshot(eng):
    z = eng.last
    tr = np.array([[t.tau_start, t.tau, t.evals_iter] for t in eng.trace])
    return [tr, z.x.copy(), z.lam.copy(), np.asarray(eng._ctx.kkt())]


def _run_case(case):
    """Runs the case's ops; returns (bits to compare, guard results)."""
    guards = []
    out = []
    if case in ("yx_nm", "xy_nm", "yx_mono_kkt", "early", "rows", "peer", "comm"):
        if case == "early":
            arr, inst = _dense(n=200, m=23, rank=6)
        else:
            arr, inst = _dense()
        shard = None
        if case == "peer":
            shard = Shard(rank=0, nranks=1, k0=0, k1=arr.m + 1, force_split=True, p2p=True,
                          exchange=lambda v: None)
        elif case == "comm":
            shard = Shard(rank=0, nranks=1, k0=0, k1=arr.m + 1, force_split=True,
                          comm=_capi.Comm(0, _capi.comm_unique_id(), 0, 1))
        mode = "xy" if case == "xy_nm" else "yx"
        cfg = R.SolverConfig(mode=mode, nonmonotone=case != "yx_mono_kkt")
        eng = R.ApdbEngine(inst, cfg, R.initial_iterate(inst), shard=shard)
        eng.run_block(25)
        eng.reinit_from("average")
        eng.run_block(15)
        out += _snapshot(eng)
        guards.append(eng._ctx.check_guards())
    elif case == "adaptive_gap":
        arr, inst = _dense()
        eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.initial_iterate(inst))
        eng.run_block(30)
        gap, cert, xc = eng.smoothed_gap(1, 0.04, 1e-9, None)
        out += _snapshot(eng) + [np.array([gap, cert.iterations, cert.residual])]
        guards.append(eng._ctx.check_guards())
    elif case in ("factored_yx", "factored_xy", "factored_phased"):
        arr, inst = _factored()
        mode = "xy" if case == "factored_xy" else "yx"
        eng = R.ApdbEngine(inst, R.SolverConfig(mode=mode, nonmonotone=True), R.initial_iterate(inst))
        eng.run_block(20)
        eng.reinit_from("last")
        eng.run_block(10)
        out += _snapshot(eng)
        guards.append(eng._ctx.check_guards())
    elif case == "egm":
        from paper_2605_29291_b200.egm import run_egm
        arr, inst = _dense()
        res = run_egm(inst, 0.01, R.initial_iterate(inst), 40)
        out += [np.asarray(res.last.x), np.asarray(res.average.x)]
        guards.append(res._ctx.check_guards())
    elif case == "points":
        arr, inst = _dense()
        x = np.linspace(-1, 1, arr.n)
        z = R.Iterate(x, np.zeros(0), np.abs(np.linspace(0, 1, arr.m)))
        met = R.kkt_residual(inst, z)
        out += [np.array([inst.f_value(x), R.coupling_value(inst, z), met.kkt_residual, met.infeas]),
                np.asarray(inst.g_value(x)), np.asarray(R.grad_x_coupling(inst, z))]
        guards.append(inst._evaluator().ctx.check_guards())
    return out, guards


@pytest.mark.parametrize("case", CASES)
def test_guards_and_determinism(case, monkeypatch):
    monkeypatch.setenv("RAPDB_GUARD", "1")
    if case == "early":
        monkeypatch.setenv("RAPDB_EARLY_CHUNKS", "4")
    if case == "rows":
        monkeypatch.setenv("RAPDB_LAYOUT", "rows")
    if case == "factored_phased":   # several row phases of R^T (one gradient launch each)
        monkeypatch.setenv("RAPDB_RT_PHASE_ROWS", "300")
    a, ga = _run_case(case)
    b, gb = _run_case(case)
    for n_bad, rep in ga + gb:
        assert n_bad == 0, rep
    assert len(a) == len(b)
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)
