"""Small instances of every device op, for compute-sanitizer (tools/sanitize.sh):

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py run
    cases: run (OP_RUN yx/xy, nm, fixed restarts, KKT cadence), gap (OP_GAP:
           smoothed gap inside an adaptive run), early (packed sweep with the
           early reduction forced on: 24 matrices), rows (row-major layout),
           factored (factored path, host-launched kernels), factored_fused
           (RAPDB_RT_PHASE_ROWS=300: several row phases of R^T), peer (in-kernel
           peer exchange at world size 1), comm (native NCCL exchange at world
           size 1), egm (extragradient op), probe (sweep / grad_x / kkt at a point)

Each case is a few iterations: the sanitizers slow kernels down 10-100x.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

case = sys.argv[1] if len(sys.argv) > 1 else "run"
if case == "early":
    os.environ["RAPDB_EARLY_CHUNKS"] = "4"
if case == "rows":
    os.environ["RAPDB_LAYOUT"] = "rows"
if case == "factored_fused":
    os.environ["RAPDB_RT_PHASE_ROWS"] = "300"

import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from paper_2605_29291_b200.sharding import Shard  # noqa: E402

crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-9, eps_feas=1e-9)


def dense(n=130, m=9, rank=8, seed=3):
    arr = instances.dense_qcqp(n, m, rank, seed=seed)
    return arr, R.ProblemInstance.from_arrays(arr, validate=False)


if case in ("run", "rows"):
    arr, inst = dense()
    for mode in ("yx", "xy"):
        res = R.run_restarted(inst, R.SolverConfig(mode=mode, nonmonotone=True), R.FixedRestart(7),
                              budget=20, criteria=crit, metrics_every=5)
        print(case, mode, res.iterations, res.evals)
elif case == "gap":
    arr, inst = dense()
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True),
                          R.AdaptiveRestart(warmup=5, check_period=5), budget=16, criteria=crit)
    print(case, res.iterations, [e.iteration for e in res.restart_log])
elif case == "early":
    arr, inst = dense(n=200, m=23, rank=6)
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.NoRestart(),
                          budget=6, criteria=crit)
    print(case, res.iterations, res.evals)
elif case in ("factored", "factored_fused"):
    from paper_2605_29291_b200.factored import FactoredInstance
    arr = instances.factored_qcqp(n=300, mq=4, rows=30, nnz_row=10, lin_rows=150, lin_nnz=5, seed=5,
                                  x0_scale=0.2)
    inst = FactoredInstance.from_arrays(arr)
    for mode in ("yx", "xy"):
        res = R.run_restarted(inst, R.SolverConfig(mode=mode, nonmonotone=True), R.FixedRestart(4),
                              budget=8, criteria=crit, metrics_every=4)
        print(case, mode, res.iterations, res.evals)
elif case == "peer":
    arr, inst = dense()
    shard = Shard(rank=0, nranks=1, k0=0, k1=arr.m + 1, force_split=True, p2p=True, exchange=lambda v: None)
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(5),
                          budget=10, criteria=crit, shard=shard)
    print(case, res.iterations)
elif case == "comm":
    from paper_2605_29291_b200 import _capi
    arr, inst = dense()
    comm = _capi.Comm(0, _capi.comm_unique_id(), 0, 1)
    shard = Shard(rank=0, nranks=1, k0=0, k1=arr.m + 1, force_split=True, comm=comm)
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(5),
                          budget=10, criteria=crit, shard=shard)
    print(case, res.iterations)
elif case == "egm":
    arr, inst = dense()
    from paper_2605_29291_b200.egm import run_egm
    out = run_egm(inst, 0.01, R.initial_iterate(inst), 6)
    print(case, "ok")
elif case == "probe":
    arr, inst = dense()
    x = np.linspace(-1, 1, arr.n)
    print(case, inst.f_value(x), float(np.sum(inst.g_value(x))))
    z = R.Iterate(x, np.zeros(0), np.abs(np.linspace(0, 1, arr.m)))
    print(case, float(np.sum(R.grad_x_coupling(inst, z))), R.kkt_residual(inst, z).kkt_residual)
else:
    raise SystemExit(f"unknown case {case}")
