"""Golden for the sparse-Q path: the REAL reference on a QCQP whose quadratic
forms are sparse (instances.sparse_qcqp: every Q_i below the 25 % density at
which problem.py:31-40 keeps it as CSR, so the reference applies them with
scipy's csr_matvec).  Records the instance checksums, per-iteration traces and
iterates of yx monotone / non-monotone runs with FixedRestart(60), a probe
point (f, g, grad_x Phi), for the oracle pin and the GPU parity test.

    python tests/golden/make_sparse_golden.py      -> tests/golden/sparse_qcqp.npz
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import rapdb  # noqa: E402  (the reference package)
from rapdb import problem as rproblem  # noqa: E402
from rapdb.geometry import Box, NonnegOrthant  # noqa: E402
from rapdb.restarts import FixedRestart  # noqa: E402

from paper_2605_29291_b200 import instances  # noqa: E402

SPARSE_SMALL = dict(n=400, m=6, rows=60, nnz_row=4, seed=3)
SNAPS = (1, 5, 20, 60, 61, 100, 150)


def main():
    Q, q, r, lo, hi = instances.sparse_qcqp(**SPARSE_SMALL)
    n, m = SPARSE_SMALL["n"], SPARSE_SMALL["m"]
    inst = rapdb.ProblemInstance(n=n, m=m, p=0, Q=Q, q=[q[i] for i in range(m + 1)], r=r,
                                 A=np.zeros((0, n)), b=np.zeros(0), primal_set=Box(lo, hi),
                                 cone=NonnegOrthant(m), mu=0.0, name="sparse-small")
    assert all(sp.issparse(M) for M in inst.Q), "the reference must hold these forms as CSR"
    out = {"Q_checksum": np.array([float(M.data.sum()) for M in Q]),
           "Q_nnz": np.array([M.nnz for M in Q], dtype=np.int64),
           "density_max": np.array(max(M.nnz for M in Q) / (n * n))}
    rng = np.random.default_rng(5)
    x = rng.uniform(-0.5, 0.5, n)
    lam = np.abs(rng.normal(size=m))
    lam[2] = 0.0
    z = rproblem.Iterate(x, np.zeros(0), lam)
    out.update(probe_x=x, probe_lam=lam, probe_f=np.array(inst.f_value(x)), probe_g=inst.g_value(x),
               probe_gradx=rproblem.grad_x_coupling(inst, z))
    for key, nm in (("mono", False), ("nm", True)):
        snaps = {}
        orig_step = rapdb.engine.ApdbEngine.step

        def hooked(self):
            rec = orig_step(self)
            if rec.iter in SNAPS:
                snaps[rec.iter] = (self.z.x.copy(), self.z.lam.copy())
            return rec

        rapdb.engine.ApdbEngine.step = hooked
        try:
            res = rapdb.run_restarted(inst, rapdb.SolverConfig(mode="yx", nonmonotone=nm), FixedRestart(60),
                                      budget=150)
        finally:
            rapdb.engine.ApdbEngine.step = orig_step
        tr = np.array([[t.iter, t.tau_start, t.tau, t.sigma, t.gamma, t.evals_iter, t.evals_total]
                       for t in res.trace])
        keys = sorted(snaps)
        out[f"{key}/trace"] = tr
        out[f"{key}/snap_iters"] = np.array(keys, dtype=np.int64)
        out[f"{key}/snap_x"] = np.array([snaps[k][0] for k in keys])
        out[f"{key}/snap_lam"] = np.array([snaps[k][1] for k in keys])
        out[f"{key}/final_x"] = res.solution.x
        out[f"{key}/final_lam"] = res.solution.lam
        out[f"{key}/restart_iters"] = np.array([e.iteration for e in res.restart_log], dtype=np.int64)
        print(key, res.iterations, res.evals, len(keys))
    np.savez_compressed(os.path.join(HERE, "sparse_qcqp.npz"), **out)
    print("wrote", os.path.getsize(os.path.join(HERE, "sparse_qcqp.npz")))


if __name__ == "__main__":
    main()
