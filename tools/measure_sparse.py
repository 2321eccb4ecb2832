"""A sparse-Q QCQP too large to densify (default n = 200 000, m = 32: the dense
stack would be 10.6 TB), on the device's sparse path (SparseQInstance) and on
the CPU oracle (the reference's CSR storage, problem.py:31-40): the first K
iterations step for step, then the device's run to KKT 1e-6.

    python tools/measure_sparse.py [n] [m] [K]   -> one JSON line
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from oracle import rapdb_oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 32
K = int(sys.argv[3]) if len(sys.argv) > 3 else 40
t0 = time.perf_counter()
Q, q, r, lo, hi = instances.sparse_qcqp(n=n, m=m, rows=n // 5, nnz_row=5, seed=1)
gen_s = time.perf_counter() - t0
nnz = int(sum(M.nnz for M in Q))
inst = R.SparseQInstance(n, m, Q, q, r, lo, hi)
cfg = R.SolverConfig(mode="yx", nonmonotone=False)
t0 = time.perf_counter()
inst.device_data(torch.device("cuda", 0))
torch.cuda.synchronize()
up_s = time.perf_counter() - t0

# parity window: K iterations on both sides
dev = R.ApdbEngine(inst, cfg, R.initial_iterate(inst))
dev.run_block(K)
got = np.array([[t.tau_start, t.tau, t.evals_iter] for t in dev.trace])
P = O.Problem(Q, [q[i] for i in range(m + 1)], r, np.zeros((0, n)), np.zeros(0), lo, hi, 0.0)
t0 = time.perf_counter()
eng = O.Engine(P, O.Options(mode="yx", nonmonotone=False), *O.initial_point(P))
for _ in range(K):
    eng.step()
cpu_s = time.perf_counter() - t0
ref = np.array([[t.tau_start, t.tau, t.evals_iter] for t in eng.trace])
z = dev.last
rx = float(np.linalg.norm(z.x - eng.x) / max(np.linalg.norm(eng.x), 1e-300))
rl = float(np.linalg.norm(z.lam - eng.lam) / max(np.linalg.norm(eng.lam), 1e-300))

# the device's run to KKT
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
res = None
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = R.run_restarted(inst, cfg, R.FixedRestart(500), budget=20000, criteria=crit)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(json.dumps({
    "workload": f"sparse-Q QCQP n={n}, m={m}, Q_i = B_i^T B_i + 0.1 I (B_i {n // 5} x n, 5 nnz/row)",
    "nnz_total": nnz, "stack_bytes_sparse": 12 * nnz, "stack_bytes_dense": 8 * (m + 1) * n * n,
    "generate_s": gen_s, "upload_s": up_s,
    "parity_iterations": K, "steps_bitwise_equal": bool(np.array_equal(got, ref)), "rel_x": rx, "rel_lam": rl,
    "cpu_oracle_iters_per_s": K / cpu_s, "cpu_evals": int(ref[:, 2].sum()),
    "device": {"iterations": res.iterations, "evals": res.evals, "converged": bool(res.converged),
               "final_kkt": res.metrics.kkt_residual, "time_s": dt, "iters_per_s": res.iterations / dt,
               "us_per_eval": 1e6 * dt / max(res.evals, 1)},
}))
