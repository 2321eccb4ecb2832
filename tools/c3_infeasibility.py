"""Certificate that BASELINE config 3 as specified (x0 ~ U(-1, 1)) has no
feasible point, which is why the timed factored runs use C3f
(x0 ~ U(-0.01, 0.01)).  Host-only (scipy), run here:

    python tools/c3_infeasibility.py [n] > profiles/r02_c3_infeasibility.json

Two bounds on ||x|| for a feasible x:
* lower, from the linear rows A x <= b alone: for any mu >= 0 with
  b'mu < 0, 0 >= mu'(A x - b) >= -||A'mu|| ||x|| - b'mu, so
  ||x|| >= -b'mu / ||A'mu||.  mu maximises the min-norm dual
  -1/2 ||A'mu||^2 - b'mu over mu >= 0 (L-BFGS-B).
* upper, from the sum of the quadratic rows: sum_i g_i(x) <= 0 gives
  1/2 x'M x + c'x + sum d <= 0 with M = sum_i R_i'R_i, c = sum c_i, so with
  l <= lambda_min(M):  ||x|| <= (||c|| + sqrt(||c||^2 - 2 l sum d)) / l.
  lambda_min(M) is estimated by Lanczos (eigsh); the report also gives the
  smallest l for which the two bounds would still be consistent
  (l_crit) -- the certificate holds whenever lambda_min(M) > l_crit.
"""
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as sla
from scipy.optimize import minimize

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29291_b200 import instances  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
scale = n / 1_000_000
t0 = time.time()
arr = instances.factored_qcqp(n=n, rows=max(1, int(100_000 * scale)), lin_rows=max(1, int(500_000 * scale)))
gen_s = time.time() - t0
A = arr.A.tocsr()
b = arr.b
At = A.T.tocsr()


def dual(mu):
    v = At @ mu
    f = 0.5 * float(v @ v) + float(b @ mu)          # minimise the negated dual
    g = A @ v + b
    return f, g


t0 = time.time()
res = minimize(dual, np.zeros(A.shape[0]), jac=True, method="L-BFGS-B",
               bounds=[(0.0, None)] * A.shape[0], options={"maxiter": 500, "maxcor": 20})
mu = np.maximum(res.x, 0.0)
atmu = At @ mu
r_min = -float(b @ mu) / float(np.linalg.norm(atmu))
dual_s = time.time() - t0

# quadratic rows 1..mq: M = sum R_i'R_i, c = sum c_i, sum d
R = arr.R.tocsr()
rows = arr.rows
Rq = R[rows:]                                       # blocks 1..mq (block 0 is the objective)
c = arr.C[1:].sum(axis=0)
sum_d = float(arr.d[1:].sum())
M = sla.LinearOperator((n, n), matvec=lambda x: Rq.T @ (Rq @ x), dtype=float)
t0 = time.time()
lam_min = float(sla.eigsh(M, k=1, which="SA", tol=1e-3, maxiter=3000, return_eigenvectors=False)[0])
eig_s = time.time() - t0
cn = float(np.linalg.norm(c))
r_max = (cn + np.sqrt(cn * cn - 2.0 * lam_min * sum_d)) / lam_min
# smallest l with 1/2 l r_min^2 - ||c|| r_min + sum d > 0 (no feasible x of norm >= r_min)
l_crit = 2.0 * (cn * r_min - sum_d) / (r_min * r_min)
out = {"n": n, "mq": arr.mq, "linear_rows": A.shape[0], "generate_s": gen_s,
       "norm_lower_bound_from_Ax_le_b": r_min, "norm_sq_lower_bound": r_min ** 2,
       "norm_sq_lower_bound_over_n": r_min ** 2 / n, "dual_lbfgsb": {"iterations": int(res.nit), "s": dual_s},
       "lambda_min_M_estimate": lam_min, "eigsh_s": eig_s, "norm_c": cn, "sum_d": sum_d,
       "norm_upper_bound_from_quadratic_rows": r_max, "norm_sq_upper_bound": r_max ** 2,
       "lambda_min_needed": l_crit, "lambda_margin": lam_min / l_crit,
       "infeasible": bool(r_min > r_max)}
print(json.dumps(out))
