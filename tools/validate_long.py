"""Long-horizon parity of a full-size BASELINE config against the CPU oracle
(the numpy restatement of the reference, oracle/rapdb_oracle.py), run on the
GPU box's host: run_restarted with FixedRestart(500) and KKT every 10
iterations for K iterations on both sides.  Reports where the accepted step
sizes first differ (if at all), the KKT trajectories at the checkpoints, and
the final iterates -- evidence that a slow or stalled convergence on the
device (C1 non-monotone) is the method's behaviour, not a device defect.

    python tools/validate_long.py C1 nm 1500  -> one JSON line
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from oracle import rapdb_oracle as O  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
nm = (sys.argv[2] if len(sys.argv) > 2 else "nm") == "nm"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
arr = instances.config_instance(name)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
P = O.Problem.from_arrays(arr)

t0 = time.time()
dev = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.FixedRestart(500), budget=K,
                      criteria=R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6))
gpu_s = time.time() - t0
t0 = time.time()
ref = O.run_restarted(P, O.Options(mode="yx", nonmonotone=nm), O.Policy(kind="fixed", period=500), budget=K,
                      criteria=dict(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6), metrics_every=10)
cpu_s = time.time() - t0

td = np.array([[t.tau_start, t.tau, t.evals_iter] for t in dev.trace])
tr = np.array([[t.tau_start, t.tau, t.evals_iter] for t in ref.trace])
k = min(len(td), len(tr))
same = np.all(td[:k] == tr[:k], axis=1)
first_diff = int(np.argmin(same)) + 1 if not same.all() else None
kd = {t.iter: t.kkt for t in dev.trace if t.kkt is not None}
kr = {t.iter: t.kkt for t in ref.trace if t.kkt is not None}
common = sorted(set(kd) & set(kr))
krel = [abs(kd[i] - kr[i]) / kr[i] for i in common]


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


out = {
    "config": name, "mode": "yx nm" if nm else "yx mono", "policy": "FixedRestart(500)", "budget": K,
    "device": {"iterations": dev.iterations, "evals": dev.evals, "converged": bool(dev.converged),
               "final_kkt": dev.metrics.kkt_residual, "wall_s": gpu_s},
    "oracle": {"iterations": ref.iterations, "evals": ref.evals, "converged": bool(ref.converged),
               "final_kkt": ref.metrics.kkt_residual, "wall_s": cpu_s},
    "steps_identical": int(same[:k].sum()), "steps_compared": k, "first_step_difference": first_diff,
    "kkt_checkpoints": len(common), "kkt_max_rel_diff": max(krel) if krel else None,
    "kkt_at": {str(i): [kd[i], kr[i]] for i in common[::max(1, len(common) // 15)]},
    "final_x_rel": rel(dev.solution.x, ref.x), "final_lam_rel": rel(dev.solution.lam, ref.lam),
}
print(json.dumps(out))
