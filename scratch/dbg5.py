import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
arr = instances.dense_qcqp(2000, 200, 200, seed=0)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
def solve():
    return R.run_restarted(inst, R.SolverConfig(mode="yx"), R.FixedRestart(500), budget=50000, criteria=crit, device=torch.device("cuda", 0))
inst.device_data(torch.device("cuda", 0))
r = solve(); print("solve1", r.iterations, flush=True)
ev = inst._evaluator(); print("eval made", flush=True)
inst.pin_host(); print("pinned", flush=True)
for k in range(3):
    inst.drop_device_data(); print("dropped", flush=True)
    t = time.time()
    try:
        d = inst.device_data(torch.device("cuda", 0)); torch.cuda.synchronize(); print("uploaded", time.time() - t, float(d.Q[5, 7, 9]), arr.Q[5, 7, 9], flush=True)
        r = solve(); print("solve", k, r.iterations, time.time() - t, flush=True)
    except Exception as e:
        print("FAIL", e, flush=True)
