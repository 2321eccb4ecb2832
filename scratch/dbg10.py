import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
arr = instances.dense_qcqp(2000, 200, 20, seed=0)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
dev = torch.device("cuda", 0)
def solve():
    return R.run_restarted(inst, R.SolverConfig(mode="yx"), R.FixedRestart(500), budget=300, device=dev)
inst.device_data(dev)
r = solve(); print("solve1", r.iterations, flush=True)
inst.pin_host()
for k in range(6):
    inst.drop_device_data()
    try:
        r = solve(); print("solve", k, r.iterations, flush=True)
    except Exception as e:
        print("FAIL", k, str(e), flush=True); break
