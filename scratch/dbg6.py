import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
variant = sys.argv[1]
arr = instances.dense_qcqp(int(sys.argv[2]), int(sys.argv[3]), 20, seed=0)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
dev = torch.device("cuda", 0)
def solve():
    return R.run_restarted(inst, R.SolverConfig(mode="yx"), R.FixedRestart(500), budget=300, device=dev)
inst.device_data(dev)
r = solve(); print(variant, "solve1", r.iterations, flush=True)
if variant == "pin":
    inst.pin_host()
for k in range(2):
    inst.drop_device_data()
    try:
        r = solve(); print(variant, "solve", k, r.iterations, flush=True)
    except Exception as e:
        print(variant, "FAIL", str(e)[:80], flush=True); break
