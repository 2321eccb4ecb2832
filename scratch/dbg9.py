import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.problem import DeviceData
n, m = int(sys.argv[1]), int(sys.argv[2])
arr = instances.dense_qcqp(n, m, 20, seed=0)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
dev = torch.device("cuda", 0)
def solve():
    return R.run_restarted(inst, R.SolverConfig(mode="yx"), R.FixedRestart(500), budget=20, device=dev)
inst.device_data(dev)
r = solve(); print("solve1", r.iterations, flush=True)
pinned = torch.from_numpy(inst.Q).pin_memory()
for k in range(4):
    inst.drop_device_data()
    d = DeviceData.upload(inst, dev, None); d.Q = pinned.to(dev)
    inst._dev[str(dev)] = d
    try:
        r = solve(); print("solve", k, r.iterations, flush=True)
    except Exception as e:
        print("FAIL", k, str(e)[:100], flush=True); break
