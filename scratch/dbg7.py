import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.problem import DeviceData
v = sys.argv[1]
arr = instances.dense_qcqp(2000, 200, 20, seed=0)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
dev = torch.device("cuda", 0)
def solve():
    return R.run_restarted(inst, R.SolverConfig(mode="yx"), R.FixedRestart(500), budget=50, device=dev)
inst.device_data(dev)
r = solve(); print(v, "solve1", r.iterations, flush=True)
pinned = torch.from_numpy(inst.Q).pin_memory() if v != "nopin" else None
print(v, "pinned", flush=True)
try:
    if v == "pin_nodrop":
        r = solve(); print(v, "solve2", r.iterations, flush=True)
    elif v == "pin_sync":
        inst.drop_device_data()
        d = DeviceData.upload(inst, dev, None)   # pageable path
        inst._dev[str(dev)] = d
        r = solve(); print(v, "solve2", r.iterations, flush=True)
    elif v == "pin_blocking":
        inst.drop_device_data()
        Qd = pinned.to(dev, non_blocking=False)
        d = DeviceData.upload(inst, dev, None); d.Q = Qd
        inst._dev[str(dev)] = d
        r = solve(); print(v, "solve2", r.iterations, flush=True)
    elif v == "nopin":
        inst.drop_device_data()
        r = solve(); print(v, "solve2", r.iterations, flush=True)
    r = solve(); print(v, "solve3", r.iterations, flush=True)
except Exception as e:
    print(v, "FAIL", str(e)[:100], flush=True)
