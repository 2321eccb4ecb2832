import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from paper_2605_29291_b200.problem import DeviceData
arr = instances.dense_qcqp(2000, 200, 20, seed=0)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
dev = torch.device("cuda", 0)
d0 = inst.device_data(dev)
print("Q0 ptr", hex(d0.Q.data_ptr()), flush=True)
pinned = torch.from_numpy(inst.Q).pin_memory()
print("pinned ptr", hex(pinned.data_ptr()), flush=True)
Qb = pinned.to(dev)
print("Qb ptr", hex(Qb.data_ptr()), Qb.is_contiguous(), Qb.stride(), flush=True)
Qc = torch.from_numpy(inst.Q).to(dev)
print("Qc ptr", hex(Qc.data_ptr()), flush=True)
print("sums", float(Qb.sum()), float(Qc.sum()), float(d0.Q.sum()), flush=True)
for name, Q in (("Qc", Qc), ("Qb", Qb)):
    inst.drop_device_data()
    d = DeviceData.upload(inst, dev, None); d.Q = Q
    inst._dev[str(dev)] = d
    ev = inst._evaluator()
    x = torch.from_numpy(np.ones(2000)).to(dev)
    try:
        u, g, ms = ev.ctx.probe_sweep(x)
        print(name, "probe ok", float(u.sum()), ms, flush=True)
    except Exception as e:
        print(name, "probe FAIL", str(e)[:100], flush=True)
