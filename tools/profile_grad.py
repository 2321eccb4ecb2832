"""One OP_GRAD launch (sweep + gradient recombination) at a random point, for
ncu: python tools/profile_grad.py [C3|C1|...] [calls]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if name == "C3":
    inst = R.FactoredInstance.from_arrays(instances.factored_qcqp())
else:
    inst = R.ProblemInstance.from_arrays(instances.config_instance(name), validate=False)
ev = inst._evaluator()
rng = np.random.default_rng(0)
dev = ev.ctx.device
x = torch.from_numpy(rng.uniform(-1, 1, inst.n)).to(dev)
v = torch.zeros(max(inst.p, 1), dtype=torch.float64, device=dev)
lam = torch.from_numpy(rng.uniform(0, 1, inst.m)).to(dev)
for _ in range(calls):
    ev.ctx.grad_x(x, v, lam)
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(5):
    ev.ctx.grad_x(x, v, lam)
s1.record()
torch.cuda.synchronize()
print(f"{name}: grad_x (sweep + recombination) {s0.elapsed_time(s1) / 5:.3f} ms/call")
