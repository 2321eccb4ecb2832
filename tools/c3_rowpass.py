"""Time the factored row pass and gradient alone (CUPTI): repeated g(x) and
grad_x Phi(x, lam) evaluations of the C3f instance through the public point
evaluators.  python tools/c3_rowpass.py [reps]   (RAPDB_LIB selects an A/B build)"""
import os
import sys
from collections import defaultdict

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
inst = R.FactoredInstance.from_arrays(instances.factored_qcqp(x0_scale=0.01))
rng = np.random.default_rng(0)
x = rng.uniform(-0.01, 0.01, inst.n)
lam = np.abs(rng.normal(size=inst.m)) * 0.01
z = R.Iterate(x, np.zeros(0), lam)
inst.g_value(x)
R.grad_x_coupling(inst, z)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        inst.g_value(x)
        R.grad_x_coupling(inst, z)
    torch.cuda.synchronize()
tot = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "fac_" in e.name:
        tot[e.name[:50]][0] += 1
        tot[e.name[:50]][1] += e.device_time_total
for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"  {c:5d}  {t / c:8.1f} us/launch  {k}")
