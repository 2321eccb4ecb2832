"""One fused C1 sweep (OP_PROBE launch) for ncu --set full; also prints its
CUDA-event time.  Usage: python tools/profile_sweep.py [C1|C0|C2 ...] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
arr = instances.config_instance(name)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
ev = inst._evaluator()
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, arr.n)).cuda()
for _ in range(2):
    ev.ctx.probe_sweep(x, reps=1)
u, g, ms = ev.ctx.probe_sweep(x, reps=reps)
bytes_ = (arr.m + 1) * arr.n * arr.n * 8
print(f"{name}: {ms:.4f} ms/sweep  {bytes_ / ms / 1e6:.1f} GB/s  (reps={reps})")
