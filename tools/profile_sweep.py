"""One fused sweep (OP_PROBE launch) for ncu --set full; also prints its
CUDA-event time.  Usage: python tools/profile_sweep.py [C1|C0|C2 ...] [reps]
(env RAPDB_LAYOUT=rows|packed selects the Q-stack layout)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import _capi, instances  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if name == "C2":   # device-generated: the host instance takes minutes and 69 GB
    inst = R.DeviceDenseInstance(4096, 512, 256)
    arr = inst
else:
    arr = instances.config_instance(name)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
ev = inst._evaluator()
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, arr.n)).cuda()
for _ in range(2):
    ev.ctx.probe_sweep(x, reps=1)
u, g, ms = ev.ctx.probe_sweep(x, reps=reps)
dense = (arr.m + 1) * arr.n * arr.n * 8
layout = getattr(ev.ctx.data, "layout", "rows")
streamed = (arr.m + 1) * _capi.packed_doubles(arr.n) * 8 if layout == "packed" else dense
print(f"{name} [{layout}]: {ms:.4f} ms/sweep  {streamed / ms / 1e6:.1f} GB/s streamed "
      f"({streamed / 1e9:.3f} GB)  {dense / ms / 1e6:.1f} GB/s dense-equivalent  (reps={reps})")
os.makedirs("gpurun_out", exist_ok=True)
open(f"gpurun_out/streamed_{name}.txt", "w").write(str(int(streamed)))
