"""Standalone packed-sweep time vs stack shape (device-generated dense
instances): separates the per-unit cost from the per-sweep fixed cost.
python tools/sweep_scan.py n m1 m2 ...   (env passes through, e.g. RAPDB_EARLY_CHUNKS)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import _capi  # noqa: E402

n = int(sys.argv[1])
for m in [int(a) for a in sys.argv[2:]]:
    inst = R.DeviceDenseInstance(n, m, min(n, 64), seed=1)
    ev = inst._evaluator()
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    for _ in range(2):
        ev.ctx.probe_sweep(x, reps=1)
    _, _, ms = ev.ctx.probe_sweep(x, reps=100)
    b = (m + 1) * _capi.packed_doubles(n) * 8
    units = (m + 1) * ((n + 63) // 64) * ((n + 63) // 64 + 1) // 2
    print(f"n={n} m+1={m + 1}: {ms * 1e3:8.2f} us/sweep  {b / ms / 1e6:7.1f} GB/s  units={units}  "
          f"{ms * 1e3 / units * 148:6.3f} us per unit per CTA", flush=True)
    del ev, inst
    torch.cuda.empty_cache()
