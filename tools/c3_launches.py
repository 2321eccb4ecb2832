"""A short C3f solve (x0 ~ U(-0.01, 0.01)) for a kernel launch list:
ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
    --log-file gpurun_out/c3.csv python tools/c3_launches.py [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
inst = R.FactoredInstance.from_arrays(instances.factored_qcqp(x0_scale=0.01))
cfg = R.SolverConfig(mode="yx")
R.run_restarted(inst, cfg, R.FixedRestart(500), budget=3)   # warm-up (binds, uploads)
torch.cuda.synchronize()
res = R.run_restarted(inst, cfg, R.FixedRestart(500), budget=iters)
torch.cuda.synchronize()
print(res.iterations, res.evals)
