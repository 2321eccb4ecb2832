import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
for (n, m, r) in [(2000, 10, 20), (2000, 200, 200)]:
    arr = instances.dense_qcqp(n, m, r, seed=0)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
    for it in range(3):
        t = time.time()
        try:
            eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx"), R.initial_iterate(inst))
            print(n, m, "reinit ok", time.time() - t, flush=True)
            eng.run_block(20)
            print(n, m, "run ok", time.time() - t, eng.trace[-1].tau, flush=True)
        except Exception as e:
            print(n, m, "FAIL", type(e).__name__, e, time.time() - t, flush=True)
