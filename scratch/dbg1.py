import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200.geometry import Box, NonnegOrthant
g = load_golden("small_qcqp")
inst = R.ProblemInstance(n=20, m=3, p=0, Q=g["Q"], q=g["q"], r=g["r"], A=np.zeros((0,20)), b=np.zeros(0), primal_set=Box(g["lower"], g["upper"]), cone=NonnegOrthant(3))
key = "yx_mono"
tg = g[f"{key}/trace"]
for chunks in ([10], [1,1,8], [2, 8], [1, 9]):
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx"), R.initial_iterate(inst))
    for c in chunks:
        eng.run_block(c)
    tr = np.array([[t.tau_start, t.tau, t.evals_iter] for t in eng.trace])
    x = eng.last.x
    print(chunks, "x err", np.linalg.norm(x - g[f"{key}/snap_x"][9]) / np.linalg.norm(g[f"{key}/snap_x"][9]))
    print(np.c_[tr, tg[:10, 1:3], tg[:10,5]])
