import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200.geometry import Box, NonnegOrthant
g = load_golden("small_qcqp")
inst = R.ProblemInstance(n=20, m=3, p=0, Q=g["Q"], q=g["q"], r=g["r"], A=np.zeros((0,20)), b=np.zeros(0), primal_set=Box(g["lower"], g["upper"]), cone=NonnegOrthant(3))
for key, nm in (("yx_mono", False), ("yx_nm", True)):
    eng = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.initial_iterate(inst))
    for k in range(1, 13):
        eng.run_block(1)
        z = eng.last
        xs = g[f"{key}/snap_x"][k-1]; ls = g[f"{key}/snap_lam"][k-1]
        print(key, k, "x", np.linalg.norm(z.x-xs)/np.linalg.norm(xs), "lam", z.lam, ls)
