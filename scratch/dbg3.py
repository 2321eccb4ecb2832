import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_golden
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
g = load_golden("c0")
arr = instances.config_instance("C0")
inst = R.ProblemInstance.from_arrays(arr, validate=False)
tg = g["nm_fixed500/trace"]
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
for rec in (False, True):
    res = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=True), R.FixedRestart(500), budget=1200, criteria=crit, record_restart_points=rec)
    tr = np.array([[t.iter, t.tau_start, t.tau, t.evals_iter, np.nan if t.kkt is None else t.kkt, t.restart_flag] for t in res.trace])
    k = min(len(tr), len(tg))
    bad = np.nonzero((tr[:k,1] != tg[:k,1]) | (tr[:k,2] != tg[:k,2]))[0]
    print("record", rec, "iters", res.iterations, "first diff", bad[:5])
    if len(bad):
        i = bad[0]
        print(np.c_[tr[i-3:i+3], tg[i-3:i+3][:, [0,1,2,5,7,10]]])
    print("kkt rows", tr[490:510:10, [0,4]].tolist(), tg[490:510:10][:, [0,7]].tolist())
