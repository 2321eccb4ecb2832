import cProfile, pstats, os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
arr = instances.config_instance("C1")
inst = R.ProblemInstance.from_arrays(arr, validate=False)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
cfg = R.SolverConfig(mode="yx", nonmonotone=False)
for _ in range(2):
    R.run_restarted(inst, cfg, R.FixedRestart(500), criteria=crit)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
res = R.run_restarted(inst, cfg, R.FixedRestart(500), criteria=crit)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0, "kernel", res.device_stats["kernel_ms"])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
