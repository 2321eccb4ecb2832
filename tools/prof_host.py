"""Host-side profile of one warm solve: python tools/prof_host.py [C1] [fixed|adaptive]"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
pol_name = sys.argv[2] if len(sys.argv) > 2 else "fixed"
arr = instances.config_instance(name)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
cfg = R.SolverConfig(mode="yx", nonmonotone=False)
pol = R.FixedRestart(500) if pol_name == "fixed" else R.AdaptiveRestart()
for _ in range(2):
    R.run_restarted(inst, cfg, pol, criteria=crit)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
res = R.run_restarted(inst, cfg, pol, criteria=crit)
torch.cuda.synchronize()
print("wall", time.perf_counter() - t0, "kernel", res.device_stats["kernel_ms"], "iters", res.iterations)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
