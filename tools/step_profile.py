"""Per-step device time of one solve (CTA 0 globaltimer, rapdb_step_profile).
python tools/step_profile.py [C1] [mono|nm]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from paper_2605_29291_b200.engine import ApdbEngine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
nm = len(sys.argv) > 2 and sys.argv[2] == "nm"
mode = sys.argv[3] if len(sys.argv) > 3 else "yx"
pol_name = sys.argv[4] if len(sys.argv) > 4 else "fixed"
arr = instances.config_instance(name)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
cfg = R.SolverConfig(mode=mode, nonmonotone=nm)
pol = R.FixedRestart(500) if pol_name == "fixed" else R.AdaptiveRestart()
for k in range(int(os.environ.get("REPS", "2"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = R.run_restarted(inst, cfg, pol, budget=1000 if nm else 50_000, criteria=crit)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"solve {k}: {dt * 1e3:.1f} ms wall, kernel {res.device_stats['kernel_ms']:.1f} ms", flush=True)
print(f"{name} {'nm' if nm else 'mono'}: {res.iterations} it, {res.evals} evals, {dt * 1e3:.1f} ms "
      f"({res.iterations / dt:.1f} it/s), kernel {res.device_stats['kernel_ms']:.1f} ms, "
      f"sweeps {res.device_stats['sweeps']} in {res.device_stats['sweep_ns'] / 1e6:.1f} ms")
prof = res.device_stats.get("step_profile") or {}
tot = sum(v[0] for v in prof.values())
for k, (ms, cnt) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:10s} {ms:9.3f} ms  {cnt:7d} calls  {1e3 * ms / max(cnt, 1):8.2f} us/call  {100 * ms / tot:5.1f}%")
