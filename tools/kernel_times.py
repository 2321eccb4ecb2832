"""Per-kernel device time of a short solve via CUPTI (torch.profiler), not
under ncu (warm caches, real clocks): python tools/kernel_times.py C3f|C1|C4 [iters]"""
import os
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3f"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if name == "C3f":
    inst = R.FactoredInstance.from_arrays(instances.factored_qcqp(x0_scale=0.01))
else:
    inst = R.ProblemInstance.from_arrays(instances.config_instance(name), validate=False)
cfg = R.SolverConfig(mode="yx", nonmonotone=name == "C4")
R.run_restarted(inst, cfg, R.FixedRestart(500), budget=3)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    res = R.run_restarted(inst, cfg, R.FixedRestart(500), budget=iters)
    t1.record()
    torch.cuda.synchronize()
tot = defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        k = e.name[:60]
        tot[k][0] += 1
        tot[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
span = t0.elapsed_time(t1) * 1e3
busy = sum(v[1] for v in tot.values())
print(f"{name}: {res.iterations} it, {res.evals} evals; span {span / 1e3:.2f} ms, kernels {busy / 1e3:.2f} ms "
      f"({100 * busy / span:.1f}% busy); per eval {span / max(res.evals, 1):.1f} us")
for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {c:6d}  {t / 1e3:9.2f} ms  {t / c:8.1f} us/launch  {t / max(res.evals, 1):7.1f} us/eval  {k}")
# idle gap in front of each device activity (start - end of the previous one), by activity name
evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
             key=lambda e: e.time_range.start)
gap = defaultdict(lambda: [0, 0.0])
prev_end = None
for e in evs:
    if prev_end is not None:
        g = max(0.0, e.time_range.start - prev_end)
        gap[e.name[:60]][0] += 1
        gap[e.name[:60]][1] += g
    prev_end = max(prev_end or 0, e.time_range.end)
print("idle before:")
for k, (c, t) in sorted(gap.items(), key=lambda kv: -kv[1][1])[:8]:
    print(f"  {c:6d}  {t / 1e3:9.2f} ms  {t / c:8.1f} us each  {t / max(res.evals, 1):7.1f} us/eval  {k}")
