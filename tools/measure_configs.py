"""Full-size runs of the BASELINE configs other than the bench workload (C1):
time per iteration, sweep bandwidth, time-to-KKT where the budget allows.
Prints one JSON object per run (append to profiles/ by hand).

    python tools/measure_configs.py C2 [budget] [mono|nm]      (device-generated dense stack)
    python tools/measure_configs.py C3 [budget] [mono|nm]      (factored sparse, host CounterRng)
    python tools/measure_configs.py C4 [budget] [mono|nm]      (KML epigraph, host CounterRng)
    python tools/measure_configs.py C0 [budget] [mono|nm]
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import _capi, instances  # noqa: E402

name = sys.argv[1]
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
nm = len(sys.argv) > 3 and sys.argv[3] == "nm"
policy_name = sys.argv[4] if len(sys.argv) > 4 else "fixed500"
t0 = time.perf_counter()
if name == "C2":
    inst = R.DeviceDenseInstance(4096, 512, 256, seed=0, name="C2 (device-generated)")
elif name == "C3":
    arr = instances.factored_qcqp()
    inst = R.FactoredInstance.from_arrays(arr)
elif name == "C3f":   # C3 with x0 ~ U(-0.01, 0.01): the BASELINE C3 (x0 ~ U(-1, 1)) is infeasible
    arr = instances.factored_qcqp(x0_scale=0.01)
    inst = R.FactoredInstance.from_arrays(arr)
else:
    arr = instances.config_instance(name)
    inst = R.ProblemInstance.from_arrays(arr, validate=False)
gen_s = time.perf_counter() - t0
dev = torch.device("cuda", 0)
t0 = time.perf_counter()
inst.device_data(dev)
torch.cuda.synchronize()
up_s = time.perf_counter() - t0
cfg = R.SolverConfig(mode="yx", nonmonotone=nm)
pol = R.FixedRestart(500) if policy_name == "fixed500" else (
    R.AdaptiveRestart() if policy_name == "adaptive" else R.NoRestart())
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
os.environ["RAPDB_STEP_PROFILE"] = "1"
res = None
for rep in range(1 if name == "C4" else 2):   # the first run of a process carries one-time host setup
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = R.run_restarted(inst, cfg, pol, budget=budget, criteria=crit, device=dev)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
st = res.device_stats
factored = hasattr(inst, "rblk")
prof = st.get("step_profile") or {}
sweep_ms = sum(v[0] for k, v in prof.items() if k.endswith("SWEEP"))
sweeps = sum(v[1] for k, v in prof.items() if k.endswith("SWEEP"))
out = {
    "config": name, "instance": getattr(inst, "name", ""), "n": inst.n, "m": inst.m,
    "policy": f"yx {'nonmonotone' if nm else 'monotone'} + {policy_name}", "budget": budget,
    "iterations": res.iterations, "evals": res.evals, "converged": res.converged,
    "final_kkt": res.metrics.kkt_residual, "final_infeas": res.metrics.infeas,
    "f": res.metrics.f_value, "wall_s": dt, "iters_per_s": res.iterations / dt,
    "ms_per_iter": 1e3 * dt / max(res.iterations, 1), "kernel_ms": st["kernel_ms"],
    "sweep_bytes": st["sweep_bytes"], "sweeps": sweeps, "sweep_ms_total": sweep_ms,
    "sweep_ms_each": sweep_ms / max(sweeps, 1),
    # the in-kernel sweep timer does not see the factored path's host-launched
    # kernels: no sweep GB/s there (see eval_* below)
    "sweep_gbs": None if factored else st["sweep_bytes"] * sweeps / max(sweep_ms, 1e-9) / 1e6,
    "time_to_kkt_s": dt if res.converged else None,
    "generate_s": gen_s, "upload_s": up_s,
    "step_profile_ms": {k: round(v[0], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])[:8]},
}
if factored:
    # SURVEY 8(d) algorithmic bytes of one test evaluation (12 B per CSR nnz):
    # R x and R^T(w W) over R, c_i . x and sum w_i c_i over C, A x and A^T mu
    nnz_r, nnz_a = int(inst.R.nnz), int(inst.A.nnz)
    eval_bytes = 2 * 12 * nnz_r + 2 * 8 * (inst.mq + 1) * inst.n + 2 * 12 * nnz_a
    per_eval = dt / max(res.evals, 1)
    out.update({"eval_bytes": eval_bytes, "us_per_eval": 1e6 * per_eval,
                "eval_gbs": eval_bytes / per_eval / 1e9, "eval_frac_of_6552": eval_bytes / per_eval / 1e9 / 6552.0})
print(json.dumps(out))
