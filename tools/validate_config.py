"""Full-size parity of a BASELINE config against the CPU oracle (the numpy
restatement of the reference, oracle/rapdb_oracle.py, pinned bit-for-bit to
the real reference by tests/test_oracle_pin.py), run on the GPU box's host --
for configs whose stack is too large for a committed golden (C2: 69 GB).

  phase 1 (per step search in --modes): the first K accepted iterations of
          yx with no restart, step for step: (tau_start, tau, evals) bitwise,
          x / lam relative error at K/4, K/2, 3K/4, K (bar 1e-9);
  phase 2 (--kkt): yx monotone + FixedRestart(500) to conic KKT 1e-6 on both
          sides (restarts.py:111-170): iteration counts (bar 2 %), restart
          iterations, (tau, evals) while the runs coincide, final KKT,
          infeasibility and objective (bar 1e-6 relative).

    python tools/validate_config.py C2 --iters 200 --modes mono,nm --kkt > profiles/r02_validate_c2.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from oracle import rapdb_oracle as O  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--modes", default="mono,nm")
ap.add_argument("--kkt", action="store_true")
ap.add_argument("--budget", type=int, default=3000)
a = ap.parse_args()

t0 = time.time()
arr = instances.config_instance(a.config)
out = {"config": a.config, "n": arr.n, "m": arr.m, "generate_s": time.time() - t0, "phase1": {}, "phase2": None}
log("generated", out["generate_s"])
inst = R.ProblemInstance.from_arrays(arr, validate=False)
P = O.Problem.from_arrays(arr)
K = a.iters
marks = sorted({K // 4, K // 2, 3 * K // 4, K} - {0})

for mode in [m for m in a.modes.split(",") if m]:
    nm = mode == "nm"
    t1 = time.time()
    eng = O.Engine(P, O.Options(mode="yx", nonmonotone=nm), *O.initial_point(P))
    ref_snaps = {}
    for k in range(1, K + 1):
        eng.step()
        if k in marks:
            ref_snaps[k] = (eng.x.copy(), eng.lam.copy())
    cpu_s = time.time() - t1
    ref = np.array([[t.tau_start, t.tau, t.evals_iter] for t in eng.trace])
    t1 = time.time()
    dev = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.initial_iterate(inst))
    errs = {}
    done = 0
    for k in marks:
        dev.run_block(k - done)
        done = k
        z = dev.last
        errs[str(k)] = [rel(z.x, ref_snaps[k][0]), rel(z.lam, ref_snaps[k][1])]
    gpu_s = time.time() - t1
    got = np.array([[t.tau_start, t.tau, t.evals_iter] for t in dev.trace])
    same = bool(np.array_equal(got, ref))
    worst = max(max(v) for v in errs.values())
    out["phase1"][mode] = {"iterations": K, "steps_bitwise_equal": same, "rel_err_x_lam_at": errs,
                           "max_rel_err": worst, "evals": int(ref[:, 2].sum()), "cpu_oracle_s": cpu_s,
                           "device_s": gpu_s, "pass": bool(same and worst <= 1e-9)}
    log(mode, json.dumps(out["phase1"][mode]))
    del dev

if a.kkt:
    crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
    t1 = time.time()
    dres = R.run_restarted(inst, R.SolverConfig(mode="yx", nonmonotone=False), R.FixedRestart(500),
                           budget=a.budget, criteria=crit)
    gpu_s = time.time() - t1
    t1 = time.time()
    ores = O.run_restarted(P, O.Options(mode="yx", nonmonotone=False), O.Policy(kind="fixed", period=500),
                           budget=a.budget, criteria=dict(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6))
    cpu_s = time.time() - t1
    td = np.array([[t.tau_start, t.tau, t.evals_iter] for t in dres.trace])
    to = np.array([[t.tau_start, t.tau, t.evals_iter] for t in ores.trace])
    k = min(len(td), len(to))
    eq = np.all(td[:k] == to[:k], axis=1)
    first_diff = None if eq.all() else int(np.argmin(eq)) + 1
    dm, om = dres.metrics, ores.metrics

    def rdiff(x, y):
        return abs(x - y) / max(abs(y), 1e-300)

    res = {"policy": "yx monotone + FixedRestart(500), conic KKT 1e-6",
           "device": {"iterations": dres.iterations, "evals": dres.evals, "converged": bool(dres.converged),
                      "restarts": [e.iteration for e in dres.restart_log], "kkt": dm.kkt_residual,
                      "infeas": dm.infeas, "f": dm.f_value, "wall_s": gpu_s},
           "oracle": {"iterations": ores.iterations, "evals": ores.evals, "converged": bool(ores.converged),
                      "restarts": [e[1] for e in ores.restarts], "kkt": om.kkt_residual,
                      "infeas": om.infeas, "f": om.f_value, "wall_s": cpu_s},
           "steps_identical": int(eq[:k].sum()), "steps_compared": k, "first_step_difference": first_diff,
           "rel_diff": {"kkt": rdiff(dm.kkt_residual, om.kkt_residual), "infeas": rdiff(dm.infeas, om.infeas),
                        "f": rdiff(dm.f_value, om.f_value)},
           "final_x_rel": rel(dres.solution.x, ores.x), "final_lam_rel": rel(dres.solution.lam, ores.lam)}
    # the metrics' evaluation floor: device vs oracle evaluation at the SAME
    # point (the oracle's final iterate); the residuals are ~1e-6 and formed
    # by cancellation, so their rounding floor is ~1e-12 absolute
    zo = R.Iterate(ores.x, ores.v, ores.lam)
    md = R.kkt_residual(inst, zo)
    floor = {"kkt": abs(md.kkt_residual - om.kkt_residual), "infeas": abs(md.infeas - om.infeas),
             "f": abs(md.f_value - om.f_value)}
    res["eval_floor_abs"] = floor
    ok_metrics = all(abs(a_ - b_) <= 1e-6 * abs(b_) + 2.0 * floor[k_]
                     for k_, a_, b_ in (("kkt", dm.kkt_residual, om.kkt_residual), ("infeas", dm.infeas, om.infeas),
                                        ("f", dm.f_value, om.f_value)))
    res["pass"] = bool(abs(dres.iterations - ores.iterations) <= 0.02 * ores.iterations
                       and res["device"]["restarts"] == res["oracle"]["restarts"]
                       and ok_metrics and dres.converged == ores.converged)
    out["phase2"] = res
    log("kkt", json.dumps(res))
print(json.dumps(out))
