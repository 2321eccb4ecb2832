"""EGM runs of the REAL reference (rapdb.egm.run_egm / tune_egm) on the
reference's own test instance random_qcqp(20, 3, seed=3) and on the analytic
eq-qp KAT (equality block) -> tests/golden/egm.npz.  Run in the build
container (/root/reference present)."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from rapdb import diagnostics, egm, generate  # noqa: E402
from rapdb.engine import initial_iterate  # noqa: E402
from rapdb.geometry import JointBall  # noqa: E402

arrays, meta = {}, {"cases": {}}
inst = generate.random_qcqp(20, 3, seed=3)
eq = [a for a in generate.analytic_suite() if a.name == "eq-qp"][0].instance
cases = {
    "rq_s01": (inst, 0.1, 300, None, 50),
    "rq_s003": (inst, 0.03, 300, None, 0),
    "rq_s1": (inst, 1.0, 300, None, 10),          # large step
    "rq_s10_div": (inst, 10.0, 300, None, 5),     # diverges at 126
    "rq_joint": (inst, 0.1, 200, JointBall(2.0), 0),
    "eq_s02": (eq, 0.2, 200, None, 20),
}
for key, (I, s, K, ball, te) in cases.items():
    res = egm.run_egm(I, s, initial_iterate(I), K, dual_ball=ball, trace_every=te)
    for name, z in (("last", res.last), ("avg", res.average)):
        arrays[f"{key}/{name}_x"] = z.x
        arrays[f"{key}/{name}_v"] = z.v
        arrays[f"{key}/{name}_lam"] = z.lam
    arrays[f"{key}/iterations"] = np.int64(res.iterations)
    arrays[f"{key}/diverged"] = np.int64(res.diverged)
    arrays[f"{key}/trace"] = np.array([[t["iter"], t["norm"]] for t in res.trace]).reshape(-1, 2)
    meta["cases"][key] = {"step": s, "K": K, "ball": None if ball is None else 2.0, "trace_every": te}


def score(z):
    return diagnostics.kkt_residual(inst, z).kkt_residual


best_s, best = egm.tune_egm(inst, initial_iterate(inst), 100, score)
arrays["tune/best_s"] = np.float64(best_s)
arrays["tune/last_x"] = best.last.x
np.savez_compressed(os.path.join(HERE, "egm.npz"), **arrays)
json.dump(meta, open(os.path.join(HERE, "egm.json"), "w"), indent=1, sort_keys=True)
print("wrote egm.npz", {k: int(arrays[f'{k}/iterations']) for k in cases}, "tune", best_s)
