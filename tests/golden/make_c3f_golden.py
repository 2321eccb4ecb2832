"""Golden for config C3f at FULL size (n = 10^6, 64 factored quadratic rows
R_i^T R_i, 5*10^5 sparse linear rows; x0 ~ U(-0.01, 0.01) because BASELINE's
x0 ~ U(-1, 1) makes C3 infeasible -- tools/c3_infeasibility.py).

The reference cannot represent this instance (problem.py:137, :142-147 densify
every Q_i and run eigvalsh on it), so the checker is the oracle's factored
restatement ``O.FactoredProblem`` (oracle/rapdb_oracle.py), itself pinned
bit-for-bit against the real reference on a densifiable instance of the same
structure (factored_small.npz, tests/test_oracle_factored.py).

Cases (offline, ~1-2 h of one host core here; never run on the GPU box):
  mono_fixed500: yx monotone + FixedRestart(500), conic KKT 1e-6 -- the
                 configuration tools/measure_configs.py times, end to end;
  nm_200:        yx non-monotone, no restart, 200 iterations.

Full 10^6-vectors are not committed: each snapshot stores a fixed index
sample (every 997th entry), the 2-norm and three projections onto seeded
CounterRng directions, enough to bound the relative error of the full vector.

    python tests/golden/make_c3f_golden.py [--only mono_fixed500|nm_200]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import rapdb_oracle as O  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from paper_2605_29291_b200.instances import CounterRng  # noqa: E402

SAMPLE_STRIDE = 997
SNAPS = (1, 2, 5, 10, 50, 100, 150, 200, 499, 500, 501, 1000)
TRACE_COLS = ["iter", "tau_start", "tau", "sigma", "gamma", "evals_iter",
              "evals_total", "kkt", "infeas", "gap_xi", "restart_flag"]


def directions(length, seed=91):
    return np.stack([CounterRng(seed, k).normal(length) for k in range(3)])


def summary(vec, dirs):
    """(sample, norm, projections) of a long vector."""
    return vec[::SAMPLE_STRIDE].copy(), float(np.linalg.norm(vec)), dirs @ vec


def trace_array(trace):
    nan = float("nan")
    return np.array([[r.iter, r.tau_start, r.tau, r.sigma, r.gamma, r.evals_iter, r.evals_total,
                      nan if r.kkt is None else r.kkt, nan if r.infeas is None else r.infeas,
                      nan if r.gap_xi is None else r.gap_xi, r.restart_flag] for r in trace])


CASES = {
    "mono_fixed500": dict(nm=False, policy=dict(kind="fixed", period=500), budget=3000,
                          criteria=dict(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)),
    "nm_200": dict(nm=True, policy=dict(kind="none"), budget=200, criteria=None),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    t0 = time.time()
    arr = instances.factored_qcqp(x0_scale=0.01)
    P = O.FactoredProblem(arr)
    print("instance", round(time.time() - t0, 1), flush=True)
    dx, dl = directions(arr.n), directions(arr.m)
    out_path = os.path.join(HERE, "c3f_full.npz")
    arrays = dict(np.load(out_path)) if os.path.exists(out_path) else {}
    arrays["R_checksum"] = np.array([float(arr.R.data.sum()), float(arr.R.indices.sum())])
    arrays["A_checksum"] = np.array([float(arr.A.data.sum()), float(arr.A.indices.sum()),
                                     float(arr.b.sum())])
    arrays["C_checksum"] = np.array([float(arr.C.sum()), float(arr.d.sum())])
    meta_path = os.path.join(HERE, "c3f_full.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {"cases": {}}
    meta.update(instance="instances.factored_qcqp(x0_scale=0.01)", sample_stride=SAMPLE_STRIDE,
                directions="CounterRng(91, k).normal(len), k = 0, 1, 2", trace_cols=TRACE_COLS)
    for key, case in CASES.items():
        if a.only and key != a.only:
            continue
        snaps = {}

        def hook(total, eng):
            if eng.iters in SNAPS:
                snaps[eng.iters] = (summary(eng.x, dx), summary(eng.lam, dl))
            if eng.iters % 25 == 0:
                print(key, eng.iters, eng.evals_total, round(time.time() - t1, 1), flush=True)

        t1 = time.time()
        res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=case["nm"]),
                              O.Policy(**case["policy"]), budget=case["budget"],
                              criteria=case["criteria"], on_iter=hook)
        wall = time.time() - t1
        keys = sorted(snaps)
        pre = key + "/"
        arrays[pre + "trace"] = trace_array(res.trace)
        arrays[pre + "snap_iters"] = np.array(keys, dtype=np.int64)
        arrays[pre + "snap_x_sample"] = np.array([snaps[k][0][0] for k in keys])
        arrays[pre + "snap_x_norm"] = np.array([snaps[k][0][1] for k in keys])
        arrays[pre + "snap_x_proj"] = np.array([snaps[k][0][2] for k in keys])
        arrays[pre + "snap_lam_sample"] = np.array([snaps[k][1][0] for k in keys])
        arrays[pre + "snap_lam_norm"] = np.array([snaps[k][1][1] for k in keys])
        arrays[pre + "snap_lam_proj"] = np.array([snaps[k][1][2] for k in keys])
        fx, fl = summary(res.x, dx), summary(res.lam, dl)
        arrays[pre + "final_x_sample"], arrays[pre + "final_x_norm"], arrays[pre + "final_x_proj"] = fx
        arrays[pre + "final_lam_sample"], arrays[pre + "final_lam_norm"], arrays[pre + "final_lam_proj"] = fl
        met = res.metrics
        arrays[pre + "metrics"] = np.array([met.kkt_residual, met.stationarity, met.primal_eq,
                                            met.complementarity, met.infeas, met.f_value,
                                            met.mean_pos_violation])
        arrays[pre + "restart_iters"] = np.array([e[1] for e in res.restarts], dtype=np.int64)
        arrays[pre + "iterations"] = np.int64(res.iterations)
        arrays[pre + "evals"] = np.int64(res.evals)
        arrays[pre + "converged"] = np.int64(res.converged)
        meta["cases"][key] = dict(case, wall_s=wall, iterations=int(res.iterations),
                                  converged=bool(res.converged))
        np.savez_compressed(out_path, **arrays)
        with open(meta_path, "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        print("wrote", key, res.iterations, res.converged, round(wall, 1),
              os.path.getsize(out_path), flush=True)


if __name__ == "__main__":
    main()
