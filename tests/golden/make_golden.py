"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures (~1 min)
    python tests/golden/make_golden.py --c1       # + C1 200-iteration traces (~10 min)

Every fixture records inputs that cannot be regenerated bit-for-bit elsewhere
(the reference's own ``random_qcqp`` instance arrays) plus the reference's
outputs: per-iteration traces (tau_start, tau, sigma, gamma, evals), restart
events, gap values, iterate snapshots, KKT metrics.  The GPU box never reads
/root/reference; tests read only these committed files.
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
sys.path.insert(0, "/root/reference/pkg/src")

import rapdb  # noqa: E402  (the reference package)
from rapdb import diagnostics, generate  # noqa: E402
from rapdb.geometry import Box, JointBall, NonnegOrthant, SplitBall  # noqa: E402
from rapdb.restarts import AdaptiveRestart, FixedRestart, NoRestart  # noqa: E402

from paper_2605_29291_b200 import instances  # noqa: E402

TRACE_COLS = ["iter", "tau_start", "tau", "sigma", "gamma", "evals_iter",
              "evals_total", "kkt", "infeas", "gap_xi", "restart_flag"]


def trace_array(trace):
    nan = float("nan")
    rows = [[r.iter, r.tau_start, r.tau, r.sigma, r.gamma, r.evals_iter, r.evals_total,
             nan if r.kkt is None else r.kkt, nan if r.infeas is None else r.infeas,
             nan if r.gap_xi is None else r.gap_xi, r.restart_flag] for r in trace]
    return np.array(rows, dtype=np.float64).reshape(-1, len(TRACE_COLS))


def ref_instance(arr):
    return rapdb.ProblemInstance(
        n=arr.n, m=arr.m, p=arr.p, Q=arr.Q_list(), q=arr.q_list(), r=arr.r,
        A=arr.A, b=arr.b, primal_set=Box(arr.lower, arr.upper),
        cone=NonnegOrthant(arr.m), mu=arr.mu, name=arr.name)


def policy_of(spec):
    kind = spec["kind"]
    if kind == "none":
        return NoRestart()
    if kind == "fixed":
        return FixedRestart(spec["period"], point=spec.get("point", "last"))
    return AdaptiveRestart(xi=spec.get("xi", 0.04), q=spec.get("q", 0.5),
                           warmup=spec.get("warmup", 50),
                           check_period=spec.get("check_period", 200),
                           point=spec.get("point", "last"))


def ball_of(spec):
    if spec is None:
        return rapdb.engine.Unbounded()
    if spec[0] == "joint":
        return JointBall(spec[1])
    return SplitBall(spec[1], spec[2])


def run_case(inst, case, snap_iters):
    """Run run_restarted with a per-iteration hook capturing snapshots."""
    cfg = rapdb.SolverConfig(mode=case.get("mode", "yx"), nonmonotone=case["nm"],
                             dual_ball=ball_of(case.get("ball")))
    crit = None
    if case.get("eps") is not None:
        if case.get("criterion", "conic") == "conic":
            crit = diagnostics.TerminationCriteria(criterion="conic", eps_kkt=case["eps"],
                                                   eps_feas=case["eps"],
                                                   f_star=case.get("f_star"))
        else:   # "paper51" (diagnostics.py:254-258): relative f-gap + mean violation
            crit = diagnostics.TerminationCriteria(criterion="paper51", eps=case["eps"],
                                                   f_star=case.get("f_star"))
    snaps_x, snaps_lam, snaps_v = {}, {}, {}
    orig_step = rapdb.engine.ApdbEngine.step

    def hooked(self):
        rec = orig_step(self)
        if rec.iter in snap_iters:
            snaps_x[rec.iter] = self.z.x.copy()
            snaps_lam[rec.iter] = self.z.lam.copy()
            snaps_v[rec.iter] = self.z.v.copy()
        return rec

    rapdb.engine.ApdbEngine.step = hooked
    try:
        t0 = time.time()
        res = rapdb.run_restarted(inst, cfg, policy_of(case["policy"]),
                                  budget=case["budget"], criteria=crit,
                                  metrics_every=10, warm_tau=case.get("warm_tau", False))
        wall = time.time() - t0
    finally:
        rapdb.engine.ApdbEngine.step = orig_step
    keys = sorted(snaps_x)
    met = res.metrics
    out = {
        "trace": trace_array(res.trace),
        "subopt": np.array([np.nan if r.subopt is None else r.subopt for r in res.trace]),
        "snap_iters": np.array(keys, dtype=np.int64),
        "snap_x": np.array([snaps_x[k] for k in keys]).reshape(len(keys), -1),
        "snap_lam": np.array([snaps_lam[k] for k in keys]).reshape(len(keys), -1),
        "snap_v": np.array([snaps_v[k] for k in keys]).reshape(len(keys), -1),
        "final_x": res.solution.x, "final_lam": res.solution.lam, "final_v": res.solution.v,
        "avg_x": res.average.x, "avg_lam": res.average.lam, "avg_v": res.average.v,
        "restart_iters": np.array([e.iteration for e in res.restart_log], dtype=np.int64),
        "restart_gaps": np.array([[np.nan if e.gap_new is None else e.gap_new,
                                   np.nan if e.gap_ref is None else e.gap_ref]
                                  for e in res.restart_log]).reshape(-1, 2),
        "metrics": np.array([met.kkt_residual, met.stationarity, met.primal_eq,
                             met.complementarity, met.infeas, met.f_value,
                             met.mean_pos_violation]),
        "iterations": np.int64(res.iterations), "evals": np.int64(res.evals),
        "converged": np.int64(res.converged),
        "subopt_final": np.float64(np.nan if met.subopt_abs is None else met.subopt_abs),
    }
    return out, wall


def save(name, arrays, meta):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    with open(os.path.join(HERE, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)/1e3:.0f} kB)")


def small_fixtures():
    # 1. the reference's own conftest instance random_qcqp(20, 3, seed=3): store arrays
    inst = generate.random_qcqp(20, 3, seed=3)
    arrays = {"Q": np.array([np.asarray(M) for M in inst.Q]), "q": np.array(inst.q),
              "r": inst.r, "lower": inst.primal_set.lower, "upper": inst.primal_set.upper}
    cases = {
        "yx_mono": dict(nm=False, policy={"kind": "none"}, budget=200),
        "yx_nm": dict(nm=True, policy={"kind": "none"}, budget=200),
        "xy_mono": dict(mode="xy", nm=False, policy={"kind": "none"}, budget=200),
        "xy_nm": dict(mode="xy", nm=True, policy={"kind": "none"}, budget=200),
        "yx_nm_joint5": dict(nm=True, ball=("joint", 5.0), policy={"kind": "none"}, budget=200),
        "yx_nm_split": dict(nm=True, ball=("split", 1.0, 0.7), policy={"kind": "none"}, budget=150),
        "yx_nm_fixed40avg": dict(nm=True, policy={"kind": "fixed", "period": 40, "point": "average"}, budget=200),
        "yx_nm_ada": dict(nm=True, policy={"kind": "adaptive", "warmup": 50, "check_period": 100},
                          budget=1500, eps=1e-8),
    }
    meta = {"instance": "rapdb.generate.random_qcqp(20, 3, seed=3)", "cases": {}}
    for key, case in cases.items():
        out, wall = run_case(inst, case, set(range(1, 201)))
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = {k: (list(v) if isinstance(v, tuple) else v) for k, v in case.items()}
        meta["cases"][key]["wall_s"] = wall
    save("small_qcqp", arrays, meta)

    # 2. analytic suite (generate.py:195-256) -- KATs
    arrays, meta = {}, {"cases": {}}
    for a in generate.analytic_suite():
        inst = a.instance
        arrays[f"{a.name}/Q"] = np.array([np.asarray(M.toarray() if hasattr(M, "toarray") else M)
                                           for M in inst.Q])
        arrays[f"{a.name}/q"] = np.array(inst.q)
        arrays[f"{a.name}/r"] = inst.r
        arrays[f"{a.name}/A"] = np.asarray(inst.A)
        arrays[f"{a.name}/b"] = inst.b
        arrays[f"{a.name}/lower"] = inst.primal_set.lower
        arrays[f"{a.name}/upper"] = inst.primal_set.upper
        arrays[f"{a.name}/mu"] = np.float64(inst.mu)
        arrays[f"{a.name}/x_star"] = a.z_star.x
        arrays[f"{a.name}/v_star"] = a.z_star.v
        arrays[f"{a.name}/lam_star"] = a.z_star.lam
        arrays[f"{a.name}/f_star"] = np.float64(a.f_star)
        for key, case in {"nm_fixed500": dict(nm=True, policy={"kind": "fixed", "period": 500},
                                              budget=5000, eps=1e-7),
                          "mono_fixed5": dict(nm=False, policy={"kind": "fixed", "period": 5}, budget=23),
                          "xy_nm": dict(mode="xy", nm=True, policy={"kind": "none"}, budget=300)}.items():
            out, wall = run_case(inst, case, set(range(1, 31)))
            for k, v in out.items():
                arrays[f"{a.name}/{key}/{k}"] = v
            meta["cases"][f"{a.name}/{key}"] = dict(case, wall_s=wall)
    save("analytic", arrays, meta)

    # 3. C0 (BASELINE config 0) -- four policies; arrays regenerated from the seed
    arr = instances.config_instance("C0")
    inst = ref_instance(arr)
    rng = np.random.default_rng(7)
    x_probe = rng.uniform(-1, 1, arr.n)
    arrays = {
        "Q_checksum": np.array([float(np.sum(arr.Q[i])) for i in range(arr.m + 1)]),
        "Q_sample": arr.Q[:, :3, :5].copy(),
        "probe_x": x_probe,
        "probe_u": np.array([np.asarray(M @ x_probe) for M in inst.Q]),
        "probe_g": inst.g_value(x_probe), "probe_f": np.float64(inst.f_value(x_probe)),
    }
    cases = {
        "nm_ada": dict(nm=True, policy={"kind": "adaptive", "xi": 0.04, "q": 0.5, "warmup": 50,
                                        "check_period": 200}, budget=50000, eps=1e-6),
        "mono_ada": dict(nm=False, policy={"kind": "adaptive", "xi": 0.04, "q": 0.5, "warmup": 50,
                                           "check_period": 200}, budget=50000, eps=1e-6),
        "nm_fixed500": dict(nm=True, policy={"kind": "fixed", "period": 500}, budget=50000, eps=1e-6),
        "mono_none": dict(nm=False, policy={"kind": "none"}, budget=50000, eps=1e-6),
        "xy_nm_none": dict(mode="xy", nm=True, policy={"kind": "none"}, budget=200),
    }
    meta = {"instance": "instances.config_instance('C0')", "cases": {}}
    for key, case in cases.items():
        out, wall = run_case(inst, case, set(range(1, 201)))
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = dict(case, wall_s=wall)
        print(key, "iterations", out["iterations"], "wall", round(wall, 2))
    save("c0", arrays, meta)

    kml_fixtures()


def kml_fixtures():
    # 4. C4-shaped small KML epigraph (N=120): p = 1, free t, zero Q0.  Both
    # step searches under FixedRestart(500): nm stops at the 3000 budget, mono
    # converges after ~12k iterations (the full-size C4 mono run is far slower)
    arr = instances.kml_epigraph(N=120, d=10)
    inst = ref_instance(arr)
    arrays, meta = {}, {"instance": "instances.kml_epigraph(N=120, d=10)", "cases": {}}
    arrays["Q_checksum"] = np.array([float(np.sum(arr.Q[i])) for i in range(arr.m + 1)])
    for key, case in {"nm_fixed500": dict(nm=True, policy={"kind": "fixed", "period": 500},
                                          budget=3000, eps=1e-6),
                      "mono_fixed500": dict(nm=False, policy={"kind": "fixed", "period": 500},
                                            budget=20000, eps=1e-6)}.items():
        out, wall = run_case(inst, case, set(range(1, 201)))
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = dict(case, wall_s=wall)
        print("kml", key, out["iterations"], out["converged"], wall)
    save("kml_small", arrays, meta)


def factored_fixtures():
    """5. C3-shaped factored instance, small enough to densify: the reference is
    given Q_i = R_i^T R_i explicitly (its _as_operator stores them as CSR) and
    the linear rows as Q = 0 orthant constraints (FactoredArrays.dense_lists)."""
    arr = instances.factored_qcqp(**FACTORED_SMALL)
    Q, q, r = arr.dense_lists()
    inst = rapdb.ProblemInstance(n=arr.n, m=arr.m, p=0, Q=Q, q=q, r=r, A=np.zeros((0, arr.n)),
                                 b=np.zeros(0), primal_set=Box(arr.lower, arr.upper),
                                 cone=NonnegOrthant(arr.m), mu=0.0, name=arr.name)
    rng = np.random.default_rng(11)
    x_probe = rng.uniform(-1, 1, arr.n)
    lam_probe = np.maximum(rng.normal(size=arr.m), 0.0)
    z = rapdb.Iterate(x_probe, np.zeros(0), lam_probe)
    arrays = {
        "R_checksum": np.array([float(arr.R.data.sum()), float(arr.R.indices.sum())]),
        "A_checksum": np.array([float(arr.A.data.sum()), float(arr.A.indices.sum()), float(arr.b.sum())]),
        "probe_x": x_probe, "probe_lam": lam_probe,
        "probe_g": inst.g_value(x_probe), "probe_f": np.float64(inst.f_value(x_probe)),
        "probe_gradx": rapdb.problem.grad_x_coupling(inst, z),
    }
    meta = {"instance": f"instances.factored_qcqp(**{FACTORED_SMALL})", "cases": {}}
    for key, case in {"mono": dict(nm=False, policy={"kind": "none"}, budget=200),
                      "nm": dict(nm=True, policy={"kind": "none"}, budget=200),
                      "nm_fixed200": dict(nm=True, policy={"kind": "fixed", "period": 200},
                                          budget=4000, eps=1e-6)}.items():
        out, wall = run_case(inst, case, set(range(1, 201)))
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = dict(case, wall_s=wall)
        print("factored", key, out["iterations"], out["converged"], round(wall, 2))
    save("factored_small", arrays, meta)


FACTORED_SMALL = dict(n=300, mq=4, rows=30, nnz_row=10, lin_rows=150, lin_nnz=5, seed=5, x0_scale=0.2)


def c1_fixtures():
    arr = instances.config_instance("C1")
    t0 = time.time()
    inst = ref_instance(arr)
    print("C1 instance", time.time() - t0)
    arrays = {"Q_checksum": np.array([float(np.sum(arr.Q[i])) for i in range(arr.m + 1)])}
    meta = {"instance": "instances.config_instance('C1')", "cases": {}}
    snaps = {1, 2, 3, 5, 10, 20, 50, 100, 150, 200}
    for key, case in {"mono": dict(nm=False, policy={"kind": "none"}, budget=200),
                      "nm": dict(nm=True, policy={"kind": "none"}, budget=200)}.items():
        out, wall = run_case(inst, case, snaps)
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = dict(case, wall_s=wall)
        print("C1", key, wall)
    save("c1_200", arrays, meta)


def scaled_fixtures(name, cfg_name, scale, cases, snaps=(1, 2, 5, 10, 20, 50, 100, 150, 200)):
    """200-iteration traces of the REAL reference on a BASELINE config
    (C4 at full size, C2 at reduced scale: the full C2 stack is 69 GB)."""
    arr = instances.config_instance(cfg_name, scale=scale)
    t0 = time.time()
    inst = ref_instance(arr)
    print(name, "instance", time.time() - t0, flush=True)
    arrays = {"Q_checksum": np.array([float(np.sum(arr.Q[i])) for i in range(arr.m + 1)])}
    meta = {"instance": f"instances.config_instance({cfg_name!r}, scale={scale!r})", "cases": {},
            "n": arr.n, "m": arr.m}
    for key, case in cases.items():
        out, wall = run_case(inst, case, set(snaps))
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = dict(case, wall_s=wall)
        print(name, key, wall, flush=True)
    save(name, arrays, meta)


def restart_option_fixtures():
    """Round 2: goldens for rows a6 (``warm_tau=True``, engine.py:111-113 via
    restarts.py:129/:153; mirrors pkg/tests/test_restarts.py:57-65) and a13
    (``criterion="paper51"`` with ``f_star``, diagnostics.py:254-258, and the
    ``subopt`` trace column, restarts.py:120).  Instances: the reference's own
    ``random_qcqp(20, 3, seed=3)`` (arrays in small_qcqp.npz), the analytic
    suite (arrays in analytic.npz) and C0 (regenerated from the seed)."""
    arrays, meta = {}, {"cases": {}}
    small = generate.random_qcqp(20, 3, seed=3)
    suite = {a.name: a for a in generate.analytic_suite()}
    c0 = ref_instance(instances.config_instance("C0"))

    # f* for small_qcqp / C0 from tight reference solves (recorded, not assumed)
    fstars = {}
    for key, inst in (("small", small), ("c0", c0)):
        out, wall = run_case(inst, dict(nm=False, policy={"kind": "none"}, budget=50000,
                                        eps=1e-10), {1})
        fstars[key] = float(out["metrics"][5])
        arrays[f"fstar/{key}"] = np.float64(fstars[key])
        meta["cases"][f"fstar/{key}"] = {"iterations": int(out["iterations"]),
                                         "converged": int(out["converged"]), "wall_s": wall}
        print("f*", key, fstars[key], out["iterations"], round(wall, 2), flush=True)

    cases = {
        # --- warm_tau (a6) ---
        "ball/warm_fixed30": ("ball", dict(nm=False, policy={"kind": "fixed", "period": 30},
                                           budget=61, warm_tau=True)),
        "ball/cold_fixed30": ("ball", dict(nm=False, policy={"kind": "fixed", "period": 30},
                                           budget=61, warm_tau=False)),
        "small/warm_nm_fixed40": ("small", dict(nm=True, policy={"kind": "fixed", "period": 40},
                                                budget=200, warm_tau=True)),
        "small/warm_mono_fixed40avg": ("small", dict(nm=False, policy={"kind": "fixed", "period": 40,
                                                                       "point": "average"},
                                                     budget=200, warm_tau=True)),
        "small/warm_xy_nm_fixed40": ("small", dict(mode="xy", nm=True,
                                                   policy={"kind": "fixed", "period": 40},
                                                   budget=200, warm_tau=True)),
        "small/warm_nm_ada": ("small", dict(nm=True, policy={"kind": "adaptive", "warmup": 50,
                                                             "check_period": 100},
                                            budget=1500, eps=1e-8, warm_tau=True)),
        "c0/warm_mono_fixed500": ("c0", dict(nm=False, policy={"kind": "fixed", "period": 500},
                                             budget=50000, eps=1e-6, warm_tau=True)),
        "c0/warm_mono_ada": ("c0", dict(nm=False, policy={"kind": "adaptive", "xi": 0.04, "q": 0.5,
                                                          "warmup": 50, "check_period": 200},
                                        budget=50000, eps=1e-6, warm_tau=True)),
        # --- paper51 + f_star, and the subopt column under "conic" (a13) ---
        "small/p51_nm_fixed100": ("small", dict(nm=True, policy={"kind": "fixed", "period": 100},
                                                budget=20000, eps=1e-6, criterion="paper51",
                                                f_star="small")),
        "small/conic_fstar_mono": ("small", dict(nm=False, policy={"kind": "none"},
                                                 budget=20000, eps=1e-7, f_star="small")),
        "small/p51_nofstar_mono": ("small", dict(nm=False, policy={"kind": "none"},
                                                 budget=20000, eps=1e-7, criterion="paper51")),
        "c0/p51_mono_fixed500": ("c0", dict(nm=False, policy={"kind": "fixed", "period": 500},
                                            budget=50000, eps=1e-6, criterion="paper51",
                                            f_star="c0")),
    }
    for name in ("ball", "box-lp", "eq-qp", "strongly-convex"):
        cases[f"{name}/p51_nm_fixed500"] = (name, dict(nm=True, policy={"kind": "fixed", "period": 500},
                                                       budget=5000, eps=1e-7, criterion="paper51",
                                                       f_star="analytic"))
    for key, (which, case) in cases.items():
        inst = small if which == "small" else c0 if which == "c0" else suite[which].instance
        run = dict(case)
        if run.get("f_star") == "analytic":
            run["f_star"] = float(suite[which].f_star)
        elif isinstance(run.get("f_star"), str):
            run["f_star"] = fstars[run["f_star"]]
        out, wall = run_case(inst, run, set(range(1, 201)))
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = dict(run, instance=which, wall_s=wall)
        print(key, "iterations", int(out["iterations"]), "conv", int(out["converged"]),
              round(wall, 2), flush=True)
    save("restart_opts", arrays, meta)


def c1_kkt_fixtures():
    """Round 2: the bench configuration end to end -- C1 yx monotone +
    FixedRestart(500) to conic KKT 1e-6 (restarts.py:111-170), plus mono +
    adaptive, by the real reference on the same seeded arrays."""
    arr = instances.config_instance("C1")
    t0 = time.time()
    inst = ref_instance(arr)
    print("C1 instance", time.time() - t0, flush=True)
    arrays = {"Q_checksum": np.array([float(np.sum(arr.Q[i])) for i in range(arr.m + 1)])}
    meta = {"instance": "instances.config_instance('C1')", "cases": {}}
    snaps = {1, 2, 5, 10, 50, 100, 200, 300, 400, 499, 500, 501, 502, 510, 550, 560, 570}
    for key, case in {"mono_fixed500": dict(nm=False, policy={"kind": "fixed", "period": 500},
                                            budget=3000, eps=1e-6),
                      "mono_ada": dict(nm=False, policy={"kind": "adaptive", "xi": 0.04, "q": 0.5,
                                                         "warmup": 50, "check_period": 200},
                                       budget=3000, eps=1e-6)}.items():
        out, wall = run_case(inst, case, snaps)
        for k, v in out.items():
            arrays[f"{key}/{k}"] = v
        meta["cases"][key] = dict(case, wall_s=wall)
        print("C1", key, int(out["iterations"]), int(out["converged"]), wall, flush=True)
        save("c1_kkt", arrays, meta)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1", action="store_true")
    ap.add_argument("--skip-small", action="store_true")
    ap.add_argument("--factored", action="store_true")
    ap.add_argument("--c4", action="store_true")
    ap.add_argument("--c2s", action="store_true")
    ap.add_argument("--kml", action="store_true")
    ap.add_argument("--restart-opts", action="store_true")
    ap.add_argument("--c1-kkt", action="store_true")
    a = ap.parse_args()
    if not a.skip_small:
        small_fixtures()
    if a.kml:
        kml_fixtures()
    if a.factored:
        factored_fixtures()
    if a.c1:
        c1_fixtures()
    if a.restart_opts:
        restart_option_fixtures()
    if a.c1_kkt:
        c1_kkt_fixtures()
    if a.c4:   # BASELINE C4 at full size (N = 4000, n = 4001): nm and mono, no restart in 200
        scaled_fixtures("c4_200", "C4", None,
                        {"nm": dict(nm=True, policy={"kind": "fixed", "period": 500}, budget=200),
                         "mono": dict(nm=False, policy={"kind": "fixed", "period": 500}, budget=200)})
    if a.c2s:  # BASELINE C2's generator at 1/4 scale (n = 1024, m = 128, rank 64)
        scaled_fixtures("c2s_200", "C2", 0.25,
                        {"nm": dict(nm=True, policy={"kind": "none"}, budget=200),
                         "mono": dict(nm=False, policy={"kind": "none"}, budget=200)})
