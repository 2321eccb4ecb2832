"""One-off full-size parity check of a BASELINE config against the CPU oracle
(too slow for the test suite): the first K accepted iterations of yx
monotone and non-monotone, step sizes bitwise, iterates to 1e-9.
python tools/validate_full.py C2 20 [mono|nm]  -> prints one JSON line"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from oracle import rapdb_oracle as O  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
only = sys.argv[3] if len(sys.argv) > 3 else None      # "mono" / "nm": one case only
t0 = time.time()
arr = instances.config_instance(name)
gen_s = time.time() - t0
inst = R.ProblemInstance.from_arrays(arr, validate=False)
P = O.Problem.from_arrays(arr)
out = {"config": name, "n": arr.n, "m": arr.m, "iterations": K, "generate_s": gen_s, "cases": {}}
for nm in (False, True):
    if only is not None and only != ("nm" if nm else "mono"):
        continue
    t0 = time.time()
    eng = O.Engine(P, O.Options(mode="yx", nonmonotone=nm), *O.initial_point(P))
    for _ in range(K):
        eng.step()
    cpu_s = time.time() - t0
    ref = np.array([[t.tau_start, t.tau, t.evals_iter] for t in eng.trace])
    t0 = time.time()
    dev = R.ApdbEngine(inst, R.SolverConfig(mode="yx", nonmonotone=nm), R.initial_iterate(inst))
    dev.run_block(K)
    gpu_s = time.time() - t0
    got = np.array([[t.tau_start, t.tau, t.evals_iter] for t in dev.trace])
    z = dev.last
    rx = float(np.linalg.norm(z.x - eng.x) / np.linalg.norm(eng.x))
    rl = float(np.linalg.norm(z.lam - eng.lam) / max(np.linalg.norm(eng.lam), 1e-300))
    out["cases"]["nm" if nm else "mono"] = {
        "steps_bitwise_equal": bool(np.array_equal(got, ref)), "rel_x": rx, "rel_lam": rl,
        "evals": int(ref[:, 2].sum()), "cpu_oracle_s": cpu_s, "device_s_incl_upload": gpu_s,
        "pass": bool(np.array_equal(got, ref) and rx <= 1e-9 and rl <= 1e-9)}
print(json.dumps(out))
