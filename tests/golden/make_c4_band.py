"""Where the reference's own C4 non-monotone run parts from itself under a
+-1-ulp jitter of every Q_i @ x (the perturbation of make_bands.py): the first
iteration whose accepted (tau_start, tau, evals) triple differs from the
unperturbed run.  The device's full-size C4 run (yx non-monotone +
FixedRestart(500)) stays bit-identical to the oracle for 782 iterations
(profiles/r02c_validate_long_c4nm.json); this shows that no arithmetic that is
not bit-identical to numpy/OpenBLAS is expected to do better.

    python tests/golden/make_c4_band.py [iterations] [seeds]   -> tests/golden/c4_band.json
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)
from oracle import rapdb_oracle as O  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402
from make_bands import Jitter  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    arr = instances.config_instance("C4")
    runs = []
    for seed in range(seeds + 1):
        P = O.Problem.from_arrays(arr)
        if seed > 0:
            rng = np.random.default_rng(seed)
            P.Q = [Jitter(M, rng) for M in P.Q]
        res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=True), O.Policy("fixed", period=500), budget=K)
        runs.append(np.array([[t.tau_start, t.tau, t.evals_iter] for t in res.trace]))
        print(seed, len(runs[-1]), int(runs[-1][:, 2].sum()), flush=True)
    base = runs[0]
    first = []
    for r in runs[1:]:
        k = min(len(r), len(base))
        same = np.all(r[:k] == base[:k], axis=1)
        first.append(int(np.argmin(same)) + 1 if not same.all() else None)
    out = {"config": "C4", "policy": "yx nonmonotone + FixedRestart(500)", "iterations": K,
           "first_step_difference_under_1ulp_jitter": first,
           "device_first_step_difference": 783}
    with open(os.path.join(HERE, "c4_band.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(out)


if __name__ == "__main__":
    main()
