"""The reference's own rounding band for the END of the bench run (C1, yx
monotone + FixedRestart(500) to conic KKT 1e-6): the oracle (bit-identical to
the reference, tests/test_oracle_pin.py) rerun with every Q_i @ x jittered by
-1/0/+1 ulp (seeded; make_bands.py's perturbation).  The final KKT residual
(~7.5e-7) is formed by cancellation, so ulp-level differences along 570
iterations move it by parts in 1e6; a device result is judged against this
spread as well as the 1e-6 relative bar (tests/test_gpu_endtoend.py).

    python tests/golden/make_c1_band.py [seeds]   # writes tests/golden/c1_band.json
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)
from make_bands import Jitter  # noqa: E402
from oracle import rapdb_oracle as O  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402


def main(seeds=3):
    arr = instances.config_instance("C1")
    crit = dict(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
    runs = []
    for seed in range(seeds + 1):
        P = O.Problem.from_arrays(arr)
        if seed > 0:
            rng = np.random.default_rng(seed)
            P.Q = [Jitter(M, rng) for M in P.Q]
        res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=False), O.Policy("fixed", period=500),
                              budget=3000, criteria=crit)
        m = res.metrics
        runs.append({"seed": seed, "iterations": int(res.iterations), "converged": bool(res.converged),
                     "restarts": [int(e[1]) for e in res.restarts], "kkt": m.kkt_residual,
                     "infeas": m.infeas, "f": m.f_value})
        print(json.dumps(runs[-1]), flush=True)
    out = {"config": "C1 yx mono + FixedRestart(500), conic 1e-6", "runs": runs}
    for k in ("kkt", "infeas", "f"):
        v = np.array([r[k] for r in runs])
        out[f"{k}_rel_spread"] = float((v.max() - v.min()) / abs(runs[0][k]))
    with open(os.path.join(HERE, "c1_band.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
