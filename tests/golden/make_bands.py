"""Perturbation bands of the reference's iteration counts (C0 policies).

The oracle (bit-identical to the reference, tests/test_oracle_pin.py) is rerun
with every Q_i @ x jittered by -1/0/+1 ulp (seeded), the perturbation SURVEY.md
section 7 hard part 4 uses.  Accept/reject decisions that the reference takes
at a margin below rounding noise then flip, and for non-monotone policies the
iteration count to KKT 1e-6 spreads widely.  A device result is judged against
this band: no arithmetic that is not bit-identical to numpy/OpenBLAS can do
better than the reference's own spread.

    python tests/golden/make_bands.py      # writes tests/golden/c0_bands.json
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import rapdb_oracle as O  # noqa: E402
from paper_2605_29291_b200 import instances  # noqa: E402


class Jitter:
    def __init__(self, M, rng):
        self.M, self.rng = M, rng

    def __matmul__(self, x):
        u = self.M @ x
        return u * (1.0 + 2.220446049250313e-16 * self.rng.choice([-1.0, 0.0, 1.0], size=u.shape))

    def toarray(self):
        return self.M

    @property
    def T(self):
        return self.M.T

    @property
    def shape(self):
        return self.M.shape


POLICIES = {
    "mono_none": (False, O.Policy("none")),
    "nm_fixed500": (True, O.Policy("fixed", period=500)),
    "mono_ada": (False, O.Policy("adaptive")),
    "nm_ada": (True, O.Policy("adaptive")),
}


def main(seeds=24):
    arr = instances.config_instance("C0")
    crit = dict(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
    out = {}
    for key, (nm, pol) in POLICIES.items():
        counts = []
        for seed in range(seeds + 1):
            P = O.Problem.from_arrays(arr)
            if seed > 0:
                rng = np.random.default_rng(seed)
                P.Q = [Jitter(M, rng) for M in P.Q]
            res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=nm), pol, budget=50000,
                                  criteria=crit)
            counts.append(int(res.iterations))
            print(key, seed, res.iterations, flush=True)
        out[key] = {"unperturbed": counts[0], "perturbed": counts[1:]}
    with open(os.path.join(HERE, "c0_bands.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
