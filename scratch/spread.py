import sys, numpy as np
sys.path.insert(0,'.')
from oracle import rapdb_oracle as O
from paper_2605_29291_b200 import instances
arr = instances.config_instance("C0")
class Jit:
    def __init__(self, M, rng): self.M, self.rng = M, rng
    def __matmul__(self, x):
        u = self.M @ x
        return u * (1.0 + 2.2e-16 * self.rng.choice([-1.0, 0.0, 1.0], size=u.shape))
    @property
    def T(self): return self.M.T
    @property
    def shape(self): return self.M.shape
crit = dict(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
pol = sys.argv[1]
for seed in range(int(sys.argv[2])):
    P = O.Problem.from_arrays(arr)
    if seed > 0:
        rng = np.random.default_rng(seed)
        P.Q = [Jit(M, rng) for M in P.Q]
    if pol == "nmfix": res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=True), O.Policy("fixed", period=500), budget=20000, criteria=crit)
    if pol == "monoada": res = O.run_restarted(P, O.Options(mode="yx", nonmonotone=False), O.Policy("adaptive"), budget=20000, criteria=crit)
    print(pol, seed, res.iterations, res.converged, flush=True)
