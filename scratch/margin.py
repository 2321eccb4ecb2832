import sys, numpy as np
sys.path.insert(0,'.')
from oracle import rapdb_oracle as O
from paper_2605_29291_b200 import instances
arr = instances.config_instance("C0")
P = O.Problem.from_arrays(arr)
opt = O.Options(mode="yx", nonmonotone=True)
log = []
orig = O.Engine._trial_yx
def wrap(self, tau, sigma):
    out = orig(self, tau, sigma)
    z, gy, E, Dp, Dd, a, b = out
    slack = 1e-13 * (1.0 + abs(P.phi(self.x, self.v, self.lam)))
    rhs = -(self.o.delta / tau) * Dp - (self.o.delta / sigma) * Dd
    log.append((self.iters + 1, tau, E, rhs, slack, Dp))
    return out
O.Engine._trial_yx = wrap
res = O.run_restarted(P, opt, O.Policy("fixed", period=500), budget=910)
for r in log:
    if 905 <= r[0] <= 908:
        it, tau, E, rhs, slack, Dp = r
        print(it, f"tau={tau:.4e} E={E:.6e} rhs={rhs:.6e} slack={slack:.2e} margin={(rhs+slack-E):.3e} rel={(rhs+slack-E)/max(abs(E),abs(rhs)):.2e}")
