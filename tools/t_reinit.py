"""Host-side setup costs per solve (bind, first reinit, C-call breakdown)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
import paper_2605_29291_b200 as R  # noqa: E402
from paper_2605_29291_b200 import instances, _capi  # noqa: E402

arr = instances.config_instance(sys.argv[1] if len(sys.argv) > 1 else "C1")
inst = R.ProblemInstance.from_arrays(arr, validate=False)
crit = R.TerminationCriteria(criterion="conic", eps_kkt=1e-6, eps_feas=1e-6)
cfg = R.SolverConfig(mode="yx", nonmonotone=False)
lib = _capi.load()
times = []


def wrap(name):
    f = getattr(lib, name)

    def g(*a):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f(*a)
        torch.cuda.synchronize()
        times.append((name.replace("rapdb_", ""), round((time.perf_counter() - t0) * 1e3, 2)))
        return r
    g.argtypes = f.argtypes
    setattr(lib, name, g)


for nm in ["rapdb_create", "rapdb_bind_dense_packed", "rapdb_set_params", "rapdb_workspace_bytes",
           "rapdb_bind_workspace", "rapdb_reinit", "rapdb_destroy"]:
    wrap(nm)
orig_empty = torch.empty
for pol in (R.AdaptiveRestart(), R.FixedRestart(500), R.AdaptiveRestart()):
    times.clear()
    t0 = time.perf_counter()
    R.run_restarted(inst, cfg, pol, criteria=crit)
    print(type(pol).__name__, round((time.perf_counter() - t0) * 1e3, 1), times)
