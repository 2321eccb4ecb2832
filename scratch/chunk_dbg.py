import os, sys, time, numpy as np, torch
sys.path.insert(0, '.')
os.environ["RAPDB_TILE_BYTES"] = sys.argv[1]
os.environ["RAPDB_STAGES"] = sys.argv[2]
import paper_2605_29291_b200 as R
from paper_2605_29291_b200 import instances
from oracle import rapdb_oracle as O
arr = instances.dense_qcqp(int(sys.argv[3]), 8, 10, seed=3)
inst = R.ProblemInstance.from_arrays(arr, validate=False)
ev = inst._evaluator()
x = np.random.default_rng(0).uniform(-1, 1, arr.n)
t = time.time()
u, g, ms = ev.ctx.probe_sweep(torch.from_numpy(x).cuda(), reps=3)
P = O.Problem.from_arrays(arr)
uu = u.cpu().numpy()
err = max(np.linalg.norm(uu[i] - arr.Q[i] @ x) / np.linalg.norm(arr.Q[i] @ x) for i in range(arr.m + 1))
print("tile", sys.argv[1], "stages", sys.argv[2], "n", arr.n, "ms", ms, "u err", err, "g err", np.max(np.abs(g.cpu().numpy()[1:] - P.g(x))), time.time() - t, flush=True)
